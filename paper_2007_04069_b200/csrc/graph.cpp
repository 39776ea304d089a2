// Graph ingest: compile the reference propagation rules into link classes,
// forced-replicated classes and class-level implication lists.
//
// Reference rule table: sharding.py:155-202 (compile), :267-302 (dot and
// reduce rules), :112-130 (the single-partition pin inside _set).
//
// Closure used by the device kernel (derivation in DESIGN.md §2): every rule
// is either an equality link between two slots or a "class X partitioned
// forces class Y replicated" implication, and nothing but a seed ever
// produces PARTITIONED.  So with link classes K:
//   P = classes of P seeds,
//   R = classes of R seeds  U  forced classes  U  Imp(P),
//   CONFLICT <=> P n R != {},  every slot takes its class's status.
#include <algorithm>
#include <cstring>
#include <numeric>
#include <unordered_set>

#include "engine.h"

namespace apb {
namespace {

struct DimView {
  const int64_t* p;
  int32_t n;
  int64_t operator[](int i) const { return p[i]; }
};

// ---- dim pairing (shape semantics of ir.py:119-196, restated) -------------

bool pair_broadcast(DimView src, DimView dst, std::vector<std::pair<int, int>>* pairs) {
  pairs->clear();
  int cursor = dst.n;
  for (int i = src.n - 1; i >= 0; --i) {
    --cursor;
    while (cursor >= 0 && dst[cursor] != src[i]) --cursor;
    if (cursor < 0) return false;
    pairs->push_back({i, cursor});
  }
  std::reverse(pairs->begin(), pairs->end());
  return true;
}

bool pair_reduce(DimView src, DimView dst, std::vector<std::pair<int, int>>* kept, std::vector<int>* reduced) {
  kept->clear();
  reduced->clear();
  int nxt = 0;
  for (int j = 0; j < dst.n; ++j) {
    while (nxt < src.n && src[nxt] != dst[j]) reduced->push_back(nxt++);
    if (nxt == src.n) return false;
    kept->push_back({nxt++, j});
  }
  while (nxt < src.n) reduced->push_back(nxt++);
  return true;
}

void pair_reshape(DimView src, DimView dst, std::vector<std::pair<int, int>>* aligned,
                  std::vector<int>* lone_src, std::vector<int>* lone_dst) {
  aligned->clear();
  lone_src->clear();
  lone_dst->clear();
  int a = 0, b = 0;
  // running products; extents of real graphs stay far below 2^63 but use
  // unsigned __int128 so a pathological graph cannot overflow silently
  unsigned __int128 off_a = 1, off_b = 1;
  while (a < src.n && b < dst.n) {
    if (off_a == off_b && src[a] == dst[b]) {
      aligned->push_back({a, b});
      off_a *= (unsigned __int128)src[a++];
      off_b *= (unsigned __int128)dst[b++];
    } else if (off_a * (unsigned __int128)src[a] <= off_b * (unsigned __int128)dst[b]) {
      lone_src->push_back(a);
      off_a *= (unsigned __int128)src[a++];
    } else {
      lone_dst->push_back(b);
      off_b *= (unsigned __int128)dst[b++];
    }
  }
  while (a < src.n) lone_src->push_back(a++);
  while (b < dst.n) lone_dst->push_back(b++);
}

struct UnionFind {
  std::vector<int64_t> parent;
  explicit UnionFind(int64_t n) : parent(n) { std::iota(parent.begin(), parent.end(), 0); }
  int64_t find(int64_t x) {
    while (parent[x] != x) {
      parent[x] = parent[parent[x]];
      x = parent[x];
    }
    return x;
  }
  void unite(int64_t a, int64_t b) {
    a = find(a);
    b = find(b);
    if (a == b) return;
    if (a < b) std::swap(a, b);
    parent[a] = b;  // keep the smaller slot as root
  }
};

}  // namespace

int build_graph(const ap_graph_desc* desc, GraphTables* g) {
  if (!desc || desc->num_instructions < 0) {
    set_error("ap_graph_create: null or negative-size descriptor");
    return AP_ERR_INVALID;
  }
  const int32_t n = desc->num_instructions;
  if (n > 0 && (!desc->opcode || !desc->rank || !desc->dims_offset || !desc->operand_offset ||
                !desc->gte_element)) {
    set_error("ap_graph_create: descriptor has null arrays");
    return AP_ERR_INVALID;
  }
  g->num_instr = n;
  g->slot_base.assign(desc->dims_offset, desc->dims_offset + n + 1);
  if (n == 0) g->slot_base.assign(1, 0);
  const int64_t S = g->slot_base[n];
  g->num_slots = S;
  g->slot_owner.assign(S, 0);
  for (int32_t p = 0; p < n; ++p) {
    if (desc->dims_offset[p + 1] - desc->dims_offset[p] != desc->rank[p]) {
      set_error("ap_graph_create: dims_offset does not match rank");
      return AP_ERR_INVALID;
    }
    for (int64_t s = g->slot_base[p]; s < g->slot_base[p + 1]; ++s) g->slot_owner[s] = p;
  }

  auto dims_of = [&](int32_t p) { return DimView{desc->dims + desc->dims_offset[p], desc->rank[p]}; };
  auto slot = [&](int32_t p, int d) { return g->slot_base[p] + d; };
  auto operand = [&](int32_t p, int k) { return desc->operands[desc->operand_offset[p] + k]; };

  struct Dot { int32_t a, b, c; };
  struct Red { int32_t a, out; std::vector<int> reduced; };
  std::vector<std::pair<int64_t, int64_t>> links;
  std::vector<Dot> dots;
  std::vector<Red> reds;
  std::vector<int64_t> forced;
  std::vector<int32_t>& prog = g->program;
  prog.clear();
  std::vector<std::pair<int, int>> pairs;
  std::vector<int> rest_a, rest_b;

  auto emit_link = [&](int64_t sa, int64_t sb, int32_t site) {
    links.push_back({sa, sb});
    prog.insert(prog.end(), {RULE_LINK, site, (int32_t)sa, (int32_t)sb});
  };

  for (int32_t p = 0; p < n; ++p) {
    const int32_t op = desc->opcode[p];
    const int32_t nops = desc->operand_offset[p + 1] - desc->operand_offset[p];
    switch (op) {
      case AP_OP_ADD: case AP_OP_SUBTRACT: case AP_OP_MULTIPLY: case AP_OP_DIVIDE:
      case AP_OP_EXP: case AP_OP_TANH:
        for (int k = 0; k < nops; ++k)
          for (int d = 0; d < desc->rank[p]; ++d) emit_link(slot(operand(p, k), d), slot(p, d), p);
        break;
      case AP_OP_DOT: {
        const int32_t a = operand(p, 0), b = operand(p, 1);
        if (desc->rank[a] != 2 || desc->rank[b] != 2 || desc->rank[p] != 2) {
          set_error("ap_graph_create: dot needs rank-2 operands and output");
          return AP_ERR_INVALID;
        }
        dots.push_back({a, b, p});
        links.push_back({slot(a, 0), slot(p, 0)});
        links.push_back({slot(b, 1), slot(p, 1)});
        links.push_back({slot(a, 1), slot(b, 0)});
        prog.insert(prog.end(), {RULE_DOT, p, a, b, p});
        break;
      }
      case AP_OP_TRANSPOSE: {
        const int32_t a = operand(p, 0);
        const int r = desc->rank[p];
        for (int d = 0; d < r; ++d) emit_link(slot(a, r - 1 - d), slot(p, d), p);
        break;
      }
      case AP_OP_RESHAPE: {
        const int32_t a = operand(p, 0);
        pair_reshape(dims_of(a), dims_of(p), &pairs, &rest_a, &rest_b);
        for (auto& pr : pairs) emit_link(slot(a, pr.first), slot(p, pr.second), p);
        for (int i : rest_a) forced.push_back(slot(a, i));
        for (int j : rest_b) forced.push_back(slot(p, j));
        break;
      }
      case AP_OP_BROADCAST: {
        const int32_t a = operand(p, 0);
        if (!pair_broadcast(dims_of(a), dims_of(p), &pairs)) {
          set_error("ap_graph_create: broadcast dims cannot be paired");
          return AP_ERR_INVALID;
        }
        std::vector<char> paired(desc->rank[p], 0);
        for (auto& pr : pairs) {
          emit_link(slot(a, pr.first), slot(p, pr.second), p);
          paired[pr.second] = 1;
        }
        for (int j = 0; j < desc->rank[p]; ++j)
          if (!paired[j]) forced.push_back(slot(p, j));
        break;
      }
      case AP_OP_REDUCE: {
        const int32_t a = operand(p, 0);
        if (!pair_reduce(dims_of(a), dims_of(p), &pairs, &rest_a)) {
          set_error("ap_graph_create: reduce dims cannot be paired");
          return AP_ERR_INVALID;
        }
        for (auto& pr : pairs) emit_link(slot(a, pr.first), slot(p, pr.second), p);
        if (!rest_a.empty() && desc->rank[p] > 0) {
          reds.push_back({a, p, rest_a});
          prog.insert(prog.end(), {RULE_REDUCE, p, a, p, (int32_t)rest_a.size()});
          prog.insert(prog.end(), rest_a.begin(), rest_a.end());
        }
        break;
      }
      case AP_OP_GET_TUPLE_ELEMENT: {
        const int32_t e = desc->gte_element[p];
        if (e < 0 || e >= n || desc->rank[e] != desc->rank[p]) {
          set_error("ap_graph_create: get-tuple-element without a matching tuple element");
          return AP_ERR_INVALID;
        }
        for (int d = 0; d < desc->rank[p]; ++d) emit_link(slot(e, d), slot(p, d), p);
        break;
      }
      case AP_OP_PARAMETER: case AP_OP_CONSTANT: case AP_OP_TUPLE:
        break;
      default:
        set_error("ap_graph_create: unknown opcode code");
        return AP_ERR_INVALID;
    }
  }
  if (S > INT32_MAX) {
    set_error("ap_graph_create: more than 2^31 slots");
    return AP_ERR_UNSUPPORTED;
  }
  g->num_links = (int32_t)links.size();

  // link classes, numbered by first slot in slot order
  UnionFind uf(S);
  for (auto& l : links) uf.unite(l.first, l.second);
  std::vector<int32_t> root_class(S, -1);
  g->class_of_slot.assign(S, 0);
  int32_t C = 0;
  for (int64_t s = 0; s < S; ++s) {
    const int64_t r = uf.find(s);
    if (root_class[r] < 0) root_class[r] = C++;
    g->class_of_slot[s] = root_class[r];
  }
  g->num_classes = C;
  auto cls = [&](int64_t s) { return g->class_of_slot[s]; };

  g->slot_forced.assign(S, 0);
  g->class_forced.assign(C, 0);
  g->forced_words.assign((size_t)(C + 31) / 32, 0u);
  g->forced_list.clear();
  for (int64_t s : forced) {
    g->forced_list.push_back((int32_t)s);
    g->slot_forced[s] = 1;
    g->class_forced[cls(s)] = 1;
    g->forced_words[(size_t)cls(s) >> 5] |= 1u << (cls(s) & 31);
  }

  // implication edges: P on class x forces R on class y
  std::vector<std::vector<int32_t>> imp(C);
  auto add_imp = [&](int64_t from_slot, int64_t to_slot) { imp[cls(from_slot)].push_back(cls(to_slot)); };
  for (int32_t p = 0; p < n; ++p) {  // single-partition pin (sharding.py:120-127)
    const int r = desc->rank[p];
    for (int d = 0; d < r; ++d)
      for (int e = 0; e < r; ++e)
        if (d != e) add_imp(slot(p, d), slot(p, e));
  }
  for (auto& t : dots) {  // dot cross rules (sharding.py:279-287)
    for (int k = 0; k < 2; ++k) {
      add_imp(slot(t.a, 0), slot(t.b, k));  // row split of A / C replicates B
      add_imp(slot(t.b, 1), slot(t.a, k));  // column split of B / C replicates A
      add_imp(slot(t.a, 1), slot(t.c, k));  // contracting split replicates C
    }
  }
  for (auto& r : reds) {  // reduce rules (sharding.py:296-301)
    const int ro = desc->rank[r.out];
    for (int rd : r.reduced)
      for (int j = 0; j < ro; ++j) {
        add_imp(slot(r.a, rd), slot(r.out, j));
        add_imp(slot(r.out, j), slot(r.a, rd));
      }
  }
  g->imp_offset.assign(C + 1, 0);
  g->imp_target.clear();
  for (int32_t c = 0; c < C; ++c) {
    auto& v = imp[c];
    std::sort(v.begin(), v.end());
    v.erase(std::unique(v.begin(), v.end()), v.end());
    for (int32_t t : v) g->imp_target.push_back(t);
    g->imp_offset[c + 1] = (int32_t)g->imp_target.size();
  }
  build_fast_graph(g);
  return AP_OK;
}

// Device tables are uploaded on first use so the host compile (and its
// export for tests) works on machines without a GPU.
int ensure_graph_on_device(GraphTables* g) {
  int cur = 0;
  AP_CUDA_CHECK(cudaGetDevice(&cur));
  if (g->uploaded) {
    if (cur != g->device) {
      set_error("graph handle used on a different device than the one it was uploaded to");
      return AP_ERR_INVALID;
    }
    return AP_OK;
  }
  g->device = cur;
  int rc;
  if ((rc = g->d_slot_class.upload(g->class_of_slot)) != AP_OK) return rc;
  if ((rc = g->d_forced_words.upload(g->forced_words)) != AP_OK) return rc;
  if ((rc = g->d_imp_offset.upload(g->imp_offset)) != AP_OK) return rc;
  if ((rc = g->d_imp_target.upload(g->imp_target)) != AP_OK) return rc;
  if ((rc = g->d_program.upload(g->program)) != AP_OK) return rc;
  if ((rc = g->d_forced_list.upload(g->forced_list)) != AP_OK) return rc;
  if ((rc = g->d_slot_base.upload(g->slot_base)) != AP_OK) return rc;
  if ((rc = g->d_slot_owner.upload(g->slot_owner)) != AP_OK) return rc;
  if (g->fast) {
    if ((rc = g->d_slot_desc.upload(g->slot_desc)) != AP_OK) return rc;
    if ((rc = g->d_slot_desc_t.upload(g->slot_desc_t)) != AP_OK) return rc;
    if ((rc = g->d_slot_cls8.upload(g->slot_cls8)) != AP_OK) return rc;
    if ((rc = g->d_imp_bits.upload(g->imp_bits)) != AP_OK) return rc;
    if ((rc = g->d_forced_bits.upload(g->forced_bits)) != AP_OK) return rc;
  }
  g->uploaded = true;
  return AP_OK;
}

int ensure_decision_on_device(DecisionTables* d) {
  if (d->uploaded) return AP_OK;
  int rc;
  if ((rc = d->d_dec_class.upload(d->dec_class)) != AP_OK) return rc;
  if ((rc = d->d_dec_flags.upload(d->dec_flags)) != AP_OK) return rc;
  if ((rc = d->d_first_same.upload(d->first_same)) != AP_OK) return rc;
  if ((rc = d->d_slots.upload(d->slots)) != AP_OK) return rc;
  if (d->fast) {
    if ((rc = d->d_dec_desc.upload(d->dec_desc)) != AP_OK) return rc;
    if ((rc = d->d_dec_masks.upload(d->dec_masks)) != AP_OK) return rc;
    if ((rc = d->d_dec_cls8.upload(d->dec_cls8)) != AP_OK) return rc;
    if ((rc = d->d_class_ncand.upload(d->class_ncand)) != AP_OK) return rc;
    if ((rc = d->d_ncand_planes.upload(d->ncand_planes)) != AP_OK) return rc;
  }
  d->uploaded = true;
  return AP_OK;
}

int build_decision(const GraphTables* g, const int64_t* slots, const uint8_t* is_cand, int32_t n,
                   DecisionTables* d) {
  if (n < 0 || (n > 0 && (!slots || !is_cand))) {
    set_error("ap_decision_create: bad arguments");
    return AP_ERR_INVALID;
  }
  d->graph = g;
  d->n = n;
  d->slots.assign(slots, slots + n);
  d->dec_class.resize(n);
  d->dec_flags.resize(n);
  d->first_same.resize(n);
  for (int32_t i = 0; i < n; ++i) {
    const int64_t s = slots[i];
    if (s < 0 || s >= g->num_slots || (i > 0 && s <= slots[i - 1])) {
      set_error("ap_decision_create: slots must be valid and strictly increasing");
      return AP_ERR_INVALID;
    }
    d->dec_class[i] = g->class_of_slot[s];
    d->dec_flags[i] = (uint8_t)((is_cand[i] ? 1 : 0) | (g->slot_forced[s] ? 2 : 0));
    const bool same = i > 0 && g->slot_owner[slots[i - 1]] == g->slot_owner[s];
    d->first_same[i] = same ? d->first_same[i - 1] : i;
  }
  build_fast_decision(g, d);
  return AP_OK;
}

}  // namespace apb
