/*
 * ap_oracle.c — CPU ORACLE (test infrastructure only).
 *
 * A plain-C restatement of the reference planner's propagation algorithm,
 * following its control flow step for step so that it reproduces not only
 * the fixed point but also the CONFLICT snapshot and conflict site:
 *
 *   rule compile      reference pkg/src/autoplan/sharding.py:155-202
 *   _set / _link      sharding.py:112-142
 *   run               sharding.py:210-248 (forced R, sorted seeds, sweep)
 *   _fixed_point      sharding.py:250-265
 *   _apply_dot        sharding.py:267-288
 *   _apply_reduce     sharding.py:290-302
 *   dim pairing       ir.py:119-196
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load this library; the product path never does.  It is pinned against
 * golden vectors generated from the reference itself (tests/golden/).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

enum { OP_PARAMETER = 0, OP_CONSTANT, OP_ADD, OP_SUBTRACT, OP_MULTIPLY, OP_DIVIDE, OP_EXP, OP_TANH, OP_DOT,
       OP_RESHAPE, OP_TRANSPOSE, OP_BROADCAST, OP_REDUCE, OP_TUPLE, OP_GTE };

typedef struct {
  int kind; /* 0 links, 1 dot, 2 reduce */
  int site;
  int nlinks;
  int64_t* links; /* 2*nlinks slots */
  int a, b;       /* dot operands / reduce operand */
  int nred;
  int* red;
} plan_t;

typedef struct {
  int n;
  const int32_t* rank;
  const int64_t* doff;
  const int64_t* dims;
  int nplans;
  plan_t* plans;
  int64_t nforced;
  int64_t* forced;
} orc_graph;

static int conflict_site;

/* sharding.py:112-130 */
static int o_set(int8_t* st, const orc_graph* g, const int32_t* owner, int64_t s, int v, int site) {
  int cur = st[s];
  if (cur == v) return 0;
  if (cur != -1) { conflict_site = site; return -1; }
  if (v == 1) {
    int o = owner[s];
    for (int64_t k = g->doff[o]; k < g->doff[o + 1]; ++k)
      if (st[k] == 1) { conflict_site = site; return -1; }
    st[s] = 1;
    for (int64_t k = g->doff[o]; k < g->doff[o + 1]; ++k)
      if (st[k] == -1) st[k] = 0;
  } else {
    st[s] = (int8_t)v;
  }
  return 1;
}

/* sharding.py:133-142 */
static int o_link(int8_t* st, const orc_graph* g, const int32_t* owner, int64_t a, int64_t b, int site) {
  int va = st[a], vb = st[b];
  if (va == vb) return 0;
  if (va == -1) return o_set(st, g, owner, a, vb, site);
  if (vb == -1) return o_set(st, g, owner, b, va, site);
  conflict_site = site;
  return -1;
}

/* ir.py:119-138 (returns number of pairs or -1) */
static int pair_bcast(const int64_t* in, int ni, const int64_t* out, int no, int* pi, int* po) {
  int j = no - 1, k = 0;
  for (int i = ni - 1; i >= 0; --i) {
    while (j >= 0 && out[j] != in[i]) --j;
    if (j < 0) return -1;
    pi[k] = i; po[k] = j; ++k; --j;
  }
  for (int x = 0; x < k / 2; ++x) {
    int t = pi[x]; pi[x] = pi[k - 1 - x]; pi[k - 1 - x] = t;
    t = po[x]; po[x] = po[k - 1 - x]; po[k - 1 - x] = t;
  }
  return k;
}

/* ir.py:141-162 */
static int pair_red(const int64_t* in, int ni, const int64_t* out, int no, int* pi, int* po, int* red, int* nred) {
  int i = 0, k = 0;
  *nred = 0;
  for (int j = 0; j < no; ++j) {
    while (i < ni && in[i] != out[j]) red[(*nred)++] = i++;
    if (i >= ni) return -1;
    pi[k] = i; po[k] = j; ++k; ++i;
  }
  while (i < ni) red[(*nred)++] = i++;
  return k;
}

/* ir.py:165-196 */
static int pair_reshape(const int64_t* in, int ni, const int64_t* out, int no, int* pi, int* po, int* ui, int* nui,
                        int* uo, int* nuo) {
  int i = 0, j = 0, k = 0;
  long double pin = 1, pout = 1; /* exact for the extents used in tests */
  *nui = *nuo = 0;
  while (i < ni && j < no) {
    if (pin == pout && in[i] == out[j]) {
      pi[k] = i; po[k] = j; ++k;
      pin *= in[i]; pout *= out[j]; ++i; ++j;
    } else if (pin * in[i] <= pout * out[j]) {
      ui[(*nui)++] = i; pin *= in[i]; ++i;
    } else {
      uo[(*nuo)++] = j; pout *= out[j]; ++j;
    }
  }
  while (i < ni) ui[(*nui)++] = i++;
  while (j < no) uo[(*nuo)++] = j++;
  return k;
}

#define MAXR 64

/* sharding.py:155-202 */
static int compile(orc_graph* g, const int32_t* opcode, const int32_t* ooff, const int32_t* ops, const int32_t* gte) {
  int n = g->n;
  g->plans = (plan_t*)calloc((size_t)2 * n + 1, sizeof(plan_t));
  g->forced = (int64_t*)malloc(sizeof(int64_t) * ((size_t)g->doff[n] + 1));
  g->nplans = 0;
  g->nforced = 0;
  int pi[MAXR], po[MAXR], ua[MAXR], ub[MAXR], red[MAXR];
  for (int p = 0; p < n; ++p) {
    int op = opcode[p], r = g->rank[p];
    if (r > MAXR) return -1;
    plan_t* pl = &g->plans[g->nplans];
    pl->site = p;
    const int64_t* od = g->dims + g->doff[p];
    if (op == OP_ADD || op == OP_SUBTRACT || op == OP_MULTIPLY || op == OP_DIVIDE || op == OP_EXP || op == OP_TANH) {
      int nops = ooff[p + 1] - ooff[p];
      pl->kind = 0;
      pl->links = (int64_t*)malloc(sizeof(int64_t) * 2 * (size_t)(nops * r + 1));
      for (int k = 0; k < nops; ++k)
        for (int d = 0; d < r; ++d) {
          pl->links[2 * pl->nlinks] = g->doff[ops[ooff[p] + k]] + d;
          pl->links[2 * pl->nlinks + 1] = g->doff[p] + d;
          pl->nlinks++;
        }
      g->nplans++;
    } else if (op == OP_DOT) {
      pl->kind = 1;
      pl->a = ops[ooff[p]];
      pl->b = ops[ooff[p] + 1];
      g->nplans++;
    } else if (op == OP_TRANSPOSE) {
      int a = ops[ooff[p]];
      pl->kind = 0;
      pl->links = (int64_t*)malloc(sizeof(int64_t) * 2 * (size_t)(r + 1));
      for (int d = 0; d < r; ++d) {
        pl->links[2 * d] = g->doff[a] + (r - 1 - d);
        pl->links[2 * d + 1] = g->doff[p] + d;
      }
      pl->nlinks = r;
      g->nplans++;
    } else if (op == OP_RESHAPE) {
      int a = ops[ooff[p]], nui, nuo;
      int k = pair_reshape(g->dims + g->doff[a], g->rank[a], od, r, pi, po, ua, &nui, ub, &nuo);
      pl->kind = 0;
      pl->links = (int64_t*)malloc(sizeof(int64_t) * 2 * (size_t)(k + 1));
      for (int x = 0; x < k; ++x) {
        pl->links[2 * x] = g->doff[a] + pi[x];
        pl->links[2 * x + 1] = g->doff[p] + po[x];
      }
      pl->nlinks = k;
      g->nplans++;
      for (int x = 0; x < nui; ++x) g->forced[g->nforced++] = g->doff[a] + ua[x];
      for (int x = 0; x < nuo; ++x) g->forced[g->nforced++] = g->doff[p] + ub[x];
    } else if (op == OP_BROADCAST) {
      int a = ops[ooff[p]];
      int k = pair_bcast(g->dims + g->doff[a], g->rank[a], od, r, pi, po);
      if (k < 0) return -2;
      pl->kind = 0;
      pl->links = (int64_t*)malloc(sizeof(int64_t) * 2 * (size_t)(k + 1));
      int paired[MAXR];
      memset(paired, 0, sizeof(paired));
      for (int x = 0; x < k; ++x) {
        pl->links[2 * x] = g->doff[a] + pi[x];
        pl->links[2 * x + 1] = g->doff[p] + po[x];
        paired[po[x]] = 1;
      }
      pl->nlinks = k;
      g->nplans++;
      for (int j = 0; j < r; ++j)
        if (!paired[j]) g->forced[g->nforced++] = g->doff[p] + j;
    } else if (op == OP_REDUCE) {
      int a = ops[ooff[p]], nred;
      int k = pair_red(g->dims + g->doff[a], g->rank[a], od, r, pi, po, red, &nred);
      if (k < 0) return -3;
      if (k > 0) {
        pl->kind = 0;
        pl->links = (int64_t*)malloc(sizeof(int64_t) * 2 * (size_t)k);
        for (int x = 0; x < k; ++x) {
          pl->links[2 * x] = g->doff[a] + pi[x];
          pl->links[2 * x + 1] = g->doff[p] + po[x];
        }
        pl->nlinks = k;
        g->nplans++;
      }
      if (nred > 0 && r > 0) {
        plan_t* q = &g->plans[g->nplans++];
        q->kind = 2;
        q->site = p;
        q->a = a;
        q->nred = nred;
        q->red = (int*)malloc(sizeof(int) * (size_t)nred);
        memcpy(q->red, red, sizeof(int) * (size_t)nred);
      }
    } else if (op == OP_GTE) {
      int e = gte[p];
      pl->kind = 0;
      pl->links = (int64_t*)malloc(sizeof(int64_t) * 2 * (size_t)(r + 1));
      for (int d = 0; d < r; ++d) {
        pl->links[2 * d] = g->doff[e] + d;
        pl->links[2 * d + 1] = g->doff[p] + d;
      }
      pl->nlinks = r;
      g->nplans++;
    }
  }
  return 0;
}

static void release(orc_graph* g) {
  for (int i = 0; i < g->nplans; ++i) {
    free(g->plans[i].links);
    free(g->plans[i].red);
  }
  free(g->plans);
  free(g->forced);
}

#define CHK(x)            \
  do {                    \
    int _r = (x);         \
    if (_r < 0) return -1; \
    ch |= _r;             \
  } while (0)

/* sharding.py:267-288 */
static int apply_dot(int8_t* st, const orc_graph* g, const int32_t* own, int a, int b, int c) {
  int ch = 0;
  int64_t A = g->doff[a], B = g->doff[b], Cc = g->doff[c];
  CHK(o_link(st, g, own, A + 0, Cc + 0, c));
  CHK(o_link(st, g, own, B + 1, Cc + 1, c));
  CHK(o_link(st, g, own, A + 1, B + 0, c));
  if (st[A] == 1 || st[Cc] == 1) { CHK(o_set(st, g, own, B, 0, c)); CHK(o_set(st, g, own, B + 1, 0, c)); }
  if (st[B + 1] == 1 || st[Cc + 1] == 1) { CHK(o_set(st, g, own, A, 0, c)); CHK(o_set(st, g, own, A + 1, 0, c)); }
  if (st[A + 1] == 1 || st[B] == 1) { CHK(o_set(st, g, own, Cc, 0, c)); CHK(o_set(st, g, own, Cc + 1, 0, c)); }
  return ch;
}

/* sharding.py:290-302 */
static int apply_reduce(int8_t* st, const orc_graph* g, const int32_t* own, int a, const int* red, int nred, int out) {
  int ch = 0, anyp = 0;
  for (int k = 0; k < nred; ++k) anyp |= st[g->doff[a] + red[k]] == 1;
  if (anyp)
    for (int64_t s = g->doff[out]; s < g->doff[out + 1]; ++s) CHK(o_set(st, g, own, s, 0, out));
  int outp = 0;
  for (int64_t s = g->doff[out]; s < g->doff[out + 1]; ++s) outp |= st[s] == 1;
  if (outp)
    for (int k = 0; k < nred; ++k) CHK(o_set(st, g, own, g->doff[a] + red[k], 0, out));
  return ch;
}

/*
 * Propagate `batch` seed rows.  Seeds are over `nseed` slots (seed_slots,
 * strictly increasing = the reference's sorted (id, dim) order); values
 * -1 none, 0 R, 1 P, 2 UNDECIDED.  init_state (nullable, [S]) replaces the
 * all-UNDECIDED start (rule_for semantics, sharding.py:336-339).
 * Writes state_out [batch, S], outcome [batch] (0 complete, 1 incomplete,
 * 2 conflict, judged on cand_slots), site [batch] (position or -1).
 * Returns 0, or <0 on a malformed graph, or -9 if the sweep cap is hit.
 */
int orc_propagate(int n, const int32_t* opcode, const int32_t* rank, const int64_t* doff, const int64_t* dims,
                  const int32_t* ooff, const int32_t* ops, const int32_t* gte, int nseed, const int64_t* seed_slots,
                  const int8_t* seeds, int64_t batch, int ncand, const int64_t* cand_slots, const int8_t* init_state,
                  int8_t* state_out, int32_t* outcome, int32_t* site) {
  orc_graph g;
  memset(&g, 0, sizeof(g));
  g.n = n;
  g.rank = rank;
  g.doff = doff;
  g.dims = dims;
  int rc = compile(&g, opcode, ooff, ops, gte);
  if (rc < 0) { release(&g); return rc; }
  int64_t S = doff[n];
  int32_t* owner = (int32_t*)malloc(sizeof(int32_t) * (size_t)(S + 1));
  for (int p = 0; p < n; ++p)
    for (int64_t s = doff[p]; s < doff[p + 1]; ++s) owner[s] = p;
  int max_rank = 0;
  for (int p = 0; p < n; ++p) if (rank[p] > max_rank) max_rank = rank[p];
  int64_t cap = (int64_t)n * (max_rank > 1 ? max_rank : 1) + 2;
  if (cap < 2) cap = 2;
  for (int64_t b = 0; b < batch; ++b) {
    int8_t* st = state_out + b * S;
    const int8_t* sr = seeds + b * nseed;
    if (init_state) memcpy(st, init_state, (size_t)S);
    else memset(st, -1, (size_t)S);
    conflict_site = -1;
    int conflict = 0;
    for (int64_t i = 0; i < g.nforced; ++i)
      if (o_set(st, &g, owner, g.forced[i], 0, owner[g.forced[i]]) < 0) { conflict = 1; break; }
    for (int j = 0; j < nseed && !conflict; ++j) {
      if (sr[j] == -1) continue;
      int64_t s = seed_slots[j];
      if (o_set(st, &g, owner, s, sr[j] == 2 ? -1 : sr[j], owner[s]) < 0) conflict = 1;
    }
    int fixed = conflict;
    for (int64_t it = 0; it < cap && !fixed; ++it) {
      int ch = 0, bad = 0;
      for (int q = 0; q < g.nplans && !bad; ++q) {
        plan_t* pl = &g.plans[q];
        int r;
        if (pl->kind == 0) {
          for (int k = 0; k < pl->nlinks && !bad; ++k) {
            r = o_link(st, &g, owner, pl->links[2 * k], pl->links[2 * k + 1], pl->site);
            if (r < 0) bad = 1; else ch |= r;
          }
        } else if (pl->kind == 1) {
          r = apply_dot(st, &g, owner, pl->a, pl->b, pl->site);
          if (r < 0) bad = 1; else ch |= r;
        } else {
          r = apply_reduce(st, &g, owner, pl->a, pl->red, pl->nred, pl->site);
          if (r < 0) bad = 1; else ch |= r;
        }
      }
      if (bad) { conflict = 1; fixed = 1; }
      else if (!ch) fixed = 1;
    }
    if (!fixed) { free(owner); release(&g); return -9; }
    site[b] = conflict ? conflict_site : -1;
    if (conflict) {
      outcome[b] = 2;
    } else {
      int complete = 1;
      for (int j = 0; j < ncand; ++j) if (st[cand_slots[j]] == -1) complete = 0;
      outcome[b] = complete ? 0 : 1;
    }
  }
  free(owner);
  release(&g);
  return 0;
}
