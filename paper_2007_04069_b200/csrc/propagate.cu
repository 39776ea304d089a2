// K1 — batched sharding propagation on sm_100a.
//
// Replaces PropagationEngine.run (reference sharding.py:210-248) for a batch
// of seed vectors.  One warp owns one plan at a time (persistent grid,
// warp-strided over the batch).  Per plan:
//   1. seed pass      lanes stride the decision positions; a P (R) seed marks
//                     its link class in the warp's P (R) flag row (benign
//                     same-value byte stores, no atomics);
//   2. implications   lanes stride the classes; every P class marks its
//                     implication targets R;
//   3. class pass     status per class (P wins), conflict = any(P and R),
//                     warp vote;
//   4. candidates     per-position status, decided / newly counts (warp
//                     reductions), optional per-position output;
//   5. slots          16 slots per lane-iteration: two 16-byte class-id
//                     loads, 16 table lookups, one 16-byte store.
// Graph tables (slot->class, implication CSR, forced bitset) are staged in
// shared memory once per CTA when they fit, else read through L1/L2; the
// per-plan class flags are P / R bitsets (shared memory, or global memory for
// very wide graphs), so any class count is supported.
#include <algorithm>
#include <cstdlib>

#include "engine.h"

namespace apb {
namespace {

constexpr int kWarps = 8;
constexpr int kThreads = kWarps * 32;
constexpr unsigned kFull = 0xffffffffu;

struct PropParams {
  const int32_t* slot_class;
  const uint32_t* forced_words;  // [Cw] forced-replicated class bitset
  const int32_t* imp_offset;
  const int32_t* imp_target;
  const int32_t* dec_class;
  const uint8_t* dec_flags;
  const int32_t* first_same;
  int64_t S;
  int32_t C, Cw, D, T, ncand;  // Cw = bitset words per row (multiple of 4)
  const int8_t* seeds;
  int64_t seed_stride, batch;
  int8_t* slots_out;
  int64_t slots_stride;
  int8_t* cand_out;
  int64_t cand_stride;
  uint8_t* outcome;
  int32_t* counts;
  int stage_tables;        // copy tables to shared memory
  uint32_t* gscratch;      // per-warp P/R bitsets in global memory (nullptr: shared)
  int64_t warp_stride;     // bytes of shared scratch per warp
  // byte offsets of the staged tables inside dynamic shared memory
  int off_slot_class, off_dec_class, off_dec_flags, off_forced, off_imp_off, off_imp_tgt, off_first_same,
      off_scratch;
};

__host__ __device__ inline int64_t align16(int64_t x) { return (x + 15) & ~int64_t(15); }

__device__ inline void copy_to_smem(uint8_t* dst, const void* src, int64_t bytes) {
  const uint8_t* s = reinterpret_cast<const uint8_t*>(src);
  for (int64_t i = threadIdx.x; i < bytes; i += blockDim.x) dst[i] = s[i];
}

// status of class c from the plan's P / R bitsets and the forced bitset
__device__ __forceinline__ int class_status(const uint32_t* P, const uint32_t* R, const uint32_t* F, int32_t c) {
  const int w = c >> 5;
  const uint32_t m = 1u << (c & 31);
  return (P[w] & m) ? 1 : (((R[w] | F[w]) & m) ? 0 : -1);
}

// Generic K1 for any graph: P / R class flags are per-warp bitsets (C/4 bytes
// per plan) in shared memory, or in global memory when even that does not
// fit; class ids are 32-bit.
// kTable: also materialise a per-warp byte status table (C bytes) after the
// class pass, so candidate / slot lookups are one byte load (graphs whose
// per-warp scratch still fits in shared memory)
template <bool kVecSlots, bool kTable>
__global__ void __launch_bounds__(kThreads) propagate_kernel(PropParams p) {
  pdl_entry();
  extern __shared__ __align__(16) uint8_t smem[];
  const int32_t* slot_class = p.slot_class;
  const int32_t* dec_class = p.dec_class;
  const uint8_t* dec_flags = p.dec_flags;
  const uint32_t* F = p.forced_words;
  const int32_t* imp_offset = p.imp_offset;
  const int32_t* imp_target = p.imp_target;
  const int32_t* first_same = p.first_same;
  if (p.stage_tables) {
    copy_to_smem(smem + p.off_slot_class, p.slot_class, p.S * 4);
    copy_to_smem(smem + p.off_dec_class, p.dec_class, (int64_t)p.D * 4);
    copy_to_smem(smem + p.off_dec_flags, p.dec_flags, p.D);
    copy_to_smem(smem + p.off_forced, p.forced_words, (int64_t)p.Cw * 4);
    copy_to_smem(smem + p.off_imp_off, p.imp_offset, (int64_t)(p.C + 1) * 4);
    copy_to_smem(smem + p.off_imp_tgt, p.imp_target, (int64_t)p.T * 4);
    copy_to_smem(smem + p.off_first_same, p.first_same, (int64_t)p.D * 4);
    __syncthreads();
    slot_class = reinterpret_cast<const int32_t*>(smem + p.off_slot_class);
    dec_class = reinterpret_cast<const int32_t*>(smem + p.off_dec_class);
    dec_flags = smem + p.off_dec_flags;
    F = reinterpret_cast<const uint32_t*>(smem + p.off_forced);
    imp_offset = reinterpret_cast<const int32_t*>(smem + p.off_imp_off);
    imp_target = reinterpret_cast<const int32_t*>(smem + p.off_imp_tgt);
    first_same = reinterpret_cast<const int32_t*>(smem + p.off_first_same);
  }
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int64_t gwarp = (int64_t)blockIdx.x * kWarps + warp;
  uint32_t* P = p.gscratch ? p.gscratch + gwarp * 2 * p.Cw
                           : reinterpret_cast<uint32_t*>(smem + p.off_scratch + (int64_t)warp * p.warp_stride);
  uint32_t* R = P + p.Cw;
  int8_t* table = reinterpret_cast<int8_t*>(R + p.Cw);  // kTable only: C bytes after the bitsets
  auto status = [&](int32_t c) -> int { return kTable ? (int)table[c] : class_status(P, R, F, c); };

  const int64_t nwarps = (int64_t)gridDim.x * kWarps;
  for (int64_t b = gwarp; b < p.batch; b += nwarps) {
    // 0. clear the bitsets (Cw is a multiple of 4)
    for (int i = lane; i < (2 * p.Cw) / 4; i += 32) reinterpret_cast<uint4*>(P)[i] = make_uint4(0, 0, 0, 0);
    __syncwarp();

    // 1. seeds
    const int8_t* srow = p.seeds + b * p.seed_stride;
    bool conflict = false;
    for (int j = lane; j < p.D; j += 32) {
      const int v = srow[j];
      if (v == 1 || v == 0) {
        const int32_t c = dec_class[j];
        atomicOr(v == 1 ? &P[c >> 5] : &R[c >> 5], 1u << (c & 31));
      } else if (v == 2) {
        // an UNDECIDED seed conflicts iff its slot is already decided when it
        // is applied: forced replicated, or pinned by an earlier P seed on the
        // same tensor (sharding.py:116-118, 219-229)
        if (dec_flags[j] & 2) conflict = true;
        for (int k = first_same[j]; k < j; ++k)
          if (srow[k] == 1) conflict = true;
      }
    }
    __syncwarp();

    // 2. implications of partitioned classes (set bits of P)
    for (int w = lane; w < p.Cw; w += 32) {
      uint32_t bits = P[w];
      while (bits) {
        const int32_t c = 32 * w + __ffs(bits) - 1;
        bits &= bits - 1;
        const int e = imp_offset[c + 1];
        for (int k = imp_offset[c]; k < e; ++k) {
          const int32_t t = imp_target[k];
          atomicOr(&R[t >> 5], 1u << (t & 31));
        }
      }
    }
    __syncwarp();

    // 3. conflict: a class both partitioned and replicated (or forced)
    for (int w = lane; w < p.Cw; w += 32) conflict |= (P[w] & (R[w] | F[w])) != 0;
    conflict = __any_sync(kFull, conflict);
    if (kTable) {
      for (int c = lane; c < p.C; c += 32) table[c] = (int8_t)class_status(P, R, F, c);
      __syncwarp();
    }

    // 4. candidate positions
    int dP = 0, dR = 0, nP = 0, nR = 0;
    int8_t* crow = p.cand_out ? p.cand_out + b * p.cand_stride : nullptr;
    for (int j = lane; j < p.D; j += 32) {
      const int s = status(dec_class[j]);
      if (crow) crow[j] = (int8_t)s;
      if (dec_flags[j] & 1) {
        const bool seeded = srow[j] != -1;
        dP += (s == 1);
        dR += (s == 0);
        nP += (s == 1) && !seeded;
        nR += (s == 0) && !seeded;
      }
    }
    dP = __reduce_add_sync(kFull, dP);
    dR = __reduce_add_sync(kFull, dR);
    nP = __reduce_add_sync(kFull, nP);
    nR = __reduce_add_sync(kFull, nR);

    // 5. all slots (16 per lane-iteration on the vector path)
    if (p.slots_out) {
      int8_t* orow = p.slots_out + b * p.slots_stride;
      const int64_t full = p.S / 16;
      if (kVecSlots) {
        for (int64_t k = lane; k < full; k += 32) {
          const int4* cq = reinterpret_cast<const int4*>(slot_class) + 4 * k;
          uint32_t ow[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int4 c = cq[q];
            ow[q] = (uint32_t)(uint8_t)status(c.x) | ((uint32_t)(uint8_t)status(c.y) << 8) |
                    ((uint32_t)(uint8_t)status(c.z) << 16) | ((uint32_t)(uint8_t)status(c.w) << 24);
          }
          reinterpret_cast<uint4*>(orow)[k] = make_uint4(ow[0], ow[1], ow[2], ow[3]);
        }
        for (int64_t s = full * 16 + lane; s < p.S; s += 32) orow[s] = (int8_t)status(slot_class[s]);
      } else {
        for (int64_t s = lane; s < p.S; s += 32) orow[s] = (int8_t)status(slot_class[s]);
      }
    }
    if (lane == 0) {
      p.outcome[b] = conflict ? AP_OUTCOME_CONFLICT
                              : ((dP + dR == p.ncand) ? AP_OUTCOME_COMPLETE : AP_OUTCOME_INCOMPLETE);
      if (p.counts) {
        int4 cv = conflict ? make_int4(0, 0, 0, 0) : make_int4(dP, dR, nP, nR);
        reinterpret_cast<int4*>(p.counts)[b] = cv;
      }
    }
    __syncwarp();
  }
}

// Generic K1 for very wide graphs (per-warp scratch does not fit): the whole
// CTA works on one plan at a time, so the per-plan work (tens of thousands of
// slots, tables read through L2) is spread over 8 warps and several plans are
// in flight per SM.  Same phases as propagate_kernel with CTA barriers; P / R
// bitsets plus (kTable) a byte status table per CTA in shared memory.
template <bool kVecSlots, bool kTable>
__global__ void __launch_bounds__(kThreads) propagate_cta_kernel(PropParams p) {
  pdl_entry();
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ int s_red[kWarps][4];
  const int32_t* slot_class = p.slot_class;
  const int32_t* dec_class = p.dec_class;
  const uint8_t* dec_flags = p.dec_flags;
  const uint32_t* F = p.forced_words;
  const int32_t* imp_offset = p.imp_offset;
  const int32_t* imp_target = p.imp_target;
  const int32_t* first_same = p.first_same;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  uint32_t* P = reinterpret_cast<uint32_t*>(smem);
  uint32_t* R = P + p.Cw;
  int8_t* table = reinterpret_cast<int8_t*>(R + p.Cw);
  auto status = [&](int32_t c) -> int { return kTable ? (int)table[c] : class_status(P, R, F, c); };

  for (int64_t b = blockIdx.x; b < p.batch; b += gridDim.x) {
    for (int i = tid; i < (2 * p.Cw) / 4; i += kThreads) reinterpret_cast<uint4*>(P)[i] = make_uint4(0, 0, 0, 0);
    __syncthreads();
    const int8_t* srow = p.seeds + b * p.seed_stride;
    int conflict = 0;
    auto seed_one = [&](int j, int v) {
      if (v == 1 || v == 0) {
        const int32_t c = dec_class[j];
        atomicOr(v == 1 ? &P[c >> 5] : &R[c >> 5], 1u << (c & 31));
      } else if (v == 2) {  // sharding.py:116-118, 219-229
        if (dec_flags[j] & 2) conflict = 1;
        for (int k = first_same[j]; k < j; ++k)
          if (srow[k] == 1) conflict = 1;
      }
    };
    // 16 seeds per load (rows are 16-byte aligned); all-unseeded chunks cost one load
    const int dfull = kVecSlots ? p.D / 16 : 0;
    for (int q = tid; q < dfull; q += kThreads) {
      const uint4 w = reinterpret_cast<const uint4*>(srow)[q];
      if ((w.x & w.y & w.z & w.w) == 0xffffffffu) continue;
      const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        const int v = (int8_t)(ws[u >> 2] >> (8 * (u & 3)));
        if (v != -1) seed_one(16 * q + u, v);
      }
    }
    for (int j = 16 * dfull + tid; j < p.D; j += kThreads) seed_one(j, srow[j]);
    __syncthreads();
    // implications of every P class: a warp per bitset word, a lane per bit
    // (P is read-only here and R only gains bits, so the order is irrelevant)
    for (int w = warp; w < p.Cw; w += kWarps) {
      if (P[w] & (1u << lane)) {
        const int32_t c = 32 * w + lane;
        const int e = imp_offset[c + 1];
        for (int k = imp_offset[c]; k < e; ++k) {
          const int32_t t = imp_target[k];
          atomicOr(&R[t >> 5], 1u << (t & 31));
        }
      }
    }
    __syncthreads();
    for (int w = tid; w < p.Cw; w += kThreads) conflict |= (P[w] & (R[w] | F[w])) != 0;
    conflict = __syncthreads_or(conflict);
    if (kTable) {
      for (int c = tid; c < p.C; c += kThreads) table[c] = (int8_t)class_status(P, R, F, c);
      __syncthreads();
    }
    int dP = 0, dR = 0, nP = 0, nR = 0;
    int8_t* crow = p.cand_out ? p.cand_out + b * p.cand_stride : nullptr;
    auto tally = [&](int s, int flags, int seedv) {
      if (flags & 1) {
        const bool seeded = seedv != -1;
        dP += (s == 1);
        dR += (s == 0);
        nP += (s == 1) && !seeded;
        nR += (s == 0) && !seeded;
      }
    };
    // 16 candidates per step: class ids (4 x int4), flags and seeds (one uint4
    // each) in flight together, statuses stored as one uint4
    const bool cvec =
        kVecSlots && (!crow || (p.cand_stride % 16 == 0 && (reinterpret_cast<uintptr_t>(p.cand_out) & 15) == 0));
    const int cfull = cvec ? p.D / 16 : 0;
    for (int q = tid; q < cfull; q += kThreads) {
      const int4* cq = reinterpret_cast<const int4*>(dec_class) + 4 * q;
      const int4 c0 = cq[0], c1 = cq[1], c2 = cq[2], c3 = cq[3];
      const uint4 fl = reinterpret_cast<const uint4*>(dec_flags)[q];
      const uint4 sd = reinterpret_cast<const uint4*>(srow)[q];
      const int cls[16] = {c0.x, c0.y, c0.z, c0.w, c1.x, c1.y, c1.z, c1.w,
                           c2.x, c2.y, c2.z, c2.w, c3.x, c3.y, c3.z, c3.w};
      const uint32_t fw[4] = {fl.x, fl.y, fl.z, fl.w}, sw[4] = {sd.x, sd.y, sd.z, sd.w};
      uint32_t ow[4] = {0u, 0u, 0u, 0u};
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        const int st = status(cls[u]);
        ow[u >> 2] |= (uint32_t)(uint8_t)st << (8 * (u & 3));
        tally(st, (int)((fw[u >> 2] >> (8 * (u & 3))) & 0xffu), (int)(int8_t)(sw[u >> 2] >> (8 * (u & 3))));
      }
      if (crow) reinterpret_cast<uint4*>(crow)[q] = make_uint4(ow[0], ow[1], ow[2], ow[3]);
    }
    for (int j = 16 * cfull + tid; j < p.D; j += kThreads) {
      const int s = status(dec_class[j]);
      if (crow) crow[j] = (int8_t)s;
      tally(s, dec_flags[j], srow[j]);
    }
    if (p.slots_out) {
      int8_t* orow = p.slots_out + b * p.slots_stride;
      const int64_t full = p.S / 16;
      if (kVecSlots) {
        for (int64_t k = tid; k < full; k += kThreads) {
          const int4* cq = reinterpret_cast<const int4*>(slot_class) + 4 * k;
          uint32_t ow[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int4 c = cq[q];
            ow[q] = (uint32_t)(uint8_t)status(c.x) | ((uint32_t)(uint8_t)status(c.y) << 8) |
                    ((uint32_t)(uint8_t)status(c.z) << 16) | ((uint32_t)(uint8_t)status(c.w) << 24);
          }
          reinterpret_cast<uint4*>(orow)[k] = make_uint4(ow[0], ow[1], ow[2], ow[3]);
        }
        for (int64_t s = full * 16 + tid; s < p.S; s += kThreads) orow[s] = (int8_t)status(slot_class[s]);
      } else {
        for (int64_t s = tid; s < p.S; s += kThreads) orow[s] = (int8_t)status(slot_class[s]);
      }
    }
    dP = __reduce_add_sync(kFull, dP);
    dR = __reduce_add_sync(kFull, dR);
    nP = __reduce_add_sync(kFull, nP);
    nR = __reduce_add_sync(kFull, nR);
    if (lane == 0) {
      s_red[warp][0] = dP;
      s_red[warp][1] = dR;
      s_red[warp][2] = nP;
      s_red[warp][3] = nR;
    }
    __syncthreads();
    if (tid == 0) {
      int t[4] = {0, 0, 0, 0};
      for (int w = 0; w < kWarps; ++w)
        for (int q = 0; q < 4; ++q) t[q] += s_red[w][q];
      p.outcome[b] = conflict ? AP_OUTCOME_CONFLICT
                              : ((t[0] + t[1] == p.ncand) ? AP_OUTCOME_COMPLETE : AP_OUTCOME_INCOMPLETE);
      if (p.counts)
        reinterpret_cast<int4*>(p.counts)[b] = conflict ? make_int4(0, 0, 0, 0) : make_int4(t[0], t[1], t[2], t[3]);
    }
    __syncthreads();
  }
}

// ---- exact-order replay (one thread) --------------------------------------

struct TraceState {
  int8_t* st;
  const int64_t* base;
  const int32_t* owner;
  int conflict_site;
};

__device__ inline int tr_set(TraceState& t, int64_t s, int v, int site) {
  const int cur = t.st[s];
  if (cur == v) return 0;
  if (cur != -1) {
    t.conflict_site = site;
    return -1;
  }
  if (v == 1) {
    const int32_t o = t.owner[s];
    const int64_t lo = t.base[o], hi = t.base[o + 1];
    for (int64_t k = lo; k < hi; ++k)
      if (t.st[k] == 1) {
        t.conflict_site = site;
        return -1;
      }
    t.st[s] = 1;
    for (int64_t k = lo; k < hi; ++k)
      if (t.st[k] == -1) t.st[k] = 0;
  } else {
    t.st[s] = (int8_t)v;
  }
  return 1;
}

__device__ inline int tr_link(TraceState& t, int64_t a, int64_t b, int site) {
  const int va = t.st[a], vb = t.st[b];
  if (va == vb) return 0;
  if (va == -1) return tr_set(t, a, vb, site);
  if (vb == -1) return tr_set(t, b, va, site);
  t.conflict_site = site;
  return -1;
}

#define TR(expr)              \
  do {                        \
    const int _r = (expr);    \
    if (_r < 0) return -1;    \
    changed |= _r;            \
  } while (0)

__global__ void trace_kernel(const int32_t* prog, int64_t prog_len, const int32_t* forced, int64_t nforced,
                             const int64_t* dec_slots, const int8_t* seeds, int32_t D, int8_t* st,
                             const int64_t* base, const int32_t* owner, int64_t S, int64_t cap, bool has_init,
                             int32_t* result) {
  pdl_entry();
  TraceState t{st, base, owner, -1};
  if (!has_init)
    for (int64_t s = 0; s < S; ++s) st[s] = -1;
  int status = 0;  // 0 fixed point, 1 conflict, 2 cap exceeded
  for (int64_t i = 0; i < nforced && status == 0; ++i)
    if (tr_set(t, forced[i], 0, owner[forced[i]]) < 0) status = 1;
  for (int32_t j = 0; j < D && status == 0; ++j) {
    const int v = seeds[j];
    if (v == -1) continue;
    const int64_t s = dec_slots[j];
    if (tr_set(t, s, v == 2 ? -1 : v, owner[s]) < 0) status = 1;
  }
  auto sweep = [&](void) -> int {
    int changed = 0;
    int64_t pc = 0;
    while (pc < prog_len) {
      const int kind = prog[pc], site = prog[pc + 1];
      if (kind == RULE_LINK) {
        TR(tr_link(t, prog[pc + 2], prog[pc + 3], site));
        pc += 4;
      } else if (kind == RULE_DOT) {
        const int64_t a = base[prog[pc + 2]], b = base[prog[pc + 3]], c = base[prog[pc + 4]];
        TR(tr_link(t, a + 0, c + 0, site));
        TR(tr_link(t, b + 1, c + 1, site));
        TR(tr_link(t, a + 1, b + 0, site));
        if (st[a] == 1 || st[c] == 1) {
          TR(tr_set(t, b + 0, 0, site));
          TR(tr_set(t, b + 1, 0, site));
        }
        if (st[b + 1] == 1 || st[c + 1] == 1) {
          TR(tr_set(t, a + 0, 0, site));
          TR(tr_set(t, a + 1, 0, site));
        }
        if (st[a + 1] == 1 || st[b] == 1) {
          TR(tr_set(t, c + 0, 0, site));
          TR(tr_set(t, c + 1, 0, site));
        }
        pc += 5;
      } else {
        const int32_t a = prog[pc + 2], out = prog[pc + 3], nr = prog[pc + 4];
        const int32_t* red = prog + pc + 5;
        bool anyP = false;
        for (int k = 0; k < nr; ++k) anyP |= st[base[a] + red[k]] == 1;
        if (anyP)
          for (int64_t s = base[out]; s < base[out + 1]; ++s) TR(tr_set(t, s, 0, site));
        bool outP = false;
        for (int64_t s = base[out]; s < base[out + 1]; ++s) outP |= st[s] == 1;
        if (outP)
          for (int k = 0; k < nr; ++k) TR(tr_set(t, base[a] + red[k], 0, site));
        pc += 5 + nr;
      }
    }
    return changed;
  };
  if (status == 0) {
    status = 2;
    for (int64_t it = 0; it < cap; ++it) {
      const int r = sweep();
      if (r < 0) {
        status = 1;
        break;
      }
      if (r == 0) {
        status = 0;
        break;
      }
    }
  }
  result[0] = status;
  result[1] = t.conflict_site;
}


}  // namespace

int launch_propagate(const GraphTables* g, const DecisionTables* d, const int8_t* seeds, int64_t batch,
                     int64_t seed_stride, int8_t* slots_out, int64_t slots_stride, int8_t* cand_out,
                     int64_t cand_stride, uint8_t* outcome, int32_t* counts, cudaStream_t stream) {
  if (batch < 0 || (batch > 0 && (!seeds || !outcome)) || seed_stride < d->n ||
      (slots_out && slots_stride < g->num_slots) || (cand_out && cand_stride < d->n)) {
    set_error("ap_propagate_batch: bad arguments (null buffer or stride smaller than row)");
    return AP_ERR_INVALID;
  }
  if (d->graph != g) {
    set_error("ap_propagate_batch: decision set belongs to another graph");
    return AP_ERR_INVALID;
  }
  if (batch == 0) return AP_OK;
  PropParams p{};
  p.slot_class = g->d_slot_class.ptr;
  p.forced_words = g->d_forced_words.ptr;
  p.imp_offset = g->d_imp_offset.ptr;
  p.imp_target = g->d_imp_target.ptr;
  p.dec_class = d->d_dec_class.ptr;
  p.dec_flags = d->d_dec_flags.ptr;
  p.first_same = d->d_first_same.ptr;
  p.S = g->num_slots;
  p.C = g->num_classes;
  p.Cw = (int32_t)(((std::max(g->num_classes, 1) + 31) / 32 + 3) & ~3);  // words, multiple of 4
  p.D = d->n;
  p.T = (int32_t)g->imp_target.size();
  int ncand = 0;
  for (uint8_t f : d->dec_flags) ncand += f & 1;
  p.ncand = ncand;
  p.seeds = seeds;
  p.seed_stride = seed_stride;
  p.batch = batch;
  p.slots_out = slots_out;
  p.slots_stride = slots_stride;
  p.cand_out = cand_out;
  p.cand_stride = cand_stride;
  p.outcome = outcome;
  p.counts = counts;

  int64_t off = 0;
  auto place = [&](int64_t bytes) {
    const int64_t o = off;
    off += align16(bytes);
    return (int)o;
  };
  p.off_slot_class = place(p.S * 4);
  p.off_dec_class = place((int64_t)p.D * 4);
  p.off_dec_flags = place(p.D);
  p.off_forced = place((int64_t)p.Cw * 4);
  p.off_imp_off = place((int64_t)(p.C + 1) * 4);
  p.off_imp_tgt = place((int64_t)p.T * 4);
  p.off_first_same = place((int64_t)p.D * 4);
  const int64_t tables_bytes = off;
  const int64_t kSmemCap = 200 * 1024;
  // per-warp scratch: P / R bitsets, plus a byte status table when it fits
  const int64_t table_bytes = (int64_t)kWarps * (2 * p.Cw * 4 + align16(p.C));
  bool use_table = true, global_scratch = false;
  int64_t smem;
  // one plan per CTA when a plan is large (measured on B200: 4.4k classes / 11k
  // slots 11 -> 24 M plans/s; 320 classes / 800 slots is 3x faster per warp);
  // AP_PROPAGATE_CTA=1 forces it (tests)
  const bool force_cta = std::getenv("AP_PROPAGATE_CTA") != nullptr || p.S + p.D >= 6144;
  if (!force_cta && tables_bytes + table_bytes <= kSmemCap) {
    p.stage_tables = 1, p.off_scratch = (int)tables_bytes, smem = tables_bytes + table_bytes;
  } else if (!force_cta && table_bytes <= kSmemCap) {
    p.stage_tables = 0, p.off_scratch = 0, smem = table_bytes;
  } else {
    // very wide graphs: one plan per CTA (propagate_cta_kernel) with the
    // bitsets (+ status table when it fits) shared by the whole CTA
    // 16-byte rows: slot rows (when written) and seed rows; candidate rows are checked in the kernel
    const bool vec = (!slots_out || ((slots_stride % 16 == 0) && ((reinterpret_cast<uintptr_t>(slots_out) & 15) == 0))) &&
                     (seed_stride % 16 == 0) && ((reinterpret_cast<uintptr_t>(seeds) & 15) == 0);
    const int64_t cta_bits = (int64_t)2 * p.Cw * 4, cta_table = cta_bits + align16(p.C);
    if (cta_bits <= kSmemCap && std::getenv("AP_PROPAGATE_NO_CTA") == nullptr) {
      const bool tbl = cta_table <= kSmemCap;
      const int64_t csmem = tbl ? cta_table : cta_bits;
      auto ck = vec ? (tbl ? propagate_cta_kernel<true, true> : propagate_cta_kernel<true, false>)
                    : (tbl ? propagate_cta_kernel<false, true> : propagate_cta_kernel<false, false>);
      AP_CUDA_CHECK(cudaFuncSetAttribute(ck, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)csmem));
      int g_num_sms = 0;
      if (int rc = current_sm_count(&g_num_sms)) return rc;
      int cper = 0;
      AP_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&cper, ck, kThreads, (size_t)csmem));
      const int cgrid = (int)std::min<int64_t>(batch, (int64_t)g_num_sms * std::max(cper, 1));
      p.stage_tables = 0;
      launch_pdl(ck, dim3(cgrid), dim3(kThreads), (size_t)csmem, stream, p);
      AP_CUDA_CHECK(cudaGetLastError());
      return AP_OK;
    }
    // beyond even per-CTA bitsets in shared memory: per-warp bitsets in global memory
    p.stage_tables = 0, p.off_scratch = 0, smem = 0, use_table = false, global_scratch = true;
  }
  // per-warp layout: [P: Cw words][R: Cw words][status table: align16(C) bytes if kTable]
  p.warp_stride = (int64_t)2 * p.Cw * 4 + (use_table ? align16(p.C) : 0);
  const bool vec = slots_out && (slots_stride % 16 == 0) && ((reinterpret_cast<uintptr_t>(slots_out) & 15) == 0);
  auto kern = vec ? (use_table ? propagate_kernel<true, true> : propagate_kernel<true, false>)
                  : (use_table ? propagate_kernel<false, true> : propagate_kernel<false, false>);
  AP_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int g_num_sms = 0;
  if (int rc = current_sm_count(&g_num_sms)) return rc;
  int per_sm = 0;
  AP_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kThreads, (size_t)smem));
  per_sm = std::max(per_sm, 1);
  if (global_scratch) per_sm = std::min(per_sm, 2);  // bounds the global scratch footprint
  const int64_t want = (batch + kWarps - 1) / kWarps;
  const int grid = (int)std::min<int64_t>(want, (int64_t)g_num_sms * per_sm);
  if (global_scratch) {
    const int64_t words = (int64_t)grid * kWarps * 2 * p.Cw;
    if (words > g->scratch_words) {
      cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
      AP_CUDA_CHECK(cudaStreamIsCapturing(stream, &cs));
      if (cs != cudaStreamCaptureStatusNone) {
        set_error("ap_propagate_batch: generic scratch must grow during graph capture; launch once before");
        return AP_ERR_INVALID;
      }
      if (g->d_scratch) AP_CUDA_CHECK(cudaFree(g->d_scratch));
      AP_CUDA_CHECK(cudaMalloc(&g->d_scratch, words * sizeof(uint32_t)));
      g->scratch_words = words;
    }
    p.gscratch = g->d_scratch;
  }
  launch_pdl(kern, dim3(grid), dim3(kThreads), (size_t)smem, stream, p);
  AP_CUDA_CHECK(cudaGetLastError());
  return AP_OK;
}

int run_trace(const GraphTables* g, const DecisionTables* d, const int8_t* seeds_host, const int8_t* init_host,
              int8_t* slots_host, int32_t* outcome_host, int32_t* site_out, cudaStream_t stream) {
  const int64_t S = g->num_slots;
  int8_t* d_seeds = nullptr;
  int8_t* d_state = nullptr;
  int32_t* d_res = nullptr;
  AP_CUDA_CHECK(cudaMalloc(&d_seeds, std::max<int64_t>(d->n, 1)));
  AP_CUDA_CHECK(cudaMalloc(&d_state, std::max<int64_t>(S, 1)));
  AP_CUDA_CHECK(cudaMalloc(&d_res, 2 * sizeof(int32_t)));
  if (d->n) AP_CUDA_CHECK(cudaMemcpyAsync(d_seeds, seeds_host, d->n, cudaMemcpyHostToDevice, stream));
  if (init_host && S) AP_CUDA_CHECK(cudaMemcpyAsync(d_state, init_host, S, cudaMemcpyHostToDevice, stream));
  int max_rank = 1;
  for (int32_t q = 0; q < g->num_instr; ++q)
    max_rank = std::max<int>(max_rank, (int)(g->slot_base[q + 1] - g->slot_base[q]));
  const int64_t cap = std::max<int64_t>(2, (int64_t)g->num_instr * max_rank + 2);  // sharding.py:251-252
  launch_pdl(trace_kernel, dim3(1), dim3(1), 0, stream, g->d_program.ptr, (int64_t)g->program.size(), g->d_forced_list.ptr,
                                    (int64_t)g->forced_list.size(), d->d_slots.ptr, d_seeds, d->n, d_state,
                                    g->d_slot_base.ptr, g->d_slot_owner.ptr, S, cap, init_host != nullptr, d_res);
  AP_CUDA_CHECK(cudaGetLastError());
  int32_t res[2];
  AP_CUDA_CHECK(cudaMemcpyAsync(res, d_res, sizeof(res), cudaMemcpyDeviceToHost, stream));
  if (S) AP_CUDA_CHECK(cudaMemcpyAsync(slots_host, d_state, S, cudaMemcpyDeviceToHost, stream));
  AP_CUDA_CHECK(cudaStreamSynchronize(stream));
  cudaFree(d_seeds);
  cudaFree(d_state);
  cudaFree(d_res);
  if (res[0] == 2) {
    set_error("sharding propagation failed to reach a fixed point");
    return AP_ERR_UNSUPPORTED;
  }
  *site_out = res[1];
  if (res[0] == 1) {
    *outcome_host = AP_OUTCOME_CONFLICT;
  } else {
    bool complete = true;
    for (int32_t j = 0; j < d->n; ++j)
      if ((d->dec_flags[j] & 1) && slots_host[d->slots[j]] == -1) complete = false;
    *outcome_host = complete ? AP_OUTCOME_COMPLETE : AP_OUTCOME_INCOMPLETE;
  }
  return AP_OK;
}

}  // namespace apb
