// K1 fast path — descriptor-driven batched propagation (graphs with <= 255
// link classes, 16-byte aligned seed / output rows).
//
// Same closure as propagate.cu (see graph.cpp header), restructured so the
// per-plan instruction count scales with the number of 16-wide chunks instead
// of the number of slots:
//
// * slot chunk descriptor (static per graph, 16 B): the <= 8 distinct link
//   classes of 16 consecutive slots plus four PRMT selectors.  Emitting 16
//   slot statuses = <= 8 shared-memory table lookups, 3-6 PRMT to pack the
//   looked-up statuses into an 8-byte table, 4 PRMT with the selectors, one
//   16-byte store.  (BERT-48: every chunk has <= 4 distinct classes.)
// * decision chunk descriptor (static per decision set, 32 B): the chunk's
//   <= 8 local classes, one 16-bit position mask per local class and the
//   selectors for per-candidate output.  The seed pass turns 16 seed bytes
//   into P / R / U position masks with 3 LOP3 per word, then marks the
//   local class flags with one AND per class.
// * counts: decided P/R = sum over classes of (#candidates in class), newly =
//   decided - seeded (popcounts of the P/R masks); UNDECIDED seeds take a
//   per-position slow path.
// * the next plan's seed chunks are prefetched into registers while the
//   current plan is evaluated.
// Bit order of the 16-bit position masks: position t = 4*i + b (word i, byte b)
// is bit 4*b + i: OR-ing (word_i & 0x01010101) << i puts it at 8*b + i, and
// `squeeze` packs those nibbles into 16 bits.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <set>

#include "engine.h"

namespace apb {
namespace {

#ifndef AP_K1_MIN_BLOCKS
#define AP_K1_MIN_BLOCKS 2
#endif
#ifndef AP_K1_MAX_CTAS_PER_SM
#define AP_K1_MAX_CTAS_PER_SM 0  // 0: as many as fit
#endif
#ifndef AP_K1_WARPS
#define AP_K1_WARPS 12  // 12 warps x 2 CTAs per SM: measured best on B200 (BERT-48)
#endif
constexpr int kWarpsF = AP_K1_WARPS;
constexpr int kThreadsF = kWarpsF * 32;
constexpr unsigned kFullMask = 0xffffffffu;
constexpr uint32_t kOnes = 0x01010101u;
constexpr int kScratchPerWarp = 1024;  // flagP[256] flagR[256] table[256] codes[256]
constexpr int kLaneMaxDecChunks = 32;   // K1-lane limits: |D| <= 512
constexpr int kLaneMaxSlotChunks = 32;  //                 |S| <= 512 (measured: BERT-base's 1,421 slots run faster warp-per-plan)

// 16-bit position mask bit of chunk position t = 4*i + b (word i, byte b)
inline int perm_bit(int t) { return 4 * (t & 3) + (t >> 2); }

// Local classes of one 16-wide chunk, first-appearance order.  Returns false
// when the chunk has more than 8 distinct classes.
bool local_classes(const int32_t* cls, int count, std::vector<int>* uniq, int local[16]) {
  uniq->clear();
  for (int t = 0; t < 16; ++t) {
    const int c = t < count ? cls[t] : cls[0];
    auto it = std::find(uniq->begin(), uniq->end(), c);
    if (it == uniq->end()) {
      if (uniq->size() == 8) return false;
      uniq->push_back(c);
      local[t] = (int)uniq->size() - 1;
    } else {
      local[t] = (int)(it - uniq->begin());
    }
  }
  return true;
}

void pack_classes(const std::vector<int>& uniq, uint32_t* w0, uint32_t* w1) {
  uint8_t b[8];
  for (int j = 0; j < 8; ++j) b[j] = j < (int)uniq.size() ? (uint8_t)uniq[j] : 0xFF;
  std::memcpy(w0, b, 4);
  std::memcpy(w1, b + 4, 4);
  if (uniq.size() <= 4) *w1 = 0xFFFFFFFFu;  // marker: four lookups suffice
}

void pack_selectors(const int local[16], uint32_t* z, uint32_t* w) {
  uint32_t sel[4];
  for (int j = 0; j < 4; ++j) {
    sel[j] = 0;
    for (int b = 0; b < 4; ++b) sel[j] |= (uint32_t)local[4 * j + b] << (4 * b);
  }
  *z = sel[0] | (sel[1] << 16);
  *w = sel[2] | (sel[3] << 16);
}

// Transposed selectors for the packed 2-bit output: word j, byte b selects slot
// 4*b + j, so OR-ing word j shifted left by 2*j puts slot t's code at bits 2*t.
// Slots past the row end select byte 4 (a zero operand): codes 0 in the padding.
void pack_selectors_t(const int local[16], int count, uint32_t* z, uint32_t* w) {
  uint32_t sel[4];
  for (int j = 0; j < 4; ++j) {
    sel[j] = 0;
    for (int b = 0; b < 4; ++b) sel[j] |= (uint32_t)(4 * b + j < count ? local[4 * b + j] : 4) << (4 * b);
  }
  *z = sel[0] | (sel[1] << 16);
  *w = sel[2] | (sel[3] << 16);
}

}  // namespace

void build_fast_graph(GraphTables* g) {
  g->fast = g->num_classes <= kMaxFastClasses;
  if (!g->fast) return;
  const int64_t S = g->num_slots;
  const int64_t nq = (S + 15) / 16;
  g->slot_desc.assign(nq * 4, 0);
  g->slot_desc_t.assign(nq * 4, 0);
  g->slot_cls8.assign(nq * 16, 0xFF);
  std::vector<int> uniq;
  int local[16];
  for (int64_t q = 0; q < nq; ++q) {
    const int count = (int)std::min<int64_t>(16, S - 16 * q);
    for (int t = 0; t < count; ++t) g->slot_cls8[16 * q + t] = (uint8_t)g->class_of_slot[16 * q + t];
    uint32_t* d = &g->slot_desc[4 * q];
    uint32_t* dt = &g->slot_desc_t[4 * q];
    if (!local_classes(&g->class_of_slot[16 * q], count, &uniq, local)) {
      d[0] = 0xFFFFFFFFu;  // fallback: per-slot lookups through slot_cls8
      dt[0] = 0xFFFFFFFFu;
      continue;
    }
    pack_classes(uniq, &d[0], &d[1]);
    pack_selectors(local, &d[2], &d[3]);
    dt[0] = d[0];
    dt[1] = d[1];
    pack_selectors_t(local, count, &dt[2], &dt[3]);
  }
  g->slot_fallback_chunks = 0;
  g->slot_all_k4 = true;
  for (int64_t q = 0; q < nq; ++q) {
    if ((g->slot_desc[4 * q] & 0xFF) == 0xFF) {
      g->slot_fallback_chunks++;
      g->slot_all_k4 = false;
    } else if (g->slot_desc[4 * q + 1] != 0xFFFFFFFFu) {
      g->slot_all_k4 = false;
    }
  }
  const int C = g->num_classes;
  g->imp_bits.assign((size_t)std::max(C, 1) * 8, 0);
  g->forced_bits.assign(8, 0);
  for (int c = 0; c < C; ++c) {
    for (int k = g->imp_offset[c]; k < g->imp_offset[c + 1]; ++k) {
      const int t = g->imp_target[k];
      g->imp_bits[(size_t)8 * c + (t >> 5)] |= 1u << (t & 31);
    }
    if (g->class_forced[c]) g->forced_bits[c >> 5] |= 1u << (c & 31);
  }
}

void build_fast_decision(const GraphTables* g, DecisionTables* d) {
  d->fast = g->fast && d->n <= 32 * kFastMaxChunks * 16 && d->n < 65536;
  if (!d->fast) return;
  const int n = d->n;
  const int nq = (n + 15) / 16;
  d->dec_desc.assign((size_t)nq * 8, 0);
  d->dec_masks.assign(nq, 0);
  d->dec_cls8.assign((size_t)nq * 16, 0xFF);
  d->class_ncand.assign(256, 0);
  d->ncand = 0;
  std::vector<int32_t> cls(n);
  for (int i = 0; i < n; ++i) {
    cls[i] = g->class_of_slot[d->slots[i]];
    d->dec_cls8[i] = (uint8_t)cls[i];
    if (d->dec_flags[i] & 1) {
      d->class_ncand[cls[i]]++;
      d->ncand++;
    }
  }
  d->ncand_planes.assign(16 * 4, 0);
  for (int c = 0; c < std::min(g->num_classes, 128); ++c)
    for (int k = 0; k < 16; ++k)
      if ((d->class_ncand[c] >> k) & 1) d->ncand_planes[4 * k + (c >> 5)] |= 1u << (c & 31);
  std::vector<int> uniq;
  int local[16];
  for (int q = 0; q < nq; ++q) {
    const int count = std::min(16, n - 16 * q);
    uint32_t valid = 0, cand = 0;
    for (int t = 0; t < count; ++t) {
      valid |= 1u << perm_bit(t);
      if (d->dec_flags[16 * q + t] & 1) cand |= 1u << perm_bit(t);
    }
    d->dec_masks[q] = valid | (cand << 16);
    uint32_t* w = &d->dec_desc[(size_t)8 * q];
    if (!local_classes(&cls[16 * q], count, &uniq, local)) {
      w[0] = 0xFFFFFFFFu;  // fallback chunk
      continue;
    }
    pack_classes(uniq, &w[0], &w[1]);
    uint32_t m[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int t = 0; t < count; ++t) m[local[t]] |= 1u << perm_bit(t);
    w[2] = m[0] | (m[1] << 16);
    w[3] = m[2] | (m[3] << 16);
    w[4] = m[4] | (m[5] << 16);
    w[5] = m[6] | (m[7] << 16);
    pack_selectors(local, &w[6], &w[7]);
  }
}

namespace {

struct FastParams {
  const uint4* slot_desc;
  const uint8_t* slot_cls8;
  const uint4* dec_desc;
  const uint32_t* dec_masks;
  const uint8_t* dec_cls8;
  const uint32_t* forced_bits;  // [8]
  const uint16_t* ncand;        // [256]
  const uint32_t* imp_bits;     // [C * 8]
  const uint8_t* dec_flags;     // global, slow path only
  const int32_t* first_same;    // global, slow path only
  int32_t nq_s, nq_d, C, D, any_slot_fallback, slot_all_k4, ncand_total;
  int64_t S;
  const int8_t* seeds;
  int64_t seed_stride, batch;
  int8_t* slots_out;
  int64_t slots_stride;
  int8_t* cand_out;
  int64_t cand_stride;
  int cand_vec;
  uint8_t* outcome;
  int32_t* counts;
  uint32_t* packed_out;     // 2-bit slot codes, [batch, packed_stride] 32-bit words, or null
  int64_t packed_stride;    // in 32-bit words
  const uint4* slot_desc_t; // transposed-selector descriptors (packed output)
  int bulk;                 // int8 slot rows staged in shared memory, stored by TMA bulk copies
  const uint32_t* ncand_planes;  // lane kernel: [16][4] classes whose candidate count has bit k
  int nplanes;
  int lane_pitch;   // lane kernel: per-row pitch of the warp's shared-memory output block (0: direct stores)
  int off_lane_stage;
  int off_lane_tab, lane_tab_stride;  // lane kernel: per-thread class status (or code) table
  int64_t stage_bytes;      // per-warp staging row (16 * nq_s)
  int off_slot_desc, off_slot_cls8, off_dec_desc, off_dec_masks, off_dec_cls8, off_ncand, off_imp_bits, off_scratch;
  int off_stage;
};

__device__ __forceinline__ uint32_t lds_u8(uint32_t addr) {
  uint32_t v;
  asm volatile("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(addr));
  return v;
}
__device__ __forceinline__ void sts_u8(uint32_t addr, uint32_t v) {
  asm volatile("st.shared.u8 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}
__device__ __forceinline__ uint4 ldg_stream(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ void stg_stream(void* p, uint4 v) {
  asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}

// predicated streaming store: one @p STG, no branch around it
__device__ __forceinline__ void stg_stream_if(void* p, uint4 v, int pred) {
  asm volatile(
      "{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %5, 0;\n\t@q st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};\n\t}" ::"l"(p),
      "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w), "r"(pred)
      : "memory");
}

// address of byte `k` of packed class word `w` inside a 256-aligned table at `base`
#define TBL_ADDR(w, base, k) __byte_perm((w), (base), 0x7650 + (k))

// Status table of up to 8 local classes as two words (bytes = int8 statuses).
__device__ __forceinline__ void local_table(uint32_t c03, uint32_t c47, uint32_t tb, uint32_t* lo, uint32_t* hi) {
  const uint32_t s0 = lds_u8(TBL_ADDR(c03, tb, 0));
  const uint32_t s1 = lds_u8(TBL_ADDR(c03, tb, 1));
  const uint32_t s2 = lds_u8(TBL_ADDR(c03, tb, 2));
  const uint32_t s3 = lds_u8(TBL_ADDR(c03, tb, 3));
  *lo = __byte_perm(__byte_perm(s0, s1, 0x0040), __byte_perm(s2, s3, 0x0040), 0x5410);
  if (c47 == 0xFFFFFFFFu) {
    *hi = *lo;
  } else {
    const uint32_t s4 = lds_u8(TBL_ADDR(c47, tb, 0));
    const uint32_t s5 = lds_u8(TBL_ADDR(c47, tb, 1));
    const uint32_t s6 = lds_u8(TBL_ADDR(c47, tb, 2));
    const uint32_t s7 = lds_u8(TBL_ADDR(c47, tb, 3));
    *hi = __byte_perm(__byte_perm(s4, s5, 0x0040), __byte_perm(s6, s7, 0x0040), 0x5410);
  }
}

// raw PRMT: the selectors are stored with clear mode bits, so skip the
// 0x7777 masking __byte_perm adds; PRMT reads only selector bits [15:0]
__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t s) {
  uint32_t d;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(s));
  return d;
}

__device__ __forceinline__ uint4 select16(uint32_t lo, uint32_t hi, uint32_t z, uint32_t w) {
  uint4 o;
  o.x = prmt(lo, hi, z);
  o.y = prmt(lo, hi, z >> 16);
  o.z = prmt(lo, hi, w);
  o.w = prmt(lo, hi, w >> 16);
  return o;
}

// Status word of 4 local classes (k <= 4 chunks).
__device__ __forceinline__ uint32_t local_table4(uint32_t c03, uint32_t tb) {
  const uint32_t s0 = lds_u8(TBL_ADDR(c03, tb, 0));
  const uint32_t s1 = lds_u8(TBL_ADDR(c03, tb, 1));
  const uint32_t s2 = lds_u8(TBL_ADDR(c03, tb, 2));
  const uint32_t s3 = lds_u8(TBL_ADDR(c03, tb, 3));
  return prmt(prmt(s0, s1, 0x0040), prmt(s2, s3, 0x0040), 0x5410);
}

// Squeeze bits {8b + i : b, i < 4} into bits {4b + i}: one shift-or and one PRMT.
__device__ __forceinline__ uint32_t squeeze(uint32_t x) {
  const uint32_t y = x | (x >> 4);
  return prmt(y, 0u, 0x4420);
}

// P / R / U position masks of one 16-byte seed chunk (bit 4*b + i for word i, byte b)
__device__ __forceinline__ void seed_masks(uint4 s, uint32_t* xp, uint32_t* xr, uint32_t* xu) {
  const uint32_t w[4] = {s.x, s.y, s.z, s.w};
  uint32_t p = 0, r = 0, u = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const uint32_t a = w[i], b = w[i] >> 1;
    p |= ((a & ~b) & kOnes) << i;   // byte == 1 (bit0 set, bit1 clear)
    r |= ((~a & ~b) & kOnes) << i;  // byte == 0
    u |= ((~a & b) & kOnes) << i;   // byte == 2
  }
  *xp = squeeze(p);
  *xr = squeeze(r);
  *xu = squeeze(u);
}

// MAXCH: 16-byte seed chunks per lane; NW: 32-bit class words (classes <= 32*NW)
template <int MAXCH, int NW>
__global__ void __launch_bounds__(kThreadsF, AP_K1_MIN_BLOCKS) propagate_fast_kernel(FastParams p) {
  pdl_entry();
  extern __shared__ __align__(16) uint8_t smem[];
  // stage the static tables
  auto stage = [&](int off, const void* src, int64_t bytes) {
    const uint4* s = reinterpret_cast<const uint4*>(src);
    uint4* d = reinterpret_cast<uint4*>(smem + off);
    const int64_t n16 = bytes / 16;
    for (int64_t i = threadIdx.x; i < n16; i += blockDim.x) d[i] = s[i];
    const uint8_t* sb = reinterpret_cast<const uint8_t*>(src);
    for (int64_t i = n16 * 16 + threadIdx.x; i < bytes; i += blockDim.x) smem[off + i] = sb[i];
  };
  if (p.packed_out) {
    stage(p.off_slot_desc, p.slot_desc_t, (int64_t)p.nq_s * 16);  // packed rows only use the transposed set
  } else {
    stage(p.off_slot_desc, p.slot_desc, (int64_t)p.nq_s * 16);
  }
  if (p.any_slot_fallback) stage(p.off_slot_cls8, p.slot_cls8, (int64_t)p.nq_s * 16);
  stage(p.off_dec_desc, p.dec_desc, (int64_t)p.nq_d * 32);
  stage(p.off_dec_masks, p.dec_masks, (int64_t)p.nq_d * 4);
  stage(p.off_dec_cls8, p.dec_cls8, (int64_t)p.nq_d * 16);
  stage(p.off_ncand, p.ncand, 512);
  stage(p.off_imp_bits, p.imp_bits, (int64_t)p.C * 32);
  __syncthreads();

  const uint4* slot_desc = reinterpret_cast<const uint4*>(smem + p.off_slot_desc);
  const uint8_t* slot_cls8 = smem + p.off_slot_cls8;
  const uint4* dec_desc = reinterpret_cast<const uint4*>(smem + p.off_dec_desc);
  const uint32_t* dec_masks = reinterpret_cast<const uint32_t*>(smem + p.off_dec_masks);
  const uint8_t* dec_cls8 = smem + p.off_dec_cls8;
  const uint16_t* ncand = reinterpret_cast<const uint16_t*>(smem + p.off_ncand);
  const uint4* imp_bits = reinterpret_cast<const uint4*>(smem + p.off_imp_bits);
  uint32_t forced_bits[NW];
#pragma unroll
  for (int k = 0; k < NW; ++k) forced_bits[k] = p.forced_bits[k];

  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  // per-warp scratch, 256-aligned in the shared window so table / flag
  // addresses are base | class (one PRMT each)
  const uint32_t smem_sa = (uint32_t)__cvta_generic_to_shared(smem);
  const uint32_t scratch_sa = (smem_sa + (uint32_t)p.off_scratch + 255u) & ~255u;
  uint8_t* scratch = smem + (scratch_sa - smem_sa) + warp * kScratchPerWarp;
  uint8_t* flagP = scratch;
  uint8_t* flagR = scratch + 256;
  int8_t* table = reinterpret_cast<int8_t*>(scratch + 512);
  uint8_t* codes = scratch + 768;  // status + 1 per class (packed output)
  const uint32_t fb = (uint32_t)__cvta_generic_to_shared(flagP);  // flagR = fb + 256
  const uint32_t tb = fb + 512;
  const uint32_t cb = fb + 768;
  const uint32_t stage_sa = smem_sa + (uint32_t)p.off_stage + (uint32_t)(warp * p.stage_bytes);
  uint64_t evict_first = 0;
  if (p.bulk) asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(evict_first));

  const int64_t nwarps = (int64_t)gridDim.x * kWarpsF;
  int64_t b = (int64_t)blockIdx.x * kWarpsF + warp;
  uint4 cur[MAXCH];
  if (b < p.batch) {
#pragma unroll
    for (int i = 0; i < MAXCH; ++i) cur[i] = ldg_stream(p.seeds + b * p.seed_stride + 16 * min(lane + 32 * i, p.nq_d - 1));
  }

  for (; b < p.batch; b += nwarps) {
    // 0. clear flags (512 bytes: one 16-byte store per lane)
    reinterpret_cast<uint4*>(scratch)[lane] = make_uint4(0, 0, 0, 0);
    __syncwarp();

    // 1. seed pass
    int nPs = 0, nRs = 0;
    uint32_t anyU = 0;
#pragma unroll
    for (int i = 0; i < MAXCH; ++i) {
      const int q = lane + 32 * i;
      if (q < p.nq_d) {
        uint32_t xp, xr, xu;
        seed_masks(cur[i], &xp, &xr, &xu);
        const uint32_t vm = dec_masks[q];
        const uint32_t valid = vm & 0xFFFF, cand = vm >> 16;
        xp &= valid;
        xr &= valid;
        anyU |= xu & valid;
        nPs += __popc(xp & cand);
        nRs += __popc(xr & cand);
        const uint4 d0 = dec_desc[2 * q];
        if ((d0.x & 0xFF) != 0xFF) {
          const uint32_t mw[4] = {d0.z, d0.w, 0, 0};
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const uint32_t m = (j & 1) ? (mw[j >> 1] >> 16) : (mw[j >> 1] & 0xFFFF);
            const uint32_t a = TBL_ADDR(d0.x, fb, j);
            if (xp & m) sts_u8(a, 1);
            if (xr & m) sts_u8(a + 256, 1);
          }
          if (d0.y != 0xFFFFFFFFu) {
            const uint4 d1 = dec_desc[2 * q + 1];
            const uint32_t mw2[2] = {d1.x, d1.y};
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const uint32_t m = (j & 1) ? (mw2[j >> 1] >> 16) : (mw2[j >> 1] & 0xFFFF);
              const uint32_t a = TBL_ADDR(d0.y, fb, j);
              if (xp & m) sts_u8(a, 1);
              if (xr & m) sts_u8(a + 256, 1);
            }
          }
        } else {
#pragma unroll
          for (int t = 0; t < 16; ++t) {
            const uint32_t bit = 1u << (4 * (t & 3) + (t >> 2));
            const uint32_t c = dec_cls8[16 * q + t];
            if (xp & bit) flagP[c] = 1;
            if (xr & bit) flagR[c] = 1;
          }
        }
      }
    }
    const bool hasU = __any_sync(kFullMask, anyU != 0);
    __syncwarp();

    // prefetch the next plan's seeds while this one is evaluated.  The loads
    // are unconditional (addresses clamped into the batch) so they land in
    // cur[] directly; a guarded load compiles to load-to-temp + predicated
    // move, which waits out the DRAM latency right here.
    const int64_t bn = b + nwarps < p.batch ? b + nwarps : b;
    const int8_t* nrow = p.seeds + bn * p.seed_stride;
#pragma unroll
    for (int i = 0; i < MAXCH; ++i) {
      const int q = min(lane + 32 * i, p.nq_d - 1);
      cur[i] = ldg_stream(nrow + 16 * q);
    }

    // 2. class bitsets: word k holds classes 32k..32k+31 (flags beyond C stay 0)
    uint32_t Pw[NW], Rw[NW], acc[NW];
    uint32_t myP = 0;  // bit k: this lane's class 32k+lane is partitioned
#pragma unroll
    for (int k = 0; k < NW; ++k) {
      acc[k] = 0;
      Pw[k] = __ballot_sync(kFullMask, flagP[32 * k + lane] != 0);
      Rw[k] = __ballot_sync(kFullMask, flagR[32 * k + lane] != 0) | forced_bits[k];
      myP |= ((Pw[k] >> lane) & 1u) << k;
    }
    // 3. implications: each lane ORs the rows of its own partitioned classes
    //    (rows are 8 words apart, only the first NW matter), then one warp
    //    OR-reduction per word
    while (myP) {
      const int k = __ffs(myP) - 1;
      myP &= myP - 1;
      const uint32_t* row = reinterpret_cast<const uint32_t*>(imp_bits + 2 * (32 * k + lane));
      if (NW <= 4) {
        const uint4 a = *reinterpret_cast<const uint4*>(row);
        const uint32_t aw[4] = {a.x, a.y, a.z, a.w};
#pragma unroll
        for (int w = 0; w < NW; ++w) acc[w] |= aw[w];
      } else {
        const uint4 a = *reinterpret_cast<const uint4*>(row), c = *reinterpret_cast<const uint4*>(row + 4);
        const uint32_t aw[8] = {a.x, a.y, a.z, a.w, c.x, c.y, c.z, c.w};
#pragma unroll
        for (int w = 0; w < NW; ++w) acc[w] |= aw[w];
      }
    }
    uint32_t clash = 0;
#pragma unroll
    for (int k = 0; k < NW; ++k) {
      Rw[k] |= __reduce_or_sync(kFullMask, acc[k]);
      clash |= Pw[k] & Rw[k];
    }
    bool conflict = clash != 0;  // warp-uniform

    // 4. class status table and decided counts (lane-owned classes)
    uint32_t dPR = 0;  // decided P | decided R << 16
#pragma unroll
    for (int k = 0; k < NW; ++k) {
      const int c = 32 * k + lane;
      const bool isP = (Pw[k] >> lane) & 1u;
      const bool isR = (Rw[k] >> lane) & 1u;
      table[c] = isP ? 1 : (isR ? 0 : -1);
      if (p.packed_out) codes[c] = isP ? 2 : (isR ? 1 : 0);
      const uint32_t nc = ncand[c];
      dPR += isP ? nc : (isR ? (nc << 16) : 0u);
    }
    dPR = __reduce_add_sync(kFullMask, dPR);
    uint32_t sPR = __reduce_add_sync(kFullMask, (uint32_t)nPs | ((uint32_t)nRs << 16));
    __syncwarp();

    int dP = dPR & 0xFFFF, dR = dPR >> 16;
    int nP = dP - (int)(sPR & 0xFFFF), nR = dR - (int)(sPR >> 16);
    if (hasU) {
      // UNDECIDED seeds: conflict rule and exact per-position newly counts
      const int8_t* srow = p.seeds + b * p.seed_stride;
      bool uconf = false;
      int np = 0, nr = 0;
      for (int j = lane; j < p.D; j += 32) {
        const int v = srow[j];
        if (v == 2) {
          if (p.dec_flags[j] & 2) uconf = true;
          for (int k = p.first_same[j]; k < j; ++k)
            if (srow[k] == 1) uconf = true;
        }
        if ((p.dec_flags[j] & 1) && v == -1) {
          const int s = table[dec_cls8[j]];
          np += s == 1;
          nr += s == 0;
        }
      }
      conflict |= __any_sync(kFullMask, uconf);
      nP = __reduce_add_sync(kFullMask, np);
      nR = __reduce_add_sync(kFullMask, nr);
    }

    // 4. per-candidate statuses
    if (p.cand_out) {
      int8_t* crow = p.cand_out + b * p.cand_stride;
      for (int q = lane; q < p.nq_d; q += 32) {
        const uint4 d0 = dec_desc[2 * q];
        if (p.cand_vec && (d0.x & 0xFF) != 0xFF) {
          const uint4 d1 = dec_desc[2 * q + 1];
          uint32_t lo, hi;
          local_table(d0.x, d0.y, tb, &lo, &hi);
          const uint4 o = select16(lo, hi, d1.z, d1.w);
          if (16 * q + 16 <= p.D) {
            reinterpret_cast<uint4*>(crow)[q] = o;
          } else {
            for (int t = 0; 16 * q + t < p.D; ++t) {
              const uint32_t wv = (t >> 2) == 0 ? o.x : ((t >> 2) == 1 ? o.y : ((t >> 2) == 2 ? o.z : o.w));
              crow[16 * q + t] = (int8_t)(wv >> (8 * (t & 3)));
            }
          }
        } else {
          for (int t = 0; t < 16 && 16 * q + t < p.D; ++t) crow[16 * q + t] = table[dec_cls8[16 * q + t]];
        }
      }
    }

    // 5. all slot statuses
    if (p.packed_out) {
      // 2-bit codes, 16 slots per 32-bit word, one coalesced 4-byte store per lane
      uint32_t* prow = p.packed_out + b * p.packed_stride;
      if (p.slot_all_k4) {
        const int rounds = (p.nq_s + 31) >> 5;
        const int last = p.nq_s - 1;
#pragma unroll 4
        for (int it = 0; it < rounds; ++it) {
          const int q = lane + 32 * it;
          const uint4 d = slot_desc[min(q, last)];
          const uint32_t lo = local_table4(d.x, cb);
          const uint32_t w0 = prmt(lo, 0u, d.z), w1 = prmt(lo, 0u, d.z >> 16);
          const uint32_t w2 = prmt(lo, 0u, d.w), w3 = prmt(lo, 0u, d.w >> 16);
          const uint32_t word = w0 | (w1 << 2) | (w2 << 4) | (w3 << 6);
          if (q <= last) __stcs(prow + q, word);
        }
      } else {
        for (int q = lane; q < p.nq_s; q += 32) {
          const uint4 d = slot_desc[q];
          uint32_t word = 0;
          if ((d.x & 0xFF) != 0xFF) {  // <= 8 local classes: the same selection on code bytes
            uint32_t lo, hi;
            local_table(d.x, d.y, cb, &lo, &hi);
            word = prmt(lo, hi, d.z) | (prmt(lo, hi, d.z >> 16) << 2) | (prmt(lo, hi, d.w) << 4) |
                   (prmt(lo, hi, d.w >> 16) << 6);
            const int64_t rem = p.S - 16 * (int64_t)q;  // padding codes are 0
            if (rem < 16) word &= (1u << (2 * rem)) - 1u;
          } else {
            for (int t = 0; t < 16 && 16 * q + t < p.S; ++t) word |= (uint32_t)codes[slot_cls8[16 * q + t]] << (2 * t);
          }
          __stcs(prow + q, word);
        }
      }
    } else if (p.slots_out && p.slot_all_k4 && p.bulk) {
      // stage the row in shared memory, one TMA bulk store per plan (issued by lane 0)
      if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      __syncwarp();
      const int rounds = (p.nq_s + 31) >> 5;
      const int last = p.nq_s - 1;
#pragma unroll 4
      for (int it = 0; it < rounds; ++it) {
        const int q = lane + 32 * it;
        const uint4 d = slot_desc[min(q, last)];
        const uint32_t lo = local_table4(d.x, tb);
        const uint4 o = select16(lo, lo, d.z, d.w);
        if (q <= last)
          asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(stage_sa + 16 * q), "r"(o.x), "r"(o.y),
                       "r"(o.z), "r"(o.w)
                       : "memory");
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) {
        asm volatile(
            "cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(
                p.slots_out + b * p.slots_stride),
            "r"(stage_sa), "r"((uint32_t)p.stage_bytes), "l"(evict_first)
            : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      }
    } else if (p.slots_out && p.slot_all_k4) {
      // common case (BERT-48): branch-free, four lookups per 16 slots
      // warp-uniform trip count: a per-lane `q < nq_s` bound diverges in the
      // last round and runs the unrolled body's remainder paths back to back
      int8_t* orow = p.slots_out + b * p.slots_stride + 16 * lane;
      const int rounds = (p.nq_s + 31) >> 5;
      const int last = p.nq_s - 1;
#pragma unroll 4
      for (int it = 0; it < rounds; ++it) {
        const int q = lane + 32 * it;
        const uint4 d = slot_desc[min(q, last)];
        const uint32_t lo = local_table4(d.x, tb);
        stg_stream_if(orow + 512 * it, select16(lo, lo, d.z, d.w), q <= last);
      }
    } else if (p.slots_out) {
      int8_t* orow = p.slots_out + b * p.slots_stride;
      for (int q = lane; q < p.nq_s; q += 32) {
        const uint4 d = slot_desc[q];
        uint4 o;
        if ((d.x & 0xFF) != 0xFF) {
          uint32_t lo, hi;
          local_table(d.x, d.y, tb, &lo, &hi);
          o = select16(lo, hi, d.z, d.w);
        } else {
          uint32_t ow[4] = {0, 0, 0, 0};
          for (int t = 0; t < 16; ++t) ow[t >> 2] |= (uint32_t)(uint8_t)table[slot_cls8[16 * q + t]] << (8 * (t & 3));
          o = make_uint4(ow[0], ow[1], ow[2], ow[3]);
        }
        stg_stream(orow + 16 * q, o);
      }
    }
    if (lane == 0) {
      // complete iff every candidate is decided (sharding.py:246-247)
      p.outcome[b] = conflict ? AP_OUTCOME_CONFLICT
                              : ((dP + dR == p.ncand_total) ? AP_OUTCOME_COMPLETE : AP_OUTCOME_INCOMPLETE);
      if (p.counts)
        reinterpret_cast<int4*>(p.counts)[b] = conflict ? make_int4(0, 0, 0, 0) : make_int4(dP, dR, nP, nR);
    }
    __syncwarp();
  }
  if (p.bulk && lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}


// ---------------------------------------------------------------------------
// K1-lane: one THREAD per plan for small graphs (<= 128 link classes, |D| <= 512,
// |S| <= 512: MLP2, VGG-19, the zoo blocks).  A warp per plan spends most of its
// ~400 instructions on per-plan fixed costs (ballots, reductions, flag tables) when
// a plan has only a few chunks; here the class bitsets live in one thread's
// registers (<= 2 words), so the same closure costs a few dozen instructions:
// seed chunks -> P / R class bits through the decision descriptors, forced classes,
// OR of the implication rows of the P classes, conflict = P & R, decided counts as
// popcounts against per-bit planes of the candidate-per-class counts, and slot
// chunks emitted from the same descriptors as the warp kernel (status of class c =
// bit c of P / R).  Same outputs bit for bit (tests/test_bench_batches_gpu.py).
// word c >> 5 of a register bitset (NW <= 4) without dynamic indexing
template <int NW>
__device__ __forceinline__ uint32_t lane_word(const uint32_t* w, uint32_t c) {
  uint32_t v = w[0];
#pragma unroll
  for (int k = 1; k < NW; ++k) v = (c >> 5) == (uint32_t)k ? w[k] : v;
  return v;
}

template <int NW>
__device__ __forceinline__ uint32_t lane_status(const uint32_t* Pw, const uint32_t* Rw, uint32_t c, bool codes) {
  const uint32_t pw = lane_word<NW>(Pw, c);
  const uint32_t rw = lane_word<NW>(Rw, c);
  const uint32_t sh = c & 31u;
  const uint32_t pb = (pw >> sh) & 1u, rb = (rw >> sh) & 1u;
  if (codes) return pb ? 2u : (rb ? 1u : 0u);
  return pb ? 1u : (rb ? 0u : 0xFFu);
}

template <int NW>
__device__ __forceinline__ uint32_t lane_word4(const uint32_t* Pw, const uint32_t* Rw, uint32_t cls4, bool codes) {
  const uint32_t s0 = lane_status<NW>(Pw, Rw, cls4 & 0xFF, codes);
  const uint32_t s1 = lane_status<NW>(Pw, Rw, (cls4 >> 8) & 0xFF, codes);
  const uint32_t s2 = lane_status<NW>(Pw, Rw, (cls4 >> 16) & 0xFF, codes);
  const uint32_t s3 = lane_status<NW>(Pw, Rw, cls4 >> 24, codes);
  return s0 | (s1 << 8) | (s2 << 16) | (s3 << 24);
}

template <int NW>
__device__ __forceinline__ void lane_set(uint32_t* w, uint32_t c) {
  const uint32_t bit = 1u << (c & 31u);
#pragma unroll
  for (int k = 0; k < NW; ++k) w[k] |= (c >> 5) == (uint32_t)k ? bit : 0u;
}

// local classes of a decision chunk (<= 4 in `cls4`, position masks in two words)
template <int NW>
__device__ __forceinline__ void lane_mark(uint32_t cls4, uint32_t m01, uint32_t m23, uint32_t xp, uint32_t xr,
                                          uint32_t* Pw, uint32_t* Rw) {
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const uint32_t c = (cls4 >> (8 * j)) & 0xFF;
    const uint32_t m = (j & 1) ? ((j < 2 ? m01 : m23) >> 16) : ((j < 2 ? m01 : m23) & 0xFFFF);
    if (c == 0xFF) continue;
    if (xp & m) lane_set<NW>(Pw, c);
    if (xr & m) lane_set<NW>(Rw, c);
  }
}

// the thread's class table: byte c = status of class c (codes: status + 1), four classes per
// 32-bit store, straight from the register bitsets
template <int NW>
__device__ __forceinline__ void lane_write_table(uint32_t* tab, const uint32_t* Pw, const uint32_t* Rw, int C,
                                                 bool codes) {
#pragma unroll
  for (int k = 0; k < NW; ++k) {
#pragma unroll
    for (int n = 0; n < 8; ++n) {
      const int c4 = 8 * k + n;
      if (4 * c4 >= C) break;
      const uint32_t p4 = (Pw[k] >> (4 * n)) & 0xFu, r4 = (Rw[k] >> (4 * n)) & 0xFu;
      uint32_t w = 0;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint32_t pb = (p4 >> j) & 1u, rb = (r4 >> j) & 1u;
        const uint32_t v = codes ? (pb ? 2u : (rb ? 1u : 0u)) : (pb ? 1u : (rb ? 0u : 0xFFu));
        w |= v << (8 * j);
      }
      tab[c4] = w;
    }
  }
}

// status word of 4 classes (bytes of `cls4`) from the thread's table
__device__ __forceinline__ uint32_t lane_tab4(const uint8_t* tab, uint32_t cls4) {
  const uint32_t s0 = tab[cls4 & 0xFF], s1 = tab[(cls4 >> 8) & 0xFF], s2 = tab[(cls4 >> 16) & 0xFF],
                 s3 = tab[cls4 >> 24];
  return prmt(prmt(s0, s1, 0x0040), prmt(s2, s3, 0x0040), 0x5410);
}

template <int NW>
__global__ void __launch_bounds__(256) propagate_lane_kernel(FastParams p) {
  pdl_entry();
  extern __shared__ __align__(16) uint8_t smem[];
  auto stage = [&](int off, const void* src, int64_t bytes) {
    const uint4* s = reinterpret_cast<const uint4*>(src);
    uint4* d = reinterpret_cast<uint4*>(smem + off);
    const int64_t n16 = bytes / 16;
    for (int64_t i = threadIdx.x; i < n16; i += blockDim.x) d[i] = s[i];
    const uint8_t* sb = reinterpret_cast<const uint8_t*>(src);
    for (int64_t i = n16 * 16 + threadIdx.x; i < bytes; i += blockDim.x) smem[off + i] = sb[i];
  };
  stage(p.off_slot_desc, p.packed_out ? p.slot_desc_t : p.slot_desc, (int64_t)p.nq_s * 16);
  if (p.any_slot_fallback) stage(p.off_slot_cls8, p.slot_cls8, (int64_t)p.nq_s * 16);
  stage(p.off_dec_desc, p.dec_desc, (int64_t)p.nq_d * 32);
  stage(p.off_dec_masks, p.dec_masks, (int64_t)p.nq_d * 4);
  stage(p.off_dec_cls8, p.dec_cls8, (int64_t)p.nq_d * 16);
  stage(p.off_ncand, p.ncand_planes, 256);
  stage(p.off_imp_bits, p.imp_bits, (int64_t)p.C * 32);
  __syncthreads();
  const uint4* slot_desc = reinterpret_cast<const uint4*>(smem + p.off_slot_desc);
  const uint8_t* slot_cls8 = smem + p.off_slot_cls8;
  const uint4* dec_desc = reinterpret_cast<const uint4*>(smem + p.off_dec_desc);
  const uint32_t* dec_masks = reinterpret_cast<const uint32_t*>(smem + p.off_dec_masks);
  const uint8_t* dec_cls8 = smem + p.off_dec_cls8;
  const uint32_t* planes = reinterpret_cast<const uint32_t*>(smem + p.off_ncand);  // [16][4]
  const uint32_t* imp = reinterpret_cast<const uint32_t*>(smem + p.off_imp_bits);  // [C][8]
  uint32_t forced[NW];
#pragma unroll
  for (int k = 0; k < NW; ++k) forced[k] = p.forced_bits[k];
  const bool codes = p.packed_out != nullptr;
  const int lane = threadIdx.x & 31;
  // 32 consecutive plans per warp: their output rows form one contiguous block, staged in
  // shared memory (row pitch an odd number of 16-byte units: conflict-free 16-byte stores)
  // and written back with coalesced stores instead of 32 scattered row stores
  uint8_t* ostage = p.lane_pitch ? smem + p.off_lane_stage + (threadIdx.x >> 5) * 32 * p.lane_pitch : nullptr;
  const int64_t nwarps_total = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t base = ((int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * 32; base < p.batch;
       base += nwarps_total * 32) {
   const int64_t b = base + lane;
   if (b < p.batch) {
    uint32_t Pw[NW], Rw[NW];
#pragma unroll
    for (int k = 0; k < NW; ++k) Pw[k] = Rw[k] = 0;
    int nPs = 0, nRs = 0;
    uint32_t anyU = 0;
    const int8_t* srow = p.seeds + b * p.seed_stride;
    for (int q = 0; q < p.nq_d; ++q) {
      uint32_t xp, xr, xu;
      seed_masks(ldg_stream(srow + 16 * q), &xp, &xr, &xu);
      const uint32_t vm = dec_masks[q];
      const uint32_t valid = vm & 0xFFFF, cand = vm >> 16;
      xp &= valid;
      xr &= valid;
      anyU |= xu & valid;
      nPs += __popc(xp & cand);
      nRs += __popc(xr & cand);
      const uint4 d0 = dec_desc[2 * q];
      if ((d0.x & 0xFF) != 0xFF) {
        lane_mark<NW>(d0.x, d0.z, d0.w, xp, xr, Pw, Rw);
        if (d0.y != 0xFFFFFFFFu) {
          const uint4 d1 = dec_desc[2 * q + 1];
          lane_mark<NW>(d0.y, d1.x, d1.y, xp, xr, Pw, Rw);
        }
      } else {
        for (int t = 0; t < 16; ++t) {
          const uint32_t bit = 1u << (4 * (t & 3) + (t >> 2));
          const uint32_t c = dec_cls8[16 * q + t];
          if (xp & bit) lane_set<NW>(Pw, c);
          if (xr & bit) lane_set<NW>(Rw, c);
        }
      }
    }
    // implications of the partitioned classes, conflict
    uint32_t acc[NW];
#pragma unroll
    for (int k = 0; k < NW; ++k) acc[k] = 0;
#pragma unroll
    for (int k = 0; k < NW; ++k) {
      uint32_t t = Pw[k];
      while (t) {
        const int c = 32 * k + __ffs(t) - 1;
        t &= t - 1;
#pragma unroll
        for (int w = 0; w < NW; ++w) acc[w] |= imp[8 * c + w];
      }
    }
    uint32_t clash = 0;
#pragma unroll
    for (int k = 0; k < NW; ++k) {
      Rw[k] |= forced[k] | acc[k];
      clash |= Pw[k] & Rw[k];
    }
    bool conflict = clash != 0;
    int dP = 0, dR = 0;
    for (int k = 0; k < p.nplanes; ++k) {
      int cp = 0, cr = 0;
#pragma unroll
      for (int w = 0; w < NW; ++w) {
        cp += __popc(Pw[w] & planes[4 * k + w]);
        cr += __popc(Rw[w] & ~Pw[w] & planes[4 * k + w]);
      }
      dP += cp << k;
      dR += cr << k;
    }
    int nP = dP - nPs, nR = dR - nRs;
    if (anyU) {  // UNDECIDED seeds: conflict rule and exact per-position newly counts
      bool uconf = false;
      int np = 0, nr = 0;
      for (int j = 0; j < p.D; ++j) {
        const int v = srow[j];
        if (v == 2) {
          if (p.dec_flags[j] & 2) uconf = true;
          for (int k = p.first_same[j]; k < j; ++k)
            if (srow[k] == 1) uconf = true;
        }
        if ((p.dec_flags[j] & 1) && v == -1) {
          const uint32_t st = lane_status<NW>(Pw, Rw, dec_cls8[j], false);
          np += st == 1;
          nr += st == 0;
        }
      }
      conflict |= uconf;
      nP = np;
      nR = nr;
    }
    p.outcome[b] = conflict ? AP_OUTCOME_CONFLICT
                            : ((dP + dR == p.ncand_total) ? AP_OUTCOME_COMPLETE : AP_OUTCOME_INCOMPLETE);
    if (p.counts)
      reinterpret_cast<int4*>(p.counts)[b] = conflict ? make_int4(0, 0, 0, 0) : make_int4(dP, dR, nP, nR);
    uint8_t* tab = smem + p.off_lane_tab + threadIdx.x * p.lane_tab_stride;
    // statuses (slots / candidates) or codes (packed rows); the packed mode's candidate statuses
    // come from the bitsets directly
    lane_write_table<NW>(reinterpret_cast<uint32_t*>(tab), Pw, Rw, p.C, codes);
    if (p.cand_out) {
      int8_t* crow = p.cand_out + b * p.cand_stride;
      for (int q = 0; q < p.nq_d; ++q) {
        const uint4 d0 = dec_desc[2 * q];
        uint4 o;
        if ((d0.x & 0xFF) != 0xFF) {
          const uint4 d1 = dec_desc[2 * q + 1];
          const uint32_t lo = codes ? lane_word4<NW>(Pw, Rw, d0.x, false) : lane_tab4(tab, d0.x);
          const uint32_t hi = d0.y == 0xFFFFFFFFu ? lo : (codes ? lane_word4<NW>(Pw, Rw, d0.y, false)
                                                                : lane_tab4(tab, d0.y));
          o = select16(lo, hi, d1.z, d1.w);
        } else {
          uint32_t ow[4] = {0, 0, 0, 0};
          for (int t = 0; t < 16; ++t) ow[t >> 2] |= lane_status<NW>(Pw, Rw, dec_cls8[16 * q + t], false) << (8 * (t & 3));
          o = make_uint4(ow[0], ow[1], ow[2], ow[3]);
        }
        if (p.cand_vec && 16 * q + 16 <= p.D) {
          reinterpret_cast<uint4*>(crow)[q] = o;
        } else {
          for (int t = 0; 16 * q + t < p.D && t < 16; ++t) {
            const uint32_t wv = (t >> 2) == 0 ? o.x : ((t >> 2) == 1 ? o.y : ((t >> 2) == 2 ? o.z : o.w));
            crow[16 * q + t] = (int8_t)(wv >> (8 * (t & 3)));
          }
        }
      }
    }
    if (p.slots_out) {
      int8_t* orow = ostage ? reinterpret_cast<int8_t*>(ostage + lane * p.lane_pitch) : p.slots_out + b * p.slots_stride;
      for (int q = 0; q < p.nq_s; ++q) {
        const uint4 d = slot_desc[q];
        uint4 o;
        if ((d.x & 0xFF) != 0xFF) {
          const uint32_t lo = lane_tab4(tab, d.x);
          const uint32_t hi = d.y == 0xFFFFFFFFu ? lo : lane_tab4(tab, d.y);
          o = select16(lo, hi, d.z, d.w);
        } else {
          uint32_t ow[4] = {0, 0, 0, 0};
          for (int t = 0; t < 16; ++t) ow[t >> 2] |= (uint32_t)tab[slot_cls8[16 * q + t]] << (8 * (t & 3));
          o = make_uint4(ow[0], ow[1], ow[2], ow[3]);
        }
        if (ostage)
          *reinterpret_cast<uint4*>(orow + 16 * q) = o;
        else
          stg_stream(orow + 16 * q, o);
      }
    } else if (codes) {
      uint32_t* prow = ostage ? reinterpret_cast<uint32_t*>(ostage + lane * p.lane_pitch) : p.packed_out + b * p.packed_stride;
      for (int q = 0; q < p.nq_s; ++q) {
        const uint4 d = slot_desc[q];  // transposed selectors
        uint32_t word = 0;
        if ((d.x & 0xFF) != 0xFF) {
          const uint32_t lo = lane_tab4(tab, d.x);
          const uint32_t hi = d.y == 0xFFFFFFFFu ? 0u : lane_tab4(tab, d.y);
          word = prmt(lo, hi, d.z) | (prmt(lo, hi, d.z >> 16) << 2) | (prmt(lo, hi, d.w) << 4) |
                 (prmt(lo, hi, d.w >> 16) << 6);
          const int64_t rem = p.S - 16 * (int64_t)q;
          if (rem < 16) word &= (1u << (2 * rem)) - 1u;
        } else {
          for (int t = 0; t < 16 && 16 * q + t < p.S; ++t) word |= (uint32_t)tab[slot_cls8[16 * q + t]] << (2 * t);
        }
        if (ostage)
          prow[q] = word;
        else
          __stcs(prow + q, word);
      }
    }
   }
    if (ostage) {  // the warp's block of rows [base, base + rows) -> global, coalesced
      __syncwarp();
      const int rows = p.batch - base < 32 ? (int)(p.batch - base) : 32;
      // only each row's nq_s data units: the caller's row stride may leave bytes it owns
      const int nq = p.nq_s;
      if (p.slots_out) {
        const int64_t ld16 = p.slots_stride / 16;
        uint4* dst = reinterpret_cast<uint4*>(p.slots_out + base * p.slots_stride);
        int r = lane / nq, c = lane - r * nq;
        const int dr = 32 / nq, dc = 32 - dr * nq;
        for (int i = lane; i < rows * nq; i += 32) {
          __stcs(dst + r * ld16 + c, *reinterpret_cast<const uint4*>(ostage + r * p.lane_pitch + 16 * c));
          r += dr, c += dc;
          if (c >= nq) c -= nq, ++r;
        }
      } else {
        uint32_t* dst = p.packed_out + base * p.packed_stride;
        int r = lane / nq, c = lane - r * nq;
        const int dr = 32 / nq, dc = 32 - dr * nq;
        for (int i = lane; i < rows * nq; i += 32) {
          __stcs(dst + r * p.packed_stride + c, *reinterpret_cast<const uint32_t*>(ostage + r * p.lane_pitch + 4 * c));
          r += dr, c += dc;
          if (c >= nq) c -= nq, ++r;
        }
      }
      __syncwarp();
    }
  }
}

template <int MAXCH, int NW>
int launch_fast_t(const FastParams& p, int64_t smem, cudaStream_t stream) {
  int num_sms = 0;
  if (int rc = current_sm_count(&num_sms)) return rc;
  auto kern = propagate_fast_kernel<MAXCH, NW>;
  AP_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int per_sm = 0;
  AP_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kThreadsF, (size_t)smem));
  if (AP_K1_MAX_CTAS_PER_SM > 0) per_sm = std::min(per_sm, AP_K1_MAX_CTAS_PER_SM);
  per_sm = std::max(per_sm, 1);
  const int64_t want = (p.batch + kWarpsF - 1) / kWarpsF;
  const int grid = (int)std::min<int64_t>(want, (int64_t)num_sms * per_sm);
  launch_pdl(kern, dim3(grid), dim3(kThreadsF), (size_t)smem, stream, p);
  AP_CUDA_CHECK(cudaGetLastError());
  return AP_OK;
}

inline int64_t a16(int64_t x) { return (x + 15) & ~int64_t(15); }

template <int MAXCH>
int dispatch_nw(int nw, const FastParams& p, int64_t smem, cudaStream_t stream) {
  switch (nw <= 1 ? 1 : nw) {
    case 1: return launch_fast_t<MAXCH, 1>(p, smem, stream);
    case 2: return launch_fast_t<MAXCH, 2>(p, smem, stream);
    case 3: return launch_fast_t<MAXCH, 3>(p, smem, stream);
    case 4: return launch_fast_t<MAXCH, 4>(p, smem, stream);
    case 5: return launch_fast_t<MAXCH, 5>(p, smem, stream);
    case 6: return launch_fast_t<MAXCH, 6>(p, smem, stream);
    case 7: return launch_fast_t<MAXCH, 7>(p, smem, stream);
    default: return launch_fast_t<MAXCH, 8>(p, smem, stream);
  }
}

}  // namespace

int launch_propagate_fast(const GraphTables* g, const DecisionTables* d, const int8_t* seeds, int64_t batch,
                          int64_t seed_stride, int8_t* slots_out, int64_t slots_stride, int8_t* cand_out,
                          int64_t cand_stride, uint8_t* outcome, int32_t* counts, cudaStream_t stream,
                          uint8_t* packed_out, int64_t packed_stride) {
  if (!g->fast || !d->fast || d->n == 0) return AP_ERR_UNSUPPORTED;
  if (packed_out && (slots_out || packed_stride % 4 || (reinterpret_cast<uintptr_t>(packed_out) & 3) ||
                     packed_stride < 4 * ((g->num_slots + 15) / 16)))
    return AP_ERR_UNSUPPORTED;
  const int nq_d = (d->n + 15) / 16;
  const int64_t nq_s = (g->num_slots + 15) / 16;
  auto aligned = [](const void* ptr) { return (reinterpret_cast<uintptr_t>(ptr) & 15) == 0; };
  if (seed_stride % 16 || !aligned(seeds) || seed_stride < 16 * nq_d) return AP_ERR_UNSUPPORTED;
  if (slots_out && (slots_stride % 16 || !aligned(slots_out) || slots_stride < 16 * nq_s)) return AP_ERR_UNSUPPORTED;
  FastParams p{};
  p.slot_desc = reinterpret_cast<const uint4*>(g->d_slot_desc.ptr);
  p.slot_cls8 = g->d_slot_cls8.ptr;
  p.dec_desc = reinterpret_cast<const uint4*>(d->d_dec_desc.ptr);
  p.dec_masks = d->d_dec_masks.ptr;
  p.dec_cls8 = d->d_dec_cls8.ptr;
  p.forced_bits = g->d_forced_bits.ptr;
  p.ncand = d->d_class_ncand.ptr;
  p.imp_bits = g->d_imp_bits.ptr;
  p.dec_flags = d->d_dec_flags.ptr;
  p.first_same = d->d_first_same.ptr;
  p.nq_s = (int32_t)nq_s;
  p.nq_d = nq_d;
  p.C = g->num_classes;
  p.D = d->n;
  p.any_slot_fallback = g->slot_fallback_chunks > 0;
  p.slot_all_k4 = g->slot_all_k4;
  p.ncand_total = d->ncand;
  p.S = g->num_slots;
  p.seeds = seeds;
  p.seed_stride = seed_stride;
  p.batch = batch;
  p.slots_out = slots_out;
  p.slots_stride = slots_stride;
  p.cand_out = cand_out;
  p.cand_stride = cand_stride;
  p.cand_vec = cand_out && cand_stride % 16 == 0 && aligned(cand_out);
  p.outcome = outcome;
  p.counts = counts;
  p.packed_out = reinterpret_cast<uint32_t*>(packed_out);
  p.packed_stride = packed_stride / 4;
  p.slot_desc_t = reinterpret_cast<const uint4*>(g->d_slot_desc_t.ptr);
  // TMA bulk row stores (AP_K1_BULK=1): int8 rows of k<=4 graphs, staged per warp in shared memory
  const char* bulk_env = std::getenv("AP_K1_BULK");
  p.bulk = slots_out && g->slot_all_k4 && bulk_env && bulk_env[0] == '1';
  p.stage_bytes = 16 * nq_s;
  int64_t off = 0;
  auto place = [&](int64_t bytes) {
    const int64_t o = off;
    off += a16(bytes);
    return (int)o;
  };
  p.off_slot_desc = place(nq_s * 16);
  p.off_slot_cls8 = p.any_slot_fallback ? place(nq_s * 16) : 0;
  p.off_dec_desc = place((int64_t)nq_d * 32);
  p.off_dec_masks = place((int64_t)nq_d * 4);
  p.off_dec_cls8 = place((int64_t)nq_d * 16);
  p.off_ncand = place(512);
  p.off_imp_bits = place((int64_t)std::max(p.C, 1) * 32);
  p.off_scratch = (int)off;
  off += 256 + (int64_t)kWarpsF * kScratchPerWarp;
  p.off_stage = (int)a16(off);
  if (p.bulk) {
    off = p.off_stage + (int64_t)kWarpsF * p.stage_bytes;
    if (off > 110 * 1024) p.bulk = 0, off = p.off_stage;  // keep 2 CTAs per SM
  }
  const int64_t smem = off;
  if (smem > 200 * 1024) return AP_ERR_UNSUPPORTED;
  // K1-lane (one thread per plan) for small graphs; AP_K1_LANE=0 forces the warp kernel
  const char* lane_env = std::getenv("AP_K1_LANE");
  const bool lane_ok = p.C <= 128 && nq_d <= kLaneMaxDecChunks && nq_s <= kLaneMaxSlotChunks && !p.bulk;
  if (lane_ok && !(lane_env && lane_env[0] == '0')) {
    p.ncand_planes = d->d_ncand_planes.ptr;
    int maxc = 0;
    for (int c = 0; c < p.C; ++c) maxc = std::max<int>(maxc, d->class_ncand[c]);
    p.nplanes = 0;
    while ((1 << p.nplanes) <= maxc) ++p.nplanes;
    // per-warp output staging when a warp's 32 rows fit (pitch: odd count of 16-byte units)
    const int64_t row_bytes = slots_out ? slots_stride : (packed_out ? packed_stride : 0);
    int64_t pitch = (row_bytes + 15) / 16;
    if (pitch % 2 == 0) ++pitch;
    pitch *= 16;
    p.lane_pitch = 0;
    p.off_lane_stage = (int)a16(p.off_scratch);
    const char* st_env = std::getenv("AP_K1_LANE_STAGE");
    if (row_bytes > 16 && pitch <= 400 && !(st_env && st_env[0] == '0')) p.lane_pitch = (int)pitch;
    int64_t lsmem = p.lane_pitch ? p.off_lane_stage + 8 * 32 * pitch : p.off_scratch;
    int tw = (p.C + 3) / 4;  // 32-bit words per thread table, odd: conflict-free byte lookups
    if (tw % 2 == 0) ++tw;
    p.lane_tab_stride = 4 * tw;
    p.off_lane_tab = (int)a16(lsmem);
    // + 256: unused local-class bytes (0xFF) of a descriptor index past the thread's row; the
    // selectors never pick those bytes, the loads only have to stay inside the allocation
    lsmem = p.off_lane_tab + 256 * (int64_t)p.lane_tab_stride + 256;
    int sms = 0;
    if (int rc = current_sm_count(&sms)) return rc;
    const int64_t want = (batch + 255) / 256;
    auto go = [&](auto kern) -> int {
      AP_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)lsmem));
      launch_pdl(kern, dim3((unsigned)std::min<int64_t>(want, (int64_t)sms * 8)), dim3(256), (size_t)lsmem, stream, p);
      return AP_OK;
    };
    const int lnw = (p.C + 31) / 32;
    if (lnw <= 1) go(propagate_lane_kernel<1>);
    else if (lnw == 2) go(propagate_lane_kernel<2>);
    else if (lnw == 3) go(propagate_lane_kernel<3>);
    else go(propagate_lane_kernel<4>);
    AP_CUDA_CHECK(cudaGetLastError());
    return AP_OK;
  }
  const int chunks = (nq_d + 31) / 32;
  const int nw = (p.C + 31) / 32;
  if (chunks <= 1) return dispatch_nw<1>(nw, p, smem, stream);
  if (chunks <= 2) return dispatch_nw<2>(nw, p, smem, stream);
  if (chunks <= 3) return dispatch_nw<3>(nw, p, smem, stream);
  if (chunks <= 4) return dispatch_nw<4>(nw, p, smem, stream);
  if (chunks <= 8) return dispatch_nw<8>(nw, p, smem, stream);
  return AP_ERR_UNSUPPORTED;
}

}  // namespace apb
