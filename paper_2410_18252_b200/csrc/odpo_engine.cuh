// odpo_engine.cuh -- persistent TMA-ring row engine (sm_100a).
//
// One CTA = NCW consumer warps + 1 producer warp.  The producer's elected lane draws work
// tickets from a global counter, decodes them into row items, and streams each row's
// vocabulary in CH-byte chunks into an S-stage shared-memory ring with 1-D TMA bulk copies
// (cp.async.bulk ... mbarrier::complete_tx, with an L2 cache policy per item kind).
// Consumers wait on the stage's full barrier, process the chunk out of shared memory, and
// release it on the stage's empty barrier, so the next rows' loads are always in flight
// while the current row is reduced.
#pragma once

#include <cstddef>

#include "odpo_device.cuh"

namespace odpo {

// Engine geometry (tuned on B200 for the BASELINE shapes; see profiles/ and DESIGN.md).
// Geometry 0 (default): 4 consumer warps per CTA, a 3 x 16 KB TMA ring, 4 CTAs per SM.
// Geometry 1 (large rows): 8 consumer warps, a 6 x 16 KB ring, 2 CTAs per SM -- half as many
// rows in flight, so a row's unscaled backward re-read stays in L2 for 256 KB rows.
#ifndef ODPO_NCW
#define ODPO_NCW 4
#endif
#ifndef ODPO_STAGES
#define ODPO_STAGES 3
#endif
#ifndef ODPO_CHUNK
#define ODPO_CHUNK 16384
#endif
#ifndef ODPO_CTAS_PER_SM
#define ODPO_CTAS_PER_SM 4
#endif
#ifndef ODPO_CLUSTER
#define ODPO_CLUSTER 1
#endif
constexpr int kCS = ODPO_CLUSTER;          // CTAs per thread-block cluster (one row per cluster)
#ifndef ODPO_NEPI
#define ODPO_NEPI 2
#endif
constexpr int kNEpi = ODPO_NEPI;           // row-epilogue warps (slot s -> warp s % kNEpi)
constexpr int kChunk = ODPO_CHUNK;         // bytes per stage
constexpr int kCV = kChunk / 16;           // 16-byte vectors per chunk
constexpr int kSlots = 8;                  // rows in flight per CTA (row-slot ring)
constexpr int kLook = 1;                   // default rows decoded ahead of the row being pushed
// Experimental (build flag): FUSED forward rows dispatched as ODPO_FSPLIT vocabulary parts
// (separate work units, merged in part order by the unit that finishes last) to shorten the
// pair-completion latency; 1 = whole rows (default).
#ifndef ODPO_FSPLIT
#define ODPO_FSPLIT 1
#endif
constexpr int kFS = ODPO_FSPLIT;
static_assert(kSlots % kNEpi == 0, "epilogue warps must tile the slot ring");

template <int NCW_, int STAGES_, int CPS_>
struct Geo {
  static constexpr int NCW = NCW_;         // consumer warps (warps 0..NCW-1)
  static constexpr int NCT = NCW * 32;     // consumer threads
  static constexpr int STAGES = STAGES_;   // TMA ring stages of kChunk bytes
  static constexpr int CPS = CPS_;         // CTAs per SM (launch bounds)
  static constexpr int UB = kCV / NCT;     // vectors per consumer thread per chunk
  static constexpr int PROD = NCW;         // TMA producer warp
  static constexpr int PAR = NCW + 1;      // backward-parameter prefetch warp
  static constexpr int EPI = NCW + 2;      // first row-epilogue warp
  static constexpr int THREADS = NCT + 64 + 32 * kNEpi;
  static constexpr int SMEM = STAGES * kChunk;
  static_assert(kCV % NCT == 0, "chunk must split evenly over consumers");
};
using Geo0 = Geo<ODPO_NCW, ODPO_STAGES, ODPO_CTAS_PER_SM>;
#ifndef ODPO_G1_NCW
#define ODPO_G1_NCW 8
#endif
#ifndef ODPO_G1_STAGES
#define ODPO_G1_STAGES 6
#endif
#ifndef ODPO_G1_CPS
#define ODPO_G1_CPS 2
#endif
using Geo1 = Geo<ODPO_G1_NCW, ODPO_G1_STAGES, ODPO_G1_CPS>;

// ------------------------------------------------------------------ mbarrier / TMA PTX
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
// All barrier operations below take 32-bit shared-window addresses (hoisted out of loops).
__device__ __forceinline__ void mbar_arrive(uint32_t b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(b) : "memory");
}
__device__ __forceinline__ void mbar_arrive_n(uint32_t b, uint32_t n) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(n) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint32_t b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes)
               : "memory");
}
// ---- thread-block cluster helpers (DSMEM): 32-bit shared::cluster addresses
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t mapa(uint32_t local_addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local_addr), "r"(rank));
  return r;
}
__device__ __forceinline__ void st_cl_u32(uint32_t addr, uint32_t v) {
  asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}
__device__ __forceinline__ void st_cl_u64(uint32_t addr, uint64_t v) {
  asm volatile("st.shared::cluster.u64 [%0], %1;" ::"r"(addr), "l"(v) : "memory");
}
__device__ __forceinline__ void mbar_arrive_cl(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive_cl_n(uint32_t cluster_addr, uint32_t n) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0], %1;" ::"r"(cluster_addr),
               "r"(n)
               : "memory");
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release;\n\tbarrier.cluster.wait.acquire;" ::: "memory");
}

// Blocking wait on the phase with the given parity (cluster-scope acquire: a barrier may
// receive arrivals, and the data they publish, from other CTAs of the cluster).
__device__ __forceinline__ void mbar_wait_cl(uint32_t b, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1, %2;\n\t"
      "@!p bra WAIT%=;\n}" ::"r"(b),
      "r"(parity), "r"(1000000u)
      : "memory");
}

// Blocking wait on the phase with the given parity.  The suspend-time hint lets the hardware
// park the warp until the phase completes instead of spinning through issue slots.
__device__ __forceinline__ void mbar_wait(uint32_t b, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
      "@!p bra WAIT%=;\n}" ::"r"(b),
      "r"(parity), "r"(1000000u)
      : "memory");
}
__device__ __forceinline__ void tma_load_1d(uint32_t dst_smem, const void* src, uint32_t bytes,
                                            uint32_t bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1], %2, [%3], %4;" ::"r"(dst_smem),
      "l"(src), "r"(bytes), "r"(bar), "l"(pol)
      : "memory");
}
// ------------------------------------------------------------------ row slots
enum { K_END = 0, K_F = 1, K_FSKIP = 2, K_B = 3, K_ZERO = 4, K_NONE = 5 };

// One row in flight.  Written by the producer before it signals slot_full (epilogue) and
// before the row's first stage (consumers); B-row parameters are added before param_ready;
// per-warp partials and x_tok are added by the consumers before part_ready.
struct RowSlot {
  int32_t kind;
  int32_t tok;
  int32_t nchunk;
  uint32_t pphase;  // parity of the param_ready phase this (B) row waits for
  int32_t fslot;    // UNSC backward rows: the slot holding the same row's forward pass
  int32_t part;    // FUSED forward rows split in ODPO_FSPLIT vocabulary parts: this part
  int64_t p;       // pair (FUSED) or sequence (SEQ)
  int64_t s;       // sequence
  int64_t g;       // row = s*T + t
  const char* row;
  char* drow;
  float c, coef, gtok, xtok;
  float xm;              // backward rows: the row max m (fp32 inputs form (x - m) k2, bwd_const)
  float pm[32], pr[32];  // per-warp (m, r) partials: [cluster rank * kNCW + warp]
};
// the header (kind .. drow) is what the cluster leader broadcasts to its peers
constexpr int kSlotHeaderBytes = 64;
static_assert(offsetof(RowSlot, c) == kSlotHeaderBytes, "slot header layout");

// ------------------------------------------------------------------ per-batch online update
// fp32 inputs (DT 0): exact exclusion of one max element (log1p form, 1e-5 contract).
// bf16 inputs (DT 1): uniform fast path; a batch that raises the running max subtracts the
// max element's own term (value exactly as added: p(0) = 1 for the polynomial and
// ex2(delta) for MUFU agree to ~1e-13), keeping r free of the "1" (error ~1e-6 relative,
// far inside the 2e-3 bf16 contract).  NPF of every 8 elements use the FMA-pipe exp2.
// XM: form the exp2 arguments as (x - m) k2 (fwd_arg; default for fp32 logits).  The LM-head
// epilogue (fp32 accumulators of O(1) magnitude) keeps the single-FFMA form.
template <int DT, int NB, int NPF, bool XM = (DT == 0)>
__device__ __forceinline__ void mr_batch(const uint4 (&v)[NB], float k2, float& m, float& r) {
  constexpr int N = Traits<DT>::N;
  float mc;
  if constexpr (DT == 1) {
    uint32_t w = Traits<1>::vmax2(v[0]);
#pragma unroll
    for (int u = 1; u < NB; ++u) w = bmax2_nan(w, Traits<1>::vmax2(v[u]));
    mc = fmax_nan(bf_lo(w), bf_hi(w));
  } else {
    mc = Traits<0>::vmax(v[0]);
#pragma unroll
    for (int u = 1; u < NB; ++u) mc = fmax_nan(mc, Traits<0>::vmax(v[u]));
  }
  const bool rec = !(mc <= m);
  // nothing finite yet and an all -inf batch (legal zero-probability entries, R14): no
  // contribution (the exponent x k2 - m k2 would be -inf + inf = NaN)
  if (!rec && m == -INFINITY) return;
  if (rec) {
    const float sc = (m == -INFINITY) ? 0.f : ex2((m - mc) * k2);
    r = (1.f + r) * sc;
    m = mc;
  }
  const float mk = m * k2;
  if (DT == 0 && rec) {
    float s = 0.f;
    int neq = 0;
#pragma unroll
    for (int u = 0; u < NB; ++u) {
      float f[N];
      Traits<DT>::unpack(v[u], f);
#pragma unroll
      for (int j = 0; j < N; ++j) {
        if (f[j] == m) ++neq;
        else s += ex2(XM ? (f[j] - m) * k2 : fmaf(f[j], k2, -mk));
      }
    }
    r += s + (float)(neq - 1);
    return;
  }
  // fast path: exp2 arguments two at a time (bf16: x k2 - m k2 in one FFMA2; fp32: (x - m) k2,
  // FADD2 + FMUL2, see fwd_arg) and two running sums (FADD2)
  const f32x2 K2 = pk2(k2, k2), NMK = pk2(-mk, -mk), NM = pk2(-m, -m);
  f32x2 acc = pk2(0.f, 0.f);
#pragma unroll
  for (int u = 0; u < NB; ++u) {
    float f[N];
    Traits<DT>::unpack(v[u], f);
#pragma unroll
    for (int j = 0; j < N; j += 2) {
      float e0, e1;
      if constexpr (XM) upk2(fmul2(fadd2(pk2(f[j], f[j + 1]), NM), K2), e0, e1);
      else upk2(ffma2(pk2(f[j], f[j + 1]), K2, NMK), e0, e1);
      acc = fadd2(acc, pk2((j < NPF) ? ex2_poly4(e0) : ex2(e0), (j + 1 < NPF) ? ex2_poly4(e1) : ex2(e1)));
    }
  }
  float s0, s1;
  upk2(acc, s0, s1);
  float s = s0 + s1;
  if (DT == 1 && rec) s -= ex2(fmaf(m, k2, -mk));
  r += s;
}

#ifndef ODPO_PARTIAL_OLD
#define ODPO_PARTIAL_OLD 0
#endif
// A partial chunk (cnv vectors, fewer than a full chunk): a thread with at most half a batch
// of vectors takes them in batches of 2.  One 8-vector batch padded with -inf would spend an
// exp2 on every padding element: for Pythia's 100.6 KB rows (six 16 KB chunks and a 2.3 KB
// one) that was a seventh chunk's worth of MUFU work per row.
template <int DT, int UB, int NPF>
__device__ __forceinline__ void mr_partial(const uint4* sv, int tid, int stride, int cnv, float k2,
                                           float& m, float& r) {
  const uint32_t NI = Traits<DT>::kNegInfWord;
  // this thread's vectors in the chunk; more than half a batch: the padded full batch (the
  // extra max checks of 2-vector batches cost more than the padding's exp2s there; measured)
  const int nr = (cnv - tid + stride - 1) / stride;
  if (ODPO_PARTIAL_OLD || 2 * nr > UB) {
    uint4 w[UB];
#pragma unroll
    for (int u = 0; u < UB; ++u) w[u] = tid + u * stride < cnv ? sv[tid + u * stride] : make_uint4(NI, NI, NI, NI);
    mr_batch<DT, UB, NPF>(w, k2, m, r);
    return;
  }
#pragma unroll
  for (int u = 0; u < UB; u += 2) {
    const int i0 = tid + u * stride;
    if (i0 >= cnv) break;
    const int i1 = i0 + stride;
    uint4 v[2];
    v[0] = sv[i0];
    v[1] = (u + 1 < UB && i1 < cnv) ? sv[i1] : make_uint4(NI, NI, NI, NI);
    mr_batch<DT, 2, NPF>(v, k2, m, r);
  }
}

// warp-level fixed-order (m, r) merge; result valid in lane 0
__device__ __forceinline__ MR warp_merge(MR v, float k2) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    MR o;
    o.m = __shfl_down_sync(kFull, v.m, off);
    o.r = __shfl_down_sync(kFull, v.r, off);
    v = mr_merge(v, o, k2);
  }
  return v;
}

}  // namespace odpo
