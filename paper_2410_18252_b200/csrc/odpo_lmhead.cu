// odpo_lmhead.cu -- NEXT-2, forward part: sequence log-probs straight from the
// LM head, logits never written to HBM (sm_100a, tcgen05 / TMEM / TMA).
//
//   logits[row, v] = invT * <hidden[row, :], W[v, :]>           (the LM head, bf16 x bf16 -> fp32)
//   logp[row]      = logits[row, tok] - logsumexp_v logits[row, v]      (Sec 2.1)
//   S_b            = sum_t mask[b, t] logp[b*T + t]                     (reading R2)
//
// K6a k_lmhead_fwd: persistent, one CTA per SM, warp-specialised; CTA c owns an equal contiguous
// range of the (128-row block, 256-wide vocabulary tile) grid (see Args).  Warp 0 (one lane) streams 128x64 hidden tiles and 256x64 weight
// tiles (bf16, 128-byte swizzle) into a 4-stage shared-memory ring with 2-D TMA; warp 1 (one
// lane) issues tcgen05.mma.cta_group::1.kind::f16 (M=128, N=256, K=16) into one of two TMEM
// accumulators (2 x 256 fp32 columns) and commits stage/accumulator barriers; warps 2..5 drain
// the finished accumulator with tcgen05.ld.32x32b.x32 (TMEM lane = row, so each thread owns one
// row) and fold the 256 logits into the row's online (m, r) state -- the same fp32 log1p-form
// update as the logits path (mr_batch<fp32>) -- while the tensor cores fill the other buffer.
// K6b k_lmhead_merge: per row, the pieces' (m, r, x_tok) in fixed (CTA) order -> logp, lse; per
// sequence, the fixed-order masked sum.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>

#include <mutex>

#include "odpo.h"
#include "odpo_device.cuh"
#include "odpo_engine.cuh"

namespace odpo {
namespace lmh {

#ifndef ODPO_LMH_NOEPI
#define ODPO_LMH_NOEPI 0   // A/B power probe only: the forward's epilogue skips its TMEM reads
#endif
constexpr int BM = 128;            // rows per tile (UMMA M)
constexpr int BN = 256;            // vocabulary per tile (UMMA N)
constexpr int BK = 64;             // hidden elements per stage (128 B = one swizzle row)
constexpr int UK = 16;             // UMMA K for kind::f16
constexpr int STAGES = 4;
constexpr int A_BYTES = BM * BK * 2;   // 16 KB
constexpr int B_BYTES = BN * BK * 2;   // 32 KB
constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int SMEM = STAGES * STAGE_BYTES + 1024;  // + alignment slack (SW128 atoms: 1024 B)
constexpr int THREADS = 192;       // producer, MMA, 4 epilogue warps
constexpr int TMEM_COLS = 2 * BN;  // two fp32 accumulators

// instruction descriptor: D fp32 (bits 4-5 = 1), A/B bf16 (bits 7-9, 10-12 = 1), both K-major,
// N >> 3 at bits 17-22, M >> 4 at bits 24-28
constexpr uint32_t kIdesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BN >> 3) << 17) |
                            ((uint32_t)(BM >> 4) << 24);

// shared-memory matrix descriptor, K-major, 128-byte swizzle: start address >> 4, LBO = 1
// (unused for swizzled K-major), SBO = 1024 B between 8-row atoms, version 1, layout 2
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | (1ull << 16) | ((uint64_t)(1024 >> 4) << 32) |
         (1ull << 46) | (2ull << 61);
}

__device__ __forceinline__ void tma_2d(uint32_t dst, const CUtensorMap* map, int c0, int c1,
                                       uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
      "l"(map), "r"(c0), "r"(c1), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void mma_bf16(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(kIdesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void mma_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
               : "memory");
}
__device__ __forceinline__ void tm_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr)
      : "memory");
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// Work split: the nrb x NT grid of (128-row block, 256-wide vocabulary tile) tiles, ordered in
// groups of G row blocks, vocabulary-major inside a group, and dealt round-robin to the
// persistent CTAs (tile i*grid + c to CTA c) -- in this single-CTA kernel; the CTA-pair kernels
// below claim tiles dynamically (see "Dynamic tile order").  The ~grid tiles in flight at any moment span G
// row blocks x grid/G vocabulary tiles, so their hidden blocks and weight tiles are shared
// through L2.  Every tile writes its rows' partial (m, r) -- the merge order (vocabulary tile
// order) does not depend on the CTA mapping.
struct Args {
  int64_t R, d, V;     // rows, hidden size, vocabulary
  int64_t nrb, NT;     // row blocks, vocabulary tiles per row block
  int64_t Ttot;        // nrb * NT
  int G;               // row blocks per raster group
  float invT;
  const int32_t* tokens;  // [R]
  const uint8_t* mask;    // [R]
  float2* parts;          // [R][NT] (m, r) of each vocabulary tile
  float* xtok;            // [R] the sampled token's logit (written by the tile holding it)
  int64_t nrb2;           // 2-CTA kernel: 256-row blocks (one per CTA pair)
  // GRAD epilogue (backward): G[row, v] = row_scale[row] (softmax - onehot), bf16 [R][ldg]
  const float* row_lse;   // [R] logsumexp of invT * logits (natural log), from the forward
  const float* row_scale; // [R] coef_b * mask (d loss / d logits = row_scale * G)
  __nv_bfloat16* gout;   // [R][ldg]
  int64_t ldg;
  // LOGITS epilogue (the chunked learner step): the bf16 logits into gout, and per (row, tile)
  // the vocabulary-parallel partial (m, log1p r, x_tok, owns tok) of those bf16 values, [NT][R]
  float4* parts4;
  unsigned long long* tile_ctr;  // CTA-pair kernels: the dynamic tile counter (zeroed per launch)
};

__device__ __forceinline__ void tile_coords(const Args& a, int64_t t, int64_t& rb, int64_t& n) {
  const int64_t grp = t / ((int64_t)a.G * a.NT);
  const int64_t r0 = grp * a.G;
  const int64_t gg = min((int64_t)a.G, a.nrb - r0);
  const int64_t idx = t - grp * (int64_t)a.G * a.NT;
  n = idx / gg;
  rb = r0 + idx % gg;
}

// ---------------------------------------------------------------- K6a: GEMM + online LSE
__global__ void __launch_bounds__(THREADS, 1)
    k_lmhead_fwd(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB,
                 Args a) {
  extern __shared__ uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t full[STAGES], empty[STAGES], tfull[2], tempty[2];
  __shared__ uint32_t tmem_sh;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t base = (smem_u32(smem_raw) + 1023u) & ~1023u;  // SW128 atoms need 1024 B
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], 4);
    }
    mbar_fence_init();
    asm volatile("prefetch.tensormap [%0];" ::"l"(&mapA) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&mapB) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&tmem_sh)),
                 "n"(TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_sh;
  const uint32_t full_s = smem_u32(full), empty_s = smem_u32(empty);
  const uint32_t tfull_s = smem_u32(tfull), tempty_s = smem_u32(tempty);
  const int nkb = (int)(a.d / BK);

  if (warp == 0) {
    if (lane == 0) {
      // ================= TMA producer
      int st = 0;
      uint32_t ph = 0;
      for (int64_t t = blockIdx.x; t < a.Ttot; t += gridDim.x) {
        int64_t rb, nt;
        tile_coords(a, t, rb, nt);
        const int vrow = (int)(nt * BN);
        {
          for (int kb = 0; kb < nkb; ++kb) {
            mbar_wait(empty_s + 8 * st, ph ^ 1u);
            const uint32_t sa = base + (uint32_t)(st * STAGE_BYTES);
            mbar_arrive_tx(full_s + 8 * st, STAGE_BYTES);
            tma_2d(sa, &mapA, kb * BK, (int)(rb * BM), full_s + 8 * st);
            tma_2d(sa + A_BYTES, &mapB, kb * BK, vrow, full_s + 8 * st);
            if (++st == STAGES) { st = 0; ph ^= 1u; }
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ================= MMA issuer (one thread)
      int st = 0;
      uint32_t ph = 0;
      int acc = 0;
      uint32_t aph = 0;
      for (int64_t t = blockIdx.x; t < a.Ttot; t += gridDim.x) {
        {
          mbar_wait(tempty_s + 8 * acc, aph ^ 1u);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint32_t td = tmem + (uint32_t)(acc * BN);
          for (int kb = 0; kb < nkb; ++kb) {
            mbar_wait(full_s + 8 * st, ph);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const uint32_t sa = base + (uint32_t)(st * STAGE_BYTES);
            const uint64_t da = sdesc(sa), db = sdesc(sa + A_BYTES);
#pragma unroll
            for (int k = 0; k < BK / UK; ++k)  // +32 bytes along K inside the swizzle atom
              mma_bf16(td, da + (uint64_t)(2 * k), db + (uint64_t)(2 * k), (kb | k) != 0);
            mma_commit(empty_s + 8 * st);  // frees the stage once these MMAs have read it
            if (++st == STAGES) { st = 0; ph ^= 1u; }
          }
          mma_commit(tfull_s + 8 * acc);   // accumulator complete
          if (++acc == 2) { acc = 0; aph ^= 1u; }
        }
      }
    }
  } else {
    // ================= epilogue warps 2..5: TMEM lane quadrant = warp % 4, one row per thread
    const int q = warp & 3;
    const uint32_t lane_base = (uint32_t)(32 * q) << 16;
    const float k2 = a.invT * kLog2e;
    int acc = 0;
    uint32_t aph = 0;
    for (int64_t t = blockIdx.x; t < a.Ttot; t += gridDim.x) {
      int64_t rb, n;
      tile_coords(a, t, rb, n);
      const int64_t row = rb * BM + 32 * q + lane;
      const bool live = row < a.R;
      const int tok = live ? a.tokens[row] : -1;
      MR s{-INFINITY, 0.f};
      mbar_wait(tfull_s + 8 * acc, aph);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const int64_t c0 = n * BN;
#pragma unroll 1
      for (int c = 0; c < BN / 32; ++c) {
        uint32_t r[32];
        tm_ld32(tmem + lane_base + (uint32_t)(acc * BN + c * 32), r);
        const int64_t cb = c0 + 32 * c;  // first vocabulary index of these 32 columns
        if (cb >= a.V) break;
        if (cb + 32 > a.V) {
#pragma unroll
          for (int j = 0; j < 32; ++j)
            if (cb + j >= a.V) r[j] = Traits<0>::kNegInfWord;
        }
        if (live && tok >= cb && tok < cb + 32) {
          float x = 0.f;
#pragma unroll
          for (int j = 0; j < 32; ++j)
            if (tok == cb + j) x = __uint_as_float(r[j]);
          a.xtok[row] = x;
        }
        uint4 v[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) v[j] = make_uint4(r[4 * j], r[4 * j + 1], r[4 * j + 2], r[4 * j + 3]);
        mr_batch<0, 8, 0, false>(v, k2, s.m, s.r);
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(tempty_s + 8 * acc);
      if (++acc == 2) { acc = 0; aph ^= 1u; }
      if (live) a.parts[row * a.NT + n] = make_float2(s.m, s.r);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(TMEM_COLS)
                 : "memory");
  }
}

// ---------------------------------------------------------------- K6a2: the same, on CTA pairs
// Thread-block clusters of 2 CTAs on the two SMs of a TPC run tcgen05.mma.cta_group::2 with
// M = 256, N = 256: each CTA stages its own 128 hidden rows and HALF of the 256 weight rows of
// the tile, so a CTA's tensor core reads 128 + 128 operand rows per K step instead of 128 + 256
// (the 1-CTA kernel is bound by those shared-memory operand reads: ncu sm__mem_tensor 94%).
// The leader (rank 0) issues the MMAs and commits with a 2-CTA multicast to both CTAs' stage /
// accumulator barriers; both CTAs' TMA loads complete on the leader's stage barrier
// (.cta_group::2 TMA, peer bit cleared), which expects both CTAs' bytes; the epilogue warps of
// both CTAs release the leader's accumulator barrier (remote arrive).  Accumulator rows 0-127 sit
// in the leader's TMEM, 128-255 in the peer's, so each CTA's epilogue drains its own rows.
constexpr int STAGES2 = 6;
constexpr int HALF_B = (BN / 2) * BK * 2;          // 16 KB: this CTA's half of the weight tile
constexpr int STAGE2_BYTES = A_BYTES + HALF_B;     // 32 KB per CTA per stage
constexpr int SMEM2 = STAGES2 * STAGE2_BYTES + 1024;
constexpr uint32_t kIdesc2 = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BN >> 3) << 17) |
                             ((uint32_t)(256 >> 4) << 24);
constexpr uint32_t kPeerMask = 0xFEFFFFFFu;  // shared::cluster address -> the leader CTA's copy

__device__ __forceinline__ void tma_2d_pair(uint32_t dst, const CUtensorMap* map, int c0, int c1,
                                            uint32_t bar_leader) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
      "l"(map), "r"(c0), "r"(c1), "r"(bar_leader)
      : "memory");
}
__device__ __forceinline__ void mma_bf16_pair(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(kIdesc2), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void mma_commit_pair(uint32_t bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(bar),
      "h"((uint16_t)3)
      : "memory");
}

__device__ __forceinline__ void tile_coords2(const Args& a, int64_t t, int64_t& rb2, int64_t& n) {
  const int64_t grp = t / ((int64_t)a.G * a.NT);
  const int64_t r0 = grp * a.G;
  const int64_t gg = min((int64_t)a.G, a.nrb2 - r0);
  const int64_t idx = t - grp * (int64_t)a.G * a.NT;
  n = idx / gg;
  rb2 = r0 + idx % gg;
}

// Dynamic tile order of the CTA-pair kernels.  With tiles dealt round-robin to the persistent
// pairs, a pair that runs 1% slower falls tens of tiles behind by the end of a LLaMA-size call:
// the pairs that should share a hidden block or a weight tile through L2 drift apart in K and
// fetch it again from HBM (ncu: 170-400 GB of DRAM reads per LLaMA-head forward against 62 GB
// for cuBLAS's GEMM), which at the 1000 W cap costs clock (profiles/r02/next2/power_dram.md).
// Instead the leader's producer claims the next tile from a global counter, so the tiles in
// flight are always a contiguous window of the raster order, and hands the index to every other
// role of the pair through a small ring in shared memory (the peer's copy written over DSMEM):
// qfull[q] (1 arrival: the leader's producer) in each CTA, qempty[q] in the leader (kTQCons
// arrivals: the leader's MMA thread and 4 epilogue warps, the peer's producer and 4 epilogue
// warps).  Index -1 ends the sequence.  ODPO_LMH_STATIC=1 (A/B only) keeps the round-robin deal.
#ifndef ODPO_LMH_STATIC
#define ODPO_LMH_STATIC 0
#endif
constexpr bool kStaticTiles = ODPO_LMH_STATIC != 0;
constexpr int kTQ = 8;
// Host: the counter to use for a launch of `tiles` tiles over `clusters` pairs, or nullptr for
// the round-robin deal.  The drift that the dynamic order removes grows with the tiles each pair
// runs; below ~512 per pair (the Pythia head: 283) the round-robin deal measured 2% faster (the
// ring hand-off costs more than the drift), above it (the LLaMA head: 3466) the dynamic order
// cuts DRAM reads 2x and runs 9-13% faster at the power cap (profiles/r02/next2/dyn/).
#ifndef ODPO_DYN_MIN
#define ODPO_DYN_MIN 512   // tiles per pair from which the dynamic order is used (A/B knob)
#endif
static unsigned long long* tile_mode(unsigned long long* ctr, int64_t tiles, int clusters) {
  if (kStaticTiles || clusters <= 0 || tiles < (int64_t)ODPO_DYN_MIN * clusters) return nullptr;
  return ctr;
}
// Host: pair-blocks (256 rows) per raster group of the head kernels: ~40 MB of hidden rows kept
// for reuse across the group's pass over the weight (measured with the dynamic order: LLaMA
// d = 4096 best at 12-24 pair-blocks, Pythia d = 2560 at 32), clamped to [8, 32].
static int lmh_group(int64_t d) {
  int64_t g = (40ll << 20) / (512 * d);
  if (g < 8) g = 8;
  if (g > 32) g = 32;
  return (int)g;
}
constexpr int kTQCons = 10;
struct TileRing {
  uint32_t full_s, empty_leader;   // this CTA's qfull, the leader's qempty (cluster address)
  long long* tq;
  uint32_t tq_peer;                // the peer's tq (cluster address; leader only)
};
// The leader's producer: publish the i-th tile of this pair (claimed one tile ahead, so the
// counter's round trip overlaps the previous tile's loads) to both CTAs.
__device__ __forceinline__ int64_t tile_publish(const TileRing& R, int i, long long t,
                                                uint32_t empty_local) {
  const int q = i % kTQ;
  const uint32_t ph = (uint32_t)((i / kTQ) & 1);
  mbar_wait(empty_local + 8 * q, ph ^ 1u);
  R.tq[q] = t;
  st_cl_u64(R.tq_peer + 8 * q, (uint64_t)t);
  asm volatile("fence.acq_rel.cluster;" ::: "memory");
  mbar_arrive(R.full_s + 8 * q);
  mbar_arrive_cl(mapa(R.full_s + 8 * q, 1));
  return (int64_t)t;
}
// Every other role: read the i-th tile index (one thread), release the slot.  The release is
// a relaxed arrive: the slot's value has been consumed (the caller's branch on it) before the
// arrive can be performed, and a release fence here would wait for this thread's own
// outstanding stores (the epilogue's) at every tile.
__device__ __forceinline__ void tile_release(const TileRing& R, int i) {
  const int q = i % kTQ;
  asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(R.empty_leader + 8 * q)
               : "memory");
}
__device__ __forceinline__ int64_t tile_read(const TileRing& R, int i) {
  const int q = i % kTQ;
  const uint32_t ph = (uint32_t)((i / kTQ) & 1);
  mbar_wait_cl(R.full_s + 8 * q, ph);
  long long t;
  asm volatile("ld.volatile.shared.s64 %0, [%1];" : "=l"(t) : "r"(smem_u32(R.tq + q)) : "memory");
  // consume the value before releasing the slot (the branch orders the load before the arrive)
  if (t < -1) __trap();
  tile_release(R, i);
  return (int64_t)t;
}

// Epilogue kinds.  LSE: fold each tile into the rows' online logsumexp partials (forward).
// GRAD: the same GEMM tiles, but the epilogue writes the row's gradient with respect to the
// logits, G = row_scale (softmax(invT x) - onehot) in bf16, instead of folding an online
// logsumexp (the backward recomputes the logits a row chunk at a time; see odpo_lmhead_grad).
// LOGITS: store the logits in bf16 AND fold the stored (rounded) values into one partial per
// (row, tile) in the vocabulary-parallel format, so the chunked learner step's loss needs no
// forward pass over the logits (odpo_lmhead_dpo_step).
constexpr int kEpiLse = 0, kEpiGrad = 1, kEpiLogits = 2;
template <int EPI>
__global__ void __launch_bounds__(THREADS, 1)
    k_lmhead_fwd2(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB,
                  Args a) {
  constexpr bool GRAD = EPI == kEpiGrad, LOGITS = EPI == kEpiLogits;
  extern __shared__ uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t full[STAGES2], empty[STAGES2], tfull[2], tempty[2];
  __shared__ __align__(8) uint64_t qfull[kTQ], qempty[kTQ];
  __shared__ __align__(8) long long tq[kTQ];
  // GRAD / LOGITS epilogue: per epilogue warp a 32-row x 64-byte staging tile (rows padded to 80 B)
  __shared__ __align__(16) uint4 gstage[4][(GRAD || LOGITS) ? 32 * 5 : 1];
  __shared__ uint32_t tmem_sh;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  const uint32_t base = (smem_u32(smem_raw) + 1023u) & ~1023u;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES2; ++s) {
      mbar_init(&full[s], 1);    // the leader's producer (expect_tx of both CTAs' bytes)
      mbar_init(&empty[s], 1);   // the leader's multicast MMA commit
    }
    for (int q = 0; q < kTQ; ++q) {
      mbar_init(&qfull[q], 1);         // the leader's producer (tile index published)
      mbar_init(&qempty[q], kTQCons);  // every reader of the pair (leader's copy is the one used)
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull[s], 1);   // multicast commit
      mbar_init(&tempty[s], 8);  // 4 epilogue warps x 2 CTAs (leader's copy is the one used)
    }
    mbar_fence_init();
    asm volatile("prefetch.tensormap [%0];" ::"l"(&mapA) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&mapB) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&tmem_sh)),
                 "n"(TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  cluster_sync_all();  // both CTAs' barriers initialised and TMEM allocated
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_sh;
  const uint32_t full_s = smem_u32(full), empty_s = smem_u32(empty);
  const uint32_t tfull_s = smem_u32(tfull), tempty_s = smem_u32(tempty);
  TileRing R;
  R.full_s = smem_u32(qfull);
  R.empty_leader = mapa(smem_u32(qempty), 0);
  R.tq = tq;
  R.tq_peer = mapa(smem_u32(tq), 1);
  const uint32_t qempty_s = smem_u32(qempty);
  const int nkb = (int)(a.d / BK);
  const int64_t cl = blockIdx.x >> 1, ncl = gridDim.x >> 1;
  const int64_t Tt = a.nrb2 * a.NT;
  const bool stat = a.tile_ctr == nullptr;   // round-robin deal (short calls, see tile_mode)

  if (warp == 0) {
    if (lane == 0) {
      // ================= TMA producer (both CTAs): own hidden rows + own half of the weights
      int st = 0;
      uint32_t ph = 0;
      long long nxt = (!stat && leader) ? (long long)atomicAdd(a.tile_ctr, 1ull) : 0;
      for (int i = 0;; ++i) {
        int64_t t;
        if (stat) {
          t = cl + (int64_t)i * ncl < Tt ? cl + (int64_t)i * ncl : (int64_t)-1;
        } else if (leader) {
          t = tile_publish(R, i, nxt < Tt ? nxt : -1, qempty_s);
          if (t >= 0) nxt = (long long)atomicAdd(a.tile_ctr, 1ull);   // used at the next tile
        } else {
          t = tile_read(R, i);
        }
        if (t < 0) break;
        int64_t rb2, nt;
        tile_coords2(a, t, rb2, nt);
        const int arow = (int)(rb2 * 256 + rank * 128);
        const int vrow = (int)(nt * BN + rank * (BN / 2));
        for (int kb = 0; kb < nkb; ++kb) {
          mbar_wait(empty_s + 8 * st, ph ^ 1u);
          const uint32_t sa = base + (uint32_t)(st * STAGE2_BYTES);
          const uint32_t fb = (full_s + 8 * st) & kPeerMask;
          if (leader) mbar_arrive_tx(full_s + 8 * st, 2 * STAGE2_BYTES);
          tma_2d_pair(sa, &mapA, kb * BK, arow, fb);
          tma_2d_pair(sa + A_BYTES, &mapB, kb * BK, vrow, fb);
          if (++st == STAGES2) { st = 0; ph ^= 1u; }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && leader) {
      // ================= MMA issuer (leader CTA, one thread): M = 256 across the pair
      int st = 0;
      uint32_t ph = 0;
      int acc = 0;
      uint32_t aph = 0;
      for (int i = 0;; ++i) {
        const int64_t t = stat ? (cl + (int64_t)i * ncl < Tt ? cl + (int64_t)i * ncl : (int64_t)-1) : tile_read(R, i);
        if (t < 0) break;
        mbar_wait(tempty_s + 8 * acc, aph ^ 1u);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t td = tmem + (uint32_t)(acc * BN);
        for (int kb = 0; kb < nkb; ++kb) {
          mbar_wait(full_s + 8 * st, ph);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint32_t sa = base + (uint32_t)(st * STAGE2_BYTES);
          const uint64_t da = sdesc(sa), db = sdesc(sa + A_BYTES);
#pragma unroll
          for (int k = 0; k < BK / UK; ++k)
            mma_bf16_pair(td, da + (uint64_t)(2 * k), db + (uint64_t)(2 * k), (kb | k) != 0);
          mma_commit_pair(empty_s + 8 * st);  // frees this stage in both CTAs
          if (++st == STAGES2) { st = 0; ph ^= 1u; }
        }
        mma_commit_pair(tfull_s + 8 * acc);   // accumulator complete in both CTAs
        if (++acc == 2) { acc = 0; aph ^= 1u; }
      }
    }
  } else {
    // ================= epilogue warps 2..5 (both CTAs): this CTA's 128 accumulator rows
    const int q = warp & 3;
    const uint32_t lane_base = (uint32_t)(32 * q) << 16;
    const uint32_t tempty_leader = mapa(tempty_s, 0);
    const float k2 = a.invT * kLog2e;
    int acc = 0;
    uint32_t aph = 0;
    for (int i = 0;; ++i) {
      int64_t t;
      if (stat) {
        t = cl + (int64_t)i * ncl < Tt ? cl + (int64_t)i * ncl : (int64_t)-1;
      } else {
        long long v = 0;
        if (lane == 0) v = tile_read(R, i);
        t = __shfl_sync(kFull, v, 0);
      }
      if (t < 0) break;
      int64_t rb2, n;
      tile_coords2(a, t, rb2, n);
      const int64_t row = rb2 * 256 + rank * 128 + 32 * q + lane;
      const bool live = row < a.R;
      const int tok = live ? a.tokens[row] : -1;
      MR s{-INFINITY, 0.f};
      float g_rs = 0.f, g_c = 0.f, xt = 0.f, own = 0.f;
      if (GRAD && live) {
        g_rs = a.row_scale[row];
        g_c = g_rs != 0.f ? a.row_lse[row] * kLog2e : INFINITY;  // p = 2^(acc invT log2e - lse log2e)
      }
      if (GRAD && !live) g_c = INFINITY;
      mbar_wait(tfull_s + 8 * acc, aph);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const int64_t c0 = n * BN;
#pragma unroll 1
      for (int c = 0; c < (ODPO_LMH_NOEPI ? 0 : BN / 32); ++c) {   // NOEPI: A/B power probe only
        uint32_t r[32];
        tm_ld32(tmem + lane_base + (uint32_t)(acc * BN + c * 32), r);
        const int64_t cb = c0 + 32 * c;
        if (cb >= a.V) break;
        if (GRAD) {
          // g_j = row_scale * p_j; at the sampled token row_scale * expm1(log p) (no p - 1
          // cancellation); rows with row_scale 0 (masked, unreferenced) get exact zeros
          // two logits per FFMA2 / FMUL2; rows with row_scale 0 carry g_c = +inf (exact zeros,
          // never 0 * inf: a masked row's lse is not its own)
          uint32_t w[16];
          const f32x2 K2 = pk2(k2, k2), NC = pk2(-g_c, -g_c), RS = pk2(g_rs, g_rs);
#pragma unroll
          for (int j = 0; j < 32; j += 2) {
            float e0, e1, g0, g1;
            upk2(ffma2(pk2(__uint_as_float(r[j]), __uint_as_float(r[j + 1])), K2, NC), e0, e1);
            upk2(fmul2(pk2(ex2(e0), ex2(e1)), RS), g0, g1);
            w[j / 2] = pack_bf16x2(g0, g1);
          }
          if (tok >= cb && tok < cb + 32 && g_rs != 0.f) {
            // the sampled token: row_scale * expm1(log p) (no p - 1 cancellation)
            const int jt = tok - (int)cb;
            float xt = 0.f;
#pragma unroll
            for (int j = 0; j < 32; ++j) xt = j == jt ? __uint_as_float(r[j]) : xt;
            const float gt = g_rs * expm1f(fmaf(xt, a.invT, -a.row_lse[row]));
            const uint32_t hb = pack_bf16x2(gt, 0.f) & 0xFFFFu;
#pragma unroll
            for (int j = 0; j < 16; ++j)
              if (j == jt / 2) w[j] = (jt & 1) ? ((w[j] & 0xFFFFu) | (hb << 16)) : ((w[j] & 0xFFFF0000u) | hb);
          }
          if (cb + 32 <= a.V) {
            // stage the warp's 32 rows x 64 B, then store row-contiguous: each store
            // instruction writes 64 B to each of 8 rows instead of 16 B to each of 32
            uint4* st_w = gstage[q];
#pragma unroll
            for (int k = 0; k < 4; ++k)
              st_w[lane * 5 + k] = make_uint4(w[4 * k], w[4 * k + 1], w[4 * k + 2], w[4 * k + 3]);
            __syncwarp();
            const int64_t row0 = rb2 * 256 + rank * 128 + 32 * q;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const int rr = 8 * k + (lane >> 2), sg = lane & 3;
              if (row0 + rr < a.R) {
                // streaming store: G is consumed by the next GEMM, not by this kernel's tiles,
                // so it must not evict the hidden / weight tiles the CTAs share through L2
                st16_stream(reinterpret_cast<uint4*>(a.gout + (row0 + rr) * a.ldg + cb) + sg,
                            st_w[rr * 5 + sg]);
              }
            }
            __syncwarp();
          } else if (live) {
            unsigned short* d2 = reinterpret_cast<unsigned short*>(a.gout + row * a.ldg + cb);
            for (int j = 0; j < 32 && cb + j < a.V; ++j)
              d2[j] = (unsigned short)((w[j / 2] >> (16 * (j & 1))) & 0xFFFFu);
          }
          continue;
        }
        if (LOGITS) {
          // round to bf16 (the chunk's logits, round-to-nearest-even) and fold exactly the
          // stored values: the loss is the one of the logits tensor the backward reads
          uint32_t w[16];
#pragma unroll
          for (int j = 0; j < 32; j += 2) {
            w[j / 2] = pack_bf16x2(__uint_as_float(r[j]), __uint_as_float(r[j + 1]));
            r[j] = w[j / 2] << 16;
            r[j + 1] = w[j / 2] & 0xFFFF0000u;
          }
          if (cb + 32 <= a.V) {
            uint4* st_w = gstage[q];
#pragma unroll
            for (int k = 0; k < 4; ++k)
              st_w[lane * 5 + k] = make_uint4(w[4 * k], w[4 * k + 1], w[4 * k + 2], w[4 * k + 3]);
            __syncwarp();
            const int64_t row0 = rb2 * 256 + rank * 128 + 32 * q;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const int rr = 8 * k + (lane >> 2), sg = lane & 3;
              if (row0 + rr < a.R)
                st16_stream(reinterpret_cast<uint4*>(a.gout + (row0 + rr) * a.ldg + cb) + sg,
                            st_w[rr * 5 + sg]);
            }
            __syncwarp();
          } else if (live) {
            unsigned short* d2 = reinterpret_cast<unsigned short*>(a.gout + row * a.ldg + cb);
            for (int j = 0; j < 32 && cb + j < a.V; ++j)
              d2[j] = (unsigned short)((w[j / 2] >> (16 * (j & 1))) & 0xFFFFu);
          }
        }
        if (cb + 32 > a.V) {
#pragma unroll
          for (int j = 0; j < 32; ++j)
            if (cb + j >= a.V) r[j] = Traits<0>::kNegInfWord;
        }
        if (live && tok >= cb && tok < cb + 32) {
          float x = 0.f;
#pragma unroll
          for (int j = 0; j < 32; ++j)
            if (tok == cb + j) x = __uint_as_float(r[j]);
          if (LOGITS) {
            xt = x;
            own = 1.f;
          } else {
            a.xtok[row] = x;
          }
        }
        uint4 v[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) v[j] = make_uint4(r[4 * j], r[4 * j + 1], r[4 * j + 2], r[4 * j + 3]);
        mr_batch<0, 8, 0, false>(v, k2, s.m, s.r);
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive_cl(tempty_leader + 8 * acc);
      if (++acc == 2) { acc = 0; aph ^= 1u; }
      if (EPI == kEpiLse && live) a.parts[row * a.NT + n] = make_float2(s.m, s.r);
      if (LOGITS && live) a.parts4[n * a.R + row] = make_float4(s.m, log1pf(s.r), xt, own);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  cluster_sync_all();  // no CTA frees TMEM (or exits) while its peer can still touch it
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(TMEM_COLS)
                 : "memory");
  }
}

// ---------------------------------------------------------------- K6d: TN GEMM on CTA pairs
// The two backward GEMMs of NEXT-2 (dhidden = G W, dweight = G^T H) as one hand-written kernel:
//   C[M, N] (fp32, row-major, ldc) = (acc ? C : 0) + A[M, K] B[N, K]^T,   A, B bf16 K-major.
// Same machinery as k_lmhead_fwd2: thread-block clusters of 2 CTAs, tcgen05.mma.cta_group::2
// (M = 256 across the pair, N = 256, K = 16), operands staged by 2-D TMA (128-byte swizzle) into a
// 6-stage ring, fp32 accumulators double-buffered in TMEM; the epilogue warps drain each
// accumulator with tcgen05.ld (one row per thread), stage 32 x 32 blocks in shared memory and
// store (or add into) C row-contiguously.  Every output element is written by exactly one
// thread in a fixed K order: deterministic, no atomics.  M/N/K tails: TMA zero-fills the
// out-of-range parts of a box; stores are masked.
struct GemmArgs {
  int64_t M, N, K;
  float* C;           // fp32 output (out_bf16 = 0)
  __nv_bfloat16* Cb;  // bf16 output, round-to-nearest-even (out_bf16 = 1; acc must be 0)
  int out_bf16;
  int64_t ldc;
  int64_t nmb2, nnb;  // 256-row blocks (one per CTA pair), 256-column blocks
  int G;              // row blocks per raster group
  int acc;            // 1: C += A B^T
  unsigned long long* tile_ctr;  // the dynamic tile counter (zeroed per launch)
};

__device__ __forceinline__ void gemm_coords(const GemmArgs& g, int64_t t, int64_t& mb, int64_t& nb) {
  const int64_t grp = t / ((int64_t)g.G * g.nnb);
  const int64_t r0 = grp * g.G;
  const int64_t gg = min((int64_t)g.G, g.nmb2 - r0);
  const int64_t idx = t - grp * (int64_t)g.G * g.nnb;
  nb = idx / gg;
  mb = r0 + idx % gg;
}

constexpr int kCPitch = 36;  // staging row pitch (floats): 16-byte rows, conflict-free float4 use

// MN-major operands (A_MN / B_MN): the operand's M (or N) index is the contiguous one in memory
// -- G read as G^T for dweight, W and H read as they are stored -- so no transposed copy is made.
// TMA boxes of 64 (MN, 128 B) x 64 (K) with 128-byte swizzle land as 8 K-row groups of 1024 B;
// a CTA's 128 MN rows are two such boxes 8 KB apart.  UMMA canonical MN-major SW128 layout:
// LBO = 8192 B between 64-element MN blocks, SBO = 1024 B between 8-row K groups, +2048 B per
// K = 16 step; instruction-descriptor bit 15 (A) / 16 (B) = MN-major.
__device__ __forceinline__ uint64_t sdesc_mn(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)(8192 >> 4) << 16) |
         ((uint64_t)(1024 >> 4) << 32) | (1ull << 46) | (2ull << 61);
}
template <bool A_MN, bool B_MN>
__device__ __forceinline__ void mma_gemm_pair(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t acc) {
  constexpr uint32_t idesc = kIdesc2 | (A_MN ? (1u << 15) : 0u) | (B_MN ? (1u << 16) : 0u);
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(acc)
      : "memory");
}

template <bool A_MN, bool B_MN>
__global__ void __launch_bounds__(THREADS, 1)
    k_gemm_tn2(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB,
               GemmArgs g) {
  extern __shared__ uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t full[STAGES2], empty[STAGES2], tfull[2], tempty[2];
  __shared__ __align__(8) uint64_t qfull[kTQ], qempty[kTQ];
  __shared__ __align__(8) long long tq[kTQ];
  __shared__ __align__(16) float cstage[4][32 * kCPitch];
  __shared__ uint32_t tmem_sh;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  const uint32_t base = (smem_u32(smem_raw) + 1023u) & ~1023u;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES2; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int q = 0; q < kTQ; ++q) {
      mbar_init(&qfull[q], 1);         // the leader's producer (tile index published)
      mbar_init(&qempty[q], kTQCons);  // every reader of the pair (leader's copy is the one used)
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], 8);
    }
    mbar_fence_init();
    asm volatile("prefetch.tensormap [%0];" ::"l"(&mapA) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&mapB) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&tmem_sh)),
                 "n"(TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  cluster_sync_all();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_sh;
  const uint32_t full_s = smem_u32(full), empty_s = smem_u32(empty);
  const uint32_t tfull_s = smem_u32(tfull), tempty_s = smem_u32(tempty);
  TileRing R;
  R.full_s = smem_u32(qfull);
  R.empty_leader = mapa(smem_u32(qempty), 0);
  R.tq = tq;
  R.tq_peer = mapa(smem_u32(tq), 1);
  const uint32_t qempty_s = smem_u32(qempty);
  const int nkb = (int)((g.K + BK - 1) / BK);
  const int64_t cl = blockIdx.x >> 1, ncl = gridDim.x >> 1;
  const int64_t Tt = g.nmb2 * g.nnb;
  const bool stat = g.tile_ctr == nullptr;   // round-robin deal (short calls, see tile_mode)

  if (warp == 0) {
    if (lane == 0) {
      int st = 0;
      uint32_t ph = 0;
      long long nxt = (!stat && leader) ? (long long)atomicAdd(g.tile_ctr, 1ull) : 0;
      for (int i = 0;; ++i) {
        int64_t t;
        if (stat) {
          t = cl + (int64_t)i * ncl < Tt ? cl + (int64_t)i * ncl : (int64_t)-1;
        } else if (leader) {
          t = tile_publish(R, i, nxt < Tt ? nxt : -1, qempty_s);
          if (t >= 0) nxt = (long long)atomicAdd(g.tile_ctr, 1ull);   // used at the next tile
        } else {
          t = tile_read(R, i);
        }
        if (t < 0) break;
        int64_t mb, nb;
        gemm_coords(g, t, mb, nb);
        const int arow = (int)(mb * 256 + rank * 128);
        const int brow = (int)(nb * BN + rank * (BN / 2));
        for (int kb = 0; kb < nkb; ++kb) {
          mbar_wait(empty_s + 8 * st, ph ^ 1u);
          const uint32_t sa = base + (uint32_t)(st * STAGE2_BYTES);
          const uint32_t fb = (full_s + 8 * st) & kPeerMask;
          if (leader) mbar_arrive_tx(full_s + 8 * st, 2 * STAGE2_BYTES);
          if (A_MN) {
            tma_2d_pair(sa, &mapA, arow, kb * BK, fb);
            tma_2d_pair(sa + 8192, &mapA, arow + 64, kb * BK, fb);
          } else {
            tma_2d_pair(sa, &mapA, kb * BK, arow, fb);
          }
          if (B_MN) {
            tma_2d_pair(sa + A_BYTES, &mapB, brow, kb * BK, fb);
            tma_2d_pair(sa + A_BYTES + 8192, &mapB, brow + 64, kb * BK, fb);
          } else {
            tma_2d_pair(sa + A_BYTES, &mapB, kb * BK, brow, fb);
          }
          if (++st == STAGES2) { st = 0; ph ^= 1u; }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && leader) {
      int st = 0;
      uint32_t ph = 0;
      int acc = 0;
      uint32_t aph = 0;
      // per K = 16 step: +32 B inside a K-major swizzle atom, +2048 B (16 K rows) MN-major
      constexpr uint64_t stepA = A_MN ? 2048 >> 4 : 2, stepB = B_MN ? 2048 >> 4 : 2;
      for (int i = 0;; ++i) {
        const int64_t t = stat ? (cl + (int64_t)i * ncl < Tt ? cl + (int64_t)i * ncl : (int64_t)-1) : tile_read(R, i);
        if (t < 0) break;
        mbar_wait(tempty_s + 8 * acc, aph ^ 1u);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t td = tmem + (uint32_t)(acc * BN);
        for (int kb = 0; kb < nkb; ++kb) {
          mbar_wait(full_s + 8 * st, ph);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint32_t sa = base + (uint32_t)(st * STAGE2_BYTES);
          const uint64_t da = A_MN ? sdesc_mn(sa) : sdesc(sa);
          const uint64_t db = B_MN ? sdesc_mn(sa + A_BYTES) : sdesc(sa + A_BYTES);
#pragma unroll
          for (int k = 0; k < BK / UK; ++k)
            mma_gemm_pair<A_MN, B_MN>(td, da + stepA * k, db + stepB * k, (kb | k) != 0);
          mma_commit_pair(empty_s + 8 * st);
          if (++st == STAGES2) { st = 0; ph ^= 1u; }
        }
        mma_commit_pair(tfull_s + 8 * acc);
        if (++acc == 2) { acc = 0; aph ^= 1u; }
      }
    }
  } else {
    const int q = warp & 3;
    const uint32_t lane_base = (uint32_t)(32 * q) << 16;
    const uint32_t tempty_leader = mapa(tempty_s, 0);
    float* stg = cstage[q];
    int acc = 0;
    uint32_t aph = 0;
    for (int i = 0;; ++i) {
      int64_t t;
      if (stat) {
        t = cl + (int64_t)i * ncl < Tt ? cl + (int64_t)i * ncl : (int64_t)-1;
      } else {
        long long v = 0;
        if (lane == 0) v = tile_read(R, i);
        t = __shfl_sync(kFull, v, 0);
      }
      if (t < 0) break;
      int64_t mb, nb;
      gemm_coords(g, t, mb, nb);
      const int64_t row0 = mb * 256 + rank * 128 + 32 * q;
      mbar_wait(tfull_s + 8 * acc, aph);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll 1
      for (int c = 0; c < BN / 32; ++c) {
        uint32_t r[32];
        tm_ld32(tmem + lane_base + (uint32_t)(acc * BN + c * 32), r);
        const int64_t cb = nb * BN + 32 * c;
        if (cb >= g.N) break;
#pragma unroll
        for (int k = 0; k < 8; ++k)
          *reinterpret_cast<float4*>(stg + lane * kCPitch + 4 * k) =
              make_float4(__uint_as_float(r[4 * k]), __uint_as_float(r[4 * k + 1]),
                          __uint_as_float(r[4 * k + 2]), __uint_as_float(r[4 * k + 3]));
        __syncwarp();
        const int sg = lane & 7;
        const int64_t col = cb + 4 * sg;
        // C += A B^T: the 8 passes' old values are loaded together first (the stores below
        // could alias them, so the compiler would otherwise serialise one HBM round trip per
        // pass and the epilogue, not the tensor cores, would set the pace)
        float4 old[8];
        if (g.acc && !g.out_bf16 && col + 4 <= g.N) {
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const int64_t row = row0 + 4 * k + (lane >> 3);
            old[k] = row < g.M ? __ldcs(reinterpret_cast<const float4*>(g.C + row * g.ldc + col))
                               : make_float4(0.f, 0.f, 0.f, 0.f);
          }
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) {  // 8 lanes x 16 B per row: 4 rows per pass
          const int rr = 4 * k + (lane >> 3);
          const int64_t row = row0 + rr;
          if (row < g.M && col < g.N && g.out_bf16) {
            // bf16 output (the chunked learner step's logits): 4 values = 8 bytes per lane
            const float4 v = *reinterpret_cast<const float4*>(stg + rr * kCPitch + 4 * sg);
            __nv_bfloat16* dst = g.Cb + row * g.ldc + col;
            if (col + 4 <= g.N) {
              *reinterpret_cast<uint2*>(dst) = make_uint2(pack_bf16x2(v.x, v.y), pack_bf16x2(v.z, v.w));
            } else {
              const float vv[4] = {v.x, v.y, v.z, v.w};
              for (int e = 0; col + e < g.N; ++e)
                reinterpret_cast<unsigned short*>(dst)[e] = (unsigned short)(pack_bf16x2(vv[e], 0.f) & 0xFFFFu);
            }
          } else if (row < g.M && col < g.N) {
            float4 v = *reinterpret_cast<const float4*>(stg + rr * kCPitch + 4 * sg);
            float* dst = g.C + row * g.ldc + col;
            if (col + 4 <= g.N) {
              if (g.acc) {
                v.x += old[k].x; v.y += old[k].y; v.z += old[k].z; v.w += old[k].w;
              }
              *reinterpret_cast<float4*>(dst) = v;
            } else {
              const float vv[4] = {v.x, v.y, v.z, v.w};
              for (int e = 0; col + e < g.N; ++e) dst[e] = g.acc ? dst[e] + vv[e] : vv[e];
            }
          }
        }
        __syncwarp();
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive_cl(tempty_leader + 8 * acc);
      if (++acc == 2) { acc = 0; aph ^= 1u; }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  cluster_sync_all();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(TMEM_COLS)
                 : "memory");
  }
}

// bf16 transpose dst[c][r] = src[r][c] in 64 x 64 tiles (ODPO_GEMM_KB: the K-major copies of
// W and of a hidden chunk, for comparing the MN-major operand path against K-major B operands).
__global__ void __launch_bounds__(256) k_transpose_bf16(const unsigned short* __restrict__ src,
                                                         int64_t rows, int64_t cols, int64_t lds,
                                                         unsigned short* __restrict__ dst,
                                                         int64_t ldd) {
  __shared__ unsigned short tile[64][66];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int64_t r0 = (int64_t)blockIdx.y * 64, c0 = (int64_t)blockIdx.x * 64;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int r = ty + 8 * i;
    const int64_t gr = r0 + r, gc = c0 + 2 * tx;
    tile[r][2 * tx] = (gr < rows && gc < cols) ? src[gr * lds + gc] : (unsigned short)0;
    tile[r][2 * tx + 1] = (gr < rows && gc + 1 < cols) ? src[gr * lds + gc + 1] : (unsigned short)0;
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int c = ty + 8 * i;
    const int64_t gc = c0 + c, gr = r0 + 2 * tx;
    if (gc >= cols) continue;
    if (gr < rows) dst[gc * ldd + gr] = tile[2 * tx][c];
    if (gr + 1 < rows) dst[gc * ldd + gr + 1] = tile[2 * tx + 1][c];
  }
}

// ---------------------------------------------------------------- K6b: merge, K6c: sequence sums
// K6b: one warp per row: lane l merges vocabulary tiles l, l+32, ... in order, then the fixed
// shfl_down tree; lane 0 forms logp and lse (the logits path's arithmetic).
__global__ void __launch_bounds__(256) k_lmhead_merge(Args a, float* tok_logp, float* row_lse,
                                                       uint32_t* status) {
  const int64_t row = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= a.R) return;
  const float k2 = a.invT * kLog2e;
  MR v{-INFINITY, 0.f};
  for (int64_t n = lane; n < a.NT; n += 32) {
    const float2 p = a.parts[row * a.NT + n];
    v = mr_merge(v, MR{p.x, p.y}, k2);
  }
  v = warp_merge(v, k2);
  if (lane != 0) return;
  uint32_t fl = 0;
  float logp = 0.f, lse = 0.f;
  if (a.mask[row]) {
    const float l1p = log1pf(v.r);
    const int tok = a.tokens[row];
    if (tok < 0 || tok >= a.V) {
      fl |= ODPO_FLAG_TOKEN_RANGE;
    } else {
      logp = __fsub_rn(__fmul_rn(__fsub_rn(a.xtok[row], v.m), a.invT), l1p);
      if (!isfinite(logp)) fl |= ODPO_FLAG_NONFINITE_LOGIT;
    }
    if (!isfinite(v.m) || !isfinite(v.r)) fl |= ODPO_FLAG_NONFINITE_LOGIT;
    lse = __fadd_rn(__fmul_rn(v.m, a.invT), l1p);
  }
  tok_logp[row] = logp;
  if (row_lse) row_lse[row] = lse;
  if (fl && status) atomicOr(status, fl);
}

// K6c: one warp per sequence, seq_sum_warp's fixed order.
__global__ void __launch_bounds__(32) k_lmhead_seqsum(const float* tok_logp, const uint8_t* mask,
                                                       int64_t T, float* seq_logp, uint32_t* status) {
  const int64_t b = blockIdx.x;
  double S;
  int n;
  seq_sum_warp(tok_logp + b * T, mask + b * T, T, S, n);
  if (threadIdx.x == 0) {
    seq_logp[b] = n ? (float)S : 0.f;
    if (!n && status) atomicOr(status, ODPO_FLAG_EMPTY_SEQ);
  }
}

// ---------------------------------------------------------------- host
typedef CUresult (*EncodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static EncodeTiled encode_fn() {
  static EncodeTiled fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (EncodeTiled)p;
  }
  return fn;
}
static bool make_map(CUtensorMap* m, const void* base, int64_t rows, int64_t cols, int64_t ld,
                     int box_rows) {
  EncodeTiled enc = encode_fn();
  if (!enc) return false;
  const cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {(cuuint64_t)(ld * 2)};
  const cuuint32_t box[2] = {(cuuint32_t)BK, (cuuint32_t)box_rows};
  const cuuint32_t es[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// MN-major operand map: memory [kdim rows][mndim cols] (row pitch ld elements), 64 x 64 boxes
// (64 MN elements = 128 B inner, 64 K rows), 128-byte swizzle.
static bool make_map_mn(CUtensorMap* m, const void* base, int64_t kdim, int64_t mndim, int64_t ld) {
  EncodeTiled enc = encode_fn();
  if (!enc) return false;
  const cuuint64_t dims[2] = {(cuuint64_t)mndim, (cuuint64_t)kdim};
  const cuuint64_t strides[1] = {(cuuint64_t)(ld * 2)};
  const cuuint32_t box[2] = {64, (cuuint32_t)BK};
  const cuuint32_t es[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

static int sm_count() {
  int dev = 0, n = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n;
}

// Build-time tuning knobs (no environment lookups in the library): ODPO_LMH_1CTA=1 builds the
// single-CTA forward as the default (comparison), ODPO_LMH_G the raster group size.
#ifndef ODPO_LMH_1CTA
#define ODPO_LMH_1CTA 0
#endif
constexpr bool kLmhPair = ODPO_LMH_1CTA == 0;
#ifndef ODPO_LMH_G
#define ODPO_LMH_G 64
#endif
constexpr int kRasterG = ODPO_LMH_G;
#ifndef ODPO_GEMM_G
#define ODPO_GEMM_G 8
#endif
constexpr int kGemmG = ODPO_GEMM_G;   // backward GEMMs: 256-row blocks per raster group (round-robin deal, burst: 8/16/32/64 -> 1636/1723/1751/1802 TF/s; dynamic order at the power cap: 8 best, profiles/r02/next2/gemm_ab/)

}  // namespace lmh
}  // namespace odpo

using namespace odpo;
using namespace odpo::lmh;

// Scratch of odpo_lmhead_grad: G [CR][Vp] bf16, CR = chunk_rows rounded up to 256, Vp = V rounded
// up to 8 (16-byte rows for TMA).
#ifndef ODPO_GEMM_KB
#define ODPO_GEMM_KB 0
#endif
constexpr bool kGemmKB = ODPO_GEMM_KB != 0;   // B operands as K-major copies (W^T, H^T)
static size_t grad_layout(int64_t chunk_rows, int64_t d, int64_t V) {
  const int64_t CR = (chunk_rows + 255) / 256 * 256;
  const int64_t Vp = (V + 7) / 8 * 8;
  size_t n = ((size_t)CR * Vp * 2 + 255) & ~(size_t)255;
  if (kGemmKB) n += (((size_t)d * Vp * 2 + 255) & ~(size_t)255) + (size_t)d * CR * 2;
  return n + 512;   // the last 256 bytes: the CTA-pair kernels' tile counter
}

static void launch_pair(const void* kern, int clusters, cudaStream_t s, void** args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(2 * clusters));
  cfg.blockDim = dim3(THREADS);
  cfg.dynamicSmemBytes = SMEM2;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelExC(&cfg, kern, args);
}

// One GEMM operand as stored in memory: `mn_major` = its M (or N) index is the contiguous one
// (memory [K][MN] with row pitch ld), else K is (memory [MN][K]).
struct Operand {
  const void* p;
  int64_t ld;
  bool mn_major;
};

// C[M, N] (+)= A B^T on the CTA-pair tcgen05 kernel.
template <bool A_MN, bool B_MN>
static odpo_status gemm2(Operand A, Operand B, int64_t M, int64_t N, int64_t K, float* C,
                         int64_t ldc, bool acc, int sms, cudaStream_t s, unsigned long long* ctr,
                         __nv_bfloat16* Cb = nullptr) {
  CUtensorMap mA, mB;
  const bool okA = A_MN ? make_map_mn(&mA, A.p, K, M, A.ld) : make_map(&mA, A.p, M, K, A.ld, BM);
  const bool okB = B_MN ? make_map_mn(&mB, B.p, K, N, B.ld) : make_map(&mB, B.p, N, K, B.ld, BN / 2);
  if (!okA || !okB) return ODPO_ERR_CUDA;
  GemmArgs g{};
  g.M = M; g.N = N; g.K = K; g.C = C; g.ldc = ldc;
  g.Cb = Cb;
  g.out_bf16 = Cb != nullptr;
  g.nmb2 = (M + 255) / 256;
  g.nnb = (N + BN - 1) / BN;
  g.G = kGemmG;
  g.acc = acc ? 1 : 0;
  int clusters = sms / 2;
  if (clusters > g.nmb2 * g.nnb) clusters = (int)(g.nmb2 * g.nnb);
  // the backward GEMMs take the dynamic order at every size (few, long-K tiles: measured with
  // 8-row-block raster groups, LLaMA-head grad 310.8 -> 298.8-300.1 ms, profiles/r02/next2/gemm_ab/)
  g.tile_ctr = kStaticTiles ? nullptr : ctr;
  if (g.tile_ctr && cudaMemsetAsync(g.tile_ctr, 0, sizeof(unsigned long long), s) != cudaSuccess)
    return ODPO_ERR_CUDA;
  void* args[] = {&mA, &mB, &g};
  launch_pair((const void*)k_gemm_tn2<A_MN, B_MN>, clusters, s, args);
  return cudaGetLastError() == cudaSuccess ? ODPO_OK : ODPO_ERR_CUDA;
}

extern "C" {

size_t odpo_lmhead_workspace_bytes(int64_t B, int64_t T, int64_t V) {
  if (B <= 0 || T <= 0 || V <= 0) return 0;
  const int64_t R = B * T;
  const int64_t NT = (V + BN - 1) / BN;
  // per row: NT (m, r) partials, the sampled logit, and an fp32 log-prob scratch
  return (size_t)R * (size_t)NT * sizeof(float2) + (size_t)R * 8 + 512;   // last 256: tile counter
}

odpo_status odpo_lmhead_seq_logprobs(const void* hidden, const void* weight, int64_t B, int64_t T,
                                     int64_t d, int64_t V, const int32_t* tokens,
                                     const uint8_t* mask, float inv_temperature, float* tok_logp,
                                     float* row_lse, float* seq_logp, uint32_t* status,
                                     void* workspace, size_t workspace_bytes, void* stream) {
  if (!hidden || !weight || !tokens || !mask || !seq_logp) return ODPO_ERR_INVALID_ARG;
  if (B <= 0 || T <= 0 || V <= 0 || d <= 0) return ODPO_ERR_INVALID_ARG;
  if (!(isfinite(inv_temperature) && inv_temperature > 0.f)) return ODPO_ERR_INVALID_ARG;
  if (d % BK) return ODPO_ERR_UNSUPPORTED;
  if (((uintptr_t)hidden & 15u) || ((uintptr_t)weight & 15u)) return ODPO_ERR_ALIGNMENT;
  const int64_t R = B * T;
  if (R > (int64_t)INT32_MAX || V > (int64_t)INT32_MAX || d > (1 << 20)) return ODPO_ERR_UNSUPPORTED;
  if (!workspace || workspace_bytes < odpo_lmhead_workspace_bytes(B, T, V)) return ODPO_ERR_WORKSPACE;
  const bool pair = kLmhPair;
  CUtensorMap mA, mB;
  if (!make_map(&mA, hidden, R, d, d, BM) || !make_map(&mB, weight, V, d, d, pair ? BN / 2 : BN))
    return ODPO_ERR_CUDA;
  // kernel attributes are per device: set them once for each device this process uses
  static std::once_flag attr_once[128];
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 128) return ODPO_ERR_UNSUPPORTED;
  std::call_once(attr_once[dev], []() {
    cudaFuncSetAttribute(k_lmhead_fwd, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
    cudaFuncSetAttribute(k_lmhead_fwd2<kEpiLse>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM2);
    cudaFuncSetAttribute(k_lmhead_fwd2<kEpiGrad>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM2);
  });
  const int sms = sm_count();
  Args a;
  a.R = R; a.d = d; a.V = V;
  a.nrb = (R + BM - 1) / BM;
  a.NT = (V + BN - 1) / BN;
  a.Ttot = a.nrb * a.NT;
  a.G = kRasterG;
  a.invT = inv_temperature;
  a.tokens = tokens; a.mask = mask;
  a.parts = reinterpret_cast<float2*>(workspace);
  a.xtok = reinterpret_cast<float*>(reinterpret_cast<char*>(workspace) + (size_t)R * a.NT * sizeof(float2));
  float* tlp = tok_logp ? tok_logp : a.xtok + R;  // log-prob scratch when not requested
  cudaStream_t s = (cudaStream_t)stream;
  if (pair) {
    a.nrb2 = (R + 255) / 256;
    a.G = lmh_group(d);
    const int64_t t2 = a.nrb2 * a.NT;
    int clusters = sms / 2;
    if (clusters > t2) clusters = (int)t2;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(2 * clusters));
    cfg.blockDim = dim3(THREADS);
    cfg.dynamicSmemBytes = SMEM2;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    a.tile_ctr = tile_mode(reinterpret_cast<unsigned long long*>(
                               reinterpret_cast<char*>(workspace) + odpo_lmhead_workspace_bytes(B, T, V) - 256),
                           t2, clusters);
    if (a.tile_ctr && cudaMemsetAsync(a.tile_ctr, 0, sizeof(unsigned long long), s) != cudaSuccess)
      return ODPO_ERR_CUDA;
    cudaLaunchKernelEx(&cfg, k_lmhead_fwd2<kEpiLse>, mA, mB, a);
  } else {
    const int grid = (int)(a.Ttot < sms ? a.Ttot : sms);
    k_lmhead_fwd<<<grid, THREADS, SMEM, s>>>(mA, mB, a);
  }
  if (cudaGetLastError() != cudaSuccess) return ODPO_ERR_CUDA;
  k_lmhead_merge<<<(unsigned)((R + 7) / 8), 256, 0, s>>>(a, tlp, row_lse, status);
  if (cudaGetLastError() != cudaSuccess) return ODPO_ERR_CUDA;
  k_lmhead_seqsum<<<(unsigned)B, 32, 0, s>>>(tlp, mask, T, seq_logp, status);
  return cudaGetLastError() == cudaSuccess ? ODPO_OK : ODPO_ERR_CUDA;
}

size_t odpo_lmhead_grad_scratch_bytes(int64_t chunk_rows, int64_t d, int64_t V) {
  if (chunk_rows <= 0 || d <= 0 || V <= 0) return 0;
  return grad_layout(chunk_rows, d, V);
}

odpo_status odpo_lmhead_grad(const void* hidden, const void* weight, int64_t R, int64_t d,
                             int64_t V, const int32_t* tokens, const float* row_lse,
                             const float* row_scale, float inv_temperature, float* dhidden,
                             float* dweight, void* scratch, size_t scratch_bytes,
                             int64_t chunk_rows, void* stream) {
  if (!hidden || !weight || !tokens || !row_lse || !row_scale || !dhidden || !dweight)
    return ODPO_ERR_INVALID_ARG;
  if (R <= 0 || d <= 0 || V <= 0 || chunk_rows <= 0) return ODPO_ERR_INVALID_ARG;
  if (!(isfinite(inv_temperature) && inv_temperature > 0.f)) return ODPO_ERR_INVALID_ARG;
  if (d % BK) return ODPO_ERR_UNSUPPORTED;
  if (R > (int64_t)INT32_MAX || V > (int64_t)INT32_MAX || d > (1 << 20)) return ODPO_ERR_UNSUPPORTED;
  if (((uintptr_t)hidden & 15u) || ((uintptr_t)weight & 15u) || ((uintptr_t)scratch & 15u) ||
      ((uintptr_t)dhidden & 15u) || ((uintptr_t)dweight & 15u))
    return ODPO_ERR_ALIGNMENT;
  if (chunk_rows > R) chunk_rows = R;
  const int64_t CR = (chunk_rows + 255) / 256 * 256;  // whole CTA-pair row blocks
  if (!scratch || scratch_bytes < odpo_lmhead_grad_scratch_bytes(CR, d, V))
    return ODPO_ERR_WORKSPACE;
  int dev = 0;
  cudaGetDevice(&dev);
  static std::once_flag attr_once[128];
  if (dev < 0 || dev >= 128) return ODPO_ERR_UNSUPPORTED;
  std::call_once(attr_once[dev], []() {
    cudaFuncSetAttribute(k_lmhead_fwd2<kEpiGrad>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM2);
    cudaFuncSetAttribute(k_gemm_tn2<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM2);
    cudaFuncSetAttribute(k_gemm_tn2<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM2);
    cudaFuncSetAttribute(k_gemm_tn2<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM2);
    cudaFuncSetAttribute(k_gemm_tn2<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM2);
  });
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t Vp = (V + 7) / 8 * 8;
  const int sms = sm_count();
  unsigned long long* ctr = reinterpret_cast<unsigned long long*>(
      reinterpret_cast<char*>(scratch) + odpo_lmhead_grad_scratch_bytes(CR, d, V) - 256);
  __nv_bfloat16* G = reinterpret_cast<__nv_bfloat16*>(scratch);
  char* Wt = reinterpret_cast<char*>(scratch) + (((size_t)CR * Vp * 2 + 255) & ~(size_t)255);
  char* Ht = Wt + (((size_t)d * Vp * 2 + 255) & ~(size_t)255);
  if (kGemmKB)
    k_transpose_bf16<<<dim3((unsigned)((d + 63) / 64), (unsigned)((V + 63) / 64)), 256, 0, s>>>(
        reinterpret_cast<const unsigned short*>(weight), V, d, d,
        reinterpret_cast<unsigned short*>(Wt), Vp);
  CUtensorMap mB;
  if (!make_map(&mB, weight, V, d, d, BN / 2)) return ODPO_ERR_CUDA;
  for (int64_t r0 = 0; r0 < R; r0 += CR) {
    const int64_t Rc = min(CR, R - r0);
    const char* hc = reinterpret_cast<const char*>(hidden) + r0 * d * 2;
    CUtensorMap mA;
    if (!make_map(&mA, hc, Rc, d, d, BM)) return ODPO_ERR_CUDA;
    Args a{};
    a.R = Rc; a.d = d; a.V = V;
    a.nrb = (Rc + BM - 1) / BM;
    a.NT = (V + BN - 1) / BN;
    a.Ttot = a.nrb * a.NT;
    a.nrb2 = (Rc + 255) / 256;
    a.G = lmh_group(d);
    a.invT = inv_temperature;
    a.tokens = tokens + r0;
    a.row_lse = row_lse + r0;
    a.row_scale = row_scale + r0;
    a.gout = G;
    a.ldg = Vp;
    int clusters = sms / 2;
    if (clusters > a.nrb2 * a.NT) clusters = (int)(a.nrb2 * a.NT);
    a.tile_ctr = tile_mode(ctr, a.nrb2 * a.NT, clusters);
    if (a.tile_ctr && cudaMemsetAsync(a.tile_ctr, 0, sizeof(unsigned long long), s) != cudaSuccess)
      return ODPO_ERR_CUDA;
    void* args[] = {&mA, &mB, &a};
    launch_pair((const void*)k_lmhead_fwd2<kEpiGrad>, clusters, s, args);
    if (cudaGetLastError() != cudaSuccess) return ODPO_ERR_CUDA;
    odpo_status e;
    if (kGemmKB) {
      k_transpose_bf16<<<dim3((unsigned)((d + 63) / 64), (unsigned)((Rc + 63) / 64)), 256, 0, s>>>(
          reinterpret_cast<const unsigned short*>(hc), Rc, d, d,
          reinterpret_cast<unsigned short*>(Ht), CR);
      e = gemm2<false, false>(Operand{G, Vp, false}, Operand{Wt, Vp, false}, Rc, d, V,
                              dhidden + r0 * d, d, false, sms, s, ctr);
      if (e != ODPO_OK) return e;
      e = gemm2<true, false>(Operand{G, Vp, true}, Operand{Ht, CR, false}, V, d, Rc, dweight, d,
                             r0 > 0, sms, s, ctr);
      if (e != ODPO_OK) return e;
      continue;
    }
    // dhidden[r0 : r0 + Rc] = G W: A = G (K = V contiguous), B = W read N-major (N = d contiguous)
    e = gemm2<false, true>(Operand{G, Vp, false}, Operand{weight, d, true}, Rc, d, V,
                           dhidden + r0 * d, d, false, sms, s, ctr);
    if (e != ODPO_OK) return e;
    // dweight (+)= G^T H: A = G read M-major (M = V contiguous), B = H chunk read N-major
    e = gemm2<true, true>(Operand{G, Vp, true}, Operand{hc, d, true}, V, d, Rc, dweight, d, r0 > 0,
                          sms, s, ctr);
    if (e != ODPO_OK) return e;
  }
  return ODPO_OK;
}


// ---------------------------------------------------------------- the chunked LM-head learner step
// (NEXT-2): per chunk of whole pairs, logits = H W^T in bf16 into a chunk
// buffer by the head kernel's LOGITS epilogue, which also folds the stored logits into one
// (m, log1p r, x_tok) partial per (row, 256-entry vocabulary tile); the loss then merges those
// partials exactly as the vocabulary-parallel path merges its shards' (odpo_vp_loss_fwd_bwd with
// one "shard" per tile: row statistics, masked sums, z, loss, statistics, and dlogits = coef
// (softmax - onehot) in place over the chunk), so the logits are read ONCE (by the backward)
// instead of twice; then dhidden = dlogits W and dweight += dlogits^T H (library GEMMs,
// MN-major operands).  Three head GEMMs (the recomputing step needs four), one chunk of logits.
// Build flag ODPO_STEP_FWD_PASS=1: the round-2 variant (plain bf16 GEMM + the full loss call,
// which re-reads the chunk for its forward pass), kept for the A/B measurement.
#ifndef ODPO_STEP_FWD_PASS
#define ODPO_STEP_FWD_PASS 0
#endif
__global__ void k_stats_add(double* total, const double* part, int n, int first) {
  const int i = threadIdx.x;
  if (i < n) total[i] = first ? part[i] : total[i] + part[i];
}

size_t odpo_lmhead_dpo_step_scratch_bytes(int64_t chunk_pairs, int64_t T, int64_t V) {
  if (chunk_pairs <= 0 || T <= 0 || V <= 0) return 0;
  const int64_t Vp = (V + 7) / 8 * 8;
  const int64_t Rc = 2 * chunk_pairs * T;
  auto al = [](size_t x) { return (x + 255) & ~(size_t)255; };
  const int64_t NT = (V + BN - 1) / BN;
  return al((size_t)Rc * Vp * 2) + al(odpo_workspace_bytes(2 * chunk_pairs, T, chunk_pairs)) +
         al(16 * sizeof(double)) + al((size_t)NT * Rc * sizeof(float4)) + 512;   // last 256: tile counter
}

odpo_status odpo_lmhead_dpo_step(const void* hidden, const void* weight, int64_t P, int64_t T,
                                 int64_t d, int64_t V, const float* ref_logp,
                                 const int32_t* tokens, const uint8_t* mask, int64_t P_global,
                                 float beta, float inv_temperature, float* dhidden,
                                 float* dweight, float* seq_logp, float* pair_logit,
                                 double* stats, uint32_t* status, void* scratch,
                                 size_t scratch_bytes, int64_t chunk_pairs, void* stream) {
  if (!hidden || !weight || !ref_logp || !tokens || !mask || !dhidden || !dweight || !seq_logp ||
      !stats)
    return ODPO_ERR_INVALID_ARG;
  if (P <= 0 || T <= 0 || d <= 0 || V <= 0 || chunk_pairs <= 0 || P_global < P)
    return ODPO_ERR_INVALID_ARG;
  if (!(isfinite(beta) && beta > 0.f) || !(isfinite(inv_temperature) && inv_temperature > 0.f))
    return ODPO_ERR_INVALID_ARG;
  if (d % BK) return ODPO_ERR_UNSUPPORTED;
  if (2 * P * T > (int64_t)INT32_MAX || V > (int64_t)INT32_MAX || d > (1 << 20))
    return ODPO_ERR_UNSUPPORTED;
  if (((uintptr_t)hidden & 15u) || ((uintptr_t)weight & 15u) || ((uintptr_t)scratch & 255u) ||
      ((uintptr_t)dhidden & 15u) || ((uintptr_t)dweight & 15u))
    return ODPO_ERR_ALIGNMENT;
  if (chunk_pairs > P) chunk_pairs = P;
  if (!scratch || scratch_bytes < odpo_lmhead_dpo_step_scratch_bytes(chunk_pairs, T, V))
    return ODPO_ERR_WORKSPACE;
  int dev = 0;
  cudaGetDevice(&dev);
  static std::once_flag attr_once[128];
  if (dev < 0 || dev >= 128) return ODPO_ERR_UNSUPPORTED;
  std::call_once(attr_once[dev], []() {
    cudaFuncSetAttribute(k_gemm_tn2<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM2);
    cudaFuncSetAttribute(k_gemm_tn2<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM2);
    cudaFuncSetAttribute(k_gemm_tn2<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM2);
    cudaFuncSetAttribute(k_lmhead_fwd2<kEpiLogits>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM2);
  });
  cudaStream_t s = (cudaStream_t)stream;
  const int sms = sm_count();
  const int64_t Vp = (V + 7) / 8 * 8;
  const int64_t NT = (V + BN - 1) / BN;
  auto al = [](size_t x) { return (x + 255) & ~(size_t)255; };
  char* base = reinterpret_cast<char*>(scratch);
  unsigned long long* ctr = reinterpret_cast<unsigned long long*>(
      base + odpo_lmhead_dpo_step_scratch_bytes(chunk_pairs, T, V) - 256);
  __nv_bfloat16* L = reinterpret_cast<__nv_bfloat16*>(base);
  const int64_t Rmax = 2 * chunk_pairs * T;
  char* ws = base + al((size_t)Rmax * Vp * 2);
  const size_t wsb = odpo_workspace_bytes(2 * chunk_pairs, T, chunk_pairs);
  double* cst = reinterpret_cast<double*>(ws + al(wsb));
  float4* parts4 = reinterpret_cast<float4*>(reinterpret_cast<char*>(cst) + al(16 * sizeof(double)));
  CUtensorMap mB;
  if (!make_map(&mB, weight, V, d, d, BN / 2)) return ODPO_ERR_CUDA;
  for (int64_t p0 = 0; p0 < P; p0 += chunk_pairs) {
    const int64_t np = min(chunk_pairs, P - p0);
    const int64_t r0 = 2 * p0 * T, Rc = 2 * np * T;
    const char* hc = reinterpret_cast<const char*>(hidden) + r0 * d * 2;
    odpo_status e;
    if (ODPO_STEP_FWD_PASS) {
      // logits chunk [Rc, V] (row pitch Vp) = H_c W^T, bf16; the full loss call in place
      e = gemm2<false, false>(Operand{hc, d, false}, Operand{weight, d, false}, Rc, V, d, nullptr,
                              Vp, false, sms, s, ctr, L);
      if (e != ODPO_OK) return e;
      e = odpo_online_dpo_loss_fwd_bwd(L, ODPO_BF16, 2 * np, T, V, T * Vp, Vp, ref_logp + 2 * p0,
                                       tokens + r0, mask + r0, nullptr, np, P_global, beta,
                                       inv_temperature, L, T * Vp, Vp, seq_logp + 2 * p0,
                                       pair_logit ? pair_logit + p0 : nullptr, cst, status, ws,
                                       wsb, stream);
      if (e != ODPO_OK) return e;
    } else {
      // logits chunk [Rc, V] (row pitch Vp) = H_c W^T in bf16 + the per-tile partials
      CUtensorMap mA;
      if (!make_map(&mA, hc, Rc, d, d, BM)) return ODPO_ERR_CUDA;
      Args a{};
      a.R = Rc; a.d = d; a.V = V;
      a.nrb = (Rc + BM - 1) / BM;
      a.NT = NT;
      a.Ttot = a.nrb * a.NT;
      a.nrb2 = (Rc + 255) / 256;
      a.G = lmh_group(d);
      a.invT = inv_temperature;
      a.tokens = tokens + r0;
      a.mask = mask + r0;
      a.gout = L;
      a.ldg = Vp;
      a.parts4 = parts4;
      int clusters = sms / 2;
      if (clusters > a.nrb2 * a.NT) clusters = (int)(a.nrb2 * a.NT);
      a.tile_ctr = tile_mode(ctr, a.nrb2 * a.NT, clusters);
      if (a.tile_ctr && cudaMemsetAsync(a.tile_ctr, 0, sizeof(unsigned long long), s) != cudaSuccess)
        return ODPO_ERR_CUDA;
      void* args[] = {&mA, &mB, &a};
      launch_pair((const void*)k_lmhead_fwd2<kEpiLogits>, clusters, s, args);
      if (cudaGetLastError() != cudaSuccess) return ODPO_ERR_CUDA;
      // row statistics from the NT partials, pair reduction, dlogits in place (one read)
      e = odpo_vp_loss_fwd_bwd(reinterpret_cast<const float*>(parts4), (int32_t)NT, L, ODPO_BF16,
                               2 * np, T, V, T * Vp, Vp, 0, V, ref_logp + 2 * p0, tokens + r0,
                               mask + r0, nullptr, np, P_global, beta, inv_temperature, L, T * Vp,
                               Vp, seq_logp + 2 * p0, pair_logit ? pair_logit + p0 : nullptr, cst,
                               nullptr, 0u, status, ws, wsb, stream);
      if (e != ODPO_OK) return e;
    }
    k_stats_add<<<1, 32, 0, s>>>(stats, cst, ODPO_NSTATS, p0 == 0);
    if (cudaGetLastError() != cudaSuccess) return ODPO_ERR_CUDA;
    // dhidden = dlogits W (W read N-major); dweight += dlogits^T H (both read MN-major)
    e = gemm2<false, true>(Operand{L, Vp, false}, Operand{weight, d, true}, Rc, d, V,
                           dhidden + r0 * d, d, false, sms, s, ctr);
    if (e != ODPO_OK) return e;
    e = gemm2<true, true>(Operand{L, Vp, true}, Operand{hc, d, true}, V, d, Rc, dweight, d, p0 > 0,
                          sms, s, ctr);
    if (e != ODPO_OK) return e;
  }
  return ODPO_OK;
}

}  // extern "C"
