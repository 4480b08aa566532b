// odpo_resident.cuh -- the RESIDENT schedule of the scaled Online-DPO call (K5r, sm_100a).
//
// Included by odpo.cu (outside namespace odpo) after LossArgs, pair_reduce_warp and the
// engine helpers.
//
// The scaled output dlogits = coef_b (softmax - onehot) needs the pair's coefficient, known
// only after BOTH sequences' forward passes (Eq. 3 / SURVEY.md §8(a) S3-S5).  The
// FUSED engine re-reads a row for its backward; on B200 that re-read misses L2 (DESIGN.md
// section 4) and the call moves 2R+1W.  This schedule keeps rows ON CHIP between their
// forward and backward passes instead (an explicit option: measured slower than FUSED, see
// DESIGN.md section 4 for the numbers and the Little's-law reason):
//
//   * one persistent CTA per SM (grid = #SMs, all co-resident);
//   * a forward TMA ring (ODPO_RES_RF x 16 KB stages, 1-D bulk copies) feeds 4 forward warps,
//     which run the online (m, r) pass from registers and, when the row owns a TMEM slot, write
//     the same registers to TENSOR MEMORY (tcgen05.st; 512 columns x 128 lanes x 32 bit = 256 KB
//     per SM = NSL row slots, two Pythia rows);
//   * 8 backward warps read a TMEM row back (tcgen05.ld; warps 4+j and 8+j read the two column
//     halves forward warp j wrote: same lane quadrant j, same vectors).  Rows beyond the TMEM
//     slots are "L2-backed" (forward loads evict_last): a backward thread re-streams them
//     through a second TMA ring (ODPO_RES_RB stages); at most `cap` of them per SM;
//   * the forward warps reproduce geometry 0's per-row reduction tree (128 threads x 8 vectors
//     per chunk, then the same fixed-order merge), so row statistics, sequence sums, loss and
//     dlogits are bit-identical to FUSED / TWO_PASS and seq_logprobs;
//   * a producer warp (claims rows in pair order, owns the TMEM allocation), a parameter warp
//     (UN = 0: polls the sequence's packed ready+coefficient word from the pair reduction;
//     UN = 1: the factored gradient or a known coefficient, no wait) and an epilogue warp (row
//     statistics, pair counting, pair reduction);
//   * deadlock freedom (UN = 0): the producer claims a row only while holding a TMEM slot or an
//     L2 allowance, so a claimed row's forward pass waits on nothing but its own TMA; a pair
//     completes once all its 2T rows are claimed, which needs SMs * min(NSL + cap, 8) >= 2T
//     (the host requires twice that).
#pragma once

namespace odpo {

#ifndef ODPO_RES_FW
#define ODPO_RES_FW 4
#endif
constexpr int kResFW = ODPO_RES_FW;            // forward warps per group (4: geometry 0's tree; or 8)
// forward warp groups (experiment): each group of kResFW warps streams every kResFGr-th live
// row, so kResFGr rows are in their forward pass at once per SM
#ifndef ODPO_RES_FGROUPS
#define ODPO_RES_FGROUPS 1
#endif
constexpr int kResFGr = ODPO_RES_FGROUPS;
constexpr int kResFWt = kResFW * kResFGr;      // all forward warps
constexpr int kResBW = 8;                      // backward warps
constexpr int kResProd = kResFWt + kResBW;     // producer warp, TMEM owner
constexpr int kResPar = kResProd + 1;          // parameter warp (13)
constexpr int kResEpi = kResProd + 2;          // epilogue warp (14)
constexpr int kResThreads = (kResEpi + 1) * 32;
constexpr int kResFT = kResFW * 32;            // forward threads (128)
constexpr int kResUB = kCV / kResFT;           // vectors per forward thread per chunk (8)
constexpr int kResCols = 32;                   // TMEM columns per lane per chunk (8 vectors)
constexpr int kResFG = kResFW / 4;             // forward warps per TMEM lane quadrant
constexpr int kResMaxRing = 13;                // forward / backward ring stages (max each)
// ring split of the 13 16-KB stages that fit: the forward ring sets the bytes in flight per SM
// (HBM latency x bandwidth share), the backward ring re-streams L2-backed rows
#ifndef ODPO_RES_RF
#define ODPO_RES_RF 10
#endif
#ifndef ODPO_RES_RB
#define ODPO_RES_RB 3
#endif
constexpr int kResRF = ODPO_RES_RF, kResRB = ODPO_RES_RB;
static_assert(kResRF + kResRB <= 13 && kResRB >= 1 && kResRF >= 1, "13 x 16 KB stages fit");
constexpr int kResMaxSL = 4;                   // TMEM row slots (max)
constexpr int kResMaxCh = 8;                   // 16 KB chunks per row (max: 128 KB rows)
constexpr int kResNIt = 8;                     // item (row descriptor) ring
#ifndef ODPO_RES_CAP
#define ODPO_RES_CAP 2
#endif
constexpr int kResCapDefault = ODPO_RES_CAP;   // L2-backed rows in flight per CTA (default)
// live rows claimed but not yet through the forward warps (bounds the per-SM forward queue,
// whose tail latency decides when a pair completes)
#ifndef ODPO_RES_FQ
#define ODPO_RES_FQ 8
#endif
constexpr int kResFQ = ODPO_RES_FQ;
constexpr int kResTmemCols = 512;
// dynamic shared memory: row buffers (at most this much); every launch asks for at least
// kResSmemMin so that exactly one CTA (one 512-column TMEM allocation) fits per SM
constexpr int kResSmemMax = 227 * 1024 - 6 * 1024;
constexpr int kResSmemMin = 120 * 1024;
static_assert(kResFW == 4 || kResFW == 8, "4 or 8 forward warps");
static_assert(kResFGr == 1 || kResFW == 4, "forward groups of 4 warps");
static_assert(kResUB * 4 * kResFG == kResCols, "a chunk fills 32 columns of every lane");


enum { R_END = 0, R_LIVE = 1, R_MASK = 2, R_NONE = 3, R_ZERO = 4 };

struct ResItem {
  int32_t kind;
  int32_t tok;
  int32_t tslot;  // TMEM slot, -1 = L2-backed row (the backward re-streams it)
  int32_t pad_;
  int64_t p, s, g, tk;
  const char* row;
  char* drow;
  float m, l1p, logp;  // row statistics (epilogue -> parameter warp)
  float c, coef, gtok, xtok;
  float pm[kResFW], pr[kResFW];
};

struct ResGeo {
  int nsl, nch;  // TMEM row slots, 16 KB chunks per row
  int rf, rbs;   // forward / backward TMA ring stages (16 KB each)
  int cap;       // L2-backed rows in flight per CTA (rows beyond the TMEM stash)
};

#ifdef ODPO_RES_DEBUG
// debug builds: per pair-row ticket [claim, first chunk landed, last chunk landed, forward
// merged, coefficient acquired, backward start, backward done, -]
constexpr int kResDbgRows = 1 << 16;
__device__ unsigned long long g_res_dbg[kResDbgRows][8];
#define RES_DBG(tk, k)                                                    \
  do {                                                                    \
    if ((tk) >= 0 && (tk) < kResDbgRows) g_res_dbg[(tk)][(k)] = gtimer(); \
  } while (0)
#else
#define RES_DBG(tk, k) \
  do {                 \
  } while (0)
#endif

__device__ __forceinline__ bool mbar_test(uint32_t b, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n}"
      : "=r"(ok)
      : "r"(b), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void tm_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tm_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
// 32 consecutive 32-bit TMEM columns of this thread's lane <- 8 16-byte vectors
__device__ __forceinline__ void tm_st32(uint32_t taddr, const uint4 (&v)[8]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(v[0].x), "r"(v[0].y), "r"(v[0].z), "r"(v[0].w), "r"(v[1].x), "r"(v[1].y), "r"(v[1].z),
      "r"(v[1].w), "r"(v[2].x), "r"(v[2].y), "r"(v[2].z), "r"(v[2].w), "r"(v[3].x), "r"(v[3].y),
      "r"(v[3].z), "r"(v[3].w), "r"(v[4].x), "r"(v[4].y), "r"(v[4].z), "r"(v[4].w), "r"(v[5].x),
      "r"(v[5].y), "r"(v[5].z), "r"(v[5].w), "r"(v[6].x), "r"(v[6].y), "r"(v[6].z), "r"(v[6].w),
      "r"(v[7].x), "r"(v[7].y), "r"(v[7].z), "r"(v[7].w)
      : "memory");
}
__device__ __forceinline__ void tm_st16(uint32_t taddr, const uint4 (&v)[4]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
      "r"(v[0].x), "r"(v[0].y), "r"(v[0].z), "r"(v[0].w), "r"(v[1].x), "r"(v[1].y), "r"(v[1].z),
      "r"(v[1].w), "r"(v[2].x), "r"(v[2].y), "r"(v[2].z), "r"(v[2].w), "r"(v[3].x), "r"(v[3].y),
      "r"(v[3].z), "r"(v[3].w)
      : "memory");
}
template <int NV>
__device__ __forceinline__ void tm_st(uint32_t taddr, const uint4 (&v)[NV]) {
  if constexpr (NV == 8) tm_st32(taddr, v);
  else tm_st16(taddr, v);
}
// 16 consecutive 32-bit TMEM columns of this thread's lane -> 4 16-byte vectors (no wait)
__device__ __forceinline__ void tm_ld16_nw(uint32_t taddr, uint4 (&v)[4]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(v[0].x), "=r"(v[0].y), "=r"(v[0].z), "=r"(v[0].w), "=r"(v[1].x), "=r"(v[1].y),
        "=r"(v[1].z), "=r"(v[1].w), "=r"(v[2].x), "=r"(v[2].y), "=r"(v[2].z), "=r"(v[2].w),
        "=r"(v[3].x), "=r"(v[3].y), "=r"(v[3].z), "=r"(v[3].w)
      : "r"(taddr)
      : "memory");
}
__device__ __forceinline__ void tm_wait_ld() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
// 16 consecutive 32-bit TMEM columns of this thread's lane -> 4 16-byte vectors
__device__ __forceinline__ void tm_ld16(uint32_t taddr, uint4 (&v)[4]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(v[0].x), "=r"(v[0].y), "=r"(v[0].z), "=r"(v[0].w), "=r"(v[1].x), "=r"(v[1].y),
        "=r"(v[1].z), "=r"(v[1].w), "=r"(v[2].x), "=r"(v[2].y), "=r"(v[2].z), "=r"(v[2].w),
        "=r"(v[3].x), "=r"(v[3].y), "=r"(v[3].z), "=r"(v[3].w)
      : "r"(taddr)
      : "memory");
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// UN = 0: the scaled Online-DPO output (the coefficient waits for the pair).  UN = 1: the
// factored gradient G = softmax - onehot, or coef_b G with a coefficient known before the call
// (App B losses, a.coef_known) -- no row waits on another row, so a row's backward follows its
// forward straight out of TMEM (exactly 1R+1W, no pair-completion latency).
template <int DT, int PV, int UN>
__global__ void __launch_bounds__(kResThreads, 1) k_resident(LossArgs a, ResGeo G) {
#if ODPO_EXPERIMENTAL  // measured slower than FUSED: built only on request
  constexpr int N = Traits<DT>::N;
  constexpr int NPF = DT == 1 ? kPoly[PV].npf : 0;  // exp2 split
  constexpr int NPB = DT == 1 ? kPoly[PV].npb : 0;
  extern __shared__ __align__(128) uint8_t rbuf[];  // [rf] forward stages, [rbs] backward stages
  __shared__ __align__(8) uint64_t f_full[kResMaxRing];
  __shared__ __align__(8) uint64_t f_empty[kResMaxRing];
  __shared__ __align__(8) uint64_t b_full[kResMaxRing];
  __shared__ __align__(8) uint64_t b_empty[kResMaxRing];
  __shared__ __align__(8) uint64_t tm_free[kResMaxSL];
  __shared__ __align__(8) uint64_t it_full[kResNIt];
  __shared__ __align__(8) uint64_t it_empty[kResNIt];
  __shared__ __align__(8) uint64_t part_ready[kResNIt];
  __shared__ __align__(8) uint64_t param_ready[kResNIt];
  __shared__ __align__(8) uint64_t stat_ready[kResNIt];  // epilogue -> parameter warp
  __shared__ __align__(16) ResItem items[kResNIt];
  __shared__ uint32_t tm_base_sh;
  __shared__ int l2_out;  // L2-backed rows claimed and not yet through their backward
  __shared__ int f_q;     // live rows claimed and not yet through the forward warps
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int q = 0; q < kResMaxRing; ++q) {
      mbar_init(&f_full[q], 1);
      mbar_init(&f_empty[q], kResFW);
      mbar_init(&b_full[q], 1);
      mbar_init(&b_empty[q], kResBW);
    }
    for (int j = 0; j < kResMaxSL; ++j) mbar_init(&tm_free[j], 1);
    for (int i = 0; i < kResNIt; ++i) {
      mbar_init(&it_full[i], 1);
      mbar_init(&it_empty[i], 2 + kResBW);  // epilogue + parameter warp + backward warps
      mbar_init(&part_ready[i], kResFW);
      mbar_init(&param_ready[i], 1);
      mbar_init(&stat_ready[i], 1);
    }
    l2_out = 0;
    f_q = 0;
    mbar_fence_init();
  }
  if (warp == kResProd) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&tm_base_sh)),
                 "n"(kResTmemCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tm_fence_before();
  __syncthreads();
  tm_fence_after();
  const uint32_t tm_base = tm_base_sh;

  const uint32_t fring_s = smem_u32(rbuf);
  const uint32_t bring_s = fring_s + (uint32_t)(G.rf * kChunk);
  const uint32_t ffull_s = smem_u32(f_full), fempty_s = smem_u32(f_empty);
  const uint32_t bfull_s = smem_u32(b_full), bempty_s = smem_u32(b_empty);
  const uint32_t tfree_s = smem_u32(tm_free);
  const uint32_t itf_s = smem_u32(it_full), ite_s = smem_u32(it_empty);
  const uint32_t pready_s = smem_u32(part_ready), mready_s = smem_u32(param_ready);
  const uint32_t sready_s = smem_u32(stat_ready);
  const int64_t T = a.T;
  const int V = (int)a.V;
  const int nvec = V / N;
  const int tail = V - nvec * N;
  const float k2 = a.invT * kLog2e;
  const int nch = G.nch;
  const int scols = kResCols * nch;  // TMEM columns per row slot

  if (warp == kResProd) {
    if (lane == 0) {
      // ================= producer: a row store first (a free TMEM slot, else an L2 allowance),
      // then a ticket (pair order) -> item; the live row's chunks into the forward ring
      const uint64_t pol_drop = policy_evict_first();  // TMEM rows: read once
      const uint64_t pol_keep = policy_evict_last();   // L2 rows: read again by the backward
      const int64_t totalF = a.P * 2 * T;
      const int64_t total = totalF + (int64_t)__ldcg(&a.w.counters[C_NUNREF]) * T;
      uint32_t busy_t = 0, ut = 0;  // TMEM slot busy mask, per-slot use parities
      int fst = 0;
      uint32_t fph = 0;
      for (int64_t k = 0;; ++k) {
        const int it = (int)(k % kResNIt);
        mbar_wait(ite_s + 8 * it, (uint32_t)((k / kResNIt) & 1) ^ 1u);
        int ts = -1;
        for (;;) {
          for (int j = 0; j < G.nsl; ++j) {
            if (((busy_t >> j) & 1u) && mbar_test(tfree_s + 8 * j, (ut >> j) & 1u)) {
              busy_t &= ~(1u << j);
              ut ^= 1u << j;
            }
            if (ts < 0 && !((busy_t >> j) & 1u)) ts = j;
          }
          if ((ts >= 0 || *((volatile int*)&l2_out) < G.cap) && *((volatile int*)&f_q) < kResFQ)
            break;
          __nanosleep(32);
        }
        const int64_t tk = (int64_t)atomicAdd(&a.w.counters[C_TICKET], 1u);
        ResItem& I = items[it];
        I.tslot = -1;
        I.tok = 0;
        I.p = 0;
        I.s = -1;
        I.g = 0;
        I.row = nullptr;
        I.drow = nullptr;
        I.tk = tk < totalF ? tk : -1;
        RES_DBG(I.tk, 0);
        if (tk >= total) {
          I.kind = R_END;
          mbar_arrive(itf_s + 8 * it);
          break;
        }
        if (tk < totalF) {
          const int64_t R = 2 * T, p = tk / R, j = tk % R;
          int64_t c, r;
          pair_seqs(a, p, c, r);
          const int64_t s = j < T ? c : r, t = j < T ? j : j - T;
          I.p = p;
          I.s = s;
          I.g = s >= 0 ? s * T + t : 0;
          if (s < 0) {
            I.kind = R_NONE;
          } else if (!a.mask[I.g]) {
            I.kind = R_MASK;
            I.drow = drow_ptr(a, s, t);
          } else {
            I.kind = R_LIVE;
            I.row = row_ptr(a, s, t);
            I.drow = drow_ptr(a, s, t);
            I.tok = a.tokens[I.g];
          }
        } else {
          const int64_t q = (tk - totalF) / T, t = (tk - totalF) % T;
          const int64_t s = __ldcg(a.w.unref + q);
          I.kind = R_ZERO;
          I.s = s;
          I.g = s * T + t;
          I.drow = drow_ptr(a, s, t);
        }
        if (I.kind == R_LIVE) {
          if (ts >= 0) {
            I.tslot = ts;
            busy_t |= 1u << ts;
          } else {
            atomicAdd(&l2_out, 1);
          }
          atomicAdd(&f_q, 1);
        }
        mbar_arrive(itf_s + 8 * it);
        if (I.kind == R_LIVE) {
          const char* src = I.row;
          const uint64_t pol = ts >= 0 ? pol_drop : pol_keep;
          for (int c = 0; c < nch; ++c) {
            mbar_wait(fempty_s + 8 * fst, fph ^ 1u);
            const int nv = min(kCV, nvec - c * kCV);
            const uint32_t bytes = (uint32_t)nv * 16u;
            mbar_arrive_tx(ffull_s + 8 * fst, bytes);
            tma_load_1d(fring_s + (uint32_t)(fst * kChunk), src + (size_t)c * kChunk, bytes,
                        ffull_s + 8 * fst, pol);
            if (++fst == G.rf) { fst = 0; fph ^= 1u; }
          }
        }
      }
    }
  } else if (warp < kResFWt) {
    // ================= forward warps: (m, r) over the row out of the forward ring, exactly
    // the engine's geometry-0 consumer arithmetic; the same registers go to the TMEM slot
    const int grp = warp / kResFW;           // forward group (rows live_idx % kResFGr)
    const int gw = warp % kResFW;            // warp within the group
    const int gtid = gw * 32 + lane;         // thread within the group (the reduction tree)
    const uint32_t lane_base = (uint32_t)(32 * (gw & 3)) << 16;
    const uint32_t gcol = (uint32_t)((gw >> 2) * kResUB * 4);  // this warp's column group
    int64_t live_idx = 0;                    // live rows seen so far (ring stage bookkeeping)
    for (int64_t k = 0;; ++k) {
      const int it = (int)(k % kResNIt);
      const uint32_t ph = (uint32_t)((k / kResNIt) & 1);
      mbar_wait(itf_s + 8 * it, ph);
      ResItem& I = items[it];
      const int kind = I.kind;
      if (kind == R_END) break;
      const bool mine = kind == R_LIVE ? (live_idx % kResFGr) == grp : grp == 0;
      const int64_t li = live_idx;
      if (kind == R_LIVE) ++live_idx;
      if (!mine) continue;
      if (kind == R_LIVE) {
        const int ts = I.tslot, tok = I.tok;
        const int tvec = (tok >= 0 && tok < nvec * N) ? tok / N : -1;
        const uint32_t tcol = tm_base + lane_base + (uint32_t)(ts * scols) + gcol;
        if (ts >= 0) tm_fence_after();
        MR s{-INFINITY, 0.f};
        for (int c = 0; c < nch; ++c) {
          const int64_t qst = li * nch + c;  // this chunk's position in the forward ring
          const int fst = (int)(qst % G.rf);
          const uint32_t fph = (uint32_t)((qst / G.rf) & 1);
          mbar_wait(ffull_s + 8 * fst, fph);
          if (gtid == 0 && c == 0) RES_DBG(I.tk, 1);
          if (gtid == 0 && c == nch - 1) RES_DBG(I.tk, 2);
          const uint4* sb = reinterpret_cast<const uint4*>(rbuf + (size_t)fst * kChunk);
          const int c0 = c * kCV;
          const int cnv = min(kCV, nvec - c0);
          uint4 v[kResUB];
          if (cnv == kCV) {
#pragma unroll
            for (int u = 0; u < kResUB; ++u) v[u] = sb[gtid + u * kResFT];
            if (ts >= 0) tm_st<kResUB>(tcol + (uint32_t)(c * kResCols), v);
            mr_batch<DT, kResUB, NPF>(v, k2, s.m, s.r);
          } else {
            const uint32_t NI = Traits<DT>::kNegInfWord;
#pragma unroll
            for (int u = 0; u < kResUB; ++u) {
              const int i = gtid + u * kResFT;
              v[u] = i < cnv ? sb[i] : make_uint4(NI, NI, NI, NI);
            }
            if (ts >= 0) tm_st<kResUB>(tcol + (uint32_t)(c * kResCols), v);
            if (gtid < cnv) mr_partial<DT, kResUB, NPF>(sb, gtid, kResFT, cnv, k2, s.m, s.r);
          }
          if (tvec >= c0 && tvec < c0 + cnv && ((tvec - c0) % kResFT) == gtid) {
            float f[N];
            Traits<DT>::unpack(sb[tvec - c0], f);
            float x = f[0];
#pragma unroll
            for (int j = 1; j < N; ++j) x = (tok % N == j) ? f[j] : x;
            I.xtok = x;
          }
          __syncwarp();
          if (lane == 0) mbar_arrive(fempty_s + 8 * fst);
        }
        if (gtid < tail) {
          const int64_t vv = (int64_t)nvec * N + gtid;
          const float x = Traits<DT>::load1(I.row, vv);
          s = mr_push1(s, x, k2);
          if (vv == tok) I.xtok = x;
        }
        const MR wv = warp_merge(s, k2);
        if (ts >= 0) {
          asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
          tm_fence_before();
        }
        __syncwarp();
        if (lane == 0) {
          I.pm[gw] = wv.m;
          I.pr[gw] = wv.r;
          mbar_arrive(pready_s + 8 * it);
          if (gw == 0) atomicSub(&f_q, 1);
        }
      } else {
        __syncwarp();
        if (lane == 0) mbar_arrive(pready_s + 8 * it);
      }
    }
  } else if (warp < kResProd) {
    // ================= backward warps: dlogits = coef (softmax - onehot) from TMEM, or, for an
    // L2-backed row, re-streamed through the backward ring (TMA issued by backward thread 0);
    // warp 4 + j (8 + j) handles vectors u = 0..3 (4..7) of forward warp j's threads -- the
    // columns that forward warp wrote into lane quadrant j
    const int j = (warp - kResFWt) & 3, half = (warp - kResFWt) >> 2;
    // the forward thread whose TMEM lane / columns this thread reads, and its first vector
    const int ftid = kResFW == 4 ? j * 32 + lane : (warp - kResFWt) * 32 + lane;
    const int u0 = kResFW == 4 ? 4 * half : 0;
    const uint32_t lane_base = (uint32_t)(32 * j) << 16;
    const int btid = tid - kResFWt * 32;  // 0..255 (zero rows, tail, TMA issue)
    const uint64_t pol_drop = policy_evict_first();
    int bst = 0, ist = 0;  // backward ring: next stage to consume / to fill
    uint32_t bph = 0, iph = 0;
    for (int64_t k = 0;; ++k) {
      const int it = (int)(k % kResNIt);
      const uint32_t ph = (uint32_t)((k / kResNIt) & 1);
      mbar_wait(itf_s + 8 * it, ph);
      const ResItem& I = items[it];
      const int kind = I.kind;
      if (kind == R_END) break;
      uint4* vout = reinterpret_cast<uint4*>(I.drow);
      if (kind == R_LIVE) {
        const int ts = I.tslot, tok = I.tok;
        // an L2 row: start re-streaming it before waiting for the coefficient
        auto issue = [&](int c) {
          mbar_wait(bempty_s + 8 * ist, iph ^ 1u);
          const int nv = min(kCV, nvec - c * kCV);
          const uint32_t bytes = (uint32_t)nv * 16u;
          mbar_arrive_tx(bfull_s + 8 * ist, bytes);
          tma_load_1d(bring_s + (uint32_t)(ist * kChunk), I.row + (size_t)c * kChunk, bytes,
                      bfull_s + 8 * ist, pol_drop);
          if (++ist == G.rbs) { ist = 0; iph ^= 1u; }
        };
        const int ahead = ts < 0 ? min(nch, G.rbs) : 0;
        if (btid == 0)
          for (int c = 0; c < ahead; ++c) issue(c);
        mbar_wait(mready_s + 8 * it, ph);
        if (btid == 0) RES_DBG(I.tk, 5);
        const float bc = I.c, coef = I.coef, gtok = I.gtok, bm = I.m;
        const bool neg = coef < 0.f;
        const int tvec = (tok >= 0 && tok < nvec * N) ? tok / N : -1;
        const uint32_t tcol = tm_base + lane_base + (uint32_t)(ts * scols + half * (kResCols / 2));
        static_assert(kResBW == 8, "8 backward warps: two 16-column halves per lane quadrant");
        if (ts >= 0) tm_fence_after();
        // two chunks per TMEM round trip (one tcgen05.wait::ld for both loads)
        for (int c = 0; c < nch; c += 2) {
          uint4 v[2][4];
          const bool two = c + 1 < nch;
          if (ts >= 0) {
            tm_ld16_nw(tcol + (uint32_t)(c * kResCols), v[0]);
            if (two) tm_ld16_nw(tcol + (uint32_t)((c + 1) * kResCols), v[1]);
            tm_wait_ld();
          }
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            if (q == 1 && !two) break;
            const int cc = c + q;
            const int c0 = cc * kCV;
            const int cnv = min(kCV, nvec - c0);
            if (ts < 0) {
              mbar_wait(bfull_s + 8 * bst, bph);
              const uint4* sb = reinterpret_cast<const uint4*>(rbuf + (size_t)(G.rf + bst) * kChunk);
#pragma unroll
              for (int u = 0; u < 4; ++u) {
                const int i = ftid + (u0 + u) * kResFT;
                v[q][u] = i < cnv ? sb[i] : make_uint4(0, 0, 0, 0);
              }
              __syncwarp();
              if (lane == 0) mbar_arrive(bempty_s + 8 * bst);
              if (++bst == G.rbs) { bst = 0; bph ^= 1u; }
              if (btid == 0 && cc + G.rbs < nch) issue(cc + G.rbs);
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const int i = ftid + (u0 + u) * kResFT;
              if (i < cnv)
                st16_stream(vout + c0 + i, neg ? bwd_vec<DT, NPB, true>(v[q][u], k2, bc, bm)
                                               : bwd_vec<DT, NPB, false>(v[q][u], k2, bc, bm));
            }
            // onehot entry: the thread that stored tok's vector overwrites it (program order)
            if (tvec >= c0 && tvec < c0 + cnv && ((tvec - c0) % kResFT) == ftid &&
                (tvec - c0) / kResFT - u0 >= 0 && (tvec - c0) / kResFT - u0 < 4)
              Traits<DT>::store1(I.drow, tok, gtok);
          }
        }
        if (btid < tail) {
          const int64_t vv = (int64_t)nvec * N + btid;
          const float x = Traits<DT>::load1(I.row, vv);
          Traits<DT>::store1(I.drow, vv, vv == tok ? gtok : copysignf(ex2(bwd_arg<DT>(x, k2, bc, bm)), coef));
        }
        if (ts >= 0) tm_fence_before();
        // all eight backward warps are past the row: release its TMEM slot / L2 allowance
        asm volatile("bar.sync 3, %0;" ::"n"(kResBW * 32) : "memory");
        if (btid == 0) {
          if (ts >= 0) mbar_arrive(tfree_s + 8 * ts);
          else atomicSub(&l2_out, 1);
          RES_DBG(I.tk, 6);
        }
      } else if (kind == R_MASK || kind == R_ZERO) {
        for (int i = btid; i < nvec; i += kResBW * 32) st16_stream(vout + i, make_uint4(0, 0, 0, 0));
        if (btid < tail) Traits<DT>::store1(I.drow, (int64_t)nvec * N + btid, 0.f);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(ite_s + 8 * it);
    }
  } else if (warp == kResPar) {
    // ================= parameter warp: poll the sequence's ready+coefficient word (written by
    // the pair reduction), fold coef into the exponent with this CTA's own row statistics
    if (lane == 0) {
      for (int64_t k = 0;; ++k) {
        const int it = (int)(k % kResNIt);
        const uint32_t ph = (uint32_t)((k / kResNIt) & 1);
        mbar_wait(itf_s + 8 * it, ph);
        ResItem& I = items[it];
        const int kind = I.kind;
        if (kind == R_END) break;
        mbar_wait(sready_s + 8 * it, ph);  // this row's statistics are in the item
        if (kind == R_LIVE) {
          float coef;
          if (UN) {
            // G (coef 1) or the known coefficient (k_pg_coef ran before this kernel)
            coef = a.coef_known ? __ldcg(a.w.seq_coef + I.s) : 1.f;
          } else {
            unsigned long long w;
            while (!((w = ld_relaxed_u64(&a.w.seq_cf[I.s])) & kCfReady)) __nanosleep(20);
            fence_acq_rel_gpu();
            coef = __uint_as_float((uint32_t)w);
          }
          const float m = I.m, l1p = I.l1p, logp = I.logp;
          I.c = coef != 0.f ? bwd_const<DT>(m, l1p, k2, coef) : INFINITY;
          I.coef = coef;
          I.gtok = coef * expm1f(logp);
          RES_DBG(I.tk, 4);
        }
        mbar_arrive(mready_s + 8 * it);
        mbar_arrive(ite_s + 8 * it);
      }
    }
  } else {
    // ================= epilogue warp: merge the forward partials, row statistics, count the
    // row into its pair; the row that completes a pair runs the pair reduction (S3/S4)
    for (int64_t k = 0;; ++k) {
      const int it = (int)(k % kResNIt);
      const uint32_t ph = (uint32_t)((k / kResNIt) & 1);
      mbar_wait(itf_s + 8 * it, ph);
      ResItem& I = items[it];
      const int kind = I.kind;
      if (kind == R_END) break;
      // every item: the forward warps are done with it before its descriptor can be reused
      mbar_wait(pready_s + 8 * it, ph);
      if (kind == R_LIVE) {
        MR v;
        v.m = lane < kResFW ? I.pm[lane] : -INFINITY;
        v.r = lane < kResFW ? I.pr[lane] : 0.f;
        v = warp_merge(v, k2);
        if (lane == 0) {
          RES_DBG(I.tk, 3);
          uint32_t fl = 0;
          const float l1p = log1pf(v.r);
          float logp = 0.f;
          if (I.tok < 0 || I.tok >= V) {
            fl |= ODPO_FLAG_TOKEN_RANGE;
          } else {
            logp = __fsub_rn(__fmul_rn(__fsub_rn(I.xtok, v.m), a.invT), l1p);
            if (!isfinite(logp)) fl |= ODPO_FLAG_NONFINITE_LOGIT;
          }
          if (!isfinite(v.m) || !isfinite(v.r)) fl |= ODPO_FLAG_NONFINITE_LOGIT;
          I.m = v.m;
          I.l1p = l1p;
          I.logp = logp;
          a.w.row_m[I.g] = v.m;
          a.w.row_l1p[I.g] = l1p;
          a.w.row_logp[I.g] = logp;
          flag(a.status, fl);
        }
      }
      if (UN && kind == R_ZERO && lane == 0 && a.row_scale) a.row_scale[I.g] = 0.f;
      __syncwarp();
      if (lane == 0) mbar_arrive(sready_s + 8 * it);
      if (kind == R_LIVE || kind == R_MASK || kind == R_NONE) {
        unsigned last = 0;
        if (lane == 0) last = (atom_add_acq_rel(&a.w.pair_cnt[I.p], 1u) == (unsigned)(2 * T) - 1u);
        last = __shfl_sync(kFull, last, 0);
        if (last) {
          fence_acq_rel_gpu();
          pair_reduce_warp(a, I.p);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(ite_s + 8 * it);
    }
  }
  tm_fence_before();
  __syncthreads();
  if (warp == kResProd) {
    tm_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm_base),
                 "n"(kResTmemCols)
                 : "memory");
  }
#endif  // ODPO_EXPERIMENTAL
}

}  // namespace odpo
