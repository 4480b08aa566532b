// odpo.cu -- libodpo.so: kernels and C ABI of the Online-DPO learner hot path on B200.
//
// Kernels:
//   k_pair_select    K1  reward-ranked pair selection + selection stats
//   k_prep           --  per-call workspace init, sequence->pair map, DUP/RANGE checks
//   k_engine<SEQ>    K2+K3a persistent TMA-ring engine, forward rows; the CTA finishing a
//                        sequence's last row sums it (seq_logprobs; TWO_PASS forward)
//   k_engine<FUSED>  K5  persistent TMA-ring engine: forward rows of pair s interleaved with
//                        backward rows of pair s-lag; per-pair completion counters; the CTA
//                        finishing a pair's last forward row runs K3b; backward rows wait on
//                        the pair's ready flag; backward re-reads hit L2 (evict_last policy)
//   k_pair_reduce    K3b one warp per pair (TWO_PASS)
//   k_row_bwd_split  K4  dlogits = coef (softmax - onehot), each row in one-batch pieces
//                        (TWO_PASS; k_row_bwd: one CTA per row, for grids past INT32_MAX)
//   k_engine<UNSC>   K5' factored gradient: each row's backward right after its forward
//   k_unsc_split/tma --  (experimental build) factored gradient over thread-block clusters
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include <cstddef>
#include <cstdio>
#include <mutex>

#include "odpo.h"
#include "odpo_device.cuh"
#include "odpo_engine.cuh"

#define ODPO_VERSION_STR "odpo-b200 0.2.0 (sm_100a)"

namespace odpo {

// ------------------------------------------------------------------ workspace layout
struct Workspace {
  float* row_m;
  float* row_l1p;
  float* row_logp;
  float* seq_coef;
  int32_t* seq_pair;   // 2p (chosen of p) / 2p+1 (rejected of p) / -1 unreferenced
  int32_t* unref;      // unreferenced sequences, ascending
  unsigned* seq_cnt;   // forward rows done per sequence (SEQ mode)
  unsigned* pair_cnt;  // forward rows done per pair (FUSED)
  unsigned* pair_ready;
  unsigned* pair_bcnt; // backward rows dispensed per pair (FUSED dispatch)
  double* pair_vals;   // [P][ODPO_NSTATS]
  unsigned long long* seq_cf;  // [B] ready bit (bit 32) | fp32 bits of the sequence's coef
  float4* fparts;      // [B*T][kFS] forward-part partials (m, r, x_tok, owns tok) (kFS > 1)
  float4* psparts;     // PSYNC: piece partials of a window of pairs [kPsWinPairs][G][2]
  unsigned* fpart_cnt; // [B*T] forward parts done (kFS > 1)
  unsigned long long* dbg_t;  // debug builds: [P][4] timestamps
  unsigned* counters;  // [0] ticket, [1] pairs done, [2] n_unref
};

enum { C_TICKET = 0, C_PAIRS_DONE = 1, C_NUNREF = 2, C_BPAIR = 3, C_ZTICKET = 4, C_DBG_SUM = 5,
       C_DBG_N = 6, C_DBG_MAX = 7, C_DBG_DONE = 8, C_COUNT = 16 };

static inline size_t align256(size_t x) { return (x + 255) & ~size_t(255); }
#ifndef ODPO_EXPERIMENTAL
#define ODPO_EXPERIMENTAL 0
#endif
#define ODPO_EXPERIMENTAL_WS ODPO_EXPERIMENTAL
constexpr int kPsWinPairs = 16;    // PSYNC partial window (pairs); the lag must stay below it
constexpr int kPsMaxGrid = 1024;   // PSYNC max CTAs
constexpr unsigned long long kCfReady = 1ull << 32;

static size_t ws_layout(int64_t B, int64_t T, int64_t P, char* base, Workspace* w) {
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off += align256(bytes);
    return base ? base + o : nullptr;
  };
  const size_t rows = (size_t)B * (size_t)T;
  char* p_m = take(rows * 4);
  char* p_l = take(rows * 4);
  char* p_lp = take(rows * 4);
  char* p_c = take((size_t)B * 4);
  char* p_sp = take((size_t)B * 4);
  char* p_u = take((size_t)B * 4);
  char* p_sc = take((size_t)B * 4);
  char* p_pc = take((size_t)P * 4);
  char* p_pr = take((size_t)P * 4);
  char* p_pb = take((size_t)P * 4);
  char* p_pv = take((size_t)P * ODPO_NSTATS * 8);
  char* p_cf = take((size_t)B * 8);
  char* p_fp = kFS > 1 ? take(rows * kFS * 16) : nullptr;
  char* p_fc = kFS > 1 ? take(rows * 4) : nullptr;
  char* p_ps = ODPO_EXPERIMENTAL_WS ? take((size_t)kPsWinPairs * kPsMaxGrid * 2 * 16) : nullptr;
  char* p_ct = take(C_COUNT * 4);
#ifdef ODPO_DEBUG_LEAD
  char* p_dt = take((size_t)P * 4 * 8);
#else
  char* p_dt = nullptr;
#endif
  if (w) {
    w->dbg_t = (unsigned long long*)p_dt;
    w->row_m = (float*)p_m;
    w->row_l1p = (float*)p_l;
    w->row_logp = (float*)p_lp;
    w->seq_coef = (float*)p_c;
    w->seq_pair = (int32_t*)p_sp;
    w->unref = (int32_t*)p_u;
    w->seq_cnt = (unsigned*)p_sc;
    w->pair_cnt = (unsigned*)p_pc;
    w->pair_ready = (unsigned*)p_pr;
    w->pair_bcnt = (unsigned*)p_pb;
    w->pair_vals = (double*)p_pv;
    w->seq_cf = (unsigned long long*)p_cf;
    w->fparts = (float4*)p_fp;
    w->fpart_cnt = (unsigned*)p_fc;
    w->psparts = (float4*)p_ps;
    w->counters = (unsigned*)p_ct;
  }
  return off;
}

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void flag(uint32_t* status, uint32_t f) {
  if (f && status) atomicOr(status, f);
}
__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// ------------------------------------------------------------------ K1 pair_select
// One CTA; thread i handles prompts i, i+NT, ...; selection stats reduced in fixed order.
constexpr int kSelThreads = 256;

__global__ void __launch_bounds__(kSelThreads) k_pair_select(
    const float* __restrict__ rewards, const uint8_t* __restrict__ has_eos, float eos_penalty,
    int64_t P, int K, int32_t* chosen, int32_t* rejected, int32_t* pair_rows, float* margin,
    double* sel_stats, uint32_t* status) {
  __shared__ double sm[3][kSelThreads];
  double msum = 0.0, ndeg = 0.0, ntr = 0.0;
  uint32_t fl = 0;
  for (int64_t p = threadIdx.x; p < P; p += kSelThreads) {
    const float* rw = rewards + p * K;
    const uint8_t* ew = has_eos ? has_eos + p * K : nullptr;
    // shaped reward: the EOS penalty REPLACES the score (R7)
    auto shaped = [&](int k) { return (ew == nullptr || ew[k]) ? rw[k] : eos_penalty; };
    int best = 0, worst = K - 1;
    float rb = shaped(0), rwst = shaped(K - 1);
    for (int k = 0; k < K; ++k) {
      const float v = shaped(k);
      if (!isfinite(v)) fl |= ODPO_FLAG_NONFINITE_REWARD;
      if (ew && !ew[k]) ntr += 1.0;
    }
    for (int k = 1; k < K; ++k) {           // FIRST index of the max (R5)
      const float v = shaped(k);
      if (v > rb) { rb = v; best = k; }
    }
    for (int k = K - 2; k >= 0; --k) {      // LAST index of the min (R5)
      const float v = shaped(k);
      if (v < rwst) { rwst = v; worst = k; }
    }
    const float mg = __fsub_rn(rb, rwst);
    if (rb == rwst) { fl |= ODPO_FLAG_DEGENERATE_PAIR; ndeg += 1.0; }
    chosen[p] = best;
    rejected[p] = worst;
    if (pair_rows) {
      pair_rows[2 * p] = (int32_t)(p * K + best);
      pair_rows[2 * p + 1] = (int32_t)(p * K + worst);
    }
    if (margin) margin[p] = mg;
    msum += (double)mg;
  }
  flag(status, fl);
  if (!sel_stats) return;
  sm[0][threadIdx.x] = msum;
  sm[1][threadIdx.x] = ndeg;
  sm[2][threadIdx.x] = ntr;
  __syncthreads();
  for (int s = kSelThreads / 2; s > 0; s >>= 1) {  // fixed-order tree
    if ((int)threadIdx.x < s)
      for (int q = 0; q < 3; ++q) sm[q][threadIdx.x] += sm[q][threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    sel_stats[ODPO_SEL_MARGIN_SUM] = sm[0][0];
    sel_stats[ODPO_SEL_NDEGEN] = sm[1][0];
    sel_stats[ODPO_SEL_NTRUNC] = sm[2][0];
  }
}

// ------------------------------------------------------------------ prep
constexpr int kPrepThreads = 1024;

__global__ void __launch_bounds__(kPrepThreads) k_prep(const int32_t* __restrict__ pair_rows,
                                                       int64_t B, int64_t P, Workspace w,
                                                       uint32_t* status, int64_t rows = 0) {
  __shared__ int scan[kPrepThreads];
  const int tid = threadIdx.x;
  if (w.fpart_cnt)
    for (int64_t g = tid; g < rows; g += kPrepThreads) w.fpart_cnt[g] = 0;
  for (int64_t b = tid; b < B; b += kPrepThreads) {
    w.seq_pair[b] = -1;
    w.seq_cnt[b] = 0;
    w.seq_cf[b] = 0ull;
  }
  for (int64_t p = tid; p < P; p += kPrepThreads) {
    w.pair_cnt[p] = 0;
    w.pair_ready[p] = 0;
    w.pair_bcnt[p] = 0;
  }
  if (tid < C_COUNT) w.counters[tid] = 0;
  __syncthreads();
  uint32_t fl = 0;
  for (int64_t p = tid; p < P; p += kPrepThreads) {
    const int64_t c = pair_rows ? pair_rows[2 * p] : 2 * p;
    const int64_t r = pair_rows ? pair_rows[2 * p + 1] : 2 * p + 1;
    if (c < 0 || c >= B || r < 0 || r >= B) { fl |= ODPO_FLAG_PAIR_RANGE; continue; }
    if (atomicCAS(&w.seq_pair[c], -1, (int)(2 * p)) != -1) fl |= ODPO_FLAG_DUP_ROW;
    if (atomicCAS(&w.seq_pair[r], -1, (int)(2 * p + 1)) != -1) fl |= ODPO_FLAG_DUP_ROW;
  }
  flag(status, fl);
  __syncthreads();
  // ordered compaction of unreferenced sequences (block scan over contiguous chunks)
  const int64_t chunk = (B + kPrepThreads - 1) / kPrepThreads;
  const int64_t b0 = tid * chunk, b1 = min(B, b0 + chunk);
  int cnt = 0;
  for (int64_t b = b0; b < b1; ++b) cnt += (w.seq_pair[b] < 0);
  scan[tid] = cnt;
  __syncthreads();
  for (int off = 1; off < kPrepThreads; off <<= 1) {
    int v = tid >= off ? scan[tid - off] : 0;
    __syncthreads();
    scan[tid] += v;
    __syncthreads();
  }
  int pos = scan[tid] - cnt;
  for (int64_t b = b0; b < b1; ++b)
    if (w.seq_pair[b] < 0) w.unref[pos++] = (int32_t)b;
  if (tid == kPrepThreads - 1) w.counters[C_NUNREF] = (unsigned)scan[tid];
}

// ------------------------------------------------------------------ K1b compact the selected pairs
// dst row 2p+k <- src row pair_rows[2p+k] for tokens / mask [rows][T] and ref_logp [rows]
// (of K completions only the chosen and rejected are trained on).  One CTA per
// destination row, 16-byte copies where the row strides allow.
__global__ void k_gather_pairs(const int32_t* __restrict__ pair_rows, int64_t n_src, int64_t T,
                               const int32_t* __restrict__ tok_in, const uint8_t* __restrict__ mask_in,
                               const float* __restrict__ ref_in, int32_t* __restrict__ tok_out,
                               uint8_t* __restrict__ mask_out, float* __restrict__ ref_out,
                               uint32_t* status) {
  const int64_t d = blockIdx.x;
  const int64_t src = pair_rows[d];
  const bool ok = src >= 0 && src < n_src;
  if (!ok && threadIdx.x == 0) flag(status, ODPO_FLAG_PAIR_RANGE);
  if (threadIdx.x == 0 && ref_out) ref_out[d] = ok ? ref_in[src] : 0.f;
  for (int64_t t = threadIdx.x; t < T; t += blockDim.x) {
    if (tok_out) tok_out[d * T + t] = ok ? tok_in[src * T + t] : 0;
    if (mask_out) mask_out[d * T + t] = ok ? mask_in[src * T + t] : (uint8_t)0;
  }
}

// ------------------------------------------------------------------ shared arguments
// NEXT-4 in-kernel exchange of the vocabulary-parallel row partials over peer memory (NVLink /
// NVSwitch P2P, or CUDA IPC between processes on one GPU): rank `rank` stores each row's
// 16-byte partial into slot [rank][g] of EVERY rank's partial buffer (parts[q]: rank q's buffer,
// mapped into this process), then the last CTA to finish publishes `epoch` into every rank's
// flag word flags[q][rank] with a system-scope release.  The combine kernel on rank q waits
// for all W flags (acquire) and merges the W partials of each row in rank order.
constexpr int kVpMaxW = 8;
struct VpPut {
  float4* parts[kVpMaxW];
  uint32_t* flags[kVpMaxW];
  uint32_t* done;   // this rank's CTA completion counter (reset by the last CTA)
  int32_t rank, W;
  uint32_t epoch;
};

struct LossArgs {
  const void* logits;
  int64_t B, T, V, sb, st;  // strides in elements
  const float* ref;
  const int32_t* tokens;
  const uint8_t* mask;
  const int32_t* pair_rows;
  int64_t P;
  double Pg;
  float beta, invT;
  void* dl;
  int64_t dsb, dst;
  float* seq_logp;
  float* z_out;
  double* stats;
  uint32_t* status;
  float* tok_out;   // SEQ: optional per-token log-probs
  float* lse_out;   // SEQ: optional per-row lse
  int seqsum;       // SEQ: sum sequences (seq_logprobs) or only write row stats (TWO_PASS)
  Workspace w;
  int lag;
  int64_t max_lead;  // FUSED: cap on forward rows dispensed ahead of the backward frontier
  int look;         // producer decode lookahead (rows), <= kSlots - 2
  int esize;
  int wave_ng;      // FUSED, wave schedule: groups (0 = adaptive dispatch)
  int wave_gs;      // CTAs per group (= 2T)
  int wave_gap;     // pair-steps between a pair's forward and backward rows (0 or 1)
  float* row_scale;  // UNSC: [B*T] out, coef_b * mask (dlogits = row_scale * G)
  int row_gap;       // UNSC: forward rows streamed between a row's forward and its backward
  // coefficient-variant losses (App B): -1 = Online DPO, else ODPO_PG_* (odpo.h)
  int pg_kind;
  int coef_known;        // UNSC: seq_coef is an input (RLOO, CoPG, SFT): write coef*G directly
  const float* rewards;  // [B] per-sequence rewards (advantages A1 = R1 - R2)
  const float* old_logp; // [B] log pi_old (CoPG, Proximal RLOO)
  float clip_eps;
  // vocabulary-parallel forward (NEXT-4): this call sees columns [tok_off, tok_off + V) of a
  // V_total vocabulary and writes per-row partials (m, log1p r, x_tok, owns tok) instead of
  // log-probs
  float4* vp_parts;
  int64_t tok_off;
  int64_t V_total;
  VpPut put;            // NEXT-4 in-kernel exchange (put.W = 0: write vp_parts locally)
  const uint32_t* vp_flags;  // combine: wait until every vp_flags[q] reached vp_epoch (NULL: none)
  uint32_t vp_epoch;
};

__device__ __forceinline__ const char* row_ptr(const LossArgs& a, int64_t b, int64_t t) {
  return reinterpret_cast<const char*>(a.logits) + (b * a.sb + t * a.st) * a.esize;
}
__device__ __forceinline__ char* drow_ptr(const LossArgs& a, int64_t b, int64_t t) {
  return reinterpret_cast<char*>(a.dl) + (b * a.dsb + t * a.dst) * a.esize;
}

__device__ __forceinline__ void pair_seqs(const LossArgs& a, int64_t p, int64_t& c, int64_t& r) {
  c = a.pair_rows ? a.pair_rows[2 * p] : 2 * p;
  r = a.pair_rows ? a.pair_rows[2 * p + 1] : 2 * p + 1;
  if (c < 0 || c >= a.B) c = -1;
  if (r < 0 || r >= a.B) r = -1;
}

// A pair with an out-of-range member (flagged ODPO_FLAG_PAIR_RANGE by k_prep): its in-range
// sequence gets coefficient 0 (zero dlogits) and a published ready word, so no schedule waits
// on it or reads a stale coefficient.
__device__ __forceinline__ void invalid_pair_coefs(const LossArgs& a, int64_t c, int64_t r) {
  const int64_t y[2] = {c, r};
  for (int k = 0; k < 2; ++k) {
    if (y[k] < 0) continue;
    a.w.seq_coef[y[k]] = 0.f;
    st_release_u64(&a.w.seq_cf[y[k]], kCfReady);
  }
}

// Pair reduction (K3b) by ONE warp: fixed-order sums of both sequences, then lane 0 forms z,
// loss, sigma(-z), coef, publishes them (release) and the pair's statistics; the warp that
// completes the LAST pair reduces all pairs' statistics in fixed order.
__device__ __noinline__ void pair_reduce_warp(const LossArgs& a, int64_t p) {
  const int lane = threadIdx.x & 31;
  int64_t c, r;
  pair_seqs(a, p, c, r);
  double Sc = 0.0, Sr = 0.0;
  int nc = 0, nr = 0;
  seq_sum2_warp(c >= 0 ? a.w.row_logp + c * a.T : nullptr, c >= 0 ? a.mask + c * a.T : nullptr,
                r >= 0 ? a.w.row_logp + r * a.T : nullptr, r >= 0 ? a.mask + r * a.T : nullptr,
                a.T, Sc, nc, Sr, nr);
  unsigned last = 0;
  if (lane == 0 && a.pg_kind >= 0) {
    uint32_t fl = 0;
    double* pv = a.w.pair_vals + p * ODPO_NSTATS;
    if (c < 0 || r < 0) {
      for (int k = 0; k < ODPO_NSTATS; ++k) pv[k] = 0.0;
      invalid_pair_coefs(a, c, r);
    } else {
      if (nc == 0 || nr == 0) fl |= ODPO_FLAG_EMPTY_SEQ;
      const float fS[2] = {nc ? (float)Sc : 0.f, nr ? (float)Sr : 0.f};
      const int64_t y[2] = {c, r};
      const double A0 = (double)a.rewards[c] - (double)a.rewards[r];
      const double A[2] = {A0, -A0};
      const double scale = (double)a.invT / (2.0 * a.Pg);
      double loss = 0.0, nact = 0.0, rsum = 0.0;
      for (int k = 0; k < 2; ++k) {
        const double S = (double)fS[k];
        double cf = 0.0;
        if (a.pg_kind == ODPO_PG_RLOO) {
          loss += -0.5 * S * A[k];
          cf = A[k] * scale;
        } else if (a.pg_kind == ODPO_PG_COPG) {
          loss += -0.5 * (S - (double)a.old_logp[y[k]]) * A[k];
          cf = A[k] * scale;
        } else if (a.pg_kind == ODPO_PG_PROX_RLOO) {
          const double rt = exp(S - (double)a.old_logp[y[k]]);
          const double eps = (double)a.clip_eps;
          const double rc = fmin(fmax(rt, 1.0 - eps), 1.0 + eps);
          const double u = rt * A[k], v = rc * A[k];
          loss += -0.5 * (u <= v ? u : v);
          cf = u <= v ? rt * A[k] * scale : 0.0;
          rsum += rt;
          a.w.seq_coef[y[k]] = (float)cf;   // the only kind whose coefficient needs S
          st_release_u64(&a.w.seq_cf[y[k]], kCfReady | __float_as_uint((float)cf));
        } else if (k == 0) {               // Best-of-2 SFT on the chosen completion
          loss += -S;
          cf = 2.0 * scale;
        }
        if ((float)cf != 0.f) nact += 1.0;
        a.seq_logp[y[k]] = fS[k];
      }
      pv[ODPO_ST_NPAIRS] = 1.0;
      pv[ODPO_ST_LOSS] = loss;
      pv[ODPO_ST_NCORRECT] = nact;
      pv[ODPO_ST_Z] = rsum;
      pv[ODPO_ST_RCHOSEN] = A0;
      pv[ODPO_ST_RREJ] = fabs(A0);
      pv[ODPO_ST_SCHOSEN] = (double)fS[0];
      pv[ODPO_ST_SREJ] = (double)fS[1];
      pv[ODPO_ST_NTOK_CHOSEN] = (double)nc;
      pv[ODPO_ST_NTOK_REJ] = (double)nr;
    }
    flag(a.status, fl);
    st_release(&a.w.pair_ready[p], 1u);
    const unsigned done = atom_add_acq_rel(&a.w.counters[C_PAIRS_DONE], 1u);
    last = (done == (unsigned)(a.P - 1));
  } else if (lane == 0) {
    uint32_t fl = 0;
    double* pv = a.w.pair_vals + p * ODPO_NSTATS;
    if (c < 0 || r < 0) {
      for (int k = 0; k < ODPO_NSTATS; ++k) pv[k] = 0.0;
      if (a.z_out) a.z_out[p] = 0.f;
      invalid_pair_coefs(a, c, r);
    } else {
      if (nc == 0 || nr == 0) fl |= ODPO_FLAG_EMPTY_SEQ;
      const float fSc = nc ? (float)Sc : 0.f;
      const float fSr = nr ? (float)Sr : 0.f;
      const float dc = __fsub_rn(fSc, a.ref[c]);
      const float dr = __fsub_rn(fSr, a.ref[r]);
      const float z = __fmul_rn(a.beta, __fsub_rn(dc, dr));   // no FMA contraction (R15)
      const double zd = (double)z;
      const double loss_p = fmax(-zd, 0.0) + log1p(exp(-fabs(zd)));  // softplus(-z)
      const double sig_neg = 1.0 / (1.0 + exp(zd));                  // sigma(-z)
      const float coef = (float)((double)a.beta * sig_neg * (double)a.invT / a.Pg);
      a.w.seq_coef[c] = coef;
      a.w.seq_coef[r] = -coef;
      // the RESIDENT schedule's parameter warps poll these (ready bit + coefficient, one load)
      st_release_u64(&a.w.seq_cf[c], kCfReady | __float_as_uint(coef));
      st_release_u64(&a.w.seq_cf[r], kCfReady | __float_as_uint(-coef));
      a.seq_logp[c] = fSc;
      a.seq_logp[r] = fSr;
      if (a.z_out) a.z_out[p] = z;
      pv[ODPO_ST_NPAIRS] = 1.0;
      pv[ODPO_ST_LOSS] = loss_p;
      pv[ODPO_ST_NCORRECT] = z > 0.f ? 1.0 : 0.0;
      pv[ODPO_ST_Z] = zd;
      pv[ODPO_ST_RCHOSEN] = (double)a.beta * (double)dc;
      pv[ODPO_ST_RREJ] = (double)a.beta * (double)dr;
      pv[ODPO_ST_SCHOSEN] = (double)fSc;
      pv[ODPO_ST_SREJ] = (double)fSr;
      pv[ODPO_ST_NTOK_CHOSEN] = (double)nc;
      pv[ODPO_ST_NTOK_REJ] = (double)nr;
    }
    flag(a.status, fl);
#ifdef ODPO_DEBUG_LEAD
    if (a.w.dbg_t) a.w.dbg_t[p * 4 + 2] = gtimer();
#endif
    st_release(&a.w.pair_ready[p], 1u);  // publishes this lane's coef / stats writes
    const unsigned done = atom_add_acq_rel(&a.w.counters[C_PAIRS_DONE], 1u);
    last = (done == (unsigned)(a.P - 1));
  }
  last = __shfl_sync(kFull, last, 0);
  if (a.row_scale) {
    // UNSC: the row scales of both sequences, coef_b * mask (0 for an invalid pair)
    float coef = 0.f;
    if (lane == 0 && c >= 0 && r >= 0) coef = a.w.seq_coef[c];
    coef = __shfl_sync(kFull, coef, 0);
    for (int64_t t = lane; t < a.T; t += 32) {
      if (c >= 0) a.row_scale[c * a.T + t] = a.mask[c * a.T + t] ? coef : 0.f;
      if (r >= 0) a.row_scale[r * a.T + t] = a.mask[r * a.T + t] ? -coef : 0.f;
    }
  }
  if (!last) return;
  fence_acq_rel_gpu();
  double acc[ODPO_NSTATS];
#pragma unroll
  for (int k = 0; k < ODPO_NSTATS; ++k) acc[k] = 0.0;
  for (int64_t q = lane; q < a.P; q += 32) {
    const double* pv = a.w.pair_vals + q * ODPO_NSTATS;
#pragma unroll
    for (int k = 0; k < ODPO_NSTATS; ++k) acc[k] += __ldcg(pv + k);
  }
#pragma unroll
  for (int k = 0; k < ODPO_NSTATS; ++k) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) acc[k] += __shfl_down_sync(kFull, acc[k], off);
  }
  if (lane == 0) {
    for (int k = 0; k < ODPO_NSTATS; ++k) a.stats[k] = acc[k];
    a.stats[ODPO_ST_LOSS] = acc[ODPO_ST_LOSS] / a.Pg;
  }
}

// ------------------------------------------------------------------ K3b pair reduce (grid = P)
__global__ void __launch_bounds__(32) k_pair_reduce(LossArgs a) { pair_reduce_warp(a, blockIdx.x); }

// ------------------------------------------------------------------ NEXT-4 vocabulary-parallel merge
// Row statistics of the full vocabulary from W shard partials (m_w, log1p r_w, x_tok, owner),
// merged in rank order with the log1p form: w* = first argmax m_w,
//   R = r_w* + sum_{w != w*} exp(invT (m_w - m*)) (1 + r_w),  lse = invT m* + log1p(R).
// One thread per row.  The token's logit comes from the shard that owns it.
__global__ void k_vp_combine(LossArgs a, const float4* __restrict__ parts, int W) {
  const int64_t rows = a.B * a.T;
  if (a.vp_flags) {
    // in-kernel exchange: wait until every rank has published this epoch's partials into this
    // rank's buffer (acquire, system scope), then read them through L2
    if (threadIdx.x == 0)
      for (int q = 0; q < W; ++q)
        while ((int32_t)(ld_acquire_sys(a.vp_flags + q) - a.vp_epoch) < 0) __nanosleep(64);
    __syncthreads();
  }
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= rows || !a.mask[g]) return;
  int ws = 0;
  float ms = -INFINITY;
  for (int w = 0; w < W; ++w) {
    const float mw = __ldcg(&parts[(int64_t)w * rows + g].x);
    if (mw > ms) { ms = mw; ws = w; }
  }
  uint32_t fl = 0;
  float R = 0.f, xt = 0.f;
  int owners = 0;
  for (int w = 0; w < W; ++w) {
    const float4 pw = __ldcg(&parts[(int64_t)w * rows + g]);
    if (pw.w != 0.f) { xt = pw.z; ++owners; }
    if (w == ws) {
      R += expm1f(pw.y);
    } else if (pw.x != -INFINITY) {
      R += ex2((pw.x - ms) * (a.invT * kLog2e)) * (1.f + expm1f(pw.y));
    }
  }
  const float l1p = log1pf(R);
  float logp = 0.f;
  if (owners != 1) {
    fl |= ODPO_FLAG_TOKEN_RANGE;
  } else {
    logp = __fsub_rn(__fmul_rn(__fsub_rn(xt, ms), a.invT), l1p);
    if (!isfinite(logp)) fl |= ODPO_FLAG_NONFINITE_LOGIT;
  }
  if (!isfinite(ms)) fl |= ODPO_FLAG_NONFINITE_LOGIT;
  a.w.row_m[g] = ms;
  a.w.row_l1p[g] = l1p;
  a.w.row_logp[g] = logp;
  flag(a.status, fl);
}

// Many partials per row (W > 32: the LM-head step's one partial per 256-entry vocabulary tile,
// odpo_lmhead_dpo_step): one warp per row, the same merge with lane-strided partials.  w* = the
// first argmax (max over lanes, then the lowest index among equal maxima); each lane sums its
// partials in index order, then a fixed shfl_down tree: deterministic.
constexpr int kCombineWarps = 8;
__global__ void __launch_bounds__(32 * kCombineWarps) k_vp_combine_wide(LossArgs a,
                                                                        const float4* __restrict__ parts,
                                                                        int W) {
  const int64_t rows = a.B * a.T;
  const int64_t g = (int64_t)blockIdx.x * kCombineWarps + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (g >= rows || !a.mask[g]) return;
  float ms = -INFINITY;
  int ws = INT32_MAX;
  for (int w = lane; w < W; w += 32) {
    const float mw = __ldcg(&parts[(int64_t)w * rows + g].x);
    if (mw > ms) { ms = mw; ws = w; }
  }
#pragma unroll
  for (int off = 16; off; off >>= 1) {
    const float om = __shfl_xor_sync(kFull, ms, off);
    const int ow = __shfl_xor_sync(kFull, ws, off);
    if (om > ms || (om == ms && ow < ws)) { ms = om; ws = ow; }
  }
  if (ws == INT32_MAX) ws = 0;   // every partial -inf: the row is flagged below
  const float k2 = a.invT * kLog2e;
  float R = 0.f, xt = 0.f;
  int owners = 0;
  for (int w = lane; w < W; w += 32) {
    const float4 pw = __ldcg(&parts[(int64_t)w * rows + g]);
    if (pw.w != 0.f) { xt = pw.z; ++owners; }
    if (w == ws) {
      R += expm1f(pw.y);
    } else if (pw.x != -INFINITY) {
      R += ex2((pw.x - ms) * k2) * (1.f + expm1f(pw.y));
    }
  }
  // the token's logit from the (first) owning lane; more or fewer than one owner is flagged
  const unsigned own_mask = __ballot_sync(kFull, owners != 0);
  xt = __shfl_sync(kFull, xt, own_mask ? __ffs(own_mask) - 1 : 0);
#pragma unroll
  for (int off = 16; off; off >>= 1) {
    R += __shfl_down_sync(kFull, R, off);
    owners += __shfl_down_sync(kFull, owners, off);
  }
  if (lane != 0) return;
  uint32_t fl = 0;
  const float l1p = log1pf(R);
  float logp = 0.f;
  if (owners != 1) {
    fl |= ODPO_FLAG_TOKEN_RANGE;
  } else {
    logp = __fsub_rn(__fmul_rn(__fsub_rn(xt, ms), a.invT), l1p);
    if (!isfinite(logp)) fl |= ODPO_FLAG_NONFINITE_LOGIT;
  }
  if (!isfinite(ms)) fl |= ODPO_FLAG_NONFINITE_LOGIT;
  a.w.row_m[g] = ms;
  a.w.row_l1p[g] = l1p;
  a.w.row_logp[g] = logp;
  flag(a.status, fl);
}

// ------------------------------------------------------------------ K6 stretch: stats over peer memory
// The batch-sharded statistics reduction without NCCL: every rank stores
// its 16-double buffer into slot [rank] of every rank's exchange (peer memory), fences and
// publishes the epoch; each rank then waits for the W flags and sums the slots in RANK order,
// so every rank gets the same bits.  One warp each.
__global__ void k_stats_put(const double* __restrict__ stats, VpPut put) {
  const int lane = threadIdx.x;
  const double v = lane < 16 ? stats[lane] : 0.0;
  for (int q = 0; q < put.W; ++q)
    if (lane < 16) reinterpret_cast<double*>(put.parts[q])[put.rank * 16 + lane] = v;
  __syncwarp();
  if (lane == 0) {
    __threadfence_system();
    for (int q = 0; q < put.W; ++q) st_release_sys(put.flags[q] + put.rank, put.epoch);
  }
}

__global__ void k_stats_sum(const double* __restrict__ slots, const uint32_t* flags, int W,
                            uint32_t epoch, double* out) {
  const int lane = threadIdx.x;
  if (lane == 0)
    for (int q = 0; q < W; ++q)
      while ((int32_t)(ld_acquire_sys(flags + q) - epoch) < 0) __nanosleep(64);
  __syncwarp();
  if (lane < 16) {
    double s = 0.0;
    for (int q = 0; q < W; ++q) s += __ldcg(slots + q * 16 + lane);
    out[lane] = s;
  }
}

// ------------------------------------------------------------------ App B known coefficients
// KL proxy (R20): ppl_b = exp(-S_b / n_b) from the row log-probs
// the SEQ engine left in the workspace.  One CTA of 32 warps; warp w sums sequences
// b = w, w + 32, ... (seq_sum_warp's order, so S_b is the engine's own double sum) and keeps
// its partial statistics in b order; the 32 partials are merged in warp order.
constexpr int kPplWarps = 32;
__global__ void __launch_bounds__(32 * kPplWarps) k_seq_ppl(LossArgs a, float* ppl, double* ppl_stats) {
  __shared__ double part[kPplWarps][4];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  for (int64_t b = warp; b < a.B; b += kPplWarps) {
    double S;
    int n;
    seq_sum_warp(a.w.row_logp + b * a.T, a.mask + b * a.T, a.T, S, n);
    if (lane == 0) {
      if (n > 0) {
        const double p = exp(-S / (double)n);
        ppl[b] = (float)p;
        acc[0] += 1.0;
        acc[1] += p;
        acc[2] += S;
        acc[3] += (double)n;
      } else {
        ppl[b] = 1.f;
      }
    }
  }
  if (lane == 0)
    for (int k = 0; k < 4; ++k) part[warp][k] = acc[k];
  __syncthreads();
  if (threadIdx.x < 4) {
    double s = 0.0;
    for (int w = 0; w < kPplWarps; ++w) s += part[w][threadIdx.x];
    ppl_stats[threadIdx.x] = s;
  }
}

// RLOO / CoPG: coef_b = A_b invT / (2 P_global); Best-of-2 SFT: invT / P_global on the chosen
// completion, 0 on the other.  One thread per pair.
__global__ void k_pg_coef(LossArgs a) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= a.P) return;
  int64_t c, r;
  pair_seqs(a, p, c, r);
  if (c < 0 || r < 0) return;
  const double scale = (double)a.invT / (2.0 * a.Pg);
  if (a.pg_kind == ODPO_PG_BEST_OF_K_SFT) {
    a.w.seq_coef[c] = (float)(2.0 * scale);
    a.w.seq_coef[r] = 0.f;
  } else {
    const double A0 = (double)a.rewards[c] - (double)a.rewards[r];
    a.w.seq_coef[c] = (float)(A0 * scale);
    a.w.seq_coef[r] = (float)(-A0 * scale);
  }
}

// ------------------------------------------------------------------ K4 row backward (grid = rows)
// Short rows (vocabulary shards of NEXT-4): one WARP per row, 8 rows per CTA, each lane with 8
// 16-byte vectors in flight -- one 512-thread CTA per 12-32 KB row spends its time being
// scheduled.  Same per-element arithmetic as row_backward (bit-identical output).
constexpr int kWarpRowsPerCta = 8;
template <int DT>
__global__ void __launch_bounds__(32 * kWarpRowsPerCta) k_row_bwd_warp(LossArgs a) {
  constexpr int N = Traits<DT>::N;
  constexpr int U = 8;
  const int lane = threadIdx.x & 31;
  const int64_t g = (int64_t)blockIdx.x * kWarpRowsPerCta + (threadIdx.x >> 5);
  if (g >= a.B * a.T) return;
  const int64_t b = g / a.T, t = g % a.T;
  const int V = (int)a.V;
  const int nvec = V / N, tail = V - nvec * N;
  uint4* vout = reinterpret_cast<uint4*>(drow_ptr(a, b, t));
  if (a.w.seq_pair[b] < 0 || !a.mask[g]) {
    for (int i = lane; i < nvec; i += 32) st16_stream(vout + i, make_uint4(0, 0, 0, 0));
    if (lane < tail) Traits<DT>::store1(vout, (int64_t)nvec * N + lane, 0.f);
    return;
  }
  const float coef = a.w.seq_coef[b];
  const int64_t tl = (int64_t)a.tokens[g] - a.tok_off;
  const int tok = (tl >= 0 && tl < V) ? (int)tl : -1;
  const float k2 = a.invT * kLog2e;
  const float rm = a.w.row_m[g];
  const float c = bwd_const<DT>(rm, a.w.row_l1p[g], k2, coef);
  const float gtok = coef * expm1f(a.w.row_logp[g]);
  const bool neg = coef < 0.f;
  const uint4* vrow = reinterpret_cast<const uint4*>(row_ptr(a, b, t));
  for (int base = lane; base < nvec; base += 32 * U) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i = base + 32 * u;
      if (i < nvec) v[u] = ld16<LD_STREAM>(vrow + i, 0);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i = base + 32 * u;
      if (i < nvec)
        st16_stream(vout + i, neg ? bwd_vec<DT, 0, true>(v[u], k2, c, rm) : bwd_vec<DT, 0, false>(v[u], k2, c, rm));
    }
  }
  if (lane < tail) {
    const int64_t vv = (int64_t)nvec * N + lane;
    const float x = Traits<DT>::load1(vrow, vv);
    Traits<DT>::store1(vout, vv, vv == tok ? gtok : copysignf(ex2(bwd_arg<DT>(x, k2, c, rm)), coef));
  }
  // onehot entry: the lane that stored tok's vector overwrites it (program order)
  if (tok >= 0 && tok < nvec * N && (tok / N) % 32 == lane) Traits<DT>::store1(vout, tok, gtok);
}

// Short-row forward partials (NEXT-4 vocabulary shards): one warp per row, each lane with
// 8 16-byte vectors per batch, the online (m, r) update of the engine (mr_batch), the
// fixed-order warp merge; writes the shard partial (m, log1p r, x_tok, owns tok) as the
// engine's vocabulary-parallel epilogue does.
__device__ __forceinline__ void vp_store(const LossArgs& a, int64_t g, float4 v) {
  if (a.put.W > 0) {
    const int64_t rows = a.B * a.T;
    for (int q = 0; q < a.put.W; ++q) a.put.parts[q][(int64_t)a.put.rank * rows + g] = v;
  } else {
    a.vp_parts[g] = v;
  }
}
// End of a put kernel (every thread of the CTA calls it): each CTA releases its partial stores
// at GPU scope into the grid's counter; the last CTA acquires them all, and ONE system-scope
// fence + release per flag makes them (by causality) visible to the peer GPUs / processes before
// the epoch they poll for.
__device__ __forceinline__ void vp_signal(const LossArgs& a) {
  if (a.put.W == 0) return;
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned n = atom_add_acq_rel(a.put.done, 1u);   // release (gpu scope) + acquire
    if (n == gridDim.x - 1) {
      __threadfence_system();
      *a.put.done = 0u;   // the next call is stream-ordered after this kernel
      for (int q = 0; q < a.put.W; ++q) st_release_sys(a.put.flags[q] + a.put.rank, a.put.epoch);
    }
  }
}

template <int DT>
__device__ __forceinline__ void vp_partials_row(const LossArgs& a);
template <int DT>
__global__ void __launch_bounds__(32 * kWarpRowsPerCta) k_vp_partials_warp(LossArgs a) {
  vp_partials_row<DT>(a);
  vp_signal(a);
}

template <int DT>
__device__ __forceinline__ void vp_partials_row(const LossArgs& a) {
  constexpr int N = Traits<DT>::N;
  constexpr int U = 8;
  const int lane = threadIdx.x & 31;
  const int64_t g = (int64_t)blockIdx.x * kWarpRowsPerCta + (threadIdx.x >> 5);
  if (g >= a.B * a.T) return;
  if (!a.mask[g]) {
    if (lane == 0) vp_store(a, g, make_float4(-INFINITY, 0.f, 0.f, 0.f));
    return;
  }
  const int64_t b = g / a.T, t = g % a.T;
  const int V = (int)a.V;
  const int nvec = V / N, tail = V - nvec * N;
  const float k2 = a.invT * kLog2e;
  const int64_t tl = (int64_t)a.tokens[g] - a.tok_off;
  const int tok = (tl >= 0 && tl < V) ? (int)tl : -1;
  const uint4* vrow = reinterpret_cast<const uint4*>(row_ptr(a, b, t));
  const uint32_t NI = Traits<DT>::kNegInfWord;
  MR s{-INFINITY, 0.f};
  float xt = 0.f;
  for (int base = lane; base < nvec; base += 32 * U) {
    uint4 v[U];
    bool any = false;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i = base + 32 * u;
      any |= i < nvec;
      v[u] = i < nvec ? ld16<LD_STREAM>(vrow + i, 0) : make_uint4(NI, NI, NI, NI);
    }
    if (any) mr_batch<DT, U, 0>(v, k2, s.m, s.r);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i = base + 32 * u;
      if (tok >= 0 && i < nvec && i == tok / N) {
        float f[N];
        Traits<DT>::unpack(v[u], f);
        float x = f[0];
#pragma unroll
        for (int j = 1; j < N; ++j) x = (tok % N == j) ? f[j] : x;
        xt = x;
      }
    }
  }
  if (lane < tail) {
    const int64_t vv = (int64_t)nvec * N + lane;
    const float x = Traits<DT>::load1(vrow, vv);
    s = mr_push1(s, x, k2);
    if (vv == tok) xt = x;
  }
  const MR v = warp_merge(s, k2);
  // the sampled logit from the lane that read it
  int src = 0;
  if (tok >= 0) src = tok < nvec * N ? (tok / N) % 32 : tok - nvec * N;
  xt = __shfl_sync(kFull, xt, src);
  if (lane == 0) {
    uint32_t fl = 0;
    const int64_t gt = tl + a.tok_off;
    if (gt < 0 || gt >= a.V_total) fl |= ODPO_FLAG_TOKEN_RANGE;
    if (isnan(v.m) || v.m == INFINITY || !isfinite(v.r)) fl |= ODPO_FLAG_NONFINITE_LOGIT;
    const bool own = tok >= 0;
    vp_store(a, g, make_float4(v.m, log1pf(v.r), own ? xt : 0.f, own ? 1.f : 0.f));
    flag(a.status, fl);
  }
}

template <int DT, int NPB>
__global__ void __launch_bounds__(kRowThreads, 2) k_row_bwd(LossArgs a) {
  const int64_t g = blockIdx.x;
  const int64_t b = g / a.T, t = g % a.T;
  char* drow = drow_ptr(a, b, t);
  if (a.w.seq_pair[b] < 0 || !a.mask[g]) {
    row_zero<DT>(drow, (int)a.V);
    return;
  }
  const float coef = a.w.seq_coef[b];
  const int64_t tl = (int64_t)a.tokens[g] - a.tok_off;   // shard-local (vocabulary-parallel)
  const int tok = (tl >= 0 && tl < a.V) ? (int)tl : -1;
  row_backward<DT, LD_STREAM, NPB>(row_ptr(a, b, t), drow, (int)a.V, tok, a.invT, a.w.row_m[g],
                              a.w.row_l1p[g], a.w.row_logp[g], coef, 0);
}

// K4s: the same backward with each row cut into pieces, one CTA per piece, every piece moved in
// ONE batch of loads then stores (THR threads x U vectors of VW bytes).  Measured on B200
// (profiles/r02/copy/): a copy kernel whose CTAs each move one ~32 KB batch reaches 6.98 TB/s of
// read+write traffic, against 6.57 for cudaMemcpy and 6.60-6.63 for one 512-thread CTA looping
// over a 256 KB (LLaMA) row; 32-byte vectors (sm_100 LDG/STG.256) help on the long rows.  The
// per-element arithmetic is bwd_vec's, so the output is bit-identical to k_row_bwd's.
// Pieces: S = ceil(nv / (THR U)) per row, per = ceil(nv / S) vectors each (even split).
// VW = 32 needs 32-byte aligned rows (host check); VW = 16 is the 16-byte fallback.
template <int VW>
struct VecT;
template <>
struct VecT<16> {
  uint4 h[1];
};
template <>
struct VecT<32> {
  uint4 h[2];
};
template <int VW>
__device__ __forceinline__ VecT<VW> ldv(const char* p) {
  VecT<VW> v;
  if constexpr (VW == 32) {
    asm volatile("ld.global.nc.L1::no_allocate.L2::evict_first.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(v.h[0].x), "=r"(v.h[0].y), "=r"(v.h[0].z), "=r"(v.h[0].w),
                   "=r"(v.h[1].x), "=r"(v.h[1].y), "=r"(v.h[1].z), "=r"(v.h[1].w)
                 : "l"(p));
  } else {
    v.h[0] = ld16<LD_STREAM>(reinterpret_cast<const uint4*>(p), 0);
  }
  return v;
}
template <int VW>
__device__ __forceinline__ void stv(char* p, const VecT<VW>& v) {
  if constexpr (VW == 32) {
    asm volatile("st.global.L1::no_allocate.L2::evict_first.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};"
                 ::"l"(p), "r"(v.h[0].x), "r"(v.h[0].y), "r"(v.h[0].z), "r"(v.h[0].w),
                   "r"(v.h[1].x), "r"(v.h[1].y), "r"(v.h[1].z), "r"(v.h[1].w)
                 : "memory");
  } else {
    st16_stream(reinterpret_cast<uint4*>(p), v.h[0]);
  }
}

template <int DT, int NPB, int THR, int U, int VW>
__global__ void __launch_bounds__(THR) k_row_bwd_split(LossArgs a) {
  constexpr int N = Traits<DT>::N;            // elements per 16 bytes
  constexpr int E = N * (VW / 16);            // elements per vector
  const int V = (int)a.V;
  const int nv = V / E;                       // whole vectors per row
  const int S = (nv + THR * U - 1) / (THR * U);
  const int64_t g = blockIdx.x / (S > 0 ? S : 1);
  const int s = (int)(blockIdx.x - g * (S > 0 ? S : 1));
  const int per = S > 0 ? (nv + S - 1) / S : 0;
  const int v0 = s * per, v1 = min(nv, v0 + per);
  const int64_t b = g / a.T, t = g % a.T;
  char* drow = drow_ptr(a, b, t);
  const char* row = row_ptr(a, b, t);
  const bool last = s == (S > 0 ? S : 1) - 1;
  const int tail = V - nv * E;                 // elements after the last whole vector
  if (a.w.seq_pair[b] < 0 || !a.mask[g]) {
    VecT<VW> z;
#pragma unroll
    for (int h = 0; h < VW / 16; ++h) z.h[h] = make_uint4(0, 0, 0, 0);
    for (int i = v0 + (int)threadIdx.x; i < v1; i += THR) stv<VW>(drow + (int64_t)i * VW, z);
    if (last && (int)threadIdx.x < tail) Traits<DT>::store1(drow, (int64_t)nv * E + threadIdx.x, 0.f);
    return;
  }
  const float coef = a.w.seq_coef[b];
  const int64_t tl = (int64_t)a.tokens[g] - a.tok_off;   // shard-local (vocabulary-parallel)
  const int tok = (tl >= 0 && tl < V) ? (int)tl : -1;
  const float k2 = a.invT * kLog2e;
  const float m = a.w.row_m[g];
  const float c = bwd_const<DT>(m, a.w.row_l1p[g], k2, coef);
  const bool neg = coef < 0.f;
  VecT<VW> v[U];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const int i = v0 + (int)threadIdx.x + u * THR;
    if (i < v1) v[u] = ldv<VW>(row + (int64_t)i * VW);
  }
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const int i = v0 + (int)threadIdx.x + u * THR;
    if (i < v1) {
#pragma unroll
      for (int h = 0; h < VW / 16; ++h)
        v[u].h[h] = neg ? bwd_vec<DT, NPB, true>(v[u].h[h], k2, c, m) : bwd_vec<DT, NPB, false>(v[u].h[h], k2, c, m);
      stv<VW>(drow + (int64_t)i * VW, v[u]);
    }
  }
  const float gtok = coef * expm1f(a.w.row_logp[g]);
  if (last && (int)threadIdx.x < tail) {
    const int64_t vv = (int64_t)nv * E + threadIdx.x;
    const float x = Traits<DT>::load1(row, vv);
    Traits<DT>::store1(drow, vv, (vv == tok) ? gtok : copysignf(ex2(bwd_arg<DT>(x, k2, c, m)), coef));
  }
  // onehot entry: written by the thread that stored tok's vector (program order)
  if (tok >= 0 && tok < nv * E) {
    const int iv = tok / E;
    if (iv >= v0 && iv < v1 && (iv - v0) % THR == (int)threadIdx.x) Traits<DT>::store1(drow, tok, gtok);
  }
}

#if ODPO_EXPERIMENTAL   // measured slower than the row engine (profiles/r02/split/)
// K5c: the factored gradient (G = softmax - onehot; coef*G when the coefficient is known
// before the call, App B) with each row split over a thread-block cluster of CS CTAs, one
// vocabulary piece of <= THR*U vectors per CTA, held in registers from its load to its store:
//   load the piece (all loads in flight) -> the piece's online (m, r) and x_tok -> fixed-order
//   warp / CTA merge -> the CTA partial stored into every peer's shared memory (DSMEM) ->
//   cluster barrier -> every CTA merges the CS partials in rank order (the same bits in every
//   CTA) -> G from the registers -> rank 0 writes the row statistics and counts the row into
//   its pair (the last row of a pair runs the pair reduction, as in the engine).
// Exactly one HBM read and one write of every row, with no L2 re-read (the engine's factored
// mode re-reads each row from L2 and loses 10-16% of the re-reads to misses), and each CTA
// moves one batch: the access pattern measured fastest for read+write traffic on B200
// (profiles/r02/copy/).  Deterministic (a fixed reduction tree per (CS, THR, U)); the tree
// differs from the engine's, so its results agree with the engine's to rounding, not bitwise.
// Units: the pair-ordered rows of the engine's tickets [0, 2PT); CTAs past them zero the rows of
// unreferenced sequences (grid-stride over k_prep's list).
template <int DT, int CS, int THR, int U, int VW>
__global__ void __launch_bounds__(THR) k_unsc_split(const __grid_constant__ LossArgs a) {
  constexpr int N = Traits<DT>::N;
  constexpr int H = VW / 16;                 // 16-byte halves per vector
  constexpr int E = N * H;                   // elements per vector
  constexpr int NB = U * H;                  // 16-byte words per thread
  constexpr int NW = THR / 32;
  __shared__ float s_wm[NW], s_wr[NW], s_wx[NW];
  __shared__ int s_wo[NW];
  __shared__ float4 s_cp[CS];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int V = (int)a.V;
  const int nv = V / E;
  const int per = (nv + CS - 1) / CS;
  const int64_t T = a.T, R = 2 * T, totalF = a.P * R;
  const int64_t unit = blockIdx.x / CS;
  const int rank = (int)(blockIdx.x % CS);   // == %cluster_ctarank (1-D clusters along x)
  const int tail = V - nv * E;
  if (unit >= totalF) {   // zero workers: rows of sequences no pair references
    const int64_t nz = (int64_t)__ldcg(&a.w.counters[C_NUNREF]) * T;
    const int64_t z0 = (int64_t)blockIdx.x - totalF * CS, nzw = (int64_t)gridDim.x - totalF * CS;
    for (int64_t z = z0; z < nz; z += nzw) {
      const int64_t s = __ldcg(a.w.unref + z / T), t = z % T;
      char* drow = drow_ptr(a, s, t);
      VecT<VW> zv;
#pragma unroll
      for (int h = 0; h < H; ++h) zv.h[h] = make_uint4(0, 0, 0, 0);
      for (int i = tid; i < nv; i += THR) stv<VW>(drow + (int64_t)i * VW, zv);
      if (tid < tail) Traits<DT>::store1(drow, (int64_t)nv * E + tid, 0.f);
      if (tid == 0 && a.row_scale) a.row_scale[s * T + t] = 0.f;
    }
    return;
  }
  if (CS > 1) asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");  // started
  const int64_t p = unit / R, j = unit % R;
  int64_t c, r;
  pair_seqs(a, p, c, r);
  const int64_t s = j < T ? c : r, t = j < T ? j : j - T;
  const int64_t g = s >= 0 ? s * T + t : 0;
  const bool live = s >= 0 && a.mask[g];
  const int v0 = rank * per, v1 = min(nv, v0 + per);
  const bool tail_owner = rank == CS - 1;
  const float k2 = a.invT * kLog2e;
  if (!live) {   // the engine's K_FSKIP (counted once) + K_ZERO
    if (CS > 1) asm volatile("barrier.cluster.wait.aligned;" ::: "memory");
    if (s >= 0) {
      char* drow = drow_ptr(a, s, t);
      VecT<VW> zv;
#pragma unroll
      for (int h = 0; h < H; ++h) zv.h[h] = make_uint4(0, 0, 0, 0);
      for (int i = v0 + tid; i < v1; i += THR) stv<VW>(drow + (int64_t)i * VW, zv);
      if (tail_owner && tid < tail) Traits<DT>::store1(drow, (int64_t)nv * E + tid, 0.f);
      if (rank == 0 && tid == 0 && a.row_scale) a.row_scale[g] = 0.f;
    }
    if (rank == 0 && warp == 0) {
      unsigned last = 0;
      if (lane == 0) last = atom_add_acq_rel(&a.w.pair_cnt[p], 1u) == (unsigned)R - 1u;
      last = __shfl_sync(kFull, last, 0);
      if (last) {
        fence_acq_rel_gpu();
        pair_reduce_warp(a, p);
      }
    }
    return;
  }
  const char* row = row_ptr(a, s, t);
  char* drow = drow_ptr(a, s, t);
  const int tok = a.tokens[g];
  // ---- the piece, all loads in flight
  uint4 w[NB];
  const uint32_t NI = Traits<DT>::kNegInfWord;
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const int i = v0 + tid + u * THR;
    if (i < v1) {
      const VecT<VW> x = ldv<VW>(row + (int64_t)i * VW);
#pragma unroll
      for (int h = 0; h < H; ++h) w[u * H + h] = x.h[h];
    } else {
#pragma unroll
      for (int h = 0; h < H; ++h) w[u * H + h] = make_uint4(NI, NI, NI, NI);
    }
  }
  MR st{-INFINITY, 0.f};
  mr_batch<DT, NB, 0>(w, k2, st.m, st.r);
  float xt = 0.f;
  int own = 0;
  const int tv = (tok >= 0 && tok < nv * E) ? tok / E : -1;
  const bool tok_mine = tv >= v0 && tv < v1 && (tv - v0) % THR == tid;
  if (tok_mine) {
    const int u = (tv - v0) / THR, e = tok % E;
    const int kk = u * H + e / N;
    uint4 sel = w[0];
#pragma unroll
    for (int k = 1; k < NB; ++k) sel = (k == kk) ? w[k] : sel;   // register selects, no local copy
    float f[N];
    Traits<DT>::unpack(sel, f);
    xt = f[0];
#pragma unroll
    for (int q = 1; q < N; ++q) xt = (e % N == q) ? f[q] : xt;
    own = 1;
  }
  if (tail_owner && tid < tail) {
    const int64_t vv = (int64_t)nv * E + tid;
    const float x = Traits<DT>::load1(row, vv);
    st = mr_push1(st, x, k2);
    if (vv == tok) { xt = x; own = 1; }
  }
  // ---- fixed-order merges: warp, CTA, then the cluster's CS partials in rank order
  const MR wm = warp_merge(st, k2);
  const unsigned ob = __ballot_sync(kFull, own);
  const float wx = __shfl_sync(kFull, xt, ob ? __ffs(ob) - 1 : 0);
  if (lane == 0) { s_wm[warp] = wm.m; s_wr[warp] = wm.r; s_wx[warp] = wx; s_wo[warp] = ob != 0; }
  __syncthreads();
  if (warp == 0) {
    MR x = lane < NW ? MR{s_wm[lane], s_wr[lane]} : MR{-INFINITY, 0.f};
    x = warp_merge(x, k2);
    const int o = lane < NW ? s_wo[lane] : 0;
    const unsigned ob2 = __ballot_sync(kFull, o);
    const float cx = __shfl_sync(kFull, lane < NW ? s_wx[lane] : 0.f, ob2 ? __ffs(ob2) - 1 : 0);
    if (CS > 1) {
      const float pm = __shfl_sync(kFull, x.m, 0), pr = __shfl_sync(kFull, x.r, 0);
      asm volatile("barrier.cluster.wait.aligned;" ::: "memory");  // every peer has started
      if (lane < CS) {   // lane q stores this CTA's partial into CTA q's slot [rank]
        const uint32_t dst = mapa((uint32_t)__cvta_generic_to_shared(&s_cp[rank]), (uint32_t)lane);
        st_cl_u32(dst, __float_as_uint(pm));
        st_cl_u32(dst + 4, __float_as_uint(pr));
        st_cl_u32(dst + 8, __float_as_uint(cx));
        st_cl_u32(dst + 12, __float_as_uint(ob2 ? 1.f : 0.f));
      }
    } else if (lane == 0) {
      s_cp[0] = make_float4(x.m, x.r, cx, ob2 ? 1.f : 0.f);
    }
  } else if (CS > 1) {
    asm volatile("barrier.cluster.wait.aligned;" ::: "memory");
  }
  if (CS > 1) cluster_sync_all();
  else __syncthreads();
  MR u{-INFINITY, 0.f};
  float xr = 0.f;
#pragma unroll
  for (int q = 0; q < CS; ++q) {
    const float4 cp = s_cp[q];
    u = mr_merge(u, MR{cp.x, cp.y}, k2);
    if (cp.w != 0.f) xr = cp.z;
  }
  const float l1p = log1pf(u.r);
  const bool tok_ok = tok >= 0 && tok < V;
  const float logp = tok_ok ? __fsub_rn(__fmul_rn(__fsub_rn(xr, u.m), a.invT), l1p) : 0.f;
  // ---- G (coef * G with a known coefficient) straight from the registers
  const float cf = a.coef_known ? __ldcg(a.w.seq_coef + s) : 1.f;
  const float cc = cf != 0.f ? bwd_const<DT>(u.m, l1p, k2, cf) : INFINITY;
  const float gtok = cf * expm1f(logp);
  const bool neg = cf < 0.f;
#pragma unroll
  for (int q = 0; q < U; ++q) {
    const int i = v0 + tid + q * THR;
    if (i < v1) {
      VecT<VW> o;
#pragma unroll
      for (int h = 0; h < H; ++h)
        o.h[h] = neg ? bwd_vec<DT, 0, true>(w[q * H + h], k2, cc, u.m)
                     : bwd_vec<DT, 0, false>(w[q * H + h], k2, cc, u.m);
      stv<VW>(drow + (int64_t)i * VW, o);
    }
  }
  if (tail_owner && tid < tail) {
    const int64_t vv = (int64_t)nv * E + tid;
    const float x = Traits<DT>::load1(row, vv);
    Traits<DT>::store1(drow, vv, vv == tok ? gtok : copysignf(ex2(bwd_arg<DT>(x, k2, cc, u.m)), cf));
  }
  if (tok_mine) Traits<DT>::store1(drow, tok, gtok);   // onehot entry (program order)
  // ---- row statistics, then the row counts into its pair
  if (rank == 0 && warp == 0) {
    unsigned last = 0;
    if (lane == 0) {
      uint32_t fl = 0;
      if (!tok_ok) fl |= ODPO_FLAG_TOKEN_RANGE;
      else if (!isfinite(logp)) fl |= ODPO_FLAG_NONFINITE_LOGIT;
      if (!isfinite(u.m) || !isfinite(u.r)) fl |= ODPO_FLAG_NONFINITE_LOGIT;
      a.w.row_m[g] = u.m;
      a.w.row_l1p[g] = l1p;
      a.w.row_logp[g] = logp;
      flag(a.status, fl);
      last = atom_add_acq_rel(&a.w.pair_cnt[p], 1u) == (unsigned)R - 1u;
    }
    last = __shfl_sync(kFull, last, 0);
    if (last) {
      fence_acq_rel_gpu();
      pair_reduce_warp(a, p);
    }
  }
}

// K5t: the same split, the piece staged in shared memory by ONE 1-D bulk TMA copy instead of
// registers, so a CTA holds no data registers and up to 7 CTAs (32 KB pieces) share an SM:
// more bytes in flight per SM while other CTAs of the SM sit in their merge / barrier phases.
template <int DT, int CS, int THR>
__global__ void __launch_bounds__(THR) k_unsc_tma(const __grid_constant__ LossArgs a) {
  constexpr int N = Traits<DT>::N;
  constexpr int NW = THR / 32;
  extern __shared__ __align__(128) uint4 sm_piece[];
  __shared__ __align__(8) uint64_t s_bar;
  __shared__ float s_wm[NW], s_wr[NW];
  __shared__ float4 s_cp[CS];
  __shared__ float s_xt;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int V = (int)a.V;
  const int nv = V / N;                      // whole 16-byte vectors per row
  const int per = (nv + CS - 1) / CS;
  const int64_t T = a.T, R = 2 * T, totalF = a.P * R;
  const int64_t unit = blockIdx.x / CS;
  const int rank = (int)(blockIdx.x % CS);
  const int tail = V - nv * N;
  if (unit >= totalF) {   // zero workers: rows of sequences no pair references
    const int64_t nz = (int64_t)__ldcg(&a.w.counters[C_NUNREF]) * T;
    const int64_t z0 = (int64_t)blockIdx.x - totalF * CS, nzw = (int64_t)gridDim.x - totalF * CS;
    for (int64_t z = z0; z < nz; z += nzw) {
      const int64_t s = __ldcg(a.w.unref + z / T), t = z % T;
      uint4* drow = reinterpret_cast<uint4*>(drow_ptr(a, s, t));
      for (int i = tid; i < nv; i += THR) st16_stream(drow + i, make_uint4(0, 0, 0, 0));
      if (tid < tail) Traits<DT>::store1(drow, (int64_t)nv * N + tid, 0.f);
      if (tid == 0 && a.row_scale) a.row_scale[s * T + t] = 0.f;
    }
    return;
  }
  if (CS > 1) asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");  // started
  const int64_t p = unit / R, j = unit % R;
  int64_t c, r;
  pair_seqs(a, p, c, r);
  const int64_t s = j < T ? c : r, t = j < T ? j : j - T;
  const int64_t g = s >= 0 ? s * T + t : 0;
  const bool live = s >= 0 && a.mask[g];
  const int v0 = rank * per, v1 = min(nv, v0 + per), n = max(v1 - v0, 0);
  const bool tail_owner = rank == CS - 1;
  const float k2 = a.invT * kLog2e;
  if (!live) {   // the engine's K_FSKIP (counted once) + K_ZERO
    if (CS > 1) asm volatile("barrier.cluster.wait.aligned;" ::: "memory");
    if (s >= 0) {
      uint4* drow = reinterpret_cast<uint4*>(drow_ptr(a, s, t));
      for (int i = v0 + tid; i < v1; i += THR) st16_stream(drow + i, make_uint4(0, 0, 0, 0));
      if (tail_owner && tid < tail) Traits<DT>::store1(drow, (int64_t)nv * N + tid, 0.f);
      if (rank == 0 && tid == 0 && a.row_scale) a.row_scale[g] = 0.f;
    }
    if (rank == 0 && warp == 0) {
      unsigned last = 0;
      if (lane == 0) last = atom_add_acq_rel(&a.w.pair_cnt[p], 1u) == (unsigned)R - 1u;
      last = __shfl_sync(kFull, last, 0);
      if (last) {
        fence_acq_rel_gpu();
        pair_reduce_warp(a, p);
      }
    }
    return;
  }
  const char* row = row_ptr(a, s, t);
  char* drow = drow_ptr(a, s, t);
  const uint32_t bar = smem_u32(&s_bar);
  if (tid == 0) {
    mbar_init(&s_bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if (n > 0) {
      mbar_arrive_tx(bar, (uint32_t)n * 16u);
      tma_load_1d(smem_u32(sm_piece), row + (int64_t)v0 * 16, (uint32_t)n * 16u, bar,
                  policy_evict_first());
    } else {
      mbar_arrive(bar);
    }
  }
  const int tok = a.tokens[g];
  const int tv = (tok >= 0 && tok < nv * N) ? tok / N : -1;
  MR st{-INFINITY, 0.f};
  float xt_tail = 0.f;
  bool own_tail = false;
  if (tail_owner && tid < tail) {   // the row's last V mod N elements, straight from HBM
    const int64_t vv = (int64_t)nv * N + tid;
    const float x = Traits<DT>::load1(row, vv);
    st = mr_push1(st, x, k2);
    if (vv == tok) { xt_tail = x; own_tail = true; }
  }
  __syncthreads();          // the barrier is initialised before anyone waits on it
  mbar_wait(bar, 0);
  const uint32_t NI = Traits<DT>::kNegInfWord;
  for (int base = tid; base < n; base += 8 * THR) {
    uint4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int i = base + u * THR;
      v[u] = i < n ? sm_piece[i] : make_uint4(NI, NI, NI, NI);
    }
    mr_batch<DT, 8, 0>(v, k2, st.m, st.r);
  }
  const MR wm = warp_merge(st, k2);
  const unsigned otb = __ballot_sync(kFull, own_tail);
  if (otb) {
    const float x = __shfl_sync(kFull, xt_tail, __ffs(otb) - 1);
    if (lane == 0) s_xt = x;
  }
  if (tid == 0 && tv >= v0 && tv < v1) {
    float f[N];
    Traits<DT>::unpack(sm_piece[tv - v0], f);
    float x = f[0];
#pragma unroll
    for (int q = 1; q < N; ++q) x = (tok % N == q) ? f[q] : x;
    s_xt = x;
  }
  if (lane == 0) { s_wm[warp] = wm.m; s_wr[warp] = wm.r; }
  __syncthreads();
  if (warp == 0) {
    MR x = lane < NW ? MR{s_wm[lane], s_wr[lane]} : MR{-INFINITY, 0.f};
    x = warp_merge(x, k2);
    const bool own = (tv >= v0 && tv < v1) || (tail_owner && tok >= nv * N && tok < V);
    const float cx = own ? s_xt : 0.f;
    const float pm = __shfl_sync(kFull, x.m, 0), pr = __shfl_sync(kFull, x.r, 0);
    if (CS > 1) {
      asm volatile("barrier.cluster.wait.aligned;" ::: "memory");  // every peer has started
      if (lane < CS) {
        const uint32_t dst = mapa((uint32_t)__cvta_generic_to_shared(&s_cp[rank]), (uint32_t)lane);
        st_cl_u32(dst, __float_as_uint(pm));
        st_cl_u32(dst + 4, __float_as_uint(pr));
        st_cl_u32(dst + 8, __float_as_uint(cx));
        st_cl_u32(dst + 12, __float_as_uint(own ? 1.f : 0.f));
      }
    } else if (lane == 0) {
      s_cp[0] = make_float4(pm, pr, cx, own ? 1.f : 0.f);
    }
  } else if (CS > 1) {
    asm volatile("barrier.cluster.wait.aligned;" ::: "memory");
  }
  if (CS > 1) cluster_sync_all();
  else __syncthreads();
  MR u{-INFINITY, 0.f};
  float xr = 0.f;
#pragma unroll
  for (int q = 0; q < CS; ++q) {
    const float4 cp = s_cp[q];
    u = mr_merge(u, MR{cp.x, cp.y}, k2);
    if (cp.w != 0.f) xr = cp.z;
  }
  const float l1p = log1pf(u.r);
  const bool tok_ok = tok >= 0 && tok < V;
  const float logp = tok_ok ? __fsub_rn(__fmul_rn(__fsub_rn(xr, u.m), a.invT), l1p) : 0.f;
  const float cf = a.coef_known ? __ldcg(a.w.seq_coef + s) : 1.f;
  const float cc = cf != 0.f ? bwd_const<DT>(u.m, l1p, k2, cf) : INFINITY;
  const float gtok = cf * expm1f(logp);
  uint4* vout = reinterpret_cast<uint4*>(drow) + v0;
  if (cf < 0.f) {
    for (int i = tid; i < n; i += THR) st16_stream(vout + i, bwd_vec<DT, 0, true>(sm_piece[i], k2, cc, u.m));
  } else {
    for (int i = tid; i < n; i += THR) st16_stream(vout + i, bwd_vec<DT, 0, false>(sm_piece[i], k2, cc, u.m));
  }
  if (tail_owner && tid < tail) {
    const int64_t vv = (int64_t)nv * N + tid;
    const float x = Traits<DT>::load1(row, vv);
    Traits<DT>::store1(drow, vv, vv == tok ? gtok : copysignf(ex2(bwd_arg<DT>(x, k2, cc, u.m)), cf));
  }
  if (tv >= v0 && tv < v1 && (tv - v0) % THR == tid) Traits<DT>::store1(drow, tok, gtok);
  if (rank == 0 && warp == 0) {
    unsigned last = 0;
    if (lane == 0) {
      uint32_t fl = 0;
      if (!tok_ok) fl |= ODPO_FLAG_TOKEN_RANGE;
      else if (!isfinite(logp)) fl |= ODPO_FLAG_NONFINITE_LOGIT;
      if (!isfinite(u.m) || !isfinite(u.r)) fl |= ODPO_FLAG_NONFINITE_LOGIT;
      a.w.row_m[g] = u.m;
      a.w.row_l1p[g] = l1p;
      a.w.row_logp[g] = logp;
      flag(a.status, fl);
      last = atom_add_acq_rel(&a.w.pair_cnt[p], 1u) == (unsigned)R - 1u;
    }
    last = __shfl_sync(kFull, last, 0);
    if (last) {
      fence_acq_rel_gpu();
      pair_reduce_warp(a, p);
    }
  }
}

#endif  // ODPO_EXPERIMENTAL

// ------------------------------------------------------------------ the TMA-ring engine
// M_SEQ: forward rows only.  M_FUSED: pair-scheduled forward + scaled backward.  M_UNSC: each
// row's forward pass and then its unscaled backward G = softmax - onehot in the same CTA (the
// re-read is one row behind, so it is served from L2); the pair reducer writes row_scale.
enum { M_SEQ = 0, M_FUSED = 1, M_UNSC = 2, M_NMODES = 3 };
#ifndef ODPO_BREV
#define ODPO_BREV 1
#endif
constexpr bool kBrev = ODPO_BREV != 0;   // factored backward rows stream last chunk first

// Fused dispatch (adaptive, per-pair backward counters).  Forward rows are dispensed in pair
// order from one counter (C_TICKET).  Backward rows are dispensed pair by pair: C_BPAIR is the
// oldest pair with undispensed backward rows, and pair_bcnt[p] hands out that pair's 2T rows.
// A producer takes a backward row only from a pair whose forward pass has completed (ready
// flag), so a queued backward row never waits; otherwise it takes a forward row, and forward
// rows never wait.  Once every forward row is dispensed a producer with nothing queued may
// wait for the next pair to complete -- its forward rows are all dispensed and progressing --
// so the kernel cannot deadlock (no co-residency assumption).  The backward pass trails the
// forward pass by the completion latency only, which keeps a pair's logits L2-resident for
// the backward re-read.  Zero rows of unreferenced sequences (C_ZTICKET) come last.
struct Dispatch {
  bool f_exh;
  int64_t ready_pair;  // a pair known ready (cache; readiness is monotone)
};

// Returns 1 (a row was claimed), 0 (everything dispensed) or -1 (nothing to claim right now;
// only when may_block is false -- the producer then streams the rows it already holds).
__device__ __forceinline__ int fused_next(const LossArgs& a, int64_t totalF, int64_t nzero,
                                          Dispatch& D, bool may_block, bool& fwd, int64_t& idx) {
  const int64_t totalFp = totalF * kFS;  // forward work units (row parts)
  const int64_t R = 2 * a.T;
  unsigned* cnt = a.w.counters;
  for (;;) {
    const int64_t pb = (int64_t)ld_relaxed(&cnt[C_BPAIR]);
    if (pb < a.P) {
      bool rdy = pb == D.ready_pair;
      if (!rdy && ld_relaxed(&a.w.pair_ready[pb]) != 0u) {
        D.ready_pair = pb;
        rdy = true;
      }
      if (rdy) {
        const int64_t r = (int64_t)atomicAdd(&a.w.pair_bcnt[pb], 1u);
        if (r < R) {
#ifdef ODPO_DEBUG_LEAD
          if (r == 0) {
            a.w.dbg_t[pb * 4 + 3] = gtimer();
            const int64_t ft = (int64_t)ld_relaxed(&cnt[C_TICKET]);
            const unsigned lead = (unsigned)(ft > pb * R ? ft - pb * R : 0);
            atomicAdd(&cnt[C_DBG_SUM], lead);
            atomicAdd(&cnt[C_DBG_N], 1u);
            atomicMax(&cnt[C_DBG_MAX], lead);
          }
#endif
          fwd = false;
          idx = pb * R + r;
          return 1;
        }
        atomicCAS(&cnt[C_BPAIR], (unsigned)pb, (unsigned)(pb + 1));  // pair exhausted
        continue;
      }
    } else {
      const int64_t z = (int64_t)atomicAdd(&cnt[C_ZTICKET], 1u);
      if (z < nzero) {
        fwd = false;
        idx = totalF + z;
        return 1;
      }
      return 0;  // every backward and zero row dispensed (so every forward row too)
    }
    // the next backward pair is not ready: a forward row, unless capped or exhausted
    if (!D.f_exh) {
      bool capped = false;
      if (a.max_lead < (int64_t)INT32_MAX) {
        const int64_t ft = (int64_t)ld_relaxed(&cnt[C_TICKET]);
        capped = ft / kFS - pb * R >= a.max_lead;
      }
      if (!capped) {
        const int64_t f = (int64_t)atomicAdd(&cnt[C_TICKET], 1u);
        if (f < totalFp) {
          fwd = true;
          idx = f;
#ifdef ODPO_DEBUG_LEAD
          if (f % R == 0) a.w.dbg_t[(f / R) * 4 + 0] = gtimer();
          if (f % R == R - 1) a.w.dbg_t[(f / R) * 4 + 1] = gtimer();
#endif
          return 1;
        }
        D.f_exh = true;
      }
    }
    if (!may_block) return -1;
    __nanosleep(128);
  }
}

// Wave dispatch (ODPO_SCHED_WAVE).  CTA b belongs to group g = b % NG with rank b / NG; group
// g owns pairs g, g + NG, ... and for each of them its CTA of rank j streams rows j, j + GS, ...
// of the pair's 2T rows forward, then the same rows backward.  A pair's rows are all in flight
// at once (one per CTA), so it completes about one row-time after it starts and NG pairs'
// logits stay in L2 for the backward re-read.  Static assignment: a CTA's backward row waits
// only on forward rows that other CTAs of its group stream before their own backward row, so
// the schedule is deadlock-free when all CTAs are co-resident (the host checks the grid).
struct Wave {
  int g, rank;
  int64_t k, i;
  int phase;
  bool pairs_done;
};
__device__ __forceinline__ int wave_next(const LossArgs& a, Wave& W, int64_t totalF, int64_t nzero,
                                         bool& fwd, int64_t& idx) {
  const int64_t R = 2 * a.T;
  // per CTA: F(0), [F(1)], B(0), [F(2)], B(1), ... with wave_gap = 1 (the bracketed forward
  // rows hide the wait for the previous pair); F(0), B(0), F(1), B(1), ... with wave_gap = 0
  for (;;) {
    if (!W.pairs_done) {
      if (W.rank >= a.wave_gs) {
        W.pairs_done = true;
        continue;
      }
      // phase 0: forward rows of pair-step k; phase 1: backward rows of pair-step k - gap
      const int64_t kk = W.phase == 0 ? W.k : W.k - a.wave_gap;
      const int64_t p = W.g + kk * a.wave_ng;
      const bool valid = kk >= 0 && p < a.P;
      const int64_t j = W.rank + W.i * a.wave_gs;
      if (valid && j < R) {
        fwd = W.phase == 0;
        idx = p * R + j;
        ++W.i;
        return 1;
      }
      W.i = 0;
      if (W.phase == 0) {
        W.phase = 1;
      } else {
        W.phase = 0;
        ++W.k;
        // done once the backward of the last pair-step has been emitted
        if (W.g + (W.k - a.wave_gap) * a.wave_ng >= a.P) W.pairs_done = true;
      }
      continue;
    }
    const int64_t z = (int64_t)atomicAdd(&a.w.counters[C_ZTICKET], 1u);
    if (z < nzero) {
      fwd = false;
      idx = totalF + z;
      return 1;
    }
    return 0;
  }
}

// exp2 split variants (bf16): NPF / NPB of every 8 elements use the FMA-pipe polynomial in the
// forward / backward; the rest use MUFU.EX2.
struct PolyVariant {
  int npf, npb;
};
constexpr PolyVariant kPoly[] = {{0, 0}, {2, 2}, {2, 4}, {3, 4}, {4, 4}, {3, 3}, {2, 3}};
constexpr int kNumPoly = sizeof(kPoly) / sizeof(kPoly[0]);
constexpr int kPolyDefault = 0;

// Row decode (producer): ticket -> RowSlot fields.  Returns true if the row streams data.
template <int DT, int MODE>
__device__ __forceinline__ bool decode_row(const LossArgs& a, int64_t tk, bool fwd_in,
                                           RowSlot& S, uint64_t& pol, uint64_t pol_keep,
                                           uint64_t pol_drop) {
  const int64_t T = a.T, R = 2 * T;
  S.tok = 0;
  S.p = 0;
  S.s = -1;
  S.g = 0;
  S.row = nullptr;
  S.drow = nullptr;
  S.part = 0;
  pol = pol_drop;
  if (MODE == M_FUSED && kFS > 1 && fwd_in) {  // forward work unit = (row, vocabulary part)
    S.part = (int32_t)(tk % kFS);
    tk /= kFS;
  }
  if (MODE == M_SEQ) {
    S.g = tk;
    S.s = tk / T;
    S.p = S.s;
    if (a.mask[S.g]) {
      S.kind = K_F;
      S.row = row_ptr(a, S.s, tk % T);
      S.tok = (int32_t)(a.tokens[S.g] - a.tok_off);  // shard-local (vocabulary-parallel)
      return true;
    }
    S.kind = K_FSKIP;
    return false;
  }
  const int64_t totalF = a.P * R;
  if (tk < totalF) {
    const bool fwd = fwd_in;
    const int64_t p = tk / R;
    const int64_t j = tk % R;
    int64_t c, r;
    pair_seqs(a, p, c, r);
    const int64_t s = j < T ? c : r;
    const int64_t t = j < T ? j : j - T;
    S.p = p;
    S.s = s;
    S.g = s >= 0 ? s * T + t : 0;
    const bool live = s >= 0 && a.mask[S.g];
    if (fwd) {
      if (!live) { S.kind = S.part == 0 ? K_FSKIP : K_NONE; return false; }  // counted once
      S.kind = K_F;
      S.row = row_ptr(a, s, t);
      S.tok = a.tokens[S.g];
      pol = pol_keep;   // keep the row in L2 for its backward pass
      return true;
    }
    if (live) {
      S.kind = K_B;
      S.row = row_ptr(a, s, t);
      S.drow = drow_ptr(a, s, t);
      S.tok = a.tokens[S.g];
      return true;
    }
    if (s >= 0) {
      S.kind = K_ZERO;
      S.drow = drow_ptr(a, s, t);
    } else {
      S.kind = K_NONE;
    }
    return false;
  }
  const int64_t k = (tk - totalF) / T, t = (tk - totalF) % T;
  const int64_t s = __ldcg(a.w.unref + k);
  S.kind = K_ZERO;
  S.s = s;
  S.g = s * T + t;
  S.drow = drow_ptr(a, s, t);
  return false;
}

// Epilogue-side counting: returns true (warp-uniform) if this row completed its pair/sequence.
template <int MODE>
__device__ __forceinline__ bool count_row(const LossArgs& a, const RowSlot& S, int lane) {
  unsigned last = 0;
  if (lane == 0 && (MODE != M_SEQ || a.seqsum)) {
    // release: this row's statistics before the count; acquire: the other rows' statistics
    unsigned* cnt = MODE != M_SEQ ? &a.w.pair_cnt[S.p] : &a.w.seq_cnt[S.s];
    const unsigned need = MODE != M_SEQ ? (unsigned)(2 * a.T) : (unsigned)a.T;
    last = (atom_add_acq_rel(cnt, 1u) == need - 1u);
  }
  last = __shfl_sync(kFull, last, 0);
  if (last) fence_acq_rel_gpu();  // make the acquire visible to every lane of the warp
  return last != 0;
}

template <int MODE>
__device__ __forceinline__ void complete_unit(const LossArgs& a, const RowSlot& S, int lane) {
  if (MODE != M_SEQ) {
    pair_reduce_warp(a, S.p);
  } else {
    double Sq;
    int n;
    seq_sum_warp(a.w.row_logp + S.s * a.T, a.mask + S.s * a.T, a.T, Sq, n);
    if (lane == 0) {
      a.seq_logp[S.s] = n ? (float)Sq : 0.f;
      if (!n) flag(a.status, ODPO_FLAG_EMPTY_SEQ);
    }
  }
}

// ---- the engine.  Warps 0..kNCW-1 consume, then the TMA producer, the parameter warp and the
// epilogue warps.  With CS > 1 the kernel runs as thread-block clusters of CS CTAs on CS
// different SMs: a row is split into CS contiguous vocabulary ranges, one per CTA, so it is
// streamed with CS SMs' bandwidth; the cluster leader (rank 0) claims the work, broadcasts
// each row slot to its peers through distributed shared memory, prefetches backward
// parameters for all of them, and its epilogue merges the CS*kNCW per-warp partials (written
// into its slot through DSMEM, in fixed (rank, warp) order).  Shorter per-row latency means a
// pair completes sooner after its rows are dispensed, which keeps the forward/backward lead
// inside L2.  CS = 1 is the plain single-CTA engine.
template <int DT, int MODE, int PV, int CS, class GE>
__global__ void __launch_bounds__(GE::THREADS, GE::CPS) k_engine(LossArgs a) {
  constexpr int kNCW = GE::NCW, kNCT = GE::NCT, kUB = GE::UB, kStages = GE::STAGES;
  constexpr int kProdWarp = GE::PROD, kParWarp = GE::PAR, kEpiWarp = GE::EPI;
  constexpr int NPF = DT == 1 ? kPoly[PV].npf : 0;
  constexpr int NPB = DT == 1 ? kPoly[PV].npb : 0;
  constexpr int N = Traits<DT>::N;
  constexpr int NPART = CS * kNCW;  // partials per row
  static_assert(NPART <= 32, "one warp merges the partials");
  static_assert(MODE != M_UNSC || CS == 1, "the unscaled mode runs on single-CTA clusters");
  static_assert(kFS == 1 || CS == 1, "forward parts run on single-CTA clusters");
  extern __shared__ __align__(128) uint8_t ring[];
  __shared__ __align__(8) uint64_t full[kStages];
  __shared__ __align__(8) uint64_t empty[kStages];
  __shared__ __align__(8) uint64_t slot_full[kSlots];
  __shared__ __align__(8) uint64_t slot_empty[kSlots];
  __shared__ __align__(8) uint64_t part_ready[kSlots];
  __shared__ __align__(8) uint64_t param_ready[kSlots];
  __shared__ int32_t stage_slot[kStages];
  __shared__ int32_t stage_chunk[kStages];   // position of the chunk in its row's stream
  __shared__ int32_t stage_pchunk[kStages];  // the chunk's place in the row (vector range)
  __shared__ __align__(16) RowSlot slots[kSlots];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t crank = CS > 1 ? cluster_rank() : 0u;
  const bool leader = crank == 0;
  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kNCW);
    }
    for (int s = 0; s < kSlots; ++s) {
      mbar_init(&slot_full[s], 1);
      mbar_init(&slot_empty[s], NPART + 2);  // every consumer warp + epilogue + parameter warp
      mbar_init(&part_ready[s], NPART);
      mbar_init(&param_ready[s], 1);
    }
    mbar_fence_init();
  }
  if (CS > 1) cluster_sync_all();  // peers' barriers exist before any remote arrive
  else __syncthreads();
  // 32-bit shared-window addresses, hoisted out of every loop
  const uint32_t ring_s = smem_u32(ring);
  const uint32_t full_s = smem_u32(full), empty_s = smem_u32(empty);
  const uint32_t sfull_s = smem_u32(slot_full), sempty_s = smem_u32(slot_empty);
  const uint32_t pready_s = smem_u32(part_ready), mready_s = smem_u32(param_ready);
  const uint32_t slots_s = smem_u32(slots);
  // the leader's copies (cluster addresses) of the barriers/slots the consumers report to
  const uint32_t L_sempty = CS > 1 ? mapa(sempty_s, 0) : sempty_s;
  const uint32_t L_pready = CS > 1 ? mapa(pready_s, 0) : pready_s;
  const uint32_t L_slots = CS > 1 ? mapa(slots_s, 0) : slots_s;
  auto wait = [&](uint32_t b, uint32_t par) {
    if (CS > 1) mbar_wait_cl(b, par);
    else mbar_wait(b, par);
  };
  auto arrive_leader = [&](uint32_t b_local_offset_addr_leader, uint32_t n) {
    if (CS > 1) mbar_arrive_cl_n(b_local_offset_addr_leader, n);
    else mbar_arrive_n(b_local_offset_addr_leader, n);
  };

  const int64_t T = a.T;
  const int V = (int)a.V;
  const int nvec = V / N;
  const int tail = V - nvec * N;
  // this CTA's contiguous vector range of every row
  const int v_lo = (int)((int64_t)nvec * crank / CS);
  const int v_hi = (int)((int64_t)nvec * (crank + 1) / CS);
  const bool tail_owner = crank == CS - 1;
  const float k2 = a.invT * kLog2e;

  if (warp == kProdWarp) {
    if (lane == 0) {
      // ================= producer: (leader) tickets -> row slots, broadcast; every CTA streams
      // its own vocabulary range of each row into its TMA ring
#ifdef ODPO_KEEP_FRAC
      const uint64_t pol_keep = MODE == M_FUSED ? policy_evict_last_frac(ODPO_KEEP_FRAC) : policy_evict_last();
#else
      const uint64_t pol_keep = policy_evict_last();
#endif
      const uint64_t pol_drop = policy_evict_first();
      const int64_t totalF = a.P * 2 * T;
      const int64_t nzero = (int64_t)__ldcg(&a.w.counters[C_NUNREF]) * T;
      const int64_t total = a.B * T;  // SEQ
      Dispatch D{false, -1};
      Wave Wv{(int)(blockIdx.x % (a.wave_ng > 0 ? a.wave_ng : 1)),
              (int)(blockIdx.x / (a.wave_ng > 0 ? a.wave_ng : 1)), 0, 0, 0, false};
      int st = 0, dsl = 0, psl = 0, ahead = 0;
      uint32_t sph = 0, dph = 0, pph = 0;
      uint32_t pmask = 0;  // per-slot parity of param_ready (advances once per use)
      bool ended = false;
      int64_t u_tk = -1;   // UNSC: the row whose backward is still to be emitted
      int u_slot = -1;
      uint32_t u_ph = 0;
      for (;;) {
        if (leader) {
          // fill slot dsl: a decoded row (more) or END (!more); fs/fph: UNSC backward rows
          auto emit = [&](bool more, int64_t tk, bool fwd, int fs, uint32_t fph) {
            wait(sempty_s + 8 * dsl, dph ^ 1u);
            RowSlot& S = slots[dsl];
            uint64_t pol = pol_drop;
            bool data = false;
            if (!more) {
              S.kind = K_END;
              ended = true;
            } else {
              data = decode_row<DT, MODE>(a, tk, fwd, S, pol, pol_keep, pol_drop);
            }
            S.nchunk = data ? 1 : 0;
            if (MODE == M_UNSC) {
              // param_ready[slot] is published by the forward row's epilogue
              S.fslot = fs;
              S.pphase = fs >= 0 ? fph : (pmask >> dsl) & 1u;
              if (S.kind == K_F) pmask ^= 1u << dsl;
            } else {
              S.pphase = (pmask >> dsl) & 1u;
              if (S.kind == K_B) pmask ^= 1u << dsl;
            }
            // broadcast the slot header to the peers, then signal slot_full everywhere
            for (int r = 1; r < CS; ++r) {
              const uint32_t dst = mapa(slots_s + dsl * (uint32_t)sizeof(RowSlot), r);
              const uint64_t* src = reinterpret_cast<const uint64_t*>(&S);
#pragma unroll
              for (int q = 0; q < kSlotHeaderBytes / 8; ++q) st_cl_u64(dst + 8 * q, src[q]);
            }
            for (int r = 1; r < CS; ++r) mbar_arrive_cl(mapa(sfull_s + 8 * dsl, r));
            mbar_arrive(sfull_s + 8 * dsl);
            if (!more) {
              // every epilogue warp must see an END in one of its own slots
              for (int q = 1; q < kNEpi; ++q) {
                const int y = (dsl + q) % kSlots;
                const uint32_t yph = dph ^ (uint32_t)((dsl + q) / kSlots);
                wait(sempty_s + 8 * y, yph ^ 1u);
                slots[y].kind = K_END;
                slots[y].nchunk = 0;
                mbar_arrive(sfull_s + 8 * y);
              }
            }
            const int me = dsl;
            ++ahead;
            if (++dsl == kSlots) { dsl = 0; dph ^= 1u; }
            return me;
          };
          // decode up to a.look rows ahead of the row being streamed
          while (!ended && ahead <= a.look) {
            int64_t tk;
            bool fwd = true, more;
            if (MODE == M_UNSC) {
              // slot order F(k), U(k-1), F(k+1), U(k), ...: a row's backward streams one
              // forward row after its own forward, so its epilogue has time to publish (m, l)
              tk = (int64_t)atomicAdd(&a.w.counters[C_TICKET], 1u);
              more = tk < totalF + nzero;
              if (more && tk < totalF) {
                const uint32_t fph = (pmask >> dsl) & 1u;
                const int fs = emit(true, tk, true, -1, 0u);
                if (a.row_gap == 0) {
                  emit(true, tk, false, fs, fph);
                  continue;
                }
                if (u_tk >= 0) emit(true, u_tk, false, u_slot, u_ph);
                u_tk = tk;
                u_slot = fs;
                u_ph = fph;
              } else {
                if (u_tk >= 0) emit(true, u_tk, false, u_slot, u_ph);
                u_tk = -1;
                emit(more, tk, false, -1, 0u);
              }
              continue;
            }
            if (MODE == M_FUSED && a.wave_ng > 0) {
              more = wave_next(a, Wv, totalF, nzero, fwd, tk) > 0;
            } else if (MODE == M_FUSED) {
              const int r = fused_next(a, totalF, nzero, D, ahead == 0, fwd, tk);
              if (r < 0) break;  // stream the rows already held, then retry
              more = r > 0;
            } else {
              tk = (int64_t)atomicAdd(&a.w.counters[C_TICKET], 1u);
              more = tk < total;
            }
            emit(more, tk, fwd, -1, 0u);
          }
          if (ahead == 0) break;
        } else {
          wait(sfull_s + 8 * psl, pph);  // peers: the leader filled this slot
        }
        const RowSlot& S = slots[psl];
        const int kind = S.kind;
        if (kind == K_F || kind == K_B || kind == K_ZERO || kind == K_END) {
          int s_lo = v_lo, s_hi = v_hi;
          if (MODE == M_FUSED && kFS > 1 && kind == K_F) {
            s_lo = (int)((int64_t)nvec * S.part / kFS);
            s_hi = (int)((int64_t)nvec * (S.part + 1) / kFS);
          }
          const bool data = (kind == K_F || kind == K_B) && S.nchunk > 0 && s_hi > s_lo;
          const int nstage = data ? (s_hi - s_lo + kCV - 1) / kCV : 1;
          const uint64_t pol = (MODE != M_SEQ && kind == K_F) ? pol_keep : pol_drop;
          for (int c = 0; c < nstage; ++c) {
            wait(empty_s + 8 * st, sph ^ 1u);
            stage_slot[st] = kind == K_END ? -1 : psl;
            stage_chunk[st] = c;
            // factored-gradient backward rows stream their chunks last-first: the chunks the
            // row's forward read last are the likeliest still in L2 (elementwise backward,
            // so the order does not change any result)
            const int pc = (kBrev && MODE == M_UNSC && kind == K_B) ? nstage - 1 - c : c;
            stage_pchunk[st] = pc;
            const int vs = s_lo + pc * kCV;
            const int nv = data ? min(kCV, s_hi - vs) : 0;
            if (nv > 0) {
              const uint32_t bytes = (uint32_t)nv * 16u;
              mbar_arrive_tx(full_s + 8 * st, bytes);
              tma_load_1d(ring_s + st * kChunk, S.row + (size_t)vs * 16, bytes, full_s + 8 * st, pol);
            } else {
              mbar_arrive(full_s + 8 * st);
            }
            if (++st == kStages) { st = 0; sph ^= 1u; }
          }
        }
        if (leader) --ahead;
        if (++psl == kSlots) { psl = 0; pph ^= 1u; }
        if (kind == K_END) break;
      }
#ifdef ODPO_DEBUG_LEAD
      if (MODE == M_FUSED && leader &&
          atomicAdd(&a.w.counters[C_DBG_DONE], 1u) == gridDim.x / CS - 1) {
        const unsigned n = ld_relaxed(&a.w.counters[C_DBG_N]);
        printf("ODPO_DEBUG_LEAD: backward claims %u, mean forward lead %.1f rows, max %u rows (2T=%d)\n",
               n, n ? (double)ld_relaxed(&a.w.counters[C_DBG_SUM]) / n : 0.0,
               ld_relaxed(&a.w.counters[C_DBG_MAX]), (int)(2 * T));
        double d01 = 0, d12 = 0, d23 = 0;
        const unsigned long long* dt = a.w.dbg_t;
        for (int64_t p = 0; p < a.P; ++p) {
          d01 += (double)(dt[4 * p + 1] - dt[4 * p + 0]);
          d12 += (double)(dt[4 * p + 2] - dt[4 * p + 1]);
          d23 += (double)(dt[4 * p + 3] - dt[4 * p + 2]);
        }
        printf("ODPO_DEBUG_LEAD: per pair mean us: dispatch span %.2f, last F dispatch -> ready %.2f, "
               "ready -> first B claim %.2f\n", d01 / a.P / 1e3, d12 / a.P / 1e3, d23 / a.P / 1e3);
      }
#endif
    }
  } else if (warp == kParWarp) {
    if (lane == 0 && leader) {
      // ================= backward-parameter prefetch (leader): for each backward row, acquire
      // its pair's coefficient, publish the row constants to every CTA of the cluster
      int sl = 0;
      uint32_t lph = 0;
      for (;;) {
        wait(sfull_s + 8 * sl, lph);
        RowSlot& S = slots[sl];
        const int kind = S.kind;
        if (kind == K_END) break;
        if (MODE == M_FUSED && kind == K_B) {
          while (ld_relaxed(&a.w.pair_ready[S.p]) == 0u) __nanosleep(32);
          fence_acq_rel_gpu();
          const float m = __ldcg(a.w.row_m + S.g);
          const float l1p = __ldcg(a.w.row_l1p + S.g);
          const float logp = __ldcg(a.w.row_logp + S.g);
          const float coef = __ldcg(a.w.seq_coef + S.s);
          // coef folded into the exponent: coef * 2^e = sign * 2^(e + log2|coef|)
          const float c = bwd_const<DT>(m, l1p, k2, coef);
          const float gtok = coef * expm1f(logp);
          S.c = c;
          S.coef = coef;
          S.gtok = gtok;
          S.xm = m;
          const uint32_t off_c = (uint32_t)offsetof(RowSlot, c);
          for (int r = 1; r < CS; ++r) {
            const uint32_t dst = mapa(slots_s + sl * (uint32_t)sizeof(RowSlot) + off_c, r);
            st_cl_u32(dst, __float_as_uint(c));
            st_cl_u32(dst + 4, __float_as_uint(coef));
            st_cl_u32(dst + 8, __float_as_uint(gtok));
            st_cl_u32(dst + 16, __float_as_uint(m));
            mbar_arrive_cl(mapa(mready_s + 8 * sl, r));
          }
          mbar_arrive(mready_s + 8 * sl);
        }
        mbar_arrive(sempty_s + 8 * sl);
        if (++sl == kSlots) { sl = 0; lph ^= 1u; }
      }
    }
  } else if (warp >= kEpiWarp) {
    if (leader) {
      // ================= row epilogues (leader): merge the cluster's partials, finalize, count,
      // pair/sequence reduce.  Epilogue warp e owns slots e, e+kNEpi, ... (each in order).
      const int e = warp - kEpiWarp;
      int sl = e;
      uint32_t lph = 0;
      uint32_t rmask = 0;  // per-slot parity of part_ready (advances only on forward rows)
      for (;;) {
        wait(sfull_s + 8 * sl, lph);
        const RowSlot& S = slots[sl];
        const int kind = S.kind;
        if (kind == K_END) break;
        if (kind == K_F) {
          wait(pready_s + 8 * sl, (rmask >> sl) & 1u);
          rmask ^= 1u << sl;
          MR v;
          v.m = lane < NPART ? S.pm[lane] : -INFINITY;
          v.r = lane < NPART ? S.pr[lane] : 0.f;
          v = warp_merge(v, k2);
          float xt = S.xtok;
          bool whole = true;  // this unit completes its row (always, unless rows are split)
          if (MODE == M_FUSED && kFS > 1) {
            // a vocabulary part: publish its partial; the part that finishes last merges all
            // parts in part order (deterministic) and finalises the row
            unsigned last = 0;
            if (lane == 0) {
              const int lo = (int)((int64_t)nvec * S.part / kFS);
              const int hi = (int)((int64_t)nvec * (S.part + 1) / kFS);
              const int tv = S.tok >= 0 ? S.tok / N : -1;
              const bool own = (tv >= lo && tv < hi && S.tok < nvec * N) ||
                               (S.part == kFS - 1 && S.tok >= nvec * N && S.tok < V);
              a.w.fparts[S.g * kFS + S.part] = make_float4(v.m, v.r, own ? S.xtok : 0.f, own ? 1.f : 0.f);
              last = atom_add_acq_rel(&a.w.fpart_cnt[S.g], 1u) == (unsigned)(kFS - 1);
              if (last) {
                fence_acq_rel_gpu();
                MR u{-INFINITY, 0.f};
                for (int h = 0; h < kFS; ++h) {
                  const float4 q = __ldcg(&a.w.fparts[S.g * kFS + h]);
                  u = mr_merge(u, MR{q.x, q.y}, k2);
                  if (q.w != 0.f) xt = q.z;
                }
                v = u;
              }
            }
            whole = __shfl_sync(kFull, last, 0) != 0;
          }
          if (!whole) {
            // another part of this row is still streaming: nothing to count yet
          } else if (MODE == M_SEQ && a.vp_parts) {
            // vocabulary-parallel partial of this shard; k_vp_combine merges the shards
            if (lane == 0) {
              uint32_t fl = 0;
              const int64_t gt = (int64_t)S.tok + a.tok_off;
              if (gt < 0 || gt >= a.V_total) fl |= ODPO_FLAG_TOKEN_RANGE;
              if (isnan(v.m) || v.m == INFINITY || !isfinite(v.r)) fl |= ODPO_FLAG_NONFINITE_LOGIT;
              const bool own = S.tok >= 0 && S.tok < V;
              a.vp_parts[S.g] = make_float4(v.m, log1pf(v.r), own ? S.xtok : 0.f, own ? 1.f : 0.f);
              flag(a.status, fl);
            }
          } else if (lane == 0) {
            uint32_t fl = 0;
            const float l1p = log1pf(v.r);
            float logp = 0.f;
            if (S.tok < 0 || S.tok >= V) {
              fl |= ODPO_FLAG_TOKEN_RANGE;
            } else {
              logp = __fsub_rn(__fmul_rn(__fsub_rn(xt, v.m), a.invT), l1p);
              if (!isfinite(logp)) fl |= ODPO_FLAG_NONFINITE_LOGIT;
            }
            if (!isfinite(v.m) || !isfinite(v.r)) fl |= ODPO_FLAG_NONFINITE_LOGIT;
            a.w.row_m[S.g] = v.m;
            a.w.row_l1p[S.g] = l1p;
            a.w.row_logp[S.g] = logp;
            if (MODE == M_SEQ) {
              if (a.tok_out) a.tok_out[S.g] = logp;
              if (a.lse_out) a.lse_out[S.g] = __fadd_rn(__fmul_rn(v.m, a.invT), l1p);
            }
            if (MODE == M_UNSC) {
              // the row's backward (G = softmax - onehot) constants, for this CTA's consumers
              RowSlot& W = slots[sl];
              // known coefficient (App B losses): coef folded into the exponent as in FUSED
              const float cf = a.coef_known ? __ldcg(a.w.seq_coef + S.s) : 1.f;
              W.c = cf != 0.f ? bwd_const<DT>(v.m, l1p, k2, cf) : INFINITY;
              W.xm = v.m;
              W.coef = cf;
              W.gtok = cf * expm1f(logp);
              mbar_arrive(mready_s + 8 * sl);
            }
            flag(a.status, fl);
          }
          if (whole && count_row<MODE>(a, S, lane)) complete_unit<MODE>(a, S, lane);
        } else if (kind == K_FSKIP) {
          if (lane == 0 && MODE == M_SEQ) {
            if (a.tok_out) a.tok_out[S.g] = 0.f;
            if (a.lse_out) a.lse_out[S.g] = 0.f;
            if (a.vp_parts) a.vp_parts[S.g] = make_float4(-INFINITY, 0.f, 0.f, 0.f);
          }
          if (count_row<MODE>(a, S, lane)) complete_unit<MODE>(a, S, lane);
        } else if (MODE == M_UNSC && kind == K_ZERO) {
          if (lane == 0 && a.row_scale) a.row_scale[S.g] = 0.f;
        }
        __syncwarp();
        // rows the consumers never see also carry their NPART arrivals
        if (lane == 0)
          mbar_arrive_n(sempty_s + 8 * sl, (kind == K_FSKIP || kind == K_NONE) ? 1u + NPART : 1u);
        sl += kNEpi;
        if (sl >= kSlots) { sl -= kSlots; lph ^= 1u; }
      }
    }
  } else {
    // ================= consumers (warps 0..kNCW-1): this CTA's vocabulary range of each row
    const uint32_t NI = Traits<DT>::kNegInfWord;
    const int pidx = (int)crank * kNCW + warp;  // this warp's partial index in the leader slot
    int st = 0;
    uint32_t sph = 0;
    MR s{-INFINITY, 0.f};
    float b_c = 0.f, b_coef = 0.f, b_gtok = 0.f, b_m = 0.f;
    int r_kind = K_NONE, r_tok = 0, r_nst = 1, r_tch = -1, r_tvl = -1;
    int r_lo = v_lo, r_hi = v_hi;
    bool r_tail = tail_owner;
    const char* r_row = nullptr;
    char* r_drow = nullptr;
    for (;;) {
      wait(full_s + 8 * st, sph);
      const int sl = stage_slot[st];
      if (sl < 0) break;
      const int ch = stage_chunk[st];
      const int pch = stage_pchunk[st];
      RowSlot& S = slots[sl];
      const uint32_t Lslot = L_slots + sl * (uint32_t)sizeof(RowSlot);
      if (ch == 0) {  // a new row: cache its fields (a row's chunks occupy consecutive stages)
        r_kind = S.kind;
        r_tok = S.tok;
        r_lo = v_lo;
        r_hi = v_hi;
        r_tail = tail_owner;
        if (MODE == M_FUSED && kFS > 1 && r_kind == K_F) {
          r_lo = (int)((int64_t)nvec * S.part / kFS);
          r_hi = (int)((int64_t)nvec * (S.part + 1) / kFS);
          r_tail = S.part == kFS - 1;
        }
        r_nst = ((r_kind == K_F || r_kind == K_B) && S.nchunk > 0 && r_hi > r_lo)
                    ? (r_hi - r_lo + kCV - 1) / kCV : 1;
        r_row = S.row;
        r_drow = S.drow;
        // the vector holding tok, if it is in this CTA's range: its chunk and chunk-local index
        const int tvec = (r_tok >= 0 && r_tok < nvec * N) ? r_tok / N : -1;
        const bool mine = tvec >= r_lo && tvec < r_hi;
        r_tch = mine ? (tvec - r_lo) / kCV : -1;
        r_tvl = mine ? (tvec - r_lo) - r_tch * kCV : -1;
      }
      const int kind = r_kind;
      const bool last_chunk = ch == r_nst - 1;
      const uint4* sv = reinterpret_cast<const uint4*>(ring + (size_t)st * kChunk);
      const int c0 = r_lo + pch * kCV;  // first vector of this chunk within the row
      const int cnv = r_hi > r_lo ? min(kCV, r_hi - c0) : 0;
      const bool own_tok = pch == r_tch && (r_tvl % kNCT) == tid;
      if (kind == K_F) {
        if (ch == 0) s = MR{-INFINITY, 0.f};
        if (cnv == kCV) {  // full chunk: no predication
          uint4 v[kUB];
#pragma unroll
          for (int u = 0; u < kUB; ++u) v[u] = sv[tid + u * kNCT];
          mr_batch<DT, kUB, NPF>(v, k2, s.m, s.r);
        } else if (tid < cnv) {
          mr_partial<DT, kUB, NPF>(sv, tid, kNCT, cnv, k2, s.m, s.r);
        }
        if (own_tok) {
          float f[N];
          Traits<DT>::unpack(sv[r_tvl], f);
          float x = f[0];
#pragma unroll
          for (int j = 1; j < N; ++j) x = (r_tok % N == j) ? f[j] : x;
          if (CS > 1) st_cl_u32(Lslot + (uint32_t)offsetof(RowSlot, xtok), __float_as_uint(x));
          else S.xtok = x;
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(empty_s + 8 * st);
        if (last_chunk) {
          if (r_tail && tid < tail) {
            const int64_t vv = (int64_t)nvec * N + tid;
            const float x = Traits<DT>::load1(r_row, vv);
            s = mr_push1(s, x, k2);
            if (vv == r_tok) {
              if (CS > 1) st_cl_u32(Lslot + (uint32_t)offsetof(RowSlot, xtok), __float_as_uint(x));
              else S.xtok = x;
            }
          }
          const MR wv = warp_merge(s, k2);
          __syncwarp();
          if (lane == 0) {
            if (CS > 1) {
              st_cl_u32(Lslot + (uint32_t)offsetof(RowSlot, pm) + 4 * pidx, __float_as_uint(wv.m));
              st_cl_u32(Lslot + (uint32_t)offsetof(RowSlot, pr) + 4 * pidx, __float_as_uint(wv.r));
            } else {
              S.pm[pidx] = wv.m;
              S.pr[pidx] = wv.r;
            }
            arrive_leader(L_pready + 8 * sl, 1u);
            // UNSC: the slot is released when the row's backward has read its constants
            if (MODE != M_UNSC) arrive_leader(L_sempty + 8 * sl, 1u);
          }
        }
      } else if (kind == K_B) {
        if (ch == 0) {
          const int fs = MODE == M_UNSC ? S.fslot : sl;
          wait(mready_s + 8 * fs, S.pphase);
          b_c = slots[fs].c;
          b_coef = slots[fs].coef;
          b_gtok = slots[fs].gtok;
          b_m = slots[fs].xm;
          if (MODE == M_UNSC) {
            __syncwarp();
            if (lane == 0) mbar_arrive(sempty_s + 8 * fs);
          }
        }
        uint4* vout = reinterpret_cast<uint4*>(r_drow) + c0;
        if (cnv == kCV) {
          if (b_coef < 0.f) {
#pragma unroll
            for (int u = 0; u < kUB; ++u)
              st16_stream(vout + tid + u * kNCT, bwd_vec<DT, NPB, true>(sv[tid + u * kNCT], k2, b_c, b_m));
          } else {
#pragma unroll
            for (int u = 0; u < kUB; ++u)
              st16_stream(vout + tid + u * kNCT, bwd_vec<DT, NPB, false>(sv[tid + u * kNCT], k2, b_c, b_m));
          }
        } else {
#pragma unroll
          for (int u = 0; u < kUB; ++u) {
            const int i = tid + u * kNCT;
            if (i < cnv)
              st16_stream(vout + i, b_coef < 0.f ? bwd_vec<DT, NPB, true>(sv[i], k2, b_c, b_m)
                                                 : bwd_vec<DT, NPB, false>(sv[i], k2, b_c, b_m));
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(empty_s + 8 * st);
        // onehot entry: the thread that stored tok's vector overwrites it (program order)
        if (own_tok) Traits<DT>::store1(r_drow, r_tok, b_gtok);
        if (last_chunk) {
          if (r_tail && tid < tail) {
            const int64_t vv = (int64_t)nvec * N + tid;
            const float x = Traits<DT>::load1(r_row, vv);
            Traits<DT>::store1(r_drow, vv, vv == r_tok ? b_gtok : copysignf(ex2(bwd_arg<DT>(x, k2, b_c, b_m)), b_coef));
          }
          __syncwarp();
          if (lane == 0) arrive_leader(L_sempty + 8 * sl, 1u);
        }
      } else {  // K_ZERO: this CTA's range of the row
        __syncwarp();
        if (lane == 0) mbar_arrive(empty_s + 8 * st);
        uint4* vout = reinterpret_cast<uint4*>(r_drow);
        for (int i = v_lo + tid; i < v_hi; i += kNCT) st16_stream(vout + i, make_uint4(0, 0, 0, 0));
        if (tail_owner && tid < tail) Traits<DT>::store1(r_drow, (int64_t)nvec * N + tid, 0.f);
        __syncwarp();
        if (lane == 0) arrive_leader(L_sempty + 8 * sl, 1u);
      }
      if (++st == kStages) { st = 0; sph ^= 1u; }
    }
  }
  // no CTA may leave while a peer can still touch its shared memory
  if (CS > 1) cluster_sync_all();
}

}  // namespace odpo
#include "odpo_resident.cuh"
// Experimental schedules measured slower than FUSED, compiled only with
// -DODPO_EXPERIMENTAL=1 (build.build(defines={"ODPO_EXPERIMENTAL": 1})): PSYNC.
#ifndef ODPO_EXPERIMENTAL
#define ODPO_EXPERIMENTAL 0
#endif
#if ODPO_EXPERIMENTAL
#include "odpo_psync.cuh"
#endif
namespace odpo {

// ------------------------------------------------------------------ host side
constexpr int kPsLagDefault = 4;   // PSYNC: pairs between a pair's forward and backward pieces

struct DevInfo {
  int sms = 0;
  int l2 = 0;
  int occ[2][2][M_NMODES] = {};  // [geometry][dtype][mode] (same for every poly variant)
  int occ_ps[2] = {};            // PSYNC CTAs per SM [dtype]
};
// cluster size per mode: the unscaled mode always runs single-CTA
template <int MODE>
constexpr int mode_cs() { return MODE == M_UNSC ? 1 : kCS; }
static DevInfo g_dev[128];
static std::once_flag g_once[128];

template <int DT, int MODE, int PV, class GE>
static void setup_one(int* occ) {
  constexpr int CS = mode_cs<MODE>();
  cudaFuncSetAttribute(k_engine<DT, MODE, PV, CS, GE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       GE::SMEM);
  if (occ)
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(occ, k_engine<DT, MODE, PV, CS, GE>, GE::THREADS,
                                                  GE::SMEM);
}

// Launch an engine instantiation, as thread-block clusters of CS CTAs when CS > 1.
template <int DT, int MODE, int PV, class GE>
static void launch_k(int grid, cudaStream_t s, const LossArgs& a) {
  constexpr int CS = mode_cs<MODE>();
  auto kern = k_engine<DT, MODE, PV, CS, GE>;
  if (CS == 1 && a.wave_ng == 0) {
    kern<<<grid, GE::THREADS, GE::SMEM, s>>>(a);
    return;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(GE::THREADS);
  cfg.dynamicSmemBytes = GE::SMEM;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  if (a.wave_ng > 0) {
    // the wave schedule's CTAs wait on their peers (a backward row on its group's forward
    // rows): launched cooperatively, so the runtime guarantees every CTA is co-resident (or
    // fails the launch -> ODPO_ERR_CUDA) whatever else shares the GPU
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
  } else {
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = (unsigned)CS;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
  }
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kern, a);
}
template <int PV>
static void setup_pv() {
  setup_one<1, M_SEQ, PV, Geo0>(nullptr);
  setup_one<1, M_FUSED, PV, Geo0>(nullptr);
  setup_one<1, M_UNSC, PV, Geo0>(nullptr);
  if constexpr (PV + 1 < kNumPoly) setup_pv<PV + 1>();
}
template <class GE>
static void setup_geo(DevInfo& d, int g) {
  setup_one<0, M_SEQ, 0, GE>(&d.occ[g][0][M_SEQ]);
  setup_one<0, M_FUSED, 0, GE>(&d.occ[g][0][M_FUSED]);
  setup_one<0, M_UNSC, 0, GE>(&d.occ[g][0][M_UNSC]);
  setup_one<1, M_SEQ, 0, GE>(&d.occ[g][1][M_SEQ]);
  setup_one<1, M_FUSED, 0, GE>(&d.occ[g][1][M_FUSED]);
  setup_one<1, M_UNSC, 0, GE>(&d.occ[g][1][M_UNSC]);
}

static ResGeo res_geo(int64_t V, int64_t T, int es, int sms, int cap);
static odpo_status launched();
static const struct DevInfo& dev_info(int dev);

template <int PV>
static void setup_res() {
  cudaFuncSetAttribute(k_resident<1, PV, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, kResSmemMax);
  if constexpr (PV == 0) {
    cudaFuncSetAttribute(k_resident<0, 0, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, kResSmemMax);
    cudaFuncSetAttribute(k_resident<0, 0, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, kResSmemMax);
    cudaFuncSetAttribute(k_resident<1, 0, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, kResSmemMax);
  }
  if constexpr (PV + 1 < kNumPoly) setup_res<PV + 1>();
}
template <int PV>
static void launch_res_bf16(int pv, int grid, int smem, const LossArgs& a, const ResGeo& g,
                            cudaStream_t s) {
  if (pv == PV) {
    k_resident<1, PV, 0><<<grid, kResThreads, smem, s>>>(a, g);
    return;
  }
  if constexpr (PV + 1 < kNumPoly) launch_res_bf16<PV + 1>(pv, grid, smem, a, g, s);
}
// the factored / known-coefficient RESIDENT mode (MUFU exp2 only); no pair waits, so any
// shape whose row fits the TMEM slots applies
static odpo_status launch_res_un(int dti, const LossArgs& a, int64_t V, int64_t es, int cap,
                                 cudaStream_t s) {
  int dev = 0;
  cudaGetDevice(&dev);
  const DevInfo& di = dev_info(dev);
  ResGeo rg = res_geo(V, 1, (int)es, di.sms, cap);
  if (rg.nsl <= 0) return ODPO_ERR_UNSUPPORTED;
  const int ring_bytes = (rg.rf + rg.rbs) * kChunk;
  const int smem = ring_bytes > kResSmemMin ? ring_bytes : kResSmemMin;
  if (dti == 0) k_resident<0, 0, 1><<<di.sms, kResThreads, smem, s>>>(a, rg);
  else k_resident<1, 0, 1><<<di.sms, kResThreads, smem, s>>>(a, rg);
  return launched();
}

static const DevInfo& dev_info(int dev) {
  std::call_once(g_once[dev], [dev]() {
    DevInfo& d = g_dev[dev];
    cudaDeviceGetAttribute(&d.sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&d.l2, cudaDevAttrL2CacheSize, dev);
    setup_geo<Geo0>(d, 0);
    setup_geo<Geo1>(d, 1);
    setup_pv<1>();
    setup_res<0>();
#if ODPO_EXPERIMENTAL
    cudaFuncSetAttribute(k_psync<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, kPsSmem);
    cudaFuncSetAttribute(k_psync<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, kPsSmem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&d.occ_ps[0], k_psync<0>, kPsThreads, kPsSmem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&d.occ_ps[1], k_psync<1>, kPsThreads, kPsSmem);
#endif
  });
  return g_dev[dev];
}

static bool aligned16(const void* p) { return ((uintptr_t)p & 15u) == 0; }

// RESIDENT schedule geometry (odpo_resident.cuh): TMEM row slots per SM, forward/backward TMA
// rings, and the L2-backed rows each SM may hold beyond its TMEM stash (cap).  Applicable
// when a row spans at most 8 16-KB chunks (two TMEM slots) and the rows in flight GPU-wide,
// SMs * (slots + cap), cover two pairs (one is the deadlock-freedom bound).
static ResGeo res_geo(int64_t V, int64_t T, int es, int sms, int cap) {
  ResGeo g{0, 0, 0, 0, 0};
  if (!ODPO_EXPERIMENTAL) return g;   // RESIDENT is compiled only with -DODPO_EXPERIMENTAL=1
  const int64_t nvec = V * es / 16;   // whole 16-byte vectors per row
  if (nvec < 1) return g;
  const int64_t nch = (nvec + kCV - 1) / kCV;
  if (nch > kResMaxCh) return g;
  int64_t nsl = (kResTmemCols / kResCols) / nch;
  if (nsl > kResMaxSL) nsl = kResMaxSL;
  if (cap < 0) cap = kResCapDefault;
  if (nsl + cap > kResNIt) cap = kResNIt - (int)nsl;
  if ((int64_t)sms * (nsl + cap) < 2 * (2 * T)) return g;
  g.nsl = (int)nsl; g.nch = (int)nch; g.rf = kResRF; g.rbs = kResRB; g.cap = cap;
  return g;
}

static bool finite_pos(float x) { return isfinite(x) && x > 0.f; }

static odpo_status check_logits(const void* logits, odpo_dtype dt, int64_t B, int64_t T, int64_t V,
                                int64_t sb, int64_t st) {
  if (!logits) return ODPO_ERR_INVALID_ARG;
  if (dt != ODPO_F32 && dt != ODPO_BF16) return ODPO_ERR_INVALID_ARG;
  if (B <= 0 || T <= 0 || V <= 0 || V > (int64_t)INT32_MAX / 4) return ODPO_ERR_INVALID_ARG;
  if (st < V || sb < 0) return ODPO_ERR_INVALID_ARG;
  const int64_t es = dt == ODPO_F32 ? 4 : 2;
  if (!aligned16(logits) || (sb * es) % 16 || (st * es) % 16) return ODPO_ERR_ALIGNMENT;
  if (B * T > (int64_t)INT32_MAX) return ODPO_ERR_UNSUPPORTED;
  return ODPO_OK;
}

static odpo_status launched() {
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? ODPO_OK : ODPO_ERR_CUDA;
}

template <int MODE, int PV>
static void launch_bf16(int pv, int grid, const LossArgs& a, cudaStream_t s) {
  if (pv == PV) {
    launch_k<1, MODE, PV, Geo0>(grid, s, a);
    return;
  }
  if constexpr (PV + 1 < kNumPoly) launch_bf16<MODE, PV + 1>(pv, grid, a, s);
}
// The row backward (TWO_PASS and the vocabulary-parallel loss): k_row_bwd_split's one-batch
// pieces, 32-byte vectors when every row of the logits and of dlogits starts 32-byte aligned,
// else 16-byte.  Configurations (threads, vectors per thread), measured side by side on B200
// (profiles/r02/bwd/; all bit-identical): (512, 4) = pieces up to 64 KB is best on LLaMA (256.5
// KB rows: 14.31 vs 14.71 ms for k_row_bwd's one CTA per row) and Rho (64 KB: 3.685 vs 3.772);
// (256, 4) = up to 32 KB on Pythia (100.6 KB rows: 1.258 vs 1.269).  ODPO_BWD_CFG (build flag,
// A/B only) forces one: -1 = k_row_bwd, 2 = (256, 4), 5 = (512, 4), 6 = (256, 8), 7 = (128, 8).
#ifndef ODPO_BWD_CFG
#define ODPO_BWD_CFG 0
#endif
constexpr int kBwdCfg = ODPO_BWD_CFG;
// Short vocabulary-shard rows (<= 32 KB): the backward in one-batch pieces of 128 threads x 4
// vectors (LLaMA W = 8: 1.28 vs 1.355 ms, Pythia W = 8: 0.139 vs 0.148, Rho W = 2: 1.27 vs 1.34;
// profiles/r02/vp/); the forward partials stay warp-per-row (a CTA per row measured slower:
// five fixed-order merges per row instead of one).  ODPO_VP_WARP=1 (A/B only): the warp-per-row
// backward.
#ifndef ODPO_VP_WARP
#define ODPO_VP_WARP 0
#endif
constexpr bool kVpWarp = ODPO_VP_WARP != 0;

template <int DT, int NPB, int THR, int U>
static void launch_split(unsigned rows, const LossArgs& a, cudaStream_t s) {
  const bool a32 = ((reinterpret_cast<uintptr_t>(a.logits) | reinterpret_cast<uintptr_t>(a.dl)) & 31u) == 0 &&
                   ((a.sb | a.st | a.dsb | a.dst) * a.esize) % 32 == 0;
  const int VW = a32 ? 32 : 16;
  const int64_t nv = a.V / (Traits<DT>::N * (VW / 16));
  int64_t S = (nv + THR * U - 1) / (THR * U);
  if (S < 1) S = 1;
  if ((int64_t)rows * S > (int64_t)INT32_MAX)
    k_row_bwd<DT, NPB><<<rows, kRowThreads, 0, s>>>(a);
  else if (a32)
    k_row_bwd_split<DT, NPB, THR, U, 32><<<(unsigned)(rows * S), THR, 0, s>>>(a);
  else
    k_row_bwd_split<DT, NPB, THR, U, 16><<<(unsigned)(rows * S), THR, 0, s>>>(a);
}
template <int DT, int NPB>
static void launch_row_bwd_t(unsigned rows, const LossArgs& a, cudaStream_t s) {
  const int64_t row_bytes = a.V * a.esize;
  if constexpr (kBwdCfg == -1) k_row_bwd<DT, NPB><<<rows, kRowThreads, 0, s>>>(a);
  else if constexpr (kBwdCfg == 2) launch_split<DT, NPB, 256, 4>(rows, a, s);
  else if constexpr (kBwdCfg == 5) launch_split<DT, NPB, 512, 4>(rows, a, s);
  else if constexpr (kBwdCfg == 6) launch_split<DT, NPB, 256, 8>(rows, a, s);
  else if constexpr (kBwdCfg == 7) launch_split<DT, NPB, 128, 8>(rows, a, s);
  else if (row_bytes > (64 << 10) && row_bytes < (128 << 10)) launch_split<DT, NPB, 256, 4>(rows, a, s);
  else launch_split<DT, NPB, 512, 4>(rows, a, s);
}
template <int PV>
static void launch_bwd_bf16(int pv, unsigned rows, const LossArgs& a, cudaStream_t s) {
  if (pv == PV) {
    launch_row_bwd_t<1, kPoly[PV].npb>(rows, a, s);
    return;
  }
  if constexpr (PV + 1 < kNumPoly) launch_bwd_bf16<PV + 1>(pv, rows, a, s);
}

// Geometry choice: geometry 1 for the unscaled mode on rows longer
// than 128 KB (its re-read must stay in L2); geometry 0 elsewhere.  geo >= 0 forces one.
static int pick_geo(int mode, int64_t row_bytes, int pv, int geo) {
  if (geo >= 0) return geo;
  if (pv != 0) return 0;
  return (mode == M_UNSC && row_bytes > (128 << 10)) ? 1 : 0;
}

#if ODPO_EXPERIMENTAL
// The cluster-split factored gradient (k_unsc_split): pieces of <= 1024 32-byte vectors (256
// threads x 4) or <= 2048 (512 x 4) per CTA, CS = a power of two <= 8 CTAs per row.  Returns
// false (nothing launched) when a row needs more than 8 pieces; the caller uses the engine.
template <int DT, int CS, int THR, int VW>
static void launch_split_cs(unsigned grid, const LossArgs& a, cudaStream_t s) {
  auto kern = k_unsc_split<DT, CS, THR, 4, VW>;
  if (CS == 1) {
    kern<<<grid, THR, 0, s>>>(a);
    return;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(THR);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = (unsigned)CS;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kern, a);
}
template <int DT, int THR, int VW>
static void launch_split_thr(int cs, unsigned grid, const LossArgs& a, cudaStream_t s) {
  if (cs == 1) launch_split_cs<DT, 1, THR, VW>(grid, a, s);
  else if (cs == 2) launch_split_cs<DT, 2, THR, VW>(grid, a, s);
  else if (cs == 4) launch_split_cs<DT, 4, THR, VW>(grid, a, s);
  else launch_split_cs<DT, 8, THR, VW>(grid, a, s);
}
template <int DT, int CS, int THR>
static void launch_tma_cs(unsigned grid, int smem, const LossArgs& a, cudaStream_t s) {
  auto kern = k_unsc_tma<DT, CS, THR>;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(THR);
  cfg.dynamicSmemBytes = (size_t)smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = (unsigned)CS;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = CS > 1 ? 1 : 0;
  cudaLaunchKernelEx(&cfg, kern, a);
}
// TMA-staged variant: pieces of <= 32 KB (<= 48 KB past 256 KB rows), CS <= 8.
template <int DT>
static bool launch_unsc_tma(const LossArgs& a, cudaStream_t s) {
  const int64_t nv = a.V / Traits<DT>::N;
  int64_t need = (nv + 2047) / 2048;
  if (need > 8) need = 8;
  const int cs = need <= 1 ? 1 : need <= 2 ? 2 : need <= 4 ? 4 : 8;
  const int64_t per = (nv + cs - 1) / cs;
  if (per * 16 > (48 << 10)) return false;
  const int smem = (int)(per * 16);
  const int64_t grid = (a.P * 2 * a.T + 2 * 148) * cs;
  if (grid > (int64_t)INT32_MAX) return false;
  if (cs == 1) launch_tma_cs<DT, 1, 128>((unsigned)grid, smem, a, s);
  else if (cs == 2) launch_tma_cs<DT, 2, 128>((unsigned)grid, smem, a, s);
  else if (cs == 4) launch_tma_cs<DT, 4, 128>((unsigned)grid, smem, a, s);
  else launch_tma_cs<DT, 8, 128>((unsigned)grid, smem, a, s);
  return true;
}

template <int DT>
static bool launch_unsc_split(const LossArgs& a, cudaStream_t s) {
  const bool a32 = ((reinterpret_cast<uintptr_t>(a.logits) | reinterpret_cast<uintptr_t>(a.dl)) & 31u) == 0 &&
                   ((a.sb | a.st | a.dsb | a.dst) * a.esize) % 32 == 0;
  const int VW = a32 ? 32 : 16;
  const int64_t nv = a.V / (Traits<DT>::N * (VW / 16));
  int thr = 256;
  int64_t need = (nv + 1023) / 1024;
  if (need > 8) {
    thr = 512;
    need = (nv + 2047) / 2048;
  }
  if (need > 8) return false;
  const int cs = need <= 1 ? 1 : need <= 2 ? 2 : need <= 4 ? 4 : 8;
  const int64_t zero_workers = 2 * 148;   // rows of unreferenced sequences (grid-stride)
  const int64_t grid = (a.P * 2 * a.T + zero_workers) * cs;
  if (grid > (int64_t)INT32_MAX) return false;
  if (thr == 256) {
    if (VW == 32) launch_split_thr<DT, 256, 32>(cs, (unsigned)grid, a, s);
    else launch_split_thr<DT, 256, 16>(cs, (unsigned)grid, a, s);
  } else {
    if (VW == 32) launch_split_thr<DT, 512, 32>(cs, (unsigned)grid, a, s);
    else launch_split_thr<DT, 512, 16>(cs, (unsigned)grid, a, s);
  }
  return true;
}

#endif  // ODPO_EXPERIMENTAL

static odpo_status launch_engine(int dt, int mode, int pv, const LossArgs& a, int cps,
                                 cudaStream_t s, int geo) {
  int dev = 0;
  cudaGetDevice(&dev);
  const DevInfo& di = dev_info(dev);
  geo = pick_geo(mode, a.V * a.esize, pv, geo);
  if (geo > 1 || (geo == 1 && pv != 0)) return ODPO_ERR_UNSUPPORTED;
  int occ = di.occ[geo][dt][mode];
  if (occ < 1) occ = 1;
  if (cps <= 0 || cps > occ) cps = occ;
  const int cs = mode == M_UNSC ? 1 : kCS;
  const int grid = (di.sms * cps / cs) * cs;
  if (geo == 1) {
    if (dt == 0 && mode == M_SEQ) launch_k<0, M_SEQ, 0, Geo1>(grid, s, a);
    if (dt == 0 && mode == M_FUSED) launch_k<0, M_FUSED, 0, Geo1>(grid, s, a);
    if (dt == 0 && mode == M_UNSC) launch_k<0, M_UNSC, 0, Geo1>(grid, s, a);
    if (dt == 1 && mode == M_SEQ) launch_k<1, M_SEQ, 0, Geo1>(grid, s, a);
    if (dt == 1 && mode == M_FUSED) launch_k<1, M_FUSED, 0, Geo1>(grid, s, a);
    if (dt == 1 && mode == M_UNSC) launch_k<1, M_UNSC, 0, Geo1>(grid, s, a);
    return launched();
  }
  if (dt == 0 && mode == M_SEQ) launch_k<0, M_SEQ, 0, Geo0>(grid, s, a);
  if (dt == 0 && mode == M_FUSED) launch_k<0, M_FUSED, 0, Geo0>(grid, s, a);
  if (dt == 0 && mode == M_UNSC) launch_k<0, M_UNSC, 0, Geo0>(grid, s, a);
  if (dt == 1 && mode == M_SEQ) launch_bf16<M_SEQ, 0>(pv, grid, a, s);
  if (dt == 1 && mode == M_FUSED) launch_bf16<M_FUSED, 0>(pv, grid, a, s);
  if (dt == 1 && mode == M_UNSC) launch_bf16<M_UNSC, 0>(pv, grid, a, s);
  return launched();
}

}  // namespace odpo

using namespace odpo;

extern "C" {

const char* odpo_version(void) { return ODPO_VERSION_STR; }

#ifdef ODPO_RES_DEBUG
// debug builds only (not declared in odpo.h): copy the RESIDENT per-ticket timestamps
int odpo_res_debug_dump(unsigned long long* host, int64_t n_rows) {
  if (n_rows > kResDbgRows) n_rows = kResDbgRows;
  return (int)cudaMemcpyFromSymbol(host, g_res_dbg, (size_t)n_rows * 8 * sizeof(unsigned long long));
}
#endif

const char* odpo_status_string(odpo_status s) {
  switch (s) {
    case ODPO_OK: return "ok";
    case ODPO_ERR_INVALID_ARG: return "invalid argument";
    case ODPO_ERR_ALIGNMENT: return "logits/dlogits base or stride not 16-byte aligned";
    case ODPO_ERR_WORKSPACE: return "workspace missing or too small";
    case ODPO_ERR_UNSUPPORTED: return "unsupported shape or option";
    case ODPO_ERR_CUDA: return "CUDA launch failure";
  }
  return "unknown status";
}

size_t odpo_workspace_bytes(int64_t B, int64_t T, int64_t P) {
  if (B <= 0 || T <= 0 || P < 0) return 0;
  return ws_layout(B, T, P > 0 ? P : 1, nullptr, nullptr);
}

odpo_status odpo_pair_select(const float* rewards, const uint8_t* has_eos, float eos_penalty,
                             int64_t P, int32_t K, int32_t* chosen, int32_t* rejected,
                             int32_t* pair_rows, float* reward_margin, double* sel_stats,
                             uint32_t* status, void* stream) {
  if (P < 0 || K < 2) return ODPO_ERR_INVALID_ARG;
  if (P > 0 && (!rewards || !chosen || !rejected)) return ODPO_ERR_INVALID_ARG;
  if (P * (int64_t)K > (int64_t)INT32_MAX) return ODPO_ERR_UNSUPPORTED;
  k_pair_select<<<1, kSelThreads, 0, (cudaStream_t)stream>>>(
      rewards, has_eos, eos_penalty, P, K, chosen, rejected, pair_rows, reward_margin, sel_stats,
      status);
  return launched();
}

static void base_args(LossArgs& a, const void* logits, int64_t B, int64_t T, int64_t V, int64_t sb,
                      int64_t st, const int32_t* tokens, const uint8_t* mask, float invT,
                      uint32_t* status, const Workspace& w, int es) {
  a.logits = logits;
  a.B = B; a.T = T; a.V = V; a.sb = sb; a.st = st;
  a.ref = nullptr; a.tokens = tokens; a.mask = mask; a.pair_rows = nullptr;
  a.P = 0; a.Pg = 1.0; a.beta = 0.f; a.invT = invT;
  a.dl = nullptr; a.dsb = 0; a.dst = 0;
  a.seq_logp = nullptr; a.z_out = nullptr; a.stats = nullptr; a.status = status;
  a.tok_out = nullptr; a.lse_out = nullptr; a.seqsum = 0;
  a.w = w; a.lag = 1; a.max_lead = 1; a.look = kLook; a.esize = es;
  a.wave_ng = 0; a.wave_gs = 0; a.wave_gap = 0;
  a.row_scale = nullptr;
  a.row_gap = 0;
  a.pg_kind = -1;
  a.coef_known = 0;
  a.rewards = nullptr;
  a.old_logp = nullptr;
  a.clip_eps = 0.f;
  a.vp_parts = nullptr;
  a.tok_off = 0;
  a.V_total = V;
  a.put = VpPut{};
  a.vp_flags = nullptr;
  a.vp_epoch = 0;
}

odpo_status odpo_seq_logprobs(const void* logits, odpo_dtype dt, int64_t B, int64_t T, int64_t V,
                              int64_t stride_b, int64_t stride_t, const int32_t* tokens,
                              const uint8_t* mask, float inv_temperature, float* seq_logp,
                              float* tok_logp, float* row_lse, uint32_t* status, void* workspace,
                              size_t workspace_bytes, void* stream) {
  odpo_status e = check_logits(logits, dt, B, T, V, stride_b, stride_t);
  if (e != ODPO_OK) return e;
  if (!tokens || !mask || !seq_logp || !finite_pos(inv_temperature)) return ODPO_ERR_INVALID_ARG;
  const int64_t P = B / 2 + 1;
  if (!workspace || workspace_bytes < ws_layout(B, T, P, nullptr, nullptr)) return ODPO_ERR_WORKSPACE;
  Workspace w;
  ws_layout(B, T, P, (char*)workspace, &w);
  cudaStream_t s = (cudaStream_t)stream;
  LossArgs a;
  base_args(a, logits, B, T, V, stride_b, stride_t, tokens, mask, inv_temperature, status, w,
            dt == ODPO_F32 ? 4 : 2);
  a.seq_logp = seq_logp;
  a.tok_out = tok_logp;
  a.lse_out = row_lse;
  a.seqsum = 1;
  k_prep<<<1, kPrepThreads, 0, s>>>(nullptr, B, 0, w, nullptr, B * T);
  if ((e = launched()) != ODPO_OK) return e;
  return launch_engine(dt == ODPO_F32 ? 0 : 1, M_SEQ, kPolyDefault, a, 0, s, -1);
}

odpo_status odpo_seq_ppl(const void* logits, odpo_dtype dt, int64_t B, int64_t T, int64_t V,
                         int64_t stride_b, int64_t stride_t, const int32_t* tokens,
                         const uint8_t* mask, float inv_temperature, float* seq_logp, float* ppl,
                         double* ppl_stats, uint32_t* status, void* workspace,
                         size_t workspace_bytes, void* stream) {
  if (!ppl || !ppl_stats) return ODPO_ERR_INVALID_ARG;
  odpo_status e = odpo_seq_logprobs(logits, dt, B, T, V, stride_b, stride_t, tokens, mask,
                                    inv_temperature, seq_logp, nullptr, nullptr, status,
                                    workspace, workspace_bytes, stream);
  if (e != ODPO_OK) return e;
  Workspace w;
  ws_layout(B, T, B / 2 + 1, (char*)workspace, &w);
  LossArgs a;
  base_args(a, logits, B, T, V, stride_b, stride_t, tokens, mask, inv_temperature, status, w,
            dt == ODPO_F32 ? 4 : 2);
  k_seq_ppl<<<1, 32 * kPplWarps, 0, (cudaStream_t)stream>>>(a, ppl, ppl_stats);
  return launched();
}

// Wave schedule geometry: groups of 2T CTAs (one row per CTA per pair), as many groups as the
// resident grid holds and as keep every group's in-flight pair within half of L2; 0 when the
// wave does not apply (2T above the grid, a pair larger than the L2 budget, clusters).
#ifndef ODPO_WAVE_BUDGET_PCT
#define ODPO_WAVE_BUDGET_PCT 90
#endif
constexpr int kWaveGap = 1;
static int wave_groups(int64_t T, int64_t P, int64_t row_bytes, int cps, int geo, int dti,
                       bool busy_half, int gap) {
  if (kCS != 1) return 0;
  int dev = 0;
  cudaGetDevice(&dev);
  const DevInfo& di = dev_info(dev);
  const int g = geo >= 0 ? geo : 0;
  if (g > 1) return 0;
  int occ = di.occ[g][dti][M_FUSED];
  if (occ < 1) occ = 1;
  if (cps <= 0 || cps > occ) cps = occ;
  const int64_t grid = (int64_t)di.sms * cps;
  const int64_t R = 2 * T;
  const int64_t pair_bytes = R * row_bytes;
  if (R > grid) return 0;
  int64_t ng = grid / R;
  // logits of (1 + gap) pairs per group are held between their forward and backward rows
  const int64_t budget = (int64_t)di.l2 * ODPO_WAVE_BUDGET_PCT / 100;
  if (ng * (1 + gap) * pair_bytes > budget) ng = budget / ((1 + gap) * pair_bytes);
  if (ng > P) ng = P;
  if (ng < 1) return 0;
  if (busy_half && ng * R * 2 < grid) return 0;  // AUTO: at least half the CTAs busy
  return (int)ng;
}

// Shared argument checks of the two loss entry points (dl = dlogits or G).
static odpo_status check_loss(const void* logits, odpo_dtype dt, int64_t B, int64_t T, int64_t V,
                              int64_t sb, int64_t st, const float* ref_logp,
                              const int32_t* tokens, const uint8_t* mask,
                              const int32_t* pair_rows, int64_t P, int64_t P_global, float beta,
                              float invT, const void* dl, int64_t dsb, int64_t dst,
                              const float* seq_logp, const double* stats, const void* workspace,
                              size_t workspace_bytes) {
  odpo_status e = check_logits(logits, dt, B, T, V, sb, st);
  if (e != ODPO_OK) return e;
  if (!ref_logp || !tokens || !mask || !dl || !seq_logp || !stats) return ODPO_ERR_INVALID_ARG;
  if (P <= 0 || P_global < P || !finite_pos(beta) || !finite_pos(invT)) return ODPO_ERR_INVALID_ARG;
  if (!pair_rows && B != 2 * P) return ODPO_ERR_INVALID_ARG;
  if (dst < V || dsb < 0) return ODPO_ERR_INVALID_ARG;
  if (B > 1 && dsb < (T - 1) * dst + V) return ODPO_ERR_INVALID_ARG;
  if (dl == logits && (dsb != sb || dst != st)) return ODPO_ERR_INVALID_ARG;
  const int64_t es = dt == ODPO_F32 ? 4 : 2;
  if (!aligned16(dl) || (dsb * es) % 16 || (dst * es) % 16) return ODPO_ERR_ALIGNMENT;
  if (4 * P * T + B * T >= (int64_t)UINT32_MAX / 2 || P > (int64_t)INT32_MAX / 2)
    return ODPO_ERR_UNSUPPORTED;
  if (!workspace || workspace_bytes < ws_layout(B, T, P, nullptr, nullptr)) return ODPO_ERR_WORKSPACE;
  return ODPO_OK;
}

odpo_status odpo_online_dpo_loss_fwd_bwd_ex(const void* policy_logits, odpo_dtype dt, int64_t B,
                                            int64_t T, int64_t V, int64_t stride_b,
                                            int64_t stride_t, const float* ref_logp,
                                            const int32_t* tokens, const uint8_t* mask,
                                            const int32_t* pair_rows, int64_t P, int64_t P_global,
                                            float beta, float inv_temperature, void* dlogits,
                                            int64_t dstride_b, int64_t dstride_t, float* seq_logp,
                                            float* pair_logit, double* stats, uint32_t* status,
                                            void* workspace, size_t workspace_bytes,
                                            odpo_launch_opts* opts, void* stream) {
  odpo_status e = check_loss(policy_logits, dt, B, T, V, stride_b, stride_t, ref_logp, tokens,
                             mask, pair_rows, P, P_global, beta, inv_temperature, dlogits,
                             dstride_b, dstride_t, seq_logp, stats, workspace, workspace_bytes);
  if (e != ODPO_OK) return e;
  const int64_t es = dt == ODPO_F32 ? 4 : 2;
  int sched = opts ? opts->schedule : ODPO_SCHED_AUTO;
  if (sched < ODPO_SCHED_AUTO || sched > ODPO_SCHED_PSYNC) return ODPO_ERR_UNSUPPORTED;
  const int pv = (opts && opts->exp2_split >= 0) ? opts->exp2_split : kPolyDefault;
  if (pv >= kNumPoly) return ODPO_ERR_UNSUPPORTED;
  int wave_ng = 0;
  const int wave_gap = (opts && opts->row_gap >= 0) ? (opts->row_gap > 0 ? 1 : 0) : kWaveGap;
  int dev = 0;
  cudaGetDevice(&dev);
  const DevInfo& di = dev_info(dev);
  // AUTO = TWO_PASS: the read-only forward pass runs at the read ceiling and the backward at
  // the copy ceiling, which beats FUSED's mixed read/write stream at every BASELINE shape
  // (round 2, same bits: LLaMA 14.87 vs 15.08 ms, Rho 3.80 vs 3.86, Pythia 1.301 vs 1.297,
  // tiny 0.116 vs 0.130; profiles/r02/scripts/run_r02ab.sh).  Neither assumes co-residency.
  const ResGeo rg = res_geo(V, T, (int)es, di.sms, opts ? opts->lookahead : -1);
  const bool res_ok = rg.nsl > 0 && (!opts || (opts->ctas_per_sm <= 0 && opts->engine < 0));
  if (sched == ODPO_SCHED_AUTO) sched = ODPO_SCHED_TWO_PASS;
  if (sched == ODPO_SCHED_RESIDENT && !res_ok) return ODPO_ERR_UNSUPPORTED;
  if (sched == ODPO_SCHED_WAVE) {
    wave_ng = wave_groups(T, P, V * es, opts ? opts->ctas_per_sm : 0, opts ? opts->engine : -1,
                          dt == ODPO_F32 ? 0 : 1, false, wave_gap);
    if (wave_ng == 0) return ODPO_ERR_UNSUPPORTED;
    sched = ODPO_SCHED_FUSED;
  }

  Workspace w;
  ws_layout(B, T, P, (char*)workspace, &w);
  cudaStream_t s = (cudaStream_t)stream;

  LossArgs a;
  base_args(a, policy_logits, B, T, V, stride_b, stride_t, tokens, mask, inv_temperature, status,
            w, (int)es);
  a.ref = ref_logp; a.pair_rows = pair_rows;
  a.P = P; a.Pg = (double)P_global; a.beta = beta;
  a.dl = dlogits; a.dsb = dstride_b; a.dst = dstride_t;
  a.seq_logp = seq_logp; a.z_out = pair_logit; a.stats = stats;

  k_prep<<<1, kPrepThreads, 0, s>>>(pair_rows, B, P, w, status, B * T);
  if ((e = launched()) != ODPO_OK) return e;
  int launches = 1;
  const int dti = dt == ODPO_F32 ? 0 : 1;
  const int geo = opts ? opts->engine : -1;

  if (sched == ODPO_SCHED_PSYNC) {
#if ODPO_EXPERIMENTAL
    // pair-synchronous split-V (odpo_psync.cuh): whole 16-byte vectors per row, a piece spans
    // at most two rows, lag below the partial window; cooperative launch (co-residency)
    const int Nv = dti == 0 ? 4 : 8;
    const int64_t nvec = V / Nv;
    int occ = di.occ_ps[dti];
    if (occ < 1) occ = 1;
    int grid = di.sms * occ;
    if (grid > kPsMaxGrid) grid = kPsMaxGrid;
    if (grid > 2 * T * nvec) grid = (int)(2 * T * nvec);   // every piece non-empty (it counts)
    const int D = (opts && opts->lag_pairs > 0) ? opts->lag_pairs : kPsLagDefault;
    if (V % Nv || 2 * T * nvec / grid > nvec || D >= kPsWinPairs) return ODPO_ERR_UNSUPPORTED;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3(kPsThreads);
    cfg.dynamicSmemBytes = kPsSmem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    if (dti == 0) cudaLaunchKernelEx(&cfg, k_psync<0>, a, D);
    else cudaLaunchKernelEx(&cfg, k_psync<1>, a, D);
    if ((e = launched()) != ODPO_OK) return e;
    if (dti == 0) k_zero_unref<0><<<di.sms * 4, 256, 0, s>>>(a);
    else k_zero_unref<1><<<di.sms * 4, 256, 0, s>>>(a);
    if ((e = launched()) != ODPO_OK) return e;
    launches += 2;
#else
    return ODPO_ERR_UNSUPPORTED;   // built without ODPO_EXPERIMENTAL (measured slower: DESIGN 4)
#endif
  } else if (sched == ODPO_SCHED_RESIDENT) {
    const int ring_bytes = (rg.rf + rg.rbs) * kChunk;
    const int smem = ring_bytes > kResSmemMin ? ring_bytes : kResSmemMin;
    if (dti == 0) k_resident<0, 0, 0><<<di.sms, kResThreads, smem, s>>>(a, rg);
    else launch_res_bf16<0>(pv, di.sms, smem, a, rg, s);
    if ((e = launched()) != ODPO_OK) return e;
    launches += 1;
  } else if (sched == ODPO_SCHED_TWO_PASS) {
    a.seqsum = 0;   // forward rows only; k_pair_reduce sums the sequences
    if ((e = launch_engine(dti, M_SEQ, pv, a, opts ? opts->ctas_per_sm : 0, s, geo)) != ODPO_OK)
      return e;
    k_pair_reduce<<<(unsigned)P, 32, 0, s>>>(a);
    if ((e = launched()) != ODPO_OK) return e;
    const unsigned rows = (unsigned)(B * T);
    if (dt == ODPO_F32) launch_row_bwd_t<0, 0>(rows, a, s);
    else launch_bwd_bf16<0>(pv, rows, a, s);
    if ((e = launched()) != ODPO_OK) return e;
    launches += 3;
  } else {
    a.look = (opts && opts->lookahead >= 0) ? (opts->lookahead < kSlots - 2 ? opts->lookahead : kSlots - 2) : kLook;
    // optional cap on the forward lead (default none: measured, capping idles CTAs more than
    // it saves in L2 misses with row-granular work units)
    const int64_t R = 2 * T;
    int64_t lead = (opts && opts->lag_pairs > 0) ? (int64_t)opts->lag_pairs * R : (int64_t)INT32_MAX;
    if (lead < 2 * R) lead = 2 * R;
    a.max_lead = lead;
    a.wave_ng = wave_ng;
    a.wave_gs = (int)(2 * T);
    a.wave_gap = wave_gap;
    const int cps = opts ? opts->ctas_per_sm : 0;
    if ((e = launch_engine(dti, M_FUSED, pv, a, cps, s, geo)) != ODPO_OK) return e;
    launches += 1;
  }
  if (opts) opts->launches = launches;
  return ODPO_OK;
}

odpo_status odpo_online_dpo_loss_fwd_bwd(const void* policy_logits, odpo_dtype dt, int64_t B,
                                         int64_t T, int64_t V, int64_t stride_b, int64_t stride_t,
                                         const float* ref_logp, const int32_t* tokens,
                                         const uint8_t* mask, const int32_t* pair_rows, int64_t P,
                                         int64_t P_global, float beta, float inv_temperature,
                                         void* dlogits, int64_t dstride_b, int64_t dstride_t,
                                         float* seq_logp, float* pair_logit, double* stats,
                                         uint32_t* status, void* workspace, size_t workspace_bytes,
                                         void* stream) {
  return odpo_online_dpo_loss_fwd_bwd_ex(policy_logits, dt, B, T, V, stride_b, stride_t, ref_logp,
                                         tokens, mask, pair_rows, P, P_global, beta,
                                         inv_temperature, dlogits, dstride_b, dstride_t, seq_logp,
                                         pair_logit, stats, status, workspace, workspace_bytes,
                                         nullptr, stream);
}

odpo_status odpo_online_dpo_loss_from_token_logp(
    const float* tok_logp, int64_t B, int64_t T, const float* ref_logp, const uint8_t* mask,
    const int32_t* pair_rows, int64_t P, int64_t P_global, float beta, float inv_temperature,
    float* seq_logp, float* pair_logit, double* stats, float* row_scale, uint32_t* status,
    void* workspace, size_t workspace_bytes, void* stream) {
  if (!tok_logp || !ref_logp || !mask || !seq_logp || !stats) return ODPO_ERR_INVALID_ARG;
  if (B <= 0 || T <= 0 || P <= 0 || P_global < P) return ODPO_ERR_INVALID_ARG;
  if (!finite_pos(beta) || !finite_pos(inv_temperature)) return ODPO_ERR_INVALID_ARG;
  if (!pair_rows && B != 2 * P) return ODPO_ERR_INVALID_ARG;
  if (B * T > (int64_t)INT32_MAX || P > (int64_t)INT32_MAX / 2) return ODPO_ERR_UNSUPPORTED;
  if (!workspace || workspace_bytes < ws_layout(B, T, P, nullptr, nullptr)) return ODPO_ERR_WORKSPACE;
  Workspace w;
  ws_layout(B, T, P, (char*)workspace, &w);
  w.row_logp = const_cast<float*>(tok_logp);  // the pair reduction reads (never writes) these
  cudaStream_t s = (cudaStream_t)stream;
  LossArgs a;
  base_args(a, nullptr, B, T, 1, T, 1, nullptr, mask, inv_temperature, status, w, 2);
  a.ref = ref_logp; a.pair_rows = pair_rows;
  a.P = P; a.Pg = (double)P_global; a.beta = beta;
  a.seq_logp = seq_logp; a.z_out = pair_logit; a.stats = stats;
  a.row_scale = row_scale;
  // rows of unreferenced sequences get row_scale 0; the pair reduction writes the others
  if (row_scale && cudaMemsetAsync(row_scale, 0, (size_t)(B * T) * sizeof(float), s) != cudaSuccess)
    return ODPO_ERR_CUDA;
  k_prep<<<1, kPrepThreads, 0, s>>>(pair_rows, B, P, w, status, B * T);
  odpo_status e;
  if ((e = launched()) != ODPO_OK) return e;
  k_pair_reduce<<<(unsigned)P, 32, 0, s>>>(a);
  return launched();
}

odpo_status odpo_online_dpo_loss_fwd_bwd_unscaled(
    const void* policy_logits, odpo_dtype dt, int64_t B, int64_t T, int64_t V, int64_t stride_b,
    int64_t stride_t, const float* ref_logp, const int32_t* tokens, const uint8_t* mask,
    const int32_t* pair_rows, int64_t P, int64_t P_global, float beta, float inv_temperature,
    void* G, int64_t gstride_b, int64_t gstride_t, float* row_scale, float* seq_logp,
    float* pair_logit, double* stats, uint32_t* status, void* workspace, size_t workspace_bytes,
    odpo_launch_opts* opts, void* stream) {
  odpo_status e = check_loss(policy_logits, dt, B, T, V, stride_b, stride_t, ref_logp, tokens,
                             mask, pair_rows, P, P_global, beta, inv_temperature, G, gstride_b,
                             gstride_t, seq_logp, stats, workspace, workspace_bytes);
  if (e != ODPO_OK) return e;
  if (!row_scale) return ODPO_ERR_INVALID_ARG;
  const bool resident = opts && opts->schedule == ODPO_SCHED_RESIDENT;
  const bool split = opts && opts->schedule == ODPO_SCHED_SPLIT;
  if (opts && opts->schedule != ODPO_SCHED_AUTO && !resident && !split) return ODPO_ERR_UNSUPPORTED;
  if (resident && !ODPO_EXPERIMENTAL) return ODPO_ERR_UNSUPPORTED;
  const int pv = (opts && opts->exp2_split >= 0) ? opts->exp2_split : kPolyDefault;
  if (pv >= kNumPoly) return ODPO_ERR_UNSUPPORTED;
  if (split && pv != 0) return ODPO_ERR_UNSUPPORTED;
  Workspace w;
  ws_layout(B, T, P, (char*)workspace, &w);
  cudaStream_t s = (cudaStream_t)stream;
  LossArgs a;
  base_args(a, policy_logits, B, T, V, stride_b, stride_t, tokens, mask, inv_temperature, status,
            w, dt == ODPO_F32 ? 4 : 2);
  a.ref = ref_logp; a.pair_rows = pair_rows;
  a.P = P; a.Pg = (double)P_global; a.beta = beta;
  a.dl = G; a.dsb = gstride_b; a.dst = gstride_t;
  a.seq_logp = seq_logp; a.z_out = pair_logit; a.stats = stats;
  a.row_scale = row_scale;
  // the producer emits up to three slots per ticket; keep the decode window inside the ring
  const int look = (opts && opts->lookahead >= 0) ? opts->lookahead : kLook;
  a.look = look < kSlots - 6 ? look : kSlots - 6;
  if (opts && opts->row_gap > 1) return ODPO_ERR_UNSUPPORTED;
  a.row_gap = (opts && opts->row_gap >= 0) ? opts->row_gap : 0;
  k_prep<<<1, kPrepThreads, 0, s>>>(pair_rows, B, P, w, status, B * T);
  if ((e = launched()) != ODPO_OK) return e;
  if (split) {
#if ODPO_EXPERIMENTAL
    const bool tma = opts->engine == 2;   // A/B: 2 = the TMA-staged pieces, else registers
    if (!(tma ? (dt == ODPO_F32 ? launch_unsc_tma<0>(a, s) : launch_unsc_tma<1>(a, s))
              : (dt == ODPO_F32 ? launch_unsc_split<0>(a, s) : launch_unsc_split<1>(a, s))))
      return ODPO_ERR_UNSUPPORTED;
#else
    return ODPO_ERR_UNSUPPORTED;   // built without ODPO_EXPERIMENTAL (measured slower: DESIGN 4)
#endif
    if ((e = launched()) != ODPO_OK) return e;
    opts->launches = 2;
    return ODPO_OK;
  }
  if (resident) {
    if (pv != 0) return ODPO_ERR_UNSUPPORTED;
    if ((e = launch_res_un(dt == ODPO_F32 ? 0 : 1, a, V, dt == ODPO_F32 ? 4 : 2, opts->lookahead,
                           s)) != ODPO_OK)
      return e;
    opts->launches = 2;
    return ODPO_OK;
  }
  const int geo = opts ? opts->engine : -1;
  if ((e = launch_engine(dt == ODPO_F32 ? 0 : 1, M_UNSC, pv, a, opts ? opts->ctas_per_sm : 0, s,
                         geo)) != ODPO_OK)
    return e;
  if (opts) opts->launches = 2;
  return ODPO_OK;
}

odpo_status odpo_pg_loss_fwd_bwd(const void* policy_logits, odpo_dtype dt, int64_t B, int64_t T,
                                 int64_t V, int64_t stride_b, int64_t stride_t,
                                 const int32_t* tokens, const uint8_t* mask,
                                 const int32_t* pair_rows, int64_t P, int64_t P_global,
                                 int32_t kind, const float* rewards, const float* old_logp,
                                 float clip_eps, float inv_temperature, void* dlogits,
                                 int64_t dstride_b, int64_t dstride_t, float* seq_logp,
                                 double* stats, uint32_t* status, void* workspace,
                                 size_t workspace_bytes, odpo_launch_opts* opts, void* stream) {
  if (kind < ODPO_PG_RLOO || kind > ODPO_PG_BEST_OF_K_SFT || !rewards) return ODPO_ERR_INVALID_ARG;
  if ((kind == ODPO_PG_COPG || kind == ODPO_PG_PROX_RLOO) && !old_logp) return ODPO_ERR_INVALID_ARG;
  if (kind == ODPO_PG_PROX_RLOO && !(clip_eps >= 0.f && clip_eps < 1.f)) return ODPO_ERR_INVALID_ARG;
  // the shared checks (ref_logp is not an input here: pass a valid pointer to skip its check)
  odpo_status e = check_loss(policy_logits, dt, B, T, V, stride_b, stride_t, rewards, tokens,
                             mask, pair_rows, P, P_global, 1.f, inv_temperature, dlogits,
                             dstride_b, dstride_t, seq_logp, stats, workspace, workspace_bytes);
  if (e != ODPO_OK) return e;
  const int pv = (opts && opts->exp2_split >= 0) ? opts->exp2_split : kPolyDefault;
  if (pv >= kNumPoly) return ODPO_ERR_UNSUPPORTED;
  const int sched = opts ? opts->schedule : ODPO_SCHED_AUTO;
  if (sched < ODPO_SCHED_AUTO || sched > ODPO_SCHED_TWO_PASS) return ODPO_ERR_UNSUPPORTED;
  Workspace w;
  ws_layout(B, T, P, (char*)workspace, &w);
  cudaStream_t s = (cudaStream_t)stream;
  LossArgs a;
  base_args(a, policy_logits, B, T, V, stride_b, stride_t, tokens, mask, inv_temperature, status,
            w, dt == ODPO_F32 ? 4 : 2);
  a.pair_rows = pair_rows;
  a.P = P; a.Pg = (double)P_global; a.beta = 1.f;
  a.dl = dlogits; a.dsb = dstride_b; a.dst = dstride_t;
  a.seq_logp = seq_logp; a.stats = stats;
  a.pg_kind = kind; a.rewards = rewards; a.old_logp = old_logp; a.clip_eps = clip_eps;
  const int dti = dt == ODPO_F32 ? 0 : 1;
  const int geo = opts ? opts->engine : -1;
  const int cps = opts ? opts->ctas_per_sm : 0;
  k_prep<<<1, kPrepThreads, 0, s>>>(pair_rows, B, P, w, status, B * T);
  if ((e = launched()) != ODPO_OK) return e;
  int launches = 1;
  if (kind != ODPO_PG_PROX_RLOO) {
    // coefficients known before the forward pass: each row's scaled backward follows its own
    // forward in the same CTA (one HBM read, one write)
    k_pg_coef<<<(unsigned)((P + 255) / 256), 256, 0, s>>>(a);
    if ((e = launched()) != ODPO_OK) return e;
    a.coef_known = 1;
    const int look = (opts && opts->lookahead >= 0) ? opts->lookahead : kLook;
    a.look = look < kSlots - 6 ? look : kSlots - 6;
    a.row_gap = 0;
    if ((e = launch_engine(dti, M_UNSC, pv, a, cps, s, geo)) != ODPO_OK) return e;
    launches += 2;
  } else if (sched == ODPO_SCHED_TWO_PASS) {
    a.seqsum = 0;
    if ((e = launch_engine(dti, M_SEQ, pv, a, cps, s, geo)) != ODPO_OK) return e;
    k_pair_reduce<<<(unsigned)P, 32, 0, s>>>(a);
    if ((e = launched()) != ODPO_OK) return e;
    const unsigned rows = (unsigned)(B * T);
    if (dt == ODPO_F32) launch_row_bwd_t<0, 0>(rows, a, s);
    else launch_bwd_bf16<0>(pv, rows, a, s);
    if ((e = launched()) != ODPO_OK) return e;
    launches += 3;
  } else {
    // Proximal RLOO: the coefficient needs the sequence's own log-prob (its pair's forward)
    a.look = (opts && opts->lookahead >= 0) ? (opts->lookahead < kSlots - 2 ? opts->lookahead : kSlots - 2) : kLook;
    a.max_lead = (int64_t)INT32_MAX;
    if ((e = launch_engine(dti, M_FUSED, pv, a, cps, s, geo)) != ODPO_OK) return e;
    launches += 1;
  }
  if (opts) opts->launches = launches;
  return ODPO_OK;
}

odpo_status odpo_gather_pairs(const int32_t* pair_rows, int64_t P, int64_t n_src, int64_t T,
                              const int32_t* tokens_in, const uint8_t* mask_in,
                              const float* ref_in, int32_t* tokens_out, uint8_t* mask_out,
                              float* ref_out, uint32_t* status, void* stream) {
  if (P < 0 || n_src < 0 || T <= 0) return ODPO_ERR_INVALID_ARG;
  if (P == 0) return ODPO_OK;
  if (!pair_rows) return ODPO_ERR_INVALID_ARG;
  if ((tokens_out && !tokens_in) || (mask_out && !mask_in) || (ref_out && !ref_in))
    return ODPO_ERR_INVALID_ARG;
  if (2 * P > (int64_t)INT32_MAX) return ODPO_ERR_UNSUPPORTED;
  k_gather_pairs<<<(unsigned)(2 * P), 128, 0, (cudaStream_t)stream>>>(
      pair_rows, n_src, T, tokens_in, mask_in, ref_in, tokens_out, mask_out, ref_out, status);
  return launched();
}

odpo_status odpo_vp_row_partials(const void* logits_shard, odpo_dtype dt, int64_t B, int64_t T,
                                 int64_t V_shard, int64_t stride_b, int64_t stride_t,
                                 int64_t v0, int64_t V_total, const int32_t* tokens,
                                 const uint8_t* mask, float inv_temperature, float* parts,
                                 uint32_t* status, void* workspace, size_t workspace_bytes,
                                 void* stream) {
  odpo_status e = check_logits(logits_shard, dt, B, T, V_shard, stride_b, stride_t);
  if (e != ODPO_OK) return e;
  if (!tokens || !mask || !parts || !finite_pos(inv_temperature)) return ODPO_ERR_INVALID_ARG;
  if (v0 < 0 || V_total < v0 + V_shard) return ODPO_ERR_INVALID_ARG;
  if (((uintptr_t)parts & 15u) != 0) return ODPO_ERR_ALIGNMENT;
  const int64_t P = B / 2 + 1;
  if (!workspace || workspace_bytes < ws_layout(B, T, P, nullptr, nullptr)) return ODPO_ERR_WORKSPACE;
  Workspace w;
  ws_layout(B, T, P, (char*)workspace, &w);
  cudaStream_t s = (cudaStream_t)stream;
  LossArgs a;
  base_args(a, logits_shard, B, T, V_shard, stride_b, stride_t, tokens, mask, inv_temperature,
            status, w, dt == ODPO_F32 ? 4 : 2);
  a.vp_parts = reinterpret_cast<float4*>(parts);
  a.tok_off = v0;
  a.V_total = V_total;
  a.seqsum = 0;
  if (V_shard * (dt == ODPO_F32 ? 4 : 2) <= (32 << 10)) {  // short shard rows: a warp per row
    const int64_t rows = B * T;
    const unsigned grid = (unsigned)((rows + kWarpRowsPerCta - 1) / kWarpRowsPerCta);
    if (dt == ODPO_F32) k_vp_partials_warp<0><<<grid, 32 * kWarpRowsPerCta, 0, s>>>(a);
    else k_vp_partials_warp<1><<<grid, 32 * kWarpRowsPerCta, 0, s>>>(a);
    return launched();
  }
  k_prep<<<1, kPrepThreads, 0, s>>>(nullptr, B, 0, w, nullptr, B * T);
  if ((e = launched()) != ODPO_OK) return e;
  return launch_engine(dt == ODPO_F32 ? 0 : 1, M_SEQ, kPolyDefault, a, 0, s, -1);
}

odpo_status odpo_stats_put(const double* stats, double* const* peer_slots,
                           uint32_t* const* peer_flags, int32_t rank, int32_t W, uint32_t epoch,
                           void* stream) {
  if (!stats || !peer_slots || !peer_flags || W < 1 || W > kVpMaxW || rank < 0 || rank >= W)
    return ODPO_ERR_INVALID_ARG;
  VpPut put{};
  for (int q = 0; q < W; ++q) {
    if (!peer_slots[q] || !peer_flags[q]) return ODPO_ERR_INVALID_ARG;
    put.parts[q] = reinterpret_cast<float4*>(peer_slots[q]);
    put.flags[q] = peer_flags[q];
  }
  put.rank = rank;
  put.W = W;
  put.epoch = epoch;
  k_stats_put<<<1, 32, 0, (cudaStream_t)stream>>>(stats, put);
  return launched();
}

odpo_status odpo_stats_sum(const double* slots, const uint32_t* flags, int32_t W, uint32_t epoch,
                           double* out, void* stream) {
  if (!slots || !flags || !out || W < 1 || W > kVpMaxW) return ODPO_ERR_INVALID_ARG;
  k_stats_sum<<<1, 32, 0, (cudaStream_t)stream>>>(slots, flags, W, epoch, out);
  return launched();
}

odpo_status odpo_vp_row_partials_put(const void* logits_shard, odpo_dtype dt, int64_t B,
                                     int64_t T, int64_t V_shard, int64_t stride_b,
                                     int64_t stride_t, int64_t v0, int64_t V_total,
                                     const int32_t* tokens, const uint8_t* mask,
                                     float inv_temperature, float* const* peer_parts,
                                     uint32_t* const* peer_flags, uint32_t* done, int32_t rank,
                                     int32_t W, uint32_t epoch, uint32_t* status, void* stream) {
  odpo_status e = check_logits(logits_shard, dt, B, T, V_shard, stride_b, stride_t);
  if (e != ODPO_OK) return e;
  if (!tokens || !mask || !peer_parts || !peer_flags || !done || !finite_pos(inv_temperature))
    return ODPO_ERR_INVALID_ARG;
  if (W < 1 || W > kVpMaxW || rank < 0 || rank >= W) return ODPO_ERR_INVALID_ARG;
  if (v0 < 0 || V_total < v0 + V_shard) return ODPO_ERR_INVALID_ARG;
  LossArgs a;
  Workspace w{};
  base_args(a, logits_shard, B, T, V_shard, stride_b, stride_t, tokens, mask, inv_temperature,
            status, w, dt == ODPO_F32 ? 4 : 2);
  for (int q = 0; q < W; ++q) {
    if (!peer_parts[q] || !peer_flags[q]) return ODPO_ERR_INVALID_ARG;
    if (((uintptr_t)peer_parts[q] & 15u) != 0) return ODPO_ERR_ALIGNMENT;
    a.put.parts[q] = reinterpret_cast<float4*>(peer_parts[q]);
    a.put.flags[q] = peer_flags[q];
  }
  a.put.done = done;
  a.put.rank = rank;
  a.put.W = W;
  a.put.epoch = epoch;
  a.tok_off = v0;
  a.V_total = V_total;
  const int64_t rows = B * T;
  const unsigned grid = (unsigned)((rows + kWarpRowsPerCta - 1) / kWarpRowsPerCta);
  cudaStream_t s = (cudaStream_t)stream;
  if (dt == ODPO_F32) k_vp_partials_warp<0><<<grid, 32 * kWarpRowsPerCta, 0, s>>>(a);
  else k_vp_partials_warp<1><<<grid, 32 * kWarpRowsPerCta, 0, s>>>(a);
  return launched();
}

odpo_status odpo_vp_loss_fwd_bwd(const float* parts_all, int32_t W, const void* logits_shard,
                                 odpo_dtype dt, int64_t B, int64_t T, int64_t V_shard,
                                 int64_t stride_b, int64_t stride_t, int64_t v0, int64_t V_total,
                                 const float* ref_logp, const int32_t* tokens,
                                 const uint8_t* mask, const int32_t* pair_rows, int64_t P,
                                 int64_t P_global, float beta, float inv_temperature,
                                 void* dlogits_shard, int64_t dstride_b, int64_t dstride_t,
                                 float* seq_logp, float* pair_logit, double* stats,
                                 const uint32_t* flags, uint32_t epoch, uint32_t* status,
                                 void* workspace, size_t workspace_bytes, void* stream) {
  if (!parts_all || W < 1 || W > (flags ? kVpMaxW : 1 << 20)) return ODPO_ERR_INVALID_ARG;
  if (v0 < 0 || V_total < v0 + V_shard) return ODPO_ERR_INVALID_ARG;
  odpo_status e = check_loss(logits_shard, dt, B, T, V_shard, stride_b, stride_t, ref_logp, tokens,
                             mask, pair_rows, P, P_global, beta, inv_temperature, dlogits_shard,
                             dstride_b, dstride_t, seq_logp, stats, workspace, workspace_bytes);
  if (e != ODPO_OK) return e;
  if (((uintptr_t)parts_all & 15u) != 0) return ODPO_ERR_ALIGNMENT;
  Workspace w;
  ws_layout(B, T, P, (char*)workspace, &w);
  cudaStream_t s = (cudaStream_t)stream;
  LossArgs a;
  base_args(a, logits_shard, B, T, V_shard, stride_b, stride_t, tokens, mask, inv_temperature,
            status, w, dt == ODPO_F32 ? 4 : 2);
  a.ref = ref_logp; a.pair_rows = pair_rows;
  a.P = P; a.Pg = (double)P_global; a.beta = beta;
  a.dl = dlogits_shard; a.dsb = dstride_b; a.dst = dstride_t;
  a.seq_logp = seq_logp; a.z_out = pair_logit; a.stats = stats;
  a.tok_off = v0;
  a.V_total = V_total;
  a.vp_flags = flags;
  a.vp_epoch = epoch;
  k_prep<<<1, kPrepThreads, 0, s>>>(pair_rows, B, P, w, status, B * T);
  if ((e = launched()) != ODPO_OK) return e;
  const int64_t rows = B * T;
  if (W > 32 && !flags)
    k_vp_combine_wide<<<(unsigned)((rows + kCombineWarps - 1) / kCombineWarps), 32 * kCombineWarps,
                        0, s>>>(a, reinterpret_cast<const float4*>(parts_all), W);
  else
    k_vp_combine<<<(unsigned)((rows + 255) / 256), 256, 0, s>>>(
        a, reinterpret_cast<const float4*>(parts_all), W);
  if ((e = launched()) != ODPO_OK) return e;
  k_pair_reduce<<<(unsigned)P, 32, 0, s>>>(a);
  if ((e = launched()) != ODPO_OK) return e;
  if (V_shard * (dt == ODPO_F32 ? 4 : 2) <= (32 << 10)) {  // short shard rows: a warp per row
    const unsigned grid = (unsigned)((rows + kWarpRowsPerCta - 1) / kWarpRowsPerCta);
    if (kVpWarp) {
      if (dt == ODPO_F32) k_row_bwd_warp<0><<<grid, 32 * kWarpRowsPerCta, 0, s>>>(a);
      else k_row_bwd_warp<1><<<grid, 32 * kWarpRowsPerCta, 0, s>>>(a);
    } else if (dt == ODPO_F32) {
      launch_split<0, 0, 128, 4>((unsigned)rows, a, s);
    } else {
      launch_split<1, 0, 128, 4>((unsigned)rows, a, s);
    }
  } else if (dt == ODPO_F32) {
    launch_row_bwd_t<0, 0>((unsigned)rows, a, s);
  } else {
    launch_row_bwd_t<1, 0>((unsigned)rows, a, s);
  }
  return launched();
}

}  // extern "C"
