// odpo.cu -- libodpo.so: kernels and C ABI of the Online-DPO learner hot path on B200.
//
// Kernels:
//   k_pair_select    K1  reward-ranked pair selection + selection stats
//   k_prep           --  per-call workspace init, sequence->pair map, DUP/RANGE checks
//   k_row_fwd        K2  one CTA per row: online LSE + gather  (seq_logprobs, TWO_PASS)
//   k_seq_sum        K3a one warp per sequence: fixed-order masked sum
//   k_pair_reduce    K3b one CTA per pair: DPO logit, -log sigma, coef, stats
//   k_row_bwd        K4  one CTA per row: dlogits = coef (softmax - onehot)
//   k_fused          K5  persistent: forward rows of pair s interleaved with backward rows of
//                        pair s-lag; per-pair completion counters; backward re-reads hit L2
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include <mutex>

#include "odpo.h"
#include "odpo_device.cuh"

#define ODPO_VERSION_STR "odpo-b200 0.1.0 (sm_100a)"

namespace odpo {

// ------------------------------------------------------------------ workspace layout
struct Workspace {
  float* row_m;
  float* row_l1p;
  float* row_logp;
  float* seq_coef;
  int32_t* seq_pair;   // 2p (chosen of p) / 2p+1 (rejected of p) / -1 unreferenced
  int32_t* unref;      // unreferenced sequences, ascending
  unsigned* pair_cnt;  // forward rows done
  unsigned* pair_ready;
  double* pair_vals;   // [P][ODPO_NSTATS]
  unsigned* counters;  // [0] ticket, [1] pairs done, [2] n_unref
};

enum { C_TICKET = 0, C_PAIRS_DONE = 1, C_NUNREF = 2, C_COUNT = 8 };

static inline size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

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
  char* p_pc = take((size_t)P * 4);
  char* p_pr = take((size_t)P * 4);
  char* p_pv = take((size_t)P * ODPO_NSTATS * 8);
  char* p_ct = take(C_COUNT * 4);
  if (w) {
    w->row_m = (float*)p_m;
    w->row_l1p = (float*)p_l;
    w->row_logp = (float*)p_lp;
    w->seq_coef = (float*)p_c;
    w->seq_pair = (int32_t*)p_sp;
    w->unref = (int32_t*)p_u;
    w->pair_cnt = (unsigned*)p_pc;
    w->pair_ready = (unsigned*)p_pr;
    w->pair_vals = (double*)p_pv;
    w->counters = (unsigned*)p_ct;
  }
  return off;
}

__device__ __forceinline__ void flag(uint32_t* status, uint32_t f) {
  if (f && status) atomicOr(status, f);
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
                                                       uint32_t* status) {
  __shared__ int scan[kPrepThreads];
  const int tid = threadIdx.x;
  for (int64_t b = tid; b < B; b += kPrepThreads) w.seq_pair[b] = -1;
  for (int64_t p = tid; p < P; p += kPrepThreads) {
    w.pair_cnt[p] = 0;
    w.pair_ready[p] = 0;
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

// ------------------------------------------------------------------ shared loss arguments
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
  Workspace w;
  int lag;
  int esize;
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

// Pair reduction (K3b) by a whole CTA (>= 64 threads): warps 0/1 sum the two sequences in
// fixed order, thread 0 forms z, loss, sigma(-z), coef, publishes them and the pair's
// statistics; the CTA that completes the LAST pair reduces all pairs in fixed order.
__device__ void pair_reduce(const LossArgs& a, int64_t p, double* smd, int* smi) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int64_t c, r;
  pair_seqs(a, p, c, r);
  if (warp < 2) {
    const int64_t s = warp == 0 ? c : r;
    double S = 0.0;
    int n = 0;
    if (s >= 0) seq_sum_warp(a.w.row_logp + s * a.T, a.mask + s * a.T, a.T, S, n);
    if (lane == 0) {
      smd[warp] = S;
      smi[warp] = n;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t fl = 0;
    double* pv = a.w.pair_vals + p * ODPO_NSTATS;
    if (c < 0 || r < 0) {
      for (int k = 0; k < ODPO_NSTATS; ++k) pv[k] = 0.0;
      if (a.z_out) a.z_out[p] = 0.f;
    } else {
      const int nc = smi[0], nr = smi[1];
      if (nc == 0 || nr == 0) fl |= ODPO_FLAG_EMPTY_SEQ;
      const float Sc = nc ? (float)smd[0] : 0.f;
      const float Sr = nr ? (float)smd[1] : 0.f;
      const float dc = __fsub_rn(Sc, a.ref[c]);
      const float dr = __fsub_rn(Sr, a.ref[r]);
      const float z = __fmul_rn(a.beta, __fsub_rn(dc, dr));   // no FMA contraction (R15)
      const double zd = (double)z;
      const double loss_p = fmax(-zd, 0.0) + log1p(exp(-fabs(zd)));  // softplus(-z)
      const double sig_neg = 1.0 / (1.0 + exp(zd));                  // sigma(-z)
      const float coef = (float)((double)a.beta * sig_neg * (double)a.invT / a.Pg);
      a.w.seq_coef[c] = coef;
      a.w.seq_coef[r] = -coef;
      a.seq_logp[c] = Sc;
      a.seq_logp[r] = Sr;
      if (a.z_out) a.z_out[p] = z;
      pv[ODPO_ST_NPAIRS] = 1.0;
      pv[ODPO_ST_LOSS] = loss_p;
      pv[ODPO_ST_NCORRECT] = z > 0.f ? 1.0 : 0.0;
      pv[ODPO_ST_Z] = zd;
      pv[ODPO_ST_RCHOSEN] = (double)a.beta * (double)dc;
      pv[ODPO_ST_RREJ] = (double)a.beta * (double)dr;
      pv[ODPO_ST_SCHOSEN] = (double)Sc;
      pv[ODPO_ST_SREJ] = (double)Sr;
      pv[ODPO_ST_NTOK_CHOSEN] = (double)nc;
      pv[ODPO_ST_NTOK_REJ] = (double)nr;
    }
    flag(a.status, fl);
    __threadfence();
    st_release(&a.w.pair_ready[p], 1u);
    const unsigned done = atomicAdd(&a.w.counters[C_PAIRS_DONE], 1u);
    smi[2] = (done == (unsigned)(a.P - 1));
  }
  __syncthreads();
  if (smi[2] && warp == 0) {
    __threadfence();
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
}

// ------------------------------------------------------------------ K2 row forward (grid = rows)
struct FwdArgs {
  const void* logits;
  int64_t T, V, sb, st;
  const int32_t* tokens;
  const uint8_t* mask;
  float invT;
  float* row_m;
  float* row_l1p;
  float* row_logp;
  float* tok_logp;  // nullable (seq_logprobs output)
  float* row_lse;   // nullable
  uint32_t* status;
  int esize;
};

template <int DT>
__global__ void __launch_bounds__(kRowThreads, 2) k_row_fwd(FwdArgs a) {
  __shared__ float sm[2 * kWarps];
  const int64_t g = blockIdx.x;
  const int64_t b = g / a.T, t = g % a.T;
  if (!a.mask[g]) {
    if (threadIdx.x == 0) {
      if (a.tok_logp) a.tok_logp[g] = 0.f;
      if (a.row_lse) a.row_lse[g] = 0.f;
    }
    return;
  }
  const char* row = reinterpret_cast<const char*>(a.logits) + (b * a.sb + t * a.st) * a.esize;
  RowOut o = row_forward<DT, LD_STREAM>(row, (int)a.V, a.tokens[g], a.invT, 0, sm);
  if (threadIdx.x == 0) {
    a.row_m[g] = o.m;
    a.row_l1p[g] = o.l1p;
    a.row_logp[g] = o.logp;
    if (a.tok_logp) a.tok_logp[g] = o.logp;
    if (a.row_lse) a.row_lse[g] = o.lse;
    flag(a.status, o.flags);
  }
}

// ------------------------------------------------------------------ K3a sequence sums
__global__ void __launch_bounds__(256) k_seq_sum(const float* __restrict__ row_logp,
                                                  const uint8_t* __restrict__ mask, int64_t B,
                                                  int64_t T, float* seq_logp, uint32_t* status) {
  const int64_t s = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (s >= B) return;
  double S;
  int n;
  seq_sum_warp(row_logp + s * T, mask + s * T, T, S, n);
  if ((threadIdx.x & 31) == 0) {
    seq_logp[s] = n ? (float)S : 0.f;
    if (!n) flag(status, ODPO_FLAG_EMPTY_SEQ);
  }
}

// ------------------------------------------------------------------ K3b pair reduce (grid = P)
__global__ void __launch_bounds__(64) k_pair_reduce(LossArgs a) {
  __shared__ double smd[2];
  __shared__ int smi[3];
  pair_reduce(a, blockIdx.x, smd, smi);
}

// ------------------------------------------------------------------ K4 row backward (grid = rows)
template <int DT>
__global__ void __launch_bounds__(kRowThreads, 2) k_row_bwd(LossArgs a) {
  const int64_t g = blockIdx.x;
  const int64_t b = g / a.T, t = g % a.T;
  char* drow = drow_ptr(a, b, t);
  if (a.w.seq_pair[b] < 0 || !a.mask[g]) {
    row_zero<DT>(drow, (int)a.V);
    return;
  }
  const float coef = a.w.seq_coef[b];
  row_backward<DT, LD_STREAM>(row_ptr(a, b, t), drow, (int)a.V, a.tokens[g], a.invT, a.w.row_m[g],
                              a.w.row_l1p[g], a.w.row_logp[g], coef, 0);
}

// ------------------------------------------------------------------ K5 fused persistent kernel
// Ticket order (R = 2T rows per pair, d = lag): F(0..d-1), then B(0), F(d), B(1), F(d+1), ...,
// then the remaining B's, then Z rows (unreferenced sequences).  A B item of pair p waits for
// pair_ready[p]; every F item of p has an earlier ticket held by a running CTA and F items never
// wait, so the wait always terminates (no co-residency assumption).
__device__ __forceinline__ void decode_block(int64_t q, int64_t P, int64_t d, bool& fwd, int64_t& p) {
  if (q < d) { fwd = true; p = q; return; }
  const int64_t mid = 2 * (P - d);
  if (q < d + mid) {
    const int64_t u = q - d;
    fwd = (u & 1);
    p = fwd ? d + (u >> 1) : (u >> 1);
    return;
  }
  fwd = false;
  p = (P - d) + (q - d - mid);
}

template <int DT>
__global__ void __launch_bounds__(kRowThreads, 2) k_fused(LossArgs a) {
  __shared__ float sm[2 * kWarps];
  __shared__ unsigned s_ticket[2];
  __shared__ double smd[2];
  __shared__ int smi[3];
  __shared__ int s_last;
  const uint64_t pol_keep = policy_evict_last();
  const uint64_t pol_drop = policy_evict_first();
  const int64_t T = a.T, R = 2 * T;
  const int64_t total_fb = 2 * a.P * R;
  const int64_t total = total_fb + (int64_t)__ldcg(&a.w.counters[C_NUNREF]) * T;
  if (threadIdx.x == 0) s_ticket[0] = atomicAdd(&a.w.counters[C_TICKET], 1u);
  __syncthreads();
  for (int it = 0;; ++it) {
    const int64_t tk = s_ticket[it & 1];
    if (tk >= total) break;
    if (threadIdx.x == 0) s_ticket[(it + 1) & 1] = atomicAdd(&a.w.counters[C_TICKET], 1u);
    if (tk < total_fb) {
      bool fwd;
      int64_t p;
      decode_block(tk / R, a.P, a.lag, fwd, p);
      const int64_t j = tk % R;
      int64_t c, r;
      pair_seqs(a, p, c, r);
      const int64_t s = j < T ? c : r;
      const int64_t t = j < T ? j : j - T;
      const int64_t g = s * T + t;
      if (fwd) {
        if (s >= 0 && a.mask[g]) {
          RowOut o = row_forward<DT, LD_HINT>(row_ptr(a, s, t), (int)a.V, a.tokens[g], a.invT,
                                              pol_keep, sm);
          if (threadIdx.x == 0) {
            a.w.row_m[g] = o.m;
            a.w.row_l1p[g] = o.l1p;
            a.w.row_logp[g] = o.logp;
            flag(a.status, o.flags);
          }
        }
        if (threadIdx.x == 0) {
          __threadfence();
          const unsigned old = atomicAdd(&a.w.pair_cnt[p], 1u);
          s_last = (old == (unsigned)(R - 1));
        }
        __syncthreads();
        if (s_last) {
          __threadfence();
          pair_reduce(a, p, smd, smi);
        }
      } else {
        if (threadIdx.x == 0) {
          while (ld_acquire(&a.w.pair_ready[p]) == 0u) __nanosleep(64);
        }
        __syncthreads();
        if (s >= 0) {
          char* drow = drow_ptr(a, s, t);
          if (!a.mask[g]) {
            row_zero<DT>(drow, (int)a.V);
          } else {
            row_backward<DT, LD_HINT>(row_ptr(a, s, t), drow, (int)a.V, a.tokens[g], a.invT,
                                      __ldcg(a.w.row_m + g), __ldcg(a.w.row_l1p + g),
                                      __ldcg(a.w.row_logp + g), __ldcg(a.w.seq_coef + s),
                                      pol_drop);
          }
        }
      }
    } else {
      const int64_t k = (tk - total_fb) / T, t = (tk - total_fb) % T;
      const int64_t s = __ldcg(a.w.unref + k);
      row_zero<DT>(drow_ptr(a, s, t), (int)a.V);
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------------ host side
struct DevInfo {
  int sms = 0;
  int l2 = 0;
  int occ_fused[2] = {0, 0};
};
static DevInfo g_dev[128];
static std::once_flag g_once[128];

static const DevInfo& dev_info(int dev) {
  std::call_once(g_once[dev], [dev]() {
    DevInfo& d = g_dev[dev];
    cudaDeviceGetAttribute(&d.sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&d.l2, cudaDevAttrL2CacheSize, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&d.occ_fused[0], k_fused<0>, kRowThreads, 0);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&d.occ_fused[1], k_fused<1>, kRowThreads, 0);
  });
  return g_dev[dev];
}

static bool aligned16(const void* p) { return ((uintptr_t)p & 15u) == 0; }
static bool finite_pos(float x) { return isfinite(x) && x > 0.f; }

static odpo_status check_logits(const void* logits, odpo_dtype dt, int64_t B, int64_t T, int64_t V,
                                int64_t sb, int64_t st) {
  if (!logits) return ODPO_ERR_INVALID_ARG;
  if (dt != ODPO_F32 && dt != ODPO_BF16) return ODPO_ERR_INVALID_ARG;
  if (B <= 0 || T <= 0 || V <= 0 || V > (int64_t)INT32_MAX) return ODPO_ERR_INVALID_ARG;
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

}  // namespace odpo

using namespace odpo;

extern "C" {

const char* odpo_version(void) { return ODPO_VERSION_STR; }

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
  FwdArgs f{logits, T, V, stride_b, stride_t, tokens, mask, inv_temperature,
            w.row_m, w.row_l1p, w.row_logp, tok_logp, row_lse, status, dt == ODPO_F32 ? 4 : 2};
  const unsigned rows = (unsigned)(B * T);
  if (dt == ODPO_F32) k_row_fwd<0><<<rows, kRowThreads, 0, s>>>(f);
  else k_row_fwd<1><<<rows, kRowThreads, 0, s>>>(f);
  if ((e = launched()) != ODPO_OK) return e;
  k_seq_sum<<<(unsigned)((B + 7) / 8), 256, 0, s>>>(w.row_logp, mask, B, T, seq_logp, status);
  return launched();
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
  odpo_status e = check_logits(policy_logits, dt, B, T, V, stride_b, stride_t);
  if (e != ODPO_OK) return e;
  if (!ref_logp || !tokens || !mask || !dlogits || !seq_logp || !stats) return ODPO_ERR_INVALID_ARG;
  if (P <= 0 || P_global < P || !finite_pos(beta) || !finite_pos(inv_temperature))
    return ODPO_ERR_INVALID_ARG;
  if (!pair_rows && B != 2 * P) return ODPO_ERR_INVALID_ARG;
  if (dstride_t < V || dstride_b < 0) return ODPO_ERR_INVALID_ARG;
  if (B > 1 && dstride_b < (T - 1) * dstride_t + V) return ODPO_ERR_INVALID_ARG;
  if (dlogits == policy_logits && (dstride_b != stride_b || dstride_t != stride_t))
    return ODPO_ERR_INVALID_ARG;
  const int64_t es = dt == ODPO_F32 ? 4 : 2;
  if (!aligned16(dlogits) || (dstride_b * es) % 16 || (dstride_t * es) % 16) return ODPO_ERR_ALIGNMENT;
  if (4 * P * T + B * T >= (int64_t)UINT32_MAX / 2 || P > (int64_t)INT32_MAX / 2)
    return ODPO_ERR_UNSUPPORTED;
  if (!workspace || workspace_bytes < ws_layout(B, T, P, nullptr, nullptr)) return ODPO_ERR_WORKSPACE;
  const int sched = opts ? opts->schedule : ODPO_SCHED_AUTO;
  if (sched < ODPO_SCHED_AUTO || sched > ODPO_SCHED_TWO_PASS) return ODPO_ERR_UNSUPPORTED;

  Workspace w;
  ws_layout(B, T, P, (char*)workspace, &w);
  cudaStream_t s = (cudaStream_t)stream;
  int dev = 0;
  cudaGetDevice(&dev);
  const DevInfo& di = dev_info(dev);

  LossArgs a;
  a.logits = policy_logits;
  a.B = B; a.T = T; a.V = V; a.sb = stride_b; a.st = stride_t;
  a.ref = ref_logp; a.tokens = tokens; a.mask = mask; a.pair_rows = pair_rows;
  a.P = P; a.Pg = (double)P_global; a.beta = beta; a.invT = inv_temperature;
  a.dl = dlogits; a.dsb = dstride_b; a.dst = dstride_t;
  a.seq_logp = seq_logp; a.z_out = pair_logit; a.stats = stats; a.status = status;
  a.w = w; a.esize = (int)es; a.lag = 1;

  k_prep<<<1, kPrepThreads, 0, s>>>(pair_rows, B, P, w, status);
  if ((e = launched()) != ODPO_OK) return e;
  int launches = 1;

  if (sched == ODPO_SCHED_TWO_PASS) {
    FwdArgs f{policy_logits, T, V, stride_b, stride_t, tokens, mask, inv_temperature,
              w.row_m, w.row_l1p, w.row_logp, nullptr, nullptr, status, (int)es};
    const unsigned rows = (unsigned)(B * T);
    if (dt == ODPO_F32) k_row_fwd<0><<<rows, kRowThreads, 0, s>>>(f);
    else k_row_fwd<1><<<rows, kRowThreads, 0, s>>>(f);
    if ((e = launched()) != ODPO_OK) return e;
    k_pair_reduce<<<(unsigned)P, 64, 0, s>>>(a);
    if ((e = launched()) != ODPO_OK) return e;
    if (dt == ODPO_F32) k_row_bwd<0><<<rows, kRowThreads, 0, s>>>(a);
    else k_row_bwd<1><<<rows, kRowThreads, 0, s>>>(a);
    if ((e = launched()) != ODPO_OK) return e;
    launches += 3;
  } else {
    const int occ = di.occ_fused[dt == ODPO_F32 ? 0 : 1];
    int cps = (opts && opts->ctas_per_sm > 0) ? opts->ctas_per_sm : occ;
    if (cps > occ) cps = occ;
    if (cps < 1) cps = 1;
    const int grid = di.sms * cps;
    // lag: enough pairs that a pair's forward rows are finished before its backward rows are
    // dispensed (grid rows in flight), and no more than ~40% of L2 of logits kept resident.
    const double pair_bytes = (double)(2 * T) * (double)V * (double)es;
    int64_t lag_min = (int64_t)grid / (2 * T) + 2;
    int64_t lag_l2 = (int64_t)(0.4 * (double)di.l2 / pair_bytes);
    int64_t lag = (opts && opts->lag_pairs > 0) ? opts->lag_pairs : (lag_l2 > lag_min ? lag_l2 : lag_min);
    if (lag > P) lag = P;
    if (lag < 1) lag = 1;
    a.lag = (int)lag;
    if (dt == ODPO_F32) k_fused<0><<<grid, kRowThreads, 0, s>>>(a);
    else k_fused<1><<<grid, kRowThreads, 0, s>>>(a);
    if ((e = launched()) != ODPO_OK) return e;
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

}  // extern "C"
