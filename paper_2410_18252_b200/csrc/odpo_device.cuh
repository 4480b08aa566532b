// odpo_device.cuh -- device building blocks of the Online-DPO hot path (sm_100a).
//
// Row forward  (K2): single-read online log-sum-exp over V in "log1p form"
//                    (track r = sum_{v != argmax} exp(invT (x_v - m)), so 1 + r is never
//                    formed by adding tiny terms to 1), plus the sampled-token gather.
//                    PAPER.md:83 (log pi(y|x)); numerics: DESIGN.md section 5.
// Row backward (K4): dlogits = coef * (softmax - onehot), onehot entry via expm1(logp).
// Sequence sum (K3a): fixed-order masked sum over t (double accumulation).
//
// No library kernels; 128-bit vector loads/stores with explicit L2 cache policies.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace odpo {

constexpr int kRowThreads = 512;   // threads per row-CTA (all row kernels; fixes the reduction tree)
constexpr int kU = 8;              // 16-byte vectors in flight per thread per batch
constexpr int kWarps = kRowThreads / 32;
constexpr float kLog2e = 1.4426950408889634f;
constexpr unsigned kFull = 0xffffffffu;

// ------------------------------------------------------------------ PTX helpers
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// exp2 on the FMA pipe (Cody-Waite): 2^x = 2^j * p(f), j = rint(x), f = x - j in [-1/2, 1/2].
// B200's MUFU.EX2 issues ~8 results/clk/SM, below the rate at which HBM delivers bf16 logits,
// so a fraction of the exponentials is evaluated here instead.
// Minimax (relative) polynomials with p(0) = 1 exactly: max rel. error 1.0e-4 (deg 3),
// 2.9e-6 (deg 4).  x is clamped at -125 (result 2^-125 instead of a denormal/zero).
__device__ __forceinline__ float ex2_poly3(float x) {
  x = fmaxf(x, -125.f);
  const float t = x + 12582912.f;  // 1.5 * 2^23: rounds x to the nearest integer j
  const float f = x - (t - 12582912.f);
  const float p = fmaf(fmaf(fmaf(5.500872061e-02f, f, 2.422104627e-01f), f, 6.932829022e-01f), f, 1.0f);
  return __int_as_float(__float_as_int(p) + (__float_as_int(t) << 23));
}
__device__ __forceinline__ float ex2_poly4(float x) {
  x = fmaxf(x, -125.f);
  const float t = x + 12582912.f;
  const float f = x - (t - 12582912.f);
  const float p = fmaf(fmaf(fmaf(fmaf(9.582830593e-03f, f, 5.590637028e-02f), f, 2.402409911e-01f), f,
                            6.931241751e-01f), f, 1.0f);
  return __int_as_float(__float_as_int(p) + (__float_as_int(t) << 23));
}
// ---- packed fp32x2 arithmetic (Blackwell FFMA2 / FADD2: two lanes of fp32 per instruction)
typedef unsigned long long f32x2;
__device__ __forceinline__ f32x2 pk2(float a, float b) {
  f32x2 r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ void upk2(f32x2 v, float& a, float& b) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
}
__device__ __forceinline__ f32x2 ffma2(f32x2 a, f32x2 b, f32x2 c) {
  f32x2 r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
__device__ __forceinline__ f32x2 fadd2(f32x2 a, f32x2 b) {
  f32x2 r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ f32x2 fmul2(f32x2 a, f32x2 b) {
  f32x2 r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ float fmax_nan(float a, float b) {
  float d;
  asm("max.NaN.f32 %0, %1, %2;" : "=f"(d) : "f"(a), "f"(b));
  return d;
}
__device__ __forceinline__ uint32_t bmax2_nan(uint32_t a, uint32_t b) {
  uint32_t d;
  asm("max.NaN.bf16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
  return d;
}
__device__ __forceinline__ float bf_lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf_hi(uint32_t w) { return __uint_as_float(w & 0xFFFF0000u); }

__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
// a fraction of the lines (address-selected) evict_last, the rest evict_first (experiment:
// keep a fixed share of every forward row resident for its backward re-read)
__device__ __forceinline__ uint64_t policy_evict_last_frac(float f) {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.L2::evict_first.b64 %0, %1;" : "=l"(p) : "f"(f));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}

// Load kinds for the logits stream.
enum { LD_STREAM = 0, LD_HINT = 1 };

template <int LK>
__device__ __forceinline__ uint4 ld16(const uint4* p, uint64_t pol) {
  uint4 v;
  if (LK == LD_HINT) {
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p), "l"(pol));
  } else {
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p));
  }
  return v;
}

__device__ __forceinline__ void st16_stream(uint4* p, uint4 v) {
  asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w)
               : "memory");
}

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned ld_relaxed(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned atom_add_acq_rel(unsigned* p, unsigned v) {
  unsigned old;
  asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}
__device__ __forceinline__ void fence_acq_rel_gpu() {
  asm volatile("fence.acq_rel.gpu;" ::: "memory");
}
__device__ __forceinline__ void st_release_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// ------------------------------------------------------------------ dtype traits
// DT 0 = f32 (4 per 16 B), DT 1 = bf16 (8 per 16 B)
template <int DT>
struct Traits;

template <>
struct Traits<0> {
  static constexpr int N = 4;
  static constexpr uint32_t kNegInfWord = 0xFF800000u;
  static constexpr uint32_t kSignWord = 0x80000000u;
  __device__ static __forceinline__ float vmax(const uint4& v) {
    return fmax_nan(fmax_nan(__uint_as_float(v.x), __uint_as_float(v.y)),
                    fmax_nan(__uint_as_float(v.z), __uint_as_float(v.w)));
  }
  __device__ static __forceinline__ void unpack(const uint4& v, float* f) {
    f[0] = __uint_as_float(v.x);
    f[1] = __uint_as_float(v.y);
    f[2] = __uint_as_float(v.z);
    f[3] = __uint_as_float(v.w);
  }
  __device__ static __forceinline__ uint4 pack(const float* g) {
    return make_uint4(__float_as_uint(g[0]), __float_as_uint(g[1]), __float_as_uint(g[2]),
                      __float_as_uint(g[3]));
  }
  __device__ static __forceinline__ float load1(const void* row, int64_t v) {
    return __ldg(reinterpret_cast<const float*>(row) + v);
  }
  __device__ static __forceinline__ void store1(void* row, int64_t v, float g) {
    reinterpret_cast<float*>(row)[v] = g;
  }
};

__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
  uint32_t d;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(d) : "f"(hi), "f"(lo));
  return d;
}

template <>
struct Traits<1> {
  static constexpr int N = 8;
  static constexpr uint32_t kNegInfWord = 0xFF80FF80u;
  static constexpr uint32_t kSignWord = 0x80008000u;
  // packed max over the 16-byte vector, NaN-propagating; returns a bf16x2 word
  __device__ static __forceinline__ uint32_t vmax2(const uint4& v) {
    return bmax2_nan(bmax2_nan(v.x, v.y), bmax2_nan(v.z, v.w));
  }
  __device__ static __forceinline__ float vmax(const uint4& v) {
    uint32_t w = vmax2(v);
    return fmax_nan(bf_lo(w), bf_hi(w));
  }
  __device__ static __forceinline__ void unpack(const uint4& v, float* f) {
    f[0] = bf_lo(v.x); f[1] = bf_hi(v.x);
    f[2] = bf_lo(v.y); f[3] = bf_hi(v.y);
    f[4] = bf_lo(v.z); f[5] = bf_hi(v.z);
    f[6] = bf_lo(v.w); f[7] = bf_hi(v.w);
  }
  __device__ static __forceinline__ uint4 pack(const float* g) {
    return make_uint4(pack_bf16x2(g[0], g[1]), pack_bf16x2(g[2], g[3]), pack_bf16x2(g[4], g[5]),
                      pack_bf16x2(g[6], g[7]));
  }
  __device__ static __forceinline__ float load1(const void* row, int64_t v) {
    uint16_t b = __ldg(reinterpret_cast<const unsigned short*>(row) + v);
    return __uint_as_float(static_cast<uint32_t>(b) << 16);
  }
  __device__ static __forceinline__ void store1(void* row, int64_t v, float g) {
    uint32_t w = pack_bf16x2(g, 0.f);
    reinterpret_cast<unsigned short*>(row)[v] = static_cast<unsigned short>(w & 0xFFFFu);
  }
};

// batch max over U vectors (NaN-propagating)
template <int DT>
__device__ __forceinline__ float batch_max(const uint4* v) {
  if constexpr (DT == 1) {
    uint32_t w = Traits<1>::vmax2(v[0]);
#pragma unroll
    for (int u = 1; u < kU; ++u) w = bmax2_nan(w, Traits<1>::vmax2(v[u]));
    return fmax_nan(bf_lo(w), bf_hi(w));
  } else {
    float m = Traits<0>::vmax(v[0]);
#pragma unroll
    for (int u = 1; u < kU; ++u) m = fmax_nan(m, Traits<0>::vmax(v[u]));
    return m;
  }
}

// ------------------------------------------------------------------ (m, r) state
// 1 + r = sum_v exp(invT (x_v - m)) where m = max_v x_v (raw units); exp2 with k2 = invT*log2e.
struct MR {
  float m, r;
};

__device__ __forceinline__ MR mr_merge(MR a, MR b, float k2) {
  MR big = a, sm = b;
  if (b.m > a.m) { big = b; sm = a; }
  if (sm.m == -INFINITY) return big;
  big.r = big.r + (1.f + sm.r) * ex2((sm.m - big.m) * k2);
  return big;
}

// exp2 argument of the forward, invT (x - m) log2e.  fp32 inputs form it as (x - m) k2: the
// single-FFMA form x k2 - fl(m k2) carries the rounding of m k2 (ulp(m k2)/2, i.e. 4e-5
// relative on every term at |m| ~ 1000), above the fp32 contract of 1e-5.
// bf16 inputs keep the FFMA form (its error is far inside the 2e-3 bf16 contract).
template <int DT>
__device__ __forceinline__ float fwd_arg(float x, float k2, float m) {
  if constexpr (DT == 0) return (x - m) * k2;
  else return fmaf(x, k2, -(m * k2));
}

// Backward exponent: |g_v| = 2^(e_v) with e_v = (x_v - m) k2 - c (fp32 inputs) or
// e_v = x_v k2 - c (bf16 inputs, c then also holds m k2), c = log1p(r) log2e - log2|coef|.
template <int DT>
__device__ __forceinline__ float bwd_const(float m, float l1p, float k2, float coef) {
  if constexpr (DT == 0) return fmaf(l1p, kLog2e, -log2f(fabsf(coef)));
  else return fmaf(l1p, kLog2e, m * k2) - log2f(fabsf(coef));
}
template <int DT>
__device__ __forceinline__ float bwd_arg(float x, float k2, float c, float m) {
  if constexpr (DT == 0) return fmaf(x - m, k2, -c);
  else return fmaf(x, k2, -c);
}

// Per-thread online pass over this thread's vectors of one row.
// Vectors i = tid, tid + NT, ... (coalesced across the CTA), kU of them per batch.
template <int DT, int LK>
__device__ __forceinline__ MR row_fwd_thread(const uint4* __restrict__ vrow, int nvec, float k2,
                                             uint64_t pol) {
  constexpr int N = Traits<DT>::N;
  const uint32_t NI = Traits<DT>::kNegInfWord;
  float m = -INFINITY, r = 0.f;
  for (int base = threadIdx.x; base < nvec; base += kRowThreads * kU) {
    uint4 v[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int i = base + u * kRowThreads;
      v[u] = (i < nvec) ? ld16<LK>(vrow + i, pol) : make_uint4(NI, NI, NI, NI);
    }
    const float mc = batch_max<DT>(v);
    if (mc == -INFINITY && m == -INFINITY) continue;  // all -inf so far: no contribution
    if (!(mc <= m)) {
      // new running max (or NaN): demote the old max into r, then add this batch
      // excluding exactly ONE element equal to the new max (it is the "1" of 1 + r).
      const float sc = (m == -INFINITY) ? 0.f : ex2((m - mc) * k2);
      r = (1.f + r) * sc;
      m = mc;
      float s = 0.f;
      int neq = 0;
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        float f[N];
        Traits<DT>::unpack(v[u], f);
#pragma unroll
        for (int j = 0; j < N; ++j) {
          if (f[j] == m) ++neq;
          else s += ex2(fwd_arg<DT>(f[j], k2, m));
        }
      }
      r += s + (float)(neq - 1);
    } else {
      float s0 = 0.f, s1 = 0.f;
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        float f[N];
        Traits<DT>::unpack(v[u], f);
#pragma unroll
        for (int j = 0; j < N; j += 2) {
          s0 += ex2(fwd_arg<DT>(f[j], k2, m));
          s1 += ex2(fwd_arg<DT>(f[j + 1], k2, m));
        }
      }
      r += s0 + s1;
    }
  }
  return MR{m, r};
}

// scalar tail element (V not a multiple of the vector width): same update rules
__device__ __forceinline__ MR mr_push1(MR s, float y, float k2) {
  if (y == -INFINITY) return s;  // a zero-probability entry (R14)
  if (!(y <= s.m)) {
    const float sc = (s.m == -INFINITY) ? 0.f : ex2((s.m - y) * k2);
    s.r = (1.f + s.r) * sc;
    s.m = y;
  } else {
    s.r += ex2((y - s.m) * k2);
  }
  return s;
}

// Fixed-order CTA merge; result valid in thread 0.  smem: 2*kWarps floats.
__device__ __forceinline__ MR block_merge(MR v, float k2, float* sm) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    MR o;
    o.m = __shfl_down_sync(kFull, v.m, off);
    o.r = __shfl_down_sync(kFull, v.r, off);
    v = mr_merge(v, o, k2);
  }
  if (lane == 0) {
    sm[warp] = v.m;
    sm[kWarps + warp] = v.r;
  }
  __syncthreads();
  if (warp == 0) {
    v.m = lane < kWarps ? sm[lane] : -INFINITY;
    v.r = lane < kWarps ? sm[kWarps + lane] : 0.f;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      MR o;
      o.m = __shfl_down_sync(kFull, v.m, off);
      o.r = __shfl_down_sync(kFull, v.r, off);
      v = mr_merge(v, o, k2);
    }
  }
  return v;
}

struct RowOut {
  float m, l1p, logp, lse;
  uint32_t flags;
};

// Whole-CTA row forward; result valid in thread 0 (others get garbage).
// row: element pointer of logits[b, t, 0]; V elements; tok: sampled token.
template <int DT, int LK>
__device__ __forceinline__ RowOut row_forward(const void* row, int V, int tok, float invT,
                                              uint64_t pol, float* sm) {
  constexpr int N = Traits<DT>::N;
  const float k2 = invT * kLog2e;
  const int nvec = V / N;
  MR s = row_fwd_thread<DT, LK>(reinterpret_cast<const uint4*>(row), nvec, k2, pol);
  const int tail = V - nvec * N;
  if ((int)threadIdx.x < tail) s = mr_push1(s, Traits<DT>::load1(row, (int64_t)nvec * N + threadIdx.x), k2);
  s = block_merge(s, k2, sm);
  RowOut o;
  o.flags = 0;
  o.m = s.m;
  o.l1p = log1pf(s.r);
  o.lse = __fadd_rn(__fmul_rn(s.m, invT), o.l1p);
  if (threadIdx.x == 0) {
    if (tok < 0 || tok >= V) {
      o.flags |= ODPO_FLAG_TOKEN_RANGE;
      o.logp = 0.f;
    } else {
      const float xt = Traits<DT>::load1(row, tok);
      o.logp = __fsub_rn(__fmul_rn(__fsub_rn(xt, s.m), invT), o.l1p);
      if (!isfinite(o.logp)) o.flags |= ODPO_FLAG_NONFINITE_LOGIT;
    }
    if (!isfinite(s.m) || !isfinite(s.r)) o.flags |= ODPO_FLAG_NONFINITE_LOGIT;
  }
  return o;
}

// One 16-byte vector of the backward: |g_v| = 2^(bwd_arg) (see bwd_const), so coef rides in
// the exponent and its sign is applied to the packed result.  NPB of
// each 8 use the FMA-pipe exp2.
template <int DT, int NPB, bool NEG>
__device__ __forceinline__ uint4 bwd_vec(const uint4& v, float k2, float c, float m) {
  constexpr int N = Traits<DT>::N;
  float f[N];
  Traits<DT>::unpack(v, f);
  const f32x2 K2 = pk2(k2, k2), NC = pk2(-c, -c), NM = pk2(-m, -m);
#pragma unroll
  for (int j = 0; j < N; j += 2) {
    float e0, e1;   // two exp2 arguments per FFMA2 (fp32: x - m first, see bwd_const)
    if constexpr (DT == 0) upk2(ffma2(fadd2(pk2(f[j], f[j + 1]), NM), K2, NC), e0, e1);
    else upk2(ffma2(pk2(f[j], f[j + 1]), K2, NC), e0, e1);
    f[j] = j < NPB ? ex2_poly3(e0) : ex2(e0);
    f[j + 1] = j + 1 < NPB ? ex2_poly3(e1) : ex2(e1);
  }
  uint4 o = Traits<DT>::pack(f);
  if (NEG) {  // sign of coef applied to the packed words (one LOP per 32-bit word)
    o.x ^= Traits<DT>::kSignWord; o.y ^= Traits<DT>::kSignWord;
    o.z ^= Traits<DT>::kSignWord; o.w ^= Traits<DT>::kSignWord;
  }
  return o;
}

// Whole-CTA row backward: drow[v] = coef * (exp(invT (x_v - m) - l1p) - [v == tok]).
// tok entry written as coef * expm1(logp) (no p - 1 cancellation).
template <int DT, int LK, int NPB>
__device__ __forceinline__ void row_backward(const void* row, void* drow, int V, int tok,
                                             float invT, float m, float l1p, float logp,
                                             float coef, uint64_t pol) {
  constexpr int N = Traits<DT>::N;
  const float k2 = invT * kLog2e;
  const float c = bwd_const<DT>(m, l1p, k2, coef);
  const bool neg = coef < 0.f;
  const int nvec = V / N;
  const uint4* vrow = reinterpret_cast<const uint4*>(row);
  uint4* vout = reinterpret_cast<uint4*>(drow);
  for (int base = threadIdx.x; base < nvec; base += kRowThreads * kU) {
    uint4 v[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int i = base + u * kRowThreads;
      if (i < nvec) v[u] = ld16<LK>(vrow + i, pol);
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int i = base + u * kRowThreads;
      if (i < nvec)
        st16_stream(vout + i, neg ? bwd_vec<DT, NPB, true>(v[u], k2, c, m) : bwd_vec<DT, NPB, false>(v[u], k2, c, m));
    }
  }
  const float gtok = coef * expm1f(logp);
  const int tail = V - nvec * N;
  if ((int)threadIdx.x < tail) {
    const int64_t v = (int64_t)nvec * N + threadIdx.x;
    const float x = Traits<DT>::load1(row, v);
    Traits<DT>::store1(drow, v, (v == tok) ? gtok : copysignf(ex2(bwd_arg<DT>(x, k2, c, m)), coef));
  }
  // onehot entry: written by the thread that stored tok's vector (program order)
  if (tok >= 0 && tok < nvec * N && (tok / N) % kRowThreads == (int)threadIdx.x)
    Traits<DT>::store1(drow, tok, gtok);
}

template <int DT>
__device__ __forceinline__ void row_zero(void* drow, int V) {
  constexpr int N = Traits<DT>::N;
  const int nvec = V / N;
  uint4* vout = reinterpret_cast<uint4*>(drow);
  for (int i = threadIdx.x; i < nvec; i += kRowThreads) st16_stream(vout + i, make_uint4(0, 0, 0, 0));
  const int tail = V - nvec * N;
  if ((int)threadIdx.x < tail) Traits<DT>::store1(drow, (int64_t)nvec * N + threadIdx.x, 0.f);
}

// Fixed-order masked sum of one sequence's per-token log-probs, by ONE warp.
// lane l sums t = l, l+32, ... in order (double), then a shfl_down tree.  Valid in lane 0.
__device__ __forceinline__ void seq_sum_warp(const float* row_logp, const uint8_t* mask, int64_t T,
                                             double& S, int& n) {
  const int lane = threadIdx.x & 31;
  double s = 0.0;
  int c = 0;
  for (int64_t t = lane; t < T; t += 32) {
    if (__ldcg(mask + t)) {
      s += (double)__ldcg(row_logp + t);
      ++c;
    }
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    s += __shfl_down_sync(kFull, s, off);
    c += __shfl_down_sync(kFull, c, off);
  }
  S = s;
  n = c;
}

// Both sequences of a pair at once (the pair reduction): per sequence exactly seq_sum_warp's
// order (lane l sums t = l, l+32, ... in order, then the same shfl_down tree), with the two
// sequences' loads interleaved so their latencies overlap.  c < 0 / r < 0: that sum is 0.
__device__ __forceinline__ void seq_sum2_warp(const float* lp_c, const uint8_t* mk_c,
                                              const float* lp_r, const uint8_t* mk_r, int64_t T,
                                              double& Sc, int& nc, double& Sr, int& nr) {
  const int lane = threadIdx.x & 31;
  double sc = 0.0, sr = 0.0;
  int cc = 0, cr = 0;
#pragma unroll 2
  for (int64_t t = lane; t < T; t += 32) {
    // both masks, then both (written) log-probs: two overlapped round trips, and masked rows'
    // log-probs (never written) are never read
    const uint8_t mc = lp_c ? __ldcg(mk_c + t) : (uint8_t)0;
    const uint8_t mr = lp_r ? __ldcg(mk_r + t) : (uint8_t)0;
    const float vc = mc ? __ldcg(lp_c + t) : 0.f;
    const float vr = mr ? __ldcg(lp_r + t) : 0.f;
    if (mc) { sc += (double)vc; ++cc; }
    if (mr) { sr += (double)vr; ++cr; }
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    sc += __shfl_down_sync(kFull, sc, off);
    cc += __shfl_down_sync(kFull, cc, off);
    sr += __shfl_down_sync(kFull, sr, off);
    cr += __shfl_down_sync(kFull, cr, off);
  }
  Sc = sc; nc = cc; Sr = sr; nr = cr;
}

}  // namespace odpo
