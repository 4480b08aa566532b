// copy_bw.cu -- HBM copy-pattern microbenchmark (B200, sm_100a).  Question: is the torch
// b.copy_ figure (MEASURED_PEAKS.json hbm_gbs) the ceiling for the scaled backward's
// read-a-row / write-a-row traffic, or does another load/store pattern move R+W bytes faster?
// Variants (all move the same N bytes in and N bytes out, L2 far smaller than N):
//   grid  : grid-stride 16-byte LDG/STG, U vectors in flight per thread
//   row   : one CTA per 256 KB "row" (k_row_bwd's shape), U vectors per thread per batch
//   tma   : persistent CTAs, 1-D bulk TMA global->smem ring, bulk TMA smem->global stores
//   read  : read-only stream (reference)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o copy_bw copy_bw.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

template <int ST>
__device__ __forceinline__ void st16(uint4* p, uint4 v) {
  if (ST == 0) asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" :: "l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
  else if (ST == 1) asm volatile("st.global.v4.u32 [%0], {%1,%2,%3,%4};" :: "l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
  else asm volatile("st.global.L1::no_allocate.v4.u32 [%0], {%1,%2,%3,%4};" :: "l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}
__device__ __forceinline__ uint4 ld16(const uint4* p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  return v;
}
__device__ __forceinline__ uint4 xf(uint4 v) { v.x ^= 0x1u; return v; }

template <int U, int ST>
__global__ void __launch_bounds__(512) k_grid(const uint4* __restrict__ in, uint4* __restrict__ out, int64_t n) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; base < n; base += stride * U) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) if (base + u * stride < n) v[u] = ld16(in + base + u * stride);
#pragma unroll
    for (int u = 0; u < U; ++u) if (base + u * stride < n) st16<ST>(out + base + u * stride, xf(v[u]));
  }
}

template <int U, int ST>
__global__ void __launch_bounds__(512, 2) k_row(const uint4* __restrict__ in, uint4* __restrict__ out, int64_t nvec_row) {
  const uint4* r = in + (int64_t)blockIdx.x * nvec_row;
  uint4* o = out + (int64_t)blockIdx.x * nvec_row;
  for (int64_t base = threadIdx.x; base < nvec_row; base += 512 * U) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) if (base + 512 * u < nvec_row) v[u] = ld16(r + base + 512 * u);
#pragma unroll
    for (int u = 0; u < U; ++u) if (base + 512 * u < nvec_row) st16<ST>(o + base + 512 * u, xf(v[u]));
  }
}

// 32-byte vectors (sm_100: ld/st .v8.b32)
struct u8v { uint32_t x[8]; };
__device__ __forceinline__ u8v ld32(const u8v* p) {
  u8v v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::evict_first.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(v.x[0]), "=r"(v.x[1]), "=r"(v.x[2]), "=r"(v.x[3]), "=r"(v.x[4]), "=r"(v.x[5]), "=r"(v.x[6]), "=r"(v.x[7]) : "l"(p));
  return v;
}
__device__ __forceinline__ void st32(u8v* p, u8v v) {
  asm volatile("st.global.L1::no_allocate.L2::evict_first.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" :: "l"(p),
               "r"(v.x[0]), "r"(v.x[1]), "r"(v.x[2]), "r"(v.x[3]), "r"(v.x[4]), "r"(v.x[5]), "r"(v.x[6]), "r"(v.x[7]) : "memory");
}
template <int U>
__global__ void __launch_bounds__(512, 2) k_row32(const u8v* __restrict__ in, u8v* __restrict__ out, int64_t n_row) {
  const u8v* r = in + (int64_t)blockIdx.x * n_row;
  u8v* o = out + (int64_t)blockIdx.x * n_row;
  for (int64_t base = threadIdx.x; base < n_row; base += 512 * U) {
    u8v v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) if (base + 512 * u < n_row) v[u] = ld32(r + base + 512 * u);
#pragma unroll
    for (int u = 0; u < U; ++u) if (base + 512 * u < n_row) { v[u].x[0] ^= 1u; st32(o + base + 512 * u, v[u]); }
  }
}

template <int THR, int U, bool W32, int MINB>
__global__ void __launch_bounds__(THR, MINB) k_chunk(const char* __restrict__ in, char* __restrict__ out, int64_t chunk) {
  const char* r = in + (int64_t)blockIdx.x * chunk;
  char* o = out + (int64_t)blockIdx.x * chunk;
  if (W32) {
    const int64_t n = chunk / 32;
    const u8v* ri = reinterpret_cast<const u8v*>(r); u8v* oi = reinterpret_cast<u8v*>(o);
    for (int64_t base = threadIdx.x; base < n; base += THR * U) {
      u8v v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) if (base + THR * u < n) v[u] = ld32(ri + base + THR * u);
#pragma unroll
      for (int u = 0; u < U; ++u) if (base + THR * u < n) { v[u].x[0] ^= 1u; st32(oi + base + THR * u, v[u]); }
    }
  } else {
    const int64_t n = chunk / 16;
    const uint4* ri = reinterpret_cast<const uint4*>(r); uint4* oi = reinterpret_cast<uint4*>(o);
    for (int64_t base = threadIdx.x; base < n; base += THR * U) {
      uint4 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) if (base + THR * u < n) v[u] = ld16(ri + base + THR * u);
#pragma unroll
      for (int u = 0; u < U; ++u) if (base + THR * u < n) st16<0>(oi + base + THR * u, xf(v[u]));
    }
  }
}

__global__ void __launch_bounds__(512) k_read(const uint4* __restrict__ in, int64_t n, unsigned* sink) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  unsigned acc = 0;
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; base < n; base += stride * 8) {
    uint4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) if (base + u * stride < n) v[u] = ld16(in + base + u * stride);
#pragma unroll
    for (int u = 0; u < 8; ++u) acc ^= v[u].x ^ v[u].w;
  }
  if (acc == 0x12345678u) *sink = acc;
}

// ---- bulk TMA copy: one elected thread per CTA; STAGES x CH bytes ring
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(b)), "r"(c)); }
__device__ __forceinline__ void mbar_expect(uint64_t* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned ph) {
  asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}" :: "r"(smem_u32(b)), "r"(ph) : "memory");
}
template <int STAGES, int CH>
__global__ void __launch_bounds__(32, 1) k_tma(const char* __restrict__ in, char* __restrict__ out, int64_t nbytes) {
  extern __shared__ __align__(128) char sm[];
  __shared__ uint64_t bar[STAGES];
  if (threadIdx.x != 0) return;
  for (int s = 0; s < STAGES; ++s) mbar_init(&bar[s], 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  const int64_t nch = nbytes / CH;
  int64_t mine = 0;
  for (int64_t c = blockIdx.x; c < nch; c += gridDim.x) ++mine;
  // prologue: fill
  int64_t issued = 0, done = 0;
  auto issue = [&](int64_t k) {
    const int64_t c = blockIdx.x + k * gridDim.x;
    const int s = (int)(k % STAGES);
    mbar_expect(&bar[s], CH);
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 :: "r"(smem_u32(sm + s * CH)), "l"(in + c * CH), "r"(CH), "r"(smem_u32(&bar[s])) : "memory");
  };
  for (; issued < mine && issued < STAGES; ++issued) issue(issued);
  for (; done < mine; ++done) {
    const int s = (int)(done % STAGES);
    mbar_wait(&bar[s], (unsigned)((done / STAGES) & 1));
    const int64_t c = blockIdx.x + done * gridDim.x;
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" :: "l"(out + c * CH), "r"(smem_u32(sm + s * CH)), "r"(CH) : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    if (issued < mine) {
      // the stage about to be refilled is the one stored (STAGES-1) groups ago... simplest: wait
      // until at most STAGES-1 store groups are pending reads, so the oldest stage is free
      asm volatile("cp.async.bulk.wait_group.read %0;" :: "n"(STAGES - 1) : "memory");
      issue(issued);
      ++issued;
    }
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

static float timeit(void (*f)(void*), void* ctx, int reps, float* med) {
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  std::vector<float> t;
  for (int i = 0; i < reps + 2; ++i) {
    cudaEventRecord(a);
    f(ctx);
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    float ms; cudaEventElapsedTime(&ms, a, b);
    if (i >= 2) t.push_back(ms);
  }
  std::sort(t.begin(), t.end());
  *med = t[t.size() / 2];
  return t[0];
}

struct Ctx { uint4* in; uint4* out; int64_t nvec; int grid; unsigned* sink; };
static Ctx C;

#define RUNK(name, launch)                                                               \
  {                                                                                      \
    auto fn = [](void*) { launch; };                                                     \
    float med, best = timeit(fn, nullptr, 10, &med);                                     \
    CK(cudaGetLastError());                                                              \
    printf("%-34s best %.3f ms = %7.1f GB/s   median %7.1f GB/s\n", name, best,          \
           bytes / best / 1e6, bytes / med / 1e6);                                       \
  }

int main(int argc, char** argv) {
  const int64_t N = (argc > 1 ? atoll(argv[1]) : 8LL) << 30;   // bytes in (and out)
  CK(cudaMalloc(&C.in, N)); CK(cudaMalloc(&C.out, N)); CK(cudaMalloc(&C.sink, 4));
  CK(cudaMemset(C.in, 1, N)); CK(cudaMemset(C.out, 0, N));
  C.nvec = N / 16;
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double bytes = 2.0 * N;
  printf("N = %lld bytes in + out, %d SMs\n", (long long)N, sms);
  RUNK("torch-like cudaMemcpy D2D", cudaMemcpyAsync(C.out, C.in, C.nvec * 16, cudaMemcpyDeviceToDevice));
  static int G;

  if (argc > 2) {   // chunk sweep only
    static int64_t CHB;
    for (int64_t cb : {16384LL, 32768LL, 50304LL, 65536LL, 100608LL, 131072LL, 128256LL, 256512LL}) {
      CHB = cb;
      G = (int)(N / cb);
      double sb = bytes; bytes = 2.0 * (double)G * cb;
      char nm[64];
#define CH(T, U, W, MB) snprintf(nm, 64, "chunk %6lld T%d U%d %s mb%d", (long long)cb, T, U, W ? "v8" : "v4", MB); \
      RUNK(nm, (k_chunk<T, U, W, MB><<<G, T>>>((const char*)C.in, (char*)C.out, CHB)));
      CH(512, 8, false, 2) CH(512, 4, true, 2) CH(512, 2, true, 2) CH(256, 8, false, 4) CH(256, 4, true, 4)
      CH(1024, 4, false, 1) CH(1024, 2, true, 1) CH(128, 8, false, 8) CH(128, 4, true, 8)
      bytes = sb;
    }
    return 0;
  }
  for (int mult : {2, 4, 8}) {
    G = sms * mult;
    char nm[64];
    snprintf(nm, 64, "grid U=4 cs  grid=%dx", mult); RUNK(nm, (k_grid<4, 0><<<G, 512>>>(C.in, C.out, C.nvec)));
    snprintf(nm, 64, "grid U=8 cs  grid=%dx", mult); RUNK(nm, (k_grid<8, 0><<<G, 512>>>(C.in, C.out, C.nvec)));
    snprintf(nm, 64, "grid U=8 wb  grid=%dx", mult); RUNK(nm, (k_grid<8, 1><<<G, 512>>>(C.in, C.out, C.nvec)));
    snprintf(nm, 64, "grid U=8 ef  grid=%dx", mult); RUNK(nm, (k_grid<8, 2><<<G, 512>>>(C.in, C.out, C.nvec)));
  }
  static int64_t rowv;
  for (int64_t rowbytes : {100608LL, 256512LL, 262144LL}) {
    rowv = rowbytes / 16;
    G = (int)(C.nvec / rowv);
    double sb = bytes; bytes = 2.0 * (double)G * rowbytes;
    char nm[64];
    snprintf(nm, 64, "row %lldB U=8 cs", (long long)rowbytes); RUNK(nm, (k_row<8, 0><<<G, 512>>>(C.in, C.out, rowv)));
    snprintf(nm, 64, "row %lldB U=4 cs", (long long)rowbytes); RUNK(nm, (k_row<4, 0><<<G, 512>>>(C.in, C.out, rowv)));
    snprintf(nm, 64, "row %lldB U=8 wb", (long long)rowbytes); RUNK(nm, (k_row<8, 1><<<G, 512>>>(C.in, C.out, rowv)));
    snprintf(nm, 64, "row32 %lldB U=4", (long long)rowbytes); RUNK(nm, (k_row32<4><<<G, 512>>>((const u8v*)C.in, (u8v*)C.out, rowv / 2)));
    snprintf(nm, 64, "row32 %lldB U=8", (long long)rowbytes); RUNK(nm, (k_row32<8><<<G, 512>>>((const u8v*)C.in, (u8v*)C.out, rowv / 2)));
    snprintf(nm, 64, "row %lldB U=16 cs", (long long)rowbytes); RUNK(nm, (k_row<16, 0><<<G, 512>>>(C.in, C.out, rowv)));
    bytes = sb;
  }
  for (int mult : {1, 2, 4}) {
    G = sms * mult;
    char nm[64];
    CK(cudaFuncSetAttribute(k_tma<6, 32768>, cudaFuncAttributeMaxDynamicSharedMemorySize, 6 * 32768));
    CK(cudaFuncSetAttribute(k_tma<4, 16384>, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 16384));
    CK(cudaFuncSetAttribute(k_tma<8, 16384>, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 16384));
    if (mult == 1) { snprintf(nm, 64, "tma 6x32K grid=%dx", mult); RUNK(nm, (k_tma<6, 32768><<<G, 32, 6 * 32768>>>((const char*)C.in, (char*)C.out, C.nvec * 16))); }
    snprintf(nm, 64, "tma 4x16K grid=%dx", mult); RUNK(nm, (k_tma<4, 16384><<<G, 32, 4 * 16384>>>((const char*)C.in, (char*)C.out, C.nvec * 16)));
    if (mult <= 2) { snprintf(nm, 64, "tma 8x16K grid=%dx", mult); RUNK(nm, (k_tma<8, 16384><<<G, 32, 8 * 16384>>>((const char*)C.in, (char*)C.out, C.nvec * 16))); }
  }
  bytes = (double)N;
  for (int mult : {2, 4, 8}) {
    G = sms * mult;
    char nm[64];
    snprintf(nm, 64, "read-only U=8 grid=%dx", mult); RUNK(nm, (k_read<<<G, 512>>>(C.in, C.nvec, C.sink)));
  }
  return 0;
}
