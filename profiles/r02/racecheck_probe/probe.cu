// racecheck probe: the canonical single-producer TMA ring in its simplest form -- one thread
// issues cp.async.bulk (1-D TMA) into a shared-memory stage with mbarrier complete_tx, the
// consumers wait on that mbarrier's phase, read the stage, and release it on a second
// mbarrier before the producer refills it.  This is correct by the PTX memory model (the
// mbarrier phase completion orders the async copy's writes before the waiters' reads), and it
// is exactly the pattern libodpo's engine uses.  If compute-sanitizer --tool racecheck reports
// hazards on THIS program, its reports on the engine's ring are the same false positive.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void ring(const uint4* __restrict__ src, int nchunks, unsigned* out) {
  constexpr int STAGES = 2, VEC = 1024;   // 16 KB stages
  extern __shared__ __align__(128) uint4 buf[];
  __shared__ __align__(8) uint64_t full[STAGES], empty[STAGES];
  const int tid = threadIdx.x;
  const int ncons = blockDim.x - 32;
  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&full[s])), "r"(1));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&empty[s])), "r"(ncons / 32));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto wait = [](uint32_t b, uint32_t ph) {
    asm volatile("{\n\t.reg .pred p;\nW%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W%=;\n}"
                 ::"r"(b), "r"(ph) : "memory");
  };
  if (tid >= ncons) {
    if (tid == ncons) {   // producer
      for (int c = 0; c < nchunks; ++c) {
        const int s = c % STAGES;
        const uint32_t ph = (c / STAGES) & 1;
        wait(su32(&empty[s]), ph ^ 1u);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[s])), "r"(VEC * 16) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(su32(buf + s * VEC)), "l"(src + (size_t)c * VEC), "r"(VEC * 16), "r"(su32(&full[s])) : "memory");
      }
    }
    return;
  }
  unsigned acc = 0;
  for (int c = 0; c < nchunks; ++c) {
    const int s = c % STAGES;
    wait(su32(&full[s]), (c / STAGES) & 1);
    for (int i = tid; i < VEC; i += ncons) acc ^= buf[s * VEC + i].x;
    __syncwarp();
    if ((tid & 31) == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&empty[s])) : "memory");
  }
  atomicXor(out, acc);
}

int main() {
  const int nchunks = 64, VEC = 1024;
  uint4* src;
  unsigned* out;
  cudaMalloc(&src, (size_t)nchunks * VEC * 16);
  cudaMemset(src, 1, (size_t)nchunks * VEC * 16);
  cudaMalloc(&out, 4);
  cudaMemset(out, 0, 4);
  cudaFuncSetAttribute(ring, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * VEC * 16);
  ring<<<1, 160, 2 * VEC * 16>>>(src, nchunks, out);
  unsigned h = 0;
  cudaMemcpy(&h, out, 4, cudaMemcpyDeviceToHost);
  printf("probe done: %s xor=%08x\n", cudaGetErrorString(cudaGetLastError()), h);
  return 0;
}
