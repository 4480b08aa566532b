// synth.cu -- device twin of synth/__init__.py's counter-hash logits generator.
//
// Holds none of the method's arithmetic: it only writes x[g, v] = int8(h & 0xff) / 64 with
// h = splitmix64(idx ^ splitmix64(seed*256 + stream)), idx = g*V + v over GLOBAL row g,
// and optionally the "peaked" sampled-token logit x[g, tok[g]] = peak.  Used by tests and
// bench.py to build multi-GB inputs on the device without a host copy; the host twin
// (numpy) regenerates any sampled rows bit-identically for the oracle.
#include <cuda_runtime.h>
#include <stdint.h>

__host__ __device__ static inline uint64_t splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

template <int DT>
__global__ void fill_logits(char* out, int64_t T, int64_t V, int64_t sb, int64_t st, uint64_t key,
                            int64_t row0, const int32_t* tokens, float peak, int use_peak) {
  const int64_t g = blockIdx.x;  // local row
  const int64_t b = g / T, t = g % T;
  const int esize = DT == 0 ? 4 : 2;
  char* row = out + (b * sb + t * st) * esize;
  const uint64_t gg = (uint64_t)(row0 + g);
  int tok = -1;
  if (use_peak && tokens) tok = tokens[g];
  for (int64_t v = threadIdx.x; v < V; v += blockDim.x) {
    const uint64_t h = splitmix64((gg * (uint64_t)V + (uint64_t)v) ^ key);
    float x = (float)(int8_t)(uint8_t)(h & 0xFF) / 64.0f;
    if (v == tok) x = peak;
    if (DT == 0) {
      reinterpret_cast<float*>(row)[v] = x;
    } else {
      // exact: values are on a 1/64 grid with |x| < 2^8 (or the bf16-exact peak)
      reinterpret_cast<uint16_t*>(row)[v] = (uint16_t)(__float_as_uint(x) >> 16);
    }
  }
}

extern "C" {

uint64_t synth_stream_key(uint64_t seed, int stream) { return splitmix64(seed * 256ull + (uint64_t)stream); }

// dtype 0 = f32, 1 = bf16.  rows [0, B*T) of a [B,T,V] tensor with element strides (sb, st);
// global row index = row0 + b*T + t.  tokens: device [B*T] or NULL.
int synth_fill_logits(void* out, int dtype, int64_t B, int64_t T, int64_t V, int64_t sb, int64_t st,
                      uint64_t seed, int stream, int64_t row0, const int32_t* tokens, float peak,
                      int use_peak, void* cuda_stream) {
  if (!out || B <= 0 || T <= 0 || V <= 0) return 1;
  const uint64_t key = synth_stream_key(seed, stream);
  const unsigned rows = (unsigned)(B * T);
  cudaStream_t s = (cudaStream_t)cuda_stream;
  if (dtype == 0)
    fill_logits<0><<<rows, 256, 0, s>>>((char*)out, T, V, sb, st, key, row0, tokens, peak, use_peak);
  else
    fill_logits<1><<<rows, 256, 0, s>>>((char*)out, T, V, sb, st, key, row0, tokens, peak, use_peak);
  return cudaGetLastError() == cudaSuccess ? 0 : 2;
}

}  // extern "C"
