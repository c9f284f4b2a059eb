// Microbenchmark (tool, not product): throughput of random 32-bit atomicOr
// into an L2-resident bitmap (the alias-histogram kernel's access pattern),
// and of random 4-byte loads from it (the mask kernel's).
#include <cuda_runtime.h>
#include <cstdint>

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16;
  return x;
}

__global__ void __launch_bounds__(256) atom_kernel(uint32_t* bits, uint32_t words, int per_thread, int mode,
                                                   uint32_t* sink) {
  const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
  uint32_t acc = 0;
  for (int i = 0; i < per_thread; ++i) {
    const uint32_t h = hash32(tid * 131u + i * 7919u);
    const uint32_t w = h % words;
    if (mode == 0) acc |= atomicOr(&bits[w], 1u << (h >> 27));
    else acc |= __ldg(&bits[w]);
  }
  if (acc == 0x12345678u) sink[0] = acc;
}

extern "C" int mb_atom(uint32_t* bits, uint32_t words, int blocks, int per_thread, int mode, uint32_t* sink,
                       void* st) {
  atom_kernel<<<blocks, 256, 0, (cudaStream_t)st>>>(bits, words, per_thread, mode, sink);
  return (int)cudaGetLastError();
}
