// Host cost of kernel launches by parameter size (B200, driver 580): an
// empty kernel taking a by-value struct of 64 B ... 24 KB, cooperative vs
// plain launch, cudaMemsetAsync and cudaOccupancy queries.  nvcc -O2 -o
// mb_launch tools/mb_launch.cu -gencode arch=compute_100a,code=sm_100a
#include <chrono>
#include <cstdio>
#include <cuda_runtime.h>

template <int B>
struct P { int v[B / 4]; };

template <int B>
__global__ void k(P<B> p, int* out) {
  if (threadIdx.x == 0 && blockIdx.x == 0 && p.v[0] == 12345) out[0] = p.v[B / 4 - 1];
}

template <int B>
double time_launch(cudaStream_t st, int* out, int reps, bool coop) {
  P<B> p = {};
  for (int i = 0; i < 100; ++i) k<B><<<148, 256, 0, st>>>(p, out);
  cudaStreamSynchronize(st);
  auto t0 = std::chrono::high_resolution_clock::now();
  for (int i = 0; i < reps; ++i) {
    if (coop) {
      void* args[] = {(void*)&p, (void*)&out};
      cudaLaunchCooperativeKernel((const void*)k<B>, dim3(148), dim3(256), args, 0, st);
    } else {
      k<B><<<148, 256, 0, st>>>(p, out);
    }
  }
  auto t1 = std::chrono::high_resolution_clock::now();
  cudaStreamSynchronize(st);
  return std::chrono::duration<double, std::micro>(t1 - t0).count() / reps;
}

int main() {
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  int* out;
  cudaMalloc(&out, 64);
  const int reps = 2000;
  printf("param bytes, plain launch us, cooperative launch us\n");
  printf("%6d %8.2f %8.2f\n", 64, time_launch<64>(st, out, reps, false), time_launch<64>(st, out, reps, true));
  printf("%6d %8.2f %8.2f\n", 1024, time_launch<1024>(st, out, reps, false), time_launch<1024>(st, out, reps, true));
  printf("%6d %8.2f %8.2f\n", 4096, time_launch<4096>(st, out, reps, false), time_launch<4096>(st, out, reps, true));
  printf("%6d %8.2f %8.2f\n", 8192, time_launch<8192>(st, out, reps, false), time_launch<8192>(st, out, reps, true));
  printf("%6d %8.2f %8.2f\n", 16384, time_launch<16384>(st, out, reps, false), time_launch<16384>(st, out, reps, true));
  printf("%6d %8.2f %8.2f\n", 24576, time_launch<24576>(st, out, reps, false), time_launch<24576>(st, out, reps, true));
  auto t0 = std::chrono::high_resolution_clock::now();
  for (int i = 0; i < reps; ++i) cudaMemsetAsync(out, 0, 8, st);
  auto t1 = std::chrono::high_resolution_clock::now();
  cudaStreamSynchronize(st);
  printf("cudaMemsetAsync 8 B: %.2f us\n", std::chrono::duration<double, std::micro>(t1 - t0).count() / reps);
  int per = 0;
  t0 = std::chrono::high_resolution_clock::now();
  for (int i = 0; i < reps; ++i) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, (const void*)k<64>, 256, 0);
  t1 = std::chrono::high_resolution_clock::now();
  printf("cudaOccupancyMaxActiveBlocksPerMultiprocessor: %.2f us\n",
         std::chrono::duration<double, std::micro>(t1 - t0).count() / reps);
  int dev = 0, v = 0;
  t0 = std::chrono::high_resolution_clock::now();
  for (int i = 0; i < reps; ++i) { cudaGetDevice(&dev); cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev); }
  t1 = std::chrono::high_resolution_clock::now();
  printf("cudaGetDevice + cudaDeviceGetAttribute: %.2f us\n", std::chrono::duration<double, std::micro>(t1 - t0).count() / reps);
  cudaEvent_t e;
  cudaEventCreate(&e);
  t0 = std::chrono::high_resolution_clock::now();
  for (int i = 0; i < reps; ++i) cudaEventRecord(e, st);
  t1 = std::chrono::high_resolution_clock::now();
  printf("cudaEventRecord: %.2f us\n", std::chrono::duration<double, std::micro>(t1 - t0).count() / reps);
  return 0;
}
