// Microbenchmark: shared-memory histogram update rates on sm_100a (design input for fit_hist).
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/ub tools/ubench_smem_atomics.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int MODE>
__global__ void k(const uint32_t* __restrict__ keys, int n_iter, unsigned long long* out) {
  __shared__ uint32_t h32[4][1024];
  __shared__ unsigned long long h64[4][257];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 4 * 1024; i += blockDim.x) (&h32[0][0])[i] = 0;
  for (int i = threadIdx.x; i < 4 * 257; i += blockDim.x) (&h64[0][0])[i] = 0;
  __syncthreads();
  uint32_t key = keys[(blockIdx.x * blockDim.x + threadIdx.x) & 4095];
  uint32_t acc = 0;
  for (int it = 0; it < n_iter; ++it) {
    uint32_t b = (key + it * 2654435761u) >> 24;  // pseudo-random bin 0..255
    if (MODE == 0) atomicAdd(&h32[w][b], 1u);                          // 1x u32 random bins
    if (MODE == 1) { atomicAdd(&h32[w][b], 1u); atomicAdd(&h32[w][256 + b], b); }  // 2x u32
    if (MODE == 2) atomicAdd(&h64[w][b], 1ull + ((unsigned long long)b << 44));     // u64 (CAS)
    if (MODE == 3) atomicAdd(&h32[w][0], 1u);                           // all lanes same bin
    if (MODE == 4) atomicAdd(&h32[w][lane * 32 + (b & 31)], 1u);         // lane-private region
    if (MODE == 5) { uint32_t x = h32[w][b]; acc += x; }                  // plain LDS (reference)
  }
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = h32[0][1] + h64[0][1] + acc;
}

template <int MODE>
float run(const uint32_t* keys, unsigned long long* out, int blocks, int iters) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  k<MODE><<<blocks, 128>>>(keys, iters, out);
  cudaEventRecord(a);
  k<MODE><<<blocks, 128>>>(keys, iters, out);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms;
}

int main() {
  uint32_t* keys;
  unsigned long long* out;
  cudaMalloc(&keys, 4096 * 4);
  cudaMalloc(&out, 1 << 20);
  uint32_t h[4096];
  for (int i = 0; i < 4096; ++i) h[i] = i * 2246822519u;
  cudaMemcpy(keys, h, sizeof h, cudaMemcpyHostToDevice);
  int dev;
  cudaGetDevice(&dev);
  int sms, clk;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  const int blocks = sms * 8, iters = 4096;
  const double ops = (double)blocks * 128 * iters;
  const char* names[] = {"u32 random bins", "2x u32 random bins", "u64 packed (CAS loop)",
                         "u32 same bin (32-way)", "u32 lane-private", "plain LDS"};
  float t[6] = {run<0>(keys, out, blocks, iters), run<1>(keys, out, blocks, iters),
                run<2>(keys, out, blocks, iters), run<3>(keys, out, blocks, iters),
                run<4>(keys, out, blocks, iters), run<5>(keys, out, blocks, iters)};
  for (int m = 0; m < 6; ++m) {
    double per_s = ops / (t[m] * 1e-3);
    printf("%-24s %8.3f ms  %.3e lane-updates/s  %.2f lane-updates/clk/SM (at %d MHz)\n", names[m],
           t[m], per_s, per_s / sms / (clk * 1e3), clk / 1000);
  }
  return 0;
}
