// Random-access throughput probe: N random indices into a table of M entries.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <random>
#include <cuda_runtime.h>
__global__ void k_load32(const uint32_t* __restrict__ idx, const uint32_t* __restrict__ t, uint32_t n, uint32_t* out) {
  uint32_t acc = 0;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) acc += __ldg(t + __ldg(idx + i));
  if (acc == 0x12345) out[0] = acc;
}
__global__ void k_atom64(const uint32_t* __restrict__ idx, unsigned long long* t, uint32_t n, uint32_t* out) {
  unsigned long long acc = 0;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) acc += atomicMin(t + __ldg(idx + i), (unsigned long long)i);
  if (acc == 0x12345) out[0] = (uint32_t)acc;
}
__global__ void k_atom32(const uint32_t* __restrict__ idx, uint32_t* t, uint32_t n, uint32_t* out) {
  uint32_t acc = 0;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) acc += atomicMin(t + __ldg(idx + i), i);
  if (acc == 0x12345) out[0] = acc;
}
__global__ void k_red64(const uint32_t* __restrict__ idx, unsigned long long* t, uint32_t n, uint32_t* out) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) atomicMin(t + __ldg(idx + i), (unsigned long long)i);
}
int main() {
  const uint32_t n = 6u << 20;
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (uint32_t M : {100000u, 1000000u, 8000000u, 32000000u}) {
    std::vector<uint32_t> h(n); std::mt19937 r(1); for (auto& x : h) x = r() % M;
    uint32_t *idx, *t32, *out; unsigned long long* t64;
    cudaMalloc(&idx, n * 4); cudaMalloc(&t32, (size_t)M * 4); cudaMalloc(&t64, (size_t)M * 8); cudaMalloc(&out, 4);
    cudaMemcpy(idx, h.data(), n * 4, cudaMemcpyHostToDevice);
    cudaMemset(t32, 0xff, (size_t)M * 4); cudaMemset(t64, 0xff, (size_t)M * 8);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int kind = 0; kind < 4; ++kind) for (int bs : {512, 1024}) {
      int grid = sms * (2048 / bs);
      float best = 1e9;
      for (int rep = 0; rep < 5; ++rep) {
        cudaEventRecord(a);
        if (kind == 0) k_load32<<<grid, bs>>>(idx, t32, n, out);
        if (kind == 1) k_atom64<<<grid, bs>>>(idx, t64, n, out);
        if (kind == 2) k_atom32<<<grid, bs>>>(idx, t32, n, out);
        if (kind == 3) k_red64<<<grid, bs>>>(idx, t64, n, out);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms;
      }
      const char* nm[] = {"load32", "atomicMin64(ret)", "atomicMin32(ret)", "atomicMin64(noret)"};
      printf("M=%9u %-20s bs=%4d: %7.1f us  %6.2f G/s\n", M, nm[kind], bs, best * 1e3, n / (best * 1e6));
    }
    cudaFree(idx); cudaFree(t32); cudaFree(t64); cudaFree(out);
  }
}
