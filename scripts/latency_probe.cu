// Latency probe (developer tool): dependent-load chains on B200.
#include <cstdio>
#include <cuda_runtime.h>
extern __shared__ unsigned long long dyn[];
__global__ void chase(const unsigned* __restrict__ a, int n, int iters, unsigned long long* out, int mode) {
    unsigned idx = 0;
    // warm
    for (int i = 0; i < n; ++i) idx = mode == 0 ? __ldg(a + idx) : a[idx];
    unsigned long long t0 = clock64();
    for (int i = 0; i < iters; ++i) idx = mode == 0 ? __ldg(a + idx) : ((volatile const unsigned*)a)[idx];
    unsigned long long t1 = clock64();
    out[0] = (t1 - t0) / iters;
    out[1] = idx;
}
__global__ void smem_cas(int iters, unsigned long long* out) {
    unsigned long long* t = dyn;
    if (threadIdx.x == 0) t[0] = 0;
    __syncthreads();
    unsigned long long v = 1;
    unsigned long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        unsigned long long o = atomicCAS(t + (v & 7), 0ull, v + 1);
        v = o + 1;
    }
    unsigned long long t1 = clock64();
    unsigned long long t2 = clock64();
    for (int i = 0; i < iters; ++i) v = atomicMin(t + (v & 7), v) + 1;
    unsigned long long t3 = clock64();
    unsigned x = 1;
    unsigned* t32 = reinterpret_cast<unsigned*>(dyn + 64);
    unsigned long long t4 = clock64();
    for (int i = 0; i < iters; ++i) x = atomicMin(t32 + (x & 7), x) + 1;
    unsigned long long t5 = clock64();
    out[0] = (t1 - t0) / iters; out[1] = (t3 - t2) / iters; out[2] = (t5 - t4) / iters; out[3] = v + x;
}
int main() {
    const int n = 4096;  // 16 KB footprint
    unsigned h[n];
    for (int i = 0; i < n; ++i) h[i] = (i * 97 + 13) % n;
    unsigned* d; unsigned long long* o; cudaMalloc(&d, n * 4); cudaMalloc(&o, 64);
    cudaMemcpy(d, h, n * 4, cudaMemcpyHostToDevice);
    cudaFuncSetAttribute(chase, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    for (int smem : {0, 48 * 1024, 96 * 1024, 200 * 1024})
        for (int mode : {0, 1}) {
            chase<<<1, 32, smem>>>(d, n, 2000, o, mode);
            unsigned long long r[2]; cudaMemcpy(r, o, 16, cudaMemcpyDeviceToHost);
            printf("dyn smem %6d  %s  %llu cycles/load\n", smem, mode ? "volatile ld" : "ldg      ", r[0]);
        }
    cudaFuncSetAttribute(smem_cas, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    smem_cas<<<1, 1, 8192>>>(1000, o);
    unsigned long long r[4]; cudaMemcpy(r, o, 32, cudaMemcpyDeviceToHost);
    printf("smem CAS64 %llu  atomicMin64 %llu  atomicMin32 %llu cycles\n", r[0], r[1], r[2]);
    return 0;
}
