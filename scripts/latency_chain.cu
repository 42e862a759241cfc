// Developer probe: dependent-access latencies on B200 (one warp, data in L2).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/lc scripts/latency_chain.cu
#include <cstdio>
#include <cstdint>
__global__ void k(unsigned* a, unsigned long long* b, unsigned n, unsigned long long* out) {
    unsigned x = threadIdx.x;
    // warm L2
    for (unsigned i = threadIdx.x; i < n; i += 32) x += a[i];
    __syncwarp();
    __threadfence();
    unsigned long long t0 = clock64();
    unsigned p = x & 1;
    for (int i = 0; i < 64; ++i) p = __ldcg(a + ((p * 2654435761u + i * 7919u) % n));  // L2 loads, dependent
    unsigned long long t1 = clock64();
    for (int i = 0; i < 64; ++i) p = __ldg(a + ((p * 2654435761u + i * 7919u) % n));   // ld.global.nc
    unsigned long long t2 = clock64();
    unsigned long long q = p;
    for (int i = 0; i < 64; ++i) q = atomicMin(b + ((q * 2654435761u + i * 7919u) % n), 0xffffffffffffull + i);  // 64-bit atomic w/ return
    unsigned long long t3 = clock64();
    unsigned r = (unsigned)q;
    for (int i = 0; i < 64; ++i) r = atomicAdd(a + 5, 1u) + r;  // same-address atomic w/ return (warp-uniform? no: all lanes)
    unsigned long long t4 = clock64();
    for (int i = 0; i < 64; ++i) { unsigned v = 0; if (threadIdx.x == 0) v = atomicAdd(a + 7, 1u); r += __shfl_sync(~0u, v, 0); }
    unsigned long long t5 = clock64();
    if (threadIdx.x == 0) { out[0] = (t1 - t0) / 64; out[1] = (t2 - t1) / 64; out[2] = (t3 - t2) / 64; out[3] = (t4 - t3) / 64; out[4] = (t5 - t4) / 64; out[5] = r; }
}
int main() {
    unsigned n = 1 << 20;  // 4 MB / 8 MB: L2 resident
    unsigned* a; unsigned long long* b; unsigned long long* o;
    cudaMalloc(&a, n * 4); cudaMalloc(&b, n * 8); cudaMalloc(&o, 64);
    cudaMemset(a, 0, n * 4); cudaMemset(b, 0xff, n * 8);
    for (int rep = 0; rep < 3; ++rep) {
        k<<<1, 32>>>(a, b, n, o);
        unsigned long long h[6]; cudaMemcpy(h, o, 48, cudaMemcpyDeviceToHost);
        printf("cycles/step: ld.cg %llu  ld.nc %llu  atom.min.u64(ret) %llu  atom.add same-addr (32 lanes) %llu  atom.add 1 lane+shfl %llu\n", h[0], h[1], h[2], h[3], h[4]);
    }
}
