// Developer probe: dependent latency of warp collectives and shared-memory ops
// on B200 (one warp, clock64 over 1000 dependent iterations).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/wl scripts/warp_op_latency.cu
// Measured (cycles/iter incl. one dependent add): match_any 40, shfl (lane from
// data) 39, shfl_xor 31, ballot 29, popc(ballot) 45, reduce_add 48, smem load 36,
// smem store+load 36, smem atomicMin+load 62, IMAD 6.
#include <cstdio>
#include <cstdint>
template <int mode>
__global__ void k(unsigned* out, int n) {
    __shared__ unsigned tab[64];
    unsigned v = threadIdx.x * 7u;
    if (threadIdx.x < 64) tab[threadIdx.x] = 0xffffffffu;
    __syncwarp();
    long long t0 = clock64();
#pragma unroll 4
    for (int i = 0; i < n; ++i) {
        if (mode == 0) v = __match_any_sync(0xffffffffu, v & 7u) + v;
        else if (mode == 1) v = __shfl_sync(0xffffffffu, v, (v + 1) & 31) + 1;
        else if (mode == 2) { v = __ballot_sync(0xffffffffu, v & 1u) + v; }
        else if (mode == 3) { atomicMin(&tab[v & 63u], threadIdx.x); __syncwarp(); v = tab[(v + 1) & 63u] + v; }
        else if (mode == 4) { v = __reduce_add_sync(0xffffffffu, v) + 1; }
        else if (mode == 5) { tab[threadIdx.x & 63] = v; __syncwarp(); v = tab[(v + 3) & 31] + 1; }
        else if (mode == 6) { v = v * 3u + 1u; }
        else if (mode == 7) { v = __shfl_sync(0xffffffffu, v, 3) + 1; }
        else if (mode == 8) { v = __shfl_xor_sync(0xffffffffu, v, 1) + 1; }
        else if (mode == 9) { v = tab[v & 63u] + 1; }
        else if (mode == 10) { v = __popc(__ballot_sync(0xffffffffu, v & 1u)) + v; }
        else if (mode == 11) { __syncwarp(); v = v + 1; }
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) { out[0] = v; out[1] = (unsigned)((t1 - t0) / n); }
}
template <int m> void run(unsigned* d, const char* name) {
    k<m><<<1, 32>>>(d, 1000); cudaDeviceSynchronize();
    k<m><<<1, 32>>>(d, 1000); unsigned h[2]; cudaMemcpy(h, d, 8, cudaMemcpyDeviceToHost);
    printf("%-20s %u cycles/iter\n", name, h[1]);
}
int main() {
    unsigned* d; cudaMalloc(&d, 8);
    run<0>(d, "match_any"); run<1>(d, "shfl var"); run<2>(d, "ballot"); run<3>(d, "smem atomicMin+ld");
    run<4>(d, "reduce_add"); run<5>(d, "smem st+ld"); run<6>(d, "alu imad"); run<7>(d, "shfl const");
    run<8>(d, "shfl_xor"); run<9>(d, "smem ld"); run<10>(d, "popc(ballot)"); run<11>(d, "syncwarp+add");
}
