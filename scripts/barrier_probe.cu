// Developer probe: cost of grid-wide barrier variants on one B200
// (148 CTAs x 512 threads, cooperative launch). Not product code.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/bp scripts/barrier_probe.cu && /tmp/bp
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__device__ unsigned bar_count, bar_gen;
__device__ unsigned arrive[1024];

__device__ __forceinline__ unsigned ld_acq(const unsigned* p) { unsigned v; asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory"); return v; }
__device__ __forceinline__ unsigned ld_rlx(const unsigned* p) { unsigned v; asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory"); return v; }
__device__ __forceinline__ void st_rel(unsigned* p, unsigned v) { asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory"); }
__device__ __forceinline__ void st_rlx(unsigned* p, unsigned v) { asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory"); }
__device__ __forceinline__ unsigned atom_add_rel(unsigned* p, unsigned v) { unsigned o; asm volatile("atom.add.release.gpu.global.u32 %0, [%1], %2;" : "=r"(o) : "l"(p), "r"(v) : "memory"); return o; }

template <int V>
__global__ void k(int iters, unsigned long long* out) {
    unsigned epoch = arrive[blockIdx.x];
    unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        if (V == 0) {  // counter + generation, threadfences (engine r1)
            __syncthreads();
            if (threadIdx.x == 0) {
                volatile unsigned* vgen = &bar_gen;
                unsigned g0 = *vgen;
                __threadfence();
                unsigned a = atomicAdd(&bar_count, 1u);
                if (a == gridDim.x - 1) { bar_count = 0; __threadfence(); atomicAdd(&bar_gen, 1u); }
                else while (*vgen == g0) {}
                __threadfence();
            }
            __syncthreads();
        } else if (V == 1) {  // cg grid sync
            cg::this_grid().sync();
        } else if (V == 2) {  // flags, acquire polling
            __syncthreads(); ++epoch;
            if (threadIdx.x < 32) {
                if (threadIdx.x == 0) { __threadfence(); st_rel(arrive + blockIdx.x, epoch); }
                for (unsigned b = threadIdx.x; b < gridDim.x; b += 32) while ((int)(ld_acq(arrive + b) - epoch) < 0) {}
                __syncwarp();
            }
            __syncthreads();
        } else if (V == 3) {  // flags, relaxed polling + one fence
            __syncthreads(); ++epoch;
            if (threadIdx.x < 32) {
                if (threadIdx.x == 0) { __threadfence(); st_rlx(arrive + blockIdx.x, epoch); }
                for (unsigned b = threadIdx.x; b < gridDim.x; b += 32) while ((int)(ld_rlx(arrive + b) - epoch) < 0) {}
                __syncwarp();
                __threadfence();
            }
            __syncthreads();
        } else if (V == 4) {  // counter with release-atomic, relaxed spin on count (monotone target)
            __syncthreads(); ++epoch;
            if (threadIdx.x == 0) {
                atom_add_rel(&bar_count, 1u);
                const unsigned target = epoch * gridDim.x;
                while ((int)(ld_rlx(&bar_count) - target) < 0) {}
                __threadfence();
            }
            __syncthreads();
        } else if (V == 5) {  // flags, relaxed polling, no fences at all (lower bound, unsafe)
            __syncthreads(); ++epoch;
            if (threadIdx.x < 32) {
                if (threadIdx.x == 0) st_rlx(arrive + blockIdx.x, epoch);
                for (unsigned b = threadIdx.x; b < gridDim.x; b += 32) while ((int)(ld_rlx(arrive + b) - epoch) < 0) {}
                __syncwarp();
            }
            __syncthreads();
        }
    }
    if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = clock64() - t0;
    if (V == 4 && threadIdx.x == 0) arrive[blockIdx.x] = epoch;  // keep epoch consistent
}

template <int V>
void run(const char* name) {
    unsigned long long* d; cudaMalloc(&d, 8);
    int iters = 2000;
    void* args[] = {&iters, &d};
    unsigned z = 0;
    cudaMemcpyToSymbol(bar_count, &z, 4);
    cudaMemcpyToSymbol(bar_gen, &z, 4);
    static unsigned zz[1024] = {0};
    cudaMemcpyToSymbol(arrive, zz, sizeof zz);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int rep = 0; rep < 2; ++rep) {
        cudaMemcpyToSymbol(bar_count, &z, 4);
        cudaMemcpyToSymbol(arrive, zz, sizeof zz);
        cudaEventRecord(a);
        cudaError_t e = cudaLaunchCooperativeKernel((void*)k<V>, dim3(148), dim3(512), args, 0, nullptr);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        unsigned long long cyc; cudaMemcpy(&cyc, d, 8, cudaMemcpyDeviceToHost);
        if (rep) printf("%-40s %7.3f us/barrier  (%.0f cyc)  %s\n", name, ms * 1e3 / iters, double(cyc) / iters, cudaGetErrorString(e));
    }
}

int main() {
    run<0>("counter+gen, threadfence x2");
    run<1>("cooperative_groups grid.sync");
    run<2>("flags, ld.acquire polling");
    run<3>("flags, relaxed polling + fence");
    run<4>("release atomic count, relaxed spin");
    run<5>("flags, relaxed, no fence (unsafe bound)");
}
