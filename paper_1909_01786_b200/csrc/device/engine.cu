// yasmin-b200 device engine (sm_100a).
//
// The whole conflict-driven loop of the reference (Driver::run,
// /root/reference/proj/src/solver.cpp:248-303) runs on the device. The code is
// written once against a "group" abstraction and instantiated twice:
//   * BlockG  — one CTA owns one search; passes are separated by __syncthreads
//               and the control block lives in shared memory. Used for
//               structured/small stores and for cube-split enumeration (one
//               search per CTA, many CTAs per GPU).
//   * GridG   — every CTA of a cooperative grid works on ONE search; passes are
//               separated by a grid barrier. Used for wide propagation over
//               large stores (the 1M-nogood configurations).
//
// One propagation pass (propagate.cpp:170-205) is made exact and
// order-independent by a dense "expansion index" e: the frontier literals'
// occurrence lists, concatenated in frontier order and, per literal, in class
// (unit, binary, ternary, long) then id order, are numbered 0..T-1. The
// reference's item order (build_items, propagate.cpp:71-84) is exactly
// "ascending min-e of each nogood", and its merge (first proposal in item
// order wins an atom) is an atomicMin on (e, sign) per atom. Winners are
// compacted in e order with one group scan, which also yields the next
// frontier's occurrence offsets. Watched literals are not used: the reference
// results do not depend on them, so every check scans the
// nogood (a few literals, L1/L2 resident).
#include <cuda_runtime.h>

#include <cstdio>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "engine.cuh"
#include "engine_api.hpp"

namespace yas::dev {

// ---------------------------------------------------------------------------
// small helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ std::uint32_t atom_of(std::int32_t l) { return l < 0 ? -l : l; }
__device__ __forceinline__ std::uint32_t lidx(std::int32_t l) { return 2u * atom_of(l) + (l < 0 ? 1u : 0u); }
__device__ __forceinline__ std::uint32_t lvl_of(std::int32_t c) { return c < 0 ? -c : c; }
__device__ __forceinline__ bool may_assert(std::uint32_t guard, std::int32_t l) {
    return l < 0 || guard == kAny || guard == atom_of(l);
}
__device__ __forceinline__ std::uint32_t lane_id() { return threadIdx.x & 31u; }
__device__ __forceinline__ unsigned long long wkey(std::uint32_t gen, std::uint32_t e, bool neg) {
    return (static_cast<unsigned long long>(~gen) << 32) | (static_cast<unsigned long long>(e) << 1) | (neg ? 1ull : 0ull);
}
__device__ __forceinline__ unsigned long long ckey(std::uint32_t gen, std::uint32_t e) {
    return (static_cast<unsigned long long>(~gen) << 32) | e;
}
// L2 eviction priorities for the wide expansion: occurrence entries are
// streamed once per pass (evict-first) while the claim words they hit at
// random are reused across passes (evict-last); without the hints a wide pass
// over a store larger than L2 pushes the claims out and every claim becomes
// a DRAM read-modify-write. The policies are kernel parameters (Static), so
// they are read from the constant bank at each use and hold no register.
__device__ __forceinline__ int4 ld_stream(const int4* a, unsigned long long pol) {
#ifdef YAS_NO_L2HINT
    return __ldg(a);
#else
    int4 r;
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.s32 {%0, %1, %2, %3}, [%4], %5;"
        : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
        : "l"(a), "l"(pol));
    return r;
#endif
}
__device__ __forceinline__ unsigned long long atomic_min_keep(unsigned long long* a, unsigned long long v,
                                                              unsigned long long pol) {
#ifdef YAS_NO_L2HINT
    return atomicMin(a, v);
#else
    unsigned long long old;
    // not volatile, no memory clobber: the claims are only read again after a
    // barrier, so the atomics may be scheduled freely inside the batch
    asm("atom.global.min.L2::cache_hint.u64 %0, [%1], %2, %3;" : "=l"(old) : "l"(a), "l"(v), "l"(pol));
    return old;
#endif
}
__global__ void make_l2_policies(unsigned long long* out) {
    unsigned long long f, l;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(f));
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(l));
    out[0] = f;
    out[1] = l;
}
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ bool better(double s, std::uint32_t i, double bs, std::uint32_t bi) {
    return s > bs || (s == bs && i < bi);
}

// Warp-aggregated append: every lane of the (converged) warp calls it.
__device__ __forceinline__ std::uint32_t warp_append(std::uint32_t* ctr, bool pred) {
    const unsigned b = __ballot_sync(0xffffffffu, pred);
    if (b == 0) return 0xffffffffu;
    const int leader = __ffs(b) - 1;
    std::uint32_t base = 0;
    if (static_cast<int>(lane_id()) == leader) base = atomicAdd(ctr, static_cast<std::uint32_t>(__popc(b)));
    base = __shfl_sync(0xffffffffu, base, leader);
    return pred ? base + __popc(b & ((1u << lane_id()) - 1u)) : 0xffffffffu;
}
__device__ __forceinline__ void warp_count(unsigned long long* ctr, bool pred) {
    const unsigned b = __ballot_sync(0xffffffffu, pred);
    if (b && lane_id() == static_cast<std::uint32_t>(__ffs(b) - 1)) atomicAdd(ctr, static_cast<unsigned long long>(__popc(b)));
}

__device__ __forceinline__ void warp_sum(unsigned long long* ctr, std::uint32_t v) {
    const std::uint32_t t = __reduce_add_sync(0xffffffffu, v);
    if (lane_id() == 0 && t) atomicAdd(ctr, static_cast<unsigned long long>(t));
}

__device__ __forceinline__ unsigned long long warp_incl_scan(unsigned long long v) {
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        unsigned long long o = __shfl_up_sync(0xffffffffu, v, d);
        if (static_cast<int>(lane_id()) >= d) v += o;
    }
    return v;
}

// ---------------------------------------------------------------------------
// Groups
// ---------------------------------------------------------------------------
// Warp 0 of a CTA on its own: small passes run warp-synchronously.
// LEAN (all groups): the search runs the default configuration only (fwd
// learning, occurrence heuristic, no portfolio / trace / restarts / fanout /
// validation / profiling), so that code is compiled out of the kernel and its
// hot loop packs into fewer instruction-cache lines.
template <bool LEAN = false>
struct WarpG {
    static constexpr bool kBlock = false;
    static constexpr bool kGrid = false;
    static constexpr bool kLean = LEAN;
    Ctl* c;
    __device__ std::uint32_t tid() const { return lane_id(); }
    __device__ std::uint32_t size() const { return 32; }
    __device__ bool leader() const { return threadIdx.x == 0; }
    __device__ bool leader_warp() const { return true; }
    __device__ void sync() { __syncwarp(); }
    __device__ unsigned long long scan(unsigned long long v, unsigned long long& total) {
        const unsigned long long inc = warp_incl_scan(v);
        total = __shfl_sync(0xffffffffu, inc, 31);
        return inc - v;
    }
    __device__ void argmax(double& s, std::uint32_t& i) {
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) {
            double os = __shfl_down_sync(0xffffffffu, s, d);
            std::uint32_t oi = __shfl_down_sync(0xffffffffu, i, d);
            if (better(os, oi, s, i)) { s = os; i = oi; }
        }
        s = __shfl_sync(0xffffffffu, s, 0);
        i = __shfl_sync(0xffffffffu, i, 0);
    }
};

template <int BS, bool LEAN = false>
struct BlockG {
    static constexpr bool kBlock = true;
    static constexpr bool kGrid = false;
    static constexpr bool kLean = LEAN;
    static constexpr int kWarps = BS / 32;
    Ctl* c;
    unsigned long long* sbuf;  // kWarps+2 words of shared scratch
    double* sd;                // kWarps doubles
    std::uint32_t* si;         // kWarps words

    __device__ std::uint32_t tid() const { return threadIdx.x; }
    __device__ std::uint32_t size() const { return BS; }
    __device__ bool leader() const { return threadIdx.x == 0; }
    __device__ bool leader_warp() const { return threadIdx.x < 32; }
    __device__ void sync() { __syncthreads(); }

    // Exclusive scan of one value per thread over the whole group.
    __device__ unsigned long long scan(unsigned long long v, unsigned long long& total) {
        const std::uint32_t w = threadIdx.x >> 5;
        unsigned long long inc = warp_incl_scan(v);
        if (lane_id() == 31) sbuf[w] = inc;
        __syncthreads();
        if (w == 0) {
            unsigned long long x = lane_id() < kWarps ? sbuf[lane_id()] : 0ull;
            unsigned long long xi = warp_incl_scan(x);
            if (lane_id() < kWarps) sbuf[lane_id()] = xi - x;
            if (lane_id() == 31) sbuf[kWarps] = xi;
        }
        __syncthreads();
        const unsigned long long r = sbuf[w] + inc - v;
        total = sbuf[kWarps];
        __syncthreads();
        return r;
    }

    __device__ void argmax(double& s, std::uint32_t& i) {
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) {
            double os = __shfl_down_sync(0xffffffffu, s, d);
            std::uint32_t oi = __shfl_down_sync(0xffffffffu, i, d);
            if (better(os, oi, s, i)) { s = os; i = oi; }
        }
        const std::uint32_t w = threadIdx.x >> 5;
        if (lane_id() == 0) { sd[w] = s; si[w] = i; }
        __syncthreads();
        if (w == 0) {
            s = lane_id() < kWarps ? sd[lane_id()] : -1.0;
            i = lane_id() < kWarps ? si[lane_id()] : 0xffffffffu;
#pragma unroll
            for (int d = 16; d > 0; d >>= 1) {
                double os = __shfl_down_sync(0xffffffffu, s, d);
                std::uint32_t oi = __shfl_down_sync(0xffffffffu, i, d);
                if (better(os, oi, s, i)) { s = os; i = oi; }
            }
            if (lane_id() == 0) { sd[0] = s; si[0] = i; }
        }
        __syncthreads();
        s = sd[0];
        i = si[0];
        __syncthreads();
    }
    // Integer variant (s = score + 1, 0 = none; ties -> lowest index): two
    // warp reductions per level instead of five shuffle rounds of (double, index).
    __device__ void argmax_u(std::uint32_t& s, std::uint32_t& i) {
        std::uint32_t m = __reduce_max_sync(0xffffffffu, s);
        i = __reduce_min_sync(0xffffffffu, s == m ? i : 0xffffffffu);
        const std::uint32_t w = threadIdx.x >> 5;
        if (lane_id() == 0) sbuf[w] = (static_cast<unsigned long long>(m) << 32) | i;
        __syncthreads();
        if (w == 0) {
            const unsigned long long x = lane_id() < kWarps ? sbuf[lane_id()] : 0ull;
            const std::uint32_t xs = static_cast<std::uint32_t>(x >> 32), xi = lane_id() < kWarps ? static_cast<std::uint32_t>(x) : 0xffffffffu;
            m = __reduce_max_sync(0xffffffffu, xs);
            i = __reduce_min_sync(0xffffffffu, xs == m ? xi : 0xffffffffu);
            if (lane_id() == 0) sbuf[kWarps] = (static_cast<unsigned long long>(m) << 32) | i;
        }
        __syncthreads();
        const unsigned long long r = sbuf[kWarps];
        s = static_cast<std::uint32_t>(r >> 32);
        i = static_cast<std::uint32_t>(r);
        __syncthreads();
    }
};

template <int BS>
struct GridG {
    static constexpr bool kBlock = false;
    static constexpr bool kGrid = true;
    static constexpr bool kLean = false;
    static constexpr int kWarps = BS / 32;
    Ctl* c;
    Shared* sh;
    unsigned long long* partial;  // 2 parities x {block totals, block extras} x gridDim.x
    double* pd;                   // gridDim.x
    std::uint32_t* pi;            // gridDim.x
    unsigned long long* sbuf;
    double* sd;
    std::uint32_t* si;
    std::uint32_t parity;
    unsigned long long* bc;  // shared: per-block pass counters {checks, conflicts, literals}
    std::uint32_t epoch;     // barriers passed (same in every block)
    std::uint32_t* snap;     // shared: control words snapshotted at a barrier
    std::int32_t* scanq;     // shared: per-warp queue of nogoods needing a full scan
    std::uint32_t* scane;    //   ... and their expansion indices

    // solo: block 0 alone runs passes (tiny frontiers) while the other blocks
    // wait at the next grid barrier; ids, size and sync become block-local.
    bool solo;

    __device__ std::uint32_t tid() const { return solo ? threadIdx.x : blockIdx.x * BS + threadIdx.x; }
    __device__ std::uint32_t size() const { return solo ? BS : gridDim.x * BS; }
    __device__ bool leader() const { return blockIdx.x == 0 && threadIdx.x == 0; }
    __device__ bool leader_warp() const { return blockIdx.x == 0 && threadIdx.x < 32; }
    // Block-interleaved numbering: consecutive ids land on different SMs, so
    // a small amount of work is spread over the whole GPU.
    __device__ std::uint32_t itid() const { return solo ? threadIdx.x : threadIdx.x * gridDim.x + blockIdx.x; }
    __device__ std::uint32_t iwarp() const { return solo ? threadIdx.x >> 5 : (threadIdx.x >> 5) * gridDim.x + blockIdx.x; }

    // Exclusive scan of one value per thread over this block only.
    __device__ unsigned long long block_scan(unsigned long long v, unsigned long long& total) {
        const std::uint32_t w = threadIdx.x >> 5;
        unsigned long long inc = warp_incl_scan(v);
        if (lane_id() == 31) sbuf[w] = inc;
        __syncthreads();
        if (w == 0) {
            unsigned long long x = lane_id() < kWarps ? sbuf[lane_id()] : 0ull;
            unsigned long long xi = warp_incl_scan(x);
            if (lane_id() < kWarps) sbuf[lane_id()] = xi - x;
            if (lane_id() == 31) sbuf[kWarps] = xi;
        }
        __syncthreads();
        const unsigned long long r = sbuf[w] + inc - v;
        total = sbuf[kWarps];
        __syncthreads();
        return r;
    }

    // Grid barrier: one release-add on a monotone arrival counter per block,
    // then a relaxed spin until the counter reaches epoch * gridDim (wrap-safe
    // difference) and an acquire fence. The counter is never reset; every block
    // passes the same barriers, so each keeps its epoch in sh->arrive[block]
    // across launches (see persist()). 1.2 us per barrier on B200 with 148
    // CTAs (scripts/barrier_probe.cu), against 2.1 us for a counter+generation
    // barrier with two fences and 5.5 us for flag all-gathers.
    __device__ void sync() { sync_snap(nullptr, nullptr); }
    // Barrier that also snapshots up to two control words, read once per
    // block by thread 0 after the barrier, into shared memory (snap[0..1]):
    // all threads reading one global word would queue thousands of requests
    // on one L2 slice.
    __device__ void sync_snap(const std::uint32_t* a, const std::uint32_t* b, const std::uint32_t* d = nullptr) {
        __syncthreads();
        if (solo) {
            if (threadIdx.x == 0) {
                __threadfence_block();
                if (a) snap[0] = *reinterpret_cast<const volatile std::uint32_t*>(a);
                if (b) snap[1] = *reinterpret_cast<const volatile std::uint32_t*>(b);
                if (d) snap[2] = *reinterpret_cast<const volatile std::uint32_t*>(d);
            }
            __syncthreads();
            return;
        }
        ++epoch;
        if (threadIdx.x == 0) {
            asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(&sh->bar_count), "r"(1u) : "memory");
            const std::uint32_t target = epoch * gridDim.x;
            for (;;) {
                std::uint32_t v;
                asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(&sh->bar_count) : "memory");
                if (static_cast<int>(v - target) >= 0) break;
            }
            __threadfence();
            if (a) snap[0] = *reinterpret_cast<const volatile std::uint32_t*>(a);
            if (b) snap[1] = *reinterpret_cast<const volatile std::uint32_t*>(b);
            if (d) snap[2] = *reinterpret_cast<const volatile std::uint32_t*>(d);
        }
        __syncthreads();
    }
    // Store this block's epoch for the next launch on the same arena.
    __device__ void persist() const {
        if (threadIdx.x == 0) sh->arrive[blockIdx.x] = epoch;
    }

    __device__ unsigned long long scan(unsigned long long v, unsigned long long& total) {
        if (solo) return block_scan(v, total);
        const std::uint32_t w = threadIdx.x >> 5;
        unsigned long long inc = warp_incl_scan(v);
        if (lane_id() == 31) sbuf[w] = inc;
        __syncthreads();
        if (w == 0) {
            unsigned long long x = lane_id() < kWarps ? sbuf[lane_id()] : 0ull;
            unsigned long long xi = warp_incl_scan(x);
            if (lane_id() < kWarps) sbuf[lane_id()] = xi - x;
            if (lane_id() == 31) sbuf[kWarps] = xi;
        }
        __syncthreads();
        unsigned long long* part = partial + parity * 2 * gridDim.x;
        parity ^= 1u;
        if (threadIdx.x == 0) part[blockIdx.x] = sbuf[kWarps];
        sync();
        if (w == 0) {
            unsigned long long before = 0, all = 0;
            for (std::uint32_t b = lane_id(); b < gridDim.x; b += 32) {
                const unsigned long long x = part[b];
                all += x;
                if (b < blockIdx.x) before += x;
            }
#pragma unroll
            for (int d = 16; d > 0; d >>= 1) {
                before += __shfl_down_sync(0xffffffffu, before, d);
                all += __shfl_down_sync(0xffffffffu, all, d);
            }
            if (lane_id() == 0) { sbuf[kWarps + 1] = before; sbuf[kWarps + 2] = all; }
        }
        __syncthreads();
        const unsigned long long r = sbuf[kWarps + 1] + sbuf[w] + inc - v;
        total = sbuf[kWarps + 2];
        __syncthreads();
        return r;
    }

    // scan() that also sums one block-level value (*ex, in shared memory,
    // final when the call is made) over the grid: *ex_total on return.
    __device__ unsigned long long scan_ex(unsigned long long v, unsigned long long& total, const unsigned long long* ex,
                                          unsigned long long& ex_total) {
        const std::uint32_t w = threadIdx.x >> 5;
        unsigned long long inc = warp_incl_scan(v);
        if (lane_id() == 31) sbuf[w] = inc;
        __syncthreads();
        if (w == 0) {
            unsigned long long x = lane_id() < kWarps ? sbuf[lane_id()] : 0ull;
            unsigned long long xi = warp_incl_scan(x);
            if (lane_id() < kWarps) sbuf[lane_id()] = xi - x;
            if (lane_id() == 31) sbuf[kWarps] = xi;
        }
        __syncthreads();
        unsigned long long* part = partial + parity * 2 * gridDim.x;
        parity ^= 1u;
        if (threadIdx.x == 0) {
            part[blockIdx.x] = sbuf[kWarps];
            part[gridDim.x + blockIdx.x] = *ex;
        }
        sync();
        if (w == 0) {
            unsigned long long before = 0, all = 0, xall = 0;
            for (std::uint32_t b = lane_id(); b < gridDim.x; b += 32) {
                const unsigned long long x = part[b];
                all += x;
                xall += part[gridDim.x + b];
                if (b < blockIdx.x) before += x;
            }
#pragma unroll
            for (int d = 16; d > 0; d >>= 1) {
                before += __shfl_down_sync(0xffffffffu, before, d);
                all += __shfl_down_sync(0xffffffffu, all, d);
                xall += __shfl_down_sync(0xffffffffu, xall, d);
            }
            if (lane_id() == 0) { sbuf[kWarps + 1] = before; sbuf[kWarps + 2] = all; sbuf[kWarps + 3] = xall; }
        }
        __syncthreads();
        const unsigned long long r = sbuf[kWarps + 1] + sbuf[w] + inc - v;
        total = sbuf[kWarps + 2];
        ex_total = sbuf[kWarps + 3];
        __syncthreads();
        return r;
    }

    __device__ void argmax(double& s, std::uint32_t& i) {
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) {
            double os = __shfl_down_sync(0xffffffffu, s, d);
            std::uint32_t oi = __shfl_down_sync(0xffffffffu, i, d);
            if (better(os, oi, s, i)) { s = os; i = oi; }
        }
        const std::uint32_t w = threadIdx.x >> 5;
        if (lane_id() == 0) { sd[w] = s; si[w] = i; }
        __syncthreads();
        if (w == 0) {
            s = lane_id() < kWarps ? sd[lane_id()] : -1.0;
            i = lane_id() < kWarps ? si[lane_id()] : 0xffffffffu;
#pragma unroll
            for (int d = 16; d > 0; d >>= 1) {
                double os = __shfl_down_sync(0xffffffffu, s, d);
                std::uint32_t oi = __shfl_down_sync(0xffffffffu, i, d);
                if (better(os, oi, s, i)) { s = os; i = oi; }
            }
            if (lane_id() == 0) { pd[blockIdx.x] = s; pi[blockIdx.x] = i; }
        }
        sync();
        if (w == 0) {
            s = -1.0;
            i = 0xffffffffu;
            for (std::uint32_t b = lane_id(); b < gridDim.x; b += 32)
                if (better(pd[b], pi[b], s, i)) { s = pd[b]; i = pi[b]; }
#pragma unroll
            for (int d = 16; d > 0; d >>= 1) {
                double os = __shfl_down_sync(0xffffffffu, s, d);
                std::uint32_t oi = __shfl_down_sync(0xffffffffu, i, d);
                if (better(os, oi, s, i)) { s = os; i = oi; }
            }
            if (lane_id() == 0) { sd[0] = s; si[0] = i; }
        }
        __syncthreads();
        s = sd[0];
        i = si[0];
        // every block leaves pd/pi untouched until the next argmax, which is
        // separated from this one by at least one grid barrier.
        __syncthreads();
    }
};

// ---------------------------------------------------------------------------
// The search (one instance per group)
// ---------------------------------------------------------------------------
// Shared-memory working set of a single-CTA search. Offsets are computed on
// the host (plan_smem) and passed as a __grid_constant__ kernel parameter, so
// every array address is "dynamic-smem base + constant".
struct SmemCfg {
    std::uint32_t tcap, hcap, fcap, vwords;
    std::uint32_t o_htab, o_wtab, o_pid, o_plit, o_pslot, o_pdep, o_pmeta, o_litat, o_otat, o_bits, o_fr, o_froff,
        o_vmir, bytes;
};

extern __shared__ __align__(16) unsigned char yas_dsm[];

struct Sm {
    const SmemCfg* cfg;
    template <class T>
    __device__ __forceinline__ T* at(std::uint32_t off) const { return reinterpret_cast<T*>(yas_dsm + off); }
    __device__ __forceinline__ unsigned long long* htab() const { return at<unsigned long long>(cfg->o_htab); }  // (id+1)<<32 | min e
    __device__ __forceinline__ unsigned long long* wtab() const { return at<unsigned long long>(cfg->o_wtab); }  // (atom+1)<<32 | e<<1|neg
    __device__ __forceinline__ std::int32_t* pid() const { return at<std::int32_t>(cfg->o_pid); }
    __device__ __forceinline__ std::int32_t* plit() const { return at<std::int32_t>(cfg->o_plit); }
    __device__ __forceinline__ std::uint32_t* pslot() const { return at<std::uint32_t>(cfg->o_pslot); }  // claim | win << 16
    __device__ __forceinline__ unsigned long long* pdep() const { return at<unsigned long long>(cfg->o_pdep); }  // Deps word 0
    __device__ __forceinline__ std::uint32_t* pmeta() const { return at<std::uint32_t>(cfg->o_pmeta); }  // ovf<<31 | occ total
    __device__ __forceinline__ std::int32_t* litat() const { return at<std::int32_t>(cfg->o_litat); }
    __device__ __forceinline__ std::uint32_t* otat() const { return at<std::uint32_t>(cfg->o_otat); }
    __device__ __forceinline__ std::uint32_t* bits() const { return at<std::uint32_t>(cfg->o_bits); }
    __device__ __forceinline__ std::int32_t* fr() const { return at<std::int32_t>(cfg->o_fr); }  // frontier mirror
    __device__ __forceinline__ std::uint32_t* froff() const { return at<std::uint32_t>(cfg->o_froff); }
    // 2 bits per atom (bit 0 assigned, bit 1 true), 16 atoms per word: one load per value
    __device__ __forceinline__ std::uint32_t* vmir() const { return at<std::uint32_t>(cfg->o_vmir); }
    __device__ __forceinline__ std::uint32_t tcap() const { return cfg->tcap; }
    __device__ __forceinline__ std::uint32_t hmask() const { return cfg->hcap ? cfg->hcap - 1 : 0; }
    __device__ __forceinline__ std::uint32_t fcap() const { return cfg->fcap; }
    __device__ __forceinline__ std::uint32_t vwords() const { return cfg->vwords; }
};

__device__ __forceinline__ std::uint32_t hslot(std::uint32_t key, std::uint32_t mask) { return (key * 2654435761u) & mask; }

// Host: lay out the shared-memory arrays for a given capacity.
SmemCfg smem_layout(std::uint32_t tcap, std::uint32_t vwords) {
    SmemCfg c{};
    c.tcap = tcap;
    c.hcap = tcap ? 2 * tcap : 0;
    c.fcap = tcap ? tcap + 1 : 0;
    c.vwords = vwords;
    std::uint32_t o = 0;
    auto take = [&](std::uint32_t bytes) {
        const std::uint32_t at = o;
        o += (bytes + 15u) & ~15u;
        return at;
    };
    if (tcap) {
        c.o_htab = take(8u * c.hcap);
        c.o_wtab = take(8u * c.hcap);
        c.o_pdep = take(8u * tcap);
        c.o_pid = take(4u * tcap);
        c.o_plit = take(4u * tcap);
        c.o_pslot = take(4u * tcap);
        c.o_pmeta = take(4u * tcap);
        c.o_litat = take(4u * tcap);
        c.o_otat = take(4u * tcap);
        c.o_bits = take(4u * ((tcap + 31) / 32));
        c.o_fr = take(4u * c.fcap);
        c.o_froff = take(4u * (c.fcap + 1));
    }
    if (vwords) {
        c.o_vmir = take(8u * vwords);
    }
    c.bytes = o;
    return c;
}

template <class G>
struct Search {
    G& g;
    const Static& S;
    const Config& C;
    Slot sl;
    const Caps& K;
    Shared* sh;
    Ctl* c;
    unsigned long long t0;
    Sm sm;

    __device__ __forceinline__ Search(G& g_, const Static& s, const Config& cf, Slot slot, const Caps& k, Shared* shared,
                      unsigned long long start, const Sm& smem)
        : g(g_), S(s), C(cf), sl(slot), K(k), sh(shared), c(g_.c), t0(start), sm(smem) {}

    // ---- assignment access: 2-bit shared mirror when present --------------
    // sign of the atom's value: 0 unassigned, 1 true, -1 false
    // Whole-grid slots keep a 2-bit mirror of the assignment in global memory
    // (16 atoms per word; 25 KB for 100k atoms) next to the cells.
    __device__ __forceinline__ static int mirror_val(std::uint32_t word, std::uint32_t a) {
        const std::uint32_t v = (word >> (2 * (a & 15))) & 3u;
        return v == 0 ? 0 : (v == 3 ? 1 : -1);
    }
    // Pass-snapshot read (L1-cached): only for values that cannot change
    // during the current phase.
    __device__ __forceinline__ std::uint32_t mirror_word_snap(std::uint32_t a) const { return __ldca(sl.gmirror() + (a >> 4)); }

    __device__ __forceinline__ int val(std::uint32_t a) const {
        if constexpr (G::kGrid) return mirror_val(__ldcg(sl.gmirror() + (a >> 4)), a);
        if (sm.vwords()) return mirror_val(sm.vmir()[a >> 4], a);
        const std::int32_t cv = sl.cells()[a];
        return (cv > 0) - (cv < 0);
    }
    __device__ __forceinline__ void set_cell(std::uint32_t a, std::int32_t cv) const {
        sl.cells()[a] = cv;
        if constexpr (G::kGrid) {
            std::uint32_t* w = sl.gmirror() + (a >> 4);
            const std::uint32_t sh2 = 2 * (a & 15);
            if (cv == 0) atomicAnd(w, ~(3u << sh2));
            else atomicOr(w, (cv > 0 ? 3u : 1u) << sh2);  // bits are clear while unassigned
            return;
        }
        if (sm.vwords()) {
            std::uint32_t* w = sm.vmir() + (a >> 4);
            const std::uint32_t sh2 = 2 * (a & 15);
            if (cv == 0) atomicAnd(w, ~(3u << sh2));
            else atomicOr(w, (cv > 0 ? 3u : 1u) << sh2);  // bits are clear while unassigned
        }
    }
    __device__ __forceinline__ void rebuild_mirror() const {
        if (!sm.vwords()) return;
        for (std::uint32_t w = g.tid(); w < 2 * sm.vwords(); w += g.size()) {
            std::uint32_t bits = 0;
            for (std::uint32_t b = 0; b < 16; ++b) {
                const std::uint32_t a = 16 * w + b;
                if (a > S.A) break;
                const std::int32_t cv = sl.cells()[a];
                if (cv != 0) bits |= (cv > 0 ? 3u : 1u) << (2 * b);
            }
            sm.vmir()[w] = bits;
        }
    }

    // ---- store access ----------------------------------------------------
    __device__ __forceinline__ const std::int32_t* lits_of(std::uint32_t id, std::uint32_t& len) const {
        if (id < S.N) {
            const std::uint32_t lo = __ldg(S.off + id);
            len = __ldg(S.off + id + 1) - lo;
            return S.pool + lo;
        }
        const std::uint32_t k = id - S.N;
        const std::uint32_t lo = sl.loff()[k];
        len = sl.loff()[k + 1] - lo;
        return sl.lpool() + lo;
    }
    __device__ __forceinline__ std::int32_t lit_at(const std::int32_t* p, std::uint32_t k, std::uint32_t id) const {
        return id < S.N ? __ldg(p + k) : p[k];
    }
    __device__ __forceinline__ std::uint32_t length_of(std::uint32_t id) const {
        if (id < S.N) return __ldg(S.off + id + 1) - __ldg(S.off + id);
        return sl.loff()[id - S.N + 1] - sl.loff()[id - S.N];
    }
    __device__ __forceinline__ std::uint32_t guard_of(std::uint32_t id) const { return id < S.N ? __ldg(S.guard + id) : kNone; }
    __device__ __forceinline__ std::uint32_t occ_total(std::uint32_t li) const {
        return __ldg(S.occ_off + li * 4 + 4) - __ldg(S.occ_off + li * 4) + sl.ltot()[li];
    }
    // j-th entry of the literal's occurrence list [static c0, learned c0, ...,
    // static c3, learned c3]: {id, guard, x, y} and its length class. Entries
    // carry their class in the top two bits of the id, so with no learned
    // nogoods one offset load and one dependent 16-byte load suffice.
    __device__ __forceinline__ static int4 decode(int4 ent, std::uint32_t& cls) {
        cls = static_cast<std::uint32_t>(ent.x) >> 30;
        ent.x &= 0x3fffffff;
        return ent;
    }
    __device__ __forceinline__ int4 occ_entry(std::uint32_t li, std::uint32_t j, bool learned, std::uint32_t& cls) const {
        const std::uint32_t* oo = S.occ_off + li * 4;
        if (!learned) return decode(__ldg(S.occ + __ldg(oo) + j), cls);
        const std::uint32_t b0 = __ldg(oo), lt = sl.ltot()[li];  // one round trip
        if (lt == 0) return decode(__ldg(S.occ + b0 + j), cls);  // no learned occurrences of this literal
        std::uint32_t b[5];
#pragma unroll
        for (int k = 0; k < 5; ++k) b[k] = __ldg(oo + k);
        const std::uint32_t* h = sl.lhdr() + 12 * li;
        std::uint32_t hp[4], hn[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            hp[k] = h[3 * k];
            hn[k] = h[3 * k + 1];
        }
#pragma unroll
        for (int cl = 0; cl < 4; ++cl) {
            const std::uint32_t ns = b[cl + 1] - b[cl];
            if (j < ns) return decode(__ldg(S.occ + b[cl] + j), cls);
            j -= ns;
            if (j < hn[cl]) return decode(sl.larena()[hp[cl] + j], cls);
            j -= hn[cl];
        }
        cls = 0;
        return make_int4(-1, 0, 0, 0);
    }
    // learning mode / heuristic of this search (a portfolio varies them per search)
    __device__ __forceinline__ std::uint32_t mode() const {
        if constexpr (G::kLean) return 0u;
        if constexpr (G::kGrid) return C.mode;  // a portfolio runs single-CTA searches
        return C.portfolio ? (c->variant & 1u) : C.mode;
    }
    __device__ __forceinline__ std::uint32_t heur() const {
        if constexpr (G::kLean) return 0u;
        if constexpr (G::kGrid) return C.heur;
        return C.portfolio ? (c->variant >> 1) : C.heur;
    }
    __device__ __forceinline__ bool prof_on() const { return !G::kLean && C.phase_prof; }
    __device__ __forceinline__ bool trace_on() const { return !G::kLean && C.trace; }
    __device__ __forceinline__ bool portfolio_on() const { return !G::kLean && C.portfolio; }
    __device__ __forceinline__ std::uint32_t nwords(std::uint32_t level) const {
        const std::uint32_t nw = level <= 1 ? 1u : (level - 1) / 64 + 1;
        return nw < C.W ? nw : C.W;
    }
    // Deps rows are atom-major: the words of one atom are contiguous (row
    // stride rounded up to an even word count for 16-byte vector access).
    __device__ __forceinline__ std::uint32_t dstride() const { return (C.W + 1u) & ~1u; }
    __device__ __forceinline__ unsigned long long& dep(std::uint32_t w, std::uint32_t a) const {
        return sl.deps()[static_cast<std::size_t>(a) * dstride() + w];
    }
    // OR words [w0, w0 + 2*NQ) of the Deps rows of atoms x[k] (on[k]) into
    // acc, as 16-byte loads all issued before any is used.
    template <int NK, int NQ>
    __device__ __forceinline__ void or_rows(const std::uint32_t* x, const bool* on, std::uint32_t w0, std::uint32_t nw,
                            unsigned long long* acc) const {
        ulonglong2 v[NK][NQ];
#pragma unroll
        for (int k = 0; k < NK; ++k) {
            const ulonglong2* row = reinterpret_cast<const ulonglong2*>(sl.deps() + static_cast<std::size_t>(on[k] ? x[k] : 0u) * dstride() + w0);
#pragma unroll
            for (int q = 0; q < NQ; ++q) v[k][q] = (on[k] && w0 + 2 * q < nw) ? row[q] : make_ulonglong2(0ull, 0ull);
        }
#pragma unroll
        for (int k = 0; k < NK; ++k)
#pragma unroll
            for (int q = 0; q < NQ; ++q) {
                acc[2 * q] |= v[k][q].x;
                acc[2 * q + 1] |= v[k][q].y;
            }
    }
    template <int NQ>
    __device__ __forceinline__ void store_row(std::uint32_t a, std::uint32_t w0, std::uint32_t nw, const unsigned long long* acc) const {
        ulonglong2* row = reinterpret_cast<ulonglong2*>(sl.deps() + static_cast<std::size_t>(a) * dstride() + w0);
#pragma unroll
        for (int q = 0; q < NQ; ++q)
            if (w0 + 2 * q < nw) {
                if (w0 + 2 * q + 1 < nw) row[q] = make_ulonglong2(acc[2 * q], acc[2 * q + 1]);
                else reinterpret_cast<unsigned long long*>(row)[2 * q] = acc[2 * q];
            }
    }
    // Deps of atom a from the rows of up to two contributing atoms.
    __device__ __forceinline__ void deps_from_pair(std::uint32_t a, std::uint32_t x0, bool on0, std::uint32_t x1, bool on1,
                                   std::uint32_t nw) const {
        const std::uint32_t xs[2] = {x0, x1};
        const bool ons[2] = {on0, on1};
        for (std::uint32_t w0 = 0; w0 < nw; w0 += 8) {
            unsigned long long acc[8] = {0ull, 0ull, 0ull, 0ull, 0ull, 0ull, 0ull, 0ull};
            or_rows<2, 4>(xs, ons, w0, nw, acc);
            store_row<4>(a, w0, nw, acc);
        }
        sl.dovf()[a] = static_cast<std::uint8_t>((on0 ? sl.dovf()[x0] : 0) | (on1 ? sl.dovf()[x1] : 0));
    }
    __device__ __forceinline__ bool holds(std::int32_t l) const {
        const int v = val(atom_of(l));
        return v != 0 && ((v > 0) == (l > 0));
    }

    // phase accounting: cycles since the previous mark go to bucket k
    __device__ __forceinline__ void mark(int k) const {
        if constexpr (G::kGrid) return;  // grid passes: see stamp()
        if (prof_on() && g.leader()) {
            const unsigned long long t = clock64();
            c->prof[k] += t - c->prof_t;
            c->prof_t = t;
        }
    }

    // Diagnostics (builds with -DYAS_TINY_PROF): warp-synchronous sub-phase
    // cycles of a tiny pass, accounted like mark().
    __device__ __forceinline__ void tprof(int k) const {
#ifdef YAS_TINY_PROF
        __syncwarp();
        if (prof_on() && lane_id() == 0) {
            const unsigned long long t = clock64();
            c->prof[k] += t - c->prof_t;
            c->prof_t = t;
        }
        __syncwarp();
#else
        (void)k;
#endif
    }

    // Diagnostics: thread 0 of every block stamps the global timer at phase
    // boundaries of the first kPtracePasses passes of a grid propagation.
    static constexpr std::uint32_t kPtracePasses = 64, kPtraceStamps = 10;
    __device__ __forceinline__ void stamp(std::uint32_t pass, std::uint32_t k) const {
        if (C.ptrace && threadIdx.x == 0 && pass < kPtracePasses)
            C.ptrace[(static_cast<std::size_t>(pass) * gridDim.x + blockIdx.x) * kPtraceStamps + k] = gtimer();
    }

    // Diagnostics: in-phase stamps (clock64) of warp 0 of block 0 in pass `pass`.
    __device__ __forceinline__ void dstamp(std::uint32_t pass, std::uint32_t k) const {
        if (C.ptrace && blockIdx.x == 0 && threadIdx.x == 0 && pass < kPtracePasses)
            C.ptrace[static_cast<std::size_t>(kPtracePasses) * gridDim.x * kPtraceStamps + pass * 16 + k] = clock64();
    }

    __device__ __forceinline__ void fail(std::uint32_t status) {
        if (g.leader()) c->status = status;
    }

    // Deps of the literal derived from nogood (lits,len) on atom `a`:
    // OR of Deps[x] over the other atoms with level > 1 (propagate.cpp:49-62).
    __device__ __forceinline__ void write_deps_from(const std::int32_t* L, std::uint32_t len, std::uint32_t id, std::uint32_t a,
                                    std::uint32_t level) const {
        const std::uint32_t nw = nwords(level);
        if (len <= 8) {
            // literals, then cells + overflow bytes, then 4 Deps words of every
            // contributing literal per sweep: 2 + ceil(nw/4) round trips
            std::int32_t l[8];
#pragma unroll
            for (std::uint32_t k = 0; k < 8; ++k) l[k] = k < len ? lit_at(L, k, id) : 0;
            std::uint32_t x[8];
            bool on[8];
            std::uint8_t ov[8];
#pragma unroll
            for (std::uint32_t k = 0; k < 8; ++k) {
                x[k] = atom_of(l[k]);
                const std::int32_t cv = sl.cells()[x[k]];
                ov[k] = sl.dovf()[x[k]];
                on[k] = k < len && x[k] != a && lvl_of(cv) > 1;
            }
            std::uint8_t ovf = 0;
#pragma unroll
            for (std::uint32_t k = 0; k < 8; ++k) ovf |= on[k] ? ov[k] : 0;
            for (std::uint32_t w0 = 0; w0 < nw; w0 += 4) {
                unsigned long long acc[4] = {0ull, 0ull, 0ull, 0ull};
                or_rows<4, 2>(x, on, w0, nw, acc);
                or_rows<4, 2>(x + 4, on + 4, w0, nw, acc);
                store_row<2>(a, w0, nw, acc);
            }
            sl.dovf()[a] = ovf;
            return;
        }
        std::uint8_t ovf = 0;
        for (std::uint32_t w0 = 0; w0 < nw; w0 += 4) {  // 4 words per sweep: independent loads
            unsigned long long acc[4] = {0ull, 0ull, 0ull, 0ull};
            for (std::uint32_t k = 0; k < len; ++k) {
                const std::uint32_t x = atom_of(lit_at(L, k, id));
                if (x == a || lvl_of(sl.cells()[x]) <= 1) continue;
#pragma unroll
                for (std::uint32_t q = 0; q < 4; ++q)
                    if (w0 + q < nw) acc[q] |= dep(w0 + q, x);
                if (w0 == 0) ovf |= sl.dovf()[x];
            }
#pragma unroll
            for (std::uint32_t q = 0; q < 4; ++q)
                if (w0 + q < nw) dep(w0 + q, a) = acc[q];
        }
        sl.dovf()[a] = ovf;
    }
    __device__ __forceinline__ unsigned long long deps_word(const std::int32_t* L, std::uint32_t len, std::uint32_t id,
                                            std::uint32_t a, std::uint32_t w, std::uint8_t& ovf) const {
        unsigned long long acc = 0;
        for (std::uint32_t k = 0; k < len; ++k) {
            const std::uint32_t x = atom_of(lit_at(L, k, id));
            const std::int32_t cv = sl.cells()[x];
            const unsigned long long d = dep(w, x);
            const std::uint8_t o = w == 0 ? sl.dovf()[x] : 0;
            if (x != a && lvl_of(cv) > 1) {
                acc |= d;
                ovf |= o;
            }
        }
        return acc;
    }

    // ---- group-parallel building blocks -------------------------------------
    // Exclusive occurrence offsets of the current frontier; sets c->T. The
    // frontier and its offsets are mirrored into shared memory when they fit.
    __device__ __forceinline__ void frontier_offsets() {
        const std::uint32_t F = c->F;
        const std::int32_t* fr = sl.fr(c->cur);
        const bool mirror = sm.tcap() && F + 1 <= sm.fcap();
        if constexpr (G::kBlock) {
            if (F <= 32) {  // a decision or a few asserted literals: warp 0 alone, one barrier
                if (threadIdx.x < 32) {
                    const std::uint32_t lane = lane_id();
                    const std::int32_t lit = lane < F ? fr[lane] : 0;
                    const std::uint32_t v = lane < F ? occ_total(lidx(lit)) : 0u;
                    std::uint32_t inc = v;
#pragma unroll
                    for (int d = 1; d < 32; d <<= 1) {
                        const std::uint32_t o = __shfl_up_sync(0xffffffffu, inc, d);
                        if (lane >= static_cast<std::uint32_t>(d)) inc += o;
                    }
                    const std::uint32_t total = __shfl_sync(0xffffffffu, inc, 31);
                    if (lane < F) {
                        sl.froff()[lane] = inc - v;
                        if (mirror) {
                            sm.froff()[lane] = inc - v;
                            sm.fr()[lane] = lit;
                        }
                    }
                    if (lane == 0) {
                        sl.froff()[F] = total;
                        if (mirror) sm.froff()[F] = total;
                        c->T = total;
                        c->b[11] = 0;
                    }
                }
                g.sync();
                mark(1);
                return;
            }
        }
        unsigned long long carry = 0;
        for (std::uint32_t base = 0; base < F; base += g.size()) {
            const std::uint32_t p = base + g.tid();
            const std::int32_t lit = p < F ? fr[p] : 0;
            const unsigned long long v = p < F ? occ_total(lidx(lit)) : 0ull;
            unsigned long long tot;
            const unsigned long long pre = g.scan(v, tot) + carry;
            if (p < F) {
                sl.froff()[p] = static_cast<std::uint32_t>(pre);
                if constexpr (G::kGrid) sl.frb()[p] = __ldg(S.occ_off + lidx(lit) * 4);
                if (mirror) {
                    sm.froff()[p] = static_cast<std::uint32_t>(pre);
                    sm.fr()[p] = lit;
                }
            }
            carry += tot;
        }
        g.sync();
        if (g.leader()) {
            sl.froff()[F] = static_cast<std::uint32_t>(carry);
            if (mirror) sm.froff()[F] = static_cast<std::uint32_t>(carry);
            c->T = static_cast<std::uint32_t>(carry);
            c->b[11] = 0;
        }
        g.sync();
        mark(1);
    }

    // Winners marked in the bitmap (bits e < T) are written, in e order, to the
    // frontier buffer `dst`, appended to the trail, and the occurrence offsets
    // of that new frontier are produced by the same scan.
    template <bool SMEM>
    __device__ __forceinline__ void compact(std::uint32_t T, std::uint32_t dst, bool pass, std::uint32_t hsize) {
        const std::uint32_t nw = (T + 31) / 32;
        const std::uint32_t ts0 = c->ts;
        std::int32_t* out = sl.fr(dst);
        std::uint32_t* bsrc = SMEM ? sm.bits() : sl.bitmap();
        const std::int32_t* lat = SMEM ? sm.litat() : sl.litat();
        const std::uint32_t fcap = sm.tcap() ? sm.fcap() : 0;
        unsigned long long carry = 0;
        for (std::uint32_t base = 0; base < nw; base += g.size()) {
            const std::uint32_t wi = base + g.tid();
            const std::uint32_t bits = wi < nw ? bsrc[wi] : 0u;
            unsigned long long occ = 0;
            for (std::uint32_t b = bits; b; b &= b - 1)
                occ += SMEM ? sm.otat()[wi * 32 + __ffs(b) - 1] : occ_total(lidx(lat[wi * 32 + __ffs(b) - 1]));
            const unsigned long long v = (static_cast<unsigned long long>(__popc(bits)) << 32) | occ;
            unsigned long long tot;
            const unsigned long long pre = g.scan(v, tot) + carry;
            std::uint32_t r = static_cast<std::uint32_t>(pre >> 32);
            std::uint32_t o = static_cast<std::uint32_t>(pre);
            for (std::uint32_t b = bits; b; b &= b - 1) {
                const std::int32_t lit = lat[wi * 32 + __ffs(b) - 1];
                out[r] = lit;
                sl.froff()[r] = o;
                if constexpr (G::kGrid) sl.frb()[r] = __ldg(S.occ_off + lidx(lit) * 4);  // grid passes read it
                if (r < fcap) {
                    sm.fr()[r] = lit;
                    sm.froff()[r] = o;
                }
                sl.trail()[ts0 + r] = lit;
                sl.tpos()[atom_of(lit)] = ts0 + r;
                o += SMEM ? sm.otat()[wi * 32 + __ffs(b) - 1] : occ_total(lidx(lit));
                ++r;
            }
            if (bits) bsrc[wi] = 0u;
            carry += tot;
        }
        if (SMEM)
            for (std::uint32_t i = g.tid(); i < hsize; i += g.size()) {
                sm.htab()[i] = 0ull;
                sm.wtab()[i] = 0ull;
            }
        g.sync();
        if (g.leader()) {
            const std::uint32_t cnt = static_cast<std::uint32_t>(carry >> 32);
            sl.froff()[cnt] = static_cast<std::uint32_t>(carry);
            if (cnt + 1 <= fcap) sm.froff()[cnt] = static_cast<std::uint32_t>(carry);
            c->ts = ts0 + cnt;
            c->F = cnt;
            c->T = static_cast<std::uint32_t>(carry);
            c->st.propagations += cnt;
            c->n_props = 0;
            if (pass) {
                c->st.passes += 1;
                c->cur = dst;
                c->b[11] = c->n_confl > 0 ? 1u : 0u;
            }
            c->gen += 1;
        }
        g.sync();
    }

    // Apply proposals: per atom the smallest key wins (newly_set); an opposite
    // loser turns its nogood into a conflict (assignment.cpp:116-124).
    template <bool SMEM>
    __device__ __forceinline__ void apply(std::uint32_t level, bool unit) {
        const std::uint32_t np = c->n_props;
        const std::uint32_t dlev = level > c->cdl ? level : c->cdl;
        for (std::uint32_t base = g.tid() & ~31u; base < np; base += g.size()) {
            const std::uint32_t i = base + lane_id();
            bool lose = false;
            std::int32_t id = 0;
            if (i < np) {
                std::int32_t lit;
                std::uint32_t e;
                unsigned long long w;
                if (SMEM) {
                    id = sm.pid()[i];
                    lit = sm.plit()[i];
                    const std::uint32_t ps = sm.pslot()[i];
                    e = static_cast<std::uint32_t>(sm.htab()[ps & 0xffffu]);
                    w = sm.wtab()[ps >> 16];
                } else {
                    const int4 p = sl.props()[i];
                    id = p.x;
                    lit = p.y;
                    e = static_cast<std::uint32_t>(p.z);
                    w = sl.win()[atom_of(lit)];
                }
                const std::uint32_t a = atom_of(lit);
                if ((static_cast<std::uint32_t>(w) >> 1) == e) {
                    set_cell(a, lit > 0 ? static_cast<std::int32_t>(level) : -static_cast<std::int32_t>(level));
                    if (unit) {
                        sl.reason()[a] = kReasonUnit;
                    } else {
                        sl.reason()[a] = id;
                        if (SMEM && nwords(dlev) == 1) {
                            dep(0, a) = sm.pdep()[i];
                            sl.dovf()[a] = static_cast<std::uint8_t>(sm.pmeta()[i] >> 31);
                        } else {
                            std::uint32_t len;
                            const std::int32_t* L = lits_of(static_cast<std::uint32_t>(id), len);
                            write_deps_from(L, len, static_cast<std::uint32_t>(id), a, dlev);
                        }
                    }
                    if (SMEM) {
                        atomicOr(sm.bits() + (e >> 5), 1u << (e & 31));
                        sm.litat()[e] = lit;
                        sm.otat()[e] = sm.pmeta()[i] & 0x7fffffffu;
                    } else {
                        atomicOr(sl.bitmap() + (e >> 5), 1u << (e & 31));
                        sl.litat()[e] = lit;
                    }
                } else {
                    lose = (w & 1ull) != (lit < 0 ? 1ull : 0ull);
                }
            }
            __syncwarp();
            const std::uint32_t slot = warp_append(&c->n_confl, lose);
            if (lose) sl.confl()[slot] = id;
        }
        g.sync();
    }

    // Evaluate nogood `id` against the pass-start assignment
    // (propagate.cpp:86-168 without the watch shortcuts).
    __device__ __forceinline__ void evaluate(std::int32_t id, bool& conflict, bool& prop, std::int32_t& plit, std::uint32_t& len,
                             unsigned long long* d0 = nullptr, std::uint32_t* meta = nullptr) const {
        const std::uint32_t guard = guard_of(static_cast<std::uint32_t>(id));
        const std::int32_t* L = lits_of(static_cast<std::uint32_t>(id), len);
        if (len == 1) {
            conflict = holds(lit_at(L, 0, static_cast<std::uint32_t>(id)));
            return;
        }
        std::uint32_t nfree = 0;
        std::int32_t u1 = 0;
        bool dead = false;
        if (len <= 8) {  // all literal loads, then all value loads: two round trips
            std::int32_t l[8];
            int v[8];
#pragma unroll
            for (std::uint32_t k = 0; k < 8; ++k) l[k] = k < len ? lit_at(L, k, static_cast<std::uint32_t>(id)) : 0;
#pragma unroll
            for (std::uint32_t k = 0; k < 8; ++k) v[k] = k < len ? val(atom_of(l[k])) : 2;
#pragma unroll
            for (int k = 7; k >= 0; --k) {  // u1 = first free literal in nogood order
                if (v[k] == 0) { ++nfree; u1 = l[k]; }
                else if (v[k] != 2 && (v[k] > 0) != (l[k] > 0)) dead = true;
            }
            if (dead || nfree >= 2) return;
        } else {
            for (std::uint32_t k = 0; k < len; ++k) {
                const std::int32_t l = lit_at(L, k, static_cast<std::uint32_t>(id));
                const int v = val(atom_of(l));
                if (v == 0) {
                    if (nfree == 0) u1 = l;
                    if (++nfree == 2) return;
                } else if ((v > 0) != (l > 0)) {
                    return;  // a dead literal: satisfied
                }
            }
        }
        if (nfree == 0) conflict = true;
        else if (may_assert(guard, -u1)) {
            prop = true;
            plit = -u1;
            if (d0) {
                std::uint8_t ovf = 0;
                *d0 = deps_word(L, len, static_cast<std::uint32_t>(id), atom_of(u1), 0, ovf);
                *meta = occ_total(lidx(plit)) | (static_cast<std::uint32_t>(ovf) << 31);
            }
        }
    }

    // Evaluate the nogood of occurrence entry `ent` (class `cls`) that was
    // triggered by frontier literal `trig` (which holds). Binary and ternary
    // nogoods are decided by the two literals carried in the entry; a long one
    // only when one of them is dead or both are free, else by a full scan.
    __device__ __forceinline__ void evaluate_entry(const int4& ent, std::uint32_t cls, std::int32_t trig, bool& conflict, bool& prop,
                                   std::int32_t& plit, std::uint32_t& len, unsigned long long* d0 = nullptr,
                                   std::uint32_t* meta = nullptr) const {
        if (cls == 0) {  // length-1 entry: its literal is the trigger, which holds
            conflict = true;
            len = 1;
            return;
        }
        const int vx = val(atom_of(ent.z));
        const int sx = vx == 0 ? 0 : ((vx > 0) == (ent.z > 0) ? 1 : -1);  // 1 holds, -1 dead, 0 free
        int sy = 1;
        if (cls >= 2) {
            const int vy = val(atom_of(ent.w));
            sy = vy == 0 ? 0 : ((vy > 0) == (ent.w > 0) ? 1 : -1);
        }
        if (cls == 3) {  // long: three blockers (z, w, y); a dead one or two free ones decide without a scan
            const int vq = val(atom_of(ent.y));
            const int sq = vq == 0 ? 0 : ((vq > 0) == (ent.y > 0) ? 1 : -1);
            const bool decided = sx < 0 || sy < 0 || sq < 0 || (sx == 0) + (sy == 0) + (sq == 0) >= 2;
            if (!decided) {
                evaluate(ent.x, conflict, prop, plit, len, d0, meta);
                return;
            }
            len = C.count_lits ? length_of(static_cast<std::uint32_t>(ent.x)) : 4;
            return;  // satisfied, or two free
        }
        len = cls + 1;
        if (C.count_lits && cls == 3) len = length_of(static_cast<std::uint32_t>(ent.x));
        if (sx < 0 || sy < 0 || (sx == 0 && sy == 0)) return;  // satisfied, or two free
        if (sx > 0 && sy > 0) {
            conflict = true;
            return;
        }
        const std::int32_t u1 = sx == 0 ? ent.z : ent.w;
        if (!may_assert(static_cast<std::uint32_t>(ent.y), -u1)) return;
        prop = true;
        plit = -u1;
        if (d0) {  // Deps of the other (holding) literals: the trigger and, for ternaries, the other blocker
            const std::uint32_t ta = atom_of(trig);
            const std::uint32_t oa = cls == 2 ? atom_of(sx == 0 ? ent.w : ent.z) : ta;
            const std::int32_t ct = sl.cells()[ta], co = sl.cells()[oa];
            const unsigned long long dt = dep(0, ta), dq = dep(0, oa);
            const std::uint8_t ot = sl.dovf()[ta], oo = sl.dovf()[oa];
            unsigned long long acc = 0;
            std::uint32_t ovf = 0;
            if (lvl_of(ct) > 1) { acc |= dt; ovf |= ot; }
            if (lvl_of(co) > 1) { acc |= dq; ovf |= oo; }
            *d0 = acc;
            *meta = occ_total(lidx(plit)) | (ovf << 31);
        }
    }

    // One pass with the working set in shared memory (T <= tcap).
    __device__ __forceinline__ void pass_smem(std::uint32_t F, std::uint32_t T, std::uint32_t cur, std::uint32_t level) {
        const bool learned = c->learned_n > 0;
        std::uint32_t hs = 64;
        while (hs < 2 * T) hs <<= 1;
        if (hs > sm.hmask() + 1) hs = sm.hmask() + 1;
        const std::uint32_t hm = hs - 1;
        for (std::uint32_t base = g.tid() & ~31u; base < T; base += g.size()) {
            const std::uint32_t e = base + lane_id();
            bool first = false, conflict = false, prop = false;
            std::int32_t id = -1, plit = 0;
            std::uint32_t slot = 0, meta = 0, clen = 0;
            unsigned long long d0 = 0;
            if (e < T) {
                std::uint32_t lo = 0, hi = F;
                while (hi - lo > 1) {
                    const std::uint32_t mid = (lo + hi) >> 1;
                    if (sm.froff()[mid] <= e) lo = mid; else hi = mid;
                }
                const std::int32_t trig = sm.fr()[lo];
                std::uint32_t cls;
                const int4 ent = occ_entry(lidx(trig), e - sm.froff()[lo], learned, cls);
                id = ent.x;
                const unsigned long long key = (static_cast<unsigned long long>(id + 1) << 32) | e;
                for (std::uint32_t h = hslot(static_cast<std::uint32_t>(id), hm);; h = (h + 1) & hm) {
                    unsigned long long cur_k = sm.htab()[h];
                    if (cur_k == 0ull) {
                        cur_k = atomicCAS(sm.htab() + h, 0ull, key);
                        if (cur_k == 0ull) { first = true; slot = h; break; }
                    }
                    if ((cur_k >> 32) == static_cast<unsigned long long>(id + 1)) {
                        atomicMin(sm.htab() + h, key);
                        break;
                    }
                }
                if (first) evaluate_entry(ent, cls, trig, conflict, prop, plit, clen, &d0, &meta);
            }
            __syncwarp();
            warp_count(&c->st.checks, first);
            warp_sum(&c->st.checked_lits, clen);
            const std::uint32_t cs = warp_append(&c->n_confl, conflict);
            if (conflict) sl.confl()[cs] = id;
            const std::uint32_t ps = warp_append(&c->n_props, prop);
            if (prop) {
                sm.pid()[ps] = id;
                sm.plit()[ps] = plit;
                sm.pslot()[ps] = slot;
                sm.pdep()[ps] = d0;
                sm.pmeta()[ps] = meta;
            }
        }
        g.sync();
        mark(2);
        const std::uint32_t np = c->n_props;
        for (std::uint32_t i = g.tid(); i < np; i += g.size()) {
            const std::uint32_t e = static_cast<std::uint32_t>(sm.htab()[sm.pslot()[i]]);
            const std::int32_t lit = sm.plit()[i];
            const std::uint32_t a = atom_of(lit);
            const unsigned long long key =
                (static_cast<unsigned long long>(a + 1) << 32) | (static_cast<unsigned long long>(e) << 1) | (lit < 0 ? 1ull : 0ull);
            for (std::uint32_t h = hslot(a, hm);; h = (h + 1) & hm) {
                unsigned long long cur_k = sm.wtab()[h];
                if (cur_k == 0ull) {
                    cur_k = atomicCAS(sm.wtab() + h, 0ull, key);
                    if (cur_k == 0ull) { sm.pslot()[i] |= h << 16; break; }
                }
                if ((cur_k >> 32) == static_cast<unsigned long long>(a + 1)) {
                    atomicMin(sm.wtab() + h, key);
                    sm.pslot()[i] |= h << 16;
                    break;
                }
            }
        }
        g.sync();
        mark(3);
        apply<true>(level, false);
        mark(4);
        compact<true>(T, cur ^ 1u, true, hs);
        mark(5);
    }

    // One pass with the working set in global memory (any size; grid mode).
    __device__ __forceinline__ void pass_global(std::uint32_t F, std::uint32_t T, std::uint32_t gen, std::uint32_t cur,
                                std::uint32_t level) {
        const bool learned = c->learned_n > 0;
        const std::int32_t* fr = sl.fr(cur);
        for (std::uint32_t base = g.tid() & ~31u; base < T; base += g.size()) {
            const std::uint32_t e = base + lane_id();
            bool first = false, conflict = false, prop = false;
            std::int32_t id = -1, plit = 0;
            std::uint32_t clen = 0;
            if (e < T) {
                std::uint32_t lo = 0, hi = F;  // largest p with froff[p] <= e
                while (hi - lo > 1) {
                    const std::uint32_t mid = (lo + hi) >> 1;
                    if (sl.froff()[mid] <= e) lo = mid; else hi = mid;
                }
                const std::int32_t trig = fr[lo];
                std::uint32_t cls;
                const int4 ent = occ_entry(lidx(trig), e - sl.froff()[lo], learned, cls);
                id = ent.x;
                const unsigned long long old = atomicMin(sl.claim() + id, ckey(gen, e));
                first = static_cast<std::uint32_t>(old >> 32) != ~gen;
                if (first) evaluate_entry(ent, cls, trig, conflict, prop, plit, clen);
            }
            __syncwarp();
            warp_count(&c->st.checks, first);
            warp_sum(&c->st.checked_lits, clen);
            const std::uint32_t cs = warp_append(&c->n_confl, conflict);
            if (conflict) sl.confl()[cs] = id;
            const std::uint32_t ps = warp_append(&c->n_props, prop);
            if (prop) sl.props()[ps] = make_int4(id, plit, 0, 0);
        }
        g.sync();
        mark(2);
        // resolve: final min-e of every proposing nogood, atomicMin per atom
        const std::uint32_t np = c->n_props;
        for (std::uint32_t i = g.tid(); i < np; i += g.size()) {
            int4 p = sl.props()[i];
            const std::uint32_t e = static_cast<std::uint32_t>(sl.claim()[p.x]);
            p.z = static_cast<std::int32_t>(e);
            sl.props()[i] = p;
            atomicMin(sl.win() + atom_of(p.y), wkey(gen, e, p.y < 0));
        }
        g.sync();
        mark(3);
        apply<false>(level, false);
        mark(4);
        compact<false>(T, cur ^ 1u, true, 0);
        mark(5);
    }

    // ---- whole-grid passes (GridG) ---------------------------------------------
    // A pass costs four grid barriers: expand+evaluate | resolve | select the
    // winners + scan | place them. Every block keeps the loop state (F, T, gen,
    // frontier buffer, trail size) in registers; the pass's conflict count is
    // exchanged with the scan, so no block reads a counter another block may
    // already be bumping for the next pass.

    // Expansion entries e in [0, T) are split into one contiguous range per
    // warp. A warp locates the frontier literal of its first entry with a
    // 32-ary search, then walks: per batch of 32*U entries it loads the next 32
    // frontier offsets once and every lane finds its trigger with five register
    // shuffles. U independent entries per lane keep U gathers, U claim atomics
    // and their cell lookups in flight at once.
    // Full scan of nogood `id` against the pass snapshot (propagate.cpp:86-168
    // without watches): literals, then their values, each as one batch of
    // independent loads.
    __device__ __forceinline__ void scan_snap(std::int32_t id, bool& conflict, bool& prop, std::int32_t& plit, std::uint32_t& len) const {
        const std::uint32_t guard = guard_of(static_cast<std::uint32_t>(id));
        const std::int32_t* L = lits_of(static_cast<std::uint32_t>(id), len);
        std::uint32_t nfree = 0;
        std::int32_t u1 = 0;
        for (std::uint32_t k0 = 0; k0 < len; k0 += 8) {
            std::int32_t l[8];
            std::uint32_t w[8];
#pragma unroll
            for (std::uint32_t k = 0; k < 8; ++k) l[k] = k0 + k < len ? lit_at(L, k0 + k, static_cast<std::uint32_t>(id)) : 0;
#pragma unroll
            for (std::uint32_t k = 0; k < 8; ++k) w[k] = mirror_word_snap(atom_of(l[k]));
#pragma unroll
            for (std::uint32_t k = 0; k < 8; ++k) {
                if (k0 + k >= len) break;
                const int v = mirror_val(w[k], atom_of(l[k]));
                if (v == 0) {
                    if (nfree == 0) u1 = l[k];
                    ++nfree;
                } else if ((v > 0) != (l[k] > 0)) {
                    return;  // a dead literal: satisfied
                }
            }
            if (nfree >= 2) return;
        }
        if (nfree == 0) conflict = true;
        else if (may_assert(guard, -u1)) {
            prop = true;
            plit = -u1;
        }
    }

    // Expansion entries e in [0, T) are split into one contiguous range per
    // warp (warps numbered block-interleaved). A warp locates the frontier
    // literal of its first entry with a 32-ary search, then walks: per batch
    // of 32*U entries it loads the next 32 frontier offsets once and every
    // lane finds its trigger with five register shuffles. The U entries of a
    // lane are processed in lock step — gathers, claim atomics and the value
    // loads of the two literals carried in the entry are all issued before
    // any of them is used — and the few long nogoods the entry cannot decide
    // are compacted over the warp's lanes for one batched full scan.
    static constexpr int kExpandU = 8;

    template <int U>
    __device__ __forceinline__ void grid_expand(std::uint32_t F, std::uint32_t T, std::uint32_t cur, std::uint32_t gen, bool learned,
                                std::uint32_t pass = 0xffffffffu) {
        dstamp(pass, 0);
        const std::int32_t* fr = sl.fr(cur);
        const std::uint32_t* froff = sl.froff();
        const std::uint32_t lane = lane_id();
        const unsigned below = (1u << lane) - 1u;
        std::int32_t* scanq = g.scanq + (threadIdx.x >> 5) * (32 * U);
        std::uint32_t* scane = g.scane + (threadIdx.x >> 5) * (32 * U);
        const std::uint32_t nwarps = g.size() >> 5, wid = g.iwarp();
        const std::uint32_t per = (((T + nwarps - 1) / nwarps) + 31u) & ~31u;
        const unsigned long long start64 = static_cast<unsigned long long>(wid) * per;
        std::uint32_t checks = 0, lits = 0;
        if (start64 < T) {
            const std::uint32_t start = static_cast<std::uint32_t>(start64);
            const std::uint32_t end = T - start < per ? T : start + per;
            // froff[lo] <= start < froff[hi] = T; the first range starts at 0
            // (froff[0] = 0): the window walk copes with empty lists there
            std::uint32_t lo = 0, hi = start == 0 ? 1u : F;
            while (hi - lo > 1) {
                const std::uint32_t step = (hi - lo + 31u) >> 5;
                const std::uint32_t idx = lo + lane * step;
                const bool ok = idx < hi && froff[idx] <= start;
                const unsigned b = __ballot_sync(0xffffffffu, ok);
                lo += static_cast<std::uint32_t>(31 - __clz(b)) * step;
                hi = min(hi, lo + step);
            }
            std::uint32_t p0 = lo, f0 = lo == 0 ? 0u : froff[lo];
            dstamp(pass, 1);
            for (std::uint32_t base = start; base < end; base += 32u * U) {
                const std::uint32_t q = p0 + 1 + lane;
                const std::uint32_t v = q <= F ? froff[q] : 0xffffffffu;
                const bool narrow = __shfl_sync(0xffffffffu, v, 31) <= base + 32u * U - 1;
                std::uint32_t pe[U], se[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const std::uint32_t e = base + 32u * u + lane;
                    if (!narrow) {
                        std::uint32_t cnt = 0;
#pragma unroll
                        for (int st = 16; st >= 1; st >>= 1)
                            if (__shfl_sync(0xffffffffu, v, cnt + st - 1) <= e) cnt += st;
                        const std::uint32_t sv = __shfl_sync(0xffffffffu, v, cnt == 0 ? 0 : cnt - 1);
                        pe[u] = p0 + cnt;
                        se[u] = cnt == 0 ? f0 : sv;
                    } else {  // many empty occurrence lists inside the batch: per-lane search
                        std::uint32_t l2 = p0, h2 = F;
                        if (e < T)
                            while (h2 - l2 > 1) {
                                const std::uint32_t m = (l2 + h2) >> 1;
                                if (froff[m] <= e) l2 = m; else h2 = m;
                            }
                        pe[u] = l2;
                        se[u] = froff[l2];
                    }
                }
                if (base == start) dstamp(pass, 2);
                std::int32_t trig[U];
                std::uint32_t fb[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const bool in = base + 32u * u + lane < end;
                    trig[u] = in ? fr[pe[u]] : 0;
                    fb[u] = in ? sl.frb()[pe[u]] : 0u;  // static list base, stored with the frontier
                }
                int4 ent[U];
                std::uint32_t cls[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const std::uint32_t e = base + 32u * u + lane;
                    cls[u] = 0;
                    if (e >= end) ent[u] = make_int4(-1, 0, 0, 0);
                    else if (!learned) ent[u] = decode(U == kExpandU ? ld_stream(S.occ + fb[u] + (e - se[u]), S.pol_first)
                                                                    : __ldg(S.occ + fb[u] + (e - se[u])),
                                                       cls[u]);
                    else ent[u] = occ_entry(lidx(trig[u]), e - se[u], learned, cls[u]);
                }
                if (base == start) { asm volatile("" ::"r"(ent[0].x)); dstamp(pass, 3); }
                unsigned long long old[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const std::uint32_t e = base + 32u * u + lane;
                    old[u] = e < end ? (U == kExpandU ? atomic_min_keep(sl.claim() + ent[u].x, ckey(gen, e), S.pol_last)
                                                      : atomicMin(sl.claim() + ent[u].x, ckey(gen, e))) : ckey(gen, 0);
                }
                std::uint32_t wx[U], wy[U];  // issued while the claims are in flight
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    wx[u] = mirror_word_snap(cls[u] >= 1 ? atom_of(ent[u].z) : 0u);
                    wy[u] = mirror_word_snap(cls[u] >= 2 ? atom_of(ent[u].w) : 0u);
                }
                // An occurrence evaluates its nogood (same outcome from any of
                // them) unless an occurrence with a smaller e already claimed
                // it, and every proposing evaluation bids its own e for the
                // atom: the nogood's min-e occurrence always evaluates, so the
                // smallest bid is the item-order winner without a separate
                // resolve phase. The first toucher counts the check and reports
                // an all-true conflict.
                // decide from the entry first (values only), while the claims
                // are still in flight: 0 nothing, 1 all true, 2 proposal, 3 full scan
                std::uint32_t stt[U];
                std::int32_t plit[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    plit[u] = 0;
                    stt[u] = 0;
                    if (base + 32u * u + lane >= end) continue;
                    if (cls[u] == 0) { stt[u] = 1; continue; }
                    const int vx = mirror_val(wx[u], atom_of(ent[u].z));
                    const int sx = vx == 0 ? 0 : ((vx > 0) == (ent[u].z > 0) ? 1 : -1);  // 1 holds, -1 dead, 0 free
                    int sy = 1;
                    if (cls[u] >= 2) {
                        const int vy = mirror_val(wy[u], atom_of(ent[u].w));
                        sy = vy == 0 ? 0 : ((vy > 0) == (ent[u].w > 0) ? 1 : -1);
                    }
                    const bool decided = sx < 0 || sy < 0 || (sx == 0 && sy == 0);
                    if (cls[u] == 3) {  // long, not decided by its first two blockers: look at the third
                        if (!decided) stt[u] = 4 | (sx == 0 || sy == 0 ? 8u : 0u);  // bit 3: one of them is free
                        continue;
                    }
                    if (decided) continue;
                    if (sx > 0 && sy > 0) { stt[u] = 1; continue; }
                    const std::int32_t u1 = sx == 0 ? ent[u].z : ent[u].w;
                    if (may_assert(static_cast<std::uint32_t>(ent[u].y), -u1)) { stt[u] = 2; plit[u] = -u1; }
                }
                // long nogoods still open after two blockers: the third blocker
                // (one more mirror lookup) settles most of them without a scan
                {
                    std::uint32_t wq[U];
#pragma unroll
                    for (int u = 0; u < U; ++u) wq[u] = (stt[u] & 4u) ? mirror_word_snap(atom_of(ent[u].y)) : 0u;
#pragma unroll
                    for (int u = 0; u < U; ++u) {
                        if (!(stt[u] & 4u)) continue;
                        const int vq = mirror_val(wq[u], atom_of(ent[u].y));
                        const bool dead = vq != 0 && ((vq > 0) != (ent[u].y > 0));
                        const bool two_free = vq == 0 && (stt[u] & 8u);
                        stt[u] = dead || two_free ? 0u : 3u;
                    }
                }
                // An occurrence acts on its nogood (same outcome from any of
                // them) unless an occurrence with a smaller e already claimed
                // it, and every proposing occurrence bids its own e for the
                // atom: the nogood's min-e occurrence always acts, so the
                // smallest bid is the item-order winner without a separate
                // resolve phase. The first toucher counts the check and reports
                // an all-true conflict.
                if (base == start) { asm volatile("" ::"l"(old[0]), "r"(wx[0])); dstamp(pass, 4); }
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const std::uint32_t e = base + 32u * u + lane;
                    const bool first = e < end && static_cast<std::uint32_t>(old[u] >> 32) != ~gen;
                    const bool evl = first || e < static_cast<std::uint32_t>(old[u]);
                    if (first) {
                        ++checks;
                        if (stt[u] != 3)
                            lits += (cls[u] == 3 && C.count_lits) ? length_of(static_cast<std::uint32_t>(ent[u].x)) : cls[u] + 1;
                    }
                    if (stt[u] == 1 && !first) stt[u] = 0;       // conflicts: reported once
                    if ((stt[u] == 2 || stt[u] == 3) && !evl) stt[u] = 0;
                    if (stt[u] == 3 && first) stt[u] = 7;        // the scan remembers first-ness
                }
                unsigned cm[U], pm[U], qm[U];
                std::uint32_t nprop = 0, nscan = 0;
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    cm[u] = __ballot_sync(0xffffffffu, stt[u] == 1);
                    pm[u] = __ballot_sync(0xffffffffu, stt[u] == 2);
                    qm[u] = __ballot_sync(0xffffffffu, (stt[u] & 3u) == 3u);
                    nprop += __popc(pm[u]);
                    nscan += __popc(qm[u]);
                    if (cm[u]) {  // rare
                        std::uint32_t at = 0;
                        if (lane == 0) at = atomicAdd(&c->n_confl, static_cast<std::uint32_t>(__popc(cm[u])));
                        at = __shfl_sync(0xffffffffu, at, 0);
                        if (cm[u] >> lane & 1u) sl.confl()[at + __popc(cm[u] & below)] = ent[u].x;
                    }
                }
                if (base == start) dstamp(pass, 5);
                if (nprop) {  // one reservation per batch for all its proposals
                    std::uint32_t at = 0;
                    if (lane == 0) at = atomicAdd(&c->n_props, nprop);
                    at = __shfl_sync(0xffffffffu, at, 0);
#pragma unroll
                    for (int u = 0; u < U; ++u) {
                        if (pm[u] >> lane & 1u) {
                            const std::uint32_t e = base + 32u * u + lane;
                            atomicMin(sl.win() + atom_of(plit[u]), wkey(gen, e, plit[u] < 0));
                            sl.props()[at + __popc(pm[u] & below)] =
                                make_int4(ent[u].x, plit[u], static_cast<std::int32_t>(e), 0);
                        }
                        at += __popc(pm[u]);
                    }
                }
                if (base == start) dstamp(pass, 6);
                if (nscan) {  // long nogoods the entry could not decide: one lane each
                    std::uint32_t at = 0;
#pragma unroll
                    for (int u = 0; u < U; ++u) {
                        if (qm[u] >> lane & 1u) {
                            const std::uint32_t q = at + __popc(qm[u] & below);
                            scanq[q] = ent[u].x | ((stt[u] & 4u) ? static_cast<std::int32_t>(0x80000000u) : 0);
                            scane[q] = base + 32u * u + lane;
                        }
                        at += __popc(qm[u]);
                    }
                    __syncwarp();
                    for (std::uint32_t r = 0; r < nscan; r += 32) {
                        bool conflict = false, prop = false;
                        std::int32_t pl = 0, id = 0;
                        std::uint32_t e = 0;
                        if (r + lane < nscan) {
                            const std::int32_t qv = scanq[r + lane];
                            const bool fst = qv < 0;
                            id = qv & 0x7fffffff;
                            e = scane[r + lane];
                            std::uint32_t len = 0;
                            scan_snap(id, conflict, prop, pl, len);
                            if (fst) lits += len;
                            conflict = conflict && fst;
                            if (prop) atomicMin(sl.win() + atom_of(pl), wkey(gen, e, pl < 0));
                        }
                        const std::uint32_t cs = warp_append(&c->n_confl, conflict);
                        if (conflict) sl.confl()[cs] = id;
                        const std::uint32_t ps = warp_append(&c->n_props, prop);
                        if (prop) sl.props()[ps] = make_int4(id, pl, static_cast<std::int32_t>(e), 0);
                    }
                    __syncwarp();
                }
                if (base == start) dstamp(pass, 7);
                p0 = __shfl_sync(0xffffffffu, pe[U - 1], 31);
                f0 = __shfl_sync(0xffffffffu, se[U - 1], 31);
            }
        }
        dstamp(pass, 8);
        checks = __reduce_add_sync(0xffffffffu, checks);
        lits = __reduce_add_sync(0xffffffffu, lits);
        if (lane == 0) {
            if (checks) atomicAdd(g.bc + 0, static_cast<unsigned long long>(checks));
            if (lits) atomicAdd(g.bc + 2, static_cast<unsigned long long>(lits));
        }
    }

    // Per proposal: the winner of its atom assigns it (cell, reason, Deps),
    // records literal and occurrence count at its e and marks e in the
    // expansion bitmap; an opposite-sign loser turns its nogood into a
    // conflict (assignment.cpp:116-124).
    __device__ __forceinline__ void grid_select(std::uint32_t level, std::uint32_t dlev, std::uint32_t np) {
        const int4* props = sl.props();
        const bool one_word = nwords(dlev) == 1;
        for (std::uint32_t i = g.itid(); i < np; i += g.size()) {
            const int4 p = props[i];
            const std::uint32_t e = static_cast<std::uint32_t>(p.z);
            const std::uint32_t a = atom_of(p.y);
            const std::uint32_t id = static_cast<std::uint32_t>(p.x);
            // everything that depends only on the proposal, in one round trip
            const unsigned long long w = sl.win()[a];
            const std::uint32_t li = lidx(p.y);
            const std::uint32_t ob = __ldg(S.occ_off + li * 4), oe = __ldg(S.occ_off + li * 4 + 4), lt = sl.ltot()[li];
            std::uint32_t len;
            const std::int32_t* L = lits_of(id, len);
            if ((static_cast<std::uint32_t>(w) >> 1) == e) {
                set_cell(a, p.y > 0 ? static_cast<std::int32_t>(level) : -static_cast<std::int32_t>(level));
                sl.reason()[a] = p.x;
                if (one_word && len <= 8) {  // literals, then their cells / Deps / overflow: two round trips
                    std::int32_t l[8];
#pragma unroll
                    for (std::uint32_t k = 0; k < 8; ++k) l[k] = k < len ? lit_at(L, k, id) : 0;
                    std::int32_t cv[8];
                    unsigned long long dv[8];
                    std::uint8_t ov[8];
#pragma unroll
                    for (std::uint32_t k = 0; k < 8; ++k) {
                        const std::uint32_t x = atom_of(l[k]);
                        cv[k] = sl.cells()[x];
                        dv[k] = dep(0, x);
                        ov[k] = sl.dovf()[x];
                    }
                    unsigned long long acc = 0;
                    std::uint8_t ovf = 0;
#pragma unroll
                    for (std::uint32_t k = 0; k < 8; ++k)
                        if (k < len && atom_of(l[k]) != a && lvl_of(cv[k]) > 1) {
                            acc |= dv[k];
                            ovf |= ov[k];
                        }
                    dep(0, a) = acc;
                    sl.dovf()[a] = ovf;
                } else {
                    write_deps_from(L, len, id, a, dlev);
                }
                sl.occat()[e] = oe - ob + lt;
                sl.obat()[e] = ob;
                sl.litat()[e] = p.y;
                atomicOr(sl.bitmap() + (e >> 5), 1u << (e & 31));
            } else if ((w & 1ull) != (p.y < 0 ? 1ull : 0ull) && static_cast<std::uint32_t>(sl.claim()[id]) == e) {
                sl.confl()[atomicAdd(&c->n_confl, 1u)] = p.x;  // once per nogood: its min-e occurrence
            }
        }
    }

    // Largest lane w with key[w] <= x, key non-decreasing over the lanes and
    // key[0] <= x (five register shuffles).
    __device__ __forceinline__ static std::uint32_t lane_search(std::uint32_t key, std::uint32_t x) {
        std::uint32_t w = 0;
#pragma unroll
        for (int st = 16; st >= 1; st >>= 1)
            if (__shfl_sync(0xffffffffu, key, w + st) <= x) w += st;
        return w;
    }

    // Winner count and occurrence sum of bitmap word wi (the 32 occurrence
    // counts of a word are one aligned 128-byte line: eight vector loads).
    __device__ __forceinline__ unsigned long long word_value(std::uint32_t wi, std::uint32_t bits) const {
        if (!bits) return 0ull;
        const uint4* line = reinterpret_cast<const uint4*>(sl.occat() + static_cast<std::size_t>(wi) * 32);
        uint4 q[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) q[k] = line[k];
        std::uint32_t occ = 0;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            occ += (bits >> (4 * k) & 1u) ? q[k].x : 0u;
            occ += (bits >> (4 * k + 1) & 1u) ? q[k].y : 0u;
            occ += (bits >> (4 * k + 2) & 1u) ? q[k].z : 0u;
            occ += (bits >> (4 * k + 3) & 1u) ? q[k].w : 0u;
        }
        return (static_cast<unsigned long long>(__popc(bits)) << 32) | occ;
    }

    // Place the winners of this warp's 32 words (lane = word, `bits`), given
    // each word's exclusive (count, occurrence) prefix `pre`: the set bits are
    // dealt to the lanes 32 at a time in e order; a segmented lane scan gives
    // each winner its occurrence offset inside its word.
    __device__ __forceinline__ void place_words(std::uint32_t wi, std::uint32_t bits, unsigned long long pre, std::int32_t* out,
                                std::uint32_t ts0) {
        const std::uint32_t lane = lane_id();
        const std::uint32_t w0 = wi - lane;
        std::uint32_t inc = __popc(bits);
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const std::uint32_t o = __shfl_up_sync(0xffffffffu, inc, d);
            if (lane >= static_cast<std::uint32_t>(d)) inc += o;
        }
        const std::uint32_t exb = inc - __popc(bits);
        const std::uint32_t total = __shfl_sync(0xffffffffu, inc, 31);
        const std::uint32_t r0 = static_cast<std::uint32_t>(pre >> 32), o0 = static_cast<std::uint32_t>(pre);
        std::uint32_t carry_w = 0xffffffffu, carry_s = 0;
        for (std::uint32_t ch = 0; ch < total; ch += 32) {
            const std::uint32_t idx = ch + lane;
            const std::uint32_t w = lane_search(exb, idx);
            const std::uint32_t bw = __shfl_sync(0xffffffffu, bits, w);
            const std::uint32_t ew = __shfl_sync(0xffffffffu, exb, w);
            const std::uint32_t rw = __shfl_sync(0xffffffffu, r0, w);
            const std::uint32_t ow = __shfl_sync(0xffffffffu, o0, w);
            const bool valid = idx < total;
            const std::uint32_t k = idx - ew;
            const std::uint32_t e = (w0 + w) * 32 + (valid ? __fns(bw, 0, static_cast<int>(k + 1)) : 0u);
            const std::int32_t lit = valid ? sl.litat()[e] : 0;
            const std::uint32_t occv = valid ? sl.occat()[e] : 0u;
            const std::uint32_t ob = valid ? sl.obat()[e] : 0u;
            std::uint32_t x = occv;  // segmented inclusive scan by word
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const std::uint32_t y = __shfl_up_sync(0xffffffffu, x, d);
                const std::uint32_t wd = __shfl_up_sync(0xffffffffu, w, d);
                if (lane >= static_cast<std::uint32_t>(d) && wd == w) x += y;
            }
            if (w == carry_w) x += carry_s;
            if (valid) {
                const std::uint32_t r = rw + k;
                out[r] = lit;
                sl.frb()[r] = ob;
                sl.froff()[r] = ow + x - occv;
                sl.trail()[ts0 + r] = lit;
                sl.tpos()[atom_of(lit)] = ts0 + r;
            }
            carry_w = __shfl_sync(0xffffffffu, w, 31);
            carry_s = __shfl_sync(0xffffffffu, x, 31);
        }
    }

    // Winners, in e order, become the next frontier. Small passes are placed
    // by block 0 alone with block scans (no grid barrier); large ones by the
    // whole grid, one grid scan per round of words.
#ifndef YAS_BPW
#define YAS_BPW 512  // measured: 512 words 0.282 ms vs 2048 words 0.288 ms per call
#endif
    static constexpr std::uint32_t kBlockPlaceWords = YAS_BPW;

    __device__ __forceinline__ void grid_place(std::uint32_t T, std::uint32_t dst, std::uint32_t ts0, std::uint32_t& F_next,
                               std::uint32_t& T_next) {
        const std::uint32_t nw = (T + 31) / 32;
        std::int32_t* out = sl.fr(dst);
        std::uint32_t* bmp = sl.bitmap();
        unsigned long long carry = 0;
        if (nw <= kBlockPlaceWords) {
            if (blockIdx.x == 0) {
                for (std::uint32_t base = 0; base < nw; base += blockDim.x) {
                    const std::uint32_t wi = base + threadIdx.x;
                    const std::uint32_t bits = wi < nw ? bmp[wi] : 0u;
                    if (bits) bmp[wi] = 0u;
                    unsigned long long tot;
                    const unsigned long long pre = g.block_scan(word_value(wi, bits), tot) + carry;
                    place_words(wi, bits, pre, out, ts0);
                    carry += tot;
                }
                F_next = static_cast<std::uint32_t>(carry >> 32);
                T_next = static_cast<std::uint32_t>(carry);
                if (threadIdx.x == 0) {
                    sl.froff()[F_next] = T_next;
                    c->F = F_next;
                    c->T = T_next;
                }
            }
            return;  // other blocks read F, T after the pass barrier
        }
        for (std::uint32_t base = 0; base < nw; base += g.size()) {
            const std::uint32_t wi = base + g.tid();
            const std::uint32_t bits = wi < nw ? bmp[wi] : 0u;
            if (bits) bmp[wi] = 0u;
            unsigned long long tot;
            const unsigned long long pre = g.scan(word_value(wi, bits), tot) + carry;
            place_words(wi, bits, pre, out, ts0);
            carry += tot;
        }
        F_next = static_cast<std::uint32_t>(carry >> 32);
        T_next = static_cast<std::uint32_t>(carry);
        if (g.leader()) sl.froff()[F_next] = T_next;
    }

    // One grid pass (expand+evaluate | select | place). In solo mode block 0
    // runs it alone with block barriers. Returns the conflict count.
    __device__ __forceinline__ std::uint32_t grid_pass(std::uint32_t& F, std::uint32_t& T, std::uint32_t& cur, std::uint32_t& gen,
                                       std::uint32_t& ts, std::uint32_t level, std::uint32_t dlev, bool learned,
                                       std::uint32_t& pass) {
        stamp(pass, 0);
        // few entries per warp: short batches; many: eight per lane in flight
        if (T <= 64u * (g.size() >> 5)) grid_expand<2>(F, T, cur, gen, learned, pass);
        else grid_expand<kExpandU>(F, T, cur, gen, learned, pass);
        stamp(pass, 1);
        g.sync_snap(&c->n_props, nullptr);
        const std::uint32_t np = g.snap[0];
        stamp(pass, 2);
        stamp(pass, 3);
        stamp(pass, 4);
        std::uint32_t nconf = 0, Fn = 0, Tn = 0;
        const bool small = (T + 31) / 32 <= kBlockPlaceWords;
#ifdef YAS_NO_FUSED_SELECT
        constexpr bool kFuse = false;
#else
        constexpr bool kFuse = true;
#endif
#ifndef YAS_FUSE_NP
#define YAS_FUSE_NP 1  // proposals per thread of block 0 (4a: 1.449 / 1.464 / 1.502 ms at 1 / 2 / 4)
#endif
        if (kFuse && small && np <= static_cast<std::uint32_t>(G::kWarps * 32 * YAS_FUSE_NP)) {
            // few proposals: block 0 selects (one per thread) and places them
            // with block barriers; the grid waits at the pass barrier
            if (blockIdx.x == 0) {
                g.solo = true;
                grid_select(level, dlev, np);
                stamp(pass, 5);
                __syncthreads();  // select's writes (bitmap, occat, ...) seen by the block
                stamp(pass, 6);
                grid_place(T, cur ^ 1u, ts, Fn, Tn);
                g.solo = false;
                if (threadIdx.x == 0) {
                    c->n_props = 0;
                    c->st.passes += 1;
                }
            }
            stamp(pass, 7);
            g.sync_snap(&c->F, &c->T, &c->n_confl);
            Fn = g.snap[0];
            Tn = g.snap[1];
            nconf = g.snap[2];
        } else {
            grid_select(level, dlev, np);
            stamp(pass, 5);
            g.sync_snap(&c->n_confl, nullptr);
            stamp(pass, 6);
            // final for this pass: no block bumps it before the pass barrier
            nconf = g.snap[0];
            grid_place(T, cur ^ 1u, ts, Fn, Tn);
            if (g.leader()) {
                c->n_props = 0;  // every block read it before the select barrier
                c->st.passes += 1;
            }
            stamp(pass, 7);
            if (small) {
                g.sync_snap(&c->F, &c->T);
                Fn = g.snap[0];
                Tn = g.snap[1];
            } else {
                g.sync();
            }
        }
        stamp(pass, 8);
        if (C.ptrace && g.leader() && pass < kPtracePasses)
            C.ptrace[(static_cast<std::size_t>(pass) * gridDim.x) * kPtraceStamps + 9] =
                (static_cast<unsigned long long>(T) << 32) | F;
        ++pass;
        if (g.leader()) c->st.propagations += Fn;
        ts += Fn;
        F = Fn;
        T = Tn;
        cur ^= 1u;
        gen += 1;
        return nconf;
    }

    __device__ __forceinline__ bool propagate_grid(std::uint32_t level) {
        frontier_offsets();
        std::uint32_t F = c->F, T = c->T, gen = c->gen, cur = c->cur, ts = c->ts;
        const std::uint32_t dlev = level > c->cdl ? level : c->cdl;
        const bool learned = c->learned_n > 0;
        if (threadIdx.x < 4) g.bc[threadIdx.x] = 0;
        __syncthreads();
        bool violated = false;
        std::uint32_t pass = 0;
        while (F != 0) {
            if (T <= sm.tcap() && F + 1 <= sm.fcap()) {
                // Narrow passes: block 0 alone runs the single-CTA pass with its
                // working set in shared memory (claims / winners in hash tables, block
                // barriers) while the other blocks wait at one grid barrier.
                if (blockIdx.x == 0) {
                    g.solo = true;
                    const std::int32_t* fsrc = sl.fr(cur);
                    for (std::uint32_t p = threadIdx.x; p < F; p += blockDim.x) {
                        sm.fr()[p] = fsrc[p];
                        sm.froff()[p] = sl.froff()[p];
                    }
                    if (threadIdx.x == 0) {
                        sm.froff()[F] = T;
                        c->F = F;
                        c->T = T;
                        c->cur = cur;
                        c->gen = gen;
                        c->ts = ts;
                        c->n_props = 0;
                        c->b[11] = 0;
                    }
                    __syncthreads();
                    while (F != 0 && !violated && T <= sm.tcap() && F + 1 <= sm.fcap()) {
                        pass_smem(F, T, cur, level);  // ends with a block barrier; the leader updated c
                        F = c->F;
                        T = c->T;
                        cur = c->cur;
                        violated = c->b[11] != 0;
                        ++pass;
                    }
                    gen = c->gen;
                    ts = c->ts;
                    g.solo = false;
                    if (threadIdx.x == 0) {
                        c->F = F;
                        c->T = T;
                        c->cur = cur;
                        c->gen = gen;
                        c->ts = ts;
                        c->b[11] = violated ? 1u : 0u;
                        c->b[13] = pass;
                    }
                }
                g.sync();  // the other blocks wait here for the solo streak
                F = *reinterpret_cast<volatile std::uint32_t*>(&c->F);
                T = *reinterpret_cast<volatile std::uint32_t*>(&c->T);
                cur = *reinterpret_cast<volatile std::uint32_t*>(&c->cur);
                gen = *reinterpret_cast<volatile std::uint32_t*>(&c->gen);
                ts = *reinterpret_cast<volatile std::uint32_t*>(&c->ts);
                violated = *reinterpret_cast<volatile std::uint32_t*>(&c->b[11]) != 0;
                pass = *reinterpret_cast<volatile std::uint32_t*>(&c->b[13]);
                if (violated) break;
                continue;
            }
            if (grid_pass(F, T, cur, gen, ts, level, dlev, learned, pass)) {
                violated = true;
                break;
            }
        }
        if (threadIdx.x == 0) {
            atomicAdd(&c->st.checks, g.bc[0]);
            if (g.bc[2]) atomicAdd(&c->st.checked_lits, g.bc[2]);
        }
        g.sync();
        if (g.leader()) {
            c->F = F;
            c->T = T;
            c->cur = cur;
            c->gen = gen;
            c->ts = ts;
            c->b[11] = violated ? 1u : 0u;
        }
        g.sync();
        return violated;
    }

    // One propagation call to fixpoint or violation (propagate.cpp:170-205).
    // Returns true when conflicts were found (they are in confl[0..n_confl)).
    // passes this small run in warp 0 alone (C.warp_pass_t: larger when other
    // searches share the SM and keep it busy while the CTA's other warps wait)

    __device__ __forceinline__ bool propagate(std::uint32_t level) {
        if constexpr (G::kGrid) return propagate_grid(level);
        mark(0);
        frontier_offsets();
        for (;;) {
            const std::uint32_t F = c->F, T = c->T, gen = c->gen, cur = c->cur, viol = c->b[11];
            if (viol) return true;
            if (F == 0) return false;
            if constexpr (G::kBlock) {
                if (T <= C.warp_pass_t && T <= sm.tcap() && F + 1 <= sm.fcap()) {
                    if (threadIdx.x < 32) {
                        WarpG<G::kLean> wg{c};
                        Search<WarpG<G::kLean>> ws(wg, S, C, sl, K, sh, t0, sm);
                        ws.small_passes(level);
                    }
                    g.sync();
                    continue;
                }
            }
            const bool in_smem = sm.tcap() && T <= sm.tcap() && F + 1 <= sm.fcap();
            if (prof_on() && g.leader()) c->prof[in_smem ? 12 : 13] += 1;  // pass counts by path
            if (in_smem) pass_smem(F, T, cur, level);
            else pass_global(F, T, gen, cur, level);
        }
    }

    // Warp-synchronous passes while they stay small (called by warp 0 only).
    __device__ __forceinline__ void small_passes(std::uint32_t level) {
        for (;;) {
            __syncwarp();
            const std::uint32_t F = c->F, T = c->T, cur = c->cur, viol = c->b[11];
            __syncwarp();
            if (viol || F == 0 || T > C.warp_pass_t || T > sm.tcap() || F + 1 > sm.fcap()) return;
            if (T <= 32) {
                tiny_pass(F, T, cur, level);
                mark(8);
                if (prof_on() && threadIdx.x == 0) c->prof[10] += 1;
            } else {
                pass_smem(F, T, cur, level);
                mark(9);
            }
        }
    }

    // evaluate() of one nogood by the whole warp (results uniform): 32
    // literals per step, free/dead detection by ballot, Deps word 0 of the
    // proposal by OR-reduction (propagate.cpp:86-168, :49-62).
    __device__ __forceinline__ void w_evaluate(std::uint32_t id, bool& conflict, bool& prop, std::int32_t& plit, std::uint32_t& len,
                               unsigned long long& d0, std::uint32_t& meta) const {
        const std::uint32_t lane = lane_id();
        const std::uint32_t guard = guard_of(id);
        const std::int32_t* L = lits_of(id, len);
        conflict = prop = false;
        plit = 0;
        d0 = 0;
        meta = 0;
        std::uint32_t nfree = 0;
        std::int32_t u1 = 0;
        for (std::uint32_t k0 = 0; k0 < len; k0 += 32) {
            const std::uint32_t k = k0 + lane;
            const std::int32_t l = k < len ? lit_at(L, k, id) : 0;
            const int v = k < len ? val(atom_of(l)) : 1;
            if (__any_sync(0xffffffffu, k < len && v != 0 && (v > 0) != (l > 0))) return;  // satisfied
            const unsigned fm = __ballot_sync(0xffffffffu, k < len && v == 0);
            if (fm && nfree == 0) u1 = __shfl_sync(0xffffffffu, l, __ffs(fm) - 1);
            nfree += __popc(fm);
            if (nfree >= 2) return;
        }
        if (nfree == 0) {
            conflict = true;
            return;
        }
        if (!may_assert(guard, -u1)) return;
        prop = true;
        plit = -u1;
        const std::uint32_t ua = atom_of(u1);
        unsigned long long acc = 0;
        std::uint32_t ov = 0;
        for (std::uint32_t k = lane; k < len; k += 32) {
            const std::uint32_t x = atom_of(lit_at(L, k, id));
            if (x == ua || lvl_of(sl.cells()[x]) <= 1) continue;
            acc |= dep(0, x);
            ov |= sl.dovf()[x];
        }
        d0 = w_or64(acc);
        ov = __reduce_or_sync(0xffffffffu, ov);
        meta = occ_total(lidx(plit)) | (ov ? 0x80000000u : 0u);
    }

    // A whole pass with one expansion entry per lane (T <= 32; warp 0 of a
    // single-CTA search). Register-level replacements for the shared-memory
    // machinery of pass_smem: duplicate nogoods by __match_any_sync on the id
    // (the lowest lane has the smallest e, i.e. comes first in item order),
    // per-atom winners by __match_any_sync on the proposed atom (lowest lane =
    // smallest key), positions by ballot prefix counts and one warp scan.
    __device__ __forceinline__ void tiny_pass(std::uint32_t F, std::uint32_t T, std::uint32_t cur, std::uint32_t level) {
        const std::uint32_t lane = lane_id();
        const unsigned below = (1u << lane) - 1u;
        const bool act = lane < T;
        const bool learned = c->learned_n > 0;
        const std::uint32_t dlev = level > c->cdl ? level : c->cdl;
        std::uint32_t lo = 0, hi = F;  // frontier literal of entry e = lane
        while (hi - lo > 1) {
            const std::uint32_t mid = (lo + hi) >> 1;
            if (sm.froff()[mid] <= lane) lo = mid; else hi = mid;
        }
        const std::int32_t trig = sm.fr()[lo];
        std::uint32_t cls = 0;
        const int4 ent = act ? occ_entry(lidx(trig), lane - sm.froff()[lo], learned, cls) : make_int4(-1, 0, 0, 0);
        const std::int32_t id = ent.x;
        tprof(1);
        const unsigned same = __match_any_sync(0xffffffffu, act ? id : -2 - static_cast<std::int32_t>(lane));
        const bool first = act && static_cast<std::uint32_t>(__ffs(same) - 1) == lane;
        bool conflict = false, prop = false;
        std::int32_t plit = 0;
        std::uint32_t clen = 0, meta = 0;
        unsigned long long d0 = 0;
        // long nogoods the two literals in the entry cannot decide are scanned
        // by the whole warp, one at a time
        bool full = false;
        if (first && cls == 3) {
            const int vx = val(atom_of(ent.z)), vy = val(atom_of(ent.w)), vq = val(atom_of(ent.y));
            const int sx = vx == 0 ? 0 : ((vx > 0) == (ent.z > 0) ? 1 : -1);
            const int sy = vy == 0 ? 0 : ((vy > 0) == (ent.w > 0) ? 1 : -1);
            const int sq = vq == 0 ? 0 : ((vq > 0) == (ent.y > 0) ? 1 : -1);
            full = !(sx < 0 || sy < 0 || sq < 0 || (sx == 0) + (sy == 0) + (sq == 0) >= 2);
        }
        if (first && !full) evaluate_entry(ent, cls, trig, conflict, prop, plit, clen, &d0, &meta);
        for (unsigned need = __ballot_sync(0xffffffffu, full); need; need &= need - 1) {
            const std::uint32_t src = static_cast<std::uint32_t>(__ffs(need) - 1);
            bool cf, pr;
            std::int32_t pl;
            std::uint32_t ln, mt;
            unsigned long long dd;
            w_evaluate(static_cast<std::uint32_t>(__shfl_sync(0xffffffffu, id, src)), cf, pr, pl, ln, dd, mt);
            if (lane == src) {
                conflict = cf;
                prop = pr;
                plit = pl;
                clen = ln;
                d0 = dd;
                meta = mt;
            }
        }
#ifdef YAS_TINY_PROF
        {
            const unsigned nf = __popc(__ballot_sync(0xffffffffu, full)), ni = __popc(__ballot_sync(0xffffffffu, first));
            if (prof_on() && lane == 0) {
                c->prof[14] += nf;
                c->prof[15] += ni;
            }
        }
#endif
        tprof(2);
        // winner per proposed atom: the lowest proposing lane
        const std::uint32_t pa = atom_of(plit);
        const unsigned grp = __match_any_sync(0xffffffffu, prop ? static_cast<std::int32_t>(pa) : -2 - static_cast<std::int32_t>(lane));
        const std::uint32_t wl = static_cast<std::uint32_t>(__ffs(grp) - 1);
        const std::int32_t wlit = __shfl_sync(0xffffffffu, plit, wl);
        const bool winner = prop && wl == lane;
        const bool lose = prop && !winner && ((wlit < 0) != (plit < 0));
        const unsigned cm = __ballot_sync(0xffffffffu, conflict || lose);
        const unsigned wm = __ballot_sync(0xffffffffu, winner);
        const std::uint32_t nchk = __popc(__ballot_sync(0xffffffffu, first));
        const std::uint32_t nlit = __reduce_add_sync(0xffffffffu, clen);
        const std::uint32_t nc0 = c->n_confl, ts0 = c->ts;
        if (cm >> lane & 1u) sl.confl()[nc0 + __popc(cm & below)] = id;
        const std::uint32_t occ = winner ? (meta & 0x7fffffffu) : 0u;
        std::uint32_t oinc = occ;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const std::uint32_t o = __shfl_up_sync(0xffffffffu, oinc, d);
            if (lane >= static_cast<std::uint32_t>(d)) oinc += o;
        }
        const std::uint32_t cnt = __popc(wm), tnext = __shfl_sync(0xffffffffu, oinc, 31);
        const std::uint32_t dst = cur ^ 1u;
        tprof(3);
        __syncwarp();  // every lane has read the frontier mirror (sm.fr / sm.froff) before it is rewritten
        if (winner) {
            set_cell(pa, plit > 0 ? static_cast<std::int32_t>(level) : -static_cast<std::int32_t>(level));
            sl.reason()[pa] = id;
            if (nwords(dlev) == 1) {
                dep(0, pa) = d0;
                sl.dovf()[pa] = static_cast<std::uint8_t>(meta >> 31);
            } else if (cls == 1 || cls == 2) {  // the other literals are the trigger and the entry's blocker
                const std::uint32_t x0 = atom_of(trig);
                const std::uint32_t x1 = cls == 2 ? atom_of(pa == atom_of(ent.z) ? ent.w : ent.z) : 0u;
                deps_from_pair(pa, x0, lvl_of(sl.cells()[x0]) > 1, x1, x1 != 0 && lvl_of(sl.cells()[x1]) > 1, nwords(dlev));
            } else {
                std::uint32_t len;
                const std::int32_t* L = lits_of(static_cast<std::uint32_t>(id), len);
                write_deps_from(L, len, static_cast<std::uint32_t>(id), pa, dlev);
            }
            const std::uint32_t r = __popc(wm & below);
            sl.fr(dst)[r] = plit;
            sl.froff()[r] = oinc - occ;
            sm.fr()[r] = plit;
            sm.froff()[r] = oinc - occ;
            sl.trail()[ts0 + r] = plit;
            sl.tpos()[pa] = ts0 + r;
        }
        tprof(4);
        __syncwarp();
        if (lane == 0) {
            sl.froff()[cnt] = tnext;
            sm.froff()[cnt] = tnext;
            c->st.checks += nchk;
            c->st.checked_lits += nlit;
            c->n_confl = nc0 + __popc(cm);
            c->ts = ts0 + cnt;
            c->F = cnt;
            c->T = tnext;
            c->st.propagations += cnt;
            c->n_props = 0;
            c->st.passes += 1;
            c->cur = dst;
            c->b[11] = c->n_confl > 0 ? 1u : 0u;
            c->gen += 1;
        }
        __syncwarp();
    }

    // Initial propagation (propagate.cpp:23-47): static units in compile order
    // (conflict id -(k+1)), then every length-1 store entry in id order,
    // asserted if its guard allows, else a passive violation check. The
    // sequential semantics are reproduced with order keys e.
    __device__ __forceinline__ bool initial_propagation(bool keep_conflicts) {
        const std::uint32_t n1 = S.n_units, n2 = S.n_uids + c->lunits_n, total = n1 + n2;
        const std::uint32_t gen = c->gen;
        for (std::uint32_t base = g.tid() & ~31u; base < total; base += g.size()) {
            const std::uint32_t e = base + lane_id();
            bool conflict = false, prop = false;
            std::int32_t id = 0, lit = 0;
            if (e < total) {
                std::int32_t sigma;
                bool force = true;
                if (e < n1) {
                    sigma = __ldg(S.units + e);
                    id = -static_cast<std::int32_t>(e) - 1;
                } else {
                    const std::uint32_t m = e - n1;
                    id = m < S.n_uids ? __ldg(S.uids + m) : sl.lunits()[m - S.n_uids];
                    std::uint32_t len;
                    const std::int32_t* L = lits_of(static_cast<std::uint32_t>(id), len);
                    sigma = lit_at(L, 0, static_cast<std::uint32_t>(id));
                    force = may_assert(guard_of(static_cast<std::uint32_t>(id)), -sigma);
                }
                if (force) {
                    lit = -sigma;
                    const int cv = val(atom_of(lit));
                    if (cv != 0) {
                        conflict = (cv > 0) != (lit > 0);
                    } else {
                        prop = true;
                        atomicMin(sl.win() + atom_of(lit), wkey(gen, e, lit < 0));
                    }
                }
            }
            __syncwarp();
            const std::uint32_t cs = warp_append(&c->n_confl, conflict);
            if (conflict) sl.confl()[cs] = id;
            const std::uint32_t ps = warp_append(&c->n_props, prop);
            if (prop) sl.props()[ps] = make_int4(id, lit, static_cast<std::int32_t>(e), 0);
        }
        g.sync();
        // passive unit entries see the assignments made before them in order
        for (std::uint32_t base = g.tid() & ~31u; base < n2; base += g.size()) {
            const std::uint32_t m = base + lane_id();
            bool conflict = false;
            std::int32_t id = 0;
            if (m < n2) {
                id = m < S.n_uids ? __ldg(S.uids + m) : sl.lunits()[m - S.n_uids];
                std::uint32_t len;
                const std::int32_t* L = lits_of(static_cast<std::uint32_t>(id), len);
                const std::int32_t sigma = lit_at(L, 0, static_cast<std::uint32_t>(id));
                if (!may_assert(guard_of(static_cast<std::uint32_t>(id)), -sigma)) {
                    const std::uint32_t a = atom_of(sigma);
                    const int cv = val(a);
                    if (cv != 0) {
                        conflict = (cv > 0) == (sigma > 0);
                    } else {
                        const unsigned long long w = sl.win()[a];
                        conflict = static_cast<std::uint32_t>(w >> 32) == ~gen &&
                                   (static_cast<std::uint32_t>(w) >> 1) < n1 + m &&
                                   ((w & 1ull) != 0) == (sigma < 0);
                    }
                }
            }
            __syncwarp();
            const std::uint32_t cs = warp_append(&c->n_confl, conflict);
            if (conflict) sl.confl()[cs] = id;
        }
        g.sync();
        apply<false>(1, true);
        compact<false>(total, c->cur, false, 0);
        const bool violated = c->n_confl > 0;
        g.sync();
        if (!keep_conflicts && g.leader()) c->n_confl = 0;
        g.sync();
        return violated;
    }

    // Erase everything above `target` (assignment.cpp:166-178).
    __device__ __forceinline__ void backjump(std::uint32_t target) {
        if (g.leader()) {
            const std::uint32_t cdl = c->cdl;
            c->b[8] = target < cdl ? sl.tpos()[atom_of(sl.ldec()[target + 1])] : c->ts;
        }
        g.sync();
        const std::uint32_t from = c->b[8], to = c->ts;
        for (std::uint32_t i = from + g.tid(); i < to; i += g.size()) {
            const std::uint32_t a = atom_of(sl.trail()[i]);
            const std::uint32_t nw = nwords(lvl_of(sl.cells()[a]));
            for (std::uint32_t w = 0; w < nw; ++w) dep(w, a) = 0ull;
            sl.dovf()[a] = 0;
            set_cell(a, 0);
            sl.tpos()[a] = 0;
            sl.reason()[a] = kReasonNone;
        }
        const bool lower = target < c->cdl;  // read by every thread before the barrier
        g.sync();
        if (g.leader() && lower) {
            c->ts = from;
            c->cdl = target;
        }
        g.sync();
    }

    // ---- conflict analysis and learning: one warp (the leader's) --------------
    // The paper's Learning / fwd-learning kernels as warp code:
    // literal sets are spread over the lanes, maxima / OR-reductions /
    // compactions are warp collectives, so a step costs one memory round trip
    // instead of one per literal. All functions are called by all 32 lanes.
    __device__ __forceinline__ static unsigned long long w_or64(unsigned long long v) {
        const std::uint32_t lo = __reduce_or_sync(0xffffffffu, static_cast<std::uint32_t>(v));
        const std::uint32_t hi = __reduce_or_sync(0xffffffffu, static_cast<std::uint32_t>(v >> 32));
        return (static_cast<unsigned long long>(hi) << 32) | lo;
    }
    __device__ __forceinline__ static unsigned long long w_min64(unsigned long long v) {
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) {
            const unsigned long long o = __shfl_xor_sync(0xffffffffu, v, d);
            v = o < v ? o : v;
        }
        return v;
    }
    __device__ __forceinline__ static unsigned long long w_max64(unsigned long long v) {
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) {
            const unsigned long long o = __shfl_xor_sync(0xffffffffu, v, d);
            v = o > v ? o : v;
        }
        return v;
    }
    __device__ __forceinline__ static unsigned long long w_add64(unsigned long long v) {
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
        return v;
    }
    __device__ __forceinline__ std::int32_t* sortbuf() const { return sl.scratch() + S.A + 256; }

    // Sort v[0..n) by atom (Nogood::make order; atoms are distinct) by rank.
    __device__ __forceinline__ void w_sort(std::int32_t* v, std::uint32_t n) const {
        const std::uint32_t lane = lane_id();
        if (n <= 32) {
            const std::int32_t x = lane < n ? v[lane] : 0;
            const std::uint32_t ka = lane < n ? atom_of(x) : 0xffffffffu;
            std::uint32_t r = 0;
            for (std::uint32_t s2 = 0; s2 < n; ++s2) r += __shfl_sync(0xffffffffu, ka, s2) < ka;
            __syncwarp();
            if (lane < n) v[r] = x;
            __syncwarp();
            return;
        }
        std::int32_t* tmp = sortbuf();
        for (std::uint32_t i = lane; i < n; i += 32) {
            const std::int32_t x = v[i];
            const std::uint32_t ka = atom_of(x);
            std::uint32_t r = 0;
#pragma unroll 8
            for (std::uint32_t j = 0; j < n; ++j) r += atom_of(v[j]) < ka;
            tmp[r] = x;
        }
        __syncwarp();
        for (std::uint32_t i = lane; i < n; i += 32) v[i] = tmp[i];
        __syncwarp();
    }

    // NogoodStore::add_learned (nogood_store.cpp:81-107). Returns id or -1.
    __device__ __forceinline__ std::int32_t w_add_learned(const std::int32_t* lits, std::uint32_t len, bool count_capacity = true) {
        const std::uint32_t lane = lane_id();
        if ((count_capacity && c->learned_n >= C.learned_capacity) || c->learned_n >= K.lcap ||
            c->lpool_used + len > K.lpool) {
            __syncwarp();
            if (lane == 0) c->status = (count_capacity && c->learned_n >= C.learned_capacity) ? kErrCapacity : kErrArena;
            __syncwarp();
            return -1;
        }
        // duplicate census (learned_seen_, nogood_store.cpp:87-89)
        unsigned long long h = 0;
        for (std::uint32_t k = lane; k < len; k += 32) {
            unsigned long long x = (static_cast<unsigned long long>(static_cast<std::uint32_t>(lits[k])) << 20) ^ k;
            x *= 0x9E3779B97F4A7C15ull;
            h += x ^ (x >> 29);
        }
        h = w_add64(h) + len;
        const std::uint32_t mask = K.dupcap - 1;
        const unsigned long long tag = static_cast<unsigned long long>(c->epoch) << 32;
        for (std::uint32_t at = static_cast<std::uint32_t>(h ^ (h >> 32)) & mask;; at = (at + 1) & mask) {
            const unsigned long long ent = sl.dup()[at];
            if ((ent >> 32) != c->epoch || ent == 0) {
                __syncwarp();
                if (lane == 0) sl.dup()[at] = tag | (c->learned_n + 1);
                break;
            }
            const std::uint32_t other = static_cast<std::uint32_t>(ent) - 1;
            const std::uint32_t olo = sl.loff()[other], olen = sl.loff()[other + 1] - olo;
            bool same = olen == len;
            for (std::uint32_t k = lane; same && k < len; k += 32) same = sl.lpool()[olo + k] == lits[k];
            if (__all_sync(0xffffffffu, same)) {
                if (lane == 0) c->st.duplicate_learned += 1;
                break;
            }
        }
        const std::uint32_t k = c->learned_n;
        const std::uint32_t id = S.N + k;
        const std::uint32_t lo = c->lpool_used;
        for (std::uint32_t j = lane; j < len; j += 32) sl.lpool()[lo + j] = lits[j];
        const std::uint32_t cls = len >= 4 ? 3u : len - 1u;
        bool fail = false;
        for (std::uint32_t j = lane; j < len; j += 32) {  // distinct literals: distinct lists
            const std::uint32_t li = lidx(lits[j]);
            std::uint32_t* h3 = sl.lhdr() + 3 * (li * 4 + cls);
            std::uint32_t base = h3[0], size = h3[1], cap = h3[2];
            if (size == cap) {
                const std::uint32_t ncap = cap ? 2 * cap : 4u;
                const std::uint32_t np = atomicAdd(&c->locc_used, ncap);
                if (np + ncap > K.larena) { fail = true; continue; }
                for (std::uint32_t q = 0; q < size; ++q) sl.larena()[np + q] = sl.larena()[base + q];  // 16-byte entries
                base = np;
                h3[0] = np;
                h3[2] = ncap;
            }
            const std::int32_t o0 = j == 0 ? (len > 1 ? lits[1] : 0) : lits[0];
            const std::int32_t o1 = j <= 1 ? (len > 2 ? lits[2] : 0) : lits[1];
            const std::int32_t o2 = j <= 2 ? (len > 3 ? lits[3] : 0) : lits[2];  // long nogoods: a third blocker
            sl.larena()[base + size] = make_int4(static_cast<std::int32_t>(id | cls << 30),
                                                 cls == 3 ? o2 : static_cast<std::int32_t>(kNone), o0, o1);
            h3[1] = size + 1;
            sl.ltot()[li] += 1;
        }
        __syncwarp();
        if (__any_sync(0xffffffffu, fail)) {
            if (lane == 0) c->status = kErrArena;
            __syncwarp();
            return -1;
        }
        if (lane == 0) {
            sl.loff()[k + 1] = lo + len;
            c->lpool_used = lo + len;
            if (len == 1) sl.lunits()[c->lunits_n++] = static_cast<std::int32_t>(id);
            c->learned_n = k + 1;
        }
        __syncwarp();
        return static_cast<std::int32_t>(id);
    }

    // State of nogood `id` under the current assignment: any dead literal
    // (satisfied), number of free literals and the free one when unique.
    __device__ __forceinline__ void w_status(std::uint32_t id, bool& dead, std::uint32_t& nfree, std::int32_t& rem) const {
        std::uint32_t len;
        const std::int32_t* L = lits_of(id, len);
        std::uint32_t nf = 0;
        std::int32_t fl = 0;
        bool dd = false;
        for (std::uint32_t k = lane_id(); k < len; k += 32) {
            const std::int32_t l = lit_at(L, k, id);
            const int v = val(atom_of(l));
            if (v == 0) { ++nf; fl = l; }
            else if ((v > 0) != (l > 0)) dd = true;
        }
        dead = __any_sync(0xffffffffu, dd);
        nfree = __reduce_add_sync(0xffffffffu, nf);
        const unsigned holder = __ballot_sync(0xffffffffu, nf != 0);
        rem = holder ? __shfl_sync(0xffffffffu, fl, __ffs(holder) - 1) : 0;
    }

    // Driver::try_assert (solver.cpp:117-146) on the current frontier.
    __device__ __forceinline__ void w_try_assert(std::uint32_t id) {
        const std::uint32_t lane = lane_id();
        bool dead;
        std::uint32_t nfree;
        std::int32_t rem;
        w_status(id, dead, nfree, rem);
        if (dead || nfree >= 2) return;
        if (nfree == 0) {
            if (lane == 0) sl.pending()[c->n_pending++] = static_cast<std::int32_t>(id);
            __syncwarp();
            return;
        }
        if (!may_assert(guard_of(id), -rem)) return;
        const std::int32_t lit = -rem;
        const std::uint32_t a = atom_of(lit), cdl = c->cdl;
        std::uint32_t len;
        const std::int32_t* L = lits_of(id, len);
        const std::uint32_t nw = nwords(cdl);
        std::uint32_t ov = 0;
        for (std::uint32_t w = 0; w < nw; ++w) {  // Deps: OR over the other literals (propagate.cpp:49-62)
            unsigned long long acc = 0;
            for (std::uint32_t k = lane; k < len; k += 32) {
                const std::uint32_t x = atom_of(lit_at(L, k, id));
                if (x == a || lvl_of(sl.cells()[x]) <= 1) continue;
                acc |= dep(w, x);
                if (w == 0) ov |= sl.dovf()[x];
            }
            acc = w_or64(acc);
            if (lane == 0) dep(w, a) = acc;
        }
        ov = __reduce_or_sync(0xffffffffu, ov);
        if (lane == 0) {
            sl.dovf()[a] = static_cast<std::uint8_t>(ov);
            set_cell(a, lit > 0 ? static_cast<std::int32_t>(cdl) : -static_cast<std::int32_t>(cdl));
            sl.reason()[a] = static_cast<std::int32_t>(id);
            sl.tpos()[a] = c->ts;
            sl.trail()[c->ts++] = lit;
            sl.fr(c->cur)[c->F++] = lit;
            c->st.propagations += 1;
        }
        __syncwarp();
    }

    // fwd_learning (learn.cpp:106-142). Writes the learned literals to out and
    // returns their count, or 0xffffffff on a Deps overflow (-> res fallback).
    __device__ __forceinline__ std::uint32_t w_fwd(std::uint32_t delta, std::int32_t* out, std::uint32_t& target) {
        const std::uint32_t lane = lane_id();
        const unsigned below = (1u << lane) - 1u;
        std::uint32_t len;
        const std::int32_t* L = lits_of(delta, len);
        std::uint32_t cl = 0;
        bool ov = false;
        for (std::uint32_t k = lane; k < len; k += 32) {
            const std::uint32_t a = atom_of(lit_at(L, k, delta));
            cl = max(cl, lvl_of(sl.cells()[a]));
            ov |= sl.dovf()[a] != 0;
        }
        cl = __reduce_max_sync(0xffffffffu, cl);
        if (__any_sync(0xffffffffu, ov)) return 0xffffffffu;
        const std::uint32_t nw = nwords(c->cdl);
        std::uint32_t n = 0, tg = 0;
        for (std::uint32_t w = 0; w < nw; ++w) {
            unsigned long long m = 0;
            for (std::uint32_t k = lane; k < len; k += 32) {
                const std::uint32_t a = atom_of(lit_at(L, k, delta));
                if (lvl_of(sl.cells()[a]) > 1) m |= dep(w, a);
            }
            m = w_or64(m);
#pragma unroll
            for (int half = 0; half < 2; ++half) {
                const std::uint32_t b32 = static_cast<std::uint32_t>(m >> (32 * half));
                if (b32 >> lane & 1u) {
                    const std::uint32_t level = 64 * w + 32 * half + lane + 1;
                    out[n + __popc(b32 & below)] = sl.ldec()[level];
                    if (level < cl) tg = max(tg, level);
                }
                n += __popc(b32);
            }
        }
        target = __reduce_max_sync(0xffffffffu, tg);
        if (target == 0) target = 1;
        __syncwarp();
        w_sort(out, n);
        return n;
    }

    // res_learning (learn.cpp:53-104): resolve until a positive UIP. The set is
    // kept as atoms in out[0..n) (unordered) with membership stamps in mark[].
    __device__ __forceinline__ std::uint32_t w_res(std::uint32_t delta, std::int32_t* out, std::uint32_t& target) {
        const std::uint32_t lane = lane_id();
        const unsigned below = (1u << lane) - 1u;
        std::uint32_t* mark = sl.mark();
        const std::uint32_t stamp = c->stamp + 1;
        __syncwarp();
        if (lane == 0) c->stamp = stamp;
        std::uint32_t len;
        const std::int32_t* L = lits_of(delta, len);
        std::uint32_t n = len;
        for (std::uint32_t k = lane; k < len; k += 32) {
            const std::uint32_t a = atom_of(lit_at(L, k, delta));
            mark[a] = stamp;
            out[k] = static_cast<std::int32_t>(a);
        }
        __syncwarp();
        for (;;) {
            // sigma = greatest trail position; kappa = greatest level of the others
            unsigned long long best = 0;  // (tpos + 1) << 32 | k
            std::uint32_t m1 = 0, c1 = 0;
            for (std::uint32_t k = lane; k < n; k += 32) {
                const std::uint32_t a = static_cast<std::uint32_t>(out[k]);
                const unsigned long long key = (static_cast<unsigned long long>(sl.tpos()[a] + 1) << 32) | k;
                best = key > best ? key : best;
                const std::uint32_t lv = lvl_of(sl.cells()[a]);
                if (lv > m1) { m1 = lv; c1 = 1; } else if (lv == m1) ++c1;
            }
            best = w_max64(best);
            const std::uint32_t gm1 = __reduce_max_sync(0xffffffffu, m1);
            const std::uint32_t gc1 = __reduce_add_sync(0xffffffffu, m1 == gm1 ? c1 : 0u);
            std::uint32_t m2 = 0;
            for (std::uint32_t k = lane; k < n; k += 32) {
                const std::uint32_t lv = lvl_of(sl.cells()[out[k]]);
                if (lv < gm1) m2 = max(m2, lv);
            }
            m2 = __reduce_max_sync(0xffffffffu, m2);
            const std::uint32_t si = static_cast<std::uint32_t>(best);
            const std::uint32_t sa = static_cast<std::uint32_t>(out[si]);
            const std::int32_t scell = sl.cells()[sa];
            const std::uint32_t slev = lvl_of(scell);
            const std::uint32_t kappa = slev == gm1 ? (gc1 > 1 ? gm1 : m2) : gm1;
            if (kappa != slev && scell > 0) {
                target = kappa > 1 ? kappa : 1;
                for (std::uint32_t k = lane; k < n; k += 32) {
                    const std::int32_t a = out[k];
                    out[k] = sl.cells()[a] > 0 ? a : -a;
                }
                __syncwarp();
                w_sort(out, n);
                return n;
            }
            const std::int32_t r = sl.reason()[sa];
            __syncwarp();
            if (lane == 0) {
                out[si] = out[n - 1];
                mark[sa] = 0;
            }
            --n;
            __syncwarp();
            const std::int32_t* E = nullptr;
            std::uint32_t elen = 0;
            if (r >= 0) E = lits_of(static_cast<std::uint32_t>(r), elen);
            else if (r == kReasonCompletion) elen = c->cdl >= 2 ? c->cdl - 1 : 0;
            else {
                if (lane == 0) c->status = kErrLogic;
                __syncwarp();
                return 0;
            }
            for (std::uint32_t k0 = 0; k0 < elen; k0 += 32) {
                const std::uint32_t k = k0 + lane;
                std::uint32_t a = 0;
                if (k < elen) a = r >= 0 ? atom_of(lit_at(E, k, static_cast<std::uint32_t>(r))) : atom_of(sl.ldec()[k + 2]);
                const bool keep = k < elen && a != sa && mark[a] != stamp;
                const unsigned km = __ballot_sync(0xffffffffu, keep);
                if (keep) {
                    mark[a] = stamp;
                    out[n + __popc(km & below)] = static_cast<std::int32_t>(a);
                }
                n += __popc(km);
            }
            __syncwarp();
        }
    }

    // Driver::handle_conflicts (solver.cpp:161-214), leader-warp part: writes
    // the backjump plan to c->b.
    __device__ __forceinline__ void analyze_and_learn() {
        const std::uint32_t lane = lane_id();
        if (lane == 0) {
            c->st.conflicts += 1;
            c->b[0] = 0;
        }
        __syncwarp();
        if (c->cdl == 1) return;  // nothing to revise
        const std::uint32_t nc = c->n_confl;
        // select conflicts: min (length, id); fanout K in fwd mode (learn.cpp:148-157)
        const std::uint32_t K2 = (!G::kLean && mode() == 0 && C.fanout > 1) ? C.fanout : 1u;
        std::int32_t* added = sl.scratch();            // ids of added nogoods
        std::int32_t* levels = sl.scratch() + 64;      // their backjump levels
        std::int32_t* buf = sl.scratch() + 128;        // learned literal buffer
        std::uint32_t n_sel = 0;
        unsigned long long prev = 0;
        bool have_prev = false;
        std::uint32_t bj = 0xffffffffu;
        while (n_sel < K2) {
            unsigned long long best = ~0ull;
            for (std::uint32_t i = lane; i < nc; i += 32) {
                const std::uint32_t id = static_cast<std::uint32_t>(sl.confl()[i]);
                const unsigned long long key = (static_cast<unsigned long long>(length_of(id)) << 32) | id;
                if ((!have_prev || key > prev) && key < best) best = key;
            }
            best = w_min64(best);
            if (best == ~0ull) break;
            prev = best;
            have_prev = true;
            const std::uint32_t delta = static_cast<std::uint32_t>(best);
            std::uint32_t target = 1, n = 0xffffffffu;
            std::uint32_t used = 1;  // 0 fwd, 1 res
            if (mode() == 0) {
                n = w_fwd(delta, buf, target);
                if (n != 0xffffffffu) used = 0;
            }
            if (n == 0xffffffffu) {
                n = w_res(delta, buf, target);
                if (c->status != kRunning) return;
            }
            // structural self-checks (solver.cpp:171-186)
            if (used == 1) {
                std::uint32_t cl = 0;
                for (std::uint32_t k = lane; k < n; k += 32) cl = max(cl, lvl_of(sl.cells()[atom_of(buf[k])]));
                cl = __reduce_max_sync(0xffffffffu, cl);
                std::uint32_t at = 0;
                for (std::uint32_t k = lane; k < n; k += 32) at += lvl_of(sl.cells()[atom_of(buf[k])]) == cl;
                at = __reduce_add_sync(0xffffffffu, at);
                if (lane == 0) {
                    if (at != 1) c->st.uip_check_failures += 1;
                    c->st.res_learned += 1;
                    if (mode() == 0) c->st.fwd_fallbacks += 1;
                }
            } else {
                std::uint32_t bad = 0;
                for (std::uint32_t k = lane; k < n; k += 32) bad += sl.reason()[atom_of(buf[k])] != kReasonDecision;
                bad = __reduce_add_sync(0xffffffffu, bad);
                if (lane == 0) {
                    c->st.fwd_decision_only_failures += bad;
                    c->st.fwd_learned += 1;
                }
            }
            __syncwarp();
            const std::int32_t id = w_add_learned(buf, n);
            if (id < 0) return;
            if (heur() == 2)
                for (std::uint32_t k = lane; k < n; k += 32) sl.act()[atom_of(buf[k])] += c->act_inc;
            if (lane == 0) {
                added[n_sel] = id;
                levels[n_sel] = static_cast<std::int32_t>(target);
                c->st.learned_count += 1;
                c->st.learned_length_sum += n;
                if (trace_on() && c->n_trace < K.tcap)
                    sl.tbuf()[c->n_trace++] = make_uint4(used, static_cast<std::uint32_t>(delta), n, target);
            }
            ++n_sel;
            bj = target < bj ? target : bj;
            __syncwarp();
        }
        // Heuristic::on_conflict (decide.cpp:34-41)
        if (heur() == 2) {
            const double inc = c->act_inc / C.decay;
            if (inc > 1e100)
                for (std::uint32_t a = lane; a <= S.A; a += 32) sl.act()[a] *= 1e-100;
            __syncwarp();
            if (lane == 0) c->act_inc = inc > 1e100 ? inc * 1e-100 : inc;
        }
        if (lane == 0) {
            const bool restart = !G::kLean && C.restarts && c->st.conflicts - c->conflicts_at_restart >= c->restart_threshold;
            if (restart) {
                c->st.restarts += 1;
                c->conflicts_at_restart = c->st.conflicts;
                c->restart_threshold = static_cast<unsigned long long>(
                    ceil(static_cast<double>(c->restart_threshold) * C.restart_factor));
            }
            c->b[0] = 1;
            c->b[1] = restart ? 1u : 0u;
            c->b[2] = restart ? 1u : bj;
            c->b[3] = n_sel;
            c->F = 0;
            c->n_confl = 0;
        }
        __syncwarp();
    }

    __device__ __forceinline__ bool handle_conflicts() {
        g.sync();  // the whole group has left propagation (it reads F, T, ... at its loop top)
        if (g.leader_warp()) analyze_and_learn();
        g.sync();
#ifdef YAS_TINY_PROF
        mark(14);  // profiling build: conflict analysis + learning
#endif
        if (c->status != kRunning) return false;
        if (c->b[0] == 0) return false;
        const bool restart = c->b[1] != 0;
        const std::uint32_t target = c->b[2];
        backjump(target);
        if (restart) initial_propagation(false);
#ifdef YAS_TINY_PROF
        mark(15);  // profiling build: backjump (+ restart)
#endif
        if (g.leader_warp()) {
            const std::uint32_t n_sel = c->b[3];
            const std::int32_t* added = sl.scratch();
            const std::int32_t* levels = sl.scratch() + 64;
            if (!restart)
                for (std::uint32_t i = 0; i < n_sel; ++i)
                    if (static_cast<std::uint32_t>(levels[i]) == target) {
                        bool dead;
                        std::uint32_t nfree;
                        std::int32_t rem;
                        w_status(static_cast<std::uint32_t>(added[i]), dead, nfree, rem);
                        if ((dead || nfree != 1) && lane_id() == 0) c->st.asserting_failures += 1;
                        __syncwarp();
                    }
            for (std::uint32_t i = 0; i < n_sel; ++i) w_try_assert(static_cast<std::uint32_t>(added[i]));
        }
        g.sync();
        return true;
    }

    __device__ __forceinline__ double score(std::uint32_t head) const {
        if (heur() == 2) return sl.act()[head];
        if (heur() == 0) return static_cast<double>(occ_total(2 * head) + occ_total(2 * head + 1));
        double s = 0.0;  // Jeroslow-Wang, summed in the reference's list order
        for (std::uint32_t li = 2 * head; li <= 2 * head + 1; ++li)
            for (std::uint32_t cl = 0; cl < 4; ++cl) {
                const std::uint32_t lo = __ldg(S.occ_off + li * 4 + cl), hi = __ldg(S.occ_off + li * 4 + cl + 1);
                for (std::uint32_t j = lo; j < hi; ++j)
                    s += ldexp(1.0, -static_cast<int>(length_of(static_cast<std::uint32_t>(__ldg(S.occ + j).x) & 0x3fffffffu)));
                const std::uint32_t* h = sl.lhdr() + 3 * (li * 4 + cl);
                for (std::uint32_t j = 0; j < h[1]; ++j)
                    s += ldexp(1.0, -static_cast<int>(length_of(static_cast<std::uint32_t>(sl.larena()[h[0] + j].x) & 0x3fffffffu)));
            }
        return s;
    }

    // find_applicable + score (decide.cpp:43-79): DU rules per thread per
    // step, every load of a step issued before any is used. Packed variant:
    // 8-byte records (the rule table of a single search stays in L1) and one
    // static count + two learned counts per applicable head (occurrence heuristic).
    __device__ __forceinline__ void scan_rules_packed(std::uint32_t& best, std::uint32_t& bi) const {
        constexpr int DU = 8;
        const std::uint32_t gs = g.size();
        for (std::uint32_t r0 = g.tid(); r0 < S.R; r0 += DU * gs) {
            unsigned long long ru[DU];
#pragma unroll
            for (int k = 0; k < DU; ++k) {
                const std::uint32_t r = r0 + k * gs;
                ru[k] = r < S.R ? __ldg(S.rules8 + r) : (1ull << 63);
            }
            std::uint32_t hh[DU];
            bool app[DU];
#pragma unroll
            for (int k = 0; k < DU; ++k) {
                const std::uint32_t h = static_cast<std::uint32_t>(ru[k]) & 0x1fffffu;
                const std::uint32_t t = static_cast<std::uint32_t>(ru[k] >> 21) & 0x1fffffu;
                const std::uint32_t n = static_cast<std::uint32_t>(ru[k] >> 42) & 0x1fffffu;
                app[k] = !(ru[k] >> 63) && val(h) == 0 && (t == 0 || val(t) > 0) && (n == 0 || val(n) >= 0);
                hh[k] = app[k] ? h : 0u;
            }
            std::uint32_t so[DU], l0[DU], l1[DU];
#pragma unroll
            for (int k = 0; k < DU; ++k) {
                so[k] = __ldg(S.socc + hh[k]);
                l0[k] = sl.ltot()[2 * hh[k]];
                l1[k] = sl.ltot()[2 * hh[k] + 1];
            }
#pragma unroll
            for (int k = 0; k < DU; ++k) {  // this thread's rules come in index order: ties keep the first
                const std::uint32_t sc = so[k] + l0[k] + l1[k] + 1u;
                if (app[k] && sc > best) { best = sc; bi = r0 + k * gs; }
            }
        }
    }
    __device__ __forceinline__ void scan_rules(double& best, std::uint32_t& bi) const {
        constexpr int DU = 8;
        const std::uint32_t gs = g.size();
        for (std::uint32_t r0 = g.tid(); r0 < S.R; r0 += DU * gs) {
            uint4 ru[DU];
#pragma unroll
            for (int k = 0; k < DU; ++k) {
                const std::uint32_t r = r0 + k * gs;
                ru[k] = r < S.R ? __ldg(S.rules + r) : make_uint4(0u, 0u, 0u, 0x80000000u);
            }
            bool app[DU];
#pragma unroll
            for (int k = 0; k < DU; ++k) {
                const std::uint32_t n = ru[k].w & 0x7fffffffu;
                app[k] = !(ru[k].w >> 31) && val(ru[k].x) == 0 && (ru[k].z == 0 || val(ru[k].z) > 0) &&
                         (n == 0 || val(n) >= 0);
            }
            if (heur() == 0) {  // occurrence count: 2 x (two offsets + learned count) per head
                std::uint32_t o[DU][6];
#pragma unroll
                for (int k = 0; k < DU; ++k) {
                    const std::uint32_t h = app[k] ? ru[k].x : 0u;
                    o[k][0] = __ldg(S.occ_off + 8 * h);
                    o[k][1] = __ldg(S.occ_off + 8 * h + 4);
                    o[k][2] = sl.ltot()[2 * h];
                    o[k][3] = __ldg(S.occ_off + 8 * h + 4);
                    o[k][4] = __ldg(S.occ_off + 8 * h + 8);
                    o[k][5] = sl.ltot()[2 * h + 1];
                }
#pragma unroll
                for (int k = 0; k < DU; ++k) {
                    const double sc = static_cast<double>(o[k][1] - o[k][0] + o[k][2] + o[k][4] - o[k][3] + o[k][5]);
                    if (app[k] && better(sc, r0 + k * gs, best, bi)) { best = sc; bi = r0 + k * gs; }
                }
            } else {
#pragma unroll
                for (int k = 0; k < DU; ++k) {
                    if (!app[k]) continue;
                    const double sc = score(ru[k].x);
                    if (better(sc, r0 + k * gs, best, bi)) { best = sc; bi = r0 + k * gs; }
                }
            }
        }
    }

    // decide (decide.cpp:107-122) or complete_assignment (decide.cpp:124-135)
    __device__ __forceinline__ void decide_or_complete() {
        double best = -1.0;
        std::uint32_t bi = 0xffffffffu;
        bool packed = false;
        if constexpr (G::kBlock) {
            packed = heur() == 0 && S.rules8 != nullptr;
            if (packed) {
                std::uint32_t bu = 0;
                scan_rules_packed(bu, bi);
                g.argmax_u(bu, bi);
                if (bu == 0) bi = 0xffffffffu;
            }
        }
        if (!packed) {
            scan_rules(best, bi);
            g.argmax(best, bi);
        }
        if (bi != 0xffffffffu) {
            if (g.leader()) {
                const std::uint32_t b = __ldg(S.rules + bi).y;
                const std::uint32_t cdl = ++c->cdl;
                sl.ldec()[cdl] = static_cast<std::int32_t>(b);
                set_cell(b, static_cast<std::int32_t>(cdl));
                sl.tpos()[b] = c->ts;
                sl.trail()[c->ts++] = static_cast<std::int32_t>(b);
                sl.reason()[b] = kReasonDecision;
                const std::uint32_t bit = cdl - 1;
                if (bit >= 64 * C.W) sl.dovf()[b] = 1;
                else dep(bit / 64, b) |= 1ull << (bit % 64);
                c->st.decisions += 1;
                sl.fr(c->cur)[0] = static_cast<std::int32_t>(b);
                c->F = 1;
            }
            g.sync();
            return;
        }
        // complete: falsify open program atoms in atom order at cdl
        const std::uint32_t cdl = c->cdl, ts0 = c->ts, cur = c->cur, np = S.n_prog;
        const std::uint32_t nw = nwords(cdl);
        const std::uint32_t hi = (cdl - 1 < 64 * C.W) ? cdl - 1 : 64 * C.W - 1;  // top bit index set
        const std::uint8_t ovf = (cdl - 1 >= 64 * C.W) ? 1 : 0;
        unsigned long long carry = 0;
        for (std::uint32_t base = 0; base < np; base += g.size()) {
            const std::uint32_t a = base + g.tid() + 1;
            const bool open = a <= np && val(a) == 0;
            unsigned long long tot;
            const std::uint32_t r = static_cast<std::uint32_t>(g.scan(open ? 1ull : 0ull, tot) + carry);
            if (open) {
                set_cell(a, -static_cast<std::int32_t>(cdl));
                sl.reason()[a] = kReasonCompletion;
                for (std::uint32_t w = 0; w < nw; ++w) {
                    unsigned long long m = 0;
                    if (cdl >= 2) {
                        const std::uint32_t lo_b = w * 64, hi_b = w * 64 + 63;
                        const std::uint32_t from = lo_b > 1 ? lo_b : 1, to = hi_b < hi ? hi_b : hi;
                        if (from <= to) {
                            const std::uint32_t cnt = to - from + 1;
                            m = (cnt == 64 ? ~0ull : ((1ull << cnt) - 1)) << (from - lo_b);
                        }
                    }
                    dep(w, a) = m;
                }
                sl.dovf()[a] = ovf;
                sl.tpos()[a] = ts0 + r;
                sl.trail()[ts0 + r] = -static_cast<std::int32_t>(a);
                sl.fr(cur)[r] = -static_cast<std::int32_t>(a);
            }
            carry += tot;
        }
        g.sync();
        if (g.leader()) {
            c->ts = ts0 + static_cast<std::uint32_t>(carry);
            c->F = static_cast<std::uint32_t>(carry);
        }
        g.sync();
    }

    __device__ __forceinline__ void record_model(std::uint32_t cube) {
        const std::uint32_t m = c->n_mbuf, words = K.mwords;
        for (std::uint32_t w = g.tid(); w < words; w += g.size()) {
            std::uint32_t bits = 0;
            for (std::uint32_t b = 0; b < 32; ++b) {
                const std::uint32_t a = 32 * w + b + 1;
                if (a <= S.n_prog && val(a) > 0) bits |= 1u << b;
            }
            sl.mbuf()[static_cast<std::size_t>(m) * words + w] = bits;
        }
        g.sync();
        if (g.leader()) {
            sl.mcube()[m] = cube;
            c->n_mbuf = m + 1;
            c->st.models += 1;
            c->pad0 += 1;  // models of this search
            if (C.cube_width && C.max_models != 0) {  // cube-parallel first models: enough found anywhere?
                const std::uint32_t n = 1u + (C.fleet ? atomicAdd_system(&C.fleet->found, 1u) : atomicAdd(&sh->found, 1u));
                if (n >= C.max_models) {
                    sh->stop = 1;
                    if (C.fleet) atomicExch_system(&C.fleet->stop, 1u);
                }
            }
        }
        g.sync();
    }

    // block_current_model (solver.cpp:234-246). false = enumeration complete.
    __device__ __forceinline__ bool block_model() {
        if (g.leader_warp()) {
            const std::uint32_t lane = lane_id();
            if (lane == 0) c->b[0] = 0;
            const std::uint32_t cdl = c->cdl;
            if (cdl > 1) {
                std::int32_t* buf = sl.scratch() + 128;
                for (std::uint32_t lv = 2 + lane; lv <= cdl; lv += 32) buf[lv - 2] = sl.ldec()[lv];
                __syncwarp();
                w_sort(buf, cdl - 1);
                const std::int32_t id = w_add_learned(buf, cdl - 1);
                if (id >= 0 && lane == 0) {
                    c->st.blocking_nogoods += 1;
                    c->b[0] = 1;
                    c->b[1] = static_cast<std::uint32_t>(id);
                    c->F = 0;
                }
            }
            __syncwarp();
        }
        g.sync();
        if (c->b[0] == 0) return false;
        const std::uint32_t id = c->b[1];
        backjump(1);
        if (g.leader_warp()) w_try_assert(id);
        g.sync();
        return true;
    }

    // validate_fixpoint (propagate.cpp:251-266) for cfg.debug_validate
    __device__ __forceinline__ void validate() {
        const std::uint32_t total = S.N + c->learned_n;
        for (std::uint32_t id = g.tid(); id < total; id += g.size()) {
            std::uint32_t len, nfree = 0, nhold = 0;
            const std::int32_t* L = lits_of(id, len);
            std::int32_t open = 0;
            bool dead = false;
            for (std::uint32_t k = 0; k < len; ++k) {
                const std::int32_t l = lit_at(L, k, id);
                const int cv = val(atom_of(l));
                if (cv == 0) { ++nfree; open = l; }
                else if ((cv > 0) == (l > 0)) ++nhold;
                else dead = true;
            }
            if (dead) continue;
            if (nfree == 0 || (nfree == 1 && may_assert(guard_of(id), -open))) c->status = kErrValidate;
        }
        for (std::uint32_t k = g.tid(); k < S.n_units; k += g.size())
            if (!holds(-__ldg(S.units + k))) c->status = kErrValidate;
        g.sync();
    }

    // Fresh search in this slot: clear what the previous search touched.
    __device__ __forceinline__ void begin_search(std::uint32_t cube) {
        const std::uint32_t ts = c->ts;
        const bool wide = c->rows_wide != 0;
        for (std::uint32_t i = g.tid(); i < ts; i += g.size()) {
            const std::uint32_t a = atom_of(sl.trail()[i]);
            const std::uint32_t nw = wide ? C.W : nwords(lvl_of(sl.cells()[a]));
            for (std::uint32_t w = 0; w < nw; ++w) dep(w, a) = 0ull;
            sl.dovf()[a] = 0;
            set_cell(a, 0);
            sl.tpos()[a] = 0;
            sl.reason()[a] = kReasonNone;
        }
        const std::uint32_t keys = (2 * S.A + 2) * 4;
        if (c->epoch == 0) {  // a fresh slot: every learned occurrence header
            for (std::uint32_t i = g.tid(); i < 3 * keys; i += g.size()) sl.lhdr()[i] = 0;
            for (std::uint32_t i = g.tid(); i < 2 * S.A + 2; i += g.size()) sl.ltot()[i] = 0;
        } else if (c->learned_n > 0) {
            // only literals of learned nogoods (cube units and blocking nogoods
            // included) have learned occurrences: clear just their headers
            const std::uint32_t nl = c->lpool_used;
            for (std::uint32_t i = g.tid(); i < nl; i += g.size()) {
                const std::uint32_t li = lidx(sl.lpool()[i]);
                std::uint32_t* h = sl.lhdr() + 3 * (li * 4);
#pragma unroll
                for (int k = 0; k < 12; ++k) h[k] = 0;
                sl.ltot()[li] = 0;
            }
        }
        std::uint32_t var = C.mode | C.heur << 1;
        if constexpr (!G::kGrid)
            if (portfolio_on()) var = (C.pf_base + cube) % 6u;
        if ((var >> 1) == 2)
            for (std::uint32_t i = g.tid(); i <= S.A; i += g.size()) sl.act()[i] = 0.0;
        g.sync();
        if (g.leader()) {
            c->variant = var;
            c->cdl = 1;
            c->ts = 0;
            c->F = 0;
            c->cur = 0;
            c->T = 0;
            c->n_props = c->n_confl = c->n_pending = 0;
            c->learned_n = c->lpool_used = c->locc_used = c->lunits_n = 0;
            sl.loff()[0] = 0;
            c->cube = cube;
            c->rows_wide = 0;
            c->epoch += 1;
            if (c->gen == 0) c->gen = 1;  // claim/win keys of generation 0 equal the all-ones init
            c->pad0 = 0;
            c->restart_threshold = C.restart_base;
            c->conflicts_at_restart = c->st.conflicts;
            c->act_inc = 1.0;
            c->st.searches += 1;
            c->phase = kInit;
        }
        g.sync();
        if (C.cube_width == 0) return;
        if (g.leader_warp()) {  // cube constraints enter as unit nogoods ahead of any learned one
            std::int32_t* buf = sl.scratch() + 128;
            for (std::uint32_t k = 0; k < C.cube_width; ++k) {
                const std::int32_t l = __ldg(S.cubes + static_cast<std::size_t>(cube) * C.cube_width + k);
                if (l == 0) continue;
                if (lane_id() == 0) buf[0] = l;
                __syncwarp();
                w_add_learned(buf, 1, false);
            }
        }
        g.sync();
    }

    // The Alg. 1 state machine (solver.cpp:248-303). Returns when the search
    // is finished (phase kFinished), on error, or when it must yield.
    __device__ __forceinline__ void run() {
        for (;;) {
            const std::uint32_t ph = c->phase;
            if (c->status != kRunning) return;
            g.sync();
            if (ph == kInit) {
                const bool violated = initial_propagation(true);
                if (g.leader()) {
                    c->n_confl = 0;
                    c->phase = violated ? kFinished : kLoop;
                }
                g.sync();
                continue;
            }
            if (ph == kAfterModel) {
                if (C.max_models != 0 && c->pad0 >= C.max_models) {
                    if (g.leader()) c->phase = kFinished;
                    g.sync();
                    return;
                }
                const bool more = block_model();
                if (c->status != kRunning) return;
                if (g.leader()) c->phase = more ? kLoop : kFinished;
                g.sync();
                if (!more) return;
                continue;
            }
            if (ph != kLoop) return;
            // yield check at the loop top (clean state)
            if (g.leader()) {
                // a portfolio search another GPU / process has beaten ends here
                if constexpr (!G::kGrid)
                    if ((portfolio_on() || (C.cube_width && C.max_models != 0)) && C.fleet &&
                        *reinterpret_cast<volatile std::uint32_t*>(&C.fleet->stop)) {
                        c->status = kDone;
                        c->phase = kFinished;
                    }
                bool y = sh->stop != 0;
                if (c->n_mbuf >= K.mcap || (trace_on() && c->n_trace + 64 > K.tcap)) {
                    y = true;
                    sh->stop = 1;
                }
                if (C.slice_ns && gtimer() - t0 > C.slice_ns) y = true;
                c->b[15] = y ? 1u : 0u;
            }
            g.sync();
            mark(11);
            // every thread reads both words before anyone may change them again
            const bool ended = !G::kGrid && c->status != kRunning, yield = c->b[15] != 0;
            if (ended) return;
            if (yield) {
                g.sync();
                if (g.leader()) c->status = kYield;
                g.sync();
                return;
            }
            bool conflicted;
            if (c->n_pending == 0) {
                conflicted = propagate(c->cdl);
            } else {
                if (g.leader()) {
                    for (std::uint32_t i = 0; i < c->n_pending; ++i) sl.confl()[i] = sl.pending()[i];
                    c->n_confl = c->n_pending;
                    c->n_pending = 0;
                }
                g.sync();
                conflicted = true;
            }
            if (conflicted) {
                mark(0);
                const bool go_on = handle_conflicts();
                mark(7);
                if (!go_on) {
                    const bool ended = c->status != kRunning;
                    g.sync();  // status read everywhere before the leader moves on
                    if (ended) return;
                    if (g.leader()) c->phase = kFinished;
                    g.sync();
                    return;
                }
                continue;
            }
            if (!G::kLean && C.debug_validate) {
                validate();
                if (c->status != kRunning) return;
            }
            if (c->ts != S.A) {
                mark(0);
                decide_or_complete();
                mark(6);
                continue;
            }
            record_model(c->cube);
            if (g.leader()) c->phase = kAfterModel;
            g.sync();
        }
    }
};

// ---------------------------------------------------------------------------
// Kernels
// ---------------------------------------------------------------------------
template <class G>
__device__ void init_smem(G& g, Search<G>& s) {
    const Sm& m = s.sm;
    if (m.tcap()) {
        for (std::uint32_t i = g.tid(); i <= m.hmask(); i += g.size()) {
            m.htab()[i] = 0ull;
            m.wtab()[i] = 0ull;
        }
        for (std::uint32_t i = g.tid(); i < (m.tcap() + 31) / 32; i += g.size()) m.bits()[i] = 0u;
    }
    s.rebuild_mirror();
    g.sync();
}

template <class G>
__device__ void slot_loop(G& g, const Static& S, const Config& C, Slot sl, const Caps& K, Shared* sh,
                          const Sm& sm) {
    const unsigned long long t0 = gtimer();
    Search<G> s(g, S, C, sl, K, sh, t0, sm);
    init_smem(g, s);
    for (;;) {
        g.sync();
        if (g.c->status != kRunning) return;
        if (!G::kGrid && !G::kLean && C.portfolio && g.c->phase == kFinished) {  // first to finish: stop the others
            if (g.leader()) {
                g.c->done_ns = gtimer();
                const std::uint32_t tag = C.fleet_tag + blockIdx.x;
                const std::uint32_t prev = C.fleet ? atomicCAS_system(&C.fleet->winner, 0xffffffffu, tag)
                                                   : atomicCAS(&sh->winner, 0xffffffffu, tag);
                g.c->won = prev == 0xffffffffu ? 1u : 0u;
                sh->stop = 1;
                if (C.fleet) atomicExch_system(&C.fleet->stop, 1u);
            }
            g.sync();  // every thread has read status and phase: now the leader may finish the search
            if (g.leader()) g.c->status = kDone;
            return;
        }
        if (g.c->phase == kIdle || g.c->phase == kFinished) {
            g.sync();
            if (g.leader()) {
                g.c->phase = kIdle;
                g.c->b[9] = sh->stop ? 0xffffffffu
                            : C.fleet ? atomicAdd_system(&C.fleet->cube_next, 1u)
                                      : atomicAdd(&sh->cube_next, 1u);
            }
            g.sync();
            const std::uint32_t cube = g.c->b[9];
            if (cube >= C.n_cubes) {
                if (g.leader()) g.c->status = cube == 0xffffffffu ? kYield : kDone;
                g.sync();
                return;
            }
            s.begin_search(cube);
        }
        s.run();
    }
}

// One CTA per search slot; slot k = blockIdx.x. MINB = resident CTAs per SM the
// register budget is planned for (1: single search, 4: cube enumeration).
template <int BS, int MINB, bool LEAN = false>
__global__ void __launch_bounds__(BS, MINB)
    block_kernel(const __grid_constant__ Static S, const __grid_constant__ Config C,
                 const __grid_constant__ SlotLayout L, const __grid_constant__ Caps K, Shared* sh,
                 const __grid_constant__ SmemCfg smc) {
    __shared__ Ctl ctl;
    __shared__ unsigned long long sbuf[BS / 32 + 4];
    __shared__ double sd[BS / 32];
    __shared__ std::uint32_t si[BS / 32];
    const Slot sl{L.base + static_cast<unsigned long long>(blockIdx.x) * L.bytes, &L};
    {
        const std::uint32_t* src = reinterpret_cast<const std::uint32_t*>(sl.ctl());
        std::uint32_t* dst = reinterpret_cast<std::uint32_t*>(&ctl);
        constexpr std::uint32_t kStatus = offsetof(Ctl, status) / 4;
        for (std::uint32_t i = threadIdx.x; i < sizeof(Ctl) / 4; i += BS) {
            const std::uint32_t v = src[i];
            dst[i] = (i == kStatus && v == kYield) ? static_cast<std::uint32_t>(kRunning) : v;  // a yielded search resumes
        }
    }
    __syncthreads();
    BlockG<BS, LEAN> g{&ctl, sbuf, sd, si};
    slot_loop(g, S, C, sl, K, sh, Sm{&smc});
    __syncthreads();
    {
        const std::uint32_t* src = reinterpret_cast<const std::uint32_t*>(&ctl);
        std::uint32_t* dst = reinterpret_cast<std::uint32_t*>(sl.ctl());
        for (std::uint32_t i = threadIdx.x; i < sizeof(Ctl) / 4; i += BS) dst[i] = src[i];
    }
}

// Every CTA of a cooperative grid works on slot 0.
template <int BS>
__global__ void __launch_bounds__(BS, 1)
    grid_kernel(const __grid_constant__ Static S, const __grid_constant__ Config C,
                const __grid_constant__ SlotLayout L, const __grid_constant__ Caps K, Shared* sh,
                unsigned long long* partial, double* pd, std::uint32_t* pi, const __grid_constant__ SmemCfg smc) {
    __shared__ unsigned long long sbuf[BS / 32 + 4];
    __shared__ double sd[BS / 32];
    __shared__ std::uint32_t si[BS / 32];
    const Slot sl{L.base, &L};
    __shared__ unsigned long long gcnt[4];
    __shared__ std::uint32_t gsnap[4];
    __shared__ std::int32_t gscanq[BS / 32 * 32 * Search<GridG<BS>>::kExpandU];
    __shared__ std::uint32_t gscane[BS / 32 * 32 * Search<GridG<BS>>::kExpandU];
    GridG<BS> g{sl.ctl(), sh, partial, pd, pi, sbuf, sd, si, 0u, gcnt,
                *reinterpret_cast<volatile std::uint32_t*>(sh->arrive + blockIdx.x), gsnap, gscanq, gscane, false};
    if (g.leader() && sl.ctl()->status == kYield) sl.ctl()->status = kRunning;
    g.sync();
    slot_loop(g, S, C, sl, K, sh, Sm{&smc});
    g.persist();
}

// Low-level operations on one slot (Propagator-style API for tests and the
// propagation microbenchmark).
enum Op : std::uint32_t {
    kOpReset = 0, kOpInitial = 1, kOpPropagate = 2, kOpDecide = 3, kOpAssign = 4, kOpSeed = 5, kOpLearn = 6,
    kOpClearFrontier = 7
};

struct OpArgs {
    std::uint32_t op;
    std::uint32_t level;
    std::int32_t lit;
    std::int32_t antecedent;
    const std::int32_t* lits;  // bulk
    std::uint32_t n;
    const unsigned long long* deps;  // W words for kOpAssign
    std::uint32_t ovf;
};

// Ops recorded by a Session since its last launch run as one kernel, in order.
constexpr std::uint32_t kMaxOps = 6;
struct OpBatch {
    std::uint32_t n;
    OpArgs ops[kMaxOps];
};

template <class G>
__device__ void do_op(G& g, const Static& S, const Config& C, Slot sl, const Caps& K, Shared* sh,
                      const OpArgs& op, const Sm& sm, Search<G>& s) {
    Ctl* c = g.c;
    switch (op.op) {
        case kOpReset:
            s.begin_search(0);  // ends with a barrier
            if (g.leader()) c->phase = kLoop;  // not read before the kernel ends
            break;
        case kOpInitial: {
            if (g.leader()) {
                c->F = 0;
                c->n_confl = 0;
                c->opsnap[0] = c->st.propagations;
                c->opsnap[1] = c->st.passes;
                c->opsnap[2] = c->st.checks;
                c->opsnap[3] = c->st.checked_lits;
            }
            g.sync();
            const bool v = s.initial_propagation(true);
            if (g.leader()) c->b[10] = v;
            g.sync();
            break;
        }
        case kOpPropagate: {
            if (g.leader()) {
                if (s.nwords(op.level > c->cdl ? op.level : c->cdl) > s.nwords(op.level)) c->rows_wide = 1;
                c->n_confl = 0;
                c->opsnap[0] = c->st.propagations;
                c->opsnap[1] = c->st.passes;
                c->opsnap[2] = c->st.checks;
                c->opsnap[3] = c->st.checked_lits;
            }
            g.sync();
            const bool v = s.propagate(op.level);
            if (g.leader()) c->b[10] = v;
            g.sync();
            break;
        }
        case kOpDecide:  // push_decision(lit) (assignment.cpp:155-164)
            if (g.leader()) {
                const std::int32_t lit = op.lit;
                const std::uint32_t a = atom_of(lit);
                const std::uint32_t cdl = ++c->cdl;
                sl.ldec()[cdl] = lit;
                s.set_cell(a, lit > 0 ? static_cast<std::int32_t>(cdl) : -static_cast<std::int32_t>(cdl));
                sl.tpos()[a] = c->ts;
                sl.trail()[c->ts++] = lit;
                sl.reason()[a] = kReasonDecision;
                const std::uint32_t bit = cdl - 1;
                if (bit >= 64 * C.W) sl.dovf()[a] = 1;
                else s.dep(bit / 64, a) |= 1ull << (bit % 64);
            }
            g.sync();
            break;
        case kOpAssign: {  // assign_propagated for a bulk of literals (assignment.cpp:135-144):
                           // already assigned atoms are left alone (agreed / conflict) and
                           // only the first occurrence of a repeated atom counts
            const std::uint32_t ts0 = c->ts, gen = c->gen;
            // Deps words an atom at this level can use; more only when the caller's
            // words beyond them are not zero (then the next reset clears whole rows)
            std::uint32_t nw = s.nwords(op.level);
            if (op.deps)
                for (std::uint32_t w = nw; w < C.W; ++w)
                    if (op.deps[w]) nw = C.W;
            if (g.leader() && nw == C.W && s.nwords(op.level) < C.W) c->rows_wide = 1;
            for (std::uint32_t k = g.tid(); k < op.n; k += g.size()) {
                const std::uint32_t a = atom_of(op.lits[k]);
                if (a != 0 && a <= S.A) atomicMin(sl.win() + a, wkey(gen, k, false));  // atoms outside [1, A] are ignored
            }
            g.sync();
            unsigned long long carry = 0;
            for (std::uint32_t base = 0; base < op.n; base += g.size()) {
                const std::uint32_t k = base + g.tid();
                const std::int32_t lit = k < op.n ? op.lits[k] : 0;
                const std::uint32_t a = atom_of(lit);
                const bool fresh = k < op.n && a != 0 && a <= S.A && s.val(a) == 0 && sl.win()[a] == wkey(gen, k, false);
                unsigned long long tot;
                const std::uint32_t r = static_cast<std::uint32_t>(g.scan(fresh ? 1ull : 0ull, tot) + carry);
                if (fresh) {
                    s.set_cell(a, lit > 0 ? static_cast<std::int32_t>(op.level) : -static_cast<std::int32_t>(op.level));
                    sl.tpos()[a] = ts0 + r;
                    sl.trail()[ts0 + r] = lit;
                    sl.reason()[a] = op.antecedent;
                    for (std::uint32_t w = 0; w < nw; ++w) s.dep(w, a) = op.deps ? op.deps[w] : 0ull;  // the rest is zero
                    sl.dovf()[a] = static_cast<std::uint8_t>(op.ovf);
                }
                carry += tot;
            }
            g.sync();
            if (g.leader()) {
                c->ts = ts0 + static_cast<std::uint32_t>(carry);
                c->gen = gen + 1;
            }
            g.sync();
            break;
        }
        case kOpSeed: {  // frontier.last.push_back for a bulk of literals (at most A + 1 in total)
            const std::uint32_t F = c->F;
            if (static_cast<unsigned long long>(F) + op.n > S.A + 1ull) {
                g.sync();
                if (g.leader()) c->op_err = 1;
                g.sync();
                break;
            }
            for (std::uint32_t k = g.tid(); k < op.n; k += g.size()) sl.fr(c->cur)[F + k] = op.lits[k];
            g.sync();
            if (g.leader()) c->F = F + op.n;
            g.sync();
            break;
        }
        case kOpClearFrontier:  // Frontier::clear (assignment.hpp:160-163)
            if (g.leader()) c->F = 0;
            g.sync();
            break;
        case kOpLearn:  // NogoodStore::add_learned (kNoTruth guard)
            if (g.leader_warp()) {
                std::int32_t* buf = sl.scratch() + 128;
                for (std::uint32_t k = lane_id(); k < op.n; k += 32) buf[k] = op.lits[k];
                __syncwarp();
                s.w_sort(buf, op.n);
                const std::int32_t id = s.w_add_learned(buf, op.n);
                if (lane_id() == 0) c->b[12] = static_cast<std::uint32_t>(id);
            }
            g.sync();
            break;
        default:
            break;
    }
}

template <class G>
__device__ void do_ops(G& g, const Static& S, const Config& C, Slot sl, const Caps& K, Shared* sh,
                       const OpBatch& B, const Sm& sm) {
    Search<G> s(g, S, C, sl, K, sh, 0, sm);
    init_smem(g, s);
    for (std::uint32_t i = 0; i < B.n; ++i) do_op(g, S, C, sl, K, sh, B.ops[i], sm, s);  // each op ends with a barrier
}

template <int BS>
__global__ void __launch_bounds__(BS, 1)
    op_block_kernel(const __grid_constant__ Static S, const __grid_constant__ Config C,
                    const __grid_constant__ SlotLayout L, const __grid_constant__ Caps K, Shared* sh,
                    const __grid_constant__ OpBatch B, const __grid_constant__ SmemCfg smc) {
    __shared__ Ctl ctl;
    __shared__ unsigned long long sbuf[BS / 32 + 4];
    __shared__ double sd[BS / 32];
    __shared__ std::uint32_t si[BS / 32];
    const Slot sl{L.base, &L};
    {
        const std::uint32_t* src = reinterpret_cast<const std::uint32_t*>(sl.ctl());
        std::uint32_t* dst = reinterpret_cast<std::uint32_t*>(&ctl);
        for (std::uint32_t i = threadIdx.x; i < sizeof(Ctl) / 4; i += BS) dst[i] = src[i];
    }
    __syncthreads();
    BlockG<BS> g{&ctl, sbuf, sd, si};
    do_ops(g, S, C, sl, K, sh, B, Sm{&smc});
    __syncthreads();
    {
        const std::uint32_t* src = reinterpret_cast<const std::uint32_t*>(&ctl);
        std::uint32_t* dst = reinterpret_cast<std::uint32_t*>(sl.ctl());
        for (std::uint32_t i = threadIdx.x; i < sizeof(Ctl) / 4; i += BS) dst[i] = src[i];
    }
}

template <int BS>
__global__ void __launch_bounds__(BS, 1)
    op_grid_kernel(const __grid_constant__ Static S, const __grid_constant__ Config C,
                   const __grid_constant__ SlotLayout L, const __grid_constant__ Caps K, Shared* sh,
                   unsigned long long* partial, double* pd, std::uint32_t* pi, const __grid_constant__ OpBatch B,
                   const __grid_constant__ SmemCfg smc) {
    __shared__ unsigned long long sbuf[BS / 32 + 4];
    __shared__ double sd[BS / 32];
    __shared__ std::uint32_t si[BS / 32];
    const Slot sl{L.base, &L};
    __shared__ unsigned long long gcnt[4];
    __shared__ std::uint32_t gsnap[4];
    __shared__ std::int32_t gscanq[BS / 32 * 32 * Search<GridG<BS>>::kExpandU];
    __shared__ std::uint32_t gscane[BS / 32 * 32 * Search<GridG<BS>>::kExpandU];
    GridG<BS> g{sl.ctl(), sh, partial, pd, pi, sbuf, sd, si, 0u, gcnt,
                *reinterpret_cast<volatile std::uint32_t*>(sh->arrive + blockIdx.x), gsnap, gscanq, gscane, false};
    do_ops(g, S, C, sl, K, sh, B, Sm{&smc});
    g.persist();
}

// Per-slot initial values that are not zero.
__global__ void init_slots(const __grid_constant__ SlotLayout L, std::uint32_t A1, std::uint32_t items) {
    const Slot sl{L.base + static_cast<unsigned long long>(blockIdx.x) * L.bytes, &L};
    for (std::uint32_t i = threadIdx.x; i < items; i += blockDim.x) sl.claim()[i] = ~0ull;
    for (std::uint32_t i = threadIdx.x; i < A1; i += blockDim.x) {
        sl.win()[i] = ~0ull;
        sl.reason()[i] = kReasonNone;
    }
}

}  // namespace yas::dev

#include "engine_host.inl"
