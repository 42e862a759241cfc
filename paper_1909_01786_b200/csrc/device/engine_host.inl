// Host side of the engine: uploads, per-slot arenas, the launch/drain loop.
// Included at the end of engine.cu (needs the kernel templates).
#include <chrono>
#include <mutex>
#include <cstddef>
#include <cstdlib>

namespace yas {

namespace {

constexpr int kBlockBS = 256;
// Several searches per SM (cube enumeration, portfolios): two-warp CTAs — the
// one-warp passes run in warp 0, larger passes and rule scans use both; at 8
// per SM a search keeps 128 registers (q12 53.8 vs 55.5 ms for 4-warp CTAs
// capped at 64 registers, which spilled; 16 one-warp searches: 55.1 ms).
constexpr int kPairBS = 64;
constexpr int kGridBS = 512;

void ck(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw std::runtime_error(std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e));
}

// Arenas come from the device's stream-ordered memory pool, told to keep
// freed memory: a repeated solve (or the next cube batch) reuses the previous
// arena's pages instead of mapping gigabytes again.
void keep_pool(int device) {
    static bool done[64] = {false};
    if (device < 0 || device >= 64 || done[device]) return;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
        std::uint64_t keep = ~0ull;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
    done[device] = true;
}

template <class T>
T* dalloc(std::size_t n, std::vector<void*>& owned) {
    void* p = nullptr;
    int dev = 0;
    cudaGetDevice(&dev);
    keep_pool(dev);
    ck(cudaMallocAsync(&p, (n ? n : 1) * sizeof(T), nullptr), "cudaMallocAsync");
    owned.push_back(p);
    return static_cast<T*>(p);
}

template <class V>
typename V::value_type* dupload(const V& v, std::vector<void*>& owned) {
    using T = typename V::value_type;
    T* p = dalloc<T>(v.size(), owned);
    if (!v.empty()) ck(cudaMemcpy(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice), "upload");
    return p;
}

std::uint32_t pow2_at_least(std::uint64_t x) {
    std::uint32_t p = 1;
    while (p < x) p <<= 1;
    return p;
}

// All device memory of one run: static store + S slots.
// Pinned host staging for the drained models, grown on demand and kept by the
// host thread across calls (first-touch page faults of a fresh pageable buffer
// cost milliseconds per enumeration).
struct HostBuf {
    std::uint32_t* p = nullptr;
    std::size_t cap = 0;
    HostBuf() = default;
    HostBuf(const HostBuf&) = delete;
    HostBuf& operator=(const HostBuf&) = delete;
    ~HostBuf() {
        if (p) cudaFreeHost(p);
    }
    void reserve(std::size_t words) {
        if (words <= cap) return;
        const std::size_t ncap = std::max<std::size_t>(words, 2 * cap);
        if (p) cudaFreeHost(p);
        p = nullptr;
        cap = 0;
        ck(cudaMallocHost(&p, ncap * sizeof(std::uint32_t)), "cudaMallocHost models");
        cap = ncap;
    }
    std::uint32_t* data() const { return p; }
};
HostBuf& host_models_buf() {
    thread_local HostBuf b;
    return b;
}

// The createpolicy encodings of the expansion's two L2 policies, made on the
// device once per process (the encoding does not depend on the device).
void l2_policies(unsigned long long& first, unsigned long long& last) {
    static std::mutex mu;
    static bool made = false;
    static unsigned long long cached[2] = {0, 0};
    std::lock_guard<std::mutex> lock(mu);
    if (made) {
        first = cached[0];
        last = cached[1];
        return;
    }
    unsigned long long* d = nullptr;
    ck(cudaMalloc(&d, 2 * sizeof(unsigned long long)), "cudaMalloc");
    dev::make_l2_policies<<<1, 1>>>(d);
    unsigned long long h[2] = {0, 0};
    const cudaError_t e = cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
    cudaFree(d);
    ck(e, "L2 policies");
    first = cached[0] = h[0];
    last = cached[1] = h[1];
    made = true;
}

struct Arena {
    std::vector<void*> owned;
    dev::Static S{};
    dev::Caps K{};
    dev::SlotLayout L{};
    std::vector<dev::Slot> slots;
    dev::Shared* sh = nullptr;
    unsigned long long* partial = nullptr;
    double* pd = nullptr;
    std::uint32_t* pi = nullptr;
    std::uint32_t W = 16;
    std::uint32_t A = 0;

    ~Arena() {
        for (void* p : owned) cudaFreeAsync(p, nullptr);
        cudaStreamSynchronize(nullptr);
    }

    void upload_static(const StaticStore& st, const std::vector<RuleRec>& rules, std::uint32_t n_prog,
                       const std::vector<std::int32_t>& cubes) {
        l2_policies(S.pol_first, S.pol_last);
        S.A = st.total_atoms;
        S.n_prog = n_prog;
        S.N = st.size();
        S.n_units = static_cast<std::uint32_t>(st.units.size());
        S.n_uids = static_cast<std::uint32_t>(st.unit_ids.size());
        S.R = static_cast<std::uint32_t>(rules.size());
        S.off = dupload(st.off, owned);
        S.pool = dupload(st.pool, owned);
        S.guard = dupload(st.guard, owned);
        S.occ_off = dupload(st.occ_off, owned);
        {
            int4* occ = dalloc<int4>(st.occ_fat.size() / 4, owned);
            if (!st.occ_fat.empty())
                ck(cudaMemcpy(occ, st.occ_fat.data(), st.occ_fat.size() * 4, cudaMemcpyHostToDevice), "upload");
            S.occ = occ;
        }
        S.units = dupload(st.units, owned);
        S.uids = dupload(st.unit_ids, owned);
        std::vector<uint4> r(rules.size());
        for (std::size_t i = 0; i < rules.size(); ++i) r[i] = make_uint4(rules[i].head, rules[i].b, rules[i].t, rules[i].n);
        S.rules = dupload(r, owned);
        S.rules8 = nullptr;
        if (st.total_atoms < (1u << 21)) {
            std::vector<unsigned long long> r8(rules.size());
            for (std::size_t i = 0; i < rules.size(); ++i) {
                const unsigned long long n = rules[i].n & 0x7fffffffu, vac = rules[i].n >> 31;
                r8[i] = static_cast<unsigned long long>(rules[i].head) | static_cast<unsigned long long>(rules[i].t) << 21 |
                        n << 42 | vac << 63;
            }
            S.rules8 = dupload(r8, owned);
        }
        std::vector<std::uint32_t> so(static_cast<std::size_t>(st.total_atoms) + 1);
        for (std::uint32_t a = 0; a <= st.total_atoms; ++a) so[a] = st.occ_off[8ull * a + 8] - st.occ_off[8ull * a];
        S.socc = dupload(so, owned);
        S.cubes = dupload(cubes, owned);
        A = st.total_atoms;
    }

    void alloc_slots(std::uint32_t n_slots, std::uint32_t W_, std::uint32_t lcap, std::uint32_t lpool,
                     std::uint32_t mcap, std::uint32_t tcap, std::uint32_t cube_width, std::uint32_t grid_blocks) {
        W = W_;
        const std::size_t A1 = static_cast<std::size_t>(A) + 1;
        const std::size_t keys = (2 * static_cast<std::size_t>(A) + 2) * 4;
        K.lcap = lcap + cube_width + 1;
        K.lpool = lpool + cube_width + 1;
        K.larena = 4 * K.lpool + 64;
        K.items = S.N + K.lcap + S.n_units + 64;
        K.dupcap = pow2_at_least(2ull * K.lcap + 2);
        K.mcap = mcap;
        K.tcap = tcap;
        K.mwords = (S.n_prog + 31) / 32 ? (S.n_prog + 31) / 32 : 1;
        // expansion bitmap: bounded by the literal occurrences of the store
        // (static + learned) and by the initial-propagation item count.
        std::uint64_t tbits = std::max<std::uint64_t>(pool_size_ + K.lpool, S.n_units + S.n_uids + K.lcap) + 64;
        tbits = (tbits + 31) / 32 * 32;
        K.tbits = static_cast<std::uint32_t>(tbits);
        // one contiguous chunk per slot
        unsigned long long o = 0;
        auto take = [&](std::size_t bytes) {
            const unsigned long long at = o;
            o += (bytes + 255) & ~static_cast<std::size_t>(255);
            return at;
        };
        L.o_ctl = take(sizeof(dev::Ctl));
        L.o_cells = take(4 * A1);
        L.o_tpos = take(4 * A1);
        L.o_reason = take(4 * A1);
        L.o_deps = take(8 * static_cast<std::size_t>((W + 1) & ~1u) * A1);  // atom-major rows
        L.o_dovf = take(A1);
        L.o_trail = take(4 * A1);
        L.o_ldec = take(4 * (A1 + 1));
        L.o_fr0 = take(4 * A1);
        L.o_fr1 = take(4 * A1);
        L.o_froff = take(4 * (A1 + 1));
        L.o_claim = take(8ull * K.items);
        L.o_win = take(8 * A1);
        L.o_props = take(16ull * K.items);
        L.o_confl = take(4ull * K.items);
        L.o_pending = take(4 * 64);
        L.o_bitmap = take(tbits / 8);
        L.o_litat = take(4 * tbits);
        L.o_loff = take(4ull * (K.lcap + 1));
        L.o_lpool = take(4ull * K.lpool);
        L.o_lhdr = take(4 * keys * 3);
        L.o_larena = take(16ull * K.larena);
        L.o_lunits = take(4ull * K.lcap);
        L.o_ltot = take(4 * 2 * A1);
        L.o_act = take(8 * A1);
        L.o_dup = take(8ull * K.dupcap);
        L.o_scratch = take(4 * (2 * A1 + 512));  // ids/levels, learned literals, sort buffer
        L.o_mark = take(4 * A1);
        L.o_merged = take(8 * W);
        L.o_mbuf = take(4ull * mcap * K.mwords);
        L.o_mcube = take(4ull * mcap);
        L.o_tbuf = take(16ull * tcap);
        L.o_occat = take(grid_blocks ? 4 * tbits : 0);  // whole-grid passes only
        L.o_gmirror = take(grid_blocks ? 4 * ((A1 + 15) / 16 + 1) : 0);
        L.o_obat = take(grid_blocks ? 4 * tbits : 0);
        L.o_frb = take(grid_blocks ? 4 * (A1 + 1) : 0);
        L.bytes = o;
        L.base = dalloc<char>(static_cast<std::size_t>(o) * n_slots, owned);
        // Zero only what is read before it is written: the control block and
        // per-atom state, the expansion bitmap, the epoch-tagged duplicate table,
        // stamp marks and scratch, the grid mirror. Append-only arenas (learned
        // literals and occurrences, proposals, models) stay as they are; claim /
        // win / reason are set by init_slots; learned headers are cleared by the
        // first begin_search of a slot (epoch 0). Cube searches have ~1000 slots,
        // so this is a few hundred MB instead of the whole multi-GB arena.
        if (std::getenv("YAS_POISON_ARENA"))  // tests: nothing may depend on the rest being zero
            ck(cudaMemset(L.base, 0xA5, static_cast<std::size_t>(o) * n_slots), "memset");
        auto zero = [&](unsigned long long from, unsigned long long to) {
            if (to > from)
                ck(cudaMemset2D(L.base + from, o, 0, static_cast<std::size_t>(to - from), n_slots), "memset");
        };
        zero(L.o_ctl, L.o_claim);
        zero(L.o_pending, L.o_litat);
        zero(L.o_dup, L.o_tbuf);  // ... and the model buffers: the host copies whole strided rows
        // occat (place reads whole 128-byte lines, masking bits outside the word) and the grid mirror
        zero(L.o_occat, L.o_obat);
        dev::init_slots<<<n_slots, 256>>>(L, static_cast<std::uint32_t>(A1), K.items);
        ck(cudaGetLastError(), "init_slots");
        slots.resize(n_slots);
        for (std::uint32_t s = 0; s < n_slots; ++s) slots[s] = dev::Slot{L.base + static_cast<unsigned long long>(s) * o, &L};
        sh = dalloc<dev::Shared>(1, owned);
        ck(cudaMemset(sh, 0, sizeof(dev::Shared)), "memset");
        ck(cudaMemset(&sh->winner, 0xff, sizeof(std::uint32_t)), "memset");
        const std::uint32_t gb = grid_blocks ? grid_blocks : 1;
        partial = dalloc<unsigned long long>(4 * gb, owned);
        pd = dalloc<double>(gb, owned);
        pi = dalloc<std::uint32_t>(gb, owned);
    }

    std::size_t pool_size_ = 0;
};

// Shared-memory working set of a single-CTA search: pass scratch for up to
// tcap expansion entries plus the 2-bit assignment mirror, within `budget`.
dev::SmemCfg plan_smem(std::uint32_t atoms, std::size_t budget) {
    const std::uint32_t vw = (atoms + 1 + 31) / 32;
    const std::uint32_t vwords = 2ull * 4 * vw + 64 <= budget / 2 ? vw : 0;
    for (std::uint32_t t = 16384; t >= 128; t /= 2) {
        const dev::SmemCfg x = dev::smem_layout(t, vwords);
        if (x.bytes <= budget) return x;
    }
    return dev::smem_layout(0, vwords);
}

// Whole-grid propagation hands passes of at most this many expansion entries to
// block 0 alone, with the single-CTA pass's working set in shared memory
// (YAS_GRID_SOLO_T overrides; 0 disables).
dev::SmemCfg grid_smem() {
    std::uint32_t t = 256;
    if (const char* e = std::getenv("YAS_GRID_SOLO_T")) t = static_cast<std::uint32_t>(std::strtoul(e, nullptr, 10));
    return dev::smem_layout(t, 0);
}

std::uint32_t grid_blocks_for(int device) {
    int sms = 0, per = 0;
    ck(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device), "attr");
    ck(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, dev::grid_kernel<kGridBS>, kGridBS, 0), "occupancy");
    if (per < 1) per = 1;
    return static_cast<std::uint32_t>(sms) * 1u;  // one CTA per SM: cheapest grid barrier
}

}  // namespace

std::string device_name(int device) {
    cudaDeviceProp p{};
    if (cudaGetDeviceProperties(&p, device) != cudaSuccess) return "unavailable";
    return p.name;
}

template <bool LEAN>
void launch_blocks(std::uint32_t per_sm, std::uint32_t n_slots, std::size_t smem, Arena& ar, const dev::Config& cfg,
                   const dev::SmemCfg& smc) {
    if (per_sm > 6)
        dev::block_kernel<kPairBS, 8, LEAN><<<n_slots, kPairBS, smem>>>(ar.S, cfg, ar.L, ar.K, ar.sh, smc);
    else if (per_sm > 4)
        dev::block_kernel<kPairBS, 6, LEAN><<<n_slots, kPairBS, smem>>>(ar.S, cfg, ar.L, ar.K, ar.sh, smc);
    else if (per_sm > 1)
        dev::block_kernel<kPairBS, 4, LEAN><<<n_slots, kPairBS, smem>>>(ar.S, cfg, ar.L, ar.K, ar.sh, smc);
    else
        dev::block_kernel<kBlockBS, 1, LEAN><<<n_slots, kBlockBS, smem>>>(ar.S, cfg, ar.L, ar.K, ar.sh, smc);
}

EngineResult engine_solve(const EngineProgram& prog, const dev::Config& cfg_in, const EngineOptions& opt,
                          const std::vector<std::int32_t>& cubes, std::uint32_t n_cubes,
                          std::uint32_t cube_width, const EngineCallbacks& cb) {
    ck(cudaSetDevice(opt.device), "cudaSetDevice");
    const auto w0 = std::chrono::steady_clock::now();
    EngineResult res;
    Arena ar;
    ar.pool_size_ = prog.store->pool.size();
    ar.upload_static(*prog.store, prog.rules, prog.n_prog, cubes);
    const std::uint32_t gblocks = opt.grid ? grid_blocks_for(opt.device) : 0;
    const std::uint32_t n_slots = opt.grid ? 1u : std::max<std::uint32_t>(1, std::min(opt.slots, n_cubes));
    ar.alloc_slots(n_slots, cfg_in.W, opt.lcap, opt.lpool, opt.mcap, opt.tcap, cube_width, gblocks);
    if (std::getenv("YAS_PROFILE")) {
        cudaDeviceSynchronize();
        std::fprintf(stderr, "[yas host] arena: %u slots x %.2f MB, ready after %.2f ms\n", n_slots, ar.L.bytes / 1e6,
                     std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - w0).count());
    }
    dev::Config cfg = cfg_in;
    cfg.n_cubes = n_cubes;
    cfg.phase_prof = std::getenv("YAS_PROFILE") ? 1u : 0u;
    cfg.cube_width = cube_width;
    cfg.slice_ns = static_cast<std::uint64_t>(opt.slice_ms * 1e6);
    cfg.fleet = opt.fleet;
    cfg.fleet_tag = opt.fleet_tag;

    cudaEvent_t e0, e1;
    ck(cudaEventCreate(&e0), "event");
    ck(cudaEventCreate(&e1), "event");
    std::vector<dev::Ctl> ctl(n_slots);
    std::vector<std::uint32_t> counts;
    HostBuf& mb = host_models_buf();  // pinned, kept by this host thread across calls
    dev::SmemCfg smc{};
    std::size_t smem = 0;
    std::uint32_t per_sm = 1;
    if (opt.grid) {
        smc = grid_smem();
        smem = smc.bytes;
        ck(cudaFuncSetAttribute(reinterpret_cast<const void*>(dev::grid_kernel<kGridBS>),
                                cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)),
           "smem attribute");
    }
    if (!opt.grid) {
        int sms = 148;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, opt.device);
        per_sm = std::min<std::uint32_t>(8, (n_slots + sms - 1) / sms);
        if (per_sm > 6) per_sm = 8;  // several searches per SM: two-warp CTAs (64, 6 or 4 per SM)
        else if (per_sm > 4) per_sm = 6;
        else if (per_sm > 1) per_sm = 4;
        // keep most of the unified L1 for the (read-only) static store
        std::size_t budget = per_sm == 1 ? 96u * 1024u : (227u * 1024u) / per_sm - 3072;
        if (const char* kb = std::getenv("YAS_SMEM_KB")) budget = std::min<std::size_t>(budget, std::strtoul(kb, nullptr, 10) * 1024u);
        smc = plan_smem(ar.A, budget);
        smem = smc.bytes;
        // several searches per SM: one-warp passes up to 256 entries (q12 55 vs 61 ms at
        // 96); a lone search: 96 (ham200 107 vs 110 ms at 160)
        cfg.warp_pass_t = per_sm > 1 ? 256u : 96u;
        if (const char* e = std::getenv("YAS_WARP_PASS_T")) cfg.warp_pass_t = static_cast<std::uint32_t>(std::strtoul(e, nullptr, 10));
        // portfolio searches race each other: one per SM (a CTA needs more than half the array)
        if (cfg.portfolio) smem = std::max<std::size_t>(smem, 116u * 1024u);
        // the rest of the 228 KB unified array stays L1 for the static store
        const int carve = static_cast<int>(std::min<std::size_t>(100, (per_sm * (smem + 4096) * 100 + 228 * 1024 - 1) / (228 * 1024)));
        for (auto fn : {reinterpret_cast<const void*>(dev::block_kernel<kBlockBS, 1>),
                        reinterpret_cast<const void*>(dev::block_kernel<kPairBS, 4>),
                        reinterpret_cast<const void*>(dev::block_kernel<kPairBS, 6>),
                        reinterpret_cast<const void*>(dev::block_kernel<kPairBS, 8>),
                        reinterpret_cast<const void*>(dev::block_kernel<kBlockBS, 1, true>),
                        reinterpret_cast<const void*>(dev::block_kernel<kPairBS, 4, true>),
                        reinterpret_cast<const void*>(dev::block_kernel<kPairBS, 6, true>),
                        reinterpret_cast<const void*>(dev::block_kernel<kPairBS, 8, true>)}) {
            ck(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)),
               "smem attribute");
            ck(cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, carve), "carveout");
        }
    }
    // the default configuration runs on kernels with everything else compiled out
    bool lean = cfg.mode == 0 && cfg.heur == 0 && !cfg.portfolio && !cfg.trace && !cfg.debug_validate &&
                !cfg.phase_prof && cfg.fanout <= 1 && !cfg.restarts;
    if (const char* e = std::getenv("YAS_LEAN")) lean = lean && std::strtoul(e, nullptr, 10) != 0;
    bool stop_early = false;
    std::uint32_t winner = ~0u;  // portfolio: the search that finished first
    for (;;) {
        ck(cudaEventRecord(e0), "record");
        if (opt.grid) {
            void* args[] = {&ar.S, &cfg, &ar.L, &ar.K, &ar.sh, &ar.partial, &ar.pd, &ar.pi, &smc};
            ck(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(dev::grid_kernel<kGridBS>), dim3(gblocks),
                                           dim3(kGridBS), args, smem, nullptr),
               "grid launch");
        } else {
            if (lean) launch_blocks<true>(per_sm, n_slots, smem, ar, cfg, smc);
            else launch_blocks<false>(per_sm, n_slots, smem, ar, cfg, smc);
            ck(cudaGetLastError(), "block launch");
        }
        ck(cudaEventRecord(e1), "record");
        ck(cudaEventSynchronize(e1), "kernel");
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        res.device_ms += ms;
        ++res.launches;
        const bool laps = std::getenv("YAS_PROFILE") != nullptr;
        auto lap = [&](const char* what) {
            if (laps)
                std::fprintf(stderr, "[yas host]   %s at %.2f ms\n", what,
                             std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - w0).count());
        };
        lap("kernel done");
        ck(cudaMemcpy2D(ctl.data(), sizeof(dev::Ctl), ar.slots[0].ctl(), ar.L.bytes, sizeof(dev::Ctl), n_slots,
                        cudaMemcpyDeviceToHost),
           "ctl");
        lap("ctl copied");
        bool more = false;
        std::uint32_t err = dev::kDone;
        // all slots' model buffers in two strided copies (not two per slot)
        std::uint32_t maxm = 0;
        for (std::uint32_t s = 0; s < n_slots; ++s) maxm = std::max(maxm, ctl[s].n_mbuf);
        if (maxm) {
            const std::size_t mrow = static_cast<std::size_t>(maxm) * ar.K.mwords * 4;
            const std::size_t bits_words = mrow / 4 * n_slots;
            mb.reserve(bits_words + static_cast<std::size_t>(maxm) * n_slots);
            ck(cudaMemcpy2D(mb.data(), mrow, ar.slots[0].mbuf(), ar.L.bytes, mrow, n_slots, cudaMemcpyDeviceToHost),
               "models");
            ck(cudaMemcpy2D(mb.data() + bits_words, 4ull * maxm, ar.slots[0].mcube(), ar.L.bytes, 4ull * maxm, n_slots,
                            cudaMemcpyDeviceToHost),
               "models");
        }
        // portfolio: only the search that claimed the first finish reports (its
        // model, or UNSAT); with a fleet it may be on another GPU / process
        winner = ~0u;
        if (cfg.portfolio)
            for (std::uint32_t s = 0; s < n_slots; ++s)
                if (ctl[s].status == dev::kDone && ctl[s].won) winner = s;
        lap("models copied");
        if (maxm) {  // one drain for every slot's models (decoded on the host threads)
            counts.assign(n_slots, 0u);
            for (std::uint32_t s = 0; s < n_slots; ++s)
                if (!(cfg.portfolio && s != winner)) counts[s] = ctl[s].n_mbuf;
            EngineDrain dr;
            dr.bits = mb.data();
            dr.cubes = mb.data() + static_cast<std::size_t>(maxm) * ar.K.mwords * n_slots;
            dr.counts = counts.data();
            dr.n_slots = n_slots;
            dr.stride = maxm;
            dr.nwords = ar.K.mwords;
            if (cb.on_models && !cb.on_models(dr)) stop_early = true;
        }
        for (std::uint32_t s = 0; s < n_slots; ++s) {
            dev::Ctl& c = ctl[s];
            c.n_mbuf = 0;
            if (c.n_trace) {
                std::vector<uint4> tb(c.n_trace);
                ck(cudaMemcpy(tb.data(), ar.slots[s].tbuf(), tb.size() * sizeof(uint4), cudaMemcpyDeviceToHost), "trace");
                if (cb.on_trace)
                    for (const uint4& t : tb) cb.on_trace(t.x, static_cast<std::int32_t>(t.y), t.z, t.w);
                c.n_trace = 0;
            }
            if (c.status == dev::kYield) more = true;
            else if (c.status != dev::kDone && c.status != dev::kRunning) err = c.status;
        }
        lap("models delivered");
        if (err != dev::kDone) {
            res.status = err;
            break;
        }
        if (!more || stop_early || winner != ~0u) break;
        ck(cudaMemcpy2D(ar.slots[0].ctl(), ar.L.bytes, ctl.data(), sizeof(dev::Ctl), sizeof(dev::Ctl), n_slots,
                        cudaMemcpyHostToDevice),
           "ctl");
        ck(cudaMemset(&ar.sh->stop, 0, sizeof(std::uint32_t)), "stop");
    }
    dev::Stats tot{};
    auto add = [](dev::Stats& a, const dev::Stats& b) {
        const unsigned long long* pb = &b.decisions;
        unsigned long long* pa = &a.decisions;
        for (std::size_t i = 0; i < sizeof(dev::Stats) / 8; ++i) pa[i] += pb[i];
    };
    for (const dev::Ctl& c : ctl) add(tot, c.st);
    if (winner != ~0u) {  // portfolio: the winning search's trajectory, and how many ran
        const unsigned long long searches = tot.searches;
        tot = ctl[winner].st;
        tot.searches = searches;
        res.variant = ctl[winner].variant;
        res.won = true;
    }
    res.stats = tot;
    if (std::getenv("YAS_PROFILE")) {
        std::fprintf(stderr, "[yas host]   engine end at %.2f ms\n",
                     std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - w0).count());
        static const char* names[16] = {"loop", "offsets", "expand", "resolve", "apply", "compact", "decide",
                                        "conflict", "tiny", "warp", "n.tiny", "looptop", "n.smem", "n.global", "x14", "x15"};
        unsigned long long p[16] = {0};
        for (const dev::Ctl& c : ctl)
            for (int k = 0; k < 16; ++k) p[k] += c.prof[k];
        std::fprintf(stderr, "[yas profile] passes=%llu", static_cast<unsigned long long>(tot.passes));
        for (int k = 1; k < 16; ++k) std::fprintf(stderr, " %s=%.2fM", names[k], p[k] / 1e6);
        std::fprintf(stderr, "\n");
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    res.wall_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - w0).count();
    return res;
}

// ---------------------------------------------------------------------------
// Session
// ---------------------------------------------------------------------------
struct Session::Impl {
    Arena ar;
    dev::SmemCfg smc{};
    std::size_t smem = 0;
    dev::Config cfg{};
    bool grid = false;
    std::uint32_t gblocks = 0;
    int device = 0;
    cudaStream_t stream{};
    cudaEvent_t e0{}, e1{};
    // Ops are recorded host-side and launched together, as one kernel, when a
    // result is needed (initial propagation, propagation, add_learned, any
    // read-back) or the batch is full. Bulk inputs of a batch are packed into
    // one pinned staging buffer and uploaded with one copy; the control block
    // comes back into pinned memory behind every launch.
    std::vector<dev::OpArgs> pending;
    std::vector<std::size_t> lits_off, deps_off;  // staging offsets (ints) per pending op, ~0 = none
    std::int32_t* h_stage = nullptr;               // pinned
    std::size_t h_stage_cap = 0, h_used = 0;
    cudaEvent_t staged{};                          // the last upload of h_stage has been consumed
    bool stage_inflight = false;
    std::int32_t* d_stage = nullptr;
    std::size_t d_stage_cap = 0;
    std::size_t h_uploaded = 0;  // prefix of this batch's staging already sent (bulk inputs go early)
    dev::Ctl* h_ctl = nullptr;  // pinned mirror of the slot's control block
    bool ctl_pending = false;
    // bytes moved between host and device by this session (staged inputs, kernel
    // arguments, control blocks, read-backs): counted, for end-to-end accounting
    mutable unsigned long long h2d_bytes = 0, d2h_bytes = 0;

    // check: the ints are literals that must name atoms in [1, atoms] (checked
    // while they are copied; nothing is staged when one does not)
    std::size_t append(const void* src, std::size_t ints, bool check = false, std::uint32_t atoms = 0) {
        if (stage_inflight) {  // the previous batch's upload may still read the buffer
            ck(cudaEventSynchronize(staged), "staging");
            stage_inflight = false;
        }
        const std::size_t off = (h_used + 3) & ~static_cast<std::size_t>(3);  // 16-byte aligned entries
        if (off + ints > h_stage_cap) {
            const std::size_t ncap = std::max<std::size_t>(off + ints, 2 * h_stage_cap + 1024);
            std::int32_t* nb = nullptr;
            ck(cudaMallocHost(&nb, ncap * sizeof(std::int32_t)), "cudaMallocHost staging");
            if (h_uploaded) ck(cudaStreamSynchronize(stream), "staging");  // early uploads read the old buffer
            if (h_stage) {
                std::memcpy(nb, h_stage, h_used * sizeof(std::int32_t));
                cudaFreeHost(h_stage);
            }
            h_stage = nb;
            h_stage_cap = ncap;
        }
        if (check) {
            const std::int32_t* in = static_cast<const std::int32_t*>(src);
            std::int32_t* out = h_stage + off;
            std::uint32_t bad = 0;  // branch-free: the copy-and-check loop vectorises
            for (std::size_t k = 0; k < ints; ++k) {
                const std::int32_t l = in[k];
                const std::uint32_t a = l < 0 ? 0u - static_cast<std::uint32_t>(l) : static_cast<std::uint32_t>(l);
                bad |= (a - 1u) >= atoms ? 1u : 0u;  // atom 0 or above the range
                out[k] = l;
            }
            if (bad) throw std::invalid_argument("seed: literal out of range");
        } else if (ints) {
            std::memcpy(h_stage + off, src, ints * sizeof(std::int32_t));
        }
        h_used = off + ints;
        // a bulk input starts its upload now, overlapping the caller's next
        // calls; the launch copies only what is left (stream order keeps it
        // behind the previous kernel, which may still read d_stage)
        if (ints >= kEagerInts && h_used <= d_stage_cap) {
            ck(cudaMemcpyAsync(d_stage + h_uploaded, h_stage + h_uploaded, (h_used - h_uploaded) * sizeof(std::int32_t),
                               cudaMemcpyHostToDevice, stream),
               "stage");
            h2d_bytes += (h_used - h_uploaded) * sizeof(std::int32_t);
            h_uploaded = h_used;
        }
        return off;
    }
    static constexpr std::size_t kEagerInts = 4096;
};

Session::Session(const StaticStore& store, std::uint32_t deps_words, bool grid, int device, std::uint32_t lcap,
                 std::uint32_t lpool)
    : impl_(new Impl), W_(deps_words) {
    ck(cudaSetDevice(device), "cudaSetDevice");
    impl_->device = device;
    impl_->grid = grid;
    impl_->ar.pool_size_ = store.pool.size();
    impl_->ar.upload_static(store, {}, 0, {});
    impl_->gblocks = grid ? grid_blocks_for(device) : 0;
    impl_->ar.alloc_slots(1, deps_words, lcap, lpool, 16, 128, 0, impl_->gblocks);
    if (!grid) {
        impl_->smc = plan_smem(impl_->ar.A, 96u * 1024u);
        impl_->smem = impl_->smc.bytes;
        ck(cudaFuncSetAttribute(dev::op_block_kernel<kBlockBS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(impl_->smem)),
           "smem attribute");
    } else {
        impl_->smc = grid_smem();
        impl_->smem = impl_->smc.bytes;
        ck(cudaFuncSetAttribute(dev::op_grid_kernel<kGridBS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(impl_->smem)),
           "smem attribute");
    }
    dev::Config& c = impl_->cfg;
    c.W = deps_words;
    c.decay = 0.95;
    c.restart_base = 100;
    c.restart_factor = 1.5;
    c.fanout = 1;
    c.learned_capacity = ~0ull;
    c.n_cubes = 1;
    c.warp_pass_t = 96;
    // the arena was uploaded / zeroed / initialised on the legacy stream; the
    // session's non-blocking stream is not ordered after it
    ck(cudaDeviceSynchronize(), "arena setup");
    ck(cudaStreamCreateWithFlags(&impl_->stream, cudaStreamNonBlocking), "stream");
    ck(cudaEventCreate(&impl_->e0), "event");
    ck(cudaEventCreate(&impl_->e1), "event");
    ck(cudaEventCreateWithFlags(&impl_->staged, cudaEventDisableTiming), "event");
    ck(cudaMallocHost(&impl_->h_ctl, sizeof(dev::Ctl)), "cudaMallocHost");
    std::memset(impl_->h_ctl, 0, sizeof(dev::Ctl));
    reset();
}

Session::~Session() {
    cudaStreamSynchronize(impl_->stream);
    if (impl_->d_stage) cudaFree(impl_->d_stage);
    if (impl_->h_stage) cudaFreeHost(impl_->h_stage);
    cudaEventDestroy(impl_->staged);
    cudaFreeHost(impl_->h_ctl);
    cudaEventDestroy(impl_->e0);
    cudaEventDestroy(impl_->e1);
    cudaStreamDestroy(impl_->stream);
}

namespace {
// Launch the recorded ops as one kernel (plus the control-block copy behind
// it). `ms` (when given) waits for the kernel and returns its CUDA-event time.
void flush_ops(Session::Impl& im, float* ms) {
    if (im.pending.empty()) return;
    if (im.h_used) {
        if (im.h_used > im.d_stage_cap) {
            ck(cudaStreamSynchronize(im.stream), "stream");  // the old buffer may still be read
            if (im.d_stage) cudaFree(im.d_stage);
            im.d_stage_cap = std::max<std::size_t>(im.h_used, 2 * im.d_stage_cap);
            ck(cudaMalloc(&im.d_stage, im.d_stage_cap * sizeof(std::int32_t)), "cudaMalloc staging");
            im.h_uploaded = 0;  // early uploads went to the old buffer
        }
        if (im.h_used > im.h_uploaded)
            ck(cudaMemcpyAsync(im.d_stage + im.h_uploaded, im.h_stage + im.h_uploaded,
                               (im.h_used - im.h_uploaded) * sizeof(std::int32_t), cudaMemcpyHostToDevice, im.stream),
               "stage");
        if (im.h_used > im.h_uploaded) im.h2d_bytes += (im.h_used - im.h_uploaded) * sizeof(std::int32_t);
        ck(cudaEventRecord(im.staged, im.stream), "record");
        im.stage_inflight = true;
    }
    dev::OpBatch b{};
    b.n = static_cast<std::uint32_t>(im.pending.size());
    for (std::uint32_t i = 0; i < b.n; ++i) {
        b.ops[i] = im.pending[i];
        if (im.lits_off[i] != ~static_cast<std::size_t>(0)) b.ops[i].lits = im.d_stage + im.lits_off[i];
        if (im.deps_off[i] != ~static_cast<std::size_t>(0))
            b.ops[i].deps = reinterpret_cast<const unsigned long long*>(im.d_stage + im.deps_off[i]);
    }
    im.pending.clear();
    im.lits_off.clear();
    im.deps_off.clear();
    im.h_used = 0;
    im.h_uploaded = 0;
    ck(cudaEventRecord(im.e0, im.stream), "record");
    if (im.grid) {
        void* args[] = {&im.ar.S, &im.cfg, &im.ar.L, &im.ar.K, &im.ar.sh, &im.ar.partial, &im.ar.pd, &im.ar.pi, &b,
                        &im.smc};
        ck(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(dev::op_grid_kernel<kGridBS>), dim3(im.gblocks),
                                       dim3(kGridBS), args, im.smem, im.stream),
           "op grid launch");
    } else {
        dev::op_block_kernel<kBlockBS><<<1, kBlockBS, im.smem, im.stream>>>(im.ar.S, im.cfg, im.ar.L, im.ar.K, im.ar.sh,
                                                                          b, im.smc);
        ck(cudaGetLastError(), "op launch");
    }
    ck(cudaEventRecord(im.e1, im.stream), "record");
    ck(cudaMemcpyAsync(im.h_ctl, im.ar.slots[0].ctl(), sizeof(dev::Ctl), cudaMemcpyDeviceToHost, im.stream), "ctl");
    im.h2d_bytes += sizeof(dev::OpBatch);  // the recorded ops travel as kernel arguments
    im.d2h_bytes += sizeof(dev::Ctl);
    im.ctl_pending = true;
    if (ms) {
        ck(cudaEventSynchronize(im.e1), "op kernel");
        cudaEventElapsedTime(ms, im.e0, im.e1);
    }
}

// Record one op (with optional staged literals / Deps words); a full batch is
// launched right away.
void record_op(Session::Impl& im, const dev::OpArgs& op, const std::int32_t* lits = nullptr, std::size_t n = 0,
               const unsigned long long* deps = nullptr, std::size_t nd = 0, bool check = false,
               std::uint32_t atoms = 0) {
    const std::size_t none = ~static_cast<std::size_t>(0);
    im.lits_off.push_back(lits ? im.append(lits, n, check, atoms) : none);
    im.deps_off.push_back(deps ? im.append(deps, 2 * nd) : none);
    im.pending.push_back(op);
    if (im.pending.size() == dev::kMaxOps) flush_ops(im, nullptr);
}
}  // namespace

void Session::flush() { flush_ops(*impl_, nullptr); }  // asynchronous: a rejected op raises at the next result

void Session::reset() {
    dev::OpArgs op{};
    op.op = dev::kOpReset;
    record_op(*impl_, op);
}

bool Session::initial_propagation() {
    dev::OpArgs op{};
    op.op = dev::kOpInitial;
    record_op(*impl_, op);
    flush_ops(*impl_, &last_ms_);
    const bool v = ctl().b[10] != 0;
    check_op_error();
    return v;
}

bool Session::propagate(std::uint32_t level) {
    dev::OpArgs op{};
    op.op = dev::kOpPropagate;
    op.level = level;
    record_op(*impl_, op);
    flush_ops(*impl_, &last_ms_);
    const bool v = ctl().b[10] != 0;
    check_op_error();
    return v;
}

void Session::push_decision(std::int32_t lit) {
    dev::OpArgs op{};
    op.op = dev::kOpDecide;
    op.lit = lit;
    record_op(*impl_, op);
}

void Session::assign(const std::int32_t* lits_in, std::size_t n_in, std::uint32_t level, std::int32_t antecedent,
                     const unsigned long long* deps, std::size_t n_deps, bool ovf) {
    Impl& im = *impl_;  // out-of-range atoms and repeats are resolved on the device
    const std::int32_t* lits = lits_in;
    std::vector<unsigned long long> d(W_, 0ull);
    for (std::size_t i = 0; i < n_deps && i < W_; ++i) d[i] = deps[i];
    dev::OpArgs op{};
    op.op = dev::kOpAssign;
    op.level = level;
    op.antecedent = antecedent;
    op.n = static_cast<std::uint32_t>(n_in);
    op.ovf = ovf ? 1u : 0u;
    record_op(im, op, lits, n_in, d.data(), W_);
}

void Session::seed(const std::int32_t* lits, std::size_t n) {
    const std::uint32_t A = impl_->ar.A;
    if (n > static_cast<std::size_t>(A) + 1) throw std::invalid_argument("seed: more literals than atoms");
    dev::OpArgs op{};
    op.op = dev::kOpSeed;
    op.n = static_cast<std::uint32_t>(n);
    record_op(*impl_, op, lits, n, nullptr, 0, true, A);  // the literals are range-checked while staged
}

void Session::clear_frontier() {
    dev::OpArgs op{};
    op.op = dev::kOpClearFrontier;
    record_op(*impl_, op);
}

std::int32_t Session::add_learned(const std::vector<std::int32_t>& lits_in) {
    // NogoodStore::add_learned takes a canonical Nogood (nogood.hpp:80-87):
    // atoms in [1, A], sorted, no repeats, never both signs of one atom
    for (std::int32_t l : lits_in)
        if (l == 0 || lit_atom(l) > impl_->ar.A) throw std::invalid_argument("add_learned: literal out of range");
    auto ng = Nogood::make(lits_in, kLearned, kNoTruth);
    if (!ng) throw std::invalid_argument("add_learned: vacuous nogood (both signs of one atom)");
    if (ng->lits.empty()) throw std::invalid_argument("add_learned: empty nogood");
    const std::vector<std::int32_t>& lits = ng->lits;
    dev::OpArgs op{};
    op.op = dev::kOpLearn;
    op.n = static_cast<std::uint32_t>(lits.size());
    record_op(*impl_, op, lits.data(), lits.size());
    flush_ops(*impl_, nullptr);
    const std::int32_t id = static_cast<std::int32_t>(ctl().b[12]);
    check_op_error();
    return id;
}

void Session::check_op_error() const {
    dev::Ctl& c = *impl_->h_ctl;
    if (!c.op_err) return;
    c.op_err = 0;  // cleared on both sides: the session stays usable
    const std::uint32_t zero = 0;
    ck(cudaMemcpyAsync(reinterpret_cast<char*>(impl_->ar.slots[0].ctl()) + offsetof(dev::Ctl, op_err), &zero,
                       sizeof zero, cudaMemcpyHostToDevice, impl_->stream),
       "clear op error");
    ck(cudaStreamSynchronize(impl_->stream), "clear op error");
    throw std::invalid_argument("seed: frontier capacity exceeded (more than A + 1 frontier literals)");
}

void Session::set_count_lits(bool on) { impl_->cfg.count_lits = on ? 1u : 0u; }

void Session::set_pass_trace(bool on) {
    Impl& im = *impl_;
    const std::size_t n = 64ull * std::max<std::uint32_t>(1, im.gblocks) * 10 + 64 * 16;
    if (on && !im.cfg.ptrace) {
        ck(cudaMallocAsync(&im.cfg.ptrace, n * sizeof(unsigned long long), nullptr), "cudaMallocAsync trace");
        ck(cudaMemset(im.cfg.ptrace, 0, n * sizeof(unsigned long long)), "memset trace");
        im.ar.owned.push_back(im.cfg.ptrace);
    } else if (!on) {
        im.cfg.ptrace = nullptr;  // freed with the arena
    }
}


const dev::Ctl& Session::ctl() const {
    flush_ops(*impl_, nullptr);
    if (impl_->ctl_pending) {
        ck(cudaStreamSynchronize(impl_->stream), "stream");
        impl_->ctl_pending = false;
    }
    return *impl_->h_ctl;
}

namespace {
template <class T>
std::size_t dl_into(const T* p, std::size_t n, T* out, cudaStream_t s, unsigned long long& counted) {
    if (n) {
        ck(cudaMemcpyAsync(out, p, n * sizeof(T), cudaMemcpyDeviceToHost, s), "download");
        ck(cudaStreamSynchronize(s), "download");
        counted += n * sizeof(T);
    }
    return n;
}
template <class T>
std::vector<T> dl(const T* p, std::size_t n, cudaStream_t s, unsigned long long& counted) {
    std::vector<T> v(n);
    dl_into(p, n, v.data(), s, counted);
    return v;
}
}  // namespace

void Session::transfers(unsigned long long& h2d, unsigned long long& d2h) const {
    h2d = impl_->h2d_bytes;
    d2h = impl_->d2h_bytes;
}

std::size_t Session::trail_into(std::int32_t* out, std::size_t cap) const {
    const std::size_t n = ctl().ts;
    if (out && cap >= n) dl_into(impl_->ar.slots[0].trail(), n, out, impl_->stream, impl_->d2h_bytes);
    else if (out && cap) dl_into(impl_->ar.slots[0].trail(), cap, out, impl_->stream, impl_->d2h_bytes);
    return n;
}

std::vector<std::int32_t> Session::cells() const {
    flush_ops(*impl_, nullptr);
    return dl(impl_->ar.slots[0].cells(), impl_->ar.A + 1, impl_->stream, impl_->d2h_bytes);
}
std::vector<std::int32_t> Session::trail() const { return dl(impl_->ar.slots[0].trail(), ctl().ts, impl_->stream, impl_->d2h_bytes); }
std::vector<std::int32_t> Session::reasons() const {
    flush_ops(*impl_, nullptr);
    return dl(impl_->ar.slots[0].reason(), impl_->ar.A + 1, impl_->stream, impl_->d2h_bytes);
}
std::vector<unsigned long long> Session::deps_word(std::uint32_t w) const {
    flush_ops(*impl_, nullptr);
    const std::size_t stride = (W_ + 1) & ~1u, n = impl_->ar.A + 1;
    const std::vector<unsigned long long> rows = dl(impl_->ar.slots[0].deps(), n * stride, impl_->stream, impl_->d2h_bytes);
    std::vector<unsigned long long> v(n);
    for (std::size_t a = 0; a < n; ++a) v[a] = rows[a * stride + w];
    return v;
}
std::vector<std::uint8_t> Session::deps_overflow() const {
    flush_ops(*impl_, nullptr);
    return dl(impl_->ar.slots[0].dovf(), impl_->ar.A + 1, impl_->stream, impl_->d2h_bytes);
}
std::vector<std::int32_t> Session::conflicts() const { return dl(impl_->ar.slots[0].confl(), ctl().n_confl, impl_->stream, impl_->d2h_bytes); }
std::vector<std::int32_t> Session::frontier() const {
    const dev::Ctl& c = ctl();
    return dl(impl_->ar.slots[0].fr(c.cur), c.F, impl_->stream, impl_->d2h_bytes);
}

std::vector<unsigned long long> Session::pass_trace(std::uint32_t& blocks) const {
    blocks = std::max<std::uint32_t>(1, impl_->gblocks);
    if (!impl_->cfg.ptrace) return {};
    ctl();
    return dl(impl_->cfg.ptrace, 64ull * blocks * 10 + 64 * 16, impl_->stream, impl_->d2h_bytes);
}

}  // namespace yas
