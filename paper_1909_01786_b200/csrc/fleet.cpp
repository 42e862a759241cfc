// Fleet transport: NCCL (dlopen'ed) collectives and the shared control block.
#include "fleet.hpp"

#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <stdexcept>
#include <string>

namespace yas {

namespace {

void ck(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw std::runtime_error(std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e));
}

// The NCCL entry points the fleet uses, resolved from libnccl.so.2 once.
struct NcclApi {
    ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
    ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
    const char* (*error_string)(ncclResult_t) = nullptr;

    static const NcclApi& get() {
        static const NcclApi api = load();
        if (!api.get_unique_id) throw std::runtime_error("CUDA error in fleet: libnccl.so.2 not loadable");
        return api;
    }

private:
    static NcclApi load() {
        NcclApi a;
        // an NCCL the process already holds (e.g. torch's) is reused: a second
        // copy under the same soname would shadow the newer one for later loads
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_LOCAL);
        if (!h) return a;
        auto sym = [&](auto& fn, const char* name) { fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name)); };
        sym(a.get_unique_id, "ncclGetUniqueId");
        sym(a.comm_init_rank, "ncclCommInitRank");
        sym(a.all_reduce, "ncclAllReduce");
        sym(a.broadcast, "ncclBroadcast");
        sym(a.comm_destroy, "ncclCommDestroy");
        sym(a.error_string, "ncclGetErrorString");
        if (!a.comm_init_rank || !a.all_reduce || !a.broadcast || !a.comm_destroy || !a.error_string) a.get_unique_id = nullptr;
        return a;
    }
};

void nck(ncclResult_t r, const char* what) {
    if (r != ncclSuccess)
        throw std::runtime_error(std::string("CUDA error in ") + what + " (NCCL): " + NcclApi::get().error_string(r));
}

class NcclComm final : public FleetComm {
public:
    NcclComm(const std::uint8_t id[128], int rank, int world, int device) : device_(device) {
        const NcclApi& api = NcclApi::get();
        ck(cudaSetDevice(device), "cudaSetDevice");
        ncclUniqueId uid;
        static_assert(sizeof(uid) == 128, "ncclUniqueId is 128 bytes");
        std::memcpy(&uid, id, sizeof uid);
        nck(api.comm_init_rank(&comm_, world, uid, rank), "ncclCommInitRank");
        ck(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking), "stream");
        ck(cudaMalloc(&buf_, kBuf), "cudaMalloc fleet buffer");
    }
    ~NcclComm() override {
        cudaSetDevice(device_);
        if (comm_) NcclApi::get().comm_destroy(comm_);
        if (buf_) cudaFree(buf_);
        if (stream_) cudaStreamDestroy(stream_);
    }
    void allreduce(std::uint64_t* vals, std::size_t n, Op op) override {
        if (8 * n > kBuf) throw std::invalid_argument("fleet all-reduce: too many values");
        ck(cudaSetDevice(device_), "cudaSetDevice");
        ck(cudaMemcpyAsync(buf_, vals, 8 * n, cudaMemcpyHostToDevice, stream_), "fleet upload");
        const ncclRedOp_t o = op == kSum ? ncclSum : op == kMax ? ncclMax : ncclMin;
        nck(NcclApi::get().all_reduce(buf_, buf_, n, ncclUint64, o, comm_, stream_), "ncclAllReduce");
        ck(cudaMemcpyAsync(vals, buf_, 8 * n, cudaMemcpyDeviceToHost, stream_), "fleet download");
        ck(cudaStreamSynchronize(stream_), "fleet all-reduce");
    }
    void broadcast(void* data, std::size_t bytes, int root) override {
        if (bytes > kBuf) throw std::invalid_argument("fleet broadcast: too many bytes");
        ck(cudaSetDevice(device_), "cudaSetDevice");
        ck(cudaMemcpyAsync(buf_, data, bytes, cudaMemcpyHostToDevice, stream_), "fleet upload");
        nck(NcclApi::get().broadcast(buf_, buf_, bytes, ncclUint8, root, comm_, stream_), "ncclBroadcast");
        ck(cudaMemcpyAsync(data, buf_, bytes, cudaMemcpyDeviceToHost, stream_), "fleet download");
        ck(cudaStreamSynchronize(stream_), "fleet broadcast");
    }

private:
    static constexpr std::size_t kBuf = 4096;
    int device_;
    ncclComm_t comm_ = nullptr;
    cudaStream_t stream_ = nullptr;
    void* buf_ = nullptr;
};

}  // namespace

void nccl_unique_id(std::uint8_t out[128]) {
    ncclUniqueId uid;
    nck(NcclApi::get().get_unique_id(&uid), "ncclGetUniqueId");
    std::memcpy(out, &uid, 128);
}

std::unique_ptr<FleetComm> nccl_comm(const std::uint8_t unique_id[128], int rank, int world, int device) {
    return std::make_unique<NcclComm>(unique_id, rank, world, device);
}

}  // namespace yas
