// A fleet = the GPUs (and processes) that share one cube enumeration or one
// first-model portfolio. The reference has no multi-GPU path
// (its enumeration is Driver::run's block-and-continue loop,
// /root/reference/proj/src/solver.cpp:216-246,291-293); here the cubes of one
// enumeration are dealt to every GPU from ONE queue in the home GPU's memory,
// reached over NVLink by peer mappings (CUDA IPC across processes), and the
// only collective is the final all-reduce of model counts, error and
// termination flags (NCCL, or a caller-supplied transport).
#pragma once

#include <cstddef>
#include <cstdint>
#include <memory>

#include <cuda_runtime.h>

#include "device/engine.cuh"

namespace yas {

// Small host-side collectives over the fleet's ranks (in place, every rank).
class FleetComm {
public:
    virtual ~FleetComm() = default;
    enum Op { kSum = 0, kMax = 1, kMin = 2 };
    virtual void allreduce(std::uint64_t* vals, std::size_t n, Op op) = 0;
    virtual void broadcast(void* buf, std::size_t bytes, int root) = 0;
};

// NCCL loaded at run time (libnccl.so.2): no link-time dependency, and a
// process that already holds torch's NCCL shares that copy.
std::unique_ptr<FleetComm> nccl_comm(const std::uint8_t unique_id[128], int rank, int world, int device);
void nccl_unique_id(std::uint8_t out[128]);

}  // namespace yas

struct yas_fleet {
    int rank = 0, world = 1, device = 0;
    std::unique_ptr<yas::FleetComm> comm;
    yas::dev::Fleet* ctl = nullptr;  // shared queue / claim, mapped on `device`
    bool owner = false;              // rank 0: allocated ctl
    bool ipc = false;                // ctl opened through CUDA IPC (rank > 0)
    bool dynamic = false;            // every rank reaches rank 0's ctl: one shared cube queue
};
