// Rank-to-rank exchange for the row-partitioned multi-GPU drivers.
//
// One communicator per rank (one GPU per process, or one host thread per GPU
// in a single process).  Every call is enqueued on the caller's stream, so a
// driver's level loop -- kernels and exchanges -- runs without host syncs.
//   * NcclExchange: NCCL over NVLink / NVSwitch (grouped ncclSend/ncclRecv,
//     ncclAllReduce); libnccl is opened at run time (the copy torch already
//     loaded when present), so the library itself has no link dependency.
//   * LocalExchange: N ranks as host threads on ONE device, transfers as
//     stream-ordered device copies behind host barriers -- the same level
//     loop with N ranks on a single GPU (tests; this build has one GPU).
#pragma once

#include <vector>

#include "b2sr_internal.cuh"

namespace b2sr {

struct Xfer {
    int peer;
    void *ptr;      // device buffer (send: source, recv: destination)
    size_t bytes;
};

struct Exchange {
    int rank = 0, world = 1, device = 0;
    virtual ~Exchange() = default;
    // One grouped round of point-to-point transfers on stream s.  Every send
    // to peer p must be matched by p's recv from this rank of the same size.
    virtual void sendrecv(const std::vector<Xfer> &sends, const std::vector<Xfer> &recvs, cudaStream_t s) = 0;
    // In-place element-wise int64 sum over ranks.
    virtual void allreduce_sum_i64(int64_t *d, size_t count, cudaStream_t s) = 0;
    // Variable-size all-gather in place: rank r's bytes [off[r], off[r]+len[r])
    // of buf are copied into every other rank's buf at the same offsets.
    void allgatherv(void *buf, const std::vector<size_t> &off, const std::vector<size_t> &len, cudaStream_t s);
};

Exchange *nccl_exchange(const void *unique_id, int world, int rank);
void nccl_unique_id(void *out128);
std::vector<Exchange *> local_exchanges(int world);

}  // namespace b2sr

struct b2sr_comm {
    b2sr::Exchange *ex = nullptr;
};
