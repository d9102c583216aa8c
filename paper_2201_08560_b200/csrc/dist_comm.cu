// Rank-to-rank exchange (see dist_comm.cuh): NCCL and the single-device
// thread-rank stand-in used by the tests.
#include <dlfcn.h>
#include <nccl.h>

#include <condition_variable>
#include <cstring>
#include <memory>
#include <mutex>

#include "dist_comm.cuh"

namespace b2sr {

void Exchange::allgatherv(void *buf, const std::vector<size_t> &off, const std::vector<size_t> &len,
                          cudaStream_t s) {
    std::vector<Xfer> sends, recvs;
    for (int p = 0; p < world; p++) {
        if (p == rank) continue;
        if (len[rank]) sends.push_back({p, static_cast<char *>(buf) + off[rank], len[rank]});
        if (len[p]) recvs.push_back({p, static_cast<char *>(buf) + off[p], len[p]});
    }
    sendrecv(sends, recvs, s);
}

// ---------------------------------------------------------------- NCCL
namespace {

struct NcclApi {
    ncclResult_t (*GetUniqueId)(ncclUniqueId *) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*Send)(const void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*AllReduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char *(*GetErrorString)(ncclResult_t) = nullptr;
};

const NcclApi &nccl() {
    static NcclApi api;
    static std::once_flag once;
    static std::string err;
    std::call_once(once, [] {
        // the copy torch loaded (same process, same library instance) first
        void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        const char *env = getenv("B2SR_NCCL_LIB");
        if (!h && env) h = dlopen(env, RTLD_NOW);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW);
        if (!h) {
            err = dlerror() ? dlerror() : "libnccl.so.2 not found";
            return;
        }
#define SYM(f) api.f = reinterpret_cast<decltype(api.f)>(dlsym(h, "nccl" #f))
        SYM(GetUniqueId);
        SYM(CommInitRank);
        SYM(CommDestroy);
        SYM(Send);
        SYM(Recv);
        SYM(AllReduce);
        SYM(GroupStart);
        SYM(GroupEnd);
        SYM(GetErrorString);
#undef SYM
    });
    if (!api.GetUniqueId || !api.CommInitRank || !api.Send || !api.Recv || !api.AllReduce || !api.GroupStart ||
        !api.GroupEnd)
        B2SR_THROW(B2SR_ECUDA, "NCCL unavailable: %s", err.empty() ? "missing symbols" : err.c_str());
    return api;
}

#define NCK(call)                                                                                    \
    do {                                                                                             \
        ncclResult_t r_ = (call);                                                                    \
        if (r_ != ncclSuccess)                                                                       \
            B2SR_THROW(B2SR_ECUDA, "NCCL error %d (%s) at %s:%d", (int)r_,                           \
                       nccl().GetErrorString ? nccl().GetErrorString(r_) : "?", __FILE__, __LINE__); \
    } while (0)

struct NcclExchange final : Exchange {
    ncclComm_t comm = nullptr;
    ~NcclExchange() override {
        if (comm && nccl().CommDestroy) nccl().CommDestroy(comm);
    }
    void sendrecv(const std::vector<Xfer> &sends, const std::vector<Xfer> &recvs, cudaStream_t s) override {
        const NcclApi &n = nccl();
        NCK(n.GroupStart());
        for (const Xfer &x : sends) NCK(n.Send(x.ptr, x.bytes, ncclUint8, x.peer, comm, s));
        for (const Xfer &x : recvs) NCK(n.Recv(x.ptr, x.bytes, ncclUint8, x.peer, comm, s));
        NCK(n.GroupEnd());
    }
    void allreduce_sum_i64(int64_t *d, size_t count, cudaStream_t s) override {
        NCK(nccl().AllReduce(d, d, count, ncclInt64, ncclSum, comm, s));
    }
};

// ---------------------------------------------------------------- single-device thread ranks
struct LocalHub {
    int world;
    std::mutex mu;
    std::condition_variable cv;
    int arrived = 0;
    unsigned long long gen = 0;
    std::vector<std::vector<Xfer>> sends;
    std::vector<cudaEvent_t> ready, done;
    explicit LocalHub(int w) : world(w), sends(w), ready(w), done(w) {
        for (int r = 0; r < w; r++) {
            CK(cudaEventCreateWithFlags(&ready[r], cudaEventDisableTiming));
            CK(cudaEventCreateWithFlags(&done[r], cudaEventDisableTiming));
        }
    }
    ~LocalHub() {
        for (int r = 0; r < world; r++) {
            cudaEventDestroy(ready[r]);
            cudaEventDestroy(done[r]);
        }
    }
    void barrier() {
        std::unique_lock<std::mutex> lk(mu);
        const unsigned long long g = gen;
        if (++arrived == world) {
            arrived = 0;
            gen++;
            cv.notify_all();
        } else {
            cv.wait(lk, [&] { return gen != g; });
        }
    }
};

__global__ void k_sum_ranks_i64(int64_t *d, const int64_t *parts, size_t count, int world) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < count; i += (size_t)gridDim.x * blockDim.x) {
        int64_t v = 0;
        for (int r = 0; r < world; r++) v += parts[(size_t)r * count + i];
        d[i] = v;
    }
}

struct LocalExchange final : Exchange {
    std::shared_ptr<LocalHub> hub;
    void sendrecv(const std::vector<Xfer> &sends, const std::vector<Xfer> &recvs, cudaStream_t s) override {
        LocalHub &h = *hub;
        CK(cudaEventRecord(h.ready[rank], s));
        h.sends[rank] = sends;
        h.barrier();  // every rank's sources are published and recorded
        std::vector<int> seen(world, 0);
        for (const Xfer &x : recvs) {
            // the k-th recv from p matches p's k-th send to this rank (NCCL's ordering rule)
            const Xfer *src = nullptr;
            int k = seen[x.peer]++;
            for (const Xfer &y : h.sends[x.peer])
                if (y.peer == rank && k-- == 0) {
                    src = &y;
                    break;
                }
            if (!src || src->bytes != x.bytes)
                B2SR_THROW(B2SR_EINVAL, "unmatched exchange between ranks %d and %d", x.peer, rank);
            CK(cudaStreamWaitEvent(s, h.ready[x.peer], 0));
            CK(cudaMemcpyAsync(x.ptr, src->ptr, x.bytes, cudaMemcpyDeviceToDevice, s));
        }
        CK(cudaEventRecord(h.done[rank], s));
        h.barrier();  // every copy is enqueued
        // senders reuse their buffers only after the receivers' copies
        for (int p = 0; p < world; p++)
            if (p != rank) CK(cudaStreamWaitEvent(s, h.done[p], 0));
    }
    void allreduce_sum_i64(int64_t *d, size_t count, cudaStream_t s) override {
        Buf<int64_t> parts((size_t)world * count, s);
        CK(cudaMemcpyAsync(parts.p + (size_t)rank * count, d, count * 8, cudaMemcpyDeviceToDevice, s));
        std::vector<Xfer> snd, rcv;
        for (int p = 0; p < world; p++) {
            if (p == rank) continue;
            snd.push_back({p, parts.p + (size_t)rank * count, count * 8});
            rcv.push_back({p, parts.p + (size_t)p * count, count * 8});
        }
        sendrecv(snd, rcv, s);
        LAUNCH(k_sum_ranks_i64, (unsigned)std::min<size_t>((count + 255) / 256, 1024), 256, 0, s, d, parts.p, count,
               world);
        // parts is freed stream-ordered; peers finished reading it (sendrecv's last wait)
    }
};

}  // namespace

void nccl_unique_id(void *out128) {
    ncclUniqueId id;
    NCK(nccl().GetUniqueId(&id));
    static_assert(sizeof(ncclUniqueId) == 128, "NCCL unique id size");
    memcpy(out128, &id, sizeof(id));
}

Exchange *nccl_exchange(const void *unique_id, int world, int rank) {
    auto *e = new NcclExchange();
    e->rank = rank;
    e->world = world;
    CK(cudaGetDevice(&e->device));
    ncclUniqueId id;
    memcpy(&id, unique_id, sizeof(id));
    try {
        NCK(nccl().CommInitRank(&e->comm, world, id, rank));
    } catch (...) {
        delete e;
        throw;
    }
    return e;
}

std::vector<Exchange *> local_exchanges(int world) {
    auto hub = std::make_shared<LocalHub>(world);
    std::vector<Exchange *> out;
    int dev = 0;
    CK(cudaGetDevice(&dev));
    for (int r = 0; r < world; r++) {
        auto *e = new LocalExchange();
        e->rank = r;
        e->world = world;
        e->device = dev;
        e->hub = hub;
        out.push_back(e);
    }
    return out;
}

}  // namespace b2sr

using namespace b2sr;

extern "C" {

int b2sr_comm_unique_id(uint8_t *out128) {
    API_BEGIN
    nccl_unique_id(out128);
    API_END
}

int b2sr_comm_init(const uint8_t *id128, int world, int rank, b2sr_comm **out) {
    API_BEGIN
    if (world < 1 || rank < 0 || rank >= world) B2SR_THROW(B2SR_EINVAL, "bad rank %d of %d", rank, world);
    auto *c = new b2sr_comm();
    try {
        c->ex = nccl_exchange(id128, world, rank);
    } catch (...) {
        delete c;
        throw;
    }
    *out = c;
    API_END
}

int b2sr_comm_init_local(int world, b2sr_comm **outs) {
    API_BEGIN
    if (world < 1 || world > 64) B2SR_THROW(B2SR_EINVAL, "local world size must be 1..64");
    std::vector<Exchange *> ex = local_exchanges(world);
    for (int r = 0; r < world; r++) {
        outs[r] = new b2sr_comm();
        outs[r]->ex = ex[r];
    }
    API_END
}

int b2sr_comm_free(b2sr_comm *c) {
    API_BEGIN
    if (c) {
        delete c->ex;
        delete c;
    }
    API_END
}

int b2sr_comm_allreduce_sum_i64(b2sr_comm *c, int64_t *d, uint64_t count, void *stream) {
    API_BEGIN
    c->ex->allreduce_sum_i64(d, count, (cudaStream_t)stream);
    API_END
}

}  // extern "C"
