// comm.cu -- communication backends of the z-slab decomposition:
//   * NcclComm: NCCL over NVLink/NVSwitch (ncclSend/ncclRecv to r-1/r+1 for halos,
//     ncclAllGather for deterministic reductions and setup exchanges).  libnccl is
//     dlopen'ed so the process uses the NCCL torch already loaded (no version mix).
//   * LocalComm: P handles of ONE process driven by P host threads (test backend):
//     the same collective schedule, with device-to-device copies between the
//     ranks' buffers ordered by events.  It exercises every sharded code path except
//     the NCCL transport itself, on one GPU, without kernels waiting on each other.
#include <dlfcn.h>
#include <nccl.h>

#include <condition_variable>
#include <cstring>
#include <memory>
#include <mutex>

#include "tsp_internal.cuh"

namespace tsp {

// ------------------------------------------------------------------ NCCL (dlopen)
struct NcclApi {
    void *h = nullptr;
    ncclResult_t (*GetUniqueId)(ncclUniqueId *) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*Send)(const void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*AllGather)(const void *, void *, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char *(*GetErrorString)(ncclResult_t) = nullptr;
};
static NcclApi &nccl()
{
    static NcclApi a;
    if (!a.h) {
        const char *names[] = {"libnccl.so.2", "libnccl.so"};
        for (const char *nm : names) {
            a.h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL);
            if (a.h) break;
        }
        TSP_REQUIRE(a.h, TSP_ERR_NCCL, "cannot dlopen libnccl.so.2");
#define SYM(f) a.f = (decltype(a.f))dlsym(a.h, "nccl" #f)
        SYM(GetUniqueId); SYM(CommInitRank); SYM(CommDestroy); SYM(Send); SYM(Recv); SYM(AllGather);
        SYM(GroupStart); SYM(GroupEnd); SYM(GetErrorString);
#undef SYM
        TSP_REQUIRE(a.GetUniqueId && a.CommInitRank && a.Send && a.Recv && a.AllGather && a.GroupStart && a.GroupEnd,
                    TSP_ERR_NCCL, "libnccl is missing symbols");
    }
    return a;
}
#define TSP_NCCL(x)                                                                                             \
    do {                                                                                                        \
        ncclResult_t r_ = (x);                                                                                  \
        if (r_ != ncclSuccess) throw ::tsp::Error{TSP_ERR_NCCL, std::string(#x) + ": " + nccl().GetErrorString(r_)}; \
    } while (0)

struct NcclComm : Comm {
    ncclComm_t comm = nullptr;
    NcclComm(int rank, int nranks, const void *uid)
    {
        this->rank = rank; this->nranks = nranks;
        ncclUniqueId id;
        memcpy(&id, uid, sizeof(id));
        TSP_NCCL(nccl().CommInitRank(&comm, nranks, id, rank));
    }
    ~NcclComm() override { if (comm && nccl().CommDestroy) nccl().CommDestroy(comm); }
    void neighbor_exchange(const void *send_lo, size_t bytes_send_lo, void *recv_lo, size_t bytes_recv_lo,
                           const void *send_hi, size_t bytes_send_hi, void *recv_hi, size_t bytes_recv_hi,
                           cudaStream_t s) override
    {
        auto &n = nccl();
        TSP_NCCL(n.GroupStart());
        if (rank > 0) {
            if (bytes_send_lo) TSP_NCCL(n.Send(send_lo, bytes_send_lo, ncclChar, rank - 1, comm, s));
            if (bytes_recv_lo) TSP_NCCL(n.Recv(recv_lo, bytes_recv_lo, ncclChar, rank - 1, comm, s));
        }
        if (rank < nranks - 1) {
            if (bytes_send_hi) TSP_NCCL(n.Send(send_hi, bytes_send_hi, ncclChar, rank + 1, comm, s));
            if (bytes_recv_hi) TSP_NCCL(n.Recv(recv_hi, bytes_recv_hi, ncclChar, rank + 1, comm, s));
        }
        TSP_NCCL(n.GroupEnd());
    }
    void allgather(const void *send, void *recv, size_t bytes, cudaStream_t s) override
    {
        TSP_NCCL(nccl().AllGather(send, recv, bytes, ncclChar, comm, s));
    }
    bool capturable() const override { return true; }      // NCCL >= 2.9 collectives and grouped send/recv capture
};

// ------------------------------------------------------------------ in-process test world
struct LocalWorld {
    int n;
    std::mutex m;
    std::condition_variable cv;
    int arrived = 0;
    long gen = 0;
    std::vector<const void *> ptr_a, ptr_b;     // per rank published pointers
    std::vector<size_t> sz_a, sz_b;
    std::vector<cudaEvent_t> ev;               // per rank "data ready" events
    std::vector<cudaEvent_t> done;             // per rank "my copies finished" events
    explicit LocalWorld(int n_) : n(n_), ptr_a(n_), ptr_b(n_), sz_a(n_), sz_b(n_), ev(n_), done(n_)
    {
        for (int r = 0; r < n; ++r) {
            cudaEventCreateWithFlags(&ev[r], cudaEventDisableTiming);
            cudaEventCreateWithFlags(&done[r], cudaEventDisableTiming);
        }
    }
    ~LocalWorld()
    {
        for (int r = 0; r < n; ++r) { cudaEventDestroy(ev[r]); cudaEventDestroy(done[r]); }
    }
    void barrier()
    {
        std::unique_lock<std::mutex> lk(m);
        long g = gen;
        if (++arrived == n) { arrived = 0; ++gen; cv.notify_all(); }
        else cv.wait(lk, [&] { return gen != g; });
    }
};

struct LocalComm : Comm {
    LocalWorld *w;
    LocalComm(LocalWorld *w_, int r) : w(w_) { rank = r; nranks = w_->n; }
    // publish (a, b), wait for everyone, run `body` (which enqueues copies from peers), then
    // make every rank's stream wait for all peers' copies before the buffers may be reused
    template <class F>
    void round(const void *a, size_t sa, const void *b, size_t sb, cudaStream_t s, F body)
    {
        w->ptr_a[rank] = a; w->sz_a[rank] = sa; w->ptr_b[rank] = b; w->sz_b[rank] = sb;
        TSP_CUDA(cudaEventRecord(w->ev[rank], s));
        w->barrier();
        body();
        TSP_CUDA(cudaEventRecord(w->done[rank], s));
        w->barrier();
        for (int r = 0; r < nranks; ++r)
            if (r != rank) TSP_CUDA(cudaStreamWaitEvent(s, w->done[r], 0));
        w->barrier();
    }
    void neighbor_exchange(const void *send_lo, size_t bytes_send_lo, void *recv_lo, size_t bytes_recv_lo,
                           const void *send_hi, size_t bytes_send_hi, void *recv_hi, size_t bytes_recv_hi,
                           cudaStream_t s) override
    {
        round(send_lo, bytes_send_lo, send_hi, bytes_send_hi, s, [&] {
            if (rank > 0 && bytes_recv_lo) {            // from rank-1's "hi" send
                TSP_REQUIRE(w->sz_b[rank - 1] == bytes_recv_lo, TSP_ERR_NCCL, "local halo size mismatch (lo)");
                TSP_CUDA(cudaStreamWaitEvent(s, w->ev[rank - 1], 0));
                TSP_CUDA(cudaMemcpyAsync(recv_lo, w->ptr_b[rank - 1], bytes_recv_lo, cudaMemcpyDeviceToDevice, s));
            }
            if (rank < nranks - 1 && bytes_recv_hi) {   // from rank+1's "lo" send
                TSP_REQUIRE(w->sz_a[rank + 1] == bytes_recv_hi, TSP_ERR_NCCL, "local halo size mismatch (hi)");
                TSP_CUDA(cudaStreamWaitEvent(s, w->ev[rank + 1], 0));
                TSP_CUDA(cudaMemcpyAsync(recv_hi, w->ptr_a[rank + 1], bytes_recv_hi, cudaMemcpyDeviceToDevice, s));
            }
        });
    }
    void allgather(const void *send, void *recv, size_t bytes, cudaStream_t s) override
    {
        round(send, bytes, nullptr, 0, s, [&] {
            for (int r = 0; r < nranks; ++r) {
                TSP_REQUIRE(w->sz_a[r] == bytes, TSP_ERR_NCCL, "local allgather size mismatch");
                if (r != rank) TSP_CUDA(cudaStreamWaitEvent(s, w->ev[r], 0));
                TSP_CUDA(cudaMemcpyAsync((char *)recv + r * bytes, w->ptr_a[r], bytes, cudaMemcpyDeviceToDevice, s));
            }
        });
    }
};

Comm *make_comm(int kind, void *arg, int rank, int nranks)
{
    if (nranks <= 1) return nullptr;
    if (kind == TSP_COMM_NCCL) return new NcclComm(rank, nranks, arg);
    if (kind == TSP_COMM_LOCAL) {
        LocalWorld *w = (LocalWorld *)arg;
        TSP_REQUIRE(w && w->n == nranks, TSP_ERR_INVALID_ARG, "local world size != nranks");
        return new LocalComm(w, rank);
    }
    throw Error{TSP_ERR_INVALID_ARG, "unknown communicator kind"};
}

// ------------------------------------------------------------------ host-level helpers on top of Comm
// allgather of a small host array (count T per rank): goes through device memory
template <class T>
std::vector<T> host_allgather(Ctx &c, const std::vector<T> &mine)
{
    if (!c.comm) return mine;
    const size_t b = mine.size() * sizeof(T);
    DBuf<uint8_t> s, r;
    s.alloc(std::max<size_t>(b, 1)); r.alloc(std::max<size_t>(b, 1) * c.nranks);
    if (b) TSP_CUDA(cudaMemcpyAsync(s, mine.data(), b, cudaMemcpyHostToDevice, c.s));
    c.comm->allgather(s, r, std::max<size_t>(b, 1), c.s);
    std::vector<T> out(mine.size() * c.nranks);
    for (int k = 0; k < c.nranks; ++k)
        if (b) TSP_CUDA(cudaMemcpyAsync((char *)out.data() + k * b, (char *)r.p + k * std::max<size_t>(b, 1), b, cudaMemcpyDeviceToHost, c.s));
    TSP_CUDA(cudaStreamSynchronize(c.s));
    return out;
}
template std::vector<int64_t> host_allgather<int64_t>(Ctx &, const std::vector<int64_t> &);
template std::vector<double> host_allgather<double>(Ctx &, const std::vector<double> &);

}  // namespace tsp

using namespace tsp;

extern "C" {

tsp_status tsp_nccl_unique_id(char out[128])
{
    try {
        ncclUniqueId id;
        static_assert(sizeof(ncclUniqueId) <= 128, "ncclUniqueId too large");
        TSP_NCCL(nccl().GetUniqueId(&id));
        memset(out, 0, 128);
        memcpy(out, &id, sizeof(id));
        return TSP_OK;
    } catch (const tsp::Error &e) {
        set_error(e.msg);
        return e.st;
    }
}

void *tsp_local_world_create(int nranks) { return nranks > 0 ? new LocalWorld(nranks) : nullptr; }
void tsp_local_world_destroy(void *w) { delete (LocalWorld *)w; }

}  // extern "C"
