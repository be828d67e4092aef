// Row-cluster sharding of the hot path over G = 2^g ranks and the
// exchange step between ranks.
//
// Rank r owns tree node r at level g: a contiguous internal-order row range [rb[r], re[r]).  Every
// rank-local vector lives in a PADDED layout of G segments of maxc entries, so one in-place
// allgather (count maxc per rank) assembles the full vector: internal row i of rank q sits at
// q*maxc + (i - rb[q]).
//
// Exchangers:
//  - NcclExchanger: ncclAllGather over the library's own communicator (NVLink / NVSwitch on one
//    node).  libnccl.so.2 is opened at run time (the copy torch already loaded, if any), so the
//    library has no link-time NCCL dependency and world == 1 never touches NCCL.
//  - LocalGroupExchanger: G ranks inside ONE process (one host thread per rank, any devices): the
//    same allgather done with device-to-device copies ordered by CUDA events and host barriers.  It
//    runs the sharded programs on a single GPU for testing ("virtual shards").
#include <dlfcn.h>
#include <nccl.h>

#include <condition_variable>
#include <algorithm>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>

#include "hm_internal.h"

namespace hm {

// ------------------------------------------------------------------ shard geometry
void local_range(const Geom& g, int rank, int world, int64_t* begin, int64_t* end) {
    int node = 0;
    for (int bit = world >> 1; bit > 0; bit >>= 1) {
        const Node& N = g.nodes[node];
        if (N.is_leaf()) {  // too few clusters: later ranks get empty ranges
            if (rank & (bit * 2 - 1)) {
                *begin = *end = N.end;
                return;
            }
            break;
        }
        node = N.child[(rank & bit) ? 1 : 0];
    }
    *begin = g.nodes[node].begin;
    *end = g.nodes[node].end;
}

void make_shard(Geom& g, int rank, int world) {
    Shard& S = g.shard;
    S.rank = rank;
    S.world = world;
    S.rb.assign(world, 0);
    S.re.assign(world, 0);
    S.maxc = 0;
    for (int q = 0; q < world; ++q) {
        local_range(g, q, world, &S.rb[q], &S.re[q]);
        S.maxc = std::max(S.maxc, S.re[q] - S.rb[q]);
    }
    S.maxc = std::max<int64_t>(S.maxc, 1);
    S.maxc = (S.maxc + 1) & ~int64_t(1);   // even: 16-byte aligned segments
}

int Shard::rank_of(int64_t i) const {
    for (int q = world - 1; q >= 0; --q)
        if (i >= rb[q] && i < re[q]) return q;
    return 0;
}

// ------------------------------------------------------------------ NCCL (dlopen)
namespace {

struct NcclApi {
    void* h = nullptr;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t*) = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi& nccl() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);   // torch's copy, if loaded
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) return;
        api.h = h;
        api.GetUniqueId = (decltype(api.GetUniqueId))dlsym(h, "ncclGetUniqueId");
        api.CommInitRank = (decltype(api.CommInitRank))dlsym(h, "ncclCommInitRank");
        api.AllGather = (decltype(api.AllGather))dlsym(h, "ncclAllGather");
        api.CommDestroy = (decltype(api.CommDestroy))dlsym(h, "ncclCommDestroy");
        api.Broadcast = (decltype(api.Broadcast))dlsym(h, "ncclBroadcast");
        api.CommGetAsyncError = (decltype(api.CommGetAsyncError))dlsym(h, "ncclCommGetAsyncError");
        api.GetErrorString = (decltype(api.GetErrorString))dlsym(h, "ncclGetErrorString");
    });
    if (!api.h || !api.GetUniqueId || !api.CommInitRank || !api.AllGather || !api.CommDestroy || !api.Broadcast)
        throw Error(HM_ERR_NCCL, "libnccl.so.2 not found or incomplete (needed for world > 1)");
    return api;
}

void nccl_check(ncclResult_t r, const char* what) {
    if (r == ncclSuccess) return;
    const char* m = nccl().GetErrorString ? nccl().GetErrorString(r) : "?";
    throw Error(HM_ERR_NCCL, std::string(what) + ": " + m);
}

struct NcclExchanger : Exchanger {
    ncclComm_t comm = nullptr;
    int rank, world;
    NcclExchanger(const void* id, int rank_, int world_) : rank(rank_), world(world_) {
        ncclUniqueId uid;
        std::memcpy(&uid, id, sizeof(uid));
        nccl_check(nccl().CommInitRank(&comm, world, uid, rank), "ncclCommInitRank");
    }
    ~NcclExchanger() override {
        if (comm) nccl().CommDestroy(comm);
    }
    void allgather(double* buf, int64_t count, cudaStream_t s) override {
        nccl_check(nccl().AllGather(buf + (int64_t)rank * count, buf, (size_t)count, ncclFloat64, comm, s),
                   "ncclAllGather");
    }
    void broadcast(void* buf, size_t bytes, int root, cudaStream_t s) override {
        nccl_check(nccl().Broadcast(buf, buf, bytes, ncclChar, root, comm, s), "ncclBroadcast");
    }
    const char* kind() const override { return "nccl"; }
};

// ------------------------------------------------------------------ in-process group
struct LocalGroup {
    int world;
    std::mutex mu;
    std::condition_variable cv;
    int arrived = 0;
    int64_t generation = 0;
    std::vector<double*> bufs;
    std::vector<void*> vbufs;
    std::vector<cudaEvent_t> ready[2], done[2];
    std::vector<int> devices;
    explicit LocalGroup(int w) : world(w), bufs(w, nullptr), vbufs(w, nullptr), devices(w, 0) {
        for (int p = 0; p < 2; ++p) {
            ready[p].assign(w, nullptr);
            done[p].assign(w, nullptr);
        }
    }
    void barrier() {
        std::unique_lock<std::mutex> lk(mu);
        const int64_t gen = generation;
        if (++arrived == world) {
            arrived = 0;
            ++generation;
            cv.notify_all();
        } else {
            cv.wait(lk, [&] { return generation != gen; });
        }
    }
};

std::mutex g_groups_mu;
std::map<int64_t, std::weak_ptr<LocalGroup>> g_groups;

std::shared_ptr<LocalGroup> join_group(int64_t key, int world) {
    std::lock_guard<std::mutex> lk(g_groups_mu);
    auto it = g_groups.find(key);
    if (it != g_groups.end()) {
        if (auto sp = it->second.lock()) {
            if (sp->world != world) throw Error(HM_ERR_INVALID_ARG, "local group joined with a different world size");
            return sp;
        }
    }
    auto sp = std::make_shared<LocalGroup>(world);
    g_groups[key] = sp;
    return sp;
}

struct LocalGroupExchanger : Exchanger {
    std::shared_ptr<LocalGroup> G;
    int rank, world, device;
    int64_t n_ex = 0;   // exchanges done (event double-buffer parity)
    LocalGroupExchanger(int64_t key, int rank_, int world_, int device_)
        : G(join_group(key, world_)), rank(rank_), world(world_), device(device_) {
        for (int p = 0; p < 2; ++p) {
            HM_CUDA(cudaEventCreateWithFlags(&G->ready[p][rank], cudaEventDisableTiming));
            HM_CUDA(cudaEventCreateWithFlags(&G->done[p][rank], cudaEventDisableTiming));
        }
        G->devices[rank] = device;
    }
    ~LocalGroupExchanger() override {
        for (int p = 0; p < 2; ++p) {
            if (G->ready[p][rank]) cudaEventDestroy(G->ready[p][rank]);
            if (G->done[p][rank]) cudaEventDestroy(G->done[p][rank]);
        }
    }
    // Same contract as ncclAllGather in place: on return (stream-ordered) buf[q*count ...] holds rank
    // q's segment for every q.  Host barriers make every rank's "segment ready" event visible before
    // any copy is enqueued, and every rank's "copies done" event visible before anyone may overwrite
    // its own segment again (events alternate between two sets, so a rank at most one exchange ahead
    // never re-records an event a peer still has to wait on).
    void allgather(double* buf, int64_t count, cudaStream_t s) override {
        const int par = (int)(n_ex++ & 1);
        G->bufs[rank] = buf;
        HM_CUDA(cudaEventRecord(G->ready[par][rank], s));
        G->barrier();
        for (int q = 0; q < world; ++q) {
            if (q == rank) continue;
            HM_CUDA(cudaStreamWaitEvent(s, G->ready[par][q], 0));
            HM_CUDA(cudaMemcpyPeerAsync(buf + (int64_t)q * count, device, G->bufs[q] + (int64_t)q * count,
                                        G->devices[q], (size_t)count * sizeof(double), s));
        }
        HM_CUDA(cudaEventRecord(G->done[par][rank], s));
        G->barrier();
        for (int q = 0; q < world; ++q)
            if (q != rank) HM_CUDA(cudaStreamWaitEvent(s, G->done[par][q], 0));
    }
    void broadcast(void* buf, size_t bytes, int root, cudaStream_t s) override {
        const int par = (int)(n_ex++ & 1);
        G->vbufs[rank] = buf;
        HM_CUDA(cudaEventRecord(G->ready[par][rank], s));
        G->barrier();
        if (rank != root && bytes > 0) {
            HM_CUDA(cudaStreamWaitEvent(s, G->ready[par][root], 0));
            HM_CUDA(cudaMemcpyPeerAsync(buf, device, G->vbufs[root], G->devices[root], bytes, s));
        }
        HM_CUDA(cudaEventRecord(G->done[par][rank], s));
        G->barrier();
        if (rank == root)
            for (int q = 0; q < world; ++q)
                if (q != rank) HM_CUDA(cudaStreamWaitEvent(s, G->done[par][q], 0));
    }
    const char* kind() const override { return "local-group"; }
};

}  // namespace

std::unique_ptr<Exchanger> make_exchanger(int device, int rank, int world, const void* comm_id, uint32_t flags) {
    if (world <= 1) return nullptr;
    if (!comm_id) throw Error(HM_ERR_INVALID_ARG, "world > 1 needs a communicator id");
    if (flags & HM_FLAG_LOCAL_GROUP) {
        int64_t key;
        std::memcpy(&key, comm_id, sizeof(key));
        return std::make_unique<LocalGroupExchanger>(key, rank, world, device);
    }
    return std::make_unique<NcclExchanger>(comm_id, rank, world);
}

}  // namespace hm

using namespace hm;

extern "C" {

hm_status hm_nccl_unique_id(void* id_out) {
    if (!id_out) return HM_ERR_INVALID_ARG;
    try {
        ncclUniqueId uid;
        nccl_check(nccl().GetUniqueId(&uid), "ncclGetUniqueId");
        std::memcpy(id_out, &uid, sizeof(uid));
        return HM_OK;
    } catch (const Error& e) {
        return e.code;
    }
}

// One-rank communicator on `device`, then the exact in-place allgather call the sharded hot path
// issues (NcclExchanger::allgather) and the factor broadcast's ncclBroadcast on a device buffer of
// `count` doubles, checked element by
// element.  A one-GPU box cannot run world > 1 over NCCL (duplicate device), so this is how the
// dlopen'd symbols, the unique-id handoff and the call form are exercised on real hardware.
hm_status hm_nccl_selftest(int device, int64_t count) {
    if (count < 1) return HM_ERR_INVALID_ARG;
    double* d = nullptr;
    try {
        if (cudaSetDevice(device) != cudaSuccess) return HM_ERR_CUDA;
        char id[128];
        const hm_status st = hm_nccl_unique_id(id);
        if (st != HM_OK) return st;
        NcclExchanger ex(id, 0, 1);
        std::vector<double> h((size_t)count), back((size_t)count);
        for (int64_t i = 0; i < count; ++i) h[(size_t)i] = 0.5 + (double)i;
        if (cudaMalloc(&d, sizeof(double) * (size_t)count) != cudaSuccess) return HM_ERR_OOM;
        cudaStream_t s;
        if (cudaStreamCreate(&s) != cudaSuccess) { cudaFree(d); return HM_ERR_CUDA; }
        cudaMemcpyAsync(d, h.data(), sizeof(double) * (size_t)count, cudaMemcpyHostToDevice, s);
        ex.allgather(d, count, s);
        ex.broadcast(d, sizeof(double) * (size_t)count, 0, s);   // the factor broadcast's call form
        cudaMemcpyAsync(back.data(), d, sizeof(double) * (size_t)count, cudaMemcpyDeviceToHost, s);
        const cudaError_t ce = cudaStreamSynchronize(s);
        cudaStreamDestroy(s);
        cudaFree(d);
        d = nullptr;
        if (ce != cudaSuccess) return HM_ERR_CUDA;
        ncclResult_t ar = ncclSuccess;
        nccl_check(nccl().CommGetAsyncError(ex.comm, &ar), "ncclCommGetAsyncError");
        nccl_check(ar, "ncclAllGather (async)");
        for (int64_t i = 0; i < count; ++i)
            if (back[(size_t)i] != h[(size_t)i]) return HM_ERR_NCCL;
        return HM_OK;
    } catch (const Error& e) {
        if (d) cudaFree(d);
        return e.code;
    }
}

hm_status hm_shard_plan(const hm_geom* geom, int world, int64_t* begin, int64_t* end, int64_t* maxc,
                        int64_t* block_owner) {
    if (!geom || world < 1 || (world & (world - 1)) || !begin || !end || !maxc) return HM_ERR_INVALID_ARG;
    const Geom& g = geom->g;
    *maxc = 0;
    for (int q = 0; q < world; ++q) {
        local_range(g, q, world, &begin[q], &end[q]);
        *maxc = std::max(*maxc, end[q] - begin[q]);
    }
    *maxc = (std::max<int64_t>(*maxc, 1) + 1) & ~int64_t(1);
    if (block_owner) {
        // owner of each block row: the rank whose range contains the block's rows (-1: straddles)
        for (size_t b = 0; b < g.blocks.size(); ++b) {
            const Blk& B = g.blocks[b];
            int64_t own = -1;
            for (int q = 0; q < world; ++q)
                if (B.r0 >= begin[q] && B.r1 <= end[q] && end[q] > begin[q]) own = q;
            block_owner[b] = own;
        }
    }
    return HM_OK;
}

}  // extern "C"
