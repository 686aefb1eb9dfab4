// comm.cu -- the multi-rank data plane: int64 sums of per-rank partials on
// the device (gains after memo, CELF partial gains per
// evaluation batch, the commit self-check).
//
// The reference is one process whose lanes are split over a thread pool
// (propagation.py:209-216, 244-251); here a rank is one GPU holding a lane
// window, and the partial sums meet through NCCL over NVLink/NVSwitch,
// enqueued on the context's stream in place -- no host copy of the data.
//
// Backends of an imx_comm:
//   NCCL   one rank per GPU (ncclCommInitRank; the unique id travels through
//          the caller's launcher, e.g. torch.distributed).  libnccl is opened
//          with dlopen at first use, so the library loads on hosts without it
//          and shares the process's NCCL (torch's) when one is loaded.
//   LOCAL  ranks as host threads of one process (test double for one GPU:
//          NCCL refuses two ranks on the same device): a barrier and a host
//          sum of the staged buffers.
#include <dlfcn.h>
#include <nccl.h>

#include <condition_variable>
#include <cstring>
#include <mutex>
#include <vector>

#include "ctx.cuh"

namespace imx {

namespace {

struct NcclApi {
    bool tried = false, ok = false;
    ncclResult_t (*GetUniqueId)(ncclUniqueId *) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*AllReduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    const char *(*GetErrorString)(ncclResult_t) = nullptr;
};
std::mutex g_nccl_mu;
NcclApi g_nccl;

int load_nccl() {
    std::lock_guard<std::mutex> lk(g_nccl_mu);
    if (g_nccl.tried) {
        if (!g_nccl.ok) { set_error("libnccl.so.2 not available"); return IMX_ENODEV; }
        return IMX_OK;
    }
    g_nccl.tried = true;
    void *h = nullptr;
    if (const char *p = getenv("IMX_NCCL_LIB")) h = dlopen(p, RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) { set_error("libnccl.so.2 not available: %s", dlerror()); return IMX_ENODEV; }
    g_nccl.GetUniqueId = (decltype(g_nccl.GetUniqueId))dlsym(h, "ncclGetUniqueId");
    g_nccl.CommInitRank = (decltype(g_nccl.CommInitRank))dlsym(h, "ncclCommInitRank");
    g_nccl.AllReduce = (decltype(g_nccl.AllReduce))dlsym(h, "ncclAllReduce");
    g_nccl.CommDestroy = (decltype(g_nccl.CommDestroy))dlsym(h, "ncclCommDestroy");
    g_nccl.GetErrorString = (decltype(g_nccl.GetErrorString))dlsym(h, "ncclGetErrorString");
    g_nccl.ok = g_nccl.GetUniqueId && g_nccl.CommInitRank && g_nccl.AllReduce && g_nccl.CommDestroy;
    if (!g_nccl.ok) { set_error("libnccl.so.2 lacks the needed symbols"); return IMX_ENODEV; }
    return IMX_OK;
}

int nccl_fail(ncclResult_t r, const char *what) {
    set_error("NCCL error in %s: %s", what, g_nccl.GetErrorString ? g_nccl.GetErrorString(r) : "?");
    return IMX_ENCCL;
}

}  // namespace

// ranks as threads of one process: a reusable barrier + staged host sums
struct LocalGroup {
    int nranks;
    std::mutex mu;
    std::condition_variable cv;
    int arrived = 0;
    unsigned long long gen = 0;
    std::vector<std::vector<int64_t>> bufs;
    std::vector<int64_t> sum;
    explicit LocalGroup(int n) : nranks(n), bufs(n) {}
    void barrier() {
        std::unique_lock<std::mutex> lk(mu);
        const unsigned long long g = gen;
        if (++arrived == nranks) {
            arrived = 0;
            ++gen;
            cv.notify_all();
        } else {
            cv.wait(lk, [&] { return gen != g; });
        }
    }
};

}  // namespace imx

struct imx_comm {
    int kind = 0;           // 1 NCCL, 2 LOCAL
    int dev = 0, rank = 0, nranks = 1;
    ncclComm_t nccl = nullptr;
    imx::LocalGroup *grp = nullptr;
};

namespace imx {

// buf[0, n) on the device (stream st) <- its sum over the ranks
int comm_allreduce_i64(imx_comm *cm, int64_t *dbuf, int64_t n, cudaStream_t st) {
    if (!cm || n <= 0) return IMX_OK;
    if (cm->kind == 1) {
        const ncclResult_t r = g_nccl.AllReduce(dbuf, dbuf, (size_t)n, ncclInt64, ncclSum, cm->nccl, st);
        if (r != ncclSuccess) return nccl_fail(r, "ncclAllReduce");
        return IMX_OK;
    }
    LocalGroup &G = *cm->grp;
    auto &mine = G.bufs[cm->rank];
    mine.resize((size_t)n);
    IMX_CUDA(cudaMemcpyAsync(mine.data(), dbuf, sizeof(int64_t) * n, cudaMemcpyDeviceToHost, st));
    IMX_CUDA(cudaStreamSynchronize(st));
    G.barrier();
    if (cm->rank == 0) {
        G.sum.assign((size_t)n, 0);
        for (auto &b : G.bufs)
            for (int64_t i = 0; i < n; ++i) G.sum[i] += b[i];
    }
    G.barrier();
    IMX_CUDA(cudaMemcpyAsync(dbuf, G.sum.data(), sizeof(int64_t) * n, cudaMemcpyHostToDevice, st));
    IMX_CUDA(cudaStreamSynchronize(st));
    G.barrier();            // G.sum is reused by the next call
    return IMX_OK;
}

}  // namespace imx

using namespace imx;

extern "C" int imx_comm_unique_id(uint8_t *id_out) {
    if (!id_out) { set_error("id_out is NULL"); return IMX_EINVAL; }
    IMX_TRY(load_nccl());
    ncclUniqueId id;
    const ncclResult_t r = g_nccl.GetUniqueId(&id);
    if (r != ncclSuccess) return nccl_fail(r, "ncclGetUniqueId");
    static_assert(sizeof(id) == IMX_COMM_ID_BYTES, "ncclUniqueId size");
    memcpy(id_out, &id, sizeof id);
    return IMX_OK;
}

extern "C" int imx_comm_create(int32_t device, int32_t nranks, int32_t rank, const uint8_t *id,
                               imx_comm **out) {
    if (!out || !id) { set_error("NULL argument"); return IMX_EINVAL; }
    *out = nullptr;
    if (nranks < 1 || rank < 0 || rank >= nranks) { set_error("rank %d of %d invalid", rank, nranks); return IMX_EINVAL; }
    IMX_TRY(load_nccl());
    IMX_TRY(select_device(device));
    ncclUniqueId uid;
    memcpy(&uid, id, sizeof uid);
    imx_comm *c = new imx_comm();
    c->kind = 1;
    c->dev = device;
    c->rank = rank;
    c->nranks = nranks;
    const ncclResult_t r = g_nccl.CommInitRank(&c->nccl, nranks, uid, rank);
    if (r != ncclSuccess) { delete c; return nccl_fail(r, "ncclCommInitRank"); }
    *out = c;
    return IMX_OK;
}

extern "C" int imx_local_group_create(int32_t nranks, void **out) {
    if (!out || nranks < 1) { set_error("bad argument"); return IMX_EINVAL; }
    *out = new LocalGroup(nranks);
    return IMX_OK;
}

extern "C" void imx_local_group_destroy(void *grp) { delete static_cast<LocalGroup *>(grp); }

extern "C" int imx_comm_create_local(void *grp, int32_t rank, int32_t device, imx_comm **out) {
    if (!out || !grp) { set_error("NULL argument"); return IMX_EINVAL; }
    LocalGroup *G = static_cast<LocalGroup *>(grp);
    if (rank < 0 || rank >= G->nranks) { set_error("rank %d of %d invalid", rank, G->nranks); return IMX_EINVAL; }
    imx_comm *c = new imx_comm();
    c->kind = 2;
    c->dev = device;
    c->rank = rank;
    c->nranks = G->nranks;
    c->grp = G;
    *out = c;
    return IMX_OK;
}

extern "C" void imx_comm_destroy(imx_comm *c) {
    if (!c) return;
    if (c->kind == 1 && c->nccl && g_nccl.CommDestroy) g_nccl.CommDestroy(c->nccl);
    delete c;
}

extern "C" int imx_comm_allreduce(imx_comm *c, int64_t *buf, int64_t n) {
    if (!c || (!buf && n > 0)) { set_error("NULL argument"); return IMX_EINVAL; }
    if (n <= 0) return IMX_OK;
    IMX_CUDA(cudaSetDevice(c->dev));
    cudaStream_t st;
    IMX_CUDA(acquire_stream(c->dev, &st));
    int64_t *d = nullptr;
    int rc = IMX_OK;
    if (cudaMallocAsync((void **)&d, sizeof(int64_t) * n, st) != cudaSuccess ||
        cudaMemcpyAsync(d, buf, sizeof(int64_t) * n, cudaMemcpyHostToDevice, st) != cudaSuccess) {
        rc = cuda_fail(cudaGetLastError(), "allreduce staging", __FILE__, __LINE__);
    }
    if (rc == IMX_OK) rc = comm_allreduce_i64(c, d, n, st);
    if (rc == IMX_OK && (cudaMemcpyAsync(buf, d, sizeof(int64_t) * n, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
                         cudaStreamSynchronize(st) != cudaSuccess))
        rc = cuda_fail(cudaGetLastError(), "allreduce staging", __FILE__, __LINE__);
    if (d) cudaFreeAsync(d, st);
    cudaStreamSynchronize(st);
    release_stream(c->dev, st);
    return rc;
}

extern "C" int imx_ctx_attach_comm(imx_ctx *c, imx_comm *comm) {
    CTX_CHECK(c);
    if (comm && comm->dev != c->dev) { set_error("communicator device %d != context device %d", comm->dev, c->dev); return IMX_EINVAL; }
    c->comm = comm;
    return IMX_OK;
}
