// upload.cu -- host->device copies of large pageable buffers (the caller's
// CSR arrays) through pinned staging.
//
// A pageable cudaMemcpyAsync goes through the driver's own staging at ~11-17
// GB/s on this host; a pinned copy reaches ~53 GB/s.  Here the pageable
// source is copied into two pinned slots by a small persistent pool of host
// threads (~30-45 GB/s aggregate) while the DMA of the other slot runs, so
// the transfer approaches the slower of the two instead of their sum.
#include <algorithm>
#include <condition_variable>
#include <cstring>
#include <mutex>
#include <thread>
#include <vector>

#include "ctx.cuh"

namespace imx {

namespace {

// Persistent memcpy workers: run(dst, src, n) splits n bytes over the workers
// and the calling thread and returns when all parts are copied.
class CopyPool {
public:
    static CopyPool &get() {
        static CopyPool pool;
        return pool;
    }
    void run(char *dst, const char *src, size_t n) {
        const int parts = (int)threads_.size() + 1;
        if (parts == 1 || n < (size_t)(256 << 10)) {
            memcpy(dst, src, n);
            return;
        }
        {
            std::lock_guard<std::mutex> lk(mu_);
            dst_ = dst;
            src_ = src;
            n_ = n;
            parts_ = parts;
            pending_ = parts - 1;
            ++gen_;
        }
        cv_.notify_all();
        copy_part(0);
        std::unique_lock<std::mutex> lk(mu_);
        done_.wait(lk, [&] { return pending_ == 0; });
    }
    ~CopyPool() {
        {
            std::lock_guard<std::mutex> lk(mu_);
            stop_ = true;
            ++gen_;
        }
        cv_.notify_all();
        for (auto &t : threads_) t.join();
    }

private:
    CopyPool() {
        unsigned hw = std::thread::hardware_concurrency();
        int nt = (int)std::min(8u, std::max(1u, hw / 2)) - 1;
        if (const char *e = getenv("IMX_UPLOAD_THREADS")) nt = std::max(0, atoi(e) - 1);
        for (int i = 0; i < nt; ++i) threads_.emplace_back([this, i] { worker(i + 1); });
    }
    void copy_part(int p) {
        const size_t per = (n_ + parts_ - 1) / parts_;
        const size_t a = std::min(n_, per * p), b = std::min(n_, a + per);
        if (b > a) memcpy(dst_ + a, src_ + a, b - a);
    }
    void worker(int p) {
        unsigned long long seen = 0;
        for (;;) {
            {
                std::unique_lock<std::mutex> lk(mu_);
                cv_.wait(lk, [&] { return gen_ != seen; });
                seen = gen_;
                if (stop_) return;
            }
            copy_part(p);
            {
                std::lock_guard<std::mutex> lk(mu_);
                if (--pending_ == 0) done_.notify_one();
            }
        }
    }
    std::vector<std::thread> threads_;
    std::mutex mu_;
    std::condition_variable cv_, done_;
    char *dst_ = nullptr;
    const char *src_ = nullptr;
    size_t n_ = 0;
    int parts_ = 1, pending_ = 0;
    unsigned long long gen_ = 0;
    bool stop_ = false;
};

std::mutex g_upload_mu;   // one staged upload at a time (the pool and slots are shared)

}  // namespace

// the source is page-locked host memory (cudaHostAlloc / registered): the
// DMA reads it directly at the link rate (55 GB/s measured), no staging
static bool host_pinned(const void *p);
bool host_pinned_ptr(const void *p) { return host_pinned(p); }

static bool host_pinned(const void *p) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost;
}

cudaError_t upload_h2d(void *dst, const void *src, size_t bytes, cudaStream_t st) {
    // below ~64 MB the driver's pageable path is as fast (thread hand-off and
    // the unpipelined first chunk dominate); measured on C2 / C3 / C4 CSRs
    size_t thresh = (size_t)64 << 20;
    if (const char *e = getenv("IMX_UPLOAD_STAGED_MIN")) thresh = (size_t)atoll(e);
    if (bytes < thresh || host_pinned(src)) return cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, st);
    std::lock_guard<std::mutex> lk(g_upload_mu);
    size_t chunk = std::min<size_t>(bytes, (size_t)8 << 20);
    if (const char *e = getenv("IMX_UPLOAD_CHUNK")) chunk = std::min<size_t>(bytes, std::max<size_t>(4096, (size_t)atoll(e)));
    void *slot[2] = {nullptr, nullptr};
    cudaEvent_t ev[2] = {nullptr, nullptr};
    cudaError_t e = cudaSuccess;
    for (int i = 0; i < 2 && e == cudaSuccess; ++i) {
        e = pinned_get(&slot[i], chunk);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming);
    }
    const char *s = static_cast<const char *>(src);
    char *d = static_cast<char *>(dst);
    for (size_t off = 0, k = 0; off < bytes && e == cudaSuccess; off += chunk, ++k) {
        const int b = (int)(k & 1);
        const size_t len = std::min(chunk, bytes - off);
        if (k >= 2) e = cudaEventSynchronize(ev[b]);     // the slot's previous DMA is done
        if (e != cudaSuccess) break;
        CopyPool::get().run(static_cast<char *>(slot[b]), s + off, len);
        e = cudaMemcpyAsync(d + off, slot[b], len, cudaMemcpyHostToDevice, st);
        if (e == cudaSuccess) e = cudaEventRecord(ev[b], st);
    }
    for (int i = 0; i < 2; ++i) {
        if (ev[i]) {
            cudaEventSynchronize(ev[i]);               // slots go back to the cache idle
            cudaEventDestroy(ev[i]);
        }
        pinned_put(slot[i], chunk);
    }
    return e;
}

}  // namespace imx
