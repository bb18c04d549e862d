// Host <-> device copies of PAGEABLE host memory for the drop-in entry points.
//
// A C program relinked from the reference's emitted OpenMP passes malloc'd arrays.  The driver
// copies pageable memory through its own pinned bounce buffer with one host thread: 11.2 GB/s on
// the B200 box, against 54-55 GB/s for pinned memory over the same PCIe link — so the drop-in call
// on pageable arrays ran at a fifth of the link.  Page-locking the caller's buffer around the DMA
// (cudaHostRegister) costs more than it saves (5.7-7.4 GB/s overall: registering 2 GiB takes
// 200-300 ms).  Here the bytes go through a ring of pinned chunks that a pool of host threads fills
// (memcpy, one slice per thread) while the DMA engine drains the previous chunk, and the reverse
// for device -> host: 45 GB/s with 8-16 threads (tools/probes/h2d_pageable.cu; memcpy alone
// reaches 52 GB/s, so the host's memory bandwidth, not the link, is the limit).  The GPU cannot read
// pageable memory itself on this platform (cudaDevAttrPageableMemoryAccess = 0: no HMM / ATS,
// tools/probes/hmm_probe.cu), so some host copy is unavoidable.
//
// Semantics: h2d returns when the caller's source may be reused (every chunk copied into the ring);
// the DMAs are ordered on the caller's stream.  d2h is synchronous (returns with the data in the
// caller's buffer) and ordered after the work already on the stream.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cstring>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

namespace {

// A fixed pool of host threads running one parallel job at a time (the caller takes part).
class CopyPool {
  public:
    explicit CopyPool(int n) : n_(std::max(1, n)) {
        for (int t = 1; t < n_; t++) th_.emplace_back([this, t] { loop(t); });
    }
    ~CopyPool() {
        {
            std::lock_guard<std::mutex> lk(mu_);
            stop_ = true;
            gen_++;
        }
        cv_.notify_all();
        for (auto& t : th_) t.join();
    }
    int size() const { return n_; }
    // job(t) for t = 0 .. n_ - 1, t = 0 on the caller
    void run(const std::function<void(int)>& job) {
        std::lock_guard<std::mutex> one(run_mu_);  // one job at a time (stagers of several devices share the pool)
        {
            std::lock_guard<std::mutex> lk(mu_);
            job_ = &job;
            left_ = n_ - 1;
            gen_++;
        }
        cv_.notify_all();
        job(0);
        std::unique_lock<std::mutex> lk(mu_);
        done_.wait(lk, [this] { return left_ == 0; });
        job_ = nullptr;
    }

  private:
    void loop(int t) {
        unsigned long long seen = 0;
        for (;;) {
            const std::function<void(int)>* job;
            {
                std::unique_lock<std::mutex> lk(mu_);
                cv_.wait(lk, [&] { return gen_ != seen; });
                seen = gen_;
                if (stop_) return;
                job = job_;
            }
            if (job) (*job)(t);
            {
                std::lock_guard<std::mutex> lk(mu_);
                if (--left_ == 0) done_.notify_one();
            }
        }
    }
    int n_;
    std::vector<std::thread> th_;
    std::mutex mu_, run_mu_;
    std::condition_variable cv_, done_;
    const std::function<void(int)>* job_ = nullptr;
    unsigned long long gen_ = 0;
    int left_ = 0;
    bool stop_ = false;
};

// memcpy of rows x width bytes (pitches dpitch / spitch) across the pool's threads
void par_copy(CopyPool& pool, char* dst, size_t dpitch, const char* src, size_t spitch, size_t width, size_t rows) {
    const int T = pool.size();
    if (rows == 1 || (dpitch == width && spitch == width)) {  // contiguous: split the bytes
        const size_t n = width * rows;
        pool.run([&](int t) {
            const size_t lo = n * t / T / 64 * 64, hi = t == T - 1 ? n : n * (t + 1) / T / 64 * 64;
            if (hi > lo) memcpy(dst + lo, src + lo, hi - lo);
        });
        return;
    }
    pool.run([&](int t) {  // split the rows
        for (size_t r = rows * t / T; r < rows * (t + 1) / T; r++) memcpy(dst + r * dpitch, src + r * spitch, width);
    });
}

// (Non-temporal stores for these copies — no read-for-ownership of the destination — measured the
// same: spmv_vec / axpy / conv5x5_u8 pageable 47.6-47.9 / 49.3 / 48.6-49.4 GB/s either way,
// tools/pageable_probe.py.)
// pinned ring: 4 chunks of 32 MB per device.  (Pieces of 1/16 of a transfer, 4-32 MB, measured
// worse: the pipelined SpMV's 70 MB chunks then go as 4 MB pieces and the per-piece dispatch and
// event waits cost more than the earlier overlap gains — SpMV pageable e2e 45 -> 37 GB/s.)
constexpr size_t CHUNK = 32u << 20;
constexpr int RING = 4;

struct Stager {
    std::mutex mu;
    char* ring = nullptr;
    cudaEvent_t ev[RING] = {};
    bool busy[RING] = {};  // an event recorded on the slot and not yet waited for
    int next = 0;
};

CopyPool& pool() {
    static CopyPool p(std::min(16, std::max(1, (int)std::thread::hardware_concurrency())));
    return p;
}

Stager* stager(int device) {
    static std::mutex mu;
    static std::vector<Stager*> all;
    std::lock_guard<std::mutex> lk(mu);
    if ((int)all.size() <= device) all.resize(device + 1, nullptr);
    if (!all[device]) {
        Stager* s = new Stager();
        if (cudaHostAlloc((void**)&s->ring, CHUNK * RING, cudaHostAllocPortable) != cudaSuccess) {
            cudaGetLastError();
            delete s;
            return nullptr;
        }
        for (int i = 0; i < RING; i++) cudaEventCreateWithFlags(&s->ev[i], cudaEventDisableTiming);
        all[device] = s;
    }
    return all[device];
}

// the next ring slot, its previous DMA finished
int take_slot(Stager* s) {
    const int k = s->next;
    s->next = (k + 1) % RING;
    if (s->busy[k]) {
        cudaEventSynchronize(s->ev[k]);
        s->busy[k] = false;
    }
    return k;
}

}  // namespace

// true for host memory the driver would have to stage itself (neither device, managed nor pinned)
bool host_is_pageable(const void* p) {
    if (!p) return false;
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return true;
    }
    return a.type == cudaMemoryTypeUnregistered;
}

// pageable src -> device dst, `rows` rows of `width` bytes at pitches spitch / dpitch (rows = 1:
// one contiguous run).  Returns a cudaError_t.
int staged_h2d_2d(int device, void* dst, size_t dpitch, const void* src, size_t spitch, size_t width, size_t rows,
                  cudaStream_t st) {
    Stager* s = stager(device);
    if (!s || (rows > 1 && width > CHUNK)) {  // no ring (or a row wider than a chunk): the driver's path
        return (int)(rows == 1 ? cudaMemcpyAsync(dst, src, width, cudaMemcpyHostToDevice, st)
                               : cudaMemcpy2DAsync(dst, dpitch, src, spitch, width, rows, cudaMemcpyHostToDevice, st));
    }
    std::lock_guard<std::mutex> lk(s->mu);
    if (rows == 1) {  // contiguous: chunk by bytes
        for (size_t off = 0; off < width; off += CHUNK) {
            const size_t n = std::min(CHUNK, width - off);
            const int k = take_slot(s);
            char* buf = s->ring + (size_t)k * CHUNK;
            par_copy(pool(), buf, n, (const char*)src + off, n, n, 1);
            cudaError_t e = cudaMemcpyAsync((char*)dst + off, buf, n, cudaMemcpyHostToDevice, st);
            if (e != cudaSuccess) return (int)e;
            cudaEventRecord(s->ev[k], st);
            s->busy[k] = true;
        }
        return (int)cudaSuccess;
    }
    const size_t per = std::max<size_t>(1, CHUNK / width);  // rows per chunk (packed at pitch width)
    for (size_t r0 = 0; r0 < rows; r0 += per) {
        const size_t nr = std::min(per, rows - r0);
        const int k = take_slot(s);
        char* buf = s->ring + (size_t)k * CHUNK;
        par_copy(pool(), buf, width, (const char*)src + r0 * spitch, spitch, width, nr);
        cudaError_t e = cudaMemcpy2DAsync((char*)dst + r0 * dpitch, dpitch, buf, width, width, nr,
                                          cudaMemcpyHostToDevice, st);
        if (e != cudaSuccess) return (int)e;
        cudaEventRecord(s->ev[k], st);
        s->busy[k] = true;
    }
    return (int)cudaSuccess;
}

// device src -> pageable dst (synchronous), rows x width bytes at pitches spitch / dpitch
int staged_d2h_2d(int device, void* dst, size_t dpitch, const void* src, size_t spitch, size_t width, size_t rows,
                  cudaStream_t st) {
    Stager* s = stager(device);
    if (!s || (rows > 1 && width > CHUNK)) {
        cudaError_t e = rows == 1 ? cudaMemcpyAsync(dst, src, width, cudaMemcpyDeviceToHost, st)
                                  : cudaMemcpy2DAsync(dst, dpitch, src, spitch, width, rows, cudaMemcpyDeviceToHost, st);
        if (e == cudaSuccess) e = cudaStreamSynchronize(st);
        return (int)e;
    }
    std::lock_guard<std::mutex> lk(s->mu);
    // the transfer as pieces of at most one chunk: (first row, rows) or, contiguous, (offset, bytes)
    struct Piece {
        size_t a, n;
    };
    std::vector<Piece> pieces;
    if (rows == 1)
        for (size_t off = 0; off < width; off += CHUNK) pieces.push_back({off, std::min(CHUNK, width - off)});
    else
        for (size_t r0 = 0, per = std::max<size_t>(1, CHUNK / width); r0 < rows; r0 += per)
            pieces.push_back({r0, std::min(per, rows - r0)});
    std::vector<int> slot(pieces.size());
    auto issue = [&](size_t i) -> cudaError_t {
        slot[i] = take_slot(s);
        char* buf = s->ring + (size_t)slot[i] * CHUNK;
        cudaError_t e = rows == 1 ? cudaMemcpyAsync(buf, (const char*)src + pieces[i].a, pieces[i].n,
                                                    cudaMemcpyDeviceToHost, st)
                                  : cudaMemcpy2DAsync(buf, width, (const char*)src + pieces[i].a * spitch, spitch,
                                                      width, pieces[i].n, cudaMemcpyDeviceToHost, st);
        if (e != cudaSuccess) return e;
        cudaEventRecord(s->ev[slot[i]], st);
        s->busy[slot[i]] = true;
        return cudaSuccess;
    };
    // keep RING - 1 DMAs ahead of the host copies
    size_t issued = 0;
    for (; issued < pieces.size() && issued < (size_t)RING - 1; issued++)
        if (cudaError_t e = issue(issued)) return (int)e;
    for (size_t i = 0; i < pieces.size(); i++) {
        cudaEventSynchronize(s->ev[slot[i]]);
        s->busy[slot[i]] = false;
        const char* buf = s->ring + (size_t)slot[i] * CHUNK;
        if (rows == 1) par_copy(pool(), (char*)dst + pieces[i].a, pieces[i].n, buf, pieces[i].n, pieces[i].n, 1);
        else par_copy(pool(), (char*)dst + pieces[i].a * dpitch, dpitch, buf, width, width, pieces[i].n);
        if (issued < pieces.size()) {
            if (cudaError_t e = issue(issued)) return (int)e;
            issued++;
        }
    }
    return (int)cudaSuccess;
}
