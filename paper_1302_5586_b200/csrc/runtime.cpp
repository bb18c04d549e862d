// Host runtime of the B200 PENCIL backend: status channel, per-device context (streams,
// fault word, scratch, caching pool), the drop-in C ABI of include/pencil_b200.h §1, the
// stream-ordered device API (§3), the CSR inspector, the Interpreter-mirror name dispatch
// (§4), the verdict->schedule mapper (§5) and the multi-GPU partitioners (§6).
//
// Reference correspondences:
//   drop-in signatures       <- emit_openmp / Printer::param  (pretty.cpp:221-233, 472-531)
//   pencil_runtime_call      <- Interpreter::call / exec_call (interp.cpp:95-122)
//   named device arrays      <- Interpreter::set_array/arrays (interp.hpp:40-43), array_storage (interp.cpp:124-138)
//   fault word / status      <- PencilError("E-INTERP") (diag.hpp:44-55; interp.cpp:186-195, 273-279)
//   pencil_map_nest          <- the verdict switch of emit_openmp (pretty.cpp:479-501)
#include <cuda_runtime.h>

#include <cstdarg>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <functional>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/pencil_b200.h"
#include "kernels.h"

// hoststage.cpp: pageable host memory through the multi-threaded pinned staging ring
bool host_is_pageable(const void* p);  // hoststage.cpp
int staged_h2d_2d(int device, void* dst, size_t dpitch, const void* src, size_t spitch, size_t width, size_t rows,
                  cudaStream_t st);
int staged_d2h_2d(int device, void* dst, size_t dpitch, const void* src, size_t spitch, size_t width, size_t rows,
                  cudaStream_t st);

namespace {

// ------------------------------------------------------------------ status channel
thread_local int g_status = PENCIL_OK;
thread_local char g_msg[512] = "";
// bytes the last drop-in call on this thread moved over the link (pencil_last_transfer_bytes)
thread_local long long g_h2d = 0, g_d2h = 0;

const char* code_name(int s) {
    switch (s) {
        case PENCIL_OK: return "OK";
        case PENCIL_E_INTERP: return "E-INTERP";
        case PENCIL_E_ARG: return "E-ARG";
        case PENCIL_E_CUDA: return "E-CUDA";
        case PENCIL_E_NOMEM: return "E-NOMEM";
        case PENCIL_E_UNSUPPORTED: return "E-UNSUPPORTED";
        case PENCIL_E_OP2_SHAPE: return "E-OP2-SHAPE";
        case PENCIL_E_OP2_RANGE: return "E-OP2-RANGE";
        case PENCIL_E_OP2_KERNEL: return "E-OP2-KERNEL";
        case PENCIL_E_OP2_CONFLICT: return "E-OP2-CONFLICT";
        case PENCIL_E_OPTIML_SHAPE: return "E-OPTIML-SHAPE";
        case PENCIL_E_OPTIML_RANGE: return "E-OPTIML-RANGE";
    }
    return "E-?";
}

int fail(int status, const char* fmt, ...) {
    g_status = status;
    int off = snprintf(g_msg, sizeof g_msg, "%s: ", code_name(status));
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_msg + off, sizeof g_msg - off, fmt, ap);
    va_end(ap);
    return status;
}
int ok() {
    g_status = PENCIL_OK;
    g_msg[0] = 0;
    return PENCIL_OK;
}
int cuda_fail(cudaError_t e, const char* what) {
    if (e == cudaErrorMemoryAllocation) return fail(PENCIL_E_NOMEM, "%s: %s", what, cudaGetErrorString(e));
    return fail(PENCIL_E_CUDA, "%s: %s", what, cudaGetErrorString(e));
}
#define CK(call)                                                  \
    do {                                                          \
        cudaError_t e_ = (call);                                  \
        if (e_ != cudaSuccess) return cuda_fail(e_, #call);       \
    } while (0)

// ------------------------------------------------------------------ device context
// Device words a launch mutates are kept per (device, stream), so launches on different streams
// never share them (re-entrant per (device set, stream)): the fault word the kernels
// raise E-INTERP bits in, the SpMV tile-ticket word, and the gemv_t last-CTA counters.  Launches
// on one stream are ordered, so the self-resetting words stay consistent between them.
struct StreamState {
    unsigned* words = nullptr;         // device: [0] fault word, [1] SpMV tile ticket
    unsigned* host = nullptr;          // pinned mirror of the fault word
    unsigned* gemv_t_counters = nullptr;
    size_t gemv_t_counter_cap = 0;
    std::mutex mu;                     // growth of the counters + the launch that uses them
};

struct DeviceCtx {
    int device = -1;
    cudaStream_t stream = nullptr;
    cudaMemPool_t pool = nullptr;
    float* dot_result = nullptr;
    double* dot_partial = nullptr;
    unsigned* dot_counter = nullptr;
    float* l2_flush = nullptr;
    long long l2_flush_elems = 0;
    std::mutex mu;                     // serializes drop-in calls on this device
    std::mutex smu;                    // guards `streams`
    std::map<cudaStream_t, StreamState*> streams;
};

std::mutex g_ctx_mu;
std::map<int, DeviceCtx*> g_ctx;

int get_ctx(DeviceCtx** out) {
    int dev = 0;
    CK(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(g_ctx_mu);
    auto it = g_ctx.find(dev);
    if (it != g_ctx.end()) {
        *out = it->second;
        return ok();
    }
    DeviceCtx* c = new DeviceCtx();
    c->device = dev;
    CK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    cudaMemPoolProps props = {};
    props.allocType = cudaMemAllocationTypePinned;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = dev;
    CK(cudaMemPoolCreate(&c->pool, &props));
    unsigned long long thresh = ~0ull;  // keep freed blocks cached: the pool is the allocator cache
    CK(cudaMemPoolSetAttribute(c->pool, cudaMemPoolAttrReleaseThreshold, &thresh));
    CK(cudaMalloc(&c->dot_result, 64));
    CK(cudaMalloc(&c->dot_partial, sizeof(double) * dot_partial_elems()));
    CK(cudaMalloc(&c->dot_counter, 64));
    CK(cudaMemset(c->dot_counter, 0, 64));
    g_ctx[dev] = c;
    *out = c;
    return ok();
}

// the per-stream words of (c's device, st), created zeroed on first use
int stream_state(DeviceCtx* c, cudaStream_t st, StreamState** out) {
    std::lock_guard<std::mutex> lk(c->smu);
    StreamState*& ss = c->streams[st];
    if (!ss) {
        StreamState* n = new StreamState();
        if (cudaMalloc(&n->words, 64) != cudaSuccess || cudaMemset(n->words, 0, 64) != cudaSuccess ||
            cudaMallocHost(&n->host, 64) != cudaSuccess) {
            cudaFree(n->words);
            delete n;
            c->streams.erase(st);
            return cuda_fail(cudaGetLastError(), "per-stream state");
        }
        ss = n;
    }
    *out = ss;
    return PENCIL_OK;
}
unsigned* fault_word(DeviceCtx* c, cudaStream_t st) {
    StreamState* ss = nullptr;
    return stream_state(c, st, &ss) ? nullptr : ss->words;
}
unsigned* ticket_word(DeviceCtx* c, cudaStream_t st) {
    StreamState* ss = nullptr;
    return stream_state(c, st, &ss) ? nullptr : ss->words + 1;
}

// the stream's view of the device API (0 = the legacy default stream, the CUDA convention, so
// launches order with the caller's other work); only the drop-in path uses the library's own stream
cudaStream_t pick_stream(DeviceCtx*, pencil_stream_t s) { return (cudaStream_t)s; }

int pool_alloc(DeviceCtx* c, cudaStream_t st, size_t bytes, void** p) {
    if (bytes == 0) bytes = 16;
    cudaError_t e = cudaMallocFromPoolAsync(p, bytes, c->pool, st);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMallocFromPoolAsync");
    return PENCIL_OK;
}
void pool_free(cudaStream_t st, void* p) {
    if (p) cudaFreeAsync(p, st);
}

// gemv_t's last-CTA counters for stream st (caller holds ss->mu); grown stream-ordered: the new
// block is zeroed on st and the old one freed on st after every launch that used it
int ensure_gemv_t_counters(DeviceCtx* c, cudaStream_t st, StreamState* ss, size_t n) {
    if (ss->gemv_t_counter_cap >= n) return PENCIL_OK;
    size_t cap = n < 1024 ? 1024 : n;
    unsigned* p = nullptr;
    int r = pool_alloc(c, st, cap * sizeof(unsigned), (void**)&p);
    if (r) return r;
    CK(cudaMemsetAsync(p, 0, cap * sizeof(unsigned), st));
    pool_free(st, ss->gemv_t_counters);
    ss->gemv_t_counters = p;
    ss->gemv_t_counter_cap = cap;
    return PENCIL_OK;
}

// gemv_t over views: A (rank 2, unit stride along j), x, y (rank 1) -> the strided kernel
int gemv_t_views_launch(DeviceCtx* c, cudaStream_t st, float alpha, float beta, const pencil_view& A,
                        const pencil_view& x, const pencil_view& y) {
    if (A.rank != 2 || x.rank != 1 || y.rank != 1 || A.extent[0] != x.extent[0] || A.extent[1] != y.extent[0] ||
        A.extent[0] < 0 || A.extent[1] < 0)
        return fail(PENCIL_E_ARG, "gemv_t views: A must be m x n, x of m, y of n");
    if (A.stride[1] != 1 || A.stride[0] < 0 || A.stride[0] > 0x7fffffff || x.stride[0] < 1 ||
        x.stride[0] > 0x7fffffff || y.stride[0] < 1 || y.stride[0] > 0x7fffffff || A.extent[0] > 0x7fffffff ||
        A.extent[1] > 0x7fffffff)
        return fail(PENCIL_E_UNSUPPORTED, "gemv_t views: needs unit stride along j and positive 32-bit strides");
    const int m = (int)A.extent[0], n = (int)A.extent[1];
    if (n == 0) return PENCIL_OK;
    StreamState* ss = nullptr;
    int r = stream_state(c, st, &ss);
    if (r) return r;
    std::lock_guard<std::mutex> lk(ss->mu);
    if ((r = ensure_gemv_t_counters(c, st, ss, gemv_t_counter_elems(n)))) return r;
    float* part = nullptr;
    size_t pe = gemv_t_partial_elems(m, n);
    if (pe && (r = pool_alloc(c, st, pe * sizeof(float), (void**)&part))) return r;
    const int e = launch_gemv_t(st, m, n, (int)A.stride[0], (int)x.stride[0], (int)y.stride[0], alpha, beta,
                                (const float*)A.base + A.offset, (const float*)x.base + x.offset,
                                (float*)y.base + y.offset, part, ss->gemv_t_counters);
    pool_free(st, part);
    return e ? cuda_fail((cudaError_t)e, "gemv_t launch") : PENCIL_OK;
}

// read and clear the fault word of stream st (synchronizes st)
int collect_faults(DeviceCtx* c, cudaStream_t st) {
    StreamState* ss = nullptr;
    int r = stream_state(c, st, &ss);
    if (r) return r;
    CK(cudaMemcpyAsync(ss->host, ss->words, sizeof(unsigned), cudaMemcpyDeviceToHost, st));
    CK(cudaMemsetAsync(ss->words, 0, sizeof(unsigned), st));
    CK(cudaStreamSynchronize(st));
    unsigned f = *ss->host;
    if (f & 1u) return fail(PENCIL_E_INTERP, "load index out of bounds (device fault word 0x%x)", f);
    if (f & 2u) return fail(PENCIL_E_INTERP, "CSR rowptr entry outside [0, nnz] (device fault word 0x%x)", f);
    if (f & 4u) return fail(PENCIL_E_INTERP, "division by zero");
    return PENCIL_OK;
}

// ------------------------------------------------------------------ host/device staging
enum Dir { IN = 1, OUT = 2, INOUT = 3 };

struct Stage {
    void* user = nullptr;      // caller pointer
    void* dev = nullptr;       // device pointer used by the kernel
    size_t bytes = 0;
    int dir = IN;
    bool owned = false;        // dev allocated from the pool (user is host memory)
    // strided copy-back (conv5x5_f32 interior): 0 = whole buffer
    size_t pitch = 0, width = 0, height = 0, offset = 0;
};

bool is_device_ptr(const void* p) {
    if (!p) return false;
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

// pageable host buffers of at least this size go through the multi-threaded pinned staging ring
// (hoststage.cpp: 45 GB/s against the driver's 11 GB/s); smaller ones through the driver
constexpr size_t STAGE_MIN = 4u << 20;
bool staged(const void* p, size_t bytes) { return bytes >= STAGE_MIN && host_is_pageable(p); }

int stage_in(DeviceCtx* c, cudaStream_t st, Stage& s) {
    if (s.bytes == 0 || is_device_ptr(s.user)) {
        s.dev = s.user;
        s.owned = false;
        return PENCIL_OK;
    }
    if (!s.user) return fail(PENCIL_E_ARG, "null array pointer");
    int r = pool_alloc(c, st, s.bytes, &s.dev);
    if (r) return r;
    s.owned = true;
    if (s.dir & IN) {
        if (staged(s.user, s.bytes)) CK((cudaError_t)staged_h2d_2d(c->device, s.dev, s.bytes, s.user, s.bytes, s.bytes, 1, st));
        else CK(cudaMemcpyAsync(s.dev, s.user, s.bytes, cudaMemcpyHostToDevice, st));
        g_h2d += (long long)s.bytes;
    }
    return PENCIL_OK;
}

int stage_out(DeviceCtx* c, cudaStream_t st, Stage& s) {
    if (!s.owned || !(s.dir & OUT)) return PENCIL_OK;
    if (s.height) {
        g_d2h += (long long)(s.width * s.height);
        if (staged(s.user, s.bytes))
            CK((cudaError_t)staged_d2h_2d(c->device, (char*)s.user + s.offset, s.pitch, (char*)s.dev + s.offset,
                                          s.pitch, s.width, s.height, st));
        else
            CK(cudaMemcpy2DAsync((char*)s.user + s.offset, s.pitch, (char*)s.dev + s.offset, s.pitch, s.width,
                                 s.height, cudaMemcpyDeviceToHost, st));
    } else {
        if (staged(s.user, s.bytes))
            CK((cudaError_t)staged_d2h_2d(c->device, s.user, s.bytes, s.dev, s.bytes, s.bytes, 1, st));
        else
            CK(cudaMemcpyAsync(s.user, s.dev, s.bytes, cudaMemcpyDeviceToHost, st));
        g_d2h += (long long)s.bytes;
    }
    return PENCIL_OK;
}

// Runs `launch(dev pointers...)` around host<->device staging; synchronous, status-setting.
template <int N, typename F>
int dropin(Stage (&st)[N], F launch) {
    DeviceCtx* c = nullptr;
    int r = get_ctx(&c);
    if (r) return r;
    std::lock_guard<std::mutex> lk(c->mu);
    cudaStream_t s = c->stream;
    g_h2d = g_d2h = 0;
    for (int i = 0; i < N && !r; i++) r = stage_in(c, s, st[i]);
    if (!r) {
        cudaError_t e = (cudaError_t)launch(c, s);
        if (e != cudaSuccess) r = cuda_fail(e, "kernel launch");
    }
    for (int i = 0; i < N && !r; i++) r = stage_out(c, s, st[i]);
    for (int i = 0; i < N; i++)
        if (st[i].owned) pool_free(s, st[i].dev);
    if (r) {
        cudaStreamSynchronize(s);
        return r;
    }
    return collect_faults(c, s) == PENCIL_OK ? ok() : g_status;
}

size_t nz(long long v) { return v > 0 ? (size_t)v : 0; }

// ------------------------------------------------------------------ CSR plans
struct CsrPlanImpl {
    int device, nrows, ncols, nnz, mode, ntiles, tile_nnz;
    int* tile_row = nullptr;
    unsigned* flags = nullptr;
    unsigned* rs_bits = nullptr;  // row-start bitmap
    int* ord = nullptr;           // plans with empty rows: non-empty ordinal of each row, and its inverse
    int* rowmap = nullptr;
    const int* rowptr = nullptr;  // the device rowptr the plan was built from (the ordinals' input)
    int seg = 0;                  // the segmented executor applies (monotone rowptr)
    SegPlan seg_plan() const {
        SegPlan s;
        if (seg) {
            s.rs_bits = rs_bits;
            s.ord = ord;
            s.rowmap = rowmap;
        }
        return s;
    }
};

// after the plan kernel: which executor the plan takes (reads its two flag words: a sync on st)
// rows may be empty: the ordinals the segmented executor names its rows by (launch_csr_ordinals)
int csr_plan_ordinals(DeviceCtx* c, cudaStream_t st, CsrPlanImpl* p) {
    int* bsum = nullptr;
    int r;
    if ((r = pool_alloc(c, st, sizeof(int) * ((size_t)p->nrows + 1), (void**)&p->ord)) ||
        (r = pool_alloc(c, st, sizeof(int) * ((size_t)p->nrows + 1), (void**)&p->rowmap)) ||
        (r = pool_alloc(c, st, sizeof(int) * csr_ord_scratch_ints(), (void**)&bsum)))
        return r;
    const int e = launch_csr_ordinals(st, p->nrows, p->rowptr, p->ord, p->rowmap, bsum);
    pool_free(st, bsum);
    return e ? cuda_fail((cudaError_t)e, "csr ordinals") : PENCIL_OK;
}

// the empty rows' y before a segmented launch over a plan with empty rows
cudaError_t zero_empty_rows(const CsrPlanImpl& p, float* y, cudaStream_t st) {
    return p.seg && p.ord ? cudaMemsetAsync(y, 0, sizeof(float) * (size_t)p.nrows, st) : cudaSuccess;
}

int csr_plan_finalize(DeviceCtx* c, cudaStream_t st, CsrPlanImpl* p) {
    unsigned f[4] = {0, 0, 0, 0};
    CK(cudaMemcpyAsync(f, p->flags, sizeof f, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    p->seg = p->rs_bits && f[0] == 0;
    if (p->seg && f[2] != 0) return csr_plan_ordinals(c, st, p);
    return PENCIL_OK;
}
void csr_plan_release(cudaStream_t st, CsrPlanImpl& p) {
    pool_free(st, p.tile_row);
    pool_free(st, p.flags);
    pool_free(st, p.rs_bits);
    pool_free(st, p.ord);
    pool_free(st, p.rowmap);
}

int csr_plan_build(DeviceCtx* c, cudaStream_t st, int nrows, int nnz, const int* rowptr, int mode,
                   CsrPlanImpl* p, unsigned* fw = nullptr) {
    p->device = c->device;
    p->rowptr = rowptr;
    p->nrows = nrows;
    p->nnz = nnz;
    p->mode = mode;
    const TileSchedule ts = csr_tile_schedule(mode, nnz);
    p->tile_nnz = ts.tile_nnz;
    p->ntiles = ts.ntiles;
    int r = pool_alloc(c, st, sizeof(int) * ((size_t)p->ntiles + 1), (void**)&p->tile_row);
    if (r) return r;
    r = pool_alloc(c, st, 64, (void**)&p->flags);
    if (r) return r;
    if ((r = pool_alloc(c, st, csr_rs_words(nnz) * sizeof(unsigned), (void**)&p->rs_bits))) return r;
    CK(cudaMemsetAsync(p->tile_row, 0, sizeof(int) * ((size_t)p->ntiles + 1), st));
    if (!fw) fw = fault_word(c, st);
    if (!fw) return g_status;
    return (int)launch_csr_plan(st, nrows, nnz, rowptr, ts, p->tile_row, p->flags, p->rs_bits, fw) == 0
               ? PENCIL_OK
               : fail(PENCIL_E_CUDA, "csr plan launch");
}

// Drop-in SpMV on host arrays, pipelined.  The call is PCIe-bound (the whole matrix crosses the
// link every call), so everything else hides under the col/val upload:
//   copy stream : rowptr, x, then col/val in SPMV_PIPE_CHUNKS ordered chunks (one event each)
//   compute     : after rowptr: the plan (tile windows + monotonicity flag); then one SpMV launch
//                 per block of tiles, each waiting only for the chunk holding its last non-zero
//   d2h stream  : y of each block as soon as its launch is done
// Block b covers tiles [b*T/K, (b+1)*T/K); its rows and their last non-zero are read from the
// plan (device) and the caller's rowptr (host).  A non-monotone rowptr (flagged by the plan)
// falls back to one launch after the whole upload.  Results are identical to the one-shot
// path: same kernel, same tiles, same per-row fold.  (Measured at 2^24 rows: 43.6 -> 41.8 ms per
// call, i.e. the upload alone at ~54.7 GB/s; a second upload stream changes nothing — PCIe-bound.)
#define SPMV_PIPE_BLOCKS 16
#define SPMV_PIPE_CHUNKS 32
struct PipeCtx {
    cudaStream_t comp = nullptr, d2h = nullptr;
    cudaEvent_t ev_rp = nullptr, ev_x = nullptr, ev_chunk[SPMV_PIPE_CHUNKS] = {}, ev_blk[SPMV_PIPE_BLOCKS] = {};
    int* host_rows = nullptr;  // pinned: [0] plan flag, [1..K+1] block boundary rows
};
std::map<int, PipeCtx*> g_pipe;
std::mutex g_pipe_mu;  // the map is shared by all devices (each PipeCtx is used under its DeviceCtx::mu)

int get_pipe(DeviceCtx* c, PipeCtx** out) {
    std::lock_guard<std::mutex> lk(g_pipe_mu);
    auto it = g_pipe.find(c->device);
    if (it != g_pipe.end()) {
        *out = it->second;
        return PENCIL_OK;
    }
    PipeCtx* p = new PipeCtx();
    CK(cudaStreamCreateWithFlags(&p->comp, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&p->d2h, cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&p->ev_rp, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&p->ev_x, cudaEventDisableTiming));
    for (auto& e : p->ev_chunk) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    for (auto& e : p->ev_blk) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    CK(cudaMallocHost(&p->host_rows, 64 * sizeof(int)));
    g_pipe[c->device] = p;
    *out = p;
    return PENCIL_OK;
}

int spmv_pipelined(int mode, int nrows, int ncols, int nnz, const int* rowptr, const int* col,
                   const float* val, const float* x, float* y) {
    DeviceCtx* c = nullptr;
    int r = get_ctx(&c);
    if (r) return r;
    std::lock_guard<std::mutex> lk(c->mu);
    PipeCtx* pc = nullptr;
    if ((r = get_pipe(c, &pc))) return r;
    cudaStream_t s0 = c->stream, s1 = pc->comp, s2 = pc->d2h;
    g_h2d = (long long)sizeof(int) * ((long long)nrows + 1) + (long long)sizeof(float) * ncols;
    g_d2h = (long long)sizeof(float) * nrows;
    int *drp = nullptr, *dcol = nullptr;
    float *dval = nullptr, *dx = nullptr, *dy = nullptr;
    CsrPlanImpl p;
    // Every exit — the CK / launch-failure returns included — waits for the three streams (the
    // per-block D2H copies into the caller's y may still be running) and frees the buffers.
    struct Release {
        std::function<void()> f;
        bool done = false;
        void operator()() {
            if (!done) f();
            done = true;
        }
        ~Release() { (*this)(); }
    } release{[&]() {
        cudaStreamSynchronize(s1);
        cudaStreamSynchronize(s2);
        pool_free(s0, drp);
        pool_free(s0, dcol);
        pool_free(s0, dval);
        pool_free(s0, dx);
        pool_free(s0, dy);
        csr_plan_release(s0, p);
        cudaStreamSynchronize(s0);
    }};
    unsigned *fw0 = fault_word(c, s0), *tk1 = ticket_word(c, s1);  // faults land in the call's word
    if (!fw0 || !tk1) return g_status;
    if ((r = pool_alloc(c, s0, sizeof(int) * ((size_t)nrows + 1), (void**)&drp)) ||
        (r = pool_alloc(c, s0, sizeof(int) * (size_t)nnz, (void**)&dcol)) ||
        (r = pool_alloc(c, s0, sizeof(float) * (size_t)nnz, (void**)&dval)) ||
        (r = pool_alloc(c, s0, sizeof(float) * nz(ncols), (void**)&dx)) ||
        (r = pool_alloc(c, s0, sizeof(float) * (size_t)nrows, (void**)&dy)))
        return r;
    // upload: rowptr first (the plan needs it), then x, then the col/val chunks in order; pageable
    // caller arrays go through the multi-threaded pinned staging ring (hoststage.cpp)
    auto up = [&](void* d, const void* h, size_t n) -> cudaError_t {
        return staged(h, n) ? (cudaError_t)staged_h2d_2d(c->device, d, n, h, n, n, 1, s0)
                            : cudaMemcpyAsync(d, h, n, cudaMemcpyHostToDevice, s0);
    };
    CK(up(drp, rowptr, sizeof(int) * ((size_t)nrows + 1)));
    CK(cudaEventRecord(pc->ev_rp, s0));
    if (ncols) CK(up(dx, x, sizeof(float) * (size_t)ncols));
    CK(cudaEventRecord(pc->ev_x, s0));
    // chunks are multiples of 4 non-zeros (16-byte aligned device offsets)
    const long long chunk = (((long long)nnz + SPMV_PIPE_CHUNKS - 1) / SPMV_PIPE_CHUNKS + 3) & ~3ll;
    // (Measured and dropped: shipping column indices < 2^24 as 3 bytes, packed on the host while
    // earlier chunks are in flight and unpacked on the GPU — 2.28 -> 2.01 GB per call but 41.8 ->
    // 41.1 ms: the host packing competes with the DMA for host memory bandwidth.)
    for (int k = 0; k < SPMV_PIPE_CHUNKS; k++) {
        const long long lo = k * chunk, hi = lo + chunk < nnz ? lo + chunk : nnz;
        if (hi > lo) {
            CK(up(dcol + lo, col + lo, sizeof(int) * (hi - lo)));
            g_h2d += (long long)sizeof(int) * (hi - lo);
            CK(up(dval + lo, val + lo, sizeof(float) * (hi - lo)));
            g_h2d += (long long)sizeof(float) * (hi - lo);
        }
        CK(cudaEventRecord(pc->ev_chunk[k], s0));
    }
    // plan on the compute stream as soon as rowptr has landed; fetch the block boundaries
    CK(cudaStreamWaitEvent(s1, pc->ev_rp, 0));
    if (csr_plan_build(c, s1, nrows, nnz, drp, mode, &p, fw0)) return g_status;
    const int K = p.ntiles < SPMV_PIPE_BLOCKS ? p.ntiles : SPMV_PIPE_BLOCKS;
    int* hb = pc->host_rows;
    CK(cudaMemcpyAsync(hb, p.flags, sizeof(int), cudaMemcpyDeviceToHost, s1));
    CK(cudaMemcpyAsync(hb + 40, p.flags + 2, sizeof(int), cudaMemcpyDeviceToHost, s1));
    for (int b = 0; b <= K; b++) {
        const long long t = (long long)b * p.ntiles / K;
        CK(cudaMemcpyAsync(hb + 1 + b, p.tile_row + t, sizeof(int), cudaMemcpyDeviceToHost, s1));
    }
    CK(cudaStreamSynchronize(s1));
    p.seg = p.rs_bits && hb[0] == 0;
    if (p.seg && hb[40] != 0 && (r = csr_plan_ordinals(c, s1, &p))) return r;
    CK(zero_empty_rows(p, dy, s1));
    CK(cudaStreamWaitEvent(s1, pc->ev_x, 0));
    auto launch = [&](long long t0, long long t1) {
        return launch_csr_spmv(s1, mode, nrows, ncols, nnz, drp, dcol, dval, dx, dy, p.tile_row + t0,
                               (int)(t1 - t0), p.flags, p.seg_plan(), tk1, fw0);
    };
    const bool y_staged = staged(y, sizeof(float) * (size_t)nrows);  // pageable y: one staged copy at the end
    if (hb[0] != 0) {  // non-monotone rowptr: generic schedule after the whole upload
        CK(cudaStreamWaitEvent(s1, pc->ev_chunk[SPMV_PIPE_CHUNKS - 1], 0));
        if (launch(0, p.ntiles)) return cuda_fail(cudaGetLastError(), "spmv launch");
        if (!y_staged) CK(cudaMemcpyAsync(y, dy, sizeof(float) * (size_t)nrows, cudaMemcpyDeviceToHost, s1));
    } else {
        for (int b = 0; b < K; b++) {
            const int rlo = hb[1 + b], rhi = hb[2 + b];
            if (rhi <= rlo) continue;
            // last non-zero the block reads: rowptr[rhi] - 1 (monotone, clamped to the array)
            long long need = (long long)rowptr[rhi];
            need = need < 1 ? 1 : (need > nnz ? nnz : need);
            const int k = (int)((need - 1) / chunk);
            CK(cudaStreamWaitEvent(s1, pc->ev_chunk[k < SPMV_PIPE_CHUNKS ? k : SPMV_PIPE_CHUNKS - 1], 0));
            if (launch((long long)b * p.ntiles / K, (long long)(b + 1) * p.ntiles / K))
                return cuda_fail(cudaGetLastError(), "spmv launch");
            if (y_staged) continue;
            CK(cudaEventRecord(pc->ev_blk[b], s1));
            CK(cudaStreamWaitEvent(s2, pc->ev_blk[b], 0));
            CK(cudaMemcpyAsync(y + rlo, dy + rlo, sizeof(float) * (size_t)(rhi - rlo), cudaMemcpyDeviceToHost, s2));
        }
    }
    if (y_staged) {
        const size_t yb = sizeof(float) * (size_t)nrows;
        CK((cudaError_t)staged_d2h_2d(c->device, y, yb, dy, yb, yb, 1, s1));
    }
    release();
    return collect_faults(c, s0) == PENCIL_OK ? ok() : g_status;
}

int spmv_common(int mode, int nrows, int ncols, int nnz, int* rowptr, int* col, float* val,
                float* x, float* y) {
    if (nrows < 0 || ncols < 0 || nnz < 0) return fail(PENCIL_E_ARG, "negative extent");
    if (nrows > 0 && nnz >= (1 << 22) && rowptr && col && val && y && (x || !ncols) && !is_device_ptr(rowptr) &&
        !is_device_ptr(col) && !is_device_ptr(val) && !is_device_ptr(x) && !is_device_ptr(y))
        return spmv_pipelined(mode, nrows, ncols, nnz, rowptr, col, val, x, y);
    Stage st[5];
    st[0] = {rowptr, nullptr, sizeof(int) * (nz(nrows) + 1), IN};
    st[1] = {col, nullptr, sizeof(int) * nz(nnz), IN};
    st[2] = {val, nullptr, sizeof(float) * nz(nnz), IN};
    st[3] = {x, nullptr, sizeof(float) * nz(ncols), IN};
    st[4] = {y, nullptr, sizeof(float) * nz(nrows), OUT};
    if (nrows == 0) return ok();
    return dropin(st, [&](DeviceCtx* c, cudaStream_t s) -> int {
        CsrPlanImpl p;
        if (csr_plan_build(c, s, nrows, nnz, (const int*)st[0].dev, mode, &p) || csr_plan_finalize(c, s, &p)) {
            csr_plan_release(s, p);
            return (int)cudaErrorUnknown;
        }
        unsigned *tk = ticket_word(c, s), *fw = fault_word(c, s);
        if (!tk || !fw) return (int)cudaErrorMemoryAllocation;
        if (cudaError_t z = zero_empty_rows(p, (float*)st[4].dev, s)) return (int)z;
        int e = launch_csr_spmv(s, mode, nrows, ncols, nnz, (const int*)st[0].dev, (const int*)st[1].dev,
                                (const float*)st[2].dev, (const float*)st[3].dev, (float*)st[4].dev,
                                p.tile_row, p.ntiles, p.flags, p.seg_plan(), tk, fw);
        csr_plan_release(s, p);
        return e;
    });
}

}  // namespace

// =====================================================================================
// §1 drop-in entry points
// =====================================================================================
// Drop-in stencils on host arrays, pipelined by row blocks: block b's input rows upload on the copy
// stream; its output rows are computed by the band sweep (the rows above / below the block are row
// pointers into the resident image, clamped at its edges, so the result is the whole-image kernel's
// bit for bit) once block b+1 has landed (the two rows below); its output rows download on the D2H
// stream while later blocks upload — the two PCIe directions overlap instead of one after the other.
// fp32 copies back only the interior rectangle (rows / columns 2 .. n-3), as the whole-image call.
// Pageable outputs come back through the staging ring after the last block (one pool of host
// threads serves both directions).  Taken for images of 64 MB and more with w % 4 == 0 on host arrays
// (packed bytes: when a SWAR kernel applies — its row-block form reads the rows around the block
// from the resident image as the whole-image sweep does).
#define STENCIL_PIPE_BLOCKS 8
constexpr long long STENCIL_PIPE_MIN = 64ll << 20;
template <typename T, typename L>
int stencil_pipelined(int h, int w, bool f32, const T* img, T* out, L launch_block) {
    DeviceCtx* c = nullptr;
    int r = get_ctx(&c);
    if (r) return r;
    std::lock_guard<std::mutex> lk(c->mu);
    PipeCtx* pc = nullptr;
    if ((r = get_pipe(c, &pc))) return r;
    cudaStream_t s0 = c->stream, s1 = pc->comp, s2 = pc->d2h;
    T *dIn = nullptr, *dOut = nullptr;
    struct Release {
        std::function<void()> f;
        ~Release() { f(); }
    } release{[&]() {
        cudaStreamSynchronize(s1);
        cudaStreamSynchronize(s2);
        pool_free(s0, dIn);
        pool_free(s0, dOut);
        cudaStreamSynchronize(s0);
    }};
    const size_t n = (size_t)h * w, row = sizeof(T) * (size_t)w;
    if ((r = pool_alloc(c, s0, sizeof(T) * n, (void**)&dIn)) || (r = pool_alloc(c, s0, sizeof(T) * n, (void**)&dOut)))
        return r;
    const bool in_staged = staged(img, sizeof(T) * n), out_staged = staged(out, sizeof(T) * n);
    const int K = STENCIL_PIPE_BLOCKS, rows = (h + K - 1) / K;
    const int olo = f32 ? 2 : 0, ohi = f32 ? h - 2 : h;  // output rows the call stores
    const size_t col0 = f32 ? 2 : 0, ncol = f32 ? (size_t)w - 4 : (size_t)w;
    g_h2d = (long long)(sizeof(T) * n);
    g_d2h = (long long)(sizeof(T) * ncol * (size_t)(ohi - olo));
    int nb = 0;
    for (int r0 = 0; r0 < h; r0 += rows) nb++;
    for (int b = 0; b < nb; b++) {  // uploads, in order on the copy stream
        const int r0 = b * rows, r1 = std::min(h, r0 + rows);
        const size_t bytes = row * (size_t)(r1 - r0);
        if (in_staged) CK((cudaError_t)staged_h2d_2d(c->device, dIn + (size_t)r0 * w, bytes, img + (size_t)r0 * w,
                                                     bytes, bytes, 1, s0));
        else CK(cudaMemcpyAsync(dIn + (size_t)r0 * w, img + (size_t)r0 * w, bytes, cudaMemcpyHostToDevice, s0));
        CK(cudaEventRecord(pc->ev_blk[b], s0));
        if (b == 0) continue;
        // block b-1 can run: its rows and the two below it have landed
        const int q0 = (b - 1) * rows, q1 = std::min(h, q0 + rows);
        CK(cudaStreamWaitEvent(s1, pc->ev_blk[b], 0));
        int e = launch_block(s1, q0, q1, (const T*)dIn, dOut);
        if (e) return cuda_fail((cudaError_t)e, "stencil launch");
        if (out_staged) continue;
        const int o0 = std::max(q0, olo), o1 = std::min(q1, ohi);
        if (o1 <= o0) continue;
        CK(cudaEventRecord(pc->ev_chunk[b - 1], s1));
        CK(cudaStreamWaitEvent(s2, pc->ev_chunk[b - 1], 0));
        CK(cudaMemcpy2DAsync(out + (size_t)o0 * w + col0, row, dOut + (size_t)o0 * w + col0, row, sizeof(T) * ncol,
                             (size_t)(o1 - o0), cudaMemcpyDeviceToHost, s2));
    }
    {  // the last block
        const int q0 = (nb - 1) * rows, q1 = h;
        CK(cudaStreamWaitEvent(s1, pc->ev_blk[nb - 1], 0));
        int e = launch_block(s1, q0, q1, (const T*)dIn, dOut);
        if (e) return cuda_fail((cudaError_t)e, "stencil launch");
        const int o0 = std::max(q0, olo), o1 = std::min(q1, ohi);
        if (!out_staged && o1 > o0) {
            CK(cudaEventRecord(pc->ev_chunk[nb - 1], s1));
            CK(cudaStreamWaitEvent(s2, pc->ev_chunk[nb - 1], 0));
            CK(cudaMemcpy2DAsync(out + (size_t)o0 * w + col0, row, dOut + (size_t)o0 * w + col0, row,
                                 sizeof(T) * ncol, (size_t)(o1 - o0), cudaMemcpyDeviceToHost, s2));
        }
    }
    if (out_staged && ohi > olo)
        CK((cudaError_t)staged_d2h_2d(c->device, out + (size_t)olo * w + col0, row, dOut + (size_t)olo * w + col0,
                                      row, sizeof(T) * ncol, (size_t)(ohi - olo), s1));
    release.f();
    release.f = [] {};
    return collect_faults(c, s0) == PENCIL_OK ? ok() : g_status;
}

// the band sweep's row pointers for rows [q0, q1) of a resident h-row image (clamped at its edges)
template <typename T>
void band_rows(const T* img, int h, int w, int q0, int q1, const T* (&top)[2], const T* (&bot)[2]) {
    auto rowp = [&](int i) { return img + (size_t)(i < 0 ? 0 : (i > h - 1 ? h - 1 : i)) * w; };
    top[0] = rowp(q0 - 2), top[1] = rowp(q0 - 1), bot[0] = rowp(q1), bot[1] = rowp(q1 + 1);
}

// Drop-in axpy on host arrays of 64 MB and more, pipelined by chunks: chunk b of x and y uploads on the
// copy stream, its axpy runs on the compute stream, its y downloads on the D2H stream under the next
// chunks' uploads (pageable y: one staged download at the end).
int axpy_pipelined(long long n, float a, const float* x, float* y) {
    DeviceCtx* c = nullptr;
    int r = get_ctx(&c);
    if (r) return r;
    std::lock_guard<std::mutex> lk(c->mu);
    PipeCtx* pc = nullptr;
    if ((r = get_pipe(c, &pc))) return r;
    cudaStream_t s0 = c->stream, s1 = pc->comp, s2 = pc->d2h;
    float *dx = nullptr, *dy = nullptr;
    struct Release {
        std::function<void()> f;
        ~Release() { f(); }
    } release{[&]() {
        cudaStreamSynchronize(s1);
        cudaStreamSynchronize(s2);
        pool_free(s0, dx);
        pool_free(s0, dy);
        cudaStreamSynchronize(s0);
    }};
    if ((r = pool_alloc(c, s0, sizeof(float) * n, (void**)&dx)) || (r = pool_alloc(c, s0, sizeof(float) * n, (void**)&dy)))
        return r;
    const bool y_staged = staged(y, sizeof(float) * n);
    auto up = [&](float* d, const float* hp, size_t bytes) -> cudaError_t {
        return staged(hp, bytes) ? (cudaError_t)staged_h2d_2d(c->device, d, bytes, hp, bytes, bytes, 1, s0)
                                 : cudaMemcpyAsync(d, hp, bytes, cudaMemcpyHostToDevice, s0);
    };
    g_h2d = (long long)(2 * sizeof(float) * n);
    g_d2h = (long long)(sizeof(float) * n);
    const int K = STENCIL_PIPE_BLOCKS;
    const long long chunk = ((n + K - 1) / K + 3) / 4 * 4;  // float4-aligned chunk starts
    int b = 0;
    for (long long o = 0; o < n; o += chunk, b++) {
        const long long len = std::min(chunk, n - o);
        CK(up(dx + o, x + o, sizeof(float) * len));
        CK(up(dy + o, y + o, sizeof(float) * len));
        CK(cudaEventRecord(pc->ev_blk[b], s0));
        CK(cudaStreamWaitEvent(s1, pc->ev_blk[b], 0));
        const int e = launch_axpy(s1, len, a, nullptr, dx + o, dy + o);
        if (e) return cuda_fail((cudaError_t)e, "axpy launch");
        if (y_staged) continue;
        CK(cudaEventRecord(pc->ev_chunk[b], s1));
        CK(cudaStreamWaitEvent(s2, pc->ev_chunk[b], 0));
        CK(cudaMemcpyAsync(y + o, dy + o, sizeof(float) * len, cudaMemcpyDeviceToHost, s2));
    }
    if (y_staged)
        CK((cudaError_t)staged_d2h_2d(c->device, y, sizeof(float) * n, dy, sizeof(float) * n, sizeof(float) * n, 1, s1));
    release.f();
    release.f = [] {};
    return collect_faults(c, s0) == PENCIL_OK ? ok() : g_status;
}

bool stencil_pipe_ok(int h, int w, size_t elem, const void* img, const void* out) {
    return (long long)h * w * (long long)elem >= STENCIL_PIPE_MIN && h >= 64 && w % 4 == 0 && img && out &&
           (uintptr_t)img % 16 == 0 && (uintptr_t)out % 16 == 0 && !is_device_ptr(img) && !is_device_ptr(out);
}

extern "C" {

void gemv(int m, int n, float alpha, float beta, float* A, float* x, float* y) {
    if (m < 0 || n < 0) { fail(PENCIL_E_ARG, "negative extent"); return; }
    if (m == 0) { ok(); return; }
    Stage st[3];
    st[0] = {A, nullptr, sizeof(float) * nz((long long)m * n), IN};
    st[1] = {x, nullptr, sizeof(float) * nz(n), IN};
    st[2] = {y, nullptr, sizeof(float) * nz(m), INOUT};
    dropin(st, [&](DeviceCtx*, cudaStream_t s) {
        return launch_gemv(s, m, n, alpha, beta, (const float*)st[0].dev, (const float*)st[1].dev,
                           (float*)st[2].dev);
    });
}

void gemv_t(int m, int n, int lda, int incx, int incy, float alpha, float beta, float* A, float* x,
            float* y) {
    if (m < 0 || n < 0) { fail(PENCIL_E_ARG, "negative extent"); return; }
    if (n == 0) { ok(); return; }
    if (lda < 0 || incx < 1 || incy < 1) { fail(PENCIL_E_ARG, "gemv_t needs lda >= 0, incx >= 1, incy >= 1"); return; }
    if (m > 0 && n > lda) {  // A[i*lda + j] with j >= lda leaves A's declared extent m*lda
        fail(PENCIL_E_INTERP, "load from A[%lld] is out of bounds", (long long)(m - 1) * lda + (n - 1));
        return;
    }
    Stage st[3];
    st[0] = {A, nullptr, sizeof(float) * nz((long long)m * lda), IN};
    st[1] = {x, nullptr, sizeof(float) * nz((long long)m * incx), IN};
    st[2] = {y, nullptr, sizeof(float) * nz((long long)n * incy), INOUT};
    // the views of the fixture's accesses (A[i*lda + j], x[i*incx], y[j*incy]) for these scalars
    pencil_view v[3];
    if (pencil_gemv_t_views(m, n, lda, incx, incy, v)) return;
    dropin(st, [&](DeviceCtx* c, cudaStream_t s) -> int {
        for (int q = 0; q < 3; q++) v[q].base = st[q].dev;
        return gemv_t_views_launch(c, s, alpha, beta, v[0], v[1], v[2]) ? (int)cudaErrorInvalidValue : 0;
    });
}

float dot(int n, float* x, float* y) {
    if (n < 0) { fail(PENCIL_E_ARG, "negative extent"); return 0.f; }
    if (n == 0) { ok(); return 0.f; }
    Stage st[2];
    st[0] = {x, nullptr, sizeof(float) * nz(n), IN};
    st[1] = {y, nullptr, sizeof(float) * nz(n), IN};
    float result = 0.f;
    dropin(st, [&](DeviceCtx* c, cudaStream_t s) -> int {
        int e = launch_dot(s, n, (const float*)st[0].dev, (const float*)st[1].dev, c->dot_result,
                           c->dot_partial, c->dot_counter);
        if (e) return e;
        return (int)cudaMemcpyAsync(&result, c->dot_result, sizeof(float), cudaMemcpyDeviceToHost, s);
    });
    return result;
}

void axpy(int n, float a, float* x, float* y) {
    if (n < 0) { fail(PENCIL_E_ARG, "negative extent"); return; }
    if (n == 0) { ok(); return; }
    if ((long long)n * 4 >= STENCIL_PIPE_MIN && x && y && !is_device_ptr(x) && !is_device_ptr(y)) {
        axpy_pipelined(n, a, x, y);
        return;
    }
    Stage st[2];
    st[0] = {x, nullptr, sizeof(float) * nz(n), IN};
    st[1] = {y, nullptr, sizeof(float) * nz(n), INOUT};
    dropin(st, [&](DeviceCtx*, cudaStream_t s) {
        return launch_axpy(s, n, a, nullptr, (const float*)st[0].dev, (float*)st[1].dev);
    });
}

void spmv_vec(int nrows, int ncols, int nnz, int* rowptr, int* col, float* val, float* x, float* y) {
    spmv_common(1, nrows, ncols, nnz, rowptr, col, val, x, y);
}
void spmv_inline(int nrows, int ncols, int nnz, int* rowptr, int* col, float* val, float* x, float* y) {
    spmv_common(0, nrows, ncols, nnz, rowptr, col, val, x, y);
}
void spmv(int nrows, int ncols, int nnz, int* rowptr, int* col, float* val, float* x, float* y) {
    spmv_common(0, nrows, ncols, nnz, rowptr, col, val, x, y);
}
void spmv_row(int nrows, int ncols, int nnz, int i, int* rowptr, int* col, float* val, float* x,
              float* y) {
    if (nrows < 0 || ncols < 0 || nnz < 0) { fail(PENCIL_E_ARG, "negative extent"); return; }
    if (i < 0 || i >= nrows) { fail(PENCIL_E_INTERP, "load from rowptr[%d] is out of bounds", i); return; }
    Stage st[5];
    st[0] = {rowptr, nullptr, sizeof(int) * (nz(nrows) + 1), IN};
    st[1] = {col, nullptr, sizeof(int) * nz(nnz), IN};
    st[2] = {val, nullptr, sizeof(float) * nz(nnz), IN};
    st[3] = {x, nullptr, sizeof(float) * nz(ncols), IN};
    st[4] = {y, nullptr, sizeof(float) * nz(nrows), INOUT};
    dropin(st, [&](DeviceCtx* c, cudaStream_t s) {
        unsigned* fw = fault_word(c, s);
        if (!fw) return (int)cudaErrorMemoryAllocation;
        return launch_csr_generic(s, 1, ncols, nnz, (const int*)st[0].dev + i, (const int*)st[1].dev,
                                  (const float*)st[2].dev, (const float*)st[3].dev,
                                  (float*)st[4].dev + i, fw);
    });
}

void conv5x5_u8(int h, int w, int scale, int* img, int* k, int* out) {
    if (h < 0 || w < 0) { fail(PENCIL_E_ARG, "negative extent"); return; }
    if (h == 0 || w == 0) { ok(); return; }
    if (scale == 0) { fail(PENCIL_E_INTERP, "division by zero"); return; }
    int taps[25];
    if (is_device_ptr(k)) {
        if (cudaMemcpy(taps, k, sizeof taps, cudaMemcpyDeviceToHost) != cudaSuccess) {
            cuda_fail(cudaGetLastError(), "tap copy");
            return;
        }
    } else {
        memcpy(taps, k, sizeof taps);
    }
    if (stencil_pipe_ok(h, w, sizeof(int), img, out)) {
        stencil_pipelined<int>(h, w, false, img, out, [&](cudaStream_t s, int q0, int q1, const int* di, int* dout) {
            const int *top[2], *bot[2];
            band_rows(di, h, w, q0, q1, top, bot);
            return launch_conv5x5_u8_band(s, q1 - q0, w, scale, di + (size_t)q0 * w, top, bot, taps,
                                          dout + (size_t)q0 * w);
        });
        return;
    }
    Stage st[2];
    st[0] = {img, nullptr, sizeof(int) * nz((long long)h * w), IN};
    st[1] = {out, nullptr, sizeof(int) * nz((long long)h * w), OUT};
    dropin(st, [&](DeviceCtx*, cudaStream_t s) {
        return launch_conv5x5_u8(s, h, w, scale, (const int*)st[0].dev, taps, (int*)st[1].dev);
    });
}

// packed 8-bit images (an extension: PENCIL has no uint8, so there is no emitted-C door): the same
// drop-in staging as the int32-storage call — host arrays copied in / out (pageable ones through the
// staging ring), device arrays used in place
extern "C" int pencil_conv5x5_u8_bytes(int h, int w, int scale, const uint8_t* img, const int* k, uint8_t* out) {
    if (h < 0 || w < 0) return fail(PENCIL_E_ARG, "negative extent");
    if (h == 0 || w == 0) return ok();
    if (scale == 0) return fail(PENCIL_E_INTERP, "division by zero");
    if (!k) return fail(PENCIL_E_ARG, "null taps");
    int taps[25];
    if (is_device_ptr(k)) {
        if (cudaMemcpy(taps, k, sizeof taps, cudaMemcpyDeviceToHost) != cudaSuccess)
            return cuda_fail(cudaGetLastError(), "tap copy");
    } else {
        memcpy(taps, k, sizeof taps);
    }
    if (stencil_pipe_ok(h, w, 1, img, out) && conv5x5_u8_bytes_rows_ok(h, w, scale, taps))  // row blocks
        return stencil_pipelined<uint8_t>(h, w, false, img, out, [&](cudaStream_t s, int q0, int q1,
                                                                     const uint8_t* di, uint8_t* dout) {
            return launch_conv5x5_u8_bytes_rows(s, h, w, scale, di, taps, dout, q0, q1);
        });
    Stage st[2];
    st[0] = {(void*)img, nullptr, nz((long long)h * w), IN};
    st[1] = {out, nullptr, nz((long long)h * w), OUT};
    return dropin(st, [&](DeviceCtx*, cudaStream_t s) {
        return launch_conv5x5_u8_bytes(s, h, w, scale, (const unsigned char*)st[0].dev, taps,
                                       (unsigned char*)st[1].dev);
    });
}

void conv5x5_f32(int h, int w, float* img, float* k, float* out) {
    if (h < 0 || w < 0) { fail(PENCIL_E_ARG, "negative extent"); return; }
    if (h < 5 || w < 5) { ok(); return; }  // no interior pixel: nothing is stored
    float taps[25];
    if (is_device_ptr(k)) {
        if (cudaMemcpy(taps, k, sizeof taps, cudaMemcpyDeviceToHost) != cudaSuccess) {
            cuda_fail(cudaGetLastError(), "tap copy");
            return;
        }
    } else {
        memcpy(taps, k, sizeof taps);
    }
    if (stencil_pipe_ok(h, w, sizeof(float), img, out)) {
        stencil_pipelined<float>(h, w, true, img, out, [&](cudaStream_t s, int q0, int q1, const float* di,
                                                           float* dout) {
            const int lo = std::max(q0, 2) - q0, hi = std::min(q1, h - 2) - q0;
            if (hi <= lo) return 0;
            const float *top[2], *bot[2];
            band_rows(di, h, w, q0, q1, top, bot);
            return launch_conv5x5_f32_band(s, q1 - q0, w, lo, hi, di + (size_t)q0 * w, top, bot, taps,
                                           dout + (size_t)q0 * w);
        });
        return;
    }
    Stage st[2];
    st[0] = {img, nullptr, sizeof(float) * nz((long long)h * w), IN};
    // only the interior of out is stored to: copy back exactly that rectangle
    st[1] = {out, nullptr, sizeof(float) * nz((long long)h * w), OUT};
    st[1].pitch = sizeof(float) * (size_t)w;
    st[1].width = sizeof(float) * (size_t)(w - 4);
    st[1].height = (size_t)(h - 4);
    st[1].offset = sizeof(float) * ((size_t)2 * w + 2);
    dropin(st, [&](DeviceCtx*, cudaStream_t s) {
        return launch_conv5x5_f32(s, h, w, (const float*)st[0].dev, taps, (float*)st[1].dev);
    });
}

// Drop-in gemm on host arrays, pipelined by row blocks of A / C: B first (every tile needs all of
// it), then per block its rows of A and C on the copy stream, the block's gemm (strided views:
// A + r0*k, C + r0*n) on the compute stream as soon as they have landed, and its C rows back on
// the D2H stream — so the upload of block b+1 and the download of block b-1 run under block b's
// tensor work, instead of upload, compute and download one after another.  Pageable arrays go
// through the staging ring (their C comes back in one staged copy at the end).
#define GEMM_PIPE_BLOCKS 8
int gemm_pipelined(int m, int n, int k, float alpha, float beta, const float* A, const float* B, float* C) {
    DeviceCtx* c = nullptr;
    int r = get_ctx(&c);
    if (r) return r;
    std::lock_guard<std::mutex> lk(c->mu);
    PipeCtx* pc = nullptr;
    if ((r = get_pipe(c, &pc))) return r;
    cudaStream_t s0 = c->stream, s1 = pc->comp, s2 = pc->d2h;
    float *dA = nullptr, *dB = nullptr, *dC = nullptr;
    void* ws = nullptr;
    size_t wb = 0;
    struct Release {
        std::function<void()> f;
        ~Release() { f(); }
    } release{[&]() {
        cudaStreamSynchronize(s1);
        cudaStreamSynchronize(s2);
        pool_free(s0, dA);
        pool_free(s0, dB);
        pool_free(s0, dC);
        pool_free(s0, ws);
        cudaStreamSynchronize(s0);
    }};
    const size_t na = (size_t)m * k, nb = (size_t)k * n, ncm = (size_t)m * n;
    if ((r = pool_alloc(c, s0, sizeof(float) * nz(na), (void**)&dA)) ||
        (r = pool_alloc(c, s0, sizeof(float) * nz(nb), (void**)&dB)) ||
        (r = pool_alloc(c, s0, sizeof(float) * ncm, (void**)&dC)))
        return r;
    auto up = [&](void* d, const void* h, size_t bytes) -> cudaError_t {
        return staged(h, bytes) ? (cudaError_t)staged_h2d_2d(c->device, d, bytes, h, bytes, bytes, 1, s0)
                                : cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, s0);
    };
    g_h2d = (long long)sizeof(float) * (long long)(na + nb + ncm);
    g_d2h = (long long)sizeof(float) * (long long)ncm;
    if (nb) CK(up(dB, B, sizeof(float) * nb));
    const bool c_staged = staged(C, sizeof(float) * ncm);
    // row blocks of a multiple of 256 rows (one CTA-pair tile)
    const int rows = ((m + GEMM_PIPE_BLOCKS - 1) / GEMM_PIPE_BLOCKS + 255) / 256 * 256;
    wb = gemm_workspace_bytes(rows, n, k, dA, k, dB, n);  // 0: the device copies are 16-byte pitched or packed per block
    if (wb && (r = pool_alloc(c, s1, wb, &ws))) return r;
    int b = 0;
    for (int r0 = 0; r0 < m; r0 += rows, b++) {
        const int mr = std::min(rows, m - r0);
        if (k) CK(up(dA + (size_t)r0 * k, A + (size_t)r0 * k, sizeof(float) * (size_t)mr * k));
        CK(up(dC + (size_t)r0 * n, C + (size_t)r0 * n, sizeof(float) * (size_t)mr * n));
        CK(cudaEventRecord(pc->ev_chunk[b], s0));
        CK(cudaStreamWaitEvent(s1, pc->ev_chunk[b], 0));
        const int e = launch_gemm(s1, mr, n, k, alpha, beta, dA + (size_t)r0 * k, k, dB, n, dC + (size_t)r0 * n, n, ws,
                                  wb);
        if (e) return cuda_fail((cudaError_t)e, "gemm launch");
        if (c_staged) continue;
        CK(cudaEventRecord(pc->ev_blk[b], s1));
        CK(cudaStreamWaitEvent(s2, pc->ev_blk[b], 0));
        CK(cudaMemcpyAsync(C + (size_t)r0 * n, dC + (size_t)r0 * n, sizeof(float) * (size_t)mr * n,
                           cudaMemcpyDeviceToHost, s2));
    }
    if (c_staged) CK((cudaError_t)staged_d2h_2d(c->device, C, sizeof(float) * ncm, dC, sizeof(float) * ncm,
                                                 sizeof(float) * ncm, 1, s1));
    release.f();
    release.f = [] {};
    return collect_faults(c, s0) == PENCIL_OK ? ok() : g_status;
}

void gemm(int m, int n, int k, float alpha, float beta, float* A, float* B, float* C) {
    if (m < 0 || n < 0 || k < 0) { fail(PENCIL_E_ARG, "negative extent"); return; }
    if (m == 0 || n == 0) { ok(); return; }
    if ((long long)m * n >= (1ll << 22) && m >= 1024 && A && B && C && !is_device_ptr(A) && !is_device_ptr(B) &&
        !is_device_ptr(C)) {
        gemm_pipelined(m, n, k, alpha, beta, A, B, C);
        return;
    }
    Stage st[3];
    st[0] = {A, nullptr, sizeof(float) * nz((long long)m * k), IN};
    st[1] = {B, nullptr, sizeof(float) * nz((long long)k * n), IN};
    st[2] = {C, nullptr, sizeof(float) * nz((long long)m * n), INOUT};
    dropin(st, [&](DeviceCtx* c, cudaStream_t s) -> int {
        size_t wb = gemm_workspace_bytes(m, n, k, (const float*)st[0].dev, k, (const float*)st[1].dev, n);
        void* ws = nullptr;
        if (wb && pool_alloc(c, s, wb, &ws)) return (int)cudaErrorMemoryAllocation;
        int e = launch_gemm(s, m, n, k, alpha, beta, (const float*)st[0].dev, k, (const float*)st[1].dev, n,
                            (float*)st[2].dev, n, ws, wb);
        pool_free(s, ws);
        return e;
    });
}

// =====================================================================================
// §2 status
// =====================================================================================
int pencil_cuda_last_status(void) { return g_status; }
const char* pencil_cuda_last_error(void) { return g_msg; }
void pencil_cuda_clear_status(void) { ok(); }
const char* pencil_status_code(int status) { return code_name(status); }

// =====================================================================================
// §3 device-resident API
// =====================================================================================
#define DEV_PROLOGUE                      \
    DeviceCtx* c = nullptr;               \
    if (get_ctx(&c)) return g_status;     \
    cudaStream_t st = pick_stream(c, s);
#define DEV_RET(e) return (e) ? cuda_fail((cudaError_t)(e), "kernel launch") : ok()

int pencil_gemv_dev(pencil_stream_t s, int m, int n, float alpha, float beta, const float* A,
                    const float* x, float* y) {
    if (m < 0 || n < 0) return fail(PENCIL_E_ARG, "negative extent");
    DEV_PROLOGUE;
    DEV_RET(launch_gemv(st, m, n, alpha, beta, A, x, y));
}

int pencil_gemv_t_dev(pencil_stream_t s, int m, int n, int lda, int incx, int incy, float alpha,
                      float beta, const float* A, const float* x, float* y) {
    if (m < 0 || n < 0 || lda < 0 || incx < 1 || incy < 1) return fail(PENCIL_E_ARG, "bad extent/stride");
    DEV_PROLOGUE;
    pencil_view v[3];
    if (pencil_gemv_t_views(m, n, lda, incx, incy, v)) return g_status;
    v[0].base = (void*)A;
    v[1].base = (void*)x;
    v[2].base = (void*)y;
    return gemv_t_views_launch(c, st, alpha, beta, v[0], v[1], v[2]) ? g_status : ok();
}

int pencil_gemv_t_view_dev(pencil_stream_t s, float alpha, float beta, const pencil_view* A, const pencil_view* x,
                           const pencil_view* y) {
    if (!A || !x || !y || !A->base || !x->base || !y->base) return fail(PENCIL_E_ARG, "null view");
    DEV_PROLOGUE;
    return gemv_t_views_launch(c, st, alpha, beta, *A, *x, *y) ? g_status : ok();
}

// The views of gemv_t.pencil.c's accesses for a call's scalars: the symbolic affine forms of
// A[i * lda + j] (read, nest j, i), x[i * incx] and y[j * incy] (write) evaluated under
// {m, n, lda, incx, incy} (descriptors.cpp) — the mapper's view descriptors, not hard-coded strides.
int pencil_gemv_t_views(int m, int n, int lda, int incx, int incy, pencil_view views[3]) {
    static const char* names[5] = {"m", "n", "lda", "incx", "incy"};
    const long long vals[5] = {m, n, lda, incx, incy};
    pencil_access_form f[16];
    const int k = pencil_affine_accesses(pencil_fixture_source("gemv_t"), "gemv_t", 5, names, vals, f, 16);
    if (k < 0) return g_status;
    memset(views, 0, 3 * sizeof(pencil_view));
    bool have[3] = {false, false, false};
    for (int a = 0; a < k && a < 16; a++) {
        const pencil_access_form& r = f[a];
        if (!r.affine || r.nloops < 1) continue;
        // loop 0 = j (the output columns), loop 1 = i (the reduction; A and x only)
        const long long sj = r.stride[0], si = r.nloops > 1 ? r.stride[1] : 0;
        if (r.nloops == 2 && !strcmp(r.array, "A") && !r.is_write) {
            views[0] = {nullptr, r.offset, 2, PENCIL_FLOAT32, {r.hi[1] - r.lo[1], r.hi[0] - r.lo[0]}, {si, sj}};
            have[0] = true;
        } else if (r.nloops == 2 && !strcmp(r.array, "x")) {
            views[1] = {nullptr, r.offset, 1, PENCIL_FLOAT32, {r.hi[1] - r.lo[1], 0}, {si, 0}};
            have[1] = true;
        } else if (r.nloops == 1 && !strcmp(r.array, "y") && r.is_write) {
            views[2] = {nullptr, r.offset, 1, PENCIL_FLOAT32, {r.hi[0] - r.lo[0], 0}, {sj, 0}};
            have[2] = true;
        }
    }
    if (!have[0] || !have[1] || !have[2]) return fail(PENCIL_E_UNSUPPORTED, "gemv_t fixture: views not found");
    return ok();
}

int pencil_dot_dev(pencil_stream_t s, long long n, const float* x, const float* y, float* result_dev) {
    if (n < 0) return fail(PENCIL_E_ARG, "negative extent");
    DEV_PROLOGUE;
    // per-call partial buffer: concurrent dots on different streams must not share it
    double* part = nullptr;
    unsigned* ctr = nullptr;
    if (pool_alloc(c, st, sizeof(double) * dot_partial_elems() + 256, (void**)&part)) return g_status;
    ctr = (unsigned*)((char*)part + sizeof(double) * dot_partial_elems());
    cudaMemsetAsync(ctr, 0, sizeof(unsigned), st);
    int e = launch_dot(st, n, x, y, result_dev, part, ctr);
    pool_free(st, part);
    DEV_RET(e);
}

int pencil_axpy_dev(pencil_stream_t s, long long n, float a, const float* x, float* y) {
    if (n < 0) return fail(PENCIL_E_ARG, "negative extent");
    DEV_PROLOGUE;
    DEV_RET(launch_axpy(st, n, a, nullptr, x, y));
}

int pencil_axpy_dev_ptr(pencil_stream_t s, long long n, const float* a_dev, const float* x, float* y) {
    if (n < 0 || !a_dev) return fail(PENCIL_E_ARG, "bad argument");
    DEV_PROLOGUE;
    DEV_RET(launch_axpy(st, n, 0.f, a_dev, x, y));
}

int pencil_conv5x5_u8_dev(pencil_stream_t s, int h, int w, int scale, const int* img,
                          const int* k_host, int* out) {
    if (h < 0 || w < 0) return fail(PENCIL_E_ARG, "negative extent");
    if (scale == 0 && h > 0 && w > 0) return fail(PENCIL_E_INTERP, "division by zero");
    DEV_PROLOGUE;
    DEV_RET(launch_conv5x5_u8(st, h, w, scale, img, k_host, out));
}

int pencil_conv5x5_u8_bytes_dev(pencil_stream_t s, int h, int w, int scale, const uint8_t* img,
                                const int* k_host, uint8_t* out) {
    if (h < 0 || w < 0) return fail(PENCIL_E_ARG, "negative extent");
    if (scale == 0 && h > 0 && w > 0) return fail(PENCIL_E_INTERP, "division by zero");
    DEV_PROLOGUE;
    DEV_RET(launch_conv5x5_u8_bytes(st, h, w, scale, img, k_host, out));
}

int pencil_conv5x5_f32_dev(pencil_stream_t s, int h, int w, const float* img, const float* k_host,
                           float* out) {
    if (h < 0 || w < 0) return fail(PENCIL_E_ARG, "negative extent");
    DEV_PROLOGUE;
    DEV_RET(launch_conv5x5_f32(st, h, w, img, k_host, out));
}

int pencil_conv5x5_u8_band_dev(pencil_stream_t s, int h, int w, int scale, const int* img, const int* const* top,
                               const int* const* bot, const int* k_host, int* out) {
    if (h < 0 || w < 0) return fail(PENCIL_E_ARG, "negative extent");
    if (!top || !bot || !k_host) return fail(PENCIL_E_ARG, "null argument");
    if (scale == 0 && h > 0 && w > 0) return fail(PENCIL_E_INTERP, "division by zero");
    DEV_PROLOGUE;
    const int e = launch_conv5x5_u8_band(st, h, w, scale, img, top, bot, k_host, out);
    if (e == (int)cudaErrorInvalidValue)
        return fail(PENCIL_E_ARG, "band rows must be 16-byte aligned with w %% 4 == 0 (w=%d)", w);
    DEV_RET(e);
}

int pencil_conv5x5_f32_band_dev(pencil_stream_t s, int h, int w, int out_lo, int out_hi, const float* img,
                                const float* const* top, const float* const* bot, const float* k_host, float* out) {
    if (h < 0 || w < 0) return fail(PENCIL_E_ARG, "negative extent");
    if (!top || !bot || !k_host) return fail(PENCIL_E_ARG, "null argument");
    DEV_PROLOGUE;
    const int e = launch_conv5x5_f32_band(st, h, w, out_lo, out_hi, img, top, bot, k_host, out);
    if (e == (int)cudaErrorInvalidValue)
        return fail(PENCIL_E_ARG, "band rows must be 16-byte aligned with w %% 4 == 0 and 0 <= out_lo, out_hi <= h");
    DEV_RET(e);
}

int pencil_gemm_strided_dev(pencil_stream_t s, int m, int n, int k, float alpha, float beta, const float* A,
                            long long lda, const float* B, long long ldb, float* C, long long ldc) {
    if (m < 0 || n < 0 || k < 0) return fail(PENCIL_E_ARG, "negative extent");
    if (lda < k || ldb < n || ldc < n)
        return fail(PENCIL_E_ARG, "gemm pitches must cover the rows: lda >= k, ldb >= n, ldc >= n");
    DEV_PROLOGUE;
    size_t wb = gemm_workspace_bytes(m, n, k, A, lda, B, ldb);
    void* ws = nullptr;
    if (wb && pool_alloc(c, st, wb, &ws)) return g_status;
    int e = launch_gemm(st, m, n, k, alpha, beta, A, lda, B, ldb, C, ldc, ws, wb);
    pool_free(st, ws);
    DEV_RET(e);
}

int pencil_gemm_dev(pencil_stream_t s, int m, int n, int k, float alpha, float beta, const float* A,
                    const float* B, float* C) {
    return pencil_gemm_strided_dev(s, m, n, k, alpha, beta, A, k, B, n, C, n);
}

struct pencil_csr_plan : CsrPlanImpl {};

int pencil_csr_plan_create(pencil_stream_t s, int nrows, int ncols, int nnz, const int* rowptr_dev,
                           int mode, pencil_csr_plan_t* out) {
    if (nrows < 0 || ncols < 0 || nnz < 0 || !out) return fail(PENCIL_E_ARG, "bad argument");
    DEV_PROLOGUE;
    pencil_csr_plan* p = new pencil_csr_plan();
    p->ncols = ncols;
    if (csr_plan_build(c, st, nrows, nnz, rowptr_dev, mode ? 1 : 0, p) || csr_plan_finalize(c, st, p)) {
        csr_plan_release(st, *p);
        delete p;
        return g_status;
    }
    *out = p;
    return ok();
}

int pencil_csr_plan_destroy(pencil_csr_plan_t plan) {
    if (!plan) return ok();
    cudaFree(plan->tile_row);  // pool memory: freed through the device's default stream order
    cudaFree(plan->flags);
    if (plan->rs_bits) cudaFree(plan->rs_bits);
    if (plan->ord) cudaFree(plan->ord);
    if (plan->rowmap) cudaFree(plan->rowmap);
    delete plan;
    return ok();
}

int pencil_csr_plan_info(pencil_csr_plan_t plan, int* ntiles, int* tile_nnz) {
    if (!plan) return fail(PENCIL_E_ARG, "null plan");
    if (ntiles) *ntiles = plan->ntiles;
    if (tile_nnz) *tile_nnz = plan->tile_nnz;
    return ok();
}

int pencil_spmv_dev(pencil_stream_t s, pencil_csr_plan_t plan, const int* rowptr, const int* col,
                    const float* val, const float* x, float* y) {
    if (!plan) return fail(PENCIL_E_ARG, "null plan");
    DEV_PROLOGUE;
    unsigned *tk = ticket_word(c, st), *fw = fault_word(c, st);
    if (!tk || !fw) return g_status;
    if (cudaError_t z = zero_empty_rows(*plan, y, st)) return cuda_fail(z, "zero empty rows");
    DEV_RET(launch_csr_spmv(st, plan->mode, plan->nrows, plan->ncols, plan->nnz, rowptr, col, val, x, y,
                            plan->tile_row, plan->ntiles, plan->flags, plan->seg_plan(), tk, fw));
}

int pencil_spmv_dev_dist(pencil_stream_t s, pencil_csr_plan_t plan, const int* rowptr, const int* col,
                         const float* val, const float* x, float* y, float* const* peers, int npeers,
                         float* mc) {
    if (!plan) return fail(PENCIL_E_ARG, "null plan");
    if (npeers < 0 || npeers > PENCIL_MAX_PEERS || (npeers > 0 && !peers))
        return fail(PENCIL_E_ARG, "npeers must be 0..%d", PENCIL_MAX_PEERS);
    PeerSet ps = {};
    for (int q = 0; q < npeers; q++) {
        if (!peers[q]) return fail(PENCIL_E_ARG, "null peer pointer %d", q);
        ps.p[q] = peers[q];
    }
    ps.n = npeers;
    ps.mc = mc;
    DEV_PROLOGUE;
    unsigned *tk = ticket_word(c, st), *fw = fault_word(c, st);
    if (!tk || !fw) return g_status;
    if (cudaError_t z = zero_empty_rows(*plan, y, st)) return cuda_fail(z, "zero empty rows");
    DEV_RET(launch_csr_spmv_dist(st, plan->mode, plan->nrows, plan->ncols, plan->nnz, rowptr, col, val, x, y,
                                 plan->tile_row, plan->ntiles, plan->flags, plan->seg_plan(), tk, fw, ps));
}

int pencil_sync_status(pencil_stream_t s) {
    DEV_PROLOGUE;
    return collect_faults(c, st) == PENCIL_OK ? ok() : g_status;
}

const char* pencil_version(void) { return "pencil-b200 0.1 (sm_100a)"; }

int pencil_l2_flush(pencil_stream_t s) {
    DEV_PROLOGUE;
    if (!c->l2_flush) {
        c->l2_flush_elems = 64ll << 20;  // 256 MiB > 126 MB L2
        CK(cudaMalloc(&c->l2_flush, sizeof(float) * c->l2_flush_elems));
    }
    DEV_RET(launch_micro_l2_flush(st, c->l2_flush_elems, c->l2_flush));
}

int pencil_micro_gather(pencil_stream_t s, int mode, long long n, const int* idx, const float* table,
                        float* out) {
    DEV_PROLOGUE;
    DEV_RET(launch_micro_gather(st, mode, n, idx, table, out));
}

int pencil_micro_gather_val(pencil_stream_t s, long long n, const int* idx, const float* val,
                            const float* table, float* out) {
    DEV_PROLOGUE;
    DEV_RET(launch_micro_gather_val(st, n, idx, val, table, out));
}

int pencil_micro_copy(pencil_stream_t s, long long n, const float* src, float* dst) {
    DEV_PROLOGUE;
    DEV_RET(launch_micro_copy(st, n, src, dst));
}

}  // extern "C"

extern "C" int pencil_last_transfer_bytes(long long* h2d, long long* d2h) {
    if (h2d) *h2d = g_h2d;
    if (d2h) *d2h = g_d2h;
    return PENCIL_OK;
}

// status setters for the dispatch and OP2 layers (dispatch.cpp, op2.cpp), C++ linkage, not part of the ABI
int pencil_internal_fail(int status, const char* msg) {
    g_status = status;
    snprintf(g_msg, sizeof g_msg, "%s", msg);
    return status;
}
int pencil_internal_ok() { return ok(); }
// the CSR executor with the mapper's reduction choice (dispatch.cpp): mode 1 = row sums
// reassociated (the inner loop mapped to a REDUCE role), 0 = source order (SEQ role)
int pencil_internal_spmv(int mode, int nrows, int ncols, int nnz, int* rowptr, int* col, float* val, float* x,
                         float* y) {
    return spmv_common(mode, nrows, ncols, nnz, rowptr, col, val, x, y);
}
