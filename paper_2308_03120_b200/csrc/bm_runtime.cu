// bm_runtime.cu -- lifecycle, memory, transfers, queue entry points and
// instrumentation of libb200mat.so (the C ABI in include/b200mat.h).
//
// The reference's runtime (reference/pkg/src/devmat/runtime.py) keeps a FIFO
// command queue drained by a dispatcher thread (runtime.py:310-360); the CUDA
// stream is that queue here.  release_deferred (runtime.py:449-451) is
// cudaFreeAsync on the same stream, so a buffer is recycled only after every
// kernel queued before the release has finished.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "bm_internal.h"

namespace bmi {

State& st() {
    static State s;
    return s;
}

static thread_local std::string g_last_error;

int set_error(int code, const std::string& msg) {
    g_last_error = msg;
    return code;
}

int cuda_fail(cudaError_t e, const char* what) {
    std::string m = std::string(what) + ": " + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) + ")";
    if (e == cudaErrorNoDevice || e == cudaErrorInsufficientDriver) return set_error(BM_ERR_NODEVICE, m);
    return set_error(BM_ERR_CUDA, m);
}

int check_device_error(const char* what) {
    State& s = st();
    if (!s.err_host) return BM_OK;
    const unsigned int w = __atomic_exchange_n(s.err_host, 0u, __ATOMIC_ACQ_REL);
    if (!w) return BM_OK;
    std::string m = std::string(what) + ": ";
    if (w & 1u)
        m += "a peer rank did not publish its partial within the exchange timeout (BM_EXCH_TIMEOUT_S); "
             "the sharded result is invalid and the exchange must be re-created";
    else
        m += "device error word set";
    return set_error(BM_ERR_PEER, m);
}

int cu_fail(CUresult r, const char* what) {
    char buf[160];
    std::snprintf(buf, sizeof buf, "%s: CUresult %d", what, (int)r);
    return set_error(BM_ERR_CUDA, buf);
}

Driver& drv() {
    static Driver d;
    return d;
}

int load_driver() {
    Driver& d = drv();
    if (d.ok) return BM_OK;
    cudaDriverEntryPointQueryResult q;
#define BM_GET(sym, field)                                                                   \
    do {                                                                                     \
        void* p = nullptr;                                                                   \
        cudaError_t e = cudaGetDriverEntryPoint(#sym, &p, cudaEnableDefault, &q);            \
        if (e != cudaSuccess || q != cudaDriverEntryPointSuccess || !p)                      \
            return set_error(BM_ERR_CUDA, "cannot resolve driver entry point " #sym);        \
        d.field = reinterpret_cast<decltype(d.field)>(p);                                    \
    } while (0)
    BM_GET(cuModuleLoadData, moduleLoadData);
    BM_GET(cuModuleGetFunction, moduleGetFunction);
    BM_GET(cuLaunchKernel, launchKernel);
    BM_GET(cuLaunchKernelEx, launchKernelEx);
    BM_GET(cuOccupancyMaxActiveClusters, occupancyMaxActiveClusters);
    BM_GET(cuFuncSetAttribute, funcSetAttribute);
    BM_GET(cuFuncGetAttribute, funcGetAttribute);
    BM_GET(cuTensorMapEncodeTiled, tensorMapEncodeTiled);
#undef BM_GET
    d.ok = true;
    return BM_OK;
}

}  // namespace bmi

using namespace bmi;

extern "C" {

int bm_abi_version(void) { return BM_ABI_VERSION; }

const char* bm_last_error(void) { return g_last_error.c_str(); }

int bm_device_count(int* count) {
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess) {
        *count = 0;
        (void)cudaGetLastError();
        return cuda_fail(e, "cudaGetDeviceCount");
    }
    *count = n;
    return BM_OK;
}

int bm_init(int device) {
    State& s = st();
    std::lock_guard<std::recursive_mutex> lk(s.mu);
    if (s.initialised) return set_error(BM_ERR_ARG, "bm_init: already initialised");
    BM_CUDA(cudaSetDevice(device));
    BM_CUDA(cudaFree(nullptr));  // create the primary context
    cudaDeviceProp p;
    BM_CUDA(cudaGetDeviceProperties(&p, device));
    if (p.major < 10) return set_error(BM_ERR_NODEVICE, std::string("bm_init: device is not sm_100-class: ") + p.name);
    int rc = load_driver();
    if (rc) return rc;
    s.device = device;
    s.sm_count = p.multiProcessorCount;
    BM_CUDA(cudaStreamCreateWithFlags(&s.own_stream, cudaStreamNonBlocking));
    s.stream = s.own_stream;
    // keep freed blocks in the pool: allocation churn of temporaries is the
    // common case (expr.py:781-787 releases after last use)
    cudaMemPool_t pool;
    BM_CUDA(cudaDeviceGetDefaultMemPool(&pool, device));
    uint64_t thr = UINT64_MAX;
    BM_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
    BM_CUDA(cudaMalloc(&s.partials[0], 8 * 8192));
    BM_CUDA(cudaMalloc(&s.partials[1], 8 * 8192));
    s.partials_cap = 8192;
    s.flip = 0;
    BM_CUDA(cudaMalloc(&s.ticket, 256));
    BM_CUDA(cudaMemset(s.ticket, 0, 256));
    BM_CUDA(cudaMalloc(&s.result, 256));
    BM_CUDA(cudaMalloc(&s.fold_scratch, 8 * 8192));
    BM_CUDA(cudaMallocHost(&s.host_slot, 256));
    BM_CUDA(cudaHostAlloc((void**)&s.err_host, 64, cudaHostAllocMapped));
    *s.err_host = 0u;
    BM_CUDA(cudaHostGetDevicePointer((void**)&s.err_dev, s.err_host, 0));
    if (const char* t = std::getenv("BM_EXCH_TIMEOUT_S")) {
        const double sec = std::atof(t);
        if (sec > 0) s.exch_timeout_ns = (unsigned long long)(sec * 1e9);
    }
    BM_CUDA(cudaDeviceSynchronize());
    s.initialised = true;
    return BM_OK;
}

int bm_shutdown(void) {
    State& s = st();
    std::lock_guard<std::recursive_mutex> lk(s.mu);
    if (!s.initialised) return BM_OK;
    cudaError_t e = cudaDeviceSynchronize();
    cudaFree(s.partials[0]);
    cudaFree(s.partials[1]);
    cudaFree(s.ticket);
    cudaFree(s.result);
    cudaFree(s.fold_scratch);
    s.fold_scratch = nullptr;
    cudaFree(s.lg_scratch);
    s.lg_scratch = nullptr;
    s.lg_scratch_cap = 0;
    cudaFreeHost(s.host_slot);
    cudaFreeHost(s.err_host);
    s.err_host = s.err_dev = nullptr;
    cudaStreamDestroy(s.own_stream);
    s.partials[0] = s.partials[1] = s.result = s.host_slot = nullptr;
    s.partials_cap = 0;
    s.ticket = nullptr;
    s.own_stream = s.stream = nullptr;
    s.initialised = false;
    if (e != cudaSuccess) return cuda_fail(e, "bm_shutdown");
    return BM_OK;
}

int bm_device_info(char* name, int name_len, int* sm_count, int* cc_major, int* cc_minor, int64_t* total_mem) {
    BM_REQUIRE_INIT();
    cudaDeviceProp p;
    BM_CUDA(cudaGetDeviceProperties(&p, st().device));
    if (name && name_len > 0) {
        std::strncpy(name, p.name, name_len - 1);
        name[name_len - 1] = 0;
    }
    if (sm_count) *sm_count = p.multiProcessorCount;
    if (cc_major) *cc_major = p.major;
    if (cc_minor) *cc_minor = p.minor;
    if (total_mem) *total_mem = (int64_t)p.totalGlobalMem;
    return BM_OK;
}

int bm_set_stream(void* cuda_stream) {
    BM_REQUIRE_INIT();
    State& s = st();
    std::lock_guard<std::recursive_mutex> lk(s.mu);
    s.stream = cuda_stream ? (cudaStream_t)cuda_stream : s.own_stream;
    return BM_OK;
}

void* bm_get_stream(void) { return (void*)st().stream; }

int bm_alloc(int64_t bytes, void** out) {
    BM_REQUIRE_INIT();
    if (bytes < 0) return set_error(BM_ERR_ARG, "bm_alloc: negative size");
    std::lock_guard<std::recursive_mutex> lk(st().mu);
    // zero-length buffers still get a distinct handle (reference keeps them live)
    BM_CUDA(cudaMallocAsync(out, bytes > 0 ? (size_t)bytes : 16, st().stream));
    return BM_OK;
}

int bm_free_async(void* p) {
    BM_REQUIRE_INIT();
    if (!p) return BM_OK;
    std::lock_guard<std::recursive_mutex> lk(st().mu);
    BM_CUDA(cudaFreeAsync(p, st().stream));
    return BM_OK;
}

int bm_free(void* p) { return bm_free_async(p); }

int bm_sync(void) {
    BM_REQUIRE_INIT();
    cudaError_t e = cudaStreamSynchronize(st().stream);
    if (e != cudaSuccess) return cuda_fail(e, "bm_sync (asynchronous kernel failure)");
    return check_device_error("bm_sync");
}

int bm_stream_busy(void) {
    if (!st().initialised) return 0;
    const cudaError_t e = cudaStreamQuery(st().stream);
    if (e == cudaErrorNotReady) return 1;
    return 0;   // idle, or a sticky error that the next bm_sync reports
}

int bm_poll_device_error(void) {
    BM_REQUIRE_INIT();
    return check_device_error("device error");
}

static int copy_sync(void* dst, const void* src, int64_t bytes, cudaMemcpyKind k) {
    BM_REQUIRE_INIT();
    if (bytes <= 0) return BM_OK;
    std::lock_guard<std::recursive_mutex> lk(st().mu);
    // a scalar read (sum cache, element reads) goes through the pinned 64-B slot: a
    // pageable copy is staged by the driver and costs several microseconds more
    const bool small_d2h = k == cudaMemcpyDeviceToHost && bytes <= 64;
    BM_CUDA(cudaMemcpyAsync(small_d2h ? st().host_slot : dst, src, (size_t)bytes, k, st().stream));
    cudaError_t e = cudaStreamSynchronize(st().stream);
    if (e != cudaSuccess) return cuda_fail(e, "copy");
    if (small_d2h) std::memcpy(dst, st().host_slot, (size_t)bytes);
    return check_device_error("copy");
}

int bm_h2d(void* dst, const void* src, int64_t bytes) {
    int rc = copy_sync(dst, src, bytes, cudaMemcpyHostToDevice);
    if (!rc && bytes > 0) st().bytes_h2d += bytes;
    return rc;
}

int bm_d2h(void* dst, const void* src, int64_t bytes) {
    int rc = copy_sync(dst, src, bytes, cudaMemcpyDeviceToHost);
    if (!rc && bytes > 0) st().bytes_d2h += bytes;
    return rc;
}

int bm_d2d(void* dst, const void* src, int64_t bytes) {
    BM_REQUIRE_INIT();
    if (bytes <= 0) return BM_OK;
    std::lock_guard<std::recursive_mutex> lk(st().mu);
    BM_CUDA(cudaMemcpyAsync(dst, src, (size_t)bytes, cudaMemcpyDeviceToDevice, st().stream));
    return BM_OK;
}

int bm_h2d_async(void* dst, const void* src, int64_t bytes) {
    BM_REQUIRE_INIT();
    if (bytes <= 0) return BM_OK;
    std::lock_guard<std::recursive_mutex> lk(st().mu);
    BM_CUDA(cudaMemcpyAsync(dst, src, (size_t)bytes, cudaMemcpyHostToDevice, st().stream));
    st().bytes_h2d += bytes;
    return BM_OK;
}

int bm_d2h_async(void* dst, const void* src, int64_t bytes) {
    BM_REQUIRE_INIT();
    if (bytes <= 0) return BM_OK;
    std::lock_guard<std::recursive_mutex> lk(st().mu);
    BM_CUDA(cudaMemcpyAsync(dst, src, (size_t)bytes, cudaMemcpyDeviceToHost, st().stream));
    st().bytes_d2h += bytes;
    return BM_OK;
}

int bm_host_alloc_pinned(int64_t bytes, void** out) {
    BM_CUDA(cudaMallocHost(out, bytes > 0 ? (size_t)bytes : 16));
    return BM_OK;
}

int bm_host_free_pinned(void* p) {
    BM_CUDA(cudaFreeHost(p));
    return BM_OK;
}

int bm_read_elems(const void* base, int32_t dtype, const int64_t* idx, int64_t n, void* host_out) {
    BM_REQUIRE_INIT();
    if (!dtype_ok(dtype)) return set_error(BM_ERR_ARG, "bm_read_elems: bad dtype");
    const int64_t sz = dtype_size(dtype);
    std::lock_guard<std::recursive_mutex> lk(st().mu);
    for (int64_t i = 0; i < n; ++i)
        BM_CUDA(cudaMemcpyAsync((char*)host_out + i * sz, (const char*)base + idx[i] * sz, (size_t)sz,
                                cudaMemcpyDeviceToHost, st().stream));
    cudaError_t e = cudaStreamSynchronize(st().stream);
    if (e != cudaSuccess) return cuda_fail(e, "bm_read_elems");
    st().bytes_d2h += n * sz;
    return BM_OK;
}

int bm_write_elem(void* base, int32_t dtype, int64_t index, const void* host_value) {
    BM_REQUIRE_INIT();
    if (!dtype_ok(dtype)) return set_error(BM_ERR_ARG, "bm_write_elem: bad dtype");
    const int64_t sz = dtype_size(dtype);
    return bm_h2d((char*)base + index * sz, host_value, sz);
}

int bm_get_counters(bm_counters* out) {
    State& s = st();
    out->launches = s.launches.load();
    out->jit_compiles = s.jit_compiles.load();
    out->jit_cache_hits = s.jit_hits.load();
    out->bytes_h2d = s.bytes_h2d.load();
    out->bytes_d2h = s.bytes_d2h.load();
    return BM_OK;
}

int bm_set_gemm_algo(int32_t algo) {
    st().gemm_algo = algo;
    return BM_OK;
}

// ---- queue --------------------------------------------------------------------------

static int check_view(const bm_view& v, const char* what) {
    if (!dtype_ok(v.dtype)) return set_error(BM_ERR_ARG, std::string(what) + ": bad dtype");
    if (!v.base) return set_error(BM_ERR_ARG, std::string(what) + ": null buffer");
    return BM_OK;
}

int bm_enqueue(const bm_invocation* inv) {
    BM_REQUIRE_INIT();
    if (!inv) return set_error(BM_ERR_ARG, "bm_enqueue: null invocation");
    if (inv->n_inputs < 0 || inv->n_inputs > BM_MAX_INPUTS) return set_error(BM_ERR_ARG, "bm_enqueue: bad input count");
    for (int i = 0; i < inv->n_inputs; ++i) {
        int rc = check_view(inv->inputs[i], "input");
        if (rc) return rc;
    }
    if (inv->has_output) {
        int rc = check_view(inv->output, "output");
        if (rc) return rc;
    }
    std::lock_guard<std::recursive_mutex> lk(st().mu);
    switch (inv->kind) {
        case BM_K_EWISE:
        case BM_K_REDUCE:
            return launch_ewise_or_reduce(inv, false, nullptr);
        case BM_K_RDIM:
            return launch_rdim(inv);
        case BM_K_GEMM:
            return launch_gemm(inv);
        case BM_K_PRED_FIND:
            return launch_pred_find(inv);
        case BM_K_LOGISTIC_GRAD:
            return launch_logistic_grad(inv);
        case BM_K_GEMM_FUSED:
            return launch_gemm_fused(inv);
        case BM_K_RDIM_FUSED:
            return launch_rdim_fused(inv);
        case BM_K_GEMM_EPI:
            return launch_gemm_epi(inv);
        default:
            return launch_misc(inv);
    }
}

static int reduce_common(const bm_invocation* inv, bool to_device, void* dev_result) {
    BM_REQUIRE_INIT();
    if (!inv || (inv->kind != BM_K_REDUCE && inv->kind != BM_K_PRED_COUNT))
        return set_error(BM_ERR_ARG, "bm_execute_reduce: not a reduction");
    for (int i = 0; i < inv->n_inputs; ++i) {
        int rc = check_view(inv->inputs[i], "input");
        if (rc) return rc;
    }
    if (inv->kind == BM_K_PRED_COUNT) return launch_pred_count(inv, to_device ? dev_result : st().result);
    return launch_ewise_or_reduce(inv, to_device, dev_result);
}

int bm_execute_reduce(const bm_invocation* inv, void* host_result) {
    State& s = st();
    std::lock_guard<std::recursive_mutex> lk(s.mu);
    int rc = reduce_common(inv, false, nullptr);
    if (rc) return rc;
    BM_CUDA(cudaMemcpyAsync(s.host_slot, s.result, 8, cudaMemcpyDeviceToHost, s.stream));
    cudaError_t e = cudaStreamSynchronize(s.stream);
    if (e != cudaSuccess) return cuda_fail(e, "bm_execute_reduce");
    if (int erc = check_device_error("bm_execute_reduce")) return erc;
    const int rdt = inv->compute_dtype;
    if (inv->reduce_op == BM_R_DOT && rdt == BM_F32) {
        // f32 dot partials are accumulated in f64; round once, like numpy's
        // float32 result of the reference's sdot blocks (kernels.py:471-472)
        double d;
        std::memcpy(&d, s.host_slot, 8);
        const float f = (float)d;
        std::memcpy(host_result, &f, 4);
    } else {
        std::memcpy(host_result, s.host_slot, (size_t)dtype_size(rdt));
    }
    s.bytes_d2h += dtype_size(rdt);
    return BM_OK;
}

int bm_reduce_to_device(const bm_invocation* inv, void* dev_result) {
    std::lock_guard<std::recursive_mutex> lk(st().mu);
    return reduce_common(inv, true, dev_result);
}

int bm_combine_partials(const void* dev_partials, int64_t count, int32_t dtype, int32_t reduce_op, void* host_result) {
    BM_REQUIRE_INIT();
    State& s = st();
    std::lock_guard<std::recursive_mutex> lk(s.mu);
    int rc = combine_partials(dev_partials, count, dtype, reduce_op, s.result);
    if (rc) return rc;
    const int64_t sz = (reduce_op == BM_R_DOT && (dtype == BM_F32 || dtype == BM_F64)) ? 8 : dtype_size(dtype);
    BM_CUDA(cudaMemcpyAsync(s.host_slot, s.result, 8, cudaMemcpyDeviceToHost, s.stream));
    cudaError_t e = cudaStreamSynchronize(s.stream);
    if (e != cudaSuccess) return cuda_fail(e, "bm_combine_partials");
    std::memcpy(host_result, s.host_slot, (size_t)sz);
    return BM_OK;
}

int bm_reduce_to_device_exchange(const bm_invocation* inv, void* dev_result, void* const* dev_peer_array,
                                 int32_t world, int32_t rank, uint64_t epoch) {
    State& s = st();
    std::lock_guard<std::recursive_mutex> lk(s.mu);
    if (world < 2 || world > 64 || rank < 0 || rank >= world || epoch == 0 || !dev_peer_array)
        return set_error(BM_ERR_ARG, "fused exchange: bad world / rank / epoch");
    s.exch_peers = dev_peer_array;
    s.exch_world = world;
    s.exch_rank = rank;
    s.exch_epoch = epoch;
    const int rc = reduce_common(inv, true, dev_result);
    s.exch_world = 0;
    s.exch_peers = nullptr;
    return rc;
}

int bm_combine_partials_to_device(const void* dev_partials, int64_t count, int32_t dtype, int32_t reduce_op,
                                  void* dev_result) {
    BM_REQUIRE_INIT();
    std::lock_guard<std::recursive_mutex> lk(st().mu);
    return combine_partials(dev_partials, count, dtype, reduce_op, dev_result);
}

int bm_gemm(int32_t dtype, int32_t trans_a, int32_t trans_b, int64_t m, int64_t n, int64_t k, const void* a,
            int64_t lda, const void* b, int64_t ldb, void* c, int64_t ldc) {
    BM_REQUIRE_INIT();
    bm_invocation inv;
    std::memset(&inv, 0, sizeof inv);
    inv.kind = BM_K_GEMM;
    inv.n_inputs = 2;
    inv.trans_a = trans_a;
    inv.trans_b = trans_b;
    const int64_t ar = trans_a ? k : m, ac = trans_a ? m : k;
    const int64_t br = trans_b ? n : k, bc = trans_b ? k : n;
    inv.inputs[0] = bm_view{const_cast<void*>(a), 0, ar * ac, 1, ar, ac, lda, dtype, 1};
    inv.inputs[1] = bm_view{const_cast<void*>(b), 0, br * bc, 1, br, bc, ldb, dtype, 1};
    inv.has_output = 1;
    inv.output = bm_view{c, 0, m * n, 1, m, n, ldc, dtype, 1};
    inv.compute_dtype = dtype;
    std::lock_guard<std::recursive_mutex> lk(st().mu);
    return launch_gemm(&inv);
}

}  // extern "C"
