// bm_pred.cu -- element-vs-scalar predicates: count, all/any and find
// (reference: ops.py:202-262 find/all/any over kernels.py:643-699
// _predicate_mask / _run_count / _run_all_any / _run_find_build).
//
// The threshold is compared in the element type after the host has cast it
// like _scalar(k, dtype) (np.float32(k) / int(k)), so NaN compares false
// except for "!=", exactly numpy's ufuncs.  Counts are integers, so the
// block counts combine with integer atomics and are still exact and
// deterministic.  find writes the ascending column-major linear indices as
// u64 (np.nonzero order) in three stream-ordered steps: per-chunk counts, an
// exclusive scan of the chunk counts, then every chunk writes its indices at
// its offset (warp ballots + popc prefixes, so each chunk's output is in
// ascending order without sorting).
#include <cstring>

#include "bm_internal.h"
#include "bm_reduce.cuh"

namespace bm {

#define PRED_CHUNK 4096           // elements per CTA in find (256 threads x 16)

template <typename T>
__device__ __forceinline__ bool pred_eval(T x, int op, T k) {
    switch (op) {
        case BM_CMP_GT: return x > k;
        case BM_CMP_LT: return x < k;
        case BM_CMP_GE: return x >= k;
        case BM_CMP_LE: return x <= k;
        case BM_CMP_EQ: return x == k;
        default: return x != k;
    }
}

// count of matches over n strided elements, accumulated into *count (u64)
template <typename T>
__global__ void __launch_bounds__(256) pred_count_kernel(const T* __restrict__ x, i64 n, i64 stride, int op, T k,
                                                         unsigned long long* count) {
    unsigned c = 0;
    const i64 tid = (i64)blockIdx.x * blockDim.x + threadIdx.x, nt = (i64)gridDim.x * blockDim.x;
    if (stride == 1) {
        for (i64 i = tid; i < n; i += nt) c += pred_eval(__ldg(x + i), op, k) ? 1u : 0u;
    } else {
        for (i64 i = tid; i < n; i += nt) c += pred_eval(x[i * stride], op, k) ? 1u : 0u;
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    __shared__ unsigned ws[8];
    if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = c;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long s = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += ws[w];
        if (s) atomicAdd(count, s);
    }
}

// per-chunk match counts
template <typename T>
__global__ void __launch_bounds__(256) pred_chunk_count_kernel(const T* __restrict__ x, i64 n, i64 stride, int op, T k,
                                                               unsigned* __restrict__ chunk_count) {
    const i64 base = (i64)blockIdx.x * PRED_CHUNK;
    unsigned c = 0;
#pragma unroll 4
    for (int j = 0; j < PRED_CHUNK / 256; ++j) {
        const i64 i = base + j * 256 + threadIdx.x;
        if (i < n) c += pred_eval(x[i * stride], op, k) ? 1u : 0u;
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    __shared__ unsigned ws[8];
    if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = c;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned s = 0;
        for (int w = 0; w < 8; ++w) s += ws[w];
        chunk_count[blockIdx.x] = s;
    }
}

// exclusive scan of the chunk counts (one CTA of 1024 threads; each thread
// scans a contiguous run, the run totals are scanned in shared memory)
__global__ void __launch_bounds__(1024) pred_scan_kernel(const unsigned* __restrict__ cnt, i64 nchunks,
                                                         unsigned long long* __restrict__ off) {
    __shared__ unsigned long long tot[1024];
    const i64 per = (nchunks + 1023) / 1024;
    const i64 lo = (i64)threadIdx.x * per, hi = (lo + per < nchunks) ? lo + per : nchunks;
    unsigned long long s = 0;
    for (i64 i = lo; i < hi; ++i) s += cnt[i];
    tot[threadIdx.x] = s;
    __syncthreads();
    // Hillis-Steele inclusive scan over the 1024 run totals
    for (int d = 1; d < 1024; d <<= 1) {
        const unsigned long long v = threadIdx.x >= (unsigned)d ? tot[threadIdx.x - d] : 0ull;
        __syncthreads();
        tot[threadIdx.x] += v;
        __syncthreads();
    }
    unsigned long long run = threadIdx.x ? tot[threadIdx.x - 1] : 0ull;
    for (i64 i = lo; i < hi; ++i) {
        off[i] = run;
        run += cnt[i];
    }
}

// every chunk writes its matching indices, ascending, at its offset
template <typename T>
__global__ void __launch_bounds__(256) pred_find_kernel(const T* __restrict__ x, i64 n, i64 stride, int op, T k,
                                                        const unsigned long long* __restrict__ off,
                                                        unsigned long long* __restrict__ out) {
    __shared__ unsigned wcount[8];
    __shared__ unsigned long long run_base;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) run_base = off[blockIdx.x];
    __syncthreads();
    const i64 base = (i64)blockIdx.x * PRED_CHUNK;
    for (int j = 0; j < PRED_CHUNK / 256; ++j) {
        // 256 consecutive elements per step: warp w covers [w*32, w*32+32)
        const i64 i = base + j * 256 + threadIdx.x;
        const bool hit = i < n && pred_eval(x[i * stride], op, k);
        const unsigned ball = __ballot_sync(0xffffffffu, hit);
        if (lane == 0) wcount[warp] = __popc(ball);
        __syncthreads();
        unsigned before = 0, total = 0;
        for (int w = 0; w < 8; ++w) {
            const unsigned c = wcount[w];
            if (w < warp) before += c;
            total += c;
        }
        if (hit) out[run_base + before + __popc(ball & ((1u << lane) - 1u))] = (unsigned long long)i;
        __syncthreads();
        if (threadIdx.x == 0) run_base += total;
        __syncthreads();
    }
}

}  // namespace bm

namespace bmi {

template <typename F>
static int pred_typed(int dtype, F&& f) {
    switch (dtype) {
        case BM_F32: return f(float(0));
        case BM_F64: return f(double(0));
        case BM_I32: return f(int(0));
        case BM_U64: return f((unsigned long long)0);
    }
    return set_error(BM_ERR_ARG, "predicate: bad dtype");
}

template <typename T>
static T pred_threshold(const bm_invocation* inv) {
    if (std::is_floating_point<T>::value) return (T)inv->fscalars[0];
    return (T)inv->iscalars[0];
}

static const char* pred_ptr(const bm_view& v) {
    return (const char*)v.base + v.offset * dtype_size(v.dtype);
}

// BM_K_PRED_COUNT / BM_K_PRED_ALL_ANY: number of matches as u64 into dev_result
// (all = count == n, any = count > 0 on the host, like _combine_all/_any)
int launch_pred_count(const bm_invocation* inv, void* dev_result) {
    if (inv->n_inputs != 1) return set_error(BM_ERR_ARG, "predicate: needs one input");
    const bm_view& v = inv->inputs[0];
    const int64_t n = v.count;
    const int op = (int)inv->iparams[0];
    if (op < BM_CMP_GT || op > BM_CMP_NE) return set_error(BM_ERR_ARG, "predicate: bad comparison");
    BM_CUDA(cudaMemsetAsync(dev_result, 0, 8, st().stream));
    if (n == 0) return BM_OK;
    return pred_typed(v.dtype, [&](auto t) {
        typedef decltype(t) T;
        int64_t blocks = (n + 255) / 256;
        const int64_t cap = (int64_t)st().sm_count * 8;
        if (blocks > cap) blocks = cap;
        bm::pred_count_kernel<T><<<(unsigned)blocks, 256, 0, st().stream>>>(
            (const T*)pred_ptr(v), n, v.stride, op, pred_threshold<T>(inv), (unsigned long long*)dev_result);
        BM_CUDA(cudaGetLastError());
        st().launches++;
        return BM_OK;
    });
}

// BM_K_PRED_FIND: ascending linear indices of the matches into the u64 output
// (whose count is the match count the caller obtained first, ops.py:221-228)
int launch_pred_find(const bm_invocation* inv) {
    if (inv->n_inputs != 1 || !inv->has_output) return set_error(BM_ERR_ARG, "find: needs one input and an output");
    const bm_view& v = inv->inputs[0];
    const bm_view& o = inv->output;
    if (o.dtype != BM_U64 || o.stride != 1) return set_error(BM_ERR_ARG, "find: output must be a contiguous u64 view");
    const int64_t n = v.count;
    const int op = (int)inv->iparams[0];
    if (op < BM_CMP_GT || op > BM_CMP_NE) return set_error(BM_ERR_ARG, "predicate: bad comparison");
    if (n == 0 || o.count == 0) return BM_OK;
    const int64_t nchunks = (n + PRED_CHUNK - 1) / PRED_CHUNK;
    if (nchunks > 0x7fffffff) return set_error(BM_ERR_NOTIMPL, "find: input too large");
    cudaStream_t s = st().stream;
    unsigned* cnt = nullptr;
    unsigned long long* off = nullptr;
    BM_CUDA(cudaMallocAsync((void**)&cnt, (size_t)nchunks * 4, s));
    BM_CUDA(cudaMallocAsync((void**)&off, (size_t)nchunks * 8, s));
    int rc = pred_typed(v.dtype, [&](auto t) {
        typedef decltype(t) T;
        const T* x = (const T*)pred_ptr(v);
        const T k = pred_threshold<T>(inv);
        bm::pred_chunk_count_kernel<T><<<(unsigned)nchunks, 256, 0, s>>>(x, n, v.stride, op, k, cnt);
        bm::pred_scan_kernel<<<1, 1024, 0, s>>>(cnt, nchunks, off);
        bm::pred_find_kernel<T><<<(unsigned)nchunks, 256, 0, s>>>(
            x, n, v.stride, op, k, off, (unsigned long long*)((char*)o.base + o.offset * 8));
        BM_CUDA(cudaGetLastError());
        st().launches += 3;
        return BM_OK;
    });
    cudaFreeAsync(cnt, s);
    cudaFreeAsync(off, s);
    return rc;
}

}  // namespace bmi
