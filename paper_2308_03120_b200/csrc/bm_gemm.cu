// bm_gemm.cu -- glue_times (reference kernels.py:704-708, lowered at
// expr.py:596-605): C = op(A) * op(B), column-major, transposes folded into
// the operand addressing so `A @ B.t()` needs no mov_transpose pass.
//
// Dispatch:
//   f32  -> 3xTF32 on tcgen05 (bm_gemm_tc.cu) when the shape is tile-aligned
//   f64  -> DMMA (mma.sync m8n8k4 f64) (bm_gemm_tc.cu)
//   i32 / u64 and ragged shapes -> the SIMT kernel below (exact integer
//   arithmetic, wrapping like numpy's integer np.dot).
#include <cstring>

#include "bm_internal.h"
#include "bm_reduce.cuh"

namespace bm {

// Multiply-accumulate of the SIMT GEMM.  Floats: one fused multiply-add per
// k, in k order from zero -- the accumulation of the reference's OpenBLAS
// sgemm/dgemm micro-kernels for the small shapes this kernel serves, so the
// products match np.dot (kernels.py:704-708) bit for bit when K fits one
// OpenBLAS K-block.  Integers wrap like numpy's integer np.dot.
__device__ __forceinline__ float mac(float a, float b, float c) { return __fmaf_rn(a, b, c); }
__device__ __forceinline__ double mac(double a, double b, double c) { return __fma_rn(a, b, c); }
template <typename T>
__device__ __forceinline__ T mac(T a, T b, T c) { return OpPlus::f(c, OpTimes::f(a, b)); }

// 64x64 output tile per CTA, 256 threads x (4x4) outputs, K staged 16 at a time.
template <typename T>
__global__ void __launch_bounds__(256) gemm_simt_kernel(int ta, int tb, i64 m, i64 n, i64 k, const T* __restrict__ A,
                                                        i64 lda, const T* __restrict__ B, i64 ldb, T* __restrict__ C,
                                                        i64 ldc) {
    __shared__ T As[16][64 + 1];
    __shared__ T Bs[16][64 + 1];
    const i64 m0 = (i64)blockIdx.x * 64, n0 = (i64)blockIdx.y * 64;
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    T acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = T(0);
    for (i64 k0 = 0; k0 < k; k0 += 16) {
        for (int idx = threadIdx.x; idx < 16 * 64; idx += 256) {
            const int kk = idx / 64, mm = idx % 64;
            const i64 gi = m0 + mm, gl = k0 + kk;
            T va = T(0);
            if (gi < m && gl < k) va = ta ? A[gl + gi * lda] : A[gi + gl * lda];
            As[kk][mm] = va;
            const i64 gj = n0 + mm;
            T vb = T(0);
            if (gj < n && gl < k) vb = tb ? B[gj + gl * ldb] : B[gl + gj * ldb];
            Bs[kk][mm] = vb;
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < 16; ++kk) {
            T a[4], b[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) a[i] = As[kk][tx + 16 * i];
#pragma unroll
            for (int j = 0; j < 4; ++j) b[j] = Bs[kk][ty + 16 * j];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = mac(a[i], b[j], acc[i][j]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const i64 gi = m0 + tx + 16 * i, gj = n0 + ty + 16 * j;
            if (gi < m && gj < n) C[gi + gj * ldc] = acc[i][j];
        }
}

// ---------------------------------------------------------------------------
// matrix-vector products (the two GEMMs of the logistic step, SURVEY 8d
// config 5, are X*w and X^T*r): HBM-bound, so no tensor cores; f64
// accumulation for float types, fixed summation order (deterministic).

// y[i] = sum_l A[i + l*lda] x[l]  (A column-major m x k, rows contiguous)
template <typename T>
__global__ void __launch_bounds__(256) gemv_n_kernel(const T* __restrict__ A, i64 lda, const T* __restrict__ x,
                                                     i64 incx, T* __restrict__ y, i64 incy, i64 m, i64 k) {
    typedef typename DotAcc<T>::type Acc;
    const i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= m) return;
    Acc acc = 0;
    i64 l = 0;
    for (; l + 4 <= k; l += 4) {
        const T a0 = A[i + (l + 0) * lda], a1 = A[i + (l + 1) * lda], a2 = A[i + (l + 2) * lda],
                a3 = A[i + (l + 3) * lda];
        acc = OpPlus::f(acc, OpTimes::f((Acc)a0, (Acc)x[(l + 0) * incx]));
        acc = OpPlus::f(acc, OpTimes::f((Acc)a1, (Acc)x[(l + 1) * incx]));
        acc = OpPlus::f(acc, OpTimes::f((Acc)a2, (Acc)x[(l + 2) * incx]));
        acc = OpPlus::f(acc, OpTimes::f((Acc)a3, (Acc)x[(l + 3) * incx]));
    }
    for (; l < k; ++l) acc = OpPlus::f(acc, OpTimes::f((Acc)A[i + l * lda], (Acc)x[l * incx]));
    y[i * incy] = cvt<T>(acc);
}

// partial[s][i] = sum over the s-th K slice of A[l + i*lda] x[l] (columns contiguous)
template <typename T>
__global__ void __launch_bounds__(256) gemv_t_partial_kernel(const T* __restrict__ A, i64 lda,
                                                             const T* __restrict__ x, i64 incx,
                                                             typename DotAcc<T>::type* __restrict__ part, i64 m,
                                                             i64 k, i64 slice) {
    typedef typename DotAcc<T>::type Acc;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const i64 i = (i64)blockIdx.x * (blockDim.x >> 5) + warp;
    if (i >= m) return;
    const i64 l0 = (i64)blockIdx.y * slice;
    i64 l1 = l0 + slice;
    if (l1 > k) l1 = k;
    const T* col = A + i * lda;
    Acc acc = 0;
    for (i64 l = l0 + lane; l < l1; l += 32) acc = OpPlus::f(acc, OpTimes::f((Acc)col[l], (Acc)x[l * incx]));
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) acc = OpPlus::f(acc, warp_shfl_xor(acc, o));
    if (lane == 0) part[(i64)blockIdx.y * m + i] = acc;
}

template <typename T>
__global__ void gemv_t_finish_kernel(const typename DotAcc<T>::type* __restrict__ part, int nsplit, T* __restrict__ y,
                                     i64 incy, i64 m) {
    typedef typename DotAcc<T>::type Acc;
    const i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= m) return;
    Acc acc = 0;
    for (int s = 0; s < nsplit; ++s) acc = OpPlus::f(acc, part[(i64)s * m + i]);
    y[i * incy] = cvt<T>(acc);
}

// --- vectorised GEMVs (16-B loads, several KB in flight per warp) ---------
//
// gemv_n_vec: y = A x with A column-major m x k.  A CTA owns RB = 32*V rows
// (one 16-B vector of V rows per lane) and its 8 warps split the k columns
// into 8 contiguous slices; every lane keeps V f64 accumulators (fma, fixed
// order), the slices are added in warp order through shared memory.  Each
// warp has UNR column vectors (UNR x 512 B) in flight.
template <typename T, int UNR>
__global__ void __launch_bounds__(256) gemv_n_vec_kernel(const T* __restrict__ A, i64 lda, const T* __restrict__ x,
                                                         i64 incx, T* __restrict__ y, i64 incy, i64 m, i64 k) {
    typedef typename DotAcc<T>::type Acc;
    constexpr int V = 16 / sizeof(T);
    constexpr int RB = 32 * V;
    __shared__ Acc red[8][RB];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const i64 row0 = (i64)blockIdx.x * RB + lane * V;
    const i64 per = (k + 7) / 8;
    const i64 l0 = warp * per;
    const i64 l1 = (l0 + per < k) ? l0 + per : k;
    Acc acc[V];
#pragma unroll
    for (int v = 0; v < V; ++v) acc[v] = 0;
    if (row0 + V <= m) {
        i64 l = l0;
        for (; l + UNR <= l1; l += UNR) {
            uint4 q[UNR];
            T xv[UNR];
#pragma unroll
            for (int u = 0; u < UNR; ++u) {
                q[u] = __ldcs(reinterpret_cast<const uint4*>(A + row0 + (l + u) * lda));
                xv[u] = x[(l + u) * incx];
            }
#pragma unroll
            for (int u = 0; u < UNR; ++u) {
                const T* t = reinterpret_cast<const T*>(&q[u]);
#pragma unroll
                for (int v = 0; v < V; ++v) acc[v] = fma((Acc)t[v], (Acc)xv[u], acc[v]);
            }
        }
        for (; l < l1; ++l) {
            const uint4 q = __ldcs(reinterpret_cast<const uint4*>(A + row0 + l * lda));
            const T* t = reinterpret_cast<const T*>(&q);
            const Acc xl = (Acc)x[l * incx];
#pragma unroll
            for (int v = 0; v < V; ++v) acc[v] = fma((Acc)t[v], xl, acc[v]);
        }
    } else {
        for (i64 l = l0; l < l1; ++l) {
            const Acc xl = (Acc)x[l * incx];
#pragma unroll
            for (int v = 0; v < V; ++v)
                if (row0 + v < m) acc[v] = fma((Acc)A[row0 + v + l * lda], xl, acc[v]);
        }
    }
#pragma unroll
    for (int v = 0; v < V; ++v) red[warp][lane * V + v] = acc[v];
    __syncthreads();
    for (int r = threadIdx.x; r < RB; r += blockDim.x) {
        const i64 gi = (i64)blockIdx.x * RB + r;
        if (gi >= m) continue;
        Acc sum = red[0][r];
#pragma unroll
        for (int w = 1; w < 8; ++w) sum = sum + red[w][r];
        y[gi * incy] = cvt<T>(sum);
    }
}

// gemv_t_vec partials: part[s][j] = sum over rows [s*S, (s+1)*S) of
// A[l + j*lda] x[l] (A column-major, column j contiguous).  One warp per
// (column, slice), 16-B loads of both A and x (x stays in L2), UNR vectors
// in flight per lane, f64 fma per lane then a shuffle tree.
template <typename T, int UNR>
__global__ void __launch_bounds__(256) gemv_t_vec_kernel(const T* __restrict__ A, i64 lda, const T* __restrict__ x,
                                                         typename DotAcc<T>::type* __restrict__ part, i64 ncols,
                                                         i64 nrows, i64 S) {
    typedef typename DotAcc<T>::type Acc;
    constexpr int V = 16 / sizeof(T);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const i64 j = (i64)blockIdx.x * 8 + warp;
    if (j >= ncols) return;
    const i64 r0 = (i64)blockIdx.y * S;
    const i64 r1 = (r0 + S < nrows) ? r0 + S : nrows;
    const T* col = A + j * lda;
    Acc acc = 0;
    i64 l = r0 + lane * V;
    constexpr i64 STEP = 32 * V;
    for (; l + (UNR - 1) * STEP + V <= r1; l += UNR * STEP) {
        uint4 qa[UNR], qx[UNR];
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
            qa[u] = __ldcs(reinterpret_cast<const uint4*>(col + l + u * STEP));
            qx[u] = __ldg(reinterpret_cast<const uint4*>(x + l + u * STEP));
        }
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
            const T* ta = reinterpret_cast<const T*>(&qa[u]);
            const T* tx = reinterpret_cast<const T*>(&qx[u]);
#pragma unroll
            for (int v = 0; v < V; ++v) acc = fma((Acc)ta[v], (Acc)tx[v], acc);
        }
    }
    for (; l < r1; l += STEP) {
#pragma unroll
        for (int v = 0; v < V; ++v)
            if (l + v < r1) acc = fma((Acc)col[l + v], (Acc)x[l + v], acc);
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) acc = acc + warp_shfl_xor(acc, o);
    if (lane == 0) part[(i64)blockIdx.y * ncols + j] = acc;
}

// Tail of the fused logistic step (bm_lgrad.cuh), one launch:
//  * CTAs [0, gridDim.x - has_accu): g[c] = the per-cluster gradient partials
//    of column c folded in cluster order -- 8 warps each add a contiguous
//    eighth of the P partials (independent loads in flight, 32 columns
//    coalesced per warp), then the eight sums are added in warp order;
//  * the last CTA (accu_out != 0): accu(r) in the reference's order
//    (kernels.py:459-460 ndarray.sum per 8192-element block, combine_pairwise
//    kernels.py:380-392).  The kernel already left every 128-element numpy
//    leaf of the full blocks in `leaves`; a block value is numpy's balanced
//    tree over its 64 leaves (one warp, operand order kept), the ragged tail
//    block is pw_generic over r, and the blocks fold with combine_pairwise.
// Launched with programmatic dependent launch: griddepcontrol.wait orders it
// after the logistic kernel's writes.
__global__ void __launch_bounds__(256) lgrad_finish_kernel(const double* __restrict__ part, int P, i64 k,
                                                           float* __restrict__ g, const float* __restrict__ leaves,
                                                           const float* __restrict__ r, i64 m,
                                                           float* __restrict__ accu_out) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const bool accu_cta = accu_out != nullptr && blockIdx.x == gridDim.x - 1;
    if (!accu_cta) {
        __shared__ double ps[8][32];
        const i64 c = (i64)blockIdx.x * 32 + lane;
        const int b0 = (int)((i64)P * warp / 8), b1 = (int)((i64)P * (warp + 1) / 8);
        double s = 0.0;
        if (c < k) {
#pragma unroll 4
            for (int b = b0; b < b1; ++b) s += __ldcg(part + (i64)b * k + c);
        }
        ps[warp][lane] = s;
        __syncthreads();
        if (warp == 0 && c < k) {
            double t = ps[0][lane];
#pragma unroll
            for (int w = 1; w < 8; ++w) t += ps[w][lane];
            g[c] = (float)t;
        }
        return;
    }
    __shared__ float bv[LG_ACCU_MAX_BLOCKS];
    __shared__ float scratch[LG_ACCU_MAX_BLOCKS / 256 + 2];
    __shared__ __align__(16) char tile[BM_TILE_BYTES];
    const i64 nfull = m / BM_REDUCE_BLOCK, tail = m - nfull * BM_REDUCE_BLOCK;
    for (i64 b = warp; b < nfull; b += 8) {
        const float* lv = leaves + b * (BM_REDUCE_BLOCK / 128);
        float x = lv[2 * lane] + lv[2 * lane + 1];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const float y = warp_shfl_xor(x, o);
            x = (lane & o) ? y + x : x + y;
        }
        if (lane == 0) bv[b] = x;
    }
    if (tail && warp == 7) {
        const BufSrc<float> src{r, 1};
        const bool vec_ok = ((uintptr_t)(r + nfull * BM_REDUCE_BLOCK) & 15u) == 0;
        const float t = pw_generic<float>(src, nfull * BM_REDUCE_BLOCK, tail, tile, vec_ok);
        if (lane == 0) bv[nfull] = t;
    }
    __syncthreads();
    const float v = cta_fold_pairwise<float, 1>(bv, scratch, (int)(nfull + (tail ? 1 : 0)));
    if (threadIdx.x == 0) accu_out[0] = v + 0.0f;   // numpy: 0 + pairwise(...)
}

}  // namespace bm

namespace bmi {

// y = op(A) x, op(A) m x k; A column-major with leading dim lda.
template <typename T>
static int gemv(bool ta, int64_t m, int64_t k, const T* A, int64_t lda, const T* x, int64_t incx, T* y,
                int64_t incy) {
    typedef typename bm::DotAcc<T>::type Acc;
    cudaStream_t s = st().stream;
    constexpr int V = 16 / sizeof(T);
    const bool a_vec = ((uintptr_t)A % 16 == 0) && (lda % V == 0);
    if (!ta && a_vec && m >= 32 * V) {
        constexpr int RB = 32 * V;
        bm::gemv_n_vec_kernel<T, 8><<<(unsigned)((m + RB - 1) / RB), 256, 0, s>>>(A, lda, x, incx, y, incy, m, k);
        BM_CUDA(cudaGetLastError());
        st().launches++;
        return BM_OK;
    }
    if (ta && a_vec && incx == 1 && (uintptr_t)x % 16 == 0 && k >= 32 * V * 8) {
        // op(A) = A^T: m outputs (columns of A), k rows; slices of S rows
        int64_t S = 16384;
        while (S > 4096 && m * ((k + S - 1) / S) < 4LL * 148 * 8 * 4) S >>= 1;
        const int64_t nsplit = (k + S - 1) / S;
        Acc* part = nullptr;
        BM_CUDA(cudaMallocAsync((void**)&part, (size_t)(nsplit * m) * sizeof(Acc), s));
        dim3 grid((unsigned)((m + 7) / 8), (unsigned)nsplit);
        bm::gemv_t_vec_kernel<T, 4><<<grid, 256, 0, s>>>(A, lda, x, part, m, k, S);
        cudaError_t e = cudaGetLastError();
        if (e == cudaSuccess) {
            bm::gemv_t_finish_kernel<T><<<(unsigned)((m + 255) / 256), 256, 0, s>>>(part, (int)nsplit, y, incy, m);
            e = cudaGetLastError();
        }
        cudaFreeAsync(part, s);
        if (e != cudaSuccess) return cuda_fail(e, "gemv");
        st().launches += 2;
        return BM_OK;
    }
    if (!ta) {
        bm::gemv_n_kernel<T><<<(unsigned)((m + 255) / 256), 256, 0, s>>>(A, lda, x, incx, y, incy, m, k);
        BM_CUDA(cudaGetLastError());
        st().launches++;
        return BM_OK;
    }
    // op(A)(i, l) = A[l + i*lda]: one warp per output, K split for parallelism
    int nsplit = 1;
    while (nsplit < 64 && m * nsplit < 4LL * 148 * 8 * 4 && k / (nsplit * 2) >= 4096) nsplit *= 2;
    const int64_t slice = (k + nsplit - 1) / nsplit;
    Acc* part = nullptr;
    BM_CUDA(cudaMallocAsync((void**)&part, (size_t)(nsplit * m) * sizeof(Acc), s));
    dim3 grid((unsigned)((m + 7) / 8), (unsigned)nsplit);
    bm::gemv_t_partial_kernel<T><<<grid, 256, 0, s>>>(A, lda, x, incx, part, m, k, slice);
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) {
        bm::gemv_t_finish_kernel<T><<<(unsigned)((m + 255) / 256), 256, 0, s>>>(part, nsplit, y, incy, m);
        e = cudaGetLastError();
    }
    cudaFreeAsync(part, s);
    if (e != cudaSuccess) return cuda_fail(e, "gemv");
    st().launches += 2;
    return BM_OK;
}

int gemm_dmma_f64(int ta, int tb, int64_t m, int64_t n, int64_t k, const double* A, int64_t lda, const double* B,
                  int64_t ldb, double* C, int64_t ldc, bool* handled);

template <typename T>
static int gemm_simt(int ta, int tb, int64_t m, int64_t n, int64_t k, const void* A, int64_t lda, const void* B,
                     int64_t ldb, void* C, int64_t ldc) {
    dim3 grid((unsigned)((m + 63) / 64), (unsigned)((n + 63) / 64));
    bm::gemm_simt_kernel<T><<<grid, 256, 0, st().stream>>>(ta, tb, m, n, k, (const T*)A, lda, (const T*)B, ldb, (T*)C,
                                                            ldc);
    BM_CUDA(cudaGetLastError());
    st().launches++;
    return BM_OK;
}

int launch_gemm(const bm_invocation* inv) {
    if (inv->n_inputs != 2 || !inv->has_output) return set_error(BM_ERR_ARG, "gemm: needs two inputs and an output");
    const bm_view &a = inv->inputs[0], &b = inv->inputs[1], &c = inv->output;
    if (a.dtype != b.dtype || a.dtype != c.dtype) return set_error(BM_ERR_ARG, "gemm: operand types differ");
    const int ta = inv->trans_a, tb = inv->trans_b;
    const int64_t m = ta ? a.cols : a.rows, k = ta ? a.rows : a.cols;
    const int64_t kb = tb ? b.cols : b.rows, n = tb ? b.rows : b.cols;
    if (k != kb) return set_error(BM_ERR_ARG, "gemm: inner dimensions differ");
    if (c.rows != m || c.cols != n) return set_error(BM_ERR_ARG, "gemm: output shape mismatch");
    const int64_t sz = dtype_size(a.dtype);
    const char* A = (const char*)a.base + a.offset * sz;
    const char* B = (const char*)b.base + b.offset * sz;
    char* C = (char*)c.base + c.offset * sz;
    if (m == 0 || n == 0) return BM_OK;
    if (k == 0) {
        // inner dimension zero: C = 0 (tests/test_integration.py:98-103)
        if (c.lda == m) {
            BM_CUDA(cudaMemsetAsync(C, 0, (size_t)(m * n * sz), st().stream));
            return BM_OK;
        }
        for (int64_t j = 0; j < n; ++j) BM_CUDA(cudaMemsetAsync(C + j * c.lda * sz, 0, (size_t)(m * sz), st().stream));
        return BM_OK;
    }
    const int algo = st().gemm_algo;
    if (algo != 2 && (a.dtype == BM_F32 || a.dtype == BM_F64) && (n == 1 || m == 1)) {
        // matrix-vector product: C = op(A) x  (n == 1)  or  C^T = op(B)^T a^T  (m == 1)
        if (n == 1) {
            const int64_t incx = tb ? b.lda : 1;
            if (a.dtype == BM_F32)
                return gemv<float>(ta != 0, m, k, (const float*)A, a.lda, (const float*)B, incx, (float*)C, 1);
            return gemv<double>(ta != 0, m, k, (const double*)A, a.lda, (const double*)B, incx, (double*)C, 1);
        }
        // m == 1: C(0, j) = sum_l a(l) op(B)(l, j); op(B)^T is n x k: stored B (k x n) => transposed access
        const int64_t incx = ta ? 1 : a.lda;
        if (a.dtype == BM_F32)
            return gemv<float>(tb == 0, n, k, (const float*)B, b.lda, (const float*)A, incx, (float*)C, c.lda);
        return gemv<double>(tb == 0, n, k, (const double*)B, b.lda, (const double*)A, incx, (double*)C, c.lda);
    }
    switch (a.dtype) {
        case BM_F32: {
            if (algo != 2) {
                bool handled = false;
                int rc = gemm_tc_f32(ta, tb, m, n, k, (const float*)A, a.lda, (const float*)B, b.lda, (float*)C, c.lda,
                                     &handled);
                if (rc || handled) return rc;
                if (algo == 1) return set_error(BM_ERR_NOTIMPL, "gemm: tensor-core path cannot take this shape");
            }
            return gemm_simt<float>(ta, tb, m, n, k, A, a.lda, B, b.lda, C, c.lda);
        }
        case BM_F64: {
            if (algo != 2) {
                bool handled = false;
                int rc = gemm_dmma_f64(ta, tb, m, n, k, (const double*)A, a.lda, (const double*)B, b.lda, (double*)C,
                                       c.lda, &handled);
                if (rc || handled) return rc;
                if (algo == 1) return set_error(BM_ERR_NOTIMPL, "gemm: DMMA path cannot take this shape");
            }
            return gemm_simt<double>(ta, tb, m, n, k, A, a.lda, B, b.lda, C, c.lda);
        }
        case BM_I32: return gemm_simt<int>(ta, tb, m, n, k, A, a.lda, B, b.lda, C, c.lda);
        case BM_U64: return gemm_simt<unsigned long long>(ta, tb, m, n, k, A, a.lda, B, b.lda, C, c.lda);
    }
    return set_error(BM_ERR_ARG, "gemm: bad dtype");
}

int launch_lgrad_finish(const double* gpart, int grid, int64_t k, float* g, const float* leaves, const float* r,
                        int64_t m, float* accu_out) {
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cudaLaunchConfig_t cfg;
    std::memset(&cfg, 0, sizeof cfg);
    cfg.gridDim = dim3((unsigned)((k + 31) / 32 + (accu_out ? 1 : 0)));
    cfg.blockDim = dim3(256);
    cfg.stream = st().stream;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    BM_CUDA(cudaLaunchKernelEx(&cfg, bm::lgrad_finish_kernel, gpart, grid, (bm::i64)k, g, leaves, r, (bm::i64)m, accu_out));
    st().launches++;
    return BM_OK;
}

}  // namespace bmi
