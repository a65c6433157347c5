// bm_rdim.cu -- per-dimension reductions rdim_sum/min/max/mean/var
// (reference kernels.py:496-531, lowered at expr.py:583-594).
//
// dim 0 (one value per column): the reference runs `a[:, lo:hi].sum(axis=0)`
// on a column-major view, i.e. numpy pairwise summation down each contiguous
// column; one warp per column reproduces it with bm_reduce.cuh's pairwise
// machinery (bit-exact).
//
// dim 1 (one value per row): `a[lo:hi, :].sum(axis=1)` iterates columns in the
// outer loop and accumulates every row sequentially, 0 + a[:,0] + a[:,1] + ...
// (verified bit-exact in tests/test_oracle.py).  One thread owns one row and
// folds the columns in order; the tiles of the row slab are streamed into
// shared memory by TMA (cp.async.bulk.tensor.2d) through a 3-stage mbarrier
// pipeline so a CTA keeps ~170 KB of HBM reads in flight while its threads do
// the dependent adds.
#include <cstring>
#include <type_traits>

#include "bm_internal.h"
#include "bm_ptx.cuh"
#define BM_UNIT_UNROLL 16   // single input: all 16 rows of a pairwise unit in flight
#include "bm_reduce.cuh"
#include "bm_rdim0.cuh"


namespace bm {

// ---------------------------------------------------------------------------
// dim 0

// Sum / mean over columns whose length is a power-of-two number of
// half-units (numpy's pairwise tree is then the balanced one): each warp walks
// its (column, half-unit) pairs as one stream, loading the next half-unit --
// across column boundaries too -- while it reduces the current one, so the
// loads never drain between columns.
template <typename T, int OP>
__global__ void __launch_bounds__(256, 2) rdim0_stream_kernel(const T* __restrict__ a, i64 rows, i64 cols,
                                                                       i64 lda, T* out, i64 cnt) {
    constexpr i64 U = PwHalf<T>::value;
    constexpr int LV = 12;
    extern __shared__ __align__(16) char smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    char* tile = smem + warp * BM_TILE_BYTES;
    const i64 gw = (i64)blockIdx.x * (blockDim.x >> 5) + warp;
    const i64 nw = (i64)gridDim.x * (blockDim.x >> 5);
    if (gw >= cols) return;
    int top = 0;
    while ((1ll << top) < cnt) ++top;
    i64 c = gw, u = 0;
    T stk[LV + 1];
    HalfRows<T> cur, nxt;
    half_load<T>(BufSrc<T>{a + c * lda, 1}, 0, cur);
    while (true) {
        i64 nc = c, nu = u + 1;
        if (nu == cnt) { nu = 0; nc = c + nw; }
        if (nc < cols) half_load<T>(BufSrc<T>{a + nc * lda, 1}, nu * U, nxt);
        T v = half_reduce<T>(cur, tile);
#pragma unroll
        for (int l = 0; l <= LV; ++l) {
            if (l < LV && ((u >> l) & 1)) {
                v = stk[l] + v;
            } else {
                stk[l] = v;
                break;
            }
        }
        if (nu == 0) {
            T sum = stk[0];
#pragma unroll
            for (int l = 1; l <= LV; ++l)
                if (l == top) sum = stk[l];
            sum = sum + T(0);
            T r = sum;
            if constexpr (OP == 5) r = OpDiv::f(sum, KScal<T>::f((double)rows, rows));
            if (lane == 0) out[c] = r;
        }
        if (nc >= cols) break;
        c = nc;
        u = nu;
        cur = nxt;
    }
}

// Columns of 8*sub half-units: one CTA per column at a time (bm_rdim0.cuh)
template <typename T, int OP>
__global__ void __launch_bounds__(256, 2) rdim0_cta_kernel(const T* __restrict__ a, i64 rows, i64 cols, i64 lda,
                                                           T* out, i64 sub) {
    extern __shared__ __align__(16) char smem[];
    rdim0_cta_body<T, OP>(BufSrc<T>{a, 1}, rows, cols, lda, out, smem, sub);
}

template <typename T, int OP>
__global__ void __launch_bounds__(256, 2) rdim0_kernel(const T* __restrict__ a, i64 rows, i64 cols, i64 lda, T* out,
                                                    int vec_ok) {
    extern __shared__ __align__(16) char smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    char* tile = smem + warp * BM_TILE_BYTES;
    const i64 gw = (i64)blockIdx.x * (blockDim.x >> 5) + warp;
    const i64 nw = (i64)gridDim.x * (blockDim.x >> 5);
    for (i64 c = gw; c < cols; c += nw) {
        const T* col = a + c * lda;
        const BufSrc<T> s{col, 1};
        T r;
        if constexpr (OP == 1 || OP == 5) {
            T sum;
            if constexpr (is_float_t<T>::value) {
                sum = pw_generic<T>(s, 0, rows, tile, vec_ok != 0) + T(0);
            } else {
                T acc = 0;
                for (i64 i = lane; i < rows; i += 32) acc = OpPlus::f(acc, col[i]);
#pragma unroll
                for (int m = 16; m >= 1; m >>= 1) acc = OpPlus::f(acc, warp_shfl_xor(acc, m));
                sum = acc;
            }
            if constexpr (OP == 5) {
                // mean: eop_scalar_div_post by the extent in the element type (kernels.py:516-518)
                r = OpDiv::f(sum, KScal<T>::f((double)rows, rows));
            } else {
                r = sum;
            }
        } else if constexpr (OP == 2 || OP == 3) {
            constexpr int V = 16 / sizeof(T);
            MinMaxAcc<T, OP == 3> acc;
            i64 i = 0;
            if (vec_ok) {
                for (; i + 4 * 32 * V <= rows; i += 4 * 32 * V) {
                    T v[4][V];
#pragma unroll
                    for (int u = 0; u < 4; ++u) s.template vec<V>(i + u * 32 * V + lane * V, v[u]);
#pragma unroll
                    for (int u = 0; u < 4; ++u)
#pragma unroll
                        for (int k = 0; k < V; ++k) acc.add(v[u][k]);
                }
            }
            for (i64 j = i + lane; j < rows; j += 32) acc.add(col[j]);
            acc.warp_merge();
            r = acc.result();
        } else {
            // unbiased variance, two passes in f64 (kernels.py:519-527)
            if (rows < 2) {
                r = T(0);
            } else {
                double s1 = 0;
                for (i64 i = lane; i < rows; i += 32) s1 += cvt<double>(col[i]);
#pragma unroll
                for (int m = 16; m >= 1; m >>= 1) s1 += warp_shfl_xor(s1, m);
                const double mean = s1 / (double)rows;
                double s2 = 0;
                for (i64 i = lane; i < rows; i += 32) {
                    const double d = cvt<double>(col[i]) - mean;
                    s2 += d * d;
                }
#pragma unroll
                for (int m = 16; m >= 1; m >>= 1) s2 += warp_shfl_xor(s2, m);
                r = cvt<T>(s2 / (double)(rows - 1));
            }
        }
        if (lane == 0) out[c] = r;
    }
}

// ---------------------------------------------------------------------------
// dim 1 -- TMA-staged row slabs

#define BM_R1_ROWS 112   // rows per CTA: 16384 rows -> 147 CTAs on 148 SMs
#define BM_R1_STAGES 3

template <typename T, int OP>
__global__ void __launch_bounds__(160, 1) rdim1_tma_kernel(const __grid_constant__ CUtensorMap tm, i64 rows, i64 cols,
                                                            T* out) {
    constexpr int RT = BM_R1_ROWS;
    constexpr int CT = 64;
    constexpr int ST = BM_R1_STAGES;
    constexpr uint32_t TILE_BYTES = RT * CT * sizeof(T);
    extern __shared__ __align__(128) char smem[];
    T* tiles = reinterpret_cast<T*>(smem);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + ST * TILE_BYTES);
    uint64_t* empty = full + ST;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const i64 row0 = (i64)blockIdx.x * RT;
    const i64 ntiles = (cols + CT - 1) / CT;
    const int passes = (OP == 6) ? 2 : 1;
    if (threadIdx.x == 0) {
        for (int s = 0; s < ST; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 4);
        }
        mbar_fence_init();
        tma_prefetch_desc(&tm);
    }
    __syncthreads();
    if (warp == 0) {
        if (lane == 0) {
            i64 t = 0;
            for (int p = 0; p < passes; ++p) {
                for (i64 j = 0; j < ntiles; ++j, ++t) {
                    const int s = (int)(t % ST);
                    if (t >= ST) mbar_wait(&empty[s], (uint32_t)(((t / ST) - 1) & 1));
                    mbar_expect_tx(&full[s], TILE_BYTES);
                    tma_load_2d(tiles + (size_t)s * RT * CT, &tm, (int)row0, (int)(j * CT), &full[s]);
                }
            }
        }
        return;
    }
    const int r = (warp - 1) * 32 + lane;  // row within the slab
    const bool active = r < RT && row0 + r < rows;
    T acc = T(0);
    MinMaxAcc<T, OP == 3> mm;
    double dacc = 0.0, mean = 0.0;
    i64 t = 0;
    for (int p = 0; p < passes; ++p) {
        for (i64 j = 0; j < ntiles; ++j, ++t) {
            const int s = (int)(t % ST);
            mbar_wait(&full[s], (uint32_t)((t / ST) & 1));
            const T* tile = tiles + (size_t)s * RT * CT;
            i64 nc = cols - j * CT;
            if (nc > CT) nc = CT;
            if (active) {
                if constexpr (OP == 1 || OP == 5) {
                    for (int c = 0; c < nc; ++c) acc = OpPlus::f(acc, tile[c * RT + r]);
                } else if constexpr (OP == 2 || OP == 3) {
                    for (int c = 0; c < nc; ++c) mm.add(tile[c * RT + r]);
                } else {
                    if (p == 0) {
                        for (int c = 0; c < nc; ++c) dacc += cvt<double>(tile[c * RT + r]);
                    } else {
                        for (int c = 0; c < nc; ++c) {
                            const double d = cvt<double>(tile[c * RT + r]) - mean;
                            dacc += d * d;
                        }
                    }
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[s]);
        }
        if constexpr (OP == 6) {
            if (p == 0) {
                mean = dacc / (double)cols;
                dacc = 0.0;
            }
        }
    }
    if (!active) return;
    T res;
    if constexpr (OP == 5) res = OpDiv::f(acc, KScal<T>::f((double)cols, cols));
    else if constexpr (OP == 6) res = (cols < 2) ? T(0) : cvt<T>(dacc / (double)(cols - 1));
    else if constexpr (OP == 2 || OP == 3) res = mm.result();
    else res = acc;
    out[row0 + r] = res;
}

// The reference reduces dim 1 in blocks of DIM_BLOCK = 64 rows (kernels.py:89,
// 425-426).  A block holding exactly one row is a 1 x cols view whose
// reduction numpy runs with its pairwise inner loop instead of the row-wise
// sequential fold, so that row is summed pairwise (one warp).
template <typename T, int OP>
__global__ void __launch_bounds__(32) rdim1_lone_row_kernel(const T* __restrict__ a, i64 row, i64 cols, i64 lda,
                                                              T* out) {
    __shared__ __align__(16) char tile[BM_TILE_BYTES];
    const BufSrc<T> s{a + row, lda};
    T sum = pw_generic<T>(s, 0, cols, tile, false) + T(0);
    if constexpr (OP == 5) sum = OpDiv::f(sum, KScal<T>::f((double)cols, cols));
    if (threadIdx.x == 0) out[row] = sum;
}

// fallback for layouts TMA cannot describe (misaligned or odd leading dimension)
template <typename T, int OP>
__global__ void __launch_bounds__(128) rdim1_simple_kernel(const T* __restrict__ a, i64 rows, i64 cols, i64 lda, T* out) {
    const i64 r = (i64)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= rows) return;
    const T* p = a + r;
    if constexpr (OP == 6) {
        if (cols < 2) { out[r] = T(0); return; }
        double s1 = 0;
        for (i64 c = 0; c < cols; ++c) s1 += cvt<double>(p[c * lda]);
        const double mean = s1 / (double)cols;
        double s2 = 0;
        for (i64 c = 0; c < cols; ++c) {
            const double d = cvt<double>(p[c * lda]) - mean;
            s2 += d * d;
        }
        out[r] = cvt<T>(s2 / (double)(cols - 1));
        return;
    } else {
        T acc = (OP == 2 || OP == 3) ? p[0] : T(0);
        for (i64 c = 0; c < cols; ++c) {
            const T x = p[c * lda];
            if constexpr (OP == 2) acc = np_min(acc, x);
            else if constexpr (OP == 3) acc = np_max(acc, x);
            else acc = OpPlus::f(acc, x);
        }
        if constexpr (OP == 5) acc = OpDiv::f(acc, KScal<T>::f((double)cols, cols));
        out[r] = acc;
    }
}

}  // namespace bm

namespace bmi {

template <typename T> struct is_float_t_host { static const bool value = std::is_floating_point<T>::value; };

template <typename T, int OP>
static int rdim_launch(const bm_view& in, void* out_base, int dim) {
    const int64_t sz = sizeof(T);
    const T* a = reinterpret_cast<const T*>((const char*)in.base + in.offset * sz);
    T* out = reinterpret_cast<T*>(out_base);
    const int64_t rows = in.rows, cols = in.cols, lda = in.lda;
    cudaStream_t s = st().stream;
    if (dim == 0) {
        if (cols == 0) return BM_OK;
        const bool vec = (((uintptr_t)a & 15u) == 0) && ((lda * sz) % 16 == 0);
        int grid = (int)((cols + 7) / 8);
        const int cap = st().sm_count * 2;   // 2 resident CTAs per SM (registers / ring)
        if (grid > cap) grid = cap;
        constexpr int64_t U = 4096 / sizeof(T);   // PwHalf: 1024 f32 / 512 f64 elements
        const int64_t cnt = rows / U;
        const bool pow2 = rows % U == 0 && cnt >= 1 && cnt <= 4096 && (cnt & (cnt - 1)) == 0;
        constexpr bool fsum = (OP == 1 || OP == 5) && is_float_t_host<T>::value;
        static const bool cta_on = !std::getenv("BM_RD0_CTA") || std::atoi(std::getenv("BM_RD0_CTA"));
        if (cta_on && vec && rows % U == 0 && cnt >= 8 && cnt / 8 <= 4096 &&
            ((fsum && pow2) || ((OP == 2 || OP == 3) && cnt % 8 == 0))) {
            int cgrid = (int)cols;
            const int ccap = st().sm_count * 2;
            if (cgrid > ccap) {
                // columns per CTA k, then just enough CTAs that none gets more than k
                const int64_t k = (cols + ccap - 1) / ccap;
                cgrid = (int)((cols + k - 1) / k);
            }
            bm::rdim0_cta_kernel<T, OP><<<cgrid, 256, 8 * BM_TILE_BYTES, s>>>(a, rows, cols, lda, out, cnt / 8);
            BM_CUDA(cudaGetLastError());
            st().launches++;
            return BM_OK;
        }
        if constexpr (fsum) {
            static const bool stream_on = !std::getenv("BM_RDIM0_STREAM") || std::atoi(std::getenv("BM_RDIM0_STREAM"));
            if (stream_on && vec && pow2) {
                int sgrid = (int)((cols + 7) / 8);
                const int scap = st().sm_count * 2;
                if (sgrid > scap) {
                    const int64_t k = (cols + 8LL * scap - 1) / (8LL * scap);
                    sgrid = (int)((cols + 8 * k - 1) / (8 * k));
                }
                bm::rdim0_stream_kernel<T, OP><<<sgrid, 256, 8 * BM_TILE_BYTES, s>>>(a, rows, cols, lda, out, cnt);
                BM_CUDA(cudaGetLastError());
                st().launches++;
                return BM_OK;
            }
        }
        static bool attr = false;
        if (!attr) {
            BM_CUDA(cudaFuncSetAttribute(bm::rdim0_kernel<T, OP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         8 * BM_TILE_BYTES));
            attr = true;
        }
        bm::rdim0_kernel<T, OP><<<grid, 256, 8 * BM_TILE_BYTES, s>>>(a, rows, cols, lda, out, vec ? 1 : 0);
        BM_CUDA(cudaGetLastError());
        st().launches++;
        return BM_OK;
    }
    if (rows == 0) return BM_OK;
    int64_t rows_main = rows;
    if constexpr ((OP == 1 || OP == 5) && is_float_t_host<T>::value) {
        if (rows % 64 == 1 && cols > 0) {
            bm::rdim1_lone_row_kernel<T, OP><<<1, 32, 0, s>>>(a, rows - 1, cols, lda, out);
            BM_CUDA(cudaGetLastError());
            st().launches++;
            rows_main = rows - 1;
            if (rows_main == 0) return BM_OK;
        }
    }
    const bool tma_ok = (((uintptr_t)a & 15u) == 0) && ((lda * sz) % 16 == 0) && rows_main >= 4 * BM_R1_ROWS &&
                        cols >= 1 && rows_main < (1LL << 31) && cols < (1LL << 31);
    if (tma_ok) {
        CUtensorMap tm;
        const cuuint64_t gdim[2] = {(cuuint64_t)rows_main, (cuuint64_t)cols};
        const cuuint64_t gstride[1] = {(cuuint64_t)(lda * sz)};
        const cuuint32_t box[2] = {BM_R1_ROWS, 64};
        const cuuint32_t estr[2] = {1, 1};
        CUtensorMapDataType dt = sz == 4 ? (std::is_same<T, float>::value ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32
                                                                          : CU_TENSOR_MAP_DATA_TYPE_INT32)
                                         : (std::is_same<T, double>::value ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64
                                                                           : CU_TENSOR_MAP_DATA_TYPE_UINT64);
        CUresult r = drv().tensorMapEncodeTiled(&tm, dt, 2, (void*)a, gdim, gstride, box, estr,
                                                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                                CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) return cu_fail(r, "cuTensorMapEncodeTiled (rdim dim 1)");
        const int smem = BM_R1_STAGES * BM_R1_ROWS * 64 * (int)sz + 2 * BM_R1_STAGES * 8;
        static bool attr = false;
        if (!attr) {
            BM_CUDA(cudaFuncSetAttribute(bm::rdim1_tma_kernel<T, OP>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
            attr = true;
        }
        const int grid = (int)((rows_main + BM_R1_ROWS - 1) / BM_R1_ROWS);
        bm::rdim1_tma_kernel<T, OP><<<grid, 160, smem, s>>>(tm, rows_main, cols, out);
        BM_CUDA(cudaGetLastError());
        st().launches++;
        return BM_OK;
    }
    const int grid = (int)((rows_main + 127) / 128);
    bm::rdim1_simple_kernel<T, OP><<<grid, 128, 0, s>>>(a, rows_main, cols, lda, out);
    BM_CUDA(cudaGetLastError());
    st().launches++;
    return BM_OK;
}

template <typename T>
static int rdim_dispatch_op(const bm_view& in, void* out, int dim, int op) {
    switch (op) {
        case BM_R_ACCU: return rdim_launch<T, 1>(in, out, dim);
        case BM_R_MIN: return rdim_launch<T, 2>(in, out, dim);
        case BM_R_MAX: return rdim_launch<T, 3>(in, out, dim);
        case BM_R_MEAN: return rdim_launch<T, 5>(in, out, dim);
        case BM_R_VAR: return rdim_launch<T, 6>(in, out, dim);
    }
    return set_error(BM_ERR_ARG, "rdim: bad reduce op");
}

int launch_rdim(const bm_invocation* inv) {
    if (inv->n_inputs != 1 || !inv->has_output) return set_error(BM_ERR_ARG, "rdim: needs one input and an output");
    const bm_view& in = inv->inputs[0];
    const bm_view& o = inv->output;
    if (o.dtype != in.dtype) return set_error(BM_ERR_ARG, "rdim: output dtype must equal input dtype");
    if (o.stride != 1) return set_error(BM_ERR_ARG, "rdim: output must be contiguous");
    const int64_t extent = inv->dim == 0 ? in.rows : in.cols;
    if (extent == 0 && (inv->reduce_op == BM_R_MIN || inv->reduce_op == BM_R_MAX) &&
        (inv->dim == 0 ? in.cols : in.rows) > 0)
        return set_error(BM_ERR_EMPTY, "rdim: min/max over an empty extent");
    void* out = (char*)o.base + o.offset * dtype_size(o.dtype);
    if (inv->dim == 0 && in.rows == 0) {
        // sum/mean of nothing: numpy gives 0 (mean: 0/0); keep it simple and exact for sum
        if (inv->reduce_op == BM_R_ACCU) {
            BM_CUDA(cudaMemsetAsync(out, 0, (size_t)(in.cols * dtype_size(in.dtype)), st().stream));
            return BM_OK;
        }
    }
    switch (in.dtype) {
        case BM_F32: return rdim_dispatch_op<float>(in, out, inv->dim, inv->reduce_op);
        case BM_F64: return rdim_dispatch_op<double>(in, out, inv->dim, inv->reduce_op);
        case BM_I32: return rdim_dispatch_op<int>(in, out, inv->dim, inv->reduce_op);
        case BM_U64: return rdim_dispatch_op<unsigned long long>(in, out, inv->dim, inv->reduce_op);
    }
    return set_error(BM_ERR_ARG, "rdim: bad dtype");
}

}  // namespace bmi
