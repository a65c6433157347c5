// bm_rdim0.cuh -- dim-0 (per-column) reductions over a column-major source S
// (reference kernels.py:502-531 `a[:, lo:hi].sum(axis=0)` / min / max / mean:
// numpy's pairwise loop down each contiguous column).  Column c is elements
// [c*ld, c*ld + rows) of S's index space.  Shared by bm_rdim.cu (S = the
// matrix) and the JIT's fused variant (S = an element-wise program over
// contiguous inputs, ld = rows: sum(2*A + B, 0) without materialising 2*A + B).
#pragma once
#include "bm_reduce.cuh"

namespace bm {

// Columns of 8*sub half-units (a power-of-two count for sum/mean; any count
// for min/max): the CTA's eight warps share one column at a time, warp w
// reducing half-units [w*sub, (w+1)*sub) -- for sum the balanced subtree
// there, the CTA then adding the eight subtree sums as the top three levels
// of the same balanced tree; for min/max a NaN-propagating partial, merged in
// any order.  One CTA streams one contiguous column (e.g. 128 KiB) instead of
// eight warps streaming eight columns, which the DRAM serves faster, and each
// warp loads its next half-unit -- across columns too -- while it reduces the
// current one.  256 threads; smem = 8 half-unit tiles.
template <typename T, int OP, class S>
__device__ __forceinline__ void rdim0_cta_body(const S& s, i64 rows, i64 cols, i64 ld, T* out, char* smem, i64 sub) {
    constexpr i64 U = PwHalf<T>::value;
    constexpr int V = 16 / sizeof(T);
    constexpr int LV = 12;
    constexpr bool MM = OP == 2 || OP == 3;
    __shared__ T res[2][8];
    __shared__ int res_nan[2][8];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    char* tile = smem + warp * BM_TILE_BYTES;
    if ((i64)blockIdx.x >= cols) return;
    int top = 0;
    while ((1ll << top) < sub) ++top;
    const i64 step = gridDim.x;
    const i64 base = (i64)warp * sub * U;
    i64 c = blockIdx.x, j = 0;
    int par = 0;
    T stk[LV + 1];
    MinMaxAcc<T, OP == 3> acc;
    HalfRows<T> cur, nxt;
    half_load<T>(s, c * ld + base, cur);
    while (true) {
        i64 nc = c, nj = j + 1;
        if (nj == sub) { nj = 0; nc = c + step; }
        if (nc < cols) half_load<T>(s, nc * ld + base + nj * U, nxt);
        if constexpr (MM) {
#pragma unroll
            for (int r = 0; r < 8; ++r)
#pragma unroll
                for (int k = 0; k < V; ++k) acc.add(cur.v[r][k]);
        } else {
            T v = half_reduce<T>(cur, tile);
            // binary-counter merge: j's t trailing ones are the pending left subtrees
            // v folds with (stk[0] first), then v is parked at level t.  Constant
            // indices only, so the stack stays in registers (a `break` out of the
            // unrolled loop put it in local memory)
            const int t = __ffsll(~(long long)j) - 1;
#pragma unroll
            for (int l = 0; l < LV; ++l)
                if (l < t) v = stk[l] + v;
#pragma unroll
            for (int l = 0; l <= LV; ++l)
                if (l == t) stk[l] = v;
        }
        if (nj == 0) {
            if constexpr (MM) {
                acc.warp_merge();
                if (lane == 0) {
                    res[par][warp] = acc.v;
                    res_nan[par][warp] = acc.nan;
                }
                acc = MinMaxAcc<T, OP == 3>();
            } else {
                T r = stk[0];
#pragma unroll
                for (int l = 1; l <= LV; ++l)
                    if (l == top) r = stk[l];
                if (lane == 0) res[par][warp] = r;
            }
            __syncthreads();
            if (threadIdx.x == 0) {
                const T* q = res[par];
                T o;
                if constexpr (MM) {
                    MinMaxAcc<T, OP == 3> m;
#pragma unroll
                    for (int w = 0; w < 8; ++w) {
                        MinMaxAcc<T, OP == 3> x;
                        x.v = q[w];
                        x.nan = res_nan[par][w] != 0;
                        m.merge(x);
                    }
                    o = m.result();
                } else {
                    T sum = ((q[0] + q[1]) + (q[2] + q[3])) + ((q[4] + q[5]) + (q[6] + q[7]));
                    sum = sum + T(0);
                    o = sum;
                    if constexpr (OP == 5) o = OpDiv::f(sum, KScal<T>::f((double)rows, rows));
                }
                out[c] = o;
            }
            par ^= 1;
        }
        if (nc >= cols) break;
        c = nc;
        j = nj;
        cur = nxt;
    }
}

// Any column length: one warp per column (sum/mean: numpy's pairwise tree via
// pw_generic, integers wrap in any order; min/max: NaN-propagating, 16-byte
// loads when vec_ok -- the host guarantees ld % (16 / sizeof(T)) == 0 then).
// 256 threads; smem = 8 half-unit tiles.
template <typename T, int OP, class S>
__device__ __forceinline__ void rdim0_col_body(const S& s, i64 rows, i64 cols, i64 ld, T* out, char* smem,
                                               bool vec_ok) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    char* tile = smem + warp * BM_TILE_BYTES;
    const i64 gw = (i64)blockIdx.x * (blockDim.x >> 5) + warp;
    const i64 nw = (i64)gridDim.x * (blockDim.x >> 5);
    for (i64 c = gw; c < cols; c += nw) {
        const i64 c0 = c * ld;
        T r;
        if constexpr (OP == 1 || OP == 5) {
            T sum;
            if constexpr (is_float_t<T>::value) {
                sum = pw_generic<T>(s, c0, rows, tile, vec_ok) + T(0);
            } else {
                T acc = 0;
                for (i64 i = lane; i < rows; i += 32) acc = OpPlus::f(acc, s.at(c0 + i));
#pragma unroll
                for (int m = 16; m >= 1; m >>= 1) acc = OpPlus::f(acc, warp_shfl_xor(acc, m));
                sum = acc;
            }
            r = sum;
            if constexpr (OP == 5) r = OpDiv::f(sum, KScal<T>::f((double)rows, rows));
        } else if constexpr (OP == 6) {
            // unbiased variance, two passes in f64 (kernels.py:519-527)
            if (rows < 2) {
                r = T(0);
            } else {
                double s1 = 0;
                for (i64 i = lane; i < rows; i += 32) s1 += cvt<double>(s.at(c0 + i));
#pragma unroll
                for (int m = 16; m >= 1; m >>= 1) s1 += warp_shfl_xor(s1, m);
                const double mean = s1 / (double)rows;
                double s2 = 0;
                for (i64 i = lane; i < rows; i += 32) {
                    const double d = cvt<double>(s.at(c0 + i)) - mean;
                    s2 += d * d;
                }
#pragma unroll
                for (int m = 16; m >= 1; m >>= 1) s2 += warp_shfl_xor(s2, m);
                r = cvt<T>(s2 / (double)(rows - 1));
            }
        } else {
            constexpr int V = 16 / sizeof(T);
            MinMaxAcc<T, OP == 3> acc;
            i64 i = 0;
            if (vec_ok) {
                for (; i + 4 * 32 * V <= rows; i += 4 * 32 * V) {
                    T v[4][V];
#pragma unroll
                    for (int u = 0; u < 4; ++u) s.template vec<V>(c0 + i + u * 32 * V + lane * V, v[u]);
#pragma unroll
                    for (int u = 0; u < 4; ++u)
#pragma unroll
                        for (int k = 0; k < V; ++k) acc.add(v[u][k]);
                }
            }
            for (i64 jj = i + lane; jj < rows; jj += 32) acc.add(s.at(c0 + jj));
            acc.warp_merge();
            r = acc.result();
        }
        if (lane == 0) out[c] = r;
    }
}

}  // namespace bm

// ---------------------------------------------------------------------------
// dim 1 (one value per row) of an element-wise program, TMA-staged: the
// reference folds each row left to right, 0 + v[:,0] + v[:,1] + ... (numpy's
// row-block reduction, kernels.py:502-531).  A CTA owns 112 rows; a producer
// warp streams every input's [112 rows x CT columns] tile of the slab through
// a 3-stage mbarrier ring (CT = 64 / inputs, so a stage stays <= 56 KB), and
// thread r folds row r column by column, evaluating the program on the staged
// values (E::at over E::Pre) -- the same values and order as reducing the
// materialised matrix.  Used by the JIT's fused variant (bm_jit.cu).
#include "bm_lgrad.cuh"

namespace bm {

#define BM_R1F_ROWS 112
#define BM_R1F_STAGES 3

struct R1Args {                 // one __grid_constant__ parameter, like LgArgs
    Args a;                     // program inputs and scalars
    LgTmap m[8];                // the inputs as [rows x cols] tensor maps (up to 8)
    i64 rows, cols;
    void* out;
};

template <typename T, int OP, class E, int NIN>
__device__ __forceinline__ void rdim1_fused_body(const R1Args& P) {
    const Args& a = P.a;
    const i64 rows = P.rows, cols = P.cols;
    T* out = reinterpret_cast<T*>(P.out);
    constexpr int RT = BM_R1F_ROWS;
    constexpr int CT = NIN == 1 ? 64 : (NIN == 2 ? 32 : (NIN <= 4 ? 16 : 8));   // columns per tile: ~constant stage bytes
    constexpr int ST = BM_R1F_STAGES;
    constexpr unsigned TILE = RT * CT * sizeof(T);
    constexpr unsigned STAGE = NIN * TILE;
    extern __shared__ __align__(128) char smem[];
    unsigned long long* full = reinterpret_cast<unsigned long long*>(smem + ST * STAGE);
    unsigned long long* empty = full + ST;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const i64 row0 = (i64)blockIdx.x * RT;
    const i64 ntiles = (cols + CT - 1) / CT;
    constexpr int PASSES = OP == 6 ? 2 : 1;    // var: mean, then squared deviations
    if (threadIdx.x == 0) {
        for (int s = 0; s < ST; ++s) {
            lg_bar_init(&full[s], 1);
            lg_bar_init(&empty[s], 4);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
#pragma unroll
        for (int j = 0; j < NIN; ++j) asm volatile("prefetch.tensormap [%0];" ::"l"(&P.m[j]) : "memory");
    }
    __syncthreads();
    if (warp == 0) {
        if (lane == 0) {
            for (i64 t = 0; t < PASSES * ntiles; ++t) {
                const int s = (int)(t % ST);
                if (t >= ST) lg_wait(&empty[s], (unsigned)(((t / ST) - 1) & 1));
                lg_expect_tx(&full[s], STAGE);
#pragma unroll
                for (int j = 0; j < NIN; ++j)
                    lg_tma_2d(smem + s * STAGE + j * TILE, &P.m[j], (int)row0, (int)((t % ntiles) * CT), &full[s]);
            }
        }
        return;
    }
    const int r = (warp - 1) * 32 + lane;   // row within the slab
    const bool active = r < RT && row0 + r < rows;
    T acc = T(0);
    MinMaxAcc<T, OP == 3> mm;
    double dacc = 0.0, mean = 0.0;
    for (i64 t = 0; t < PASSES * ntiles; ++t) {
        const int s = (int)(t % ST);
        lg_wait(&full[s], (unsigned)((t / ST) & 1));
        const T* st = reinterpret_cast<const T*>(smem + s * STAGE);
        const i64 tc = t % ntiles;
        i64 nc = cols - tc * CT;
        if (nc > CT) nc = CT;
        if (active) {
            for (int c = 0; c < nc; ++c) {
                typename E::Pre pre;
#pragma unroll
                for (int j = 0; j < NIN; ++j) pre.x[j] = st[j * (TILE / sizeof(T)) + c * RT + r];
                const T v = E::at(a, pre);
                if constexpr (OP == 2 || OP == 3) {
                    mm.add(v);
                } else if constexpr (OP == 6) {
                    if (t < ntiles) {
                        dacc += cvt<double>(v);
                    } else {
                        const double d = cvt<double>(v) - mean;
                        dacc += d * d;
                    }
                } else {
                    acc = OpPlus::f(acc, v);
                }
            }
        }
        __syncwarp();
        if (lane == 0) lg_arrive(&empty[s]);
        if constexpr (OP == 6) {
            if (t == ntiles - 1) {
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

}  // namespace bm
