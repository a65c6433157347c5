// bm_misc.cu -- generators and data movement that feed the hot path:
// gen_fill_const / gen_eye / gen_linspace / gen_randu / gen_randn
// (reference kernels.py:536-575) and mov_transpose / strided extract / insert /
// resize / reshape / join / diagmat / diagvec / repmat (kernels.py:578-640).
// These are memory-movement kernels: coalesced grid-stride loops, one
// numpy-exact conversion on store.
#include <cstring>

#include "bm_internal.h"
#include "bm_reduce.cuh"

namespace bm {

template <typename T>
__global__ void fill_kernel(T* __restrict__ p, i64 n, i64 stride, T v) {
    const i64 tid = (i64)blockIdx.x * blockDim.x + threadIdx.x, nt = (i64)gridDim.x * blockDim.x;
    for (i64 i = tid; i < n; i += nt) p[i * stride] = v;
}

template <typename T>
__global__ void eye_kernel(T* __restrict__ p, i64 n, i64 rows, T one, T zero) {
    const i64 tid = (i64)blockIdx.x * blockDim.x + threadIdx.x, nt = (i64)gridDim.x * blockDim.x;
    for (i64 i = tid; i < n; i += nt) p[i] = ((i % rows) == (i / rows)) ? one : zero;
}

// linspace: start + (end - start) * i / (n - 1) in f64 (kernels.py:547-555), then
// _stage_cast to the generator type and cast_out to the output type
template <typename TG, typename TO>
__global__ void linspace_kernel(TO* __restrict__ p, i64 count, i64 stride, double start, double end, i64 n) {
    const i64 tid = (i64)blockIdx.x * blockDim.x + threadIdx.x, nt = (i64)gridDim.x * blockDim.x;
    for (i64 i = tid; i < count; i += nt) {
        double v;
        if (n == 1) v = start;
        else v = start + ((end - start) * (double)i) / (double)(n - 1);
        p[i * stride] = cvt<TO>(cvt<TG>(v));
    }
}

// splitmix64 counter RNG (kernels.py:227-245): value = f(seed, stream, index)
__device__ __forceinline__ u64 mix64(u64 x) {
    u64 z = x + 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
__device__ __forceinline__ double uniform_at(u64 key, u64 idx) {
    return (double)(mix64(idx ^ key) >> 11) * 0x1.0p-53;
}

template <typename TG, typename TO>
__global__ void randu_kernel(TO* __restrict__ p, i64 n, i64 stride, u64 key) {
    const i64 tid = (i64)blockIdx.x * blockDim.x + threadIdx.x, nt = (i64)gridDim.x * blockDim.x;
    for (i64 i = tid; i < n; i += nt) p[i * stride] = cvt<TO>(cvt<TG>(uniform_at(key, (u64)i)));
}

// Box-Muller over the paired stream (kernels.py:248-253): u1 at 2i, u2 at 2i+1
template <typename TG, typename TO>
__global__ void randn_kernel(TO* __restrict__ p, i64 n, i64 stride, u64 key) {
    const i64 tid = (i64)blockIdx.x * blockDim.x + threadIdx.x, nt = (i64)gridDim.x * blockDim.x;
    const double two_pi = 2.0 * 3.141592653589793;
    for (i64 i = tid; i < n; i += nt) {
        const double u1 = uniform_at(key, 2 * (u64)i);
        const double u2 = uniform_at(key, 2 * (u64)i + 1);
        const double z = sqrt(-2.0 * log1p(-u1)) * cos(two_pi * u2);
        p[i * stride] = cvt<TO>(cvt<TG>(z));
    }
}

// dst(r, c) = cast(src(r, c)) over rows x cols, both column-major with leading dims
template <typename TI, typename TO>
__global__ void copy2d_kernel(const TI* __restrict__ src, i64 s_ld, TO* __restrict__ dst, i64 d_ld, i64 rows, i64 cols) {
    const i64 n = rows * cols;
    const i64 tid = (i64)blockIdx.x * blockDim.x + threadIdx.x, nt = (i64)gridDim.x * blockDim.x;
    for (i64 i = tid; i < n; i += nt) {
        const i64 r = i % rows, c = i / rows;
        dst[r + c * d_ld] = cvt<TO>(src[r + c * s_ld]);
    }
}

template <typename TI, typename TO>
__global__ void repmat_kernel(const TI* __restrict__ src, i64 s_ld, i64 sr, i64 sc, TO* __restrict__ dst, i64 rows_out,
                              i64 n) {
    const i64 tid = (i64)blockIdx.x * blockDim.x + threadIdx.x, nt = (i64)gridDim.x * blockDim.x;
    for (i64 i = tid; i < n; i += nt) {
        const i64 r = (i % rows_out) % sr, c = (i / rows_out) % sc;
        dst[i] = cvt<TO>(src[r + c * s_ld]);
    }
}

// out (cols x rows) = in^T, 32x32 tiles through shared memory
template <typename TI, typename TO>
__global__ void transpose_kernel(const TI* __restrict__ src, i64 s_ld, TO* __restrict__ dst, i64 d_ld, i64 rows,
                                 i64 cols) {
    __shared__ TI tile[32][33];
    const i64 r0 = (i64)blockIdx.x * 32, c0 = (i64)blockIdx.y * 32;
    for (int k = threadIdx.y; k < 32; k += blockDim.y) {
        const i64 r = r0 + threadIdx.x, c = c0 + k;
        if (r < rows && c < cols) tile[k][threadIdx.x] = src[r + c * s_ld];
    }
    __syncthreads();
    for (int k = threadIdx.y; k < 32; k += blockDim.y) {
        // output element (c, r): row index c0 + threadIdx.x of dst, column r0 + k
        const i64 orow = c0 + threadIdx.x, ocol = r0 + k;
        if (orow < cols && ocol < rows) dst[orow + ocol * d_ld] = cvt<TO>(tile[threadIdx.x][k]);
    }
}

}  // namespace bm

namespace bmi {

static int grid_for(int64_t n) {
    int64_t g = (n + 255) / 256;
    const int64_t cap = (int64_t)st().sm_count * 16;
    if (g > cap) g = cap;
    return (int)(g < 1 ? 1 : g);
}

#define BM_LAUNCHED()                  \
    do {                               \
        BM_CUDA(cudaGetLastError());   \
        st().launches++;               \
    } while (0)

static char* view_ptr(const bm_view& v) { return (char*)v.base + v.offset * dtype_size(v.dtype); }

// element type dispatch helpers
template <typename F>
static int with_type(int dt, F&& f) {
    switch (dt) {
        case BM_F32: return f(float());
        case BM_F64: return f(double());
        case BM_I32: return f(int());
        case BM_U64: return f((unsigned long long)0);
    }
    return set_error(BM_ERR_ARG, "bad dtype");
}

template <typename TO>
static TO from_bits(int64_t bits) {
    TO v;
    std::memcpy(&v, &bits, sizeof(TO));
    return v;
}

// logical view geometry: rows x cols with leading dim (flat views are 1 x count, ld = stride)
struct Geo {
    int64_t rows, cols, ld;
};
static Geo geo(const bm_view& v) {
    if (v.is_block) return Geo{v.rows, v.cols, v.lda};
    return Geo{1, v.count, v.stride};
}

static int copy2d(const bm_view& src, int64_t s_off, int64_t s_ld, const bm_view& dst, int64_t d_off, int64_t d_ld,
                  int64_t rows, int64_t cols) {
    if (rows <= 0 || cols <= 0) return BM_OK;
    const char* sp = view_ptr(src) + s_off * dtype_size(src.dtype);
    char* dp = view_ptr(dst) + d_off * dtype_size(dst.dtype);
    return with_type(src.dtype, [&](auto ti) {
        typedef decltype(ti) TI;
        return with_type(dst.dtype, [&](auto to) {
            typedef decltype(to) TO;
            bm::copy2d_kernel<TI, TO><<<grid_for(rows * cols), 256, 0, st().stream>>>((const TI*)sp, s_ld, (TO*)dp, d_ld,
                                                                                        rows, cols);
            BM_LAUNCHED();
            return BM_OK;
        });
    });
}

static int fill_view(const bm_view& dst, int64_t bits_zero_ok) {
    (void)bits_zero_ok;
    const Geo g = geo(dst);
    if (g.rows * g.cols == 0) return BM_OK;
    char* dp = view_ptr(dst);
    if (g.rows == 1 || g.ld == g.rows) {
        if (g.rows == 1 && g.ld == 1) {
            BM_CUDA(cudaMemsetAsync(dp, 0, (size_t)(g.cols * dtype_size(dst.dtype)), st().stream));
            return BM_OK;
        }
        if (g.ld == g.rows) {
            BM_CUDA(cudaMemsetAsync(dp, 0, (size_t)(g.rows * g.cols * dtype_size(dst.dtype)), st().stream));
            return BM_OK;
        }
    }
    return with_type(dst.dtype, [&](auto to) {
        typedef decltype(to) TO;
        // zero a strided 1 x n view
        bm::fill_kernel<TO><<<grid_for(g.cols), 256, 0, st().stream>>>((TO*)dp, g.cols, g.ld, TO(0));
        BM_LAUNCHED();
        return BM_OK;
    });
}

static int launch_strided(const bm_invocation* inv) {
    const bm_view& out = inv->output;
    const Geo go = geo(out);
    switch (inv->sub_kind) {
        case BM_MOV_EXTRACT:
        case BM_MOV_INSERT: {
            // element-order copy between two views of equal element count
            const bm_view& in = inv->inputs[0];
            const Geo gi = geo(in);
            if (gi.rows * gi.cols != go.rows * go.cols) return set_error(BM_ERR_ARG, "extract/insert: size mismatch");
            if (gi.rows == go.rows || go.rows * go.cols == 0) return copy2d(in, 0, gi.ld, out, 0, go.ld, gi.rows, gi.cols);
            // shapes differ (block <-> flat): go through the contiguous side
            if (in.is_block && !out.is_block && go.ld == 1)
                return copy2d(in, 0, gi.ld, out, 0, gi.rows, gi.rows, gi.cols);
            if (!in.is_block && out.is_block && gi.ld == 1)
                return copy2d(in, 0, go.rows, out, 0, go.ld, go.rows, go.cols);
            return set_error(BM_ERR_NOTIMPL, "extract/insert: unsupported view pair");
        }
        case BM_MOV_RESIZE: {
            const bm_view& in = inv->inputs[0];
            int rc = fill_view(out, 0);
            if (rc) return rc;
            const int64_t kr = in.rows < out.rows ? in.rows : out.rows;
            const int64_t kc = in.cols < out.cols ? in.cols : out.cols;
            return copy2d(in, 0, in.lda, out, 0, out.lda, kr, kc);
        }
        case BM_MOV_RESHAPE: {
            const bm_view& in = inv->inputs[0];
            const int64_t ns = in.count, nd = out.count;
            const int64_t n = ns < nd ? ns : nd;
            if (nd > n) {
                bm_view tail = out;
                tail.offset += n;
                tail.count = nd - n;
                int rc = fill_view(tail, 0);
                if (rc) return rc;
            }
            return copy2d(in, 0, in.stride, out, 0, out.stride, 1, n);
        }
        case BM_MOV_JOIN_ROWS: {
            const bm_view &a = inv->inputs[0], &b = inv->inputs[1];
            int rc = copy2d(a, 0, a.lda, out, 0, out.lda, a.rows, a.cols);
            if (rc) return rc;
            return copy2d(b, 0, b.lda, out, a.cols * out.lda, out.lda, b.rows, b.cols);
        }
        case BM_MOV_JOIN_COLS: {
            const bm_view &a = inv->inputs[0], &b = inv->inputs[1];
            int rc = copy2d(a, 0, a.lda, out, 0, out.lda, a.rows, a.cols);
            if (rc) return rc;
            return copy2d(b, 0, b.lda, out, a.rows, out.lda, b.rows, b.cols);
        }
        case BM_MOV_DIAGMAT: {
            const bm_view& in = inv->inputs[0];
            int rc = fill_view(out, 0);
            if (rc) return rc;
            const int64_t n = out.rows < out.cols ? out.rows : out.cols;
            return copy2d(in, 0, in.stride, out, 0, out.lda + 1, 1, n);
        }
        case BM_MOV_DIAGVEC: {
            const bm_view& in = inv->inputs[0];
            const int64_t k = inv->iparams[0];
            const int64_t start = k >= 0 ? k * in.lda : -k;
            return copy2d(in, start, in.lda + 1, out, 0, out.stride, 1, out.count);
        }
        case BM_MOV_REPMAT: {
            const bm_view& in = inv->inputs[0];
            const int64_t n = out.count > 0 ? out.count : out.rows * out.cols;
            const int64_t rows_out = inv->iparams[0];
            if (n == 0) return BM_OK;
            return with_type(in.dtype, [&](auto ti) {
                typedef decltype(ti) TI;
                return with_type(out.dtype, [&](auto to) {
                    typedef decltype(to) TO;
                    bm::repmat_kernel<TI, TO><<<grid_for(n), 256, 0, st().stream>>>(
                        (const TI*)view_ptr(in), in.lda, in.rows, in.cols, (TO*)view_ptr(out), rows_out, n);
                    BM_LAUNCHED();
                    return BM_OK;
                });
            });
        }
    }
    return set_error(BM_ERR_ARG, "strided copy: bad sub kind");
}

int launch_misc(const bm_invocation* inv) {
    if (!inv->has_output) return set_error(BM_ERR_ARG, "kind needs an output view");
    const bm_view& out = inv->output;
    const int64_t n = out.is_block ? out.rows * out.cols : out.count;
    char* op = view_ptr(out);
    const int64_t ostride = out.is_block ? 1 : out.stride;
    switch (inv->kind) {
        case BM_K_FILL: {
            if (n == 0) return BM_OK;
            return with_type(out.dtype, [&](auto to) {
                typedef decltype(to) TO;
                bm::fill_kernel<TO><<<grid_for(n), 256, 0, st().stream>>>((TO*)op, n, ostride, from_bits<TO>(inv->iparams[0]));
                BM_LAUNCHED();
                return BM_OK;
            });
        }
        case BM_K_EYE: {
            if (n == 0) return BM_OK;
            return with_type(out.dtype, [&](auto to) {
                typedef decltype(to) TO;
                bm::eye_kernel<TO><<<grid_for(n), 256, 0, st().stream>>>((TO*)op, n, inv->iparams[2],
                                                                          from_bits<TO>(inv->iparams[0]), TO(0));
                BM_LAUNCHED();
                return BM_OK;
            });
        }
        case BM_K_LINSPACE:
        case BM_K_RANDU:
        case BM_K_RANDN: {
            if (n == 0) return BM_OK;
            return with_type(inv->compute_dtype, [&](auto tg) {
                typedef decltype(tg) TG;
                return with_type(out.dtype, [&](auto to) {
                    typedef decltype(to) TO;
                    if (inv->kind == BM_K_LINSPACE) {
                        bm::linspace_kernel<TG, TO><<<grid_for(n), 256, 0, st().stream>>>(
                            (TO*)op, n, ostride, inv->fscalars[0], inv->fscalars[1], inv->iparams[0]);
                    } else {
                        const unsigned long long key = (unsigned long long)inv->iparams[0];
                        if (inv->kind == BM_K_RANDU)
                            bm::randu_kernel<TG, TO><<<grid_for(n), 256, 0, st().stream>>>((TO*)op, n, ostride, key);
                        else
                            bm::randn_kernel<TG, TO><<<grid_for(n), 256, 0, st().stream>>>((TO*)op, n, ostride, key);
                    }
                    BM_LAUNCHED();
                    return BM_OK;
                });
            });
        }
        case BM_K_TRANSPOSE: {
            const bm_view& in = inv->inputs[0];
            if (in.rows * in.cols == 0) return BM_OK;
            return with_type(in.dtype, [&](auto ti) {
                typedef decltype(ti) TI;
                return with_type(out.dtype, [&](auto to) {
                    typedef decltype(to) TO;
                    dim3 grid((unsigned)((in.rows + 31) / 32), (unsigned)((in.cols + 31) / 32));
                    bm::transpose_kernel<TI, TO><<<grid, dim3(32, 8), 0, st().stream>>>(
                        (const TI*)view_ptr(in), in.lda, (TO*)op, out.lda, in.rows, in.cols);
                    BM_LAUNCHED();
                    return BM_OK;
                });
            });
        }
        case BM_K_STRIDED_COPY:
            return launch_strided(inv);
        case BM_K_COPY: {
            // mov_copy: flat element-order copy with cast (kernels.py:580-581)
            const bm_view& in = inv->inputs[0];
            return copy2d(in, 0, in.stride, out, 0, out.stride, 1, in.count);
        }
    }
    return set_error(BM_ERR_NOTIMPL, "unknown invocation kind");
}

}  // namespace bmi
