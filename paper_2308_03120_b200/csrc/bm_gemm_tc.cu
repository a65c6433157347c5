// bm_gemm_tc.cu -- tensor-core GEMMs for glue_times (reference kernels.py:704-708).
//
// f32: 3xTF32 on the 5th-generation tensor cores.  A pre-pass splits each
// operand into tf32 hi = rna(x) and lo = rna(x - hi) and lays both out K-major
// (the transpose of a column-major A or of B^T is folded into this pass, so
// `A @ B.t()` never materialises a transposed matrix).  The GEMM kernel
// streams 128x16 / 256x16 hi/lo tiles with TMA (SWIZZLE_64B) through a 4-stage
// mbarrier pipeline; one elected thread issues tcgen05.mma kind::tf32
// (lo*hi + hi*lo + hi*hi per k-step) into 128x256 f32 accumulators in TMEM;
// eight epilogue warps drain TMEM with tcgen05.ld and store column-major C.
// The dropped lo*lo term and the tf32 rounding of lo leave ~2^-22 relative
// error per product; the accumulation is promoted to round-to-nearest f32
// every 64 K (see below), so the result tracks an SGEMM.
//
// f64: DMMA (mma.sync.aligned.m8n8k4 f64) fed by a 4-stage cp.async ring.
#include <cstring>

#include "bm_internal.h"
#include "bm_gemm_tc.cuh"

namespace bm {

// ---------------------------------------------------------------------------
// 3xTF32 split pre-pass: out[r * kp + c] for r < rp (M or N), c < kp (K)

// the split kernel (split_tf32_body) lives in bm_reduce.cuh so that NVRTC can
// instantiate it over a fused element-wise operand (GEMM prologue fusion)
struct PlainSrc {
    const float* src;
    i64 ld;
    __device__ __forceinline__ float at(i64 idx) const { return src[idx]; }
    template <int V> __device__ __forceinline__ void vec(i64 idx, float (&v)[V]) const {
        const float4 q = __ldg(reinterpret_cast<const float4*>(src + idx));
        v[0] = q.x;
        v[1] = q.y;
        v[2] = q.z;
        v[3] = q.w;
    }
};
template <bool SRC_KMAJOR, bool VEC>
__global__ void __launch_bounds__(256) split_tf32_kernel(const float* __restrict__ src, i64 ld, i64 rows, i64 k,
                                                         float* __restrict__ hi, float* __restrict__ lo, i64 kp,
                                                         i64 rp, int trunc) {
    split_tf32_body<SRC_KMAJOR, VEC>(PlainSrc{src, ld}, ld, rows, k, hi, lo, kp, rp, trunc != 0);
}

// ---------------------------------------------------------------------------
// tcgen05 kernel.
//
// Tile 128 x 256 x 16 (K-major SWIZZLE_64B operands), 4-stage TMA ring,
// one elected thread issuing tcgen05.mma kind::tf32 into TMEM.  The tensor
// core adds its K=8 products into the f32 accumulator with truncation, so a
// long K chain drifts (max-normalised error ~1e-5 at K = 1024, 15x the
// reference's OpenBLAS SGEMM).  The accumulator is therefore promoted every
// 64 K: two TMEM buffers ping-pong, and eight epilogue warps add each finished
// 128x256 chunk into round-to-nearest f32 registers while the MMAs run on
// the other buffer (the same remedy DeepGEMM applies to FP8).

__global__ void __launch_bounds__(TC_THREADS, 1)
    gemm_3xtf32_kernel(const __grid_constant__ TmapBytes tm_ahi, const __grid_constant__ TmapBytes tm_alo,
                       const __grid_constant__ TmapBytes tm_bhi, const __grid_constant__ TmapBytes tm_blo,
                       float* __restrict__ C, i64 m, i64 n, i64 ldc, int nk, int group_m, int kb0, int accumulate) {
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    uint8_t* smem = smem_raw + (((raw + 1023u) & ~1023u) - raw);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + TC_STAGES * TC_STAGE_BYTES);
    uint64_t* empty = full + TC_STAGES;
    uint64_t* acc_full = empty + TC_STAGES;   // [2]
    uint64_t* acc_empty = acc_full + 2;       // [2]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // Grouped raster: the linear CTA index walks groups of group_m tile rows
    // column by column, so the ~148 CTAs resident at a time cover about
    // group_m x (148 / group_m) tiles and share each A and B slab several ways
    // through L2 (a plain row raster shares B ~1 way, which
    // made the 32768^3 product DRAM-bound).
    int m0, n0;
    {
        const int nm = (int)((m + TC_BM - 1) / TC_BM), nn = (int)((n + TC_BN - 1) / TC_BN);
        const int t = blockIdx.x;
        const int per_group = group_m * nn;
        const int g = t / per_group, first_m = g * group_m;
        const int gsize = (nm - first_m) < group_m ? (nm - first_m) : group_m;
        const int r = t - g * per_group;
        m0 = (first_m + r % gsize) * TC_BM;
        n0 = (r / gsize) * TC_BN;
    }
    const int nchunks = (nk + TC_CHUNK_KB - 1) / TC_CHUNK_KB;

    if (threadIdx.x == 0) {
        for (int s = 0; s < TC_STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&acc_full[b], 1);
            mbar_init(&acc_empty[b], 8);
        }
        mbar_fence_init();
        tma_prefetch_desc(&tm_ahi);
        tma_prefetch_desc(&tm_alo);
        tma_prefetch_desc(&tm_bhi);
        tma_prefetch_desc(&tm_blo);
    }
    if (warp == 1) tmem_alloc(tmem_slot, 2 * TC_BN);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    auto tile_ahi = [&](int s) { return smem + s * TC_STAGE_BYTES; };
    auto tile_alo = [&](int s) { return smem + s * TC_STAGE_BYTES + TC_TILE_A; };
    auto tile_bhi = [&](int s) { return smem + s * TC_STAGE_BYTES + 2 * TC_TILE_A; };
    auto tile_blo = [&](int s) { return smem + s * TC_STAGE_BYTES + 2 * TC_TILE_A + TC_TILE_B; };

    if (warp == 0) {
        if (lane == 0) {
            for (int kb = 0; kb < nk; ++kb) {
                const int s = kb % TC_STAGES;
                if (kb >= TC_STAGES) mbar_wait(&empty[s], (uint32_t)(((kb / TC_STAGES) - 1) & 1));
                mbar_expect_tx(&full[s], TC_STAGE_BYTES);
                const int kc = (kb0 + kb) * TC_BK;
                tma_load_2d(tile_ahi(s), &tm_ahi, kc, m0, &full[s]);
                tma_load_2d(tile_alo(s), &tm_alo, kc, m0, &full[s]);
                tma_load_2d(tile_bhi(s), &tm_bhi, kc, n0, &full[s]);
                tma_load_2d(tile_blo(s), &tm_blo, kc, n0, &full[s]);
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            constexpr uint32_t idesc = tf32_idesc(TC_BM, TC_BN);
            for (int c = 0; c < nchunks; ++c) {
                const int b = c & 1;
                if (c >= 2) mbar_wait(&acc_empty[b], (uint32_t)(((c >> 1) - 1) & 1));
                tc_fence_after();
                const uint32_t d = tmem + (uint32_t)(b * TC_BN);
                const int kb_end = (c + 1) * TC_CHUNK_KB < nk ? (c + 1) * TC_CHUNK_KB : nk;
                for (int kb = c * TC_CHUNK_KB; kb < kb_end; ++kb) {
                    const int s = kb % TC_STAGES;
                    mbar_wait(&full[s], (uint32_t)((kb / TC_STAGES) & 1));
                    tc_fence_after();
                    const uint64_t ahi = sw64_kmajor_desc(smem_u32(tile_ahi(s)));
                    const uint64_t alo = sw64_kmajor_desc(smem_u32(tile_alo(s)));
                    const uint64_t bhi = sw64_kmajor_desc(smem_u32(tile_bhi(s)));
                    const uint64_t blo = sw64_kmajor_desc(smem_u32(tile_blo(s)));
#pragma unroll
                    for (int kk = 0; kk < TC_BK / 8; ++kk) {
                        const uint64_t adv = (uint64_t)((kk * 32) >> 4);   // 8 tf32 = 32 B along K
                        const uint32_t first = (kb == c * TC_CHUNK_KB && kk == 0) ? 0u : 1u;
                        mma_tf32(d, alo + adv, bhi + adv, idesc, first);
                        mma_tf32(d, ahi + adv, blo + adv, idesc, 1u);
                        mma_tf32(d, ahi + adv, bhi + adv, idesc, 1u);
                    }
                    mma_commit(&empty[s]);
                }
                mma_commit(&acc_full[b]);
            }
        }
    } else {
        // epilogue warps 2..9: TMEM lane quarter q = warp % 4, column half h
        const int q = warp & 3;
        const int h = (warp - 2) >> 2;
        // a later K pass starts its chain from C (loads issued up front, their
        // latency hidden behind the first chunk's MMAs), so the chunk sums
        // add in the same order as one long pass
        const i64 row = (i64)m0 + 32 * q + lane;
        float acc[128];
        if (accumulate && row < m) {
            const float* cp = C + row + ((i64)n0 + h * 128) * ldc;
            const int ncol = (int)(n - n0 - h * 128 < 128 ? n - n0 - h * 128 : 128);
#pragma unroll
            for (int t = 0; t < 128; ++t) acc[t] = t < ncol ? __ldg(cp + t * ldc) : 0.f;
        } else {
#pragma unroll
            for (int t = 0; t < 128; ++t) acc[t] = 0.f;
        }
        for (int c = 0; c < nchunks; ++c) {
            const int b = c & 1;
            mbar_wait(&acc_full[b], (uint32_t)((c >> 1) & 1));
            tc_fence_after();
            const uint32_t base = tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)(b * TC_BN + h * 128);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                uint32_t v[32];
                tmem_ld_32x32b_x32(base + (uint32_t)(j * 32), v);
                tmem_ld_wait();
#pragma unroll
                for (int t = 0; t < 32; ++t) acc[j * 32 + t] += __uint_as_float(v[t]);
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&acc_empty[b]);
        }
        if (row < m) {
#pragma unroll
            for (int t = 0; t < 128; ++t) {
                const i64 col = (i64)n0 + h * 128 + t;
                if (col < n) C[row + col * ldc] = acc[t];
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) tmem_dealloc(tmem, 2 * TC_BN);
}

// the ahead-of-time kernels: plain stores
template <bool AMN, bool BMN>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(T2_THREADS, 1)
    gemm_3xtf32_pair_kernel(const __grid_constant__ TmapBytes tm_ahi, const __grid_constant__ TmapBytes tm_alo,
                            const __grid_constant__ TmapBytes tm_bhi, const __grid_constant__ TmapBytes tm_blo,
                            float* __restrict__ C, i64 m, i64 n, i64 ldc, int nk, int group_m, int kb0,
                            int accumulate, unsigned int* tile_ctr) {
    const Args none{};
    gemm_pair_body<PlainEpi, AMN, BMN>(tm_ahi, tm_alo, tm_bhi, tm_blo, C, m, n, ldc, nk, group_m, kb0, accumulate,
                                       none, 0, tile_ctr);
}

// lo = x - trunc_tf32(x) of a column-major rows x k matrix (ld), into a compact copy
// (ldl = rows rounded up to 4): the second operand of an MN-major 3xTF32 product, whose
// first is x itself (the tensor core truncates it).  No transpose: streamed at copy rate.
__global__ void __launch_bounds__(256) tf32_lo_kernel(const float* __restrict__ x, i64 ld, i64 rows, i64 k,
                                                       float* __restrict__ lo, i64 ldl) {
    const i64 nq = ldl / 4;                       // quads per column
    const i64 total = nq * k;
    for (i64 q = (i64)blockIdx.x * blockDim.x + threadIdx.x; q < total; q += (i64)gridDim.x * blockDim.x) {
        const i64 c = q / nq, r = (q - c * nq) * 4;
        float v[4];
        if (r + 3 < rows) {
            const float4 t = *reinterpret_cast<const float4*>(x + r + c * ld);
            v[0] = t.x; v[1] = t.y; v[2] = t.z; v[3] = t.w;
        } else {
#pragma unroll
            for (int e = 0; e < 4; ++e) v[e] = r + e < rows ? x[r + e + c * ld] : 0.f;
        }
        float4 o;
        float* op = &o.x;
#pragma unroll
        for (int e = 0; e < 4; ++e) op[e] = v[e] - __uint_as_float(__float_as_uint(v[e]) & 0xffffe000u);
        *reinterpret_cast<float4*>(lo + r + c * ldl) = o;
    }
}

template <bool TA, bool TB, int BM, int BK, int ST, bool VEC>
__global__ void __launch_bounds__(DmCfg<BM, BK, ST>::NW * 32, BM == 64 ? 2 : 1)
    gemm_dmma_kernel(const double* __restrict__ A, i64 lda, const double* __restrict__ B, i64 ldb,
                     double* __restrict__ C, i64 ldc, i64 m, i64 n, i64 k) {
    const Args none{};
    gemm_dmma_body<TA, TB, BM, BK, ST, VEC, PlainEpi>(A, lda, B, ldb, C, ldc, m, n, k, none);
}
}  // namespace bm

namespace bmi {

static_assert(sizeof(bm::TmapBytes) == sizeof(CUtensorMap), "tensor map size");

static int encode_kmajor(bm::TmapBytes* tmb, const float* p, int64_t kp, int64_t rows_p, int box_rows) {
    CUtensorMap* tm = reinterpret_cast<CUtensorMap*>(tmb);
    const cuuint64_t gdim[2] = {(cuuint64_t)kp, (cuuint64_t)rows_p};
    const cuuint64_t gstride[1] = {(cuuint64_t)(kp * 4)};
    const cuuint32_t box[2] = {TC_BK, (cuuint32_t)box_rows};
    const cuuint32_t estr[2] = {1, 1};
    CUresult r = drv().tensorMapEncodeTiled(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void*)p, gdim, gstride, box, estr,
                                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B,
                                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return cu_fail(r, "cuTensorMapEncodeTiled (gemm operand)");
    return BM_OK;
}

// an MN-major operand map: dims {rows (contiguous), k}, boxes of 32 rows x 16 K with the
// 128-B swizzle in 32-B atoms (bm_gemm_tc.cuh mn32_desc)
// as a 3-D map {32 rows, k, rows / 32} (strides ld * 4, 128 B) so one request moves the
// 4 row atoms of a 128-row tile (rows must be a multiple of 32: the caller pads)
static int encode_mn(bm::TmapBytes* tmb, const float* p, int64_t ld, int64_t rows, int64_t k) {
    CUtensorMap* tm = reinterpret_cast<CUtensorMap*>(tmb);
    const cuuint64_t gdim[3] = {32, (cuuint64_t)k, (cuuint64_t)((rows + 31) / 32)};
    const cuuint64_t gstride[2] = {(cuuint64_t)(ld * 4), 128};
    const cuuint32_t box[3] = {32, TC_BK, 4};
    const cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = drv().tensorMapEncodeTiled(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, (void*)p, gdim, gstride, box, estr,
                                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B,
                                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return cu_fail(r, "cuTensorMapEncodeTiled (gemm operand, MN-major)");
    return BM_OK;
}

// Which operands of a pair GEMM are read MN-major from the stored matrix: op(A) is M x K
// and MN-major when A is not transposed; op(B)^T is N x K and MN-major when B is.  TMA
// needs a 16-B base and a 16-B multiple row stride, and the 3-D map whole 32-row atoms
// (32 | m, 32 | n).  BM_GEMM_MN selects it (measured slower, off by default: DESIGN.md).
bool gemm_mn_enabled() {
    static const bool on = std::getenv("BM_GEMM_MN") && std::atoi(std::getenv("BM_GEMM_MN")) != 0;
    return on;
}

void pair_mn_modes(int ta, int tb, const float* A, int64_t lda, const float* B, int64_t ldb, int64_t m, int64_t n,
                   bool* amn, bool* bmn) {
    const bool on = gemm_mn_enabled();
    *amn = on && !ta && lda % 4 == 0 && m % 32 == 0 && ((uintptr_t)A & 15u) == 0;
    *bmn = on && tb && ldb % 4 == 0 && n % 32 == 0 && ((uintptr_t)B & 15u) == 0;
}

static int split_operand(const float* src, int64_t ld, bool kmajor, int64_t rows, int64_t k, float* hi, float* lo,
                         int64_t kp, int64_t rp) {
    const int tr = gemm_mn_enabled() ? 1 : 0;   // truncating split alongside in-place MN-major operands
    dim3 grid((unsigned)((kp + 63) / 64), (unsigned)((rp + 63) / 64));
    const bool vec = (ld % 4 == 0) && (((uintptr_t)src & 15u) == 0);
    if (kmajor) {
        if (vec) bm::split_tf32_kernel<true, true><<<grid, dim3(32, 8), 0, st().stream>>>(src, ld, rows, k, hi, lo, kp, rp, tr);
        else bm::split_tf32_kernel<true, false><<<grid, dim3(32, 8), 0, st().stream>>>(src, ld, rows, k, hi, lo, kp, rp, tr);
    } else {
        if (vec) bm::split_tf32_kernel<false, true><<<grid, dim3(32, 8), 0, st().stream>>>(src, ld, rows, k, hi, lo, kp, rp, tr);
        else bm::split_tf32_kernel<false, false><<<grid, dim3(32, 8), 0, st().stream>>>(src, ld, rows, k, hi, lo, kp, rp, tr);
    }
    BM_CUDA(cudaGetLastError());
    st().launches++;
    return BM_OK;
}

bool gemm_pair_persistent() {
    static const bool persist = !std::getenv("BM_GEMM_PERSIST") || std::atoi(std::getenv("BM_GEMM_PERSIST")) != 0;
    return persist;
}

// C = op(A) op(B) on the 3xTF32 tcgen05 path; split_a / split_b fill the
// K-major hi/lo copies of op(A) (m x k) and op(B)^T (n x k).
int gemm_tc_f32_core(int64_t m, int64_t n, int64_t k, const SplitFn& split_a, const SplitFn& split_b, float* C,
                     int64_t ldc, bool* handled, const PairEpilogue* epi, const MnOperand* a_mn,
                     const MnOperand* b_mn) {
    *handled = false;
    // CTA pairs (cta_group::2, 256 x 256 tiles) unless BM_GEMM_PAIR=0
    static const bool pair = !std::getenv("BM_GEMM_PAIR") || std::atoi(std::getenv("BM_GEMM_PAIR")) != 0;
    if (epi && !pair) return BM_OK;     // fused epilogues exist for the pair kernel only
    if (!pair) a_mn = b_mn = nullptr;   // the single-CTA kernel reads K-major copies only
    const int64_t tm_ = pair ? 2 * T2_BM : TC_BM, tn_ = pair ? 2 * T2_BNH : TC_BN;
    const int64_t mp = (m + tm_ - 1) / tm_ * tm_;
    const int64_t np = (n + tn_ - 1) / tn_ * tn_;
    const int64_t kp = (k + 31) / 32 * 32;   // split kernel tiles K by 32
    if ((mp / tm_) * (np / tn_) * (pair ? 2 : 1) > (1LL << 31) - 1) return BM_OK;
    cudaStream_t s = st().stream;
    float* buf = nullptr;
    // K-major operands: hi and lo copies, mp (np) x kp; MN-major ones: a lo copy only
    const int64_t lda_lo = a_mn ? (m + 3) / 4 * 4 : 0, ldb_lo = b_mn ? (n + 3) / 4 * 4 : 0;
    const int64_t a_elems = a_mn ? lda_lo * k : 2 * mp * kp, b_elems = b_mn ? ldb_lo * k : 2 * np * kp;
    constexpr int kMaxPasses = 64;     // tile counters of the persistent pairs, one per K pass
    BM_CUDA(cudaMallocAsync((void**)&buf, (size_t)((a_elems + b_elems) * 4 + kMaxPasses * 4 + 64), s));
    float* abuf = buf;
    float* bbuf = buf + (a_elems + 3) / 4 * 4;          // 16-B aligned
    unsigned int* ctr = reinterpret_cast<unsigned int*>(bbuf + (b_elems + 3) / 4 * 4);
    auto lo_pass = [&](const MnOperand* o, int64_t rows, float* lo, int64_t ldl) -> int {
        const int64_t quads = ldl / 4 * k;
        const int grid = (int)std::min<int64_t>((quads + 255) / 256, (int64_t)st().sm_count * 8);
        bm::tf32_lo_kernel<<<grid > 0 ? grid : 1, 256, 0, s>>>(o->p, o->ld, rows, k, lo, ldl);
        BM_CUDA(cudaGetLastError());
        st().launches++;
        return BM_OK;
    };
    bm::TmapBytes tm[4];
    int rc = BM_OK;
    if (a_mn) {
        rc = lo_pass(a_mn, m, abuf, lda_lo);
        if (!rc) rc = encode_mn(&tm[0], a_mn->p, a_mn->ld, m, k);
        if (!rc) rc = encode_mn(&tm[1], abuf, lda_lo, m, k);
    } else {
        rc = split_a(abuf, abuf + mp * kp, kp, mp);
        if (!rc) rc = encode_kmajor(&tm[0], abuf, kp, mp, TC_BM);
        if (!rc) rc = encode_kmajor(&tm[1], abuf + mp * kp, kp, mp, TC_BM);
    }
    if (!rc && b_mn) {
        rc = lo_pass(b_mn, n, bbuf, ldb_lo);
        if (!rc) rc = encode_mn(&tm[2], b_mn->p, b_mn->ld, n, k);
        if (!rc) rc = encode_mn(&tm[3], bbuf, ldb_lo, n, k);
    } else if (!rc) {
        rc = split_b(bbuf, bbuf + np * kp, kp, np);
        if (!rc) rc = encode_kmajor(&tm[2], bbuf, kp, np, pair ? T2_BNH : TC_BN);
        if (!rc) rc = encode_kmajor(&tm[3], bbuf + np * kp, kp, np, pair ? T2_BNH : TC_BN);
    }
    if (!rc && epi && (epi->amn != (a_mn != nullptr) || epi->bmn != (b_mn != nullptr)))
        rc = set_error(BM_ERR_ARG, "3xTF32 GEMM: epilogue kernel compiled for other operand layouts");
    if (!rc) {
        static bool attr = false;
        if (!attr) {
            cudaError_t e = cudaFuncSetAttribute(bm::gemm_3xtf32_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 TC_SMEM);
            if (e == cudaSuccess)
                e = cudaFuncSetAttribute(bm::gemm_3xtf32_pair_kernel<false, false>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, T2_SMEM);
            if (e == cudaSuccess)
                e = cudaFuncSetAttribute(bm::gemm_3xtf32_pair_kernel<true, false>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, T2_SMEM);
            if (e == cudaSuccess)
                e = cudaFuncSetAttribute(bm::gemm_3xtf32_pair_kernel<false, true>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, T2_SMEM);
            if (e == cudaSuccess)
                e = cudaFuncSetAttribute(bm::gemm_3xtf32_pair_kernel<true, true>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, T2_SMEM);
            if (e != cudaSuccess) rc = cuda_fail(e, "cudaFuncSetAttribute (3xTF32)");
            attr = true;
        }
    }
    if (!rc) {
        dim3 grid((unsigned)((np / tn_) * (mp / tm_) * (pair ? 2 : 1)));
        // Persistent CTA pairs (one per two SMs; BM_GEMM_PERSIST=0 turns them off) claiming
        // raster tiles from a global counter as they free up, with the next tile's MMAs
        // under this tile's epilogue: 0.5-1 % over one pair per tile after the barrier-scope
        // fix (8192^3 3.97-3.99 vs 4.00-4.01 ms, 16384^3 34.5-34.6 vs 34.6-35.0 ms).  (A
        // static share per pair -- tiles p, p + P, ... -- was 3-15 % slower: the pairs
        // drift apart along the raster and their operand slabs stop sharing L2.)
        const bool persist = gemm_pair_persistent();
        bool persistent = false;
        if (pair && persist && grid.x > (unsigned)(st().sm_count / 2 * 2)) {
            grid.x = (unsigned)(st().sm_count / 2 * 2);
            persistent = true;
            BM_CUDA(cudaMemsetAsync(ctr, 0, kMaxPasses * 4, s));
        }
        // tile rows per raster group (BM_GEMM_GROUP overrides): 8 single-CTA rows for the
        // single-CTA kernel; for the pair kernel see below
        static const int group_env = std::getenv("BM_GEMM_GROUP") ? std::atoi(std::getenv("BM_GEMM_GROUP")) : 0;
        // persistent pairs: 8 pair rows up to 8192 x 8192 outputs (4096^3..8192^3: 0.6-1 %
        // faster than 4, interleaved on one box), 4 above (16384^3: 1 %, 32768^3: 4 % faster
        // than 8; profiles/r02_gemm_group_sweep.txt); one pair per tile (BM_GEMM_PERSIST=0):
        // 4, as tuned for that launch shape
        const int group_m = group_env > 0 ? group_env
                                          : (pair ? (persistent && mp <= 8192 && np <= 8192 ? 8 : 4) : 8);
        // Long K runs as several stream-ordered passes of at most kpass K
        // (the later ones add into C): within one launch the resident CTAs
        // drift apart along K, and at K = 32768 their A/B slabs stop meeting
        // in L2 (4x the minimum DRAM reads, and the GPU power-throttles on
        // them); a pass restarts them together.  Measured: 32768^3 196 -> 218
        // TF/s with 8192-K passes; up to K = 16384 one pass is as fast.
        static const int64_t kpass_env = std::getenv("BM_GEMM_KPASS") ? std::atoll(std::getenv("BM_GEMM_KPASS")) : 8192;
        const int nk = (int)(kp / TC_BK);
        int pass_kb = kpass_env > 0 && kp > 2 * kpass_env ? (int)(kpass_env / (TC_BK * TC_CHUNK_KB)) * TC_CHUNK_KB : nk;
        if (pass_kb <= 0 || pass_kb >= nk) pass_kb = nk;
        if ((nk + pass_kb - 1) / pass_kb > kMaxPasses)
            pass_kb = ((nk + kMaxPasses - 1) / kMaxPasses + TC_CHUNK_KB - 1) / TC_CHUNK_KB * TC_CHUNK_KB;
        for (int kb0 = 0, pass = 0; kb0 < nk && !rc; kb0 += pass_kb, ++pass) {
            const int len = nk - kb0 < pass_kb ? nk - kb0 : pass_kb;
            unsigned int* tile_ctr = persistent ? ctr + pass : nullptr;
            if (epi) {
                // the JIT pair kernel: same geometry; the element-wise epilogue runs on the last K pass
                int64_t mm = m, nn = n, lc = ldc;
                int nkl = len, gm = group_m > 0 ? group_m : 8, k0 = kb0, acc = kb0 > 0, apply = kb0 + len >= nk;
                float* Cp = C;
                void* params[] = {&tm[0], &tm[1], &tm[2], &tm[3], &Cp, &mm, &nn, &lc, &nkl, &gm, &k0, &acc,
                                  const_cast<void*>(epi->args), &apply, &tile_ctr};
                CUresult cr = drv().launchKernel((CUfunction)epi->fn, grid.x, 1, 1, T2_THREADS, 1, 1,
                                                 epi->smem > 0 ? epi->smem : T2_SMEM, (CUstream)s,
                                                 params, nullptr);
                if (cr != CUDA_SUCCESS) {
                    rc = cu_fail(cr, "cuLaunchKernel (3xTF32 GEMM, fused epilogue)");
                    break;
                }
                st().launches++;
                continue;
            }
            if (pair) {
                const int gm = group_m > 0 ? group_m : 8;
                auto* kfn = a_mn ? (b_mn ? bm::gemm_3xtf32_pair_kernel<true, true> : bm::gemm_3xtf32_pair_kernel<true, false>)
                                 : (b_mn ? bm::gemm_3xtf32_pair_kernel<false, true> : bm::gemm_3xtf32_pair_kernel<false, false>);
                kfn<<<grid, T2_THREADS, T2_SMEM, s>>>(tm[0], tm[1], tm[2], tm[3], C, m, n, ldc, len, gm, kb0, kb0 > 0,
                                                      tile_ctr);
            }
            else
                bm::gemm_3xtf32_kernel<<<grid, TC_THREADS, TC_SMEM, s>>>(tm[0], tm[1], tm[2], tm[3], C, m, n, ldc, len,
                                                                          group_m > 0 ? group_m : 8, kb0, kb0 > 0);
            cudaError_t e = cudaGetLastError();
            if (e != cudaSuccess) rc = cuda_fail(e, "3xTF32 GEMM launch");
            else st().launches++;
        }
    }
    cudaFreeAsync(buf, s);
    if (!rc) *handled = true;
    return rc;
}

int gemm_tc_f32(int ta, int tb, int64_t m, int64_t n, int64_t k, const float* A, int64_t lda, const float* B,
                int64_t ldb, float* C, int64_t ldc, bool* handled, const PairEpilogue* epi) {
    *handled = false;
    if (m * n * k < (int64_t)1 << 21) return BM_OK;   // tiny: the SIMT kernel is cheaper than the split pass
    // op(A) is m x k; K-major iff A is stored transposed.  op(B) is k x n and we
    // need its N x K K-major form: K-major iff B is NOT transposed.  The MN-major ones
    // are read in place (pair_mn_modes); the K-major ones get hi/lo copies.
    bool amn, bmn;
    pair_mn_modes(ta, tb, A, lda, B, ldb, m, n, &amn, &bmn);
    if (epi) { amn = epi->amn; bmn = epi->bmn; }       // the modes the epilogue kernel was compiled for
    const MnOperand ao{A, lda}, bo{B, ldb};
    return gemm_tc_f32_core(
        m, n, k,
        [&](float* hi, float* lo, int64_t kp, int64_t rp) { return split_operand(A, lda, ta != 0, m, k, hi, lo, kp, rp); },
        [&](float* hi, float* lo, int64_t kp, int64_t rp) { return split_operand(B, ldb, tb == 0, n, k, hi, lo, kp, rp); },
        C, ldc, handled, epi, amn ? &ao : nullptr, bmn ? &bo : nullptr);
}

template <bool TA, bool TB, int BM, int BK, int ST, bool VEC>
static int dmma_go(int64_t m, int64_t n, int64_t k, const double* A, int64_t lda, const double* B, int64_t ldb,
                   double* C, int64_t ldc) {
    typedef bm::DmCfg<BM, BK, ST> G;
    dim3 grid((unsigned)((n + DM_BN - 1) / DM_BN), (unsigned)((m + BM - 1) / BM));
    if (grid.y > 65535) return set_error(BM_ERR_NOTIMPL, "gemm: too many row tiles");
    static bool attr = false;
    if (!attr) {
        BM_CUDA(cudaFuncSetAttribute(bm::gemm_dmma_kernel<TA, TB, BM, BK, ST, VEC>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, G::SMEM));
        attr = true;
    }
    bm::gemm_dmma_kernel<TA, TB, BM, BK, ST, VEC><<<grid, G::NW * 32, G::SMEM, st().stream>>>(A, lda, B, ldb, C, ldc,
                                                                                             m, n, k);
    BM_CUDA(cudaGetLastError());
    st().launches++;
    return BM_OK;
}

template <int BM, int BK, int ST, bool VEC>
static int dmma_launch(int ta, int tb, int64_t m, int64_t n, int64_t k, const double* A, int64_t lda,
                       const double* B, int64_t ldb, double* C, int64_t ldc) {
    if (ta) {
        if (tb) return dmma_go<true, true, BM, BK, ST, VEC>(m, n, k, A, lda, B, ldb, C, ldc);
        return dmma_go<true, false, BM, BK, ST, VEC>(m, n, k, A, lda, B, ldb, C, ldc);
    }
    if (tb) return dmma_go<false, true, BM, BK, ST, VEC>(m, n, k, A, lda, B, ldb, C, ldc);
    return dmma_go<false, false, BM, BK, ST, VEC>(m, n, k, A, lda, B, ldb, C, ldc);
}

int gemm_dmma_f64(int ta, int tb, int64_t m, int64_t n, int64_t k, const double* A, int64_t lda, const double* B,
                  int64_t ldb, double* C, int64_t ldc, bool* handled) {
    *handled = false;
    if (m * n * k < (int64_t)1 << 18) return BM_OK;
    // 16-byte pair copies need even extents/strides and 16-byte bases on the
    // contiguous operand(s)
    const bool vec = (ta || ((m | lda) % 2 == 0 && ((uintptr_t)A & 15) == 0)) &&
                     (!tb || ((n | ldb) % 2 == 0 && ((uintptr_t)B & 15) == 0));
    static const int variant = std::getenv("BM_DMMA_VARIANT") ? std::atoi(std::getenv("BM_DMMA_VARIANT")) : 0;
    int rc;
    switch (variant) {
        case 1: rc = dmma_launch<64, 16, 3, false>(ta, tb, m, n, k, A, lda, B, ldb, C, ldc); break;
        case 2: rc = vec ? dmma_launch<64, 32, 2, true>(ta, tb, m, n, k, A, lda, B, ldb, C, ldc)
                         : dmma_launch<64, 32, 2, false>(ta, tb, m, n, k, A, lda, B, ldb, C, ldc); break;
        case 3: rc = vec ? dmma_launch<64, 8, 6, true>(ta, tb, m, n, k, A, lda, B, ldb, C, ldc)
                         : dmma_launch<64, 8, 6, false>(ta, tb, m, n, k, A, lda, B, ldb, C, ldc); break;
        case 4: rc = vec ? dmma_launch<64, 16, 3, true>(ta, tb, m, n, k, A, lda, B, ldb, C, ldc)
                         : dmma_launch<64, 16, 3, false>(ta, tb, m, n, k, A, lda, B, ldb, C, ldc); break;
        case 5: rc = vec ? dmma_launch<64, 8, 8, true>(ta, tb, m, n, k, A, lda, B, ldb, C, ldc)
                         : dmma_launch<64, 8, 8, false>(ta, tb, m, n, k, A, lda, B, ldb, C, ldc); break;
        default: rc = vec ? dmma_launch<64, 16, 4, true>(ta, tb, m, n, k, A, lda, B, ldb, C, ldc)
                          : dmma_launch<64, 16, 4, false>(ta, tb, m, n, k, A, lda, B, ldb, C, ldc); break;
    }
    if (!rc) *handled = true;
    return rc;
}

}  // namespace bmi
