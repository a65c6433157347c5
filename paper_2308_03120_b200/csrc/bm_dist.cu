// bm_dist.cu -- deterministic cross-shard combine for column-block sharded
// reductions.  Every rank reduces its shard to one partial
// (bm_reduce_to_device); the partials are all-gathered in rank order and
// folded here with combine_pairwise (kernels.py:380-392).  When every shard
// holds an aligned power-of-two run of REDUCE_BLOCK blocks this reproduces the
// single-device result bit for bit ("reduction order").
#include <type_traits>

#include "bm_internal.h"
#include "bm_reduce.cuh"

namespace bm {

template <typename A, int OP>
__global__ void __launch_bounds__(256) combine_kernel(const A* __restrict__ parts, int count, A* out, int normalise) {
    __shared__ A buf[2 * 2048];
    for (int i = threadIdx.x; i < count; i += blockDim.x) buf[i] = parts[i];
    __syncthreads();
    const A r = cta_combine_pairwise<A, OP>(buf, buf + 2048, count);
    if (threadIdx.x == 0) out[0] = normalise ? OpPlus::f(r, A(0)) : r;
}

}  // namespace bm

namespace bmi {

template <typename A, int OP>
static int run_combine(const void* parts, int64_t count, void* out, int normalise) {
    bm::combine_kernel<A, OP><<<1, 256, 0, st().stream>>>((const A*)parts, (int)count, (A*)out, normalise);
    BM_CUDA(cudaGetLastError());
    st().launches++;
    return BM_OK;
}

template <typename T>
static int combine_typed(const void* parts, int64_t count, int op, void* out) {
    const int norm = std::is_floating_point<T>::value ? 1 : 0;
    switch (op) {
        case BM_R_ACCU: return run_combine<T, 1>(parts, count, out, norm);
        case BM_R_MIN: return run_combine<T, 2>(parts, count, out, 0);
        case BM_R_MAX: return run_combine<T, 3>(parts, count, out, 0);
        case BM_R_DOT: return run_combine<typename bm::DotAcc<T>::type, 1>(parts, count, out, 0);
    }
    return set_error(BM_ERR_ARG, "combine: bad reduce op");
}

template <typename P, int OP, int UPB, bool NORM>
static int fold_typed(const void* parts, int64_t nitems, int64_t nfull, bool unit_mode, int chunk, int nchunks,
                      void* result) {
    void* scratch = st().fold_scratch;   // per initialised device (bm_init / bm_shutdown)
    const int smem = 2 * chunk * (int)sizeof(P);
    static bool attr = false;
    if (!attr) {
        BM_CUDA(cudaFuncSetAttribute(bm::fold_chunks_kernel<P, OP, UPB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     160 * 1024));
        attr = true;
    }
    bm::fold_chunks_kernel<P, OP, UPB><<<nchunks, 512, smem, st().stream>>>(
        (const P*)parts, nitems, nfull, unit_mode ? 1 : 0, chunk, (P*)scratch);
    BM_CUDA(cudaGetLastError());
    bm::fold_final_kernel<P, OP, NORM><<<1, 256, (nchunks + nchunks / 256 + 1) * (int)sizeof(P), st().stream>>>(
        (const P*)scratch, nchunks, (P*)result);
    BM_CUDA(cudaGetLastError());
    st().launches += 2;
    return BM_OK;
}

int launch_fold(int dtype, int op, const void* parts, int64_t nitems, int64_t nfull, bool unit_mode, int chunk,
                int nchunks, void* result) {
#define BM_FOLD(P, UPB, NORM)                                                                                     \
    switch (op) {                                                                                                  \
        case BM_R_ACCU: return fold_typed<P, 1, UPB, NORM>(parts, nitems, nfull, unit_mode, chunk, nchunks, result); \
        case BM_R_MIN: return fold_typed<P, 2, UPB, false>(parts, nitems, nfull, unit_mode, chunk, nchunks, result); \
        case BM_R_MAX: return fold_typed<P, 3, UPB, false>(parts, nitems, nfull, unit_mode, chunk, nchunks, result); \
    }
    if (op == BM_R_DOT) {
        if (dtype == BM_F32) return fold_typed<double, 1, 8, false>(parts, nitems, nfull, unit_mode, chunk, nchunks, result);
        if (dtype == BM_F64) return fold_typed<double, 1, 16, false>(parts, nitems, nfull, unit_mode, chunk, nchunks, result);
        if (dtype == BM_I32) return fold_typed<int, 1, 8, false>(parts, nitems, nfull, unit_mode, chunk, nchunks, result);
        return fold_typed<unsigned long long, 1, 16, false>(parts, nitems, nfull, unit_mode, chunk, nchunks, result);
    }
    switch (dtype) {
        // unit-mode items are half-units (bm_reduce.cuh PwHalf): 8 per block
        // for 4-byte types, 16 for 8-byte types
        case BM_F32: BM_FOLD(float, 8, true) break;
        case BM_F64: BM_FOLD(double, 16, true) break;
        case BM_I32: BM_FOLD(int, 8, false) break;
        case BM_U64: BM_FOLD(unsigned long long, 16, false) break;
    }
#undef BM_FOLD
    return set_error(BM_ERR_ARG, "fold: bad dtype/op");
}

int combine_partials(const void* parts, int64_t count, int dtype, int op, void* out) {
    if (count < 1 || count > 2048) return set_error(BM_ERR_ARG, "combine: partial count out of range");
    switch (dtype) {
        case BM_F32: return combine_typed<float>(parts, count, op, out);
        case BM_F64: return combine_typed<double>(parts, count, op, out);
        case BM_I32: return combine_typed<int>(parts, count, op, out);
        case BM_U64: return combine_typed<unsigned long long>(parts, count, op, out);
    }
    return set_error(BM_ERR_ARG, "combine: bad dtype");
}

}  // namespace bmi
