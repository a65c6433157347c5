// bm_dist.cu -- deterministic cross-shard combine for column-block sharded
// reductions.  Every rank reduces its shard to one partial
// (bm_reduce_to_device); the partials are all-gathered in rank order and
// folded here with combine_pairwise (kernels.py:380-392).  When every shard
// holds an aligned power-of-two run of REDUCE_BLOCK blocks this reproduces the
// single-device result bit for bit ("reduction order").
#include <cstring>
#include <type_traits>

#include "bm_internal.h"
#include "bm_reduce.cuh"

namespace bm {

struct PeerPtrs {
    void* p[64];
};

template <typename A, int OP>
__global__ void __launch_bounds__(256) combine_kernel(const A* __restrict__ parts, int count, A* out, int normalise) {
    __shared__ A buf[2 * 2048];
    for (int i = threadIdx.x; i < count; i += blockDim.x) buf[i] = parts[i];
    __syncthreads();
    const A r = cta_combine_pairwise<A, OP>(buf, buf + 2048, count);
    if (threadIdx.x == 0) out[0] = normalise ? OpPlus::f(r, A(0)) : r;
}

// One CTA: publish this rank's partial to every peer, wait for all, fold
// (exchange_fold, bm_reduce.cuh).
template <typename A, int OP>
__global__ void __launch_bounds__(256) exchange_combine_kernel(const A* __restrict__ partial, PeerPtrs peers, int world,
                                                               int rank, unsigned long long epoch, A* out,
                                                               int normalise, unsigned int* err,
                                                               unsigned long long timeout_ns,
                                                               void* const* dev_peers) {
    __shared__ A xv[2 * 64];
    __shared__ void* pp[64];
    for (int i = threadIdx.x; i < world; i += blockDim.x) pp[i] = dev_peers ? dev_peers[i] : peers.p[i];
    const A v = partial ? partial[0] : A(0);   // no partial: an empty shard contributes zero (accu / dot)
    const A r = exchange_fold<A, OP>(pp, world, rank, epoch, err, timeout_ns, v, xv);
    if (threadIdx.x == 0) out[0] = normalise ? OpPlus::f(r, A(0)) : r;
}

// ---------------------------------------------------------------------------
// Vector exchange over peer memory, folded in ONE kernel: the replacement of an
// NCCL all-gather of one vector per rank plus the dim-1 reduction over the
// gathered rows x world matrix (dist.gather_columns + sum/min/max(., 1)).
//   rows  (config 2 dim-1 reductions): out[i] = x_0[i] (op) x_1[i] ...
//         in rank order -- left to right for the sum (what the dim-1 reduction
//         of the gathered matrix computes), numpy's NaN-propagating min / max;
//   gsum  (config 5, the sample-sharded logistic step): the same sum over the
//         ranks' gradients, plus every rank's folded accu(r) combined with
//         combine_pairwise + 0.0f, as the scalar exchange does for a float accu.
// Buffer of every rank, per parity (epoch & 1): [world slots of `slot` bytes]
// [world u64 flags]; a slot holds the rank's vector and, for gsum, its f32
// scalar after it.  `cap` (bm_exchange_alloc_vec) sizes the slots in 4-byte
// units: a vector of n T plus the scalar needs n * sizeof(T) / 4 + 1 <= cap.

__host__ __device__ inline size_t vx_slot_bytes(long long cap) { return (size_t)((4 * (cap + 1) + 15) / 16 * 16); }
__host__ __device__ inline size_t vx_flags_off(int world, long long cap) { return (size_t)world * vx_slot_bytes(cap); }
__host__ __device__ inline size_t vx_parity_bytes(int world, long long cap) {
    return vx_flags_off(world, cap) + (size_t)world * 8;
}

template <typename T, int OP, bool SCALAR>
__global__ void __launch_bounds__(512) exchange_vec_kernel(const T* __restrict__ x, long long n,
                                                           const float* __restrict__ s, PeerPtrs peers, int W, int R,
                                                           unsigned long long ep, long long cap, T* __restrict__ out,
                                                           float* __restrict__ s_out, unsigned int* err,
                                                           unsigned long long timeout_ns) {
    __shared__ float xv[2 * 64];
    const size_t slot = vx_slot_bytes(cap);
    const size_t base = (size_t)(ep & 1) * vx_parity_bytes(W, cap);
    const size_t flags = vx_flags_off(W, cap);
    // publish: this rank's vector (and scalar) into slot R of every rank's buffer
    for (int p = 0; p < W; ++p) {
        char* dst = reinterpret_cast<char*>(peers.p[p]) + base + (size_t)R * slot;
        for (long long i = threadIdx.x; i < n; i += blockDim.x) reinterpret_cast<T*>(dst)[i] = x[i];
        if (SCALAR && threadIdx.x == 0) *reinterpret_cast<float*>(dst + (size_t)n * sizeof(T)) = s[0];
    }
    __threadfence_system();            // every value lands before any flag says so
    __syncthreads();
    if (threadIdx.x < W) {
        unsigned long long* flag =
            reinterpret_cast<unsigned long long*>(reinterpret_cast<char*>(peers.p[threadIdx.x]) + base + flags) + R;
        asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(flag), "l"(ep) : "memory");
    }
    // wait for every rank's flag in the own buffer
    const char* mine = reinterpret_cast<const char*>(peers.p[R]) + base;
    if (threadIdx.x < W) {
        const unsigned long long* flag = reinterpret_cast<const unsigned long long*>(mine + flags) + threadIdx.x;
        unsigned long long f, t0, t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
        do {
            asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(f) : "l"(flag) : "memory");
            if (f >= ep) break;
            __nanosleep(64);
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        } while (t - t0 < timeout_ns);
        if (f < ep && err) atomicOr_system(err, BM_DEVERR_PEER_TIMEOUT);
    }
    __syncthreads();
    for (long long i = threadIdx.x; i < n; i += blockDim.x) {
        auto at = [&](int p) { return *reinterpret_cast<const volatile T*>(mine + (size_t)p * slot + (size_t)i * sizeof(T)); };
        if constexpr (OP == 1) {
            T acc = at(0);
            for (int p = 1; p < W; ++p) acc = OpPlus::f(acc, at(p));
            out[i] = acc;
        } else {
            MinMaxAcc<T, OP == 3> mm;
            for (int p = 0; p < W; ++p) mm.add(at(p));
            out[i] = mm.result();
        }
    }
    if constexpr (SCALAR) {
        for (int p = threadIdx.x; p < W; p += blockDim.x)
            xv[p] = *reinterpret_cast<const volatile float*>(mine + (size_t)p * slot + (size_t)n * sizeof(T));
        __syncthreads();
        const float r = cta_combine_pairwise<float, 1>(xv, xv + W, W);
        if (threadIdx.x == 0) s_out[0] = OpPlus::f(r, 0.0f);
    }
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
                      void* result, const bm::ExchArgs& x) {
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
        (const P*)scratch, nchunks, (P*)result, x);
    BM_CUDA(cudaGetLastError());
    st().launches += 2;
    return BM_OK;
}

int launch_fold(int dtype, int op, const void* parts, int64_t nitems, int64_t nfull, bool unit_mode, int chunk,
                int nchunks, void* result, void* const* exch_peers, int exch_world, int exch_rank,
                unsigned long long exch_epoch) {
    bm::ExchArgs x;
    x.peers = exch_peers;
    x.world = exch_world;
    x.rank = exch_rank;
    x.epoch = exch_epoch;
    x.err = st().err_dev;
    x.timeout_ns = st().exch_timeout_ns;
#define BM_FOLD(P, UPB, NORM)                                                                                     \
    switch (op) {                                                                                                  \
        case BM_R_ACCU: return fold_typed<P, 1, UPB, NORM>(parts, nitems, nfull, unit_mode, chunk, nchunks, result, x); \
        case BM_R_MIN: return fold_typed<P, 2, UPB, false>(parts, nitems, nfull, unit_mode, chunk, nchunks, result, x); \
        case BM_R_MAX: return fold_typed<P, 3, UPB, false>(parts, nitems, nfull, unit_mode, chunk, nchunks, result, x); \
    }
    if (op == BM_R_DOT) {
        if (dtype == BM_F32) return fold_typed<double, 1, 8, false>(parts, nitems, nfull, unit_mode, chunk, nchunks, result, x);
        if (dtype == BM_F64) return fold_typed<double, 1, 16, false>(parts, nitems, nfull, unit_mode, chunk, nchunks, result, x);
        if (dtype == BM_I32) return fold_typed<int, 1, 8, false>(parts, nitems, nfull, unit_mode, chunk, nchunks, result, x);
        return fold_typed<unsigned long long, 1, 16, false>(parts, nitems, nfull, unit_mode, chunk, nchunks, result, x);
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

namespace bmi {

template <typename A, int OP>
static int run_exchange(const void* partial, void* const* peers, int world, int rank, unsigned long long epoch,
                        void* out, int normalise, void* const* dev_peers = nullptr) {
    bm::PeerPtrs pp;
    std::memset(&pp, 0, sizeof pp);
    if (!dev_peers)
        for (int i = 0; i < world; ++i) pp.p[i] = peers[i];
    bm::exchange_combine_kernel<A, OP><<<1, 256, 0, st().stream>>>((const A*)partial, pp, world, rank, epoch, (A*)out,
                                                                    normalise, st().err_dev, st().exch_timeout_ns,
                                                                    dev_peers);
    BM_CUDA(cudaGetLastError());
    st().launches++;
    return BM_OK;
}

template <typename T>
static int exchange_typed(const void* partial, void* const* peers, int world, int rank, unsigned long long epoch,
                          int op, void* out) {
    const int norm = std::is_floating_point<T>::value ? 1 : 0;
    switch (op) {
        case BM_R_ACCU: return run_exchange<T, 1>(partial, peers, world, rank, epoch, out, norm);
        case BM_R_MIN: return run_exchange<T, 2>(partial, peers, world, rank, epoch, out, 0);
        case BM_R_MAX: return run_exchange<T, 3>(partial, peers, world, rank, epoch, out, 0);
        case BM_R_DOT: return run_exchange<typename bm::DotAcc<T>::type, 1>(partial, peers, world, rank, epoch, out, 0);
    }
    return set_error(BM_ERR_ARG, "exchange: bad reduce op");
}

// An empty shard of a fused sharded accu / dot: no reduction kernel, but the
// rank still takes part in the exchange with a zero (peers wait for it).
int exchange_empty_shard(int dtype, int op, void* const* dev_peers, int world, int rank, unsigned long long epoch,
                         void* out) {
    const bool f = dtype == BM_F32 || dtype == BM_F64;
    if (op == BM_R_DOT) {
        if (f) return run_exchange<double, 1>(nullptr, nullptr, world, rank, epoch, out, 0, dev_peers);
        if (dtype == BM_I32) return run_exchange<int, 1>(nullptr, nullptr, world, rank, epoch, out, 0, dev_peers);
        return run_exchange<unsigned long long, 1>(nullptr, nullptr, world, rank, epoch, out, 0, dev_peers);
    }
    if (op != BM_R_ACCU) return set_error(BM_ERR_EMPTY, "reduction over an empty range");
    switch (dtype) {
        case BM_F32: return run_exchange<float, 1>(nullptr, nullptr, world, rank, epoch, out, 1, dev_peers);
        case BM_F64: return run_exchange<double, 1>(nullptr, nullptr, world, rank, epoch, out, 1, dev_peers);
        case BM_I32: return run_exchange<int, 1>(nullptr, nullptr, world, rank, epoch, out, 0, dev_peers);
        case BM_U64: return run_exchange<unsigned long long, 1>(nullptr, nullptr, world, rank, epoch, out, 0, dev_peers);
    }
    return set_error(BM_ERR_ARG, "exchange: bad dtype");
}

static int vx_check(int32_t world, int32_t rank, uint64_t epoch, int64_t n, int64_t elem_bytes, int64_t cap) {
    if (world < 1 || world > 64 || rank < 0 || rank >= world) return set_error(BM_ERR_ARG, "exchange: bad world/rank");
    if (epoch == 0) return set_error(BM_ERR_ARG, "exchange: epochs start at 1");
    if (n < 0 || cap < 0 || n * elem_bytes > 4 * cap)
        return set_error(BM_ERR_ARG, "exchange: vector longer than the buffer's capacity");
    return BM_OK;
}

static bm::PeerPtrs vx_peers(void* const* peer_buffers, int world) {
    bm::PeerPtrs pp;
    std::memset(&pp, 0, sizeof pp);
    for (int i = 0; i < world; ++i) pp.p[i] = peer_buffers[i];
    return pp;
}

template <typename T>
static int rows_typed(const void* x, int64_t n, int op, bm::PeerPtrs pp, int world, int rank, uint64_t epoch,
                      int64_t cap, void* out) {
    switch (op) {
        case BM_R_ACCU:
            bm::exchange_vec_kernel<T, 1, false><<<1, 512, 0, st().stream>>>(
                (const T*)x, (long long)n, nullptr, pp, world, rank, epoch, (long long)cap, (T*)out, nullptr,
                st().err_dev, st().exch_timeout_ns);
            break;
        case BM_R_MIN:
            bm::exchange_vec_kernel<T, 2, false><<<1, 512, 0, st().stream>>>(
                (const T*)x, (long long)n, nullptr, pp, world, rank, epoch, (long long)cap, (T*)out, nullptr,
                st().err_dev, st().exch_timeout_ns);
            break;
        case BM_R_MAX:
            bm::exchange_vec_kernel<T, 3, false><<<1, 512, 0, st().stream>>>(
                (const T*)x, (long long)n, nullptr, pp, world, rank, epoch, (long long)cap, (T*)out, nullptr,
                st().err_dev, st().exch_timeout_ns);
            break;
        default:
            return set_error(BM_ERR_ARG, "exchange rows: op must be accu (sum), min or max");
    }
    BM_CUDA(cudaGetLastError());
    st().launches++;
    return BM_OK;
}

}  // namespace bmi

extern "C" {

int bm_exchange_alloc(int32_t world, void** dev_buffer, void* ipc_handle) {
    using namespace bmi;
    BM_REQUIRE_INIT();
    if (world < 1 || world > 64) return set_error(BM_ERR_ARG, "exchange: world out of range");
    const size_t bytes = (size_t)2 * 2 * world * 8;
    BM_CUDA(cudaMalloc(dev_buffer, bytes));
    BM_CUDA(cudaMemset(*dev_buffer, 0, bytes));
    cudaIpcMemHandle_t h;
    BM_CUDA(cudaIpcGetMemHandle(&h, *dev_buffer));
    static_assert(sizeof(h) == 64, "IPC handle size");
    std::memcpy(ipc_handle, &h, sizeof h);
    return BM_OK;
}

int bm_exchange_alloc_vec(int32_t world, int64_t cap, void** dev_buffer, void* ipc_handle) {
    using namespace bmi;
    BM_REQUIRE_INIT();
    if (world < 1 || world > 64) return set_error(BM_ERR_ARG, "exchange: world out of range");
    if (cap < 0 || cap > (1 << 22)) return set_error(BM_ERR_ARG, "exchange: vector capacity out of range");
    const size_t bytes = 2 * bm::vx_parity_bytes(world, cap);
    BM_CUDA(cudaMalloc(dev_buffer, bytes));
    BM_CUDA(cudaMemset(*dev_buffer, 0, bytes));
    cudaIpcMemHandle_t h;
    BM_CUDA(cudaIpcGetMemHandle(&h, *dev_buffer));
    std::memcpy(ipc_handle, &h, sizeof h);
    return BM_OK;
}

int bm_exchange_gsum(const float* dev_g, int64_t n, const float* dev_s, void* const* peer_buffers, int32_t world,
                     int32_t rank, uint64_t epoch, int64_t cap, float* dev_g_out, float* dev_s_out) {
    using namespace bmi;
    BM_REQUIRE_INIT();
    if (int rc = bmi::vx_check(world, rank, epoch, n, 4, cap)) return rc;
    if (!dev_s || !dev_s_out || (n > 0 && (!dev_g || !dev_g_out))) return set_error(BM_ERR_ARG, "exchange: null buffer");
    std::lock_guard<std::recursive_mutex> lk(st().mu);
    bm::exchange_vec_kernel<float, 1, true><<<1, 512, 0, st().stream>>>(
        dev_g, (long long)n, dev_s, bmi::vx_peers(peer_buffers, world), world, rank, epoch, (long long)cap, dev_g_out,
        dev_s_out, st().err_dev, st().exch_timeout_ns);
    BM_CUDA(cudaGetLastError());
    st().launches++;
    return BM_OK;
}

int bm_exchange_rows(const void* dev_x, int64_t n, int32_t dtype, int32_t reduce_op, void* const* peer_buffers,
                     int32_t world, int32_t rank, uint64_t epoch, int64_t cap, void* dev_out) {
    using namespace bmi;
    BM_REQUIRE_INIT();
    const int64_t eb = dtype == BM_F64 || dtype == BM_U64 ? 8 : 4;
    if (int rc = bmi::vx_check(world, rank, epoch, n, eb, cap)) return rc;
    if (n > 0 && (!dev_x || !dev_out)) return set_error(BM_ERR_ARG, "exchange: null buffer");
    std::lock_guard<std::recursive_mutex> lk(st().mu);
    const bm::PeerPtrs pp = bmi::vx_peers(peer_buffers, world);
    switch (dtype) {
        case BM_F32: return bmi::rows_typed<float>(dev_x, n, reduce_op, pp, world, rank, epoch, cap, dev_out);
        case BM_F64: return bmi::rows_typed<double>(dev_x, n, reduce_op, pp, world, rank, epoch, cap, dev_out);
        case BM_I32: return bmi::rows_typed<int>(dev_x, n, reduce_op, pp, world, rank, epoch, cap, dev_out);
        case BM_U64: return bmi::rows_typed<unsigned long long>(dev_x, n, reduce_op, pp, world, rank, epoch, cap, dev_out);
    }
    return set_error(BM_ERR_ARG, "exchange: bad dtype");
}

int bm_exchange_open(const void* ipc_handle, void** dev_buffer) {
    using namespace bmi;
    BM_REQUIRE_INIT();
    cudaIpcMemHandle_t h;
    std::memcpy(&h, ipc_handle, sizeof h);
    BM_CUDA(cudaIpcOpenMemHandle(dev_buffer, h, cudaIpcMemLazyEnablePeerAccess));
    return BM_OK;
}

int bm_exchange_close(void* dev_buffer, int32_t opened) {
    using namespace bmi;
    BM_REQUIRE_INIT();
    if (opened) BM_CUDA(cudaIpcCloseMemHandle(dev_buffer));
    else BM_CUDA(cudaFree(dev_buffer));
    return BM_OK;
}

int bm_exchange_combine(const void* dev_partial, void* const* peer_buffers, int32_t world, int32_t rank,
                        uint64_t epoch, int32_t dtype, int32_t reduce_op, void* dev_result) {
    using namespace bmi;
    BM_REQUIRE_INIT();
    if (world < 1 || world > 64 || rank < 0 || rank >= world) return set_error(BM_ERR_ARG, "exchange: bad world/rank");
    if (epoch == 0) return set_error(BM_ERR_ARG, "exchange: epochs start at 1");
    std::lock_guard<std::recursive_mutex> lk(st().mu);
    switch (dtype) {
        case BM_F32: return exchange_typed<float>(dev_partial, peer_buffers, world, rank, epoch, reduce_op, dev_result);
        case BM_F64: return exchange_typed<double>(dev_partial, peer_buffers, world, rank, epoch, reduce_op, dev_result);
        case BM_I32: return exchange_typed<int>(dev_partial, peer_buffers, world, rank, epoch, reduce_op, dev_result);
        case BM_U64:
            return exchange_typed<unsigned long long>(dev_partial, peer_buffers, world, rank, epoch, reduce_op,
                                                      dev_result);
    }
    return set_error(BM_ERR_ARG, "exchange: bad dtype");
}

}  // extern "C"
