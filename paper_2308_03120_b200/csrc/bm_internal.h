// bm_internal.h -- state shared by the translation units of libb200mat.so.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <atomic>
#include <cstdint>
#include <functional>
#include <mutex>
#include <string>

#include "../../include/b200mat.h"

namespace bmi {

struct State {
    bool initialised = false;
    int device = -1;
    int sm_count = 0;
    cudaStream_t own_stream = nullptr;
    cudaStream_t stream = nullptr;     // current stream (own or external)
    // reduction scratch, double-buffered: consecutive reductions alternate so
    // that a launch overlapping its predecessor's final fold (programmatic
    // dependent launch) never touches the predecessor's partials or ticket
    void* partials[2] = {nullptr, nullptr};
    int64_t partials_cap = 0;          // capacity of each, in 8-byte entries
    void* fold_scratch = nullptr;      // chunk results of the separate fold kernels (8192 x 8 B)
    void* lg_scratch = nullptr;        // fused logistic step: gradient partials + accu leaves (stream-ordered reuse)
    int64_t lg_scratch_cap = 0;        // bytes
    // pending fused exchange for the next reduction (bm_reduce_to_device_exchange)
    void* const* exch_peers = nullptr;
    int exch_world = 0, exch_rank = 0;
    unsigned long long exch_epoch = 0;
    unsigned long long exch_timeout_ns = 60ull * 1000000000ull;   // BM_EXCH_TIMEOUT_S
    // device error word: pinned, mapped host memory that kernels set (atomicOr_system)
    // and every host synchronisation point checks (BM_ERR_PEER)
    unsigned int* err_host = nullptr;
    unsigned int* err_dev = nullptr;
    int flip = 0;                      // buffer of the next reduction
    unsigned int* ticket = nullptr;    // two last-CTA counters (at +0 and +32), zero between launches
    void* result = nullptr;            // device slot of the final value
    void* host_slot = nullptr;         // pinned 64 B for scalar results
    std::recursive_mutex mu;           // serialises stream use across host threads
    std::atomic<int64_t> launches{0};
    std::atomic<int64_t> jit_compiles{0};
    std::atomic<int64_t> jit_hits{0};
    std::atomic<int64_t> bytes_h2d{0};
    std::atomic<int64_t> bytes_d2h{0};
    int gemm_algo = 0;
};

State& st();

int set_error(int code, const std::string& msg);
int cuda_fail(cudaError_t e, const char* what);
int cu_fail(CUresult r, const char* what);
// after a stream synchronisation: BM_ERR_PEER (and clear) when a kernel set the device error word
int check_device_error(const char* what);

#define BM_CUDA(call)                                           \
    do {                                                        \
        cudaError_t _e = (call);                                \
        if (_e != cudaSuccess) return bmi::cuda_fail(_e, #call); \
    } while (0)

#define BM_REQUIRE_INIT()                                                          \
    do {                                                                           \
        if (!bmi::st().initialised)                                                \
            return bmi::set_error(BM_ERR_NODEVICE, "libb200mat: bm_init not called"); \
    } while (0)

inline int64_t dtype_size(int dt) { return (dt == BM_F32 || dt == BM_I32) ? 4 : 8; }
inline bool dtype_ok(int dt) { return dt >= 0 && dt <= 3; }

// driver entry points fetched through the runtime (no link-time libcuda dependency)
struct Driver {
    PFN_cuModuleLoadData_v2000 moduleLoadData = nullptr;
    PFN_cuModuleGetFunction_v2000 moduleGetFunction = nullptr;
    PFN_cuLaunchKernel_v4000 launchKernel = nullptr;
    PFN_cuLaunchKernelEx_v11060 launchKernelEx = nullptr;
    PFN_cuOccupancyMaxActiveClusters_v11070 occupancyMaxActiveClusters = nullptr;
    PFN_cuFuncSetAttribute_v9000 funcSetAttribute = nullptr;
    PFN_cuFuncGetAttribute_v2020 funcGetAttribute = nullptr;
    PFN_cuTensorMapEncodeTiled_v12000 tensorMapEncodeTiled = nullptr;
    bool ok = false;
};
Driver& drv();
int load_driver();

// launch helpers implemented per translation unit
int launch_ewise_or_reduce(const bm_invocation* inv, bool to_device, void* dev_result);
int launch_rdim(const bm_invocation* inv);
int launch_gemm(const bm_invocation* inv);
int launch_misc(const bm_invocation* inv);
int launch_pred_count(const bm_invocation* inv, void* dev_result);
int launch_pred_find(const bm_invocation* inv);
int launch_logistic_grad(const bm_invocation* inv);
int launch_gemm_fused(const bm_invocation* inv);
int launch_rdim_fused(const bm_invocation* inv);
// fills the K-major tf32 hi/lo copies (rp x kp) of one GEMM operand
typedef std::function<int(float* hi, float* lo, int64_t kp, int64_t rp)> SplitFn;
// a JIT-compiled pair kernel with a fused element-wise epilogue (bm_gemm_tc.cuh
// gemm_pair_body<EPI>, NVRTC entry bm_gemm_epi) and its program arguments
struct PairEpilogue {
    void* fn;            // CUfunction
    const void* args;    // bm::Args
    int smem = 0;        // the kernel's dynamic shared memory (0: T2_SMEM)
    bool amn = false;    // compiled for MN-major A / B operands (pair_mn_modes)
    bool bmn = false;
};
struct MnOperand {       // an operand read MN-major in place: the stored column-major matrix
    const float* p;
    int64_t ld;
};
void pair_mn_modes(int ta, int tb, const float* A, int64_t lda, const float* B, int64_t ldb, int64_t m, int64_t n,
                   bool* amn, bool* bmn);
bool gemm_mn_enabled();   // BM_GEMM_MN=1: MN-major in-place operands + truncating splits
int gemm_tc_f32_core(int64_t m, int64_t n, int64_t k, const SplitFn& split_a, const SplitFn& split_b, float* C,
                     int64_t ldc, bool* handled, const PairEpilogue* epi = nullptr, const MnOperand* a_mn = nullptr,
                     const MnOperand* b_mn = nullptr);
bool gemm_pair_persistent();   // BM_GEMM_PERSIST (default on): persistent CTA pairs (bm_gemm_tc.cu)
int gemm_tc_f32(int ta, int tb, int64_t m, int64_t n, int64_t k, const float* A, int64_t lda, const float* B,
                int64_t ldb, float* C, int64_t ldc, bool* handled, const PairEpilogue* epi = nullptr);
int launch_gemm_epi(const bm_invocation* inv);
int gemm_epi_compile_only(const bm_invocation* inv);
int gemm_fused_compile_only(const bm_invocation* inv);
int exchange_empty_shard(int dtype, int op, void* const* dev_peers, int world, int rank, unsigned long long epoch,
                         void* dev_out);
int combine_partials(const void* dev_partials, int64_t count, int dtype, int op, void* dev_out);
// exch_world > 1: the final fold kernel also runs the cross-GPU exchange (fused sharded reductions)
int launch_fold(int dtype, int op, const void* partials, int64_t nitems, int64_t nfull, bool unit_mode, int chunk,
                int nchunks, void* result, void* const* exch_peers = nullptr, int exch_world = 0, int exch_rank = 0,
                unsigned long long exch_epoch = 0);

// grid heuristics
inline int ewise_grid(int64_t n_vec_units) {
    int64_t g = (n_vec_units + 255) / 256;
    const int64_t cap = (int64_t)st().sm_count * 8;
    if (g > cap) g = cap;
    if (g < 1) g = 1;
    return (int)g;
}

}  // namespace bmi
