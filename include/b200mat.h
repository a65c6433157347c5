/*
 * b200mat.h -- C ABI of libb200mat.so, the B200 (sm_100a) device library that
 * replaces the simulated device underneath the reference's runtime firewall.
 *
 * The reference (`/root/reference/pkg/src/devmat`) routes every device
 * operation through `Runtime` (runtime.py:366-557).  Its operator ABI is
 *
 *     KernelInvocation(kind, inputs, output, scalars, params)   runtime.py:103-109
 *     FlatView(buf, offset, count, stride)                      runtime.py:84-90
 *     BlockView(buf, offset, rows, cols, lda)                   runtime.py:93-100
 *
 * and the entry points the expression layer calls are
 *
 *     Runtime.acquire_memory      runtime.py:428   -> bm_alloc
 *     Runtime.release             runtime.py:441   -> bm_free
 *     Runtime.release_deferred    runtime.py:449   -> bm_free_async
 *     Runtime.enqueue             runtime.py:469   -> bm_enqueue
 *     Runtime.execute_reduce      runtime.py:479   -> bm_execute_reduce
 *     Runtime.synchronise         runtime.py:476   -> bm_sync
 *     Runtime.copy_h2d            runtime.py:497   -> bm_h2d
 *     Runtime.copy_d2h            runtime.py:505   -> bm_d2h
 *     Runtime.copy_d2d            runtime.py:514   -> bm_d2d
 *     Runtime.read_elems          runtime.py:525   -> bm_read_elems
 *     Runtime.write_scalar        runtime.py:534   -> bm_write_elem
 *     runtime.init / shutdown     runtime.py:602,621 -> bm_init / bm_shutdown
 *
 * Everything here is plain C: device pointers are `void*`, sizes are
 * `int64_t`, every function returns a status code (BM_OK on success) and
 * the message of the last failure on the calling thread is available from
 * bm_last_error().  Errors raised asynchronously by a kernel are sticky and
 * surface at the next bm_sync(), which is the reference's contract
 * (runtime.py:340-353: async errors re-raised at synchronise).
 *
 * Element types follow kernels.py:28-35 (f32, f64, i32, u64); matrices are
 * column-major (element (r, c) at offset + r + c*lda).
 */
#ifndef B200MAT_H
#define B200MAT_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BM_ABI_VERSION 1

/* status codes */
#define BM_OK             0
#define BM_ERR_CUDA       1   /* CUDA runtime / driver failure (incl. sticky kernel faults) */
#define BM_ERR_ARG        2   /* malformed invocation or view out of bounds */
#define BM_ERR_NOTIMPL    3   /* kind / dtype combination not provided */
#define BM_ERR_EMPTY      4   /* min/max over an empty range (reference: ValueError, runtime.py:279-281) */
#define BM_ERR_JIT        5   /* NVRTC compilation of a fused program failed */
#define BM_ERR_NODEVICE   6   /* no CUDA device / not initialised */
#define BM_ERR_PEER       7   /* a peer rank never published into a cross-GPU exchange (device error
                                 word, raised at the next synchronisation point like the reference's
                                 asynchronous errors, runtime.py:340-353) */

/* element types (kernels.py:28-35) */
#define BM_F32 0
#define BM_F64 1
#define BM_I32 2
#define BM_U64 3

/* ---- invocation kinds (reference names in kernels.py:54-79, expr.py:467-484) ---- */
#define BM_K_EWISE           1   /* eop_*, eglue_*, fused_chain: one fused kernel per program   */
#define BM_K_REDUCE          2   /* reduce_accu/min/max/dot, optionally over a fused program      */
#define BM_K_RDIM            3   /* rdim_sum/min/max/mean/var over a 2-D block view               */
#define BM_K_GEMM            4   /* gemm (glue_times), with transpose flags folding op_htrans     */
#define BM_K_COPY            5   /* mov_copy (two-way conversion)                                  */
#define BM_K_TRANSPOSE       6   /* mov_transpose                                                  */
#define BM_K_FILL            7   /* gen_fill_const                                                 */
#define BM_K_EYE             8   /* gen_eye                                                        */
#define BM_K_LINSPACE        9   /* gen_linspace                                                   */
#define BM_K_RANDU          10   /* gen_randu (splitmix64 counter RNG, kernels.py:227-245)         */
#define BM_K_RANDN          11   /* gen_randn (Box-Muller, kernels.py:248-253)                     */
#define BM_K_STRIDED_COPY   12   /* mov_extract_strided / mov_insert_strided / resize / joins      */
#define BM_K_LOGISTIC_GRAD  13   /* fused single-pass logistic step: inputs X
                                    (block view, m x k f32), w (k), r (m, written), then the
                                    program's inputs 1..; program input 0 is X w; output g (k).
                                    iparams[0] = address of an f32 device slot that receives
                                    accu(r) in the reference's order (0: not wanted; needs
                                    m <= 2^26)                                                    */
#define BM_K_PRED_COUNT     14   /* pred_count / pred_all_any: matches of an element-vs-scalar test
                                    (ops.py:202-262, kernels.py:643-699); result u64 via
                                    bm_execute_reduce; iparams[0] = BM_CMP_*, threshold in scalars[0] */
#define BM_K_PRED_FIND      15   /* pred_find_build: ascending u64 linear indices of the matches   */
#define BM_K_GEMM_FUSED     16   /* glue_times over element-wise operands (f32, 3xTF32): each operand's
                                    program is evaluated inside the split pre-pass (expr.py:596-605
                                    lowers them to separate chains).  inputs: A's program inputs
                                    (iparams[0] of them), then B's; prog: A's stages (iparams[1]),
                                    then B's (loads relative to B's inputs); iparams[2], [3] = stored
                                    rows of A and B; [4..6] = m, n, k; output C (m x n)            */
#define BM_K_RDIM_FUSED     17   /* sum / mean / min / max over dim 0 or 1 of an element-wise program
                                    (expr.py:583-594 materialises it first): inputs = the program's
                                    flat inputs of rows * cols elements (column-major); dim = 0 / 1;
                                    iparams[0] = rows, iparams[1] = cols (dim 1); reduce_op =
                                    BM_R_ACCU / MIN / MAX / MEAN / VAR; output = cols (dim 0) or rows
                                    (dim 1) values of the compute dtype.  dim 1 takes 1-8 inputs of
                                    the compute dtype, 16-B aligned, rows * size % 16 == 0 (TMA)      */

#define BM_K_GEMM_EPI       18   /* glue_times consumed by an element-wise program (expr.py:596-605 +
                                    :611-657 lower them as a GEMM and a separate chain): C = F(op(A)
                                    op(B), ...) with F compiled into the GEMM's store (3xTF32 pair
                                    kernel / DMMA).  inputs: [0] A, [1] B (block views; trans_a /
                                    trans_b), [1 + j] program input j >= 1 (m * n elements each);
                                    program input 0 is the product; output C (contiguous m x n).
                                    One f32 input (f32 compute) is staged through shared memory when
                                    it has unit stride, a 16-byte base and 4 | m; otherwise the call
                                    runs as a GEMM into a temporary and the chain (same bits) */

/* comparison of a predicate (kernels.py:643-657 _predicate_mask) */
#define BM_CMP_GT 0
#define BM_CMP_LT 1
#define BM_CMP_GE 2
#define BM_CMP_LE 3
#define BM_CMP_EQ 4
#define BM_CMP_NE 5

/* program tags for BM_K_EWISE / BM_K_REDUCE (post-order, expr.py:611-657) */
#define BM_P_LOAD   0   /* push input[arg]                            */
#define BM_P_UNARY  1   /* x = op(x [, scalar[arg]])                   */
#define BM_P_SCALAR 2   /* x = op(x, scalar[arg])                      */
#define BM_P_GLUE   3   /* b = pop; a = pop; push op(a, b)             */

/* unary ops (kernels.py:54-58) */
#define BM_U_EXP 0
#define BM_U_LOG 1
#define BM_U_LOG10 2
#define BM_U_SQRT 3
#define BM_U_SQUARE 4
#define BM_U_POW 5
#define BM_U_ABS 6
#define BM_U_COS 7
#define BM_U_SIN 8
#define BM_U_TAN 9
#define BM_U_ACOS 10
#define BM_U_ASIN 11
#define BM_U_ATAN 12

/* scalar ops (kernels.py:59-62) */
#define BM_S_PLUS 0
#define BM_S_MINUS_PRE 1
#define BM_S_MINUS_POST 2
#define BM_S_TIMES 3
#define BM_S_DIV_PRE 4
#define BM_S_DIV_POST 5

/* glue ops (kernels.py:63) */
#define BM_G_PLUS 0
#define BM_G_MINUS 1
#define BM_G_SCHUR 2
#define BM_G_DIV 3

/* reductions (kernels.py:65-66) */
#define BM_R_NONE 0
#define BM_R_ACCU 1
#define BM_R_MIN 2
#define BM_R_MAX 3
#define BM_R_DOT 4   /* program leaves two values; their products are summed */
#define BM_R_MEAN 5  /* rdim only */
#define BM_R_VAR 6   /* rdim only */

/* strided-copy sub-kinds (kernels.py:68-72) */
#define BM_MOV_EXTRACT 0
#define BM_MOV_INSERT 1
#define BM_MOV_RESIZE 2
#define BM_MOV_RESHAPE 3
#define BM_MOV_JOIN_ROWS 4
#define BM_MOV_JOIN_COLS 5
#define BM_MOV_DIAGMAT 6
#define BM_MOV_DIAGVEC 7
#define BM_MOV_REPMAT 8

#define BM_MAX_INPUTS 16
#define BM_MAX_SCALARS 16
#define BM_MAX_PROG 64

/* A view into device memory.  Flat views (is_block == 0) mirror FlatView:
 * count elements at base + offset + i*stride.  Block views mirror BlockView:
 * rows x cols column-major at base + offset with leading dimension lda. */
typedef struct bm_view {
    void*   base;
    int64_t offset;
    int64_t count;
    int64_t stride;
    int64_t rows;
    int64_t cols;
    int64_t lda;
    int32_t dtype;
    int32_t is_block;
} bm_view;

/* One device operation -- the C image of KernelInvocation (runtime.py:103-109).
 * Scalars are carried twice: as double (float compute types; converted on the
 * device with round-to-nearest exactly like np.float32(k)) and as int64 (integer
 * compute types; the host performs int(k) with numpy's overflow rules,
 * kernels.py:280-283). */
typedef struct bm_invocation {
    int32_t kind;
    int32_t n_inputs;
    bm_view inputs[BM_MAX_INPUTS];
    int32_t has_output;
    bm_view output;
    int32_t n_scalars;
    double  fscalars[BM_MAX_SCALARS];
    int64_t iscalars[BM_MAX_SCALARS];
    int32_t n_prog;                       /* number of (tag, op, arg) triples */
    int32_t prog[3 * BM_MAX_PROG];
    int32_t compute_dtype;                /* dtype every stage is rounded to (kernels.py:270-277) */
    int32_t reduce_op;                    /* BM_R_* for BM_K_REDUCE / BM_K_RDIM */
    int32_t dim;                          /* rdim: 0 = per column, 1 = per row */
    int32_t trans_a;                      /* gemm: op(A) = A^T when 1 */
    int32_t trans_b;                      /* gemm: op(B) = B^T when 1 (folds op_htrans, expr.py:543-547) */
    int32_t sub_kind;                     /* BM_MOV_* for BM_K_STRIDED_COPY */
    int64_t iparams[8];                   /* kind-specific integers (rows for eye, n for linspace,
                                             seed/stream for RNG, diagonal k, ...) */
} bm_invocation;

/* ---- lifecycle / device ---------------------------------------------------------- */
int         bm_abi_version(void);
int         bm_device_count(int* count);
int         bm_init(int device);                  /* select device, create stream + pools */
int         bm_shutdown(void);                    /* drain, free everything still live   */
int         bm_device_info(char* name, int name_len, int* sm_count, int* cc_major,
                           int* cc_minor, int64_t* total_mem);
int         bm_set_stream(void* cuda_stream);     /* run on an external stream (NULL = own) */
void*       bm_get_stream(void);
const char* bm_last_error(void);

/* ---- memory (runtime.py:428-451) ---------------------------------------------------- */
int bm_alloc(int64_t bytes, void** out);          /* stream-ordered pool allocation */
int bm_free(void* p);                             /* immediate: waits for queued work first */
int bm_free_async(void* p);                       /* stream-ordered release (release_deferred) */

/* ---- transfers (runtime.py:497-540); synchronous like the reference -------------------- */
int bm_h2d(void* dst, const void* src, int64_t bytes);
int bm_d2h(void* dst, const void* src, int64_t bytes);
int bm_d2d(void* dst, const void* src, int64_t bytes);
int bm_h2d_async(void* dst, const void* src, int64_t bytes);   /* pinned host memory */
int bm_d2h_async(void* dst, const void* src, int64_t bytes);
int bm_read_elems(const void* base, int32_t dtype, const int64_t* idx, int64_t n, void* host_out);
int bm_write_elem(void* base, int32_t dtype, int64_t index, const void* host_value);
int bm_host_alloc_pinned(int64_t bytes, void** out);
int bm_host_free_pinned(void* p);

/* ---- queue (runtime.py:469-493) ------------------------------------------------------ */
int bm_enqueue(const bm_invocation* inv);
/* Enqueue a reducing invocation, wait, and copy its scalar result (result dtype =
 * input/compute dtype, like the reference's `.item()` of an in-dtype sum) to
 * host_result.  BM_ERR_EMPTY for min/max over nothing. */
int bm_execute_reduce(const bm_invocation* inv, void* host_result);
/* Reduce variant that leaves the block partial of this shard on the device for a
 * cross-GPU combine (multi-GPU column-block sharding): writes the
 * shard's combined partial (in the result dtype) to dev_result. */
int bm_reduce_to_device(const bm_invocation* inv, void* dev_result);
/* Deterministic combine of `count` partials already on the device in rank
 * order (combine_pairwise, kernels.py:380-392) -> host_result. */
int bm_combine_partials(const void* dev_partials, int64_t count, int32_t dtype,
                        int32_t reduce_op, void* host_result);
/* same fold, result left on the device (no host synchronisation) */
int bm_combine_partials_to_device(const void* dev_partials, int64_t count, int32_t dtype,
                                  int32_t reduce_op, void* dev_result);
/* ---- peer-memory exchange of the shard partials (replaces the NCCL all-gather of
 * ShardedReduction with one kernel over NVLink; one process per GPU) ----
 * bm_exchange_alloc: an exchange buffer of 2 parities x (world values + world flags)
 * 8-byte slots, zeroed, from cudaMalloc (IPC-exportable); its 64-byte IPC handle goes
 * to every peer (torch.distributed object all-gather), which maps it with
 * bm_exchange_open.  bm_exchange_combine (one kernel): writes this rank's partial into
 * slot `rank` of every rank's buffer (parity epoch & 1), publishes `epoch` in its flag
 * with release semantics at system scope, waits until every rank's flag in the local
 * buffer reaches `epoch`, then folds the world values in rank order like
 * bm_combine_partials_to_device into dev_result. */
int bm_exchange_alloc(int32_t world, void** dev_buffer, void* ipc_handle /* 64 bytes out */);
int bm_exchange_open(const void* ipc_handle, void** dev_buffer);
/* vector variants: a buffer whose per-rank slot holds `cap` 4-byte units (plus one
 * f32 scalar), opened / closed like the scalar one.  Each call is ONE kernel that writes
 * this rank's vector into every rank's buffer over peer memory, publishes `epoch`, waits
 * for every rank and folds in rank order -- the replacement of an NCCL all-gather of
 * one vector per rank and the dim-1 reduction over the gathered rows x world matrix
 * (dist.py gather_columns + sum/min/max(., 1)); `cap` must be the allocation's.
 *   bm_exchange_rows (config 2 dim-1 reductions): out[i] = x_0[i] op x_1[i]
 *     op ... -- left to right for BM_R_ACCU (the sum), numpy's NaN-propagating min / max.
 *   bm_exchange_gsum (config 5, the sample-sharded logistic step): g_out = the rank-order
 *     sum of the ranks' n f32 gradients, s_out = combine_pairwise(s_0 .. s_{world-1}) +
 *     0.0f (every rank's folded accu(r)).
 * A peer that never publishes sets BM_ERR_PEER at the next bm_sync. */
int bm_exchange_alloc_vec(int32_t world, int64_t cap, void** dev_buffer, void* ipc_handle /* 64 bytes out */);
int bm_exchange_rows(const void* dev_x, int64_t n, int32_t dtype, int32_t reduce_op,
                     void* const* peer_buffers /* host array */, int32_t world, int32_t rank, uint64_t epoch,
                     int64_t cap, void* dev_out);
int bm_exchange_gsum(const float* dev_g, int64_t n, const float* dev_s, void* const* peer_buffers /* host array */,
                     int32_t world, int32_t rank, uint64_t epoch, int64_t cap, float* dev_g_out, float* dev_s_out);
int bm_exchange_close(void* dev_buffer, int32_t opened /* 1: mapped peer buffer, 0: own */);
/* the reduction and the exchange in ONE kernel: like bm_reduce_to_device, but the
 * reduction's last CTA publishes the shard partial into every rank's exchange buffer,
 * waits for all and writes the folded world result to dev_result.  dev_peer_array is
 * a DEVICE array of the world buffer pointers (own buffer at [rank]).  Reductions
 * large enough for the separate fold kernels run the exchange in the final fold
 * kernel instead; an empty shard (accu / dot) publishes a zero. */
int bm_reduce_to_device_exchange(const bm_invocation* inv, void* dev_result, void* const* dev_peer_array,
                                 int32_t world, int32_t rank, uint64_t epoch);
int bm_exchange_combine(const void* dev_partial, void* const* peer_buffers /* host array, world entries */,
                        int32_t world, int32_t rank, uint64_t epoch, int32_t dtype, int32_t reduce_op,
                        void* dev_result);
int bm_sync(void);   /* drain the stream; BM_ERR_CUDA on a kernel fault, BM_ERR_PEER on an exchange timeout */
/* check (and clear) the device error word without draining, after the caller synchronised
 * the stream itself (e.g. torch.cuda.synchronize): BM_ERR_PEER when a peer timed out.  The
 * peer wait of every exchange is bounded by BM_EXCH_TIMEOUT_S (default 60 s). */
int bm_poll_device_error(void);
/* 1 while queued work has not finished on the library's stream, else 0 */
int bm_stream_busy(void);

/* ---- instrumentation -------------------------------------------------------------- */
typedef struct bm_counters {
    int64_t launches;        /* kernels launched by this library */
    int64_t jit_compiles;    /* fused programs compiled by NVRTC */
    int64_t jit_cache_hits;  /* fused programs found in memory / on-disk cubin cache */
    int64_t bytes_h2d;
    int64_t bytes_d2h;
} bm_counters;
int bm_get_counters(bm_counters* out);
/* directory for the on-disk cubin cache of fused programs (NULL/"" disables) */
int bm_set_cache_dir(const char* dir);
/* generate + NVRTC-compile the fused kernel of a BM_K_EWISE / BM_K_REDUCE
 * invocation without launching it (works without a GPU; warms the cache) */
int bm_jit_compile_only(const bm_invocation* inv);

/* ---- explicit entry points a non-Python FFI would bind directly ---------------------- */
/* C = op(A) * op(B); A, B, C column-major; dtype one of BM_F32 (3xTF32 on tcgen05),
 * BM_F64 (DMMA), BM_I32, BM_U64 (exact, wrapping). */
int bm_gemm(int32_t dtype, int32_t trans_a, int32_t trans_b, int64_t m, int64_t n, int64_t k,
            const void* a, int64_t lda, const void* b, int64_t ldb, void* c, int64_t ldc);
/* force a GEMM algorithm (0 = auto, 1 = tensor core, 2 = SIMT) -- for tests / ablation */
int bm_set_gemm_algo(int32_t algo);

#ifdef __cplusplus
}
#endif
#endif /* B200MAT_H */
