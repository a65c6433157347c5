// bm_reduce.cuh -- element-wise store and reduction kernels over an abstract
// element source (a plain buffer or a fused expression program), sm_100a.
//
// Summation order.  The reference sums a block with numpy's ndarray.sum
// (kernels.py:459-460), which is numpy's pairwise summation: segments of at
// most 128 elements use 8 interleaved accumulators, longer ones split at
// n/2 rounded down to a multiple of 8; the result is 0 + pairwise(n).  Blocks
// of REDUCE_BLOCK = 8192 elements (kernels.py:87) are then folded with
// combine_pairwise (kernels.py:380-392).  This file reproduces that order
// exactly, so f32/f64 accu is bit-identical to the reference for every
// element-wise program whose element values are bit-identical.
//
// Fast path for numpy leaves of 128 elements: a warp loads 8 rows of 512 B
// fully coalesced (16-B vectors), parks them in a padded shared tile (row
// pitch 544 B) and re-reads them transposed so that each lane owns some of
// the 8 interleaved accumulators of one leaf; the 34-unit pitch makes both
// the row writes and the transposed 8-B reads bank-conflict free.  Per warp
// that is one "half-unit" of 1024 f32 / 512 f64 elements, a balanced subtree
// of numpy's split of an 8192-element block.
#pragma once
#include "bm_common.cuh"

namespace bm {

#ifndef BM_TRACE
#define BM_TRACE(k)   // fold timing hook (tools/fold_micro.cu)
#endif

#define BM_MAXIN 16
#define BM_REDUCE_BLOCK 8192
#define LG_ACCU_MAX_BLOCKS 8192           // fused logistic step: accu(r) side output up to 2^26 rows
#define BM_TILE_PITCH 544
#define BM_TILE_BYTES (8 * BM_TILE_PITCH)   // one half-unit (8 rows of 512 B)
#ifndef BM_UNIT_UNROLL
#define BM_UNIT_UNROLL 4                 // rows of a pairwise unit loaded per batch
#endif

struct Args {
    const void* in[BM_MAXIN];   // element 0 of every input view
    i64 stride[BM_MAXIN];       // element stride of every input view
    void* out;                  // element 0 of the output view
    i64 out_stride;
    i64 n;                      // number of elements
    double fk[16];              // scalars for float compute types
    i64 ik[16];                 // scalars for integer compute types
    void* partials;             // per-CTA partials scratch
    unsigned int* ticket;       // last-CTA-done counter (reset by the last CTA)
    void* result;               // device slot for the final value
    i64 blocks;                 // number of REDUCE_BLOCK blocks (informational)
    int group;                  // reductions: 1 = unit mode, 0 = block mode
    int vec_ok;                 // all views contiguous and 16-B aligned
    int smem_bytes;             // dynamic shared memory of the launch
    int ext_fold;               // 1: leave the partials for the separate fold kernels
    int grab;                   // items a warp takes per counter fetch (dynamic scheduling)
    // fused cross-GPU combine (peer-memory exchange, b200mat.h bm_reduce_to_device_exchange):
    // exch_world > 1 makes the last CTA publish its partial to every rank and fold them all
    void* const* exch_peers;    // device array of the world exchange buffers
    int exch_world, exch_rank;
    unsigned long long exch_epoch;
    unsigned int* dev_err;      // mapped host error word (bm_sync raises when it is set)
    unsigned long long exch_timeout_ns;
};

// ---------------------------------------------------------------------------
// sources

template <typename T> struct BufSrc {
    typedef T value_type;
    const T* p;
    i64 s;
    __device__ __forceinline__ T at(i64 i) const { return p[i * s]; }
    template <int V> __device__ __forceinline__ void vec(i64 i, T (&v)[V]) const {
        if (sizeof(T) * V == 16) {
            const uint4 q = __ldg(reinterpret_cast<const uint4*>(p + i));
            const T* t = reinterpret_cast<const T*>(&q);
#pragma unroll
            for (int k = 0; k < V; ++k) v[k] = t[k];
        } else {
#pragma unroll
            for (int k = 0; k < V; ++k) v[k] = p[i + k];
        }
    }
};

// vector load of V elements of TI converted to T (16-B transactions)
template <typename T, typename TI, int V>
__device__ __forceinline__ void ld_cvt(const void* base, i64 i, T (&v)[V]) {
    const TI* p = reinterpret_cast<const TI*>(base) + i;
    if ((sizeof(TI) * V) % 16 == 0) {
#pragma unroll
        for (int q = 0; q < (int)(sizeof(TI) * V / 16); ++q) {
            const uint4 w = __ldg(reinterpret_cast<const uint4*>(p) + q);
            const TI* t = reinterpret_cast<const TI*>(&w);
#pragma unroll
            for (int k = 0; k < (int)(16 / sizeof(TI)); ++k) v[q * (16 / sizeof(TI)) + k] = cvt<T>(t[k]);
        }
    } else {
#pragma unroll
        for (int k = 0; k < V; ++k) v[k] = cvt<T>(p[k]);
    }
}
template <typename T, typename TI>
__device__ __forceinline__ T ld1(const void* base, i64 i, i64 s) {
    return cvt<T>(reinterpret_cast<const TI*>(base)[i * s]);
}

// vector store of V elements converted to TO
template <typename TO, typename T, int V>
__device__ __forceinline__ void st_cvt(void* base, i64 i, const T (&v)[V]) {
    TO* p = reinterpret_cast<TO*>(base) + i;
    if ((sizeof(TO) * V) % 16 == 0) {
#pragma unroll
        for (int q = 0; q < (int)(sizeof(TO) * V / 16); ++q) {
            uint4 w;
            TO* t = reinterpret_cast<TO*>(&w);
#pragma unroll
            for (int k = 0; k < (int)(16 / sizeof(TO)); ++k) t[k] = cvt<TO>(v[q * (16 / sizeof(TO)) + k]);
            reinterpret_cast<uint4*>(p)[q] = w;
        }
    } else {
#pragma unroll
        for (int k = 0; k < V; ++k) p[k] = cvt<TO>(v[k]);
    }
}

// ---------------------------------------------------------------------------
// element-wise store: out[i] = cast_out(E(i))   (kernels.py:429-454)

template <class E, typename TO>
__device__ __forceinline__ void ewise_store(const Args& a) {
    typedef typename E::T T;
    const i64 n = a.n;
    const i64 tid = (i64)blockIdx.x * blockDim.x + threadIdx.x;
    const i64 nthr = (i64)gridDim.x * blockDim.x;
    if (a.vec_ok) {
        constexpr int V = (16 / sizeof(T)) > (16 / sizeof(TO)) ? (16 / sizeof(T)) : (16 / sizeof(TO));
        const i64 nv = n / V;
        for (i64 j = tid; j < nv; j += nthr) {
            T v[V];
            E::template vec<V>(a, j * V, v);
            st_cvt<TO, T, V>(a.out, j * V, v);
        }
        for (i64 i = nv * V + tid; i < n; i += nthr)
            reinterpret_cast<TO*>(a.out)[i] = cvt<TO>(E::at(a, i));
    } else {
        for (i64 i = tid; i < n; i += nthr)
            reinterpret_cast<TO*>(a.out)[i * a.out_stride] = cvt<TO>(E::at(a, i));
    }
}

// ---------------------------------------------------------------------------
// numpy pairwise summation

// Half a unit: 8 rows of 512 B (8 numpy leaves of f32, 4 of f64; 1024 / 512
// elements).  A half-unit is a balanced subtree of the 8192-element block, so
// half-unit partials fold into block partials exactly like units do; halving
// the work item doubles the item count, which balances the persistent CTAs'
// warps (config 1: 16384 items over 2368 warps, 6.9 rounds
// instead of 3.5 -> 4).
template <typename T> struct PwHalf { static const int value = 32 * 8 * (16 / sizeof(T)); };

// numpy pairwise value of the 8 rows parked in `tile` (pitch BM_TILE_PITCH);
// returned in every lane.  8-byte transposed reads: for both element sizes
// the 32 lanes of one read cover all 32 banks twice (2 wavefronts, ideal).
template <typename T>
__device__ __forceinline__ T pw_half_tile(const char* tile) {
    const int lane = threadIdx.x & 31;
    if constexpr (sizeof(T) == 4) {
        // 8 leaves (rows) x 4 lanes; lane (c, q) owns accumulators 2q, 2q+1
        const int c = lane >> 2, q = lane & 3;
        const char* base = tile + c * BM_TILE_PITCH + q * 8;
        uint2 w = *reinterpret_cast<const uint2*>(base);
        T r0 = __uint_as_float(w.x), r1 = __uint_as_float(w.y);
#pragma unroll
        for (int i = 1; i < 16; ++i) {
            w = *reinterpret_cast<const uint2*>(base + i * 32);
            r0 = r0 + __uint_as_float(w.x);
            r1 = r1 + __uint_as_float(w.y);
        }
        T t = r0 + r1;                   // r[2q] + r[2q+1]
        t = t + warp_shfl_xor(t, 1);     // (r0+r1)+(r2+r3) | (r4+r5)+(r6+r7)
        t = t + warp_shfl_xor(t, 2);     // leaf (128)
        t = t + warp_shfl_xor(t, 4);     // 256
        t = t + warp_shfl_xor(t, 8);     // 512
        t = t + warp_shfl_xor(t, 16);    // 1024
        return t;
    } else {
        // 4 leaves (2 rows each) x 8 lanes; lane (c, j) owns accumulator j
        const int c = lane >> 3, j = lane & 7;
        const char* base = tile + 2 * c * BM_TILE_PITCH + j * 8;
        T r = *reinterpret_cast<const T*>(base);
#pragma unroll
        for (int i = 1; i < 16; ++i) r = r + *reinterpret_cast<const T*>(base + (i >> 3) * BM_TILE_PITCH + (i & 7) * 64);
        T t = r;
        t = t + warp_shfl_xor(t, 1);
        t = t + warp_shfl_xor(t, 2);
        t = t + warp_shfl_xor(t, 4);     // leaf (128)
        t = t + warp_shfl_xor(t, 8);     // 256
        t = t + warp_shfl_xor(t, 16);    // 512
        return t;
    }
}

// one warp-cooperative half-unit: 8 rows x (32 lanes x 16 B)
template <typename T, bool VEC, class S>
__device__ __forceinline__ T pw_half(const S& s, i64 off, char* tile) {
    constexpr int V = 16 / sizeof(T);
    constexpr int W = 32 * V;
    const int lane = threadIdx.x & 31;
    constexpr int UNR = BM_UNIT_UNROLL < 8 ? BM_UNIT_UNROLL : 8;
#pragma unroll
    for (int r0 = 0; r0 < 8; r0 += UNR) {
        T v[UNR][V];
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
            const int r = r0 + u;
            if constexpr (VEC) {
                s.template vec<V>(off + r * W + lane * V, v[u]);
            } else {
#pragma unroll
                for (int k = 0; k < V; ++k) v[u][k] = s.at(off + r * W + lane * V + k);
            }
        }
#pragma unroll
        for (int u = 0; u < UNR; ++u)
            *reinterpret_cast<uint4*>(tile + (r0 + u) * BM_TILE_PITCH + lane * 16) = *reinterpret_cast<const uint4*>(v[u]);
    }
    __syncwarp();
    const T res = pw_half_tile<T>(tile);
    __syncwarp();
    return res;
}

// rows of one half-unit, loaded (program evaluated) but not yet reduced
template <typename T> struct HalfRows { T v[8][16 / sizeof(T)]; };

template <typename T, class S>
__device__ __forceinline__ void half_load(const S& s, i64 off, HalfRows<T>& h) {
    constexpr int V = 16 / sizeof(T);
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int r = 0; r < 8; ++r) s.template vec<V>(off + r * 32 * V + lane * V, h.v[r]);
}

template <typename T>
__device__ __forceinline__ T half_reduce(const HalfRows<T>& h, char* tile) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int r = 0; r < 8; ++r)
        *reinterpret_cast<uint4*>(tile + r * BM_TILE_PITCH + lane * 16) = *reinterpret_cast<const uint4*>(h.v[r]);
    __syncwarp();
    const T res = pw_half_tile<T>(tile);
    __syncwarp();
    return res;
}

// balanced pairwise tree over `count` = 2^k consecutive half-units.  The
// binary-counter stack lives in registers (levels unrolled) and, on the
// vector path, the rows of half-unit u + 1 are loaded while half-unit u is
// reduced, so every warp keeps a half-unit of loads in flight.  Not inlined:
// its double-buffered rows must not raise the register budget of the
// reduction kernels' hot half-unit loop.
template <typename T, class S>
__device__ __noinline__ T pw_balanced(const S& s, i64 off, i64 count, char* tile, bool vec_ok) {
    constexpr i64 U = PwHalf<T>::value;
    constexpr int LV = 12;                        // register levels: count <= 4096
    if (count > (1 << LV) || !vec_ok) {
        T stk[24];
        int lvl[24];
        int sp = 0;
        for (i64 u = 0; u < count; ++u) {
            T v = vec_ok ? pw_half<T, true>(s, off + u * U, tile) : pw_half<T, false>(s, off + u * U, tile);
            int l = 0;
            while (sp > 0 && lvl[sp - 1] == l) { v = stk[sp - 1] + v; --sp; ++l; }
            stk[sp] = v; lvl[sp] = l; ++sp;
        }
        return stk[0];
    }
    T stk[LV + 1];
    HalfRows<T> cur, nxt;
    half_load<T>(s, off, cur);
    for (i64 u = 0; u < count; ++u) {
        if (u + 1 < count) half_load<T>(s, off + (u + 1) * U, nxt);
        T v = half_reduce<T>(cur, tile);
        // u's trailing one bits are the pending left subtrees v merges with
#pragma unroll
        for (int l = 0; l <= LV; ++l) {
            if (l < LV && ((u >> l) & 1)) {
                v = stk[l] + v;
            } else {
                stk[l] = v;
                break;
            }
        }
        cur = nxt;
    }
    int top = 0;
    while ((1ll << top) < count) ++top;
    T res = stk[0];
#pragma unroll
    for (int l = 1; l <= LV; ++l)
        if (l == top) res = stk[l];
    return res;
}

// numpy leaf: n < 8 sequential from 0; n <= 128 eight interleaved accumulators
template <typename T, class S>
__device__ __forceinline__ T pw_leaf(const S& s, i64 off, i64 n) {
    const int lane = threadIdx.x & 31;
    if (n < 8) {
        T r = 0;
        for (i64 i = 0; i < n; ++i) r = r + s.at(off + i);
        return r;
    }
    T acc = 0;
    const i64 body = n - (n % 8);
    if (lane < 8) {
        acc = s.at(off + lane);
        for (i64 i = 8; i < body; i += 8) acc = acc + s.at(off + i + lane);
    }
    const T a0 = __shfl_sync(0xffffffffu, acc, 0), a1 = __shfl_sync(0xffffffffu, acc, 1);
    const T a2 = __shfl_sync(0xffffffffu, acc, 2), a3 = __shfl_sync(0xffffffffu, acc, 3);
    const T a4 = __shfl_sync(0xffffffffu, acc, 4), a5 = __shfl_sync(0xffffffffu, acc, 5);
    const T a6 = __shfl_sync(0xffffffffu, acc, 6), a7 = __shfl_sync(0xffffffffu, acc, 7);
    T r = ((a0 + a1) + (a2 + a3)) + ((a4 + a5) + (a6 + a7));
    for (i64 i = body; i < n; ++i) r = r + s.at(off + i);
    return r;
}

// general numpy pairwise_sum over [off, off+n): explicit post-order walk of
// the split tree (no device recursion); balanced sub-trees of whole units
// take the coalesced fast path.  Warp-uniform control flow.
template <typename T, class S>
__device__ __noinline__ T pw_generic(const S& s, i64 off, i64 n, char* tile, bool vec_ok) {
    constexpr i64 U = PwHalf<T>::value;
    if (n <= 128) return pw_leaf<T>(s, off, n);
    i64 f_off[48], f_n[48];
    int f_state[48];  // 0 = unvisited, 1 = left pending, 2 = right pending
    T f_left[48];
    int sp = 0;
    f_off[0] = off; f_n[0] = n; f_state[0] = 0; sp = 1;
    T ret = 0;
    bool have = false;  // `ret` holds a finished child value for the top frame
    while (sp > 0) {
        const int t = sp - 1;
        if (have) {
            if (f_state[t] == 1) {
                f_left[t] = ret;
                f_state[t] = 2;
                i64 n2 = f_n[t] / 2;
                n2 -= n2 % 8;
                f_off[sp] = f_off[t] + n2; f_n[sp] = f_n[t] - n2; f_state[sp] = 0; ++sp;
                have = false;
            } else {
                ret = f_left[t] + ret;
                --sp;
            }
            continue;
        }
        const i64 nn = f_n[t];
        bool direct = nn <= 128;
        bool balanced = false;
        if (!direct && nn % U == 0) {
            const i64 c = nn / U;
            balanced = (c & (c - 1)) == 0;
        }
        if (direct || balanced) {
            ret = direct ? pw_leaf<T>(s, f_off[t], nn) : pw_balanced<T>(s, f_off[t], nn / U, tile, vec_ok);
            have = true;
            --sp;
            continue;
        }
        i64 n2 = nn / 2;
        n2 -= n2 % 8;
        f_state[t] = 1;
        f_off[sp] = f_off[t]; f_n[sp] = n2; f_state[sp] = 0; ++sp;
    }
    return ret;
}

// ---------------------------------------------------------------------------
// block partials for the flat reductions (one warp per REDUCE_BLOCK block)

template <typename T, class S>
__device__ __forceinline__ T block_accu(const S& s, i64 off, i64 len, char* tile, bool vec_ok) {
    if constexpr (is_float_t<T>::value) {
        if (len == BM_REDUCE_BLOCK) return pw_balanced<T>(s, off, BM_REDUCE_BLOCK / PwHalf<T>::value, tile, vec_ok);
        return pw_generic<T>(s, off, len, tile, vec_ok);
    } else {
        // integers wrap: any summation order gives the same bits
        const int lane = threadIdx.x & 31;
        T acc = 0;
        for (i64 i = lane; i < len; i += 32) acc = OpPlus::f(acc, s.at(off + i));
#pragma unroll
        for (int m = 16; m >= 1; m >>= 1) acc = OpPlus::f(acc, warp_shfl_xor(acc, m));
        return acc;
    }
}

template <typename T, bool IS_MAX, class S>
__device__ __forceinline__ T block_minmax(const S& s, i64 off, i64 len, bool vec_ok) {
    constexpr int V = 16 / sizeof(T);
    const int lane = threadIdx.x & 31;
    MinMaxAcc<T, IS_MAX> acc;
    if (vec_ok && len % (4 * 32 * V) == 0) {
        for (i64 i = lane * V; i < len; i += 4 * 32 * V) {
            T v[4][V];
#pragma unroll
            for (int u = 0; u < 4; ++u) s.template vec<V>(off + i + u * 32 * V, v[u]);
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
                for (int k = 0; k < V; ++k) acc.add(v[u][k]);
        }
    } else {
        for (i64 i = lane; i < len; i += 32) acc.add(s.at(off + i));
    }
    acc.warp_merge();
    return acc.result();
}

// dot partials accumulate in double for float inputs (the reference block
// partial is OpenBLAS sdot/ddot, kernels.py:471-472; parity is by tolerance)
template <typename T> struct DotAcc { typedef double type; };
template <> struct DotAcc<int> { typedef int type; };
template <> struct DotAcc<u64> { typedef u64 type; };

template <typename T, class S2>
__device__ __forceinline__ typename DotAcc<T>::type block_dot(const S2& s, i64 off, i64 len, bool vec_ok) {
    typedef typename DotAcc<T>::type A;
    constexpr int V = 16 / sizeof(T);
    const int lane = threadIdx.x & 31;
    A acc = 0;
    if (vec_ok && len % (4 * 32 * V) == 0) {
        A acc2 = 0;
        for (i64 i = lane * V; i < len; i += 4 * 32 * V) {
            T x[4][V], y[4][V];
#pragma unroll
            for (int u = 0; u < 4; ++u) s.template vec2<V>(off + i + u * 32 * V, x[u], y[u]);
            asm volatile("" ::: "memory");   // keep the eight loads in flight together
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
                for (int k = 0; k < V; ++k) {
                    if (u & 1) acc2 = OpPlus::f(acc2, OpTimes::f((A)x[u][k], (A)y[u][k]));
                    else acc = OpPlus::f(acc, OpTimes::f((A)x[u][k], (A)y[u][k]));
                }
        }
        acc = OpPlus::f(acc, acc2);
    } else {
        for (i64 i = lane; i < len; i += 32) {
            T x, y;
            s.at2(off + i, x, y);
            acc = OpPlus::f(acc, OpTimes::f((A)x, (A)y));
        }
    }
#pragma unroll
    for (int m = 16; m >= 1; m >>= 1) acc = OpPlus::f(acc, warp_shfl_xor(acc, m));
    return acc;
}

// ---------------------------------------------------------------------------
// combine_pairwise (kernels.py:380-392) over `cnt` values in shared memory,
// executed by the whole CTA.  Adjacent pairs, odd element carried.
template <typename A, int OP>
__device__ __forceinline__ A combine_op(A a, A b) {
    if (OP == 2) return py_min(a, b);
    if (OP == 3) return py_max(a, b);
    return OpPlus::f(a, b);
}
template <typename A, int OP>
__device__ A cta_combine_pairwise(A* v, A* w, int cnt) {
    // ping-pong between v and w; returns the folded value (valid in every thread)
    while (cnt > 1) {
        const int half = cnt >> 1;
        for (int i = threadIdx.x; i < half; i += blockDim.x) w[i] = combine_op<A, OP>(v[2 * i], v[2 * i + 1]);
        if ((cnt & 1) && threadIdx.x == 0) w[half] = v[cnt - 1];
        __syncthreads();
        A* t = v; v = w; w = t;
        cnt = half + (cnt & 1);
    }
    const A r = v[0];
    __syncthreads();
    return r;
}


// Device error word bits (State::err_*, surfaced by bm_sync / bm_poll_device_error).
#define BM_DEVERR_PEER_TIMEOUT 1u

// ---------------------------------------------------------------------------
// Cross-GPU exchange of one value per rank over peer memory, then the fold of
// the world values in rank order (combine_pairwise, kernels.py:380-392).
// Buffer layout of every rank, per parity (epoch & 1): [world values][world
// flags], 8-byte slots.  Thread 0 writes this rank's value into slot `rank`
// of every rank's buffer (NVLink stores), fences at system scope, releases
// the epoch in its flag of every buffer; then the CTA waits for every flag of
// its own buffer with acquire loads and folds.  A peer that has not published
// after timeout_ns sets BM_DEVERR_PEER_TIMEOUT in the mapped error word, which
// bm_sync turns into BM_ERR_PEER (the reference surfaces asynchronous device
// errors at synchronise, runtime.py:340-353); the slot keeps its stale value.
// Called by every thread of ONE CTA; v is read in thread 0; xv is shared
// scratch of >= 2 * world values.  Returns the world value (all threads).
template <typename P, int OP>
__device__ P exchange_fold(void* const* peers, int W, int R, unsigned long long ep, unsigned int* err,
                           unsigned long long timeout_ns, P v, P* xv) {
    __syncthreads();
    const size_t base = (size_t)(ep & 1) * 2 * W;
    if (threadIdx.x == 0) {
        for (int p = 0; p < W; ++p)
            *reinterpret_cast<P*>(reinterpret_cast<unsigned long long*>(peers[p]) + base + R) = v;
        __threadfence_system();   // the values land before any flag says so
        for (int p = 0; p < W; ++p) {
            unsigned long long* flag = reinterpret_cast<unsigned long long*>(peers[p]) + base + W + R;
            asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(flag), "l"(ep) : "memory");
        }
    }
    __syncthreads();
    unsigned long long* mine = reinterpret_cast<unsigned long long*>(peers[R]) + base;
    for (int p = threadIdx.x; p < W; p += blockDim.x) {
        unsigned long long f, t0, t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
        do {
            asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(f) : "l"(mine + W + p) : "memory");
            if (f >= ep) break;
            __nanosleep(64);
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        } while (t - t0 < timeout_ns);
        if (f < ep && err) atomicOr_system(err, BM_DEVERR_PEER_TIMEOUT);
        xv[p] = *reinterpret_cast<volatile P*>(mine + p);
    }
    __syncthreads();
    return cta_combine_pairwise<P, OP>(xv, xv + W, W);
}

// ---------------------------------------------------------------------------
// flat reduction kernel body.
//
// Work items are either the 1024/512-element pairwise half-units of every
// full REDUCE_BLOCK block ("unit mode": always for the float accu, and for the
// other ops when blocks are scarce) or whole blocks ("block mode"); the
// ragged tail block is one extra item.  One persistent CTA per SM; warps take
// runs of items from a global counter (reduce_flat).  Every item writes one
// partial to global scratch, and the last CTA to finish folds them (ticket):
// half-unit partials -> block values with numpy's balanced tree
// (stage_block_values), then the blocks with combine_pairwise
// (cta_fold_pairwise: balanced 256-groups per warp, the ragged rest and the
// group values level by level), chunk results streamed in order.
// No float atomics: the result is the reference's bits.

template <typename A, int OP>
struct Fold {
    // combine of two block partials (combine_pairwise op, kernels.py:779-798)
    __device__ static __forceinline__ A blocks(A a, A b) { return combine_op<A, OP>(a, b); }
    // combine of two unit partials inside one block (numpy's tree / ndarray.min)
    __device__ static __forceinline__ A units(A a, A b) {
        if (OP == 2) return np_min(a, b);
        if (OP == 3) return np_max(a, b);
        return OpPlus::f(a, b);
    }
};

// combine_pairwise over `count` values produced by get(i), streamed with a
// binary-counter stack; equals the reference's level-by-level fold.
template <typename A, int OP, class G>
__device__ __forceinline__ A stream_pairwise(i64 count, const G& get) {
    A stk[40];
    int lvl[40];
    int sp = 0;
    for (i64 i = 0; i < count; ++i) {
        A v = get(i);
        int l = 0;
        while (sp > 0 && lvl[sp - 1] == l) { v = Fold<A, OP>::blocks(stk[sp - 1], v); --sp; ++l; }
        stk[sp] = v; lvl[sp] = l; ++sp;
    }
    A v = stk[sp - 1];
    for (int k = sp - 2; k >= 0; --k) v = Fold<A, OP>::blocks(stk[k], v);
    return v;
}

// combine_pairwise (kernels.py:380-392) over n <= 256 values in shared memory,
// level by level in place (pairs, odd element carried), by one warp; the
// result is returned in every lane.
template <typename A, int OP>
__device__ __forceinline__ A warp_combine_pairwise(A* t, int n) {
    const int lane = threadIdx.x & 31;
    while (n > 1) {
        const int half = n >> 1;
        A r[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int i = lane + 32 * j;
            if (i < half) r[j] = Fold<A, OP>::blocks(t[2 * i], t[2 * i + 1]);
        }
        const A carry = t[n - 1];
        __syncwarp();
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int i = lane + 32 * j;
            if (i < half) t[i] = r[j];
        }
        if ((n & 1) && lane == 0) t[half] = carry;
        __syncwarp();
        n = half + (n & 1);
    }
    return t[0];
}

// combine_pairwise (kernels.py:380-392) over `cnt` values in shared memory,
// executed by the whole CTA; the result is valid in thread 0.
// combine_pairwise of n values equals the right-nested fold of balanced trees
// over the binary segments of n, so: every aligned group of
// 256 values is a balanced subtree folded by one warp (8 values per lane in
// registers, then a shuffle butterfly that keeps left/right operand order),
// the ragged tail (< 256 values) is folded level by level by one warp, and
// one warp folds the group values plus the tail value the same way (the
// tail is innermost, exactly like an appended leaf).  Two barriers instead
// of one per level.
// `scratch` holds at least cnt / 256 + 1 values; cnt <= 65535.
template <typename A, int OP>
__device__ A cta_fold_pairwise(A* v, A* scratch, int cnt) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int G = cnt >> 8, tail = cnt & 255;
    for (int g = warp; g < G; g += nw) {
        const A* p = v + g * 256 + lane * 8;
        A x[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) x[k] = p[k];
        const A b0 = Fold<A, OP>::blocks(Fold<A, OP>::blocks(x[0], x[1]), Fold<A, OP>::blocks(x[2], x[3]));
        const A b1 = Fold<A, OP>::blocks(Fold<A, OP>::blocks(x[4], x[5]), Fold<A, OP>::blocks(x[6], x[7]));
        A c = Fold<A, OP>::blocks(b0, b1);
#pragma unroll
        for (int m = 1; m < 32; m <<= 1) {
            const A o = warp_shfl_xor(c, m);
            c = (lane & m) ? Fold<A, OP>::blocks(o, c) : Fold<A, OP>::blocks(c, o);
        }
        if (lane == 0) scratch[g] = c;
    }
    if (tail && warp == nw - 1) {
        const A tv = warp_combine_pairwise<A, OP>(v + G * 256, tail);
        if (lane == 0) scratch[G] = tv;
    }
    __syncthreads();
    A res = A(0);
    if (warp == 0) res = warp_combine_pairwise<A, OP>(scratch, G + (tail ? 1 : 0));
    __syncthreads();
    return res;
}

// Block values of blocks [c0, c0 + cn) into buf.  Block mode: the item
// partials are the block values.  Unit mode: numpy's balanced tree over each
// block's UPB half-unit partials (kernels.py:459-460 via ndarray.sum), read
// with coalesced 16-B loads -- a vector holds VP consecutive partials of one
// block and the VPB lanes holding one block combine by shuffles (left/right
// operand order kept).  The ragged tail block is the last item partial.
// Executed by the whole CTA; the caller synchronises before reading buf.
template <typename P, int OP, int UPB>
__device__ __forceinline__ void stage_block_values(const P* parts, i64 c0, int cn, i64 nfull, i64 nitems,
                                                   bool unit_mode, P* buf) {
    if (!unit_mode) {
        for (int i = threadIdx.x; i < cn; i += blockDim.x) buf[i] = __ldcg(parts + (c0 + i));
        return;
    }
    constexpr int VP = 16 / (int)sizeof(P);
    constexpr int VPB = UPB / VP;
    static_assert(VPB >= 1 && VPB <= 32 && (32 % VPB) == 0, "block vectors must tile a warp");
    const int lane = threadIdx.x & 31;
    const i64 full_end = (c0 + cn < nfull) ? c0 + cn : nfull;
    const int nvec = full_end > c0 ? (int)((full_end - c0) * VPB) : 0;
    const uint4* pv = reinterpret_cast<const uint4*>(parts + c0 * UPB);
    constexpr int BATCH = 4;
    for (int base = 0; base < nvec; base += BATCH * (int)blockDim.x) {
        uint4 q[BATCH];
#pragma unroll
        for (int k = 0; k < BATCH; ++k) {
            const int j = base + (int)threadIdx.x + k * (int)blockDim.x;
            if (j < nvec) q[k] = __ldcg(pv + j);
        }
#pragma unroll
        for (int k = 0; k < BATCH; ++k) {
            const int j = base + (int)threadIdx.x + k * (int)blockDim.x;
            const P* t = reinterpret_cast<const P*>(&q[k]);
            P x;
            if constexpr (VP == 4) {
                x = Fold<P, OP>::units(Fold<P, OP>::units(t[0], t[1]), Fold<P, OP>::units(t[2], t[3]));
            } else {
                x = Fold<P, OP>::units(t[0], t[1]);
            }
#pragma unroll
            for (int m = 1; m < VPB; m <<= 1) {
                const P o = warp_shfl_xor(x, m);
                x = (lane & m) ? Fold<P, OP>::units(o, x) : Fold<P, OP>::units(x, o);
            }
            if (j < nvec && (lane % VPB) == 0) buf[j / VPB] = x;
        }
    }
    if (threadIdx.x == 0 && nfull >= c0 && nfull < c0 + cn && nitems > nfull * UPB) buf[nfull - c0] = __ldcg(parts + (nitems - 1));
}

// partial of one work item (a half-unit, a block or the ragged tail block),
// valid in every lane
template <typename T, int OP, class S>
__device__ __forceinline__ typename cond_t<OP == 4, typename DotAcc<T>::type, T>::type reduce_item(
    const S& s, i64 off, i64 len, char* tile, bool vec_ok, bool unit) {
    if constexpr (OP == 4) {
        return block_dot<T>(s, off, len, vec_ok);
    } else if constexpr (OP == 2 || OP == 3) {
        return block_minmax<T, OP == 3>(s, off, len, vec_ok);
    } else {
        if constexpr (is_float_t<T>::value) {
            if (unit) return vec_ok ? pw_half<T, true>(s, off, tile) : pw_half<T, false>(s, off, tile);
        }
        return block_accu<T>(s, off, len, tile, vec_ok);
    }
}

// Last-CTA fold of the item partials (ticket): unit partials -> block
// partials with numpy's balanced tree (UPB items per block), then the blocks
// with combine_pairwise.
template <typename T, int OP, int UPB>
__device__ void last_cta_fold(const Args& a, i64 nitems, i64 nfull, bool has_tail, bool unit_mode) {
    typedef typename DotAcc<T>::type DA;
    typedef typename cond_t<OP == 4, DA, T>::type P;   // partial type
    extern __shared__ __align__(16) char smem[];
    const i64 tail = has_tail ? 1 : 0;
    // Ticket: the barrier orders the CTA's partial stores before thread 0's
    // gpu-scope release (cumulative), the acq_rel atomic makes every CTA's
    // partials visible to the last one.  One fence per CTA, not per thread:
    // this sits on the critical path after the slowest CTA.  a.ticket[0] is
    // the ticket, a.ticket[1] the dynamic item counter; the last CTA resets both.
    __shared__ bool am_last;
    __syncthreads();
    BM_TRACE(0);
    if (threadIdx.x == 0) {
        unsigned prev;
        asm volatile("atom.add.acq_rel.gpu.u32 %0, [%1], 1;" : "=r"(prev) : "l"(a.ticket) : "memory");
        am_last = (prev == gridDim.x - 1);
    }
    __syncthreads();
    if (!am_last) return;
    if (a.ext_fold) {   // large reductions: folded by fold_chunks_kernel / fold_final_kernel
        if (threadIdx.x == 0) { a.ticket[0] = 0u; a.ticket[1] = 0u; }
        return;
    }
    BM_TRACE(1);
    // ---- final fold (last CTA) ----
    // Block partials are staged into shared memory with coalesced, independent
    // loads (all threads), one aligned power-of-two chunk of blocks at a time,
    // folded there with combine_pairwise; chunk results fold the same way.
    // (L2 loads, ordered after the other CTAs' stores by the acquire above)
    const P* parts = reinterpret_cast<const P*>(a.partials);
    const i64 nblocks = nfull + (tail ? 1 : 0);
    const int smem_vals = (int)(a.smem_bytes / sizeof(P));
    int chunk = 1;
    while (2 * chunk <= smem_vals) chunk <<= 1;
    chunk >>= 1;                                   // ping-pong halves
    P* buf = reinterpret_cast<P*>(smem);
    P* buf2 = buf + chunk;
    __shared__ P chunk_res[1024];
    const i64 nchunks = (nblocks + chunk - 1) / chunk;
    P r = P(0);
    for (i64 ck = 0; ck < nchunks; ++ck) {
        const i64 c0 = ck * chunk;
        const int cn = (int)((nblocks - c0) < chunk ? (nblocks - c0) : chunk);
        stage_block_values<P, OP, UPB>(parts, c0, cn, nfull, nitems, unit_mode, buf);
        __syncthreads();
        BM_TRACE(2);
        const P cr = cta_fold_pairwise<P, OP>(buf, buf2, cn);
        BM_TRACE(3);
        if (threadIdx.x == 0) chunk_res[ck] = cr;     // host guarantees nchunks <= 1024
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        // combine_pairwise over the chunk results (aligned power-of-two groups)
        r = stream_pairwise<P, OP>(nchunks, [&](i64 i) { return chunk_res[i]; });
    }
    if (threadIdx.x == 0) {
        P fin = r;
        if constexpr (OP == 1 && is_float_t<T>::value) fin = r + T(0);  // numpy: 0 + pairwise(...) (-0 -> +0)
        reinterpret_cast<P*>(a.result)[0] = fin;
        a.ticket[0] = 0u;
        a.ticket[1] = 0u;
        chunk_res[0] = fin;
    }
    if (a.exch_world > 1) {
        // the collective in the same kernel: publish this rank's partial, wait
        // for every rank's, fold in rank order (exchange_fold)
        __syncthreads();
        const P g = exchange_fold<P, OP>(a.exch_peers, a.exch_world, a.exch_rank, a.exch_epoch, a.dev_err,
                                         a.exch_timeout_ns, chunk_res[0], chunk_res + 1);
        if (threadIdx.x == 0) {
            P o = g;
            if constexpr (OP == 1 && is_float_t<T>::value) o = g + T(0);
            reinterpret_cast<P*>(a.result)[0] = o;
        }
    }
    BM_TRACE(4);
}

template <typename T, int OP, class S>
__device__ void reduce_flat(const Args& a, const S& s) {
    typedef typename DotAcc<T>::type DA;
    typedef typename cond_t<OP == 4, DA, T>::type P;   // partial type
    extern __shared__ __align__(16) char smem[];
    const int nw = blockDim.x >> 5;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    char* tile = smem + warp * BM_TILE_BYTES;
    const bool vec_ok = a.vec_ok != 0;
    const bool unit_mode = a.group != 0;          // group != 0: unit mode
    constexpr i64 UE = PwHalf<T>::value;          // elements per unit-mode item (half-unit)
    constexpr int UPB = BM_REDUCE_BLOCK / UE;     // items per block
    const i64 nfull = a.n / BM_REDUCE_BLOCK;      // full blocks
    const i64 tail = a.n - nfull * BM_REDUCE_BLOCK;
    const i64 nitems_full = unit_mode ? nfull * UPB : nfull;
    const i64 nitems = nitems_full + (tail ? 1 : 0);
    P* parts = reinterpret_cast<P*>(a.partials);
    // Dynamic item scheduling: a warp takes `grab` consecutive items at a
    // time; its first run is static, the rest come from a global counter,
    // fetched one run ahead so the atomic's latency hides behind the current
    // run.  A CTA that starts late (its SM still folding the previous
    // reduction) simply takes fewer runs.  `grab` keeps the counter below
    // about one atomic per 2 ns for light items (one input).
    const i64 G = a.grab > 0 ? a.grab : 1;
    const i64 nwarps_total = (i64)gridDim.x * nw;
    i64 run = (i64)blockIdx.x * nw + warp;
    while (run * G < nitems) {
        unsigned nxt = 0;
        if (lane == 0) nxt = atomicAdd(a.ticket + 1, 1u);
        const i64 i_end = (run + 1) * G < nitems ? (run + 1) * G : nitems;
        for (i64 item = run * G; item < i_end; ++item) {
            P v;
            if (item < nitems_full) {
                const i64 off = item * (unit_mode ? UE : BM_REDUCE_BLOCK);
                v = reduce_item<T, OP>(s, off, unit_mode ? UE : BM_REDUCE_BLOCK, tile, vec_ok, unit_mode);
            } else {
                v = reduce_item<T, OP>(s, nfull * BM_REDUCE_BLOCK, tail, tile, vec_ok, false);
            }
            if (lane == 0) parts[item] = v;
        }
        run = nwarps_total + (i64)__shfl_sync(0xffffffffu, nxt, 0);
    }
    // Programmatic dependent launch (bm_jit.cu launch_reduce): everything
    // above only read this launch's inputs and wrote this launch's scratch;
    // wait for the predecessor to complete before the ticket (the scratch
    // of the launch before that is this one's), then let the successor start
    // on the SMs this grid frees while its last CTA folds.
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    last_cta_fold<T, OP, UPB>(a, nitems, nfull, tail != 0, unit_mode);
}

// ---------------------------------------------------------------------------
// 3xTF32 split pre-pass (bm_gemm_tc.cu): hi = rna_tf32(x), lo = rna_tf32(x - hi)
// -- or, with `trunc` (BM_GEMM_MN=1, so that the MN-major in-place operands and these
// copies multiply the same values), hi = x truncated to tf32 (what the tensor core does
// with an fp32 operand) and lo = x - hi -- written K-major as out[r * kp + c] for
// r < rp (M or N), c < kp (K), zero-padded.  Round to nearest is the more accurate
// pair (8192^3 normwise error 1.2e-6 against 2.1e-6).  The source is read through `src.at(linear index)`: a plain
// matrix, or (GEMM prologue fusion) the JIT-compiled element-wise program of
// the operand, evaluated on the fly so the operand is never materialised.
// SRC_KMAJOR: op(X)(r, c) = X[c + r*ld]; otherwise X[r + c*ld].

__device__ __forceinline__ float tf32_rna(float x) {
    unsigned r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return __uint_as_float(r);
}

template <bool SRC_KMAJOR, bool VEC, class SRC>
__device__ __forceinline__ void split_tf32_body(const SRC& src, i64 ld, i64 rows, i64 k, float* __restrict__ hi,
                                                float* __restrict__ lo, i64 kp, i64 rp, bool trunc = false) {
    // 64 (r) x 64 (c) tile per 256-thread CTA, moved as float4 along the
    // source's contiguous dimension and written as float4 along K (kp is a
    // multiple of 32, so a quad that starts inside [0, kp) ends inside it)
    __shared__ float tile[64][65];   // [r][c]
    const i64 r0 = (i64)blockIdx.y * 64, c0 = (i64)blockIdx.x * 64;
    const int t = threadIdx.x + threadIdx.y * blockDim.x;
#pragma unroll
    for (int q = t; q < 1024; q += 256) {
        if (SRC_KMAJOR) {                              // X[c + r * ld]: contiguous along c
            const int rr = q >> 4, cc = (q & 15) * 4;
            const i64 r = r0 + rr, c = c0 + cc;
            float v[4] = {0.f, 0.f, 0.f, 0.f};
            if (r < rows) {
                bool done = false;
                if constexpr (VEC) {
                    if (c + 3 < k) {
                        src.template vec<4>(c + r * ld, v);
                        done = true;
                    }
                }
                if (!done) {
#pragma unroll
                    for (int e = 0; e < 4; ++e)
                        if (c + e < k) v[e] = src.at(c + e + r * ld);
                }
            }
#pragma unroll
            for (int e = 0; e < 4; ++e) tile[rr][cc + e] = v[e];
        } else {                                       // X[r + c * ld]: contiguous along r
            const int cc = q >> 4, rr = (q & 15) * 4;
            const i64 r = r0 + rr, c = c0 + cc;
            float v[4] = {0.f, 0.f, 0.f, 0.f};
            if (c < k) {
                bool done = false;
                if constexpr (VEC) {
                    if (r + 3 < rows) {
                        src.template vec<4>(r + c * ld, v);
                        done = true;
                    }
                }
                if (!done) {
#pragma unroll
                    for (int e = 0; e < 4; ++e)
                        if (r + e < rows) v[e] = src.at(r + e + c * ld);
                }
            }
#pragma unroll
            for (int e = 0; e < 4; ++e) tile[rr + e][cc] = v[e];
        }
    }
    __syncthreads();
#pragma unroll
    for (int q = t; q < 1024; q += 256) {
        const int rr = q >> 4, cc = (q & 15) * 4;
        const i64 r = r0 + rr, c = c0 + cc;
        if (r < rp && c < kp) {
            float4 h, l;
            float* hp = &h.x;
            float* lp = &l.x;
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const float x = tile[rr][cc + e];
                if (trunc) {
                    hp[e] = __uint_as_float(__float_as_uint(x) & 0xffffe000u);
                    lp[e] = x - hp[e];
                } else {
                    hp[e] = tf32_rna(x);
                    lp[e] = tf32_rna(x - hp[e]);
                }
            }
            *reinterpret_cast<float4*>(hi + r * kp + c) = h;
            *reinterpret_cast<float4*>(lo + r * kp + c) = l;
        }
    }
}

// ---------------------------------------------------------------------------
// External fold for large reductions: CTA k folds the aligned chunk k of
// block partials (combine_pairwise in shared memory), then one CTA folds the
// chunk results.  Equal to one combine_pairwise over all blocks (aligned
// power-of-two groups fold independently).

template <typename P, int OP, int UPB>
__global__ void __launch_bounds__(512) fold_chunks_kernel(const P* __restrict__ parts, i64 nitems, i64 nfull,
                                                          int unit_mode, int chunk, P* __restrict__ out) {
    extern __shared__ __align__(16) char smem[];
    P* buf = reinterpret_cast<P*>(smem);
    P* buf2 = buf + chunk;
    const i64 nblocks = nfull + (nitems > (unit_mode ? nfull * UPB : nfull) ? 1 : 0);
    const i64 c0 = (i64)blockIdx.x * chunk;
    const int cn = (int)((nblocks - c0) < chunk ? (nblocks - c0) : chunk);
    stage_block_values<P, OP, UPB>(parts, c0, cn, nfull, nitems, unit_mode != 0, buf);
    __syncthreads();
    const P r = cta_fold_pairwise<P, OP>(buf, buf2, cn);
    if (threadIdx.x == 0) out[blockIdx.x] = r;
}

struct ExchArgs {
    void* const* peers;   // device array of the world exchange buffers; world < 2: no exchange
    int world, rank;
    unsigned long long epoch;
    unsigned int* err;
    unsigned long long timeout_ns;
};

template <typename P, int OP, bool NORMALISE>
__global__ void __launch_bounds__(256) fold_final_kernel(const P* __restrict__ chunks, int n, P* __restrict__ result,
                                                         ExchArgs x) {
    // the chunk values are staged in shared memory and folded by the whole CTA
    // (cta_fold_pairwise: the same combine_pairwise order); one thread
    // streaming them costs ~135 ns per value (69 us for 512 chunks)
    extern __shared__ __align__(16) char fsm[];
    __shared__ P xv[2 * 64];
    P* buf = reinterpret_cast<P*>(fsm);
    for (int i = threadIdx.x; i < n; i += blockDim.x) buf[i] = chunks[i];
    __syncthreads();
    P r = cta_fold_pairwise<P, OP>(buf, buf + n, n);
    if (NORMALISE) r = r + P(0);
    if (x.world > 1) {   // sharded reduction: the exchange of the shard values in this kernel
        r = exchange_fold<P, OP>(x.peers, x.world, x.rank, x.epoch, x.err, x.timeout_ns, r, xv);
        if (NORMALISE) r = r + P(0);
    }
    if (threadIdx.x == 0) result[0] = r;
}

}  // namespace bm
