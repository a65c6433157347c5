// bm_lgrad.cuh -- single-pass fused logistic-regression gradient (SURVEY 8f
// rank 1, config 5): g = X^T F(X w, ...) reading X from HBM once, and the
// element-wise result r = F(X w, ...) as a side output.
//
// The reference runs this as three kernels and reads X twice: z = X@w
// (sgemv per panel), r = 1/(1+exp(0-z)) - y (fused chain), g = X.t()@r
// (mov_transpose + gemm), kernels.py:584-586,704-708.
//
// Layout.  X is column-major (m x k, lda).  Work is cut into slabs of 64 rows
// x all k columns.  TMA moves 2-D boxes of 64 rows (256 B, the inner extent
// that streams at full HBM rate; 64-B rows stream at a third of it,
// tools/tma2d_probe.cu) x 128 columns.  A slab of 64 x 1024 f32 is 256 KB --
// more than one SM holds -- so a CTA pair (cluster of 2: one TPC, so 74
// pairs tile all 148 SMs, where clusters of 4 fitted only 33 times) shares
// it: CTA q owns columns [512q, 512q + 512), four boxes per slab, which a
// producer warp streams through a 6-box ring.  Each compute warp owns 32
// columns inside one box; phase 1 moves its values from shared memory into
// registers, releases the box, and parks them in TMEM (tcgen05.st, 256
// columns per slab, two slabs), so boxes refill at once and phase 2 reads
// the slab back from TMEM.  Per slab:
//   phase 1  each CTA computes partial z over its columns (f32 chains as in
//            the reference's sgemv, partials added in f64; fixed order) and
//            pushes it into the peer's shared memory (st.async, completing
//            bytes on the peer's mbarrier -- no fence, no cluster barrier);
//            once it lands both CTAs sum the two partials in rank order
//            (identical z in both);
//            the program inputs of the next slab are loaded into registers;
//   chain    r_i = F(round_f32(z_i), y_i, ...) -- the fused element-wise
//            program, every stage rounded to f32 like the unfused plan;
//   phase 2  each CTA adds sum_i X_ic r_i for its columns: a lane holds
//            4-row quads of 16 columns, then a transpose-reduce across its
//            half-warp (15 shuffles) leaves each lane one column's f64
//            accumulator for the whole kernel.
// The loop is software-pipelined: while the partials of slab j + 1 travel,
// the CTA runs phase 2 of slab j.
// Slabs are dealt to clusters in consecutive pairs (pair p = slabs 2p, 2p+1,
// pairs round-robin), so every 128-row numpy leaf of r is produced by one
// cluster: with the accu side output on, warp 0 of CTA 0 runs numpy's eight
// interleaved accumulators over the pair's r values and writes the leaf sum
// (kernels.py:459-460; ndarray.sum's pairwise leaves), and lgrad_finish folds
// leaves -> 8192-row blocks -> combine_pairwise, so accu(r) costs no pass.
// Every cluster writes its k gradient partials and lgrad_finish folds them in
// cluster order: deterministic.
// Compiled by NVRTC with the program's functor E.
#pragma once
#include "bm_reduce.cuh"

namespace bm {

#ifndef LG_RB
#define LG_RB 64            // rows per slab (256 B of f32: full-rate TMA rows)
#endif
#define LG_BOXC 128         // columns per TMA box (32 KB)
#ifndef LG_CLUSTER
#define LG_CLUSTER 2        // CTAs per slab: a CTA pair is one TPC, so pairs tile all 148 SMs
#endif                      // (k > 1024: clusters of 4 / 8, set by the launcher through NVRTC)
#define LG_COLS 512                   // columns per CTA
#define LG_KMAX (LG_CLUSTER * LG_COLS)
#define LG_KMAX_ALL (8 * LG_COLS)     // clusters of up to 8 CTAs (the portable maximum): k <= 4096
#define LG_NB (LG_COLS / LG_BOXC)     // boxes per slab per CTA
#define LG_NBOX 6                     // ring of boxes (192 KB)
#define LG_BOX_BYTES (LG_RB * LG_BOXC * 4)
#define LG_STAGES (LG_NBOX / LG_NB)   // (launcher: ring bytes = LG_STAGES * LG_STAGE_BYTES)
#define LG_STAGE_BYTES (LG_NBOX * LG_BOX_BYTES / LG_STAGES)
#define LG_CW 32                      // columns per compute warp
#define LG_THREADS (LG_COLS / LG_CW * 32)   // compute threads (16 warps)
#define LG_BLOCK (LG_THREADS + 32)    // + one TMA producer warp
#define LG_TMEM_COLS 512              // two slabs x 64 values per thread parked in TMEM

struct alignas(64) LgTmap {
    unsigned long long v[16];   // CUtensorMap (128 B, opaque)
};

struct LgArgs {
    Args a;                     // program inputs 1.. (input 0 of the program is z), scalars
    LgTmap tmx;                 // X: dim0 = rows (contiguous), dim1 = columns
    const float* w;             // k
    float* r;                   // m (side output)
    double* gpart;              // clusters x k partials
    float* leaves;              // accu(r) side output: numpy leaf sums of the full blocks (nullptr: off)
    i64 m, k;
    i64 nslabs;
    i64 nleaves;                // 128-row leaves inside full 8192-row blocks
};

__device__ __forceinline__ unsigned lg_smem(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void lg_bar_init(unsigned long long* b, unsigned cnt) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(lg_smem(b)), "r"(cnt));
}
__device__ __forceinline__ void lg_expect_tx(unsigned long long* b, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(lg_smem(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void lg_arrive(unsigned long long* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(lg_smem(b)) : "memory");
}
// try_wait polled from a C++ loop: a branch loop inside inline asm hides the
// loop from the compiler's reconvergence analysis, which deadlocked a
// warp-specialised variant of this kernel (divergent producer lane + named
// barriers)
__device__ __forceinline__ void lg_wait(unsigned long long* b, unsigned parity) {
    unsigned ok;
    do {
        asm volatile(
            "{\n"
            ".reg .pred p;\n"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
            "selp.u32 %0, 1, 0, p;\n"
            "}\n"
            : "=r"(ok)
            : "r"(lg_smem(b)), "r"(parity)
            : "memory");
    } while (!ok);
}
// the same, acquiring at cluster scope: the bytes completing the phase were
// stored by peer CTAs (st.async)
__device__ __forceinline__ void lg_wait_cluster(unsigned long long* b, unsigned parity) {
    unsigned ok;
    do {
        asm volatile(
            "{\n"
            ".reg .pred p;\n"
            "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n"
            "selp.u32 %0, 1, 0, p;\n"
            "}\n"
            : "=r"(ok)
            : "r"(lg_smem(b)), "r"(parity)
            : "memory");
    } while (!ok);
}
__device__ __forceinline__ void lg_tma_2d(void* dst, const LgTmap* tm, int c0, int c1, unsigned long long* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            lg_smem(dst)),
        "l"(tm), "r"(c0), "r"(c1), "r"(lg_smem(bar))
        : "memory");
}
__device__ __forceinline__ unsigned lg_cluster_rank() {
    unsigned r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
// TMEM as a per-thread parking space: 32 f32 of this thread's lane at column
// offset `taddr` (32x32b shape: warp w owns lanes 32 (w % 4) .. + 31)
__device__ __forceinline__ void lg_tmem_st32(unsigned taddr, const float (&v)[32]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
        "{%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16, "
        "%17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32};" ::"r"(taddr),
        "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7]), "f"(v[8]), "f"(v[9]),
        "f"(v[10]), "f"(v[11]), "f"(v[12]), "f"(v[13]), "f"(v[14]), "f"(v[15]), "f"(v[16]), "f"(v[17]), "f"(v[18]),
        "f"(v[19]), "f"(v[20]), "f"(v[21]), "f"(v[22]), "f"(v[23]), "f"(v[24]), "f"(v[25]), "f"(v[26]), "f"(v[27]),
        "f"(v[28]), "f"(v[29]), "f"(v[30]), "f"(v[31])
        : "memory");
}
__device__ __forceinline__ void lg_tmem_ld32(unsigned taddr, float (&v)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
        "%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];\n"
        "tcgen05.wait::ld.sync.aligned;"
        : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]), "=f"(v[7]), "=f"(v[8]),
          "=f"(v[9]), "=f"(v[10]), "=f"(v[11]), "=f"(v[12]), "=f"(v[13]), "=f"(v[14]), "=f"(v[15]), "=f"(v[16]),
          "=f"(v[17]), "=f"(v[18]), "=f"(v[19]), "=f"(v[20]), "=f"(v[21]), "=f"(v[22]), "=f"(v[23]), "=f"(v[24]),
          "=f"(v[25]), "=f"(v[26]), "=f"(v[27]), "=f"(v[28]), "=f"(v[29]), "=f"(v[30]), "=f"(v[31])
        : "r"(taddr)
        : "memory");
}
__device__ __forceinline__ void lg_cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
template <class E>
__device__ void logistic_grad(const LgArgs& L) {
    extern __shared__ __align__(1024) char lg_raw[];
    char* ring = lg_raw + ((1024 - (lg_smem(lg_raw) & 1023)) & 1023);
    __shared__ unsigned long long full[LG_NBOX], empty[LG_NBOX];
    __shared__ unsigned long long zbar[2];                // the peer's z partial of a slab landed (by parity)
    __shared__ double zpart[2][LG_THREADS / 32][LG_RB];   // by slab parity
    __shared__ double zq_all[2][LG_CLUSTER][LG_RB];   // the cluster's partial z, by slab parity
    __shared__ __align__(16) float rs[2][LG_RB];
    __shared__ float ws[LG_COLS];
    __shared__ unsigned tmem_slot;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const unsigned q = lg_cluster_rank();
    const i64 cluster = blockIdx.x / LG_CLUSTER, nclusters = gridDim.x / LG_CLUSTER;
    // slab j of this cluster: pair cluster + (j / 2) * nclusters, half j % 2
    const i64 npairs = (L.nslabs + 1) / 2;
    const i64 pmine = npairs > cluster ? (npairs - cluster + nclusters - 1) / nclusters : 0;
    const i64 nmine = 2 * pmine - (((L.nslabs & 1) && pmine > 0 && cluster + (pmine - 1) * nclusters == npairs - 1) ? 1 : 0);
    auto slab_of = [&](i64 j) -> i64 { return 2 * (cluster + (j >> 1) * nclusters) + (j & 1); };
    const int col0 = (int)q * LG_COLS;                  // this CTA's first column
    for (int c = tid; c < LG_COLS; c += LG_BLOCK) ws[c] = (col0 + c < L.k) ? L.w[col0 + c] : 0.f;
    if (tid == 0) {
        for (int s = 0; s < LG_NBOX; ++s) {
            lg_bar_init(&full[s], 1);
            lg_bar_init(&empty[s], LG_BOXC / LG_CW);   // the compute warps reading the box
        }
        lg_bar_init(&zbar[0], 1);
        lg_bar_init(&zbar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&L.tmx) : "memory");
    }
    if (warp == 0) {                           // 2 slabs x 256 columns of TMEM
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(lg_smem(&tmem_slot)),
                     "r"(LG_TMEM_COLS)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    lg_cluster_sync();                         // the peer's zbar initialised before anyone pushes
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");

    // ---- producer warp: boxes (slab j, box b) in order through the 6-box ring
    if (warp == LG_THREADS / 32) {
        if (lane == 0) {
            const i64 nboxes = nmine * LG_NB;
            for (i64 i = 0; i < nboxes; ++i) {
                const int s = (int)(i % LG_NBOX);
                if (i >= LG_NBOX) lg_wait(&empty[s], (unsigned)(((i / LG_NBOX) - 1) & 1));
                const i64 j = i / LG_NB;
                const int b = (int)(i % LG_NB);
                const i64 slab = slab_of(j);
                lg_expect_tx(&full[s], LG_BOX_BYTES);
                lg_tma_2d(ring + s * LG_BOX_BYTES, &L.tmx, (int)(slab * LG_RB), col0 + b * LG_BOXC, &full[s]);
            }
        }
    } else {
        // ---- compute warps
        typename E::Pre pre;                   // chain inputs of the next slab (threads < LG_RB)
        double gacc = 0.0;                     // this lane's column (see phase 2)
        // Lane layout (LG_RB = 64): warp w owns columns 32 w .. 32 w + 31 (inside box
        // w / 4); half-warp hc = lane / 16 takes 16 of them, lane hl = lane % 16 rows
        // 4 hl .. 4 hl + 3, so every shared-memory read is one 16-byte row quad.
        static_assert(LG_RB == 64, "lane layout assumes 64-row slabs");
        const int hl = lane & 15, hc = lane >> 4;
        const int cw = LG_CW * warp + 16 * hc;     // this half-warp's first column (CTA-relative)
        const int bx = (LG_CW * warp) / LG_BOXC;   // the box holding them
        const int cb = cw - bx * LG_BOXC;          // ... and their offset in it
        // TMEM parking place: the warp's lane quarter, 64 columns per warp group of 4
        const unsigned tmem_me = tmem_slot + ((unsigned)(32 * (warp & 3)) << 16) + (unsigned)(64 * (warp >> 2));
        auto ldx4 = [&](int s, int c) -> float4 {
            return *reinterpret_cast<const float4*>(ring + s * LG_BOX_BYTES + c * (LG_RB * 4) + 16 * hl);
        };
        // phase 1 of slab j: an f32 chain per row over the half-warp's 16 columns
        // (the reference's z is an f32 sgemv); the two halves, the 16 warp
        // partials and the 2 CTA partials are added in f64 in a fixed order
        auto phase1 = [&](i64 j) {
            const i64 i = j * LG_NB + bx;
            const int s = (int)(i % LG_NBOX);
            lg_wait(&full[s], (unsigned)((i / LG_NBOX) & 1));
            float xs[64];                      // [column u][row h], parked in TMEM for phase 2
#pragma unroll
            for (int u = 0; u < 16; ++u) {
                const float4 x = ldx4(s, cb + u);
                xs[4 * u] = x.x;
                xs[4 * u + 1] = x.y;
                xs[4 * u + 2] = x.z;
                xs[4 * u + 3] = x.w;
            }
            __syncwarp();
            if (lane == 0) lg_arrive(&empty[s]);   // the box is free: its values are in registers
            const unsigned t = tmem_me + (unsigned)((j & 1) * 256);
            lg_tmem_st32(t, *reinterpret_cast<const float(*)[32]>(&xs[0]));
            lg_tmem_st32(t + 32, *reinterpret_cast<const float(*)[32]>(&xs[32]));
            float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
#pragma unroll
            for (int u = 0; u < 16; ++u) {
                const float w = ws[cw + u];
                a0 = __fmaf_rn(xs[4 * u], w, a0);
                a1 = __fmaf_rn(xs[4 * u + 1], w, a1);
                a2 = __fmaf_rn(xs[4 * u + 2], w, a2);
                a3 = __fmaf_rn(xs[4 * u + 3], w, a3);
            }
            const int par = (int)(j & 1);
            double d[4] = {(double)a0, (double)a1, (double)a2, (double)a3};
#pragma unroll
            for (int h = 0; h < 4; ++h) {
                const double o = __shfl_xor_sync(0xffffffffu, d[h], 16);
                if (hc == 0) zpart[par][warp][4 * hl + h] = d[h] + o;   // low half + high half
            }
            asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        };
        // publish this CTA's partial z of slab j: st.async into the peer's zq_all,
        // completing bytes on the peer's zbar[parity] (no fence, no cluster
        // barrier); its own copy is a plain local store.  Thread 0 posts the
        // expect_tx for the peer's bytes (the phase may see the bytes first: the
        // tx-count goes negative until then).  A slot is rewritten two slabs later
        // only after its reader published the slab in between, which the writer
        // had to receive first.
        auto publish = [&](i64 j) {
            const int par = (int)(j & 1);
            if (tid == 0) lg_expect_tx(&zbar[par], (LG_CLUSTER - 1) * LG_RB * 8);
            if (tid < LG_RB) {
                // balanced tree over the warp partials (fixed order, 4 levels deep)
                double t[LG_THREADS / 32];
#pragma unroll
                for (int w = 0; w < LG_THREADS / 32; ++w) t[w] = zpart[par][w][tid];
#pragma unroll
                for (int h = 1; h < LG_THREADS / 32; h <<= 1)
#pragma unroll
                    for (int w = 0; w + h < LG_THREADS / 32; w += 2 * h) t[w] = t[w] + t[w + h];
                zq_all[par][q][tid] = t[0];
#pragma unroll
                for (unsigned p = 1; p < LG_CLUSTER; ++p) {
                    const unsigned peer = (q + p) % LG_CLUSTER;
                    unsigned raddr, rbar;
                    asm("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(raddr) : "r"(lg_smem(&zq_all[par][q][tid])), "r"(peer));
                    asm("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rbar) : "r"(lg_smem(&zbar[par])), "r"(peer));
                    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f64 [%0], %1, [%2];" ::"r"(raddr),
                                 "d"(t[0]), "r"(rbar)
                                 : "memory");
                }
            }
        };
        // z of slab j (the partials in rank order, once the peer's bytes landed) and r
        auto chain = [&](i64 j) {
            const int par = (int)(j & 1);
            if (tid < LG_RB) {
                lg_wait_cluster(&zbar[par], (unsigned)((j >> 1) & 1));
                double z = zq_all[par][0][tid];
#pragma unroll
                for (unsigned p = 1; p < LG_CLUSTER; ++p) z = z + zq_all[par][p][tid];
                const i64 row = slab_of(j) * LG_RB + tid;
                float r = 0.f;
                if (row < L.m) {
                    r = E::at(L.a, pre, (float)z);
                    if (q == 0) L.r[row] = r;
                }
                rs[par][tid] = r;
            }
        };
        // phase 2 of slab j: the slab's values back from TMEM, each lane's 4-row
        // partial sums for its 16 columns, then a transpose-reduce across the 16
        // lanes of the half-warp (15 shuffles), after which lane l owns column
        // cw + (l & 15) (bit-reversed order: 8 b3 + 4 b2 + 2 b1 + b0)
        float lacc = 0.f;                      // numpy leaf accumulator (warp 0, lanes 0..7 of CTA 0)
        auto leaf = [&](i64 j) {
            const int par = (int)(j & 1);
            const i64 pair = slab_of(j) >> 1;
            if (pair >= L.nleaves) return;     // tail block: folded from r by lgrad_finish
            const int t = lane & 7;
            float acc = (j & 1) ? lacc : rs[par][t];
#pragma unroll
            for (int i = (j & 1) ? 0 : 1; i < LG_RB / 8; ++i) acc = acc + rs[par][8 * i + t];
            if (!(j & 1)) {
                lacc = acc;
                return;
            }
            // ((r0 + r1) + (r2 + r3)) + ((r4 + r5) + (r6 + r7))
            acc = acc + __shfl_down_sync(0xffffffffu, acc, 1);
            acc = acc + __shfl_down_sync(0xffffffffu, acc, 2);
            acc = acc + __shfl_down_sync(0xffffffffu, acc, 4);
            if (lane == 0) L.leaves[pair] = acc;
        };
        auto phase2 = [&](i64 j) {
            const int par = (int)(j & 1);
            if (L.leaves != nullptr && q == 0 && warp == 0) leaf(j);
            const float4 rr = *reinterpret_cast<const float4*>(&rs[par][4 * hl]);
            float xs[64];
            const unsigned t = tmem_me + (unsigned)((j & 1) * 256);
            lg_tmem_ld32(t, *reinterpret_cast<float(*)[32]>(&xs[0]));
            lg_tmem_ld32(t + 32, *reinterpret_cast<float(*)[32]>(&xs[32]));
            float v[16];
#pragma unroll
            for (int c = 0; c < 16; ++c) {
                float acc = xs[4 * c] * rr.x;
                acc = __fmaf_rn(xs[4 * c + 1], rr.y, acc);
                acc = __fmaf_rn(xs[4 * c + 2], rr.z, acc);
                v[c] = __fmaf_rn(xs[4 * c + 3], rr.w, acc);
            }
#pragma unroll
            for (int off = 8, n = 8; off >= 1; off >>= 1, n >>= 1) {
                const bool upper = (lane & off) != 0;
#pragma unroll
                for (int c = 0; c < n; ++c) {
                    const float send = upper ? v[c] : v[c + n];
                    const float keep = upper ? v[c + n] : v[c];
                    v[c] = keep + __shfl_xor_sync(0xffffffffu, send, off);
                }
            }
            gacc += (double)v[0];
        };

        // Software pipeline: the partials of slab j + 1 travel while this CTA
        // runs phase 2 of slab j.  Named barrier 1 spans the compute warps only
        // (the producer warp never joins).
        auto csync = [&]() { asm volatile("bar.sync 1, %0;" ::"n"(LG_THREADS) : "memory"); };
        if (nmine > 0) {
            if (tid < LG_RB) {
                const i64 row = slab_of(0) * LG_RB + tid;
                if (row < L.m) E::load(L.a, row, pre);
            }
            phase1(0);
            csync();
            publish(0);
        }
        for (i64 j = 0; j < nmine; ++j) {
            chain(j);
            if (j + 1 < nmine && tid < LG_RB) {   // y & co. of slab j + 1 into registers now
                const i64 row = slab_of(j + 1) * LG_RB + tid;
                if (row < L.m) E::load(L.a, row, pre);
            }
            if (j + 1 < nmine) phase1(j + 1);
            csync();                              // r of slab j and the z partials of slab j + 1
            if (j + 1 < nmine) publish(j + 1);
            phase2(j);
        }
        asm volatile("griddepcontrol.launch_dependents;" ::: "memory");   // lgrad_finish may get resident
        {
            const int c = col0 + cw + 8 * ((lane >> 3) & 1) + 4 * ((lane >> 2) & 1) + 2 * ((lane >> 1) & 1) + (lane & 1);
            if (c < L.k) L.gpart[cluster * L.k + c] = gacc;
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    lg_cluster_sync();                             // no CTA exits while its peer may still write its zq
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_slot), "r"(LG_TMEM_COLS)
                     : "memory");
}

}  // namespace bm
