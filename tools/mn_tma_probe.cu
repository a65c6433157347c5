// mn_tma_probe.cu -- MN-major tf32 operands loaded by TMA with the 128-B swizzle in
// 32-B atoms (CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B) straight from column-major matrices,
// consumed by tcgen05.mma with descriptor layout type 1 (tools/mn_probe.cu variant 7):
// A (M x K, M contiguous, lda) and B (N x K, N contiguous, ldb), M = N = 128, K = 16 as
// two K = 8 MMAs.  A tile is 4 boxes of {32 MN, 16 K} (2 KB each): MN-atom stride 2 KB
// (LBO), 4-row K groups 512 B apart (SBO), the second MMA starts 1 KB in.  Prints the
// max error against the host product for both LBO/SBO assignments.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -I paper_2308_03120_b200/csrc \
//        -o tools/mn_tma_probe tools/mn_tma_probe.cu -lcuda && ./tools/mn_tma_probe
#include <cuda.h>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "bm_ptx.cuh"

using namespace bm;

struct alignas(64) Tmap { CUtensorMap m; };

__global__ void probe(const __grid_constant__ Tmap ta, const __grid_constant__ Tmap tb, float* C, int swap) {
    __shared__ __align__(1024) unsigned char sa[128 * 16 * 4];
    __shared__ __align__(1024) unsigned char sb[128 * 16 * 4];
    __shared__ uint64_t bar, mbar;
    __shared__ uint32_t tslot;
    const int tid = threadIdx.x;
    if (tid == 0) {
        mbar_init(&bar, 1);
        mbar_init(&mbar, 1);
        mbar_fence_init();
    }
    if (tid < 32) tmem_alloc(&tslot, 128);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tslot;
    if (tid == 0) {
        mbar_expect_tx(&bar, 2 * 128 * 16 * 4);
        for (int i = 0; i < 4; ++i) {
            tma_load_2d(sa + i * 2048, &ta.m, 32 * i, 0, &bar);
            tma_load_2d(sb + i * 2048, &tb.m, 32 * i, 0, &bar);
        }
    }
    mbar_wait(&bar, 0);
    tc_fence_after();
    if (tid == 0) {
        auto desc = [&](const void* p) {
            uint64_t d = 0;
            d |= (uint64_t)((smem_u32(p) & 0x3FFFFu) >> 4);
            const uint32_t lbo = swap ? 512u : 2048u, sbo = swap ? 2048u : 512u;
            d |= (uint64_t)(lbo >> 4) << 16;
            d |= (uint64_t)(sbo >> 4) << 32;
            d |= (uint64_t)1 << 46;
            d |= (uint64_t)1 << 61;          // layout type 1: 128-B swizzle, 32-B atoms
            return d;
        };
        const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | (1u << 15) | (1u << 16) |
                               ((uint32_t)(128 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
        mma_tf32(tmem, desc(sa), desc(sb), idesc, 0u);
        mma_tf32(tmem, desc(sa + 1024), desc(sb + 1024), idesc, 1u);
        mma_commit(&mbar);
    }
    __syncwarp();
    mbar_wait(&mbar, 0);
    tc_fence_after();
    if (tid < 128) {
        const int w = tid >> 5;
        for (int c0 = 0; c0 < 128; c0 += 32) {
            uint32_t v[32];
            tmem_ld_32x32b_x32(tmem + ((uint32_t)(32 * w) << 16) + (uint32_t)c0, v);
            tmem_ld_wait();
            for (int t = 0; t < 32; ++t) C[tid + (c0 + t) * 128] = __uint_as_float(v[t]);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (tid < 32) tmem_dealloc(tmem, 128);
}

static CUtensorMap make_map(float* p, int rows, int k, int ld) {
    CUtensorMap m;
    const cuuint64_t gdim[2] = {(cuuint64_t)rows, (cuuint64_t)k};
    const cuuint64_t gstride[1] = {(cuuint64_t)ld * 4};
    const cuuint32_t box[2] = {32, 16};
    const cuuint32_t estr[2] = {1, 1};
    CUresult r = cuTensorMapEncodeTiled(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, p, gdim, gstride, box, estr,
                                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B,
                                        CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) printf("encode failed: %d\n", (int)r);
    return m;
}

int main() {
    const int M = 128, K = 16, LD = 136;             // padded leading dimension (16-B multiple)
    std::vector<float> a(LD * K), b(LD * K), ref(M * M, 0.f), c(M * M);
    srand(3);
    for (auto& x : a) x = (float)(rand() % 7);
    for (auto& x : b) x = (float)(rand() % 7);
    for (int i = 0; i < M; ++i)
        for (int j = 0; j < M; ++j)
            for (int k = 0; k < K; ++k) ref[i + j * M] += a[i + k * LD] * b[j + k * LD];
    float *da, *db, *dc;
    cudaMalloc(&da, a.size() * 4);
    cudaMalloc(&db, b.size() * 4);
    cudaMalloc(&dc, c.size() * 4);
    cudaMemcpy(da, a.data(), a.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(db, b.data(), b.size() * 4, cudaMemcpyHostToDevice);
    Tmap ta{make_map(da, M, K, LD)}, tb{make_map(db, M, K, LD)};
    for (int swap = 0; swap < 2; ++swap) {
        cudaMemset(dc, 0, c.size() * 4);
        probe<<<1, 128>>>(ta, tb, dc, swap);
        cudaError_t e = cudaDeviceSynchronize();
        cudaMemcpy(c.data(), dc, c.size() * 4, cudaMemcpyDeviceToHost);
        double maxerr = 0, maxref = 0;
        for (int i = 0; i < M * M; ++i) {
            maxerr = std::max(maxerr, (double)std::fabs(c[i] - ref[i]));
            maxref = std::max(maxref, (double)std::fabs(ref[i]));
        }
        printf("TMA 128B_ATOM_32B + MMA type 1, %s: %s max|err| %.1f max|ref| %.1f  C[0..3]=%.0f %.0f %.0f %.0f ref %.0f %.0f %.0f %.0f\n",
               swap ? "LBO=512 (K group), SBO=2048 (MN atom)" : "LBO=2048 (MN atom), SBO=512 (K group)",
               cudaGetErrorString(e), maxerr, maxref, c[0], c[1], c[2], c[3], ref[0], ref[1], ref[2], ref[3]);
        if (e != cudaSuccess) return 1;
    }
    return 0;
}
