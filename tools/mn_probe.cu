// mn_probe.cu -- one tcgen05.mma kind::tf32 (cta_group::1, M = 128, N = 128, K = 8)
// with MN-major SWIZZLE_128B operands written by hand into shared memory, for
// variants of the smem descriptor (LBO / SBO / layout type) -- which one
// reproduces A^T B on the host.  GPU box:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -I paper_2308_03120_b200/csrc \
//        -o tools/mn_probe tools/mn_probe.cu && ./tools/mn_probe
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "bm_ptx.cuh"

using namespace bm;

// A: M x K (m contiguous), B: N x K (n contiguous); element (mn, kk) of a 128-wide
// MN-major SW128 tile: atom j = mn / 32 at j * atom_stride, row kk at kk * 128 B,
// 16-B chunk (mn % 32) / 4 XOR (kk % 8), word mn % 4
__device__ __forceinline__ int sw128_off(int mn, int kk, int atom_stride) {
    const int j = mn >> 5, w = mn & 31;
    const int chunk = (w >> 2) ^ (kk & 7);
    return j * atom_stride + kk * 128 + chunk * 16 + (w & 3) * 4;
}

__global__ void probe(const float* A, const float* B, float* C, int variant) {
    __shared__ __align__(1024) unsigned char sa[128 * 8 * 4 * 2];   // 4 atoms x 1 KB (8 rows) -- room for 2 KB stride
    __shared__ __align__(1024) unsigned char sb[128 * 8 * 4 * 2];   // (type-1 variants use 4 KB: 2 K groups x 2 KB)
    __shared__ uint64_t bar;
    __shared__ uint32_t tslot;
    const int tid = threadIdx.x;
    const int atom = (variant & 1) ? 2048 : 1024;
    for (int i = tid; i < 128 * 8; i += blockDim.x) {
        const int mn = i % 128, kk = i / 128;
        int off;
        if (variant == 4) {          // K-major, no swizzle: 8x16B core matrices, LBO (K) 128 B, SBO (MN) 256 B
            off = (mn >> 3) * 256 + (kk >> 2) * 128 + (mn & 7) * 16 + (kk & 3) * 4;
        } else if (variant == 5) {   // MN-major, no swizzle: 16 B (4 along MN) x 8 K rows; SBO (MN) 128 B, LBO (K) unused
            off = (mn >> 2) * 128 + (kk & 7) * 16 + (mn & 3) * 4;
        } else if (variant == 6) {   // K-major SWIZZLE_64B (the GEMM's layout): 64-B rows, 16-B chunk ^= (row >> 1) & 3
            off = mn * 64 + (((kk >> 2) ^ ((mn >> 1) & 3)) * 16) + (kk & 3) * 4;
        } else if (variant >= 7) {   // MN-major SWIZZLE_128B with 32-B atomicity (layout type 1):
            // 128-B rows of 32 MN elements per K index, 32-B chunks XORed with the K row
            // (7, 8: chunk ^= kk & 3; 9, 10: chunk ^= (kk >> 1) & 3), atoms of 4 K rows;
            // MN atoms 512 B apart, K atom groups 2048 B apart
            const int j = mn >> 5, w = mn & 31;
            const int swz = variant <= 8 ? (kk & 3) : ((kk >> 1) & 3);
            off = j * 512 + (kk >> 2) * 2048 + (kk & 3) * 128 + (((w >> 3) ^ swz) * 32) + (w & 7) * 4;
        } else {
            off = sw128_off(mn, kk, atom);
        }
        *reinterpret_cast<float*>(sa + off) = A[mn + kk * 128];
        *reinterpret_cast<float*>(sb + off) = B[mn + kk * 128];
    }
    if (tid == 0) {
        mbar_init(&bar, 1);
        mbar_fence_init();
    }
    if (tid < 32) tmem_alloc(&tslot, 128);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tslot;
    if (tid == 0) {
        auto desc = [&](const void* p) {
            uint64_t d = 0;
            d |= (uint64_t)((smem_u32(p) & 0x3FFFFu) >> 4);
            uint32_t lbo = (variant & 2) ? 1024u : (uint32_t)atom;   // variant bit 1: swap roles
            uint32_t sbo = (variant & 2) ? (uint32_t)atom : 1024u;
            uint32_t lt = 2;
            if (variant == 4) { lbo = 128; sbo = 256; lt = 0; }
            if (variant == 5) { lbo = 1024; sbo = 128; lt = 0; }
            if (variant == 6) { lbo = 16; sbo = 512; lt = 4; }
            if (variant >= 7) {          // type 1; 7, 9: LBO = MN atom stride; 8, 10: swapped
                lt = 1;
                const bool sw = (variant == 8 || variant == 10);
                lbo = sw ? 2048 : 512;
                sbo = sw ? 512 : 2048;
            }
            d |= (uint64_t)(lbo >> 4) << 16;
            d |= (uint64_t)(sbo >> 4) << 32;
            d |= (uint64_t)1 << 46;
            d |= (uint64_t)lt << 61;
            return d;
        };
        uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(128 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
        if (variant != 4 && variant != 6) idesc |= (1u << 15) | (1u << 16);   // MN-major: transpose A and B
        mma_tf32(tmem, desc(sa), desc(sb), idesc, 0u);
        mma_commit(&bar);
    }
    __syncwarp();
    mbar_wait(&bar, 0);
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

int main() {
    const int M = 128, N = 128, K = 8;
    std::vector<float> a(M * K), b(N * K), ref(M * N, 0.f), c(M * N);
    srand(1);
    for (auto& x : a) x = (float)(rand() % 7);
    for (auto& x : b) x = (float)(rand() % 7);
    for (int i = 0; i < M; ++i)
        for (int j = 0; j < N; ++j)
            for (int k = 0; k < K; ++k) ref[i + j * M] += a[i + k * M] * b[j + k * N];
    float *da, *db, *dc;
    cudaMalloc(&da, a.size() * 4);
    cudaMalloc(&db, b.size() * 4);
    cudaMalloc(&dc, c.size() * 4);
    cudaMemcpy(da, a.data(), a.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(db, b.data(), b.size() * 4, cudaMemcpyHostToDevice);
    for (int variant = 0; variant < 11; ++variant) {
        cudaMemset(dc, 0, c.size() * 4);
        probe<<<1, 128>>>(da, db, dc, variant);
        cudaError_t e = cudaDeviceSynchronize();
        cudaMemcpy(c.data(), dc, c.size() * 4, cudaMemcpyDeviceToHost);
        double maxerr = 0, maxref = 0, maxgot = 0;
        for (int i = 0; i < M * N; ++i) {
            maxerr = std::max(maxerr, (double)std::abs(c[i] - ref[i]));
            maxref = std::max(maxref, (double)std::abs(ref[i]));
            maxgot = std::max(maxgot, (double)std::abs(c[i]));
        }
        const char* what = variant < 4 ? ((variant & 2) ? "MN SW128, LBO=1KB,SBO=atom" : "MN SW128, LBO=atom,SBO=1KB")
                         : variant == 4 ? "K-major, no swizzle" : variant == 5 ? "MN, no swizzle"
                         : variant == 6 ? "K-major SW64 (the GEMM's)"
                         : variant == 7 ? "MN SW128/32B-atom, chunk^=k&3, LBO=MN atom 512, SBO=K group 2048"
                         : variant == 8 ? "MN SW128/32B-atom, chunk^=k&3, LBO/SBO swapped"
                         : variant == 9 ? "MN SW128/32B-atom, chunk^=(k>>1)&3" : "MN SW128/32B-atom, chunk^=(k>>1)&3, swapped";
        printf("variant %d (%s): %s max|err| %.1f max|ref| %.1f max|got| %.1f  C[0..3]=%.0f %.0f %.0f %.0f ref %.0f %.0f %.0f %.0f\n",
               variant, what,
               cudaGetErrorString(e), maxerr, maxref, maxgot, c[0], c[1], c[2], c[3], ref[0], ref[1], ref[2], ref[3]);
        if (e != cudaSuccess) return 1;
    }
    return 0;
}
