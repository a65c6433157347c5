// tf32_round_probe.cu -- how tcgen05.mma kind::tf32 converts fp32 operands: one MMA
// (M = N = 128, K = 8, K-major, no swizzle -- tools/mn_probe.cu variant 4) with A full
// fp32 values and B = 1 on one k only, so C[i][j] = A[i][k0] as the tensor core read it;
// compared with truncation and round-to-nearest of A to tf32 (10 mantissa bits).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -I paper_2308_03120_b200/csrc -o tools/tf32_round_probe tools/tf32_round_probe.cu
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "bm_ptx.cuh"

using namespace bm;

__global__ void probe(const float* A, const float* B, float* C) {
    __shared__ __align__(1024) unsigned char sa[128 * 8 * 4];
    __shared__ __align__(1024) unsigned char sb[128 * 8 * 4];
    __shared__ uint64_t bar;
    __shared__ uint32_t tslot;
    const int tid = threadIdx.x;
    for (int i = tid; i < 128 * 8; i += blockDim.x) {
        const int mn = i % 128, kk = i / 128;
        const int off = (mn >> 3) * 256 + (kk >> 2) * 128 + (mn & 7) * 16 + (kk & 3) * 4;
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
            d |= (uint64_t)(128 >> 4) << 16;
            d |= (uint64_t)(256 >> 4) << 32;
            d |= (uint64_t)1 << 46;
            return d;
        };
        const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(128 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
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

static float trunc_tf32(float x) { unsigned u; std::memcpy(&u, &x, 4); u &= 0xffffe000u; float r; std::memcpy(&r, &u, 4); return r; }
static float rne_tf32(float x) {
    unsigned u; std::memcpy(&u, &x, 4);
    const unsigned lsb = (u >> 13) & 1u;
    u = (u + 0x0fffu + lsb) & 0xffffe000u;
    float r; std::memcpy(&r, &u, 4); return r;
}
static float rna_tf32(float x) { unsigned u; std::memcpy(&u, &x, 4); u = (u + 0x1000u) & 0xffffe000u; float r; std::memcpy(&r, &u, 4); return r; }

int main() {
    const int M = 128, K = 8;
    std::vector<float> a(M * K), b(M * K, 0.f), c(M * M);
    srand(7);
    for (auto& x : a) x = 1.0f + (float)rand() / RAND_MAX;   // full 23-bit mantissas
    for (int j = 0; j < M; ++j) b[j + 0 * M] = 1.0f;            // B[j][k=0] = 1: C[i][j] = A[i][0]
    float *da, *db, *dc;
    cudaMalloc(&da, a.size() * 4);
    cudaMalloc(&db, b.size() * 4);
    cudaMalloc(&dc, c.size() * 4);
    cudaMemcpy(da, a.data(), a.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(db, b.data(), b.size() * 4, cudaMemcpyHostToDevice);
    probe<<<1, 128>>>(da, db, dc);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(c.data(), dc, c.size() * 4, cudaMemcpyDeviceToHost);
    int eq_raw = 0, eq_tr = 0, eq_rne = 0, eq_rna = 0;
    for (int i = 0; i < M; ++i) {
        const float got = c[i + 5 * M], x = a[i];
        eq_raw += got == x;
        eq_tr += got == trunc_tf32(x);
        eq_rne += got == rne_tf32(x);
        eq_rna += got == rna_tf32(x);
    }
    printf("%s: of %d operands the MMA used: raw fp32 %d, truncated tf32 %d, RNE tf32 %d, RNA tf32 %d\n",
           cudaGetErrorString(e), M, eq_raw, eq_tr, eq_rne, eq_rna);
    printf("sample: x=%.9g got=%.9g trunc=%.9g rne=%.9g\n", a[0], c[0 + 5 * M], trunc_tf32(a[0]), rne_tf32(a[0]));
    return 0;
}
