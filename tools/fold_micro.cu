// fold_micro.cu -- time the last-CTA fold of bm_reduce.cuh in isolation (GPU
// box): one CTA folding `nitems` half-unit partials, with phase timestamps.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -std=c++17 \
//        -I paper_2308_03120_b200/csrc -o tools/fold_micro tools/fold_micro.cu
#include <cstdio>
#include <vector>
__device__ unsigned long long g_t[8];
__device__ unsigned long long g_tr[8];
#define BM_TRACE(k)                                                                            \
    do {                                                                                       \
        if (threadIdx.x == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g_tr[k]));     \
    } while (0)
#include "bm_reduce.cuh"

using namespace bm;

__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

template <int UPB>
__global__ void __launch_bounds__(512) fold_only(Args a, i64 nitems, i64 nfull) {
    if (threadIdx.x == 0) g_t[0] = gtime();
    last_cta_fold<float, 1, UPB>(a, nitems, nfull, false, true);
    __syncthreads();
    if (threadIdx.x == 0) g_t[1] = gtime();
}

// the same fold with phase stamps: loads, staging, tree
__global__ void __launch_bounds__(512) fold_phases(const float* parts, int nblocks, float* out) {
    extern __shared__ __align__(16) char smem[];
    float* buf = reinterpret_cast<float*>(smem);
    float* buf2 = buf + 16384;
    unsigned long long t0 = gtime();
    for (int i0 = threadIdx.x; i0 < nblocks; i0 += 4 * blockDim.x) {
        float v[4][8];
#pragma unroll
        for (int bb = 0; bb < 4; ++bb) {
            const int i = i0 + bb * blockDim.x;
            if (i < nblocks) {
#pragma unroll
                for (int u = 0; u < 8; ++u) v[bb][u] = __ldcg(parts + (i * 8 + u));
            }
        }
#pragma unroll
        for (int bb = 0; bb < 4; ++bb) {
            const int i = i0 + bb * blockDim.x;
            if (i < nblocks) {
                float x = ((v[bb][0] + v[bb][1]) + (v[bb][2] + v[bb][3])) + ((v[bb][4] + v[bb][5]) + (v[bb][6] + v[bb][7]));
                buf[i] = x;
            }
        }
    }
    __syncthreads();
    unsigned long long t1 = gtime();
    float r = cta_combine_pairwise<float, 1>(buf, buf2, nblocks);
    unsigned long long t2 = gtime();
    if (threadIdx.x == 0) {
        out[0] = r;
        g_t[2] = t0; g_t[3] = t1; g_t[4] = t2;
    }
}

int main() {
    const int nblocks = 2048, upb = 8;
    const long long nitems = (long long)nblocks * upb;
    float* parts;
    float* res;
    unsigned* ticket;
    cudaMalloc(&parts, nitems * 8);
    cudaMalloc(&res, 64);
    cudaMalloc(&ticket, 4);
    cudaMemset(ticket, 0, 4);
    // item partials of 1 followed by pre-folded block values of 8 (one CTA owns every block)
    std::vector<float> h(2 * nitems, 8.0f);
    for (long long i = 0; i < nitems; ++i) h[i] = 1.0f;
    cudaMemcpy(parts, h.data(), nitems * 8, cudaMemcpyHostToDevice);
    Args a;
    memset(&a, 0, sizeof a);
    a.partials = parts;
    a.ticket = ticket;
    a.result = res;
    a.smem_bytes = 16 * BM_TILE_BYTES;
    cudaFuncSetAttribute(fold_only<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, a.smem_bytes);
    cudaFuncSetAttribute(fold_phases, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(e0);
        fold_only<8><<<1, 512, a.smem_bytes>>>(a, nitems, nblocks);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        unsigned long long t[8];
        cudaMemcpyFromSymbol(t, g_t, sizeof t);
        float r;
        cudaMemcpy(&r, res, 4, cudaMemcpyDeviceToHost);
        unsigned long long tr[8];
        cudaMemcpyFromSymbol(tr, g_tr, sizeof tr);
        printf("fold_only: event %.2f us, in-kernel %.2f us, result %.0f (%s)\n", ms * 1e3, (t[1] - t[0]) * 1e-3, r,
               cudaGetErrorString(cudaGetLastError()));
        printf("  start->ticket %.2f, ticket %.2f, stage %.2f, tree %.2f, tail %.2f us\n", (tr[0] - t[0]) * 1e-3,
               (tr[1] - tr[0]) * 1e-3, (tr[2] - tr[1]) * 1e-3, (tr[3] - tr[2]) * 1e-3, (tr[4] - tr[3]) * 1e-3);
    }
    for (int rep = 0; rep < 3; ++rep) {
        fold_phases<<<1, 512, 128 * 1024>>>(parts, nblocks, res);
        cudaDeviceSynchronize();
        unsigned long long t[8];
        cudaMemcpyFromSymbol(t, g_t, sizeof t);
        printf("fold_phases: loads+stage %.2f us, tree %.2f us (%s)\n", (t[3] - t[2]) * 1e-3, (t[4] - t[3]) * 1e-3,
               cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
