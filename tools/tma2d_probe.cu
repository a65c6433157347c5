// tma2d_probe.cu -- streaming throughput of 2-D TMA boxes over a column-major
// 2^20 x 1024 f32 matrix as a function of the box's inner (row) extent: the
// layout question behind the fused logistic kernel (bm_lgrad.cuh).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tma2d_probe tools/tma2d_probe.cu -lcuda
#include <cstdio>
#include <cuda.h>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned sm_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__global__ void probe2d(const __grid_constant__ CUtensorMap tm, int rb, int bc, int nbox_c, long long nslabs, int ns,
                        float* out) {
    extern __shared__ __align__(1024) char smem[];
    __shared__ unsigned long long full[8];
    const long long nmine = (nslabs - blockIdx.x + gridDim.x - 1) / gridDim.x;
    const unsigned slab_bytes = (unsigned)(rb * bc * nbox_c * 4);
    if (threadIdx.x == 0) {
        for (int s = 0; s < ns; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sm_u32(&full[s])));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    auto issue = [&](long long j) {
        const int s = (int)(j % ns);
        const long long unit = blockIdx.x + j * gridDim.x;
        const long long groups = 1024 / (bc * nbox_c);
        const long long slab = unit / groups, grp = unit % groups;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sm_u32(&full[s])), "r"(slab_bytes)
                     : "memory");
        for (int b = 0; b < nbox_c; ++b)
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
                    sm_u32(smem + (size_t)s * slab_bytes + (size_t)b * rb * bc * 4)),
                "l"(&tm), "r"((int)(slab * rb)), "r"((int)((grp * nbox_c + b) * bc)), "r"(sm_u32(&full[s]))
                : "memory");
    };
    float acc = 0.f;
    if (threadIdx.x == 0)
        for (long long j = 0; j < ns - 1 && j < nmine; ++j) issue(j);
    for (long long j = 0; j < nmine; ++j) {
        const int s = (int)(j % ns);
        const unsigned par = (unsigned)((j / ns) & 1);
        asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(
                         sm_u32(&full[s])),
                     "r"(par)
                     : "memory");
        acc += reinterpret_cast<const float*>(smem + (size_t)s * slab_bytes)[threadIdx.x];
        __syncthreads();
        if (threadIdx.x == 0 && j + ns - 1 < nmine) issue(j + ns - 1);
    }
    if (acc == 1234.5f) out[0] = acc;
}

int main() {
    const long long m = 1 << 20, k = 1024;
    float* X;
    float* out;
    cudaMalloc(&X, m * k * 4);
    cudaMalloc(&out, 64);
    cudaMemset(X, 0, m * k * 4);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaFuncSetAttribute(probe2d, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    struct Cfg { int rb, bc, swz; };
    Cfg cfgs[] = {{16, 256, 64}, {32, 256, 128}, {32, 128, 128}, {64, 128, 0}, {64, 64, 0}, {128, 64, 0}, {256, 32, 0},
                  {256, 16, 0}};
    for (const Cfg& c : cfgs) {
        CUtensorMap tm;
        const cuuint64_t gdim[2] = {(cuuint64_t)m, (cuuint64_t)k};
        const cuuint64_t gstr[1] = {(cuuint64_t)(m * 4)};
        const cuuint32_t box[2] = {(cuuint32_t)c.rb, (cuuint32_t)c.bc};
        const cuuint32_t es[2] = {1, 1};
        CUtensorMapSwizzle sw = c.swz == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : c.swz == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
                                                                                       : CU_TENSOR_MAP_SWIZZLE_NONE;
        CUresult r = cuTensorMapEncodeTiled(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, X, gdim, gstr, box, es,
                                            CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) { printf("encode failed rb=%d bc=%d: %d\n", c.rb, c.bc, (int)r); continue; }
        // a stage holds `per` boxes of rb x bc (a whole slab when it fits)
        const int nbox_c = (int)(k / c.bc);
        const long long box_bytes = (long long)c.rb * c.bc * 4;
        int per = nbox_c;
        while (per > 1 && 3 * per * box_bytes > 192 * 1024) per >>= 1;
        const long long slab_bytes = per * box_bytes;
        int ns = (int)((192 * 1024) / slab_bytes);
        if (ns > 8) ns = 8;
        const long long nslabs = (m / c.rb) * (nbox_c / per);   // stage units, row-block major
        const int smem = (int)(ns * slab_bytes);
        auto run = [&] { probe2d<<<sms, 256, smem>>>(tm, c.rb, c.bc, per, nslabs, ns, out); };
        run();
        cudaDeviceSynchronize();
        float best = 1e9;
        for (int rep = 0; rep < 5; ++rep) {
            cudaEventRecord(a);
            run();
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (ms < best) best = ms;
        }
        printf("rb=%3d box=%3dx%3d swz=%3d boxes/stage=%d stages=%d: %7.1f GB/s %s\n", c.rb, c.rb, c.bc, c.swz, per, ns,
               m * k * 4 / (best * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
