// tma_probe.cu -- streaming-read microbenchmark for the staged reduction
// design (run on the GPU box): how fast can one SM pull HBM data into shared
// memory with 1-D cp.async.bulk copies of various sizes, ring depths and
// issuing lanes, compared with plain 16-B LDG streaming?
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/tma_probe tools/tma_probe.cu && /tmp/tma_probe
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned sm_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void bar_init(unsigned long long* b, unsigned c) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sm_u32(b)), "r"(c));
}
__device__ __forceinline__ void expect_tx(unsigned long long* b, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sm_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void arrive(unsigned long long* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sm_u32(b)) : "memory");
}
__device__ __forceinline__ void wait(unsigned long long* b, unsigned par) {
    asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(
                     sm_u32(b)),
                 "r"(par)
                 : "memory");
}
__device__ __forceinline__ void bulk(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     sm_u32(dst)),
                 "l"(src), "r"(bytes), "r"(sm_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void bulk_hint(void* dst, const void* src, unsigned bytes, unsigned long long* bar,
                                          unsigned long long pol) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            sm_u32(dst)),
        "l"(src), "r"(bytes), "r"(sm_u32(bar)), "l"(pol)
        : "memory");
}

// ring of NS stages of STAGE bytes, split into `pieces` copies issued by lanes
// 0..pieces-1 of warp 0; NC consumer warps (stage k -> warp k % NC) sum it.
__global__ void probe_bulk(const float* __restrict__ src, long long nbytes, int stage, int ns, int pieces, int hint,
                           float* out) {
    extern __shared__ __align__(128) char smem[];
    __shared__ unsigned long long full[64], empty[64];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nc = (blockDim.x >> 5) - 1;
    const long long nst = nbytes / stage;
    const long long per = nst / gridDim.x;
    const long long first = per * blockIdx.x;
    if (threadIdx.x == 0) {
        for (int i = 0; i < ns; ++i) { bar_init(&full[i], 1); bar_init(&empty[i], 1); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    unsigned long long pol = 0;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    if (warp == 0) {
        const int piece = stage / pieces;
        for (long long k = 0; k < per; ++k) {
            const int s = (int)(k % ns);
            const unsigned it = (unsigned)(k / ns);
            if (it > 0) wait(&empty[s], (it - 1) & 1);
            if (lane == 0) expect_tx(&full[s], stage);
            __syncwarp();
            if (lane < pieces) {
                const char* g = reinterpret_cast<const char*>(src) + (first + k) * stage + lane * piece;
                if (hint) bulk_hint(smem + (size_t)s * stage + lane * piece, g, piece, &full[s], pol);
                else bulk(smem + (size_t)s * stage + lane * piece, g, piece, &full[s]);
            }
        }
    } else {
        float acc = 0.f;
        for (long long k = warp - 1; k < per; k += nc) {
            const int s = (int)(k % ns);
            wait(&full[s], (unsigned)(k / ns) & 1);
            const float4* p = reinterpret_cast<const float4*>(smem + (size_t)s * stage);
            for (int i = lane; i < stage / 16; i += 32) {
                float4 v = p[i];
                acc += v.x + v.y + v.z + v.w;
            }
            __syncwarp();
            if (lane == 0) arrive(&empty[s]);
        }
        if (acc == 12345.f) out[0] = acc;
    }
}

__global__ void probe_ldg(const float4* __restrict__ src, long long n4, float* out) {
    float acc = 0.f;
    const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x, nt = (long long)gridDim.x * blockDim.x;
    long long i = tid;
    for (; i + 3 * nt < n4; i += 4 * nt) {
        float4 a = __ldg(src + i), b = __ldg(src + i + nt), c = __ldg(src + i + 2 * nt), d = __ldg(src + i + 3 * nt);
        acc += a.x + b.y + c.z + d.w;
    }
    for (; i < n4; i += nt) acc += __ldg(src + i).x;
    if (acc == 12345.f) out[0] = acc;
}

int main() {
    const long long nbytes = 1ll << 30;
    float* buf;
    float* out;
    cudaMalloc(&buf, nbytes);
    cudaMalloc(&out, 64);
    cudaMemset(buf, 0, nbytes);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaFuncSetAttribute(probe_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    auto timeit = [&](auto launch) {
        launch();
        cudaDeviceSynchronize();
        float best = 1e9;
        for (int r = 0; r < 5; ++r) {
            cudaEventRecord(a);
            launch();
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (ms < best) best = ms;
        }
        return nbytes / (best * 1e-3) / 1e9;
    };
    for (int blk : {256, 512, 1024}) {
        for (int per : {1, 2, 4}) {
            double g = timeit([&] { probe_ldg<<<sms * per, blk>>>((const float4*)buf, nbytes / 16, out); });
            printf("ldg   block=%4d ctas/sm=%d                         %7.1f GB/s\n", blk, per, g);
        }
    }
    struct Cfg { int stage, ns, pieces, nc, hint; };
    Cfg cfgs[] = {
        {8192, 20, 1, 4, 0}, {8192, 24, 1, 8, 0}, {8192, 20, 2, 4, 0},
        {16384, 12, 1, 4, 0}, {16384, 12, 2, 4, 0}, {16384, 12, 1, 6, 0},
        {32768, 6, 1, 3, 0}, {32768, 6, 1, 6, 0}, {32768, 6, 2, 6, 0}, {32768, 6, 4, 6, 0},
        {65536, 3, 1, 3, 0}, {65536, 3, 2, 3, 0}, {4096, 40, 1, 4, 0}, {4096, 48, 1, 8, 0},
        {8192, 20, 1, 4, 1}, {32768, 6, 1, 6, 1}, {16384, 12, 1, 12, 0}, {16384, 8, 1, 8, 0},
    };
    for (const Cfg& c : cfgs) {
        const int smem = c.stage * c.ns;
        if (smem > 200 * 1024) continue;
        double g = timeit([&] {
            probe_bulk<<<sms, 32 * (1 + c.nc), smem>>>(buf, nbytes, c.stage, c.ns, c.pieces, c.hint, out);
        });
        cudaError_t e = cudaGetLastError();
        printf("bulk  stage=%6d ns=%2d pieces=%2d consumers=%d hint=%d  %7.1f GB/s %s\n", c.stage, c.ns, c.pieces, c.nc,
               c.hint, g, e == cudaSuccess ? "" : cudaGetErrorString(e));
    }
    return 0;
}
