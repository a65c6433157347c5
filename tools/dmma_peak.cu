// dmma_peak.cu -- issue-rate ceiling of DMMA (mma.sync m8n8k4 f64) on this GPU: every
// warp runs chains of independent DMMAs on register operands (no memory traffic), for
// several warps per SM; prints TFLOP/s.  The roofline denominator for the f64 GEMM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/dmma_peak tools/dmma_peak.cu && ./tools/dmma_peak
#include <cstdio>

template <int CH>
__global__ void dmma_loop(double* out, int iters, double seed) {
    double c[CH][2];
    double a = seed + threadIdx.x * 1e-9, b = seed - threadIdx.x * 1e-9;
#pragma unroll
    for (int j = 0; j < CH; ++j) c[j][0] = c[j][1] = 0.0;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < CH; ++j)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                         : "+d"(c[j][0]), "+d"(c[j][1])
                         : "d"(a), "d"(b));
    }
    double s = 0;
#pragma unroll
    for (int j = 0; j < CH; ++j) s += c[j][0] + c[j][1];
    if (s == 12345.678) out[threadIdx.x] = s;   // keep the chains alive
}

template <int CH>
void run(int sms, int warps, int iters) {
    double* out;
    cudaMalloc(&out, 4096 * sizeof(double));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    dmma_loop<CH><<<sms, warps * 32>>>(out, 100, 1.0);
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(e0);
        dmma_loop<CH><<<sms, warps * 32>>>(out, iters, 1.0);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    const double flops = 2.0 * 8 * 8 * 4 * (double)CH * iters * warps * sms;
    printf("chains %d warps/SM %2d: %.2f ms  %.2f TFLOP/s  (%s)\n", CH, warps, best, flops / best / 1e9,
           cudaGetErrorString(cudaGetLastError()));
    cudaFree(out);
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    printf("SMs %d\n", sms);
    const int iters = 20000;
    for (int w : {4, 8, 16, 32}) {
        run<4>(sms, w, iters);
        run<8>(sms, w, iters);
    }
    return 0;
}
