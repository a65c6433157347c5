// scalar_read_probe.cu -- host latency of reading one scalar a kernel produced, per
// iteration of [tiny kernel; get the value on the host]:
//   memcpy: cudaMemcpyAsync 8 B D2H into pinned memory + cudaStreamSynchronize
//   mapped: the kernel stores into mapped pinned memory + cudaStreamSynchronize
//   spin:   the kernel stores value + flag into mapped pinned memory, the host spins on the flag
// (what the config-5 step pays after its kernel for accu(r)).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/scalar_read_probe tools/scalar_read_probe.cu
#include <chrono>
#include <cstdio>

__global__ void produce(double* dev, double* host_val, volatile unsigned* host_flag, unsigned seq, int mode) {
    const double v = 1.0 + seq;
    if (mode == 0) *dev = v;
    if (mode >= 1) *host_val = v;
    if (mode == 2) {
        __threadfence_system();
        *host_flag = seq;
    }
}

int main() {
    double *dev, *pinned;
    unsigned* flag;
    cudaMalloc(&dev, 8);
    cudaHostAlloc(&pinned, 64, cudaHostAllocMapped);
    cudaHostAlloc(&flag, 64, cudaHostAllocMapped);
    double* pinned_d;
    unsigned* flag_d;
    cudaHostGetDevicePointer(&pinned_d, pinned, 0);
    cudaHostGetDevicePointer(&flag_d, flag, 0);
    cudaStream_t s;
    cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    const char* names[3] = {"memcpy+sync", "mapped+sync", "mapped flag spin"};
    for (int rep = 0; rep < 2; ++rep)
        for (int mode = 0; mode < 3; ++mode) {
            const int n = 2000;
            double sum = 0;
            *flag = 0;
            auto t0 = std::chrono::steady_clock::now();
            for (int i = 1; i <= n; ++i) {
                produce<<<1, 1, 0, s>>>(dev, pinned_d, flag_d, (unsigned)i, mode);
                if (mode == 0) {
                    cudaMemcpyAsync(pinned, dev, 8, cudaMemcpyDeviceToHost, s);
                    cudaStreamSynchronize(s);
                } else if (mode == 1) {
                    cudaStreamSynchronize(s);
                } else {
                    while (*reinterpret_cast<volatile unsigned*>(flag) != (unsigned)i) {
                    }
                }
                sum += *reinterpret_cast<volatile double*>(pinned);
            }
            if (mode == 2) cudaStreamSynchronize(s);
            auto t1 = std::chrono::steady_clock::now();
            printf("%-18s %.2f us/iter (check %.0f)\n", names[mode],
                   std::chrono::duration<double, std::micro>(t1 - t0).count() / n, sum);
        }
    return 0;
}
