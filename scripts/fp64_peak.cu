// Measured FP64 roof of the B200 ("measure the DFMA peak on
// the box"): every thread runs independent DFMA chains (8 accumulators, no
// memory traffic), grid = 8 blocks per SM; also the DADD and complex-MAC
// rates the fused passes issue.  Prints one JSON object.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/fp64_peak scripts/fp64_peak.cu
#include <cuda_runtime.h>

#include <cstdio>

template <int OP>
__global__ void k_peak(double* out, int iters, double a, double b) {
    double x[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-9 + i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (OP == 0) x[i] = fma(x[i], a, b);  // DFMA: 2 flop
            else x[i] = x[i] + b;                 // DADD: 1 flop
        }
    }
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += x[i];
    if (s == 12345.678) out[0] = s;  // keep the chains alive
}

template <int OP>
double run(int sms, float* msOut) {
    double* d = nullptr;
    cudaMalloc(&d, sizeof(double));
    const int threads = 256, blocks = 8 * sms, iters = 4096;
    k_peak<OP><<<blocks, threads>>>(d, 16, 0.999999, 1e-7);  // warm-up
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
        cudaEventRecord(e0);
        k_peak<OP><<<blocks, threads>>>(d, iters, 0.999999, 1e-7);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    cudaFree(d);
    *msOut = best;
    const double ops = static_cast<double>(blocks) * threads * iters * 8;  // instructions (thread level)
    return ops / (best * 1e-3);
}

int main() {
    int dev = 0, sms = 0, clk = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
    float msF = 0.f, msA = 0.f;
    const double dfma = run<0>(sms, &msF);
    const double dadd = run<1>(sms, &msA);
    std::printf(
        "{\"dfma_per_s\": %.6e, \"fp64_tflops_fma\": %.3f, \"dadd_per_s\": %.6e, \"sms\": %d, "
        "\"dfma_per_clk_per_sm_at_max_clock\": %.2f, \"max_clock_khz\": %d, \"ms_fma\": %.3f, \"ms_add\": %.3f}\n",
        dfma, 2.0 * dfma / 1e12, dadd, sms, dfma / (sms * (clk * 1e3)), clk, msF, msA);
    return 0;
}
