// tools/fp64_peak.cu -- DEVELOPER TOOL: measures the B200's FP64 pipe peak
// (DFMA and DMNMX/DSETP throughput) at the running clock, because
// MEASURED_PEAKS.json carries no FP64 figure.  The result is written to
// profiles/fp64_peak_rNN.json and is the denominator of bench.py's roofline.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp64_peak tools/fp64_peak.cu
//   tools/fp64_peak            (prints one JSON line)
#include <cstdio>
#include <cuda_runtime.h>

constexpr int CHAINS = 8;   // independent dependency chains per thread
constexpr int ITERS = 4096;

__global__ void dfma_kernel(double* out, double a, double b) {
    double x[CHAINS];
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) x[c] = threadIdx.x * 1e-9 + c;
    for (int i = 0; i < ITERS; ++i) {
#pragma unroll
        for (int c = 0; c < CHAINS; ++c) x[c] = fma(x[c], a, b);
    }
    double s = 0;
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) s += x[c];
    if (s == 12345.678) out[0] = s;  // never true; keeps the chains alive
}

__global__ void dmnmx_kernel(double* out, double a, double b) {
    double x[CHAINS];
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) x[c] = threadIdx.x * 1e-9 + c;
    for (int i = 0; i < ITERS; ++i) {
#pragma unroll
        for (int c = 0; c < CHAINS; ++c) x[c] = fmax(fmin(x[c], a), b);
    }
    double s = 0;
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) s += x[c];
    if (s == 12345.678) out[0] = s;
}

int main() {
    int dev = 0, sms = 0, clk_khz = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev);
    double* out;
    cudaMalloc(&out, 8);
    const int threads = 256, blocks = sms * 8;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    double best_fma = 1e30, best_mnmx = 1e30;
    for (int rep = 0; rep < 6; ++rep) {
        float ms;
        cudaEventRecord(e0);
        dfma_kernel<<<blocks, threads>>>(out, 0.999999, 1e-7);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        if (rep) best_fma = ms < best_fma ? ms : best_fma;
        cudaEventRecord(e0);
        dmnmx_kernel<<<blocks, threads>>>(out, 0.5, -0.5);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        if (rep) best_mnmx = ms < best_mnmx ? ms : best_mnmx;
    }
    const double thr = (double)blocks * threads;
    const double fma_per_s = thr * ITERS * CHAINS / (best_fma * 1e-3);
    const double mnmx_per_s = thr * ITERS * CHAINS * 2 / (best_mnmx * 1e-3);
    printf("{\"sms\": %d, \"clock_rate_mhz\": %.0f, \"dfma_per_s\": %.4e, \"fp64_tflops\": %.3f, "
           "\"dmnmx_per_s\": %.4e, \"dfma_per_sm_per_clk_at_max\": %.2f, \"err\": \"%s\"}\n",
           sms, clk_khz / 1e3, fma_per_s, 2 * fma_per_s / 1e12, mnmx_per_s,
           fma_per_s / sms / (clk_khz * 1e3), cudaGetErrorString(cudaGetLastError()));
    return 0;
}
