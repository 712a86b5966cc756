// tools/lat_probe.cu -- DEVELOPER TOOL: single-warp dependent-chain latencies
// (cycles per op, clock64) of the ops on the k = 0 tree's critical path:
// DFMA, DMUL, 64-bit integer max, SHFL of a double, and one full tree node
// (DMUL + DFMA + integer max).  One JSON line.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/lat_probe tools/lat_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int IT = 4096;

__global__ void probe(double a, double b, long long* cyc, double* sink) {
    double x = threadIdx.x * 1e-9 + 1.0;
    long long t0, t1;
    // DFMA chain
    t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < IT; ++i) x = fma(x, a, b);
    t1 = clock64();
    cyc[0] = t1 - t0;
    // DMUL chain
    t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < IT; ++i) x = x * a;
    t1 = clock64();
    cyc[1] = t1 - t0;
    // 64-bit integer max chain (bit patterns)
    long long y = __double_as_longlong(x);
    t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < IT; ++i) y = max(y, (long long)i) ^ 1;
    t1 = clock64();
    cyc[2] = t1 - t0;
    // SHFL chain
    double z = x;
    t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < IT; ++i) z = __shfl_down_sync(0xffffffffu, z, 1) + 0.0;
    t1 = clock64();
    cyc[3] = t1 - t0;
    // tree node chain: v = max(ex, pu v + pd v)
    double v = x, ex = 0.25;
    t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < IT; ++i) {
        const double c = fma(a, v, b * v);
        v = __longlong_as_double(max(__double_as_longlong(ex), __double_as_longlong(c)));
    }
    t1 = clock64();
    cyc[4] = t1 - t0;
    // DADD chain
    t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < IT; ++i) z = z + b;
    t1 = clock64();
    cyc[5] = t1 - t0;
    // FFMA (fp32) chain for comparison
    float f = (float)x;
    t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < IT; ++i) f = fmaf(f, (float)a, (float)b);
    t1 = clock64();
    cyc[6] = t1 - t0;
    if (threadIdx.x == 0) sink[0] = x + y + z + v + f;
}

// the k = 0 tree's level loop (amtc_tree.cu) for M columns per lane, timed per
// level on one warp (clock64), warps = blockDim / 32 on one SM
template <int M>
__global__ void level_loop(double pu, double pd, double d, double c0, int levels, long long* cyc, double* sink) {
    double V[M], X[M];
#pragma unroll
    for (int q = 0; q < M; ++q) { V[q] = 1.0 + 1e-3 * (threadIdx.x * M + q); X[q] = 0.5 - 1e-3 * q; }
    const long long t0 = clock64();
    for (int l = 0; l < levels; ++l) {
        const double nb = __shfl_down_sync(0xffffffffu, V[0], 1);
#pragma unroll
        for (int q = 0; q < M; ++q) {
            const double vn = (q + 1 < M) ? V[q + 1] : nb;
            X[q] = fma(d, X[q], c0);
            const double cont = fma(pu, V[q], pd * vn);
            V[q] = __longlong_as_double(max(__double_as_longlong(X[q]), __double_as_longlong(cont)));
        }
    }
    const long long t1 = clock64();
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
    double sum = 0;
#pragma unroll
    for (int q = 0; q < M; ++q) sum += V[q];
    if (sum == 1234.5) sink[0] = sum;
}

template <int M>
static double per_level(int warps, long long* d, double* s) {
    const int L = 4096;
    level_loop<M><<<1, 32 * warps>>>(0.49, 0.5, 0.99, 0.01, L, d, s);
    level_loop<M><<<1, 32 * warps>>>(0.49, 0.5, 0.99, 0.01, L, d, s);
    long long h;
    cudaMemcpy(&h, d, sizeof(h), cudaMemcpyDeviceToHost);
    return (double)h / L;
}

int main() {
    long long* d;
    double* s;
    cudaMalloc(&d, 8 * sizeof(long long));
    cudaMalloc(&s, sizeof(double));
    probe<<<1, 32>>>(0.999999, 1e-7, d, s);
    probe<<<1, 32>>>(0.999999, 1e-7, d, s);
    long long h[8];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    printf("{\"tool\": \"lat_probe\", \"cycles_per_op\": {\"dfma\": %.2f, \"dmul\": %.2f, \"imax64_xor\": %.2f, "
           "\"shfl_f64_dadd\": %.2f, \"tree_node\": %.2f, \"dadd\": %.2f, \"ffma\": %.2f}}\n",
           (double)h[0] / IT, (double)h[1] / IT, (double)h[2] / IT, (double)h[3] / IT, (double)h[4] / IT,
           (double)h[5] / IT, (double)h[6] / IT);
    printf("{\"tool\": \"lat_probe\", \"tree_level_cycles\": {");
    const int ws[] = {1, 4, 8, 16};
    for (int wi = 0; wi < 4; ++wi) {
        const int w = ws[wi];
        printf("%s\"w%d\": {\"M4\": %.1f, \"M8\": %.1f, \"M12\": %.1f, \"M16\": %.1f}", wi ? ", " : "", w,
               per_level<4>(w, d, s), per_level<8>(w, d, s), per_level<12>(w, d, s), per_level<16>(w, d, s));
    }
    printf("}}\n");
    return 0;
}
