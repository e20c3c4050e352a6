// fp64_peak.cu -- N8: measured FP64 issue peak of this B200 (DFMA chains) and
// the FP64 min/max (DMNMX) and DADD rates that the PredINTF inner loop uses.
// MEASURED_PEAKS.json has no FP64 figure; this supplies one for context next
// to the derived roofline peak (148 SM x 64 lanes x 1.965 GHz).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp64_peak tools/fp64_peak.cu
//   tools/fp64_peak            -> one JSON line
#include <cstdio>
#include <cuda_runtime.h>

template <int OP>
__global__ void k_chain(double* out, int iters, double a, double b) {
    // 8 independent chains per thread to cover the DFMA latency
    double x[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) x[j] = threadIdx.x * 1e-9 + j;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            if (OP == 0) x[j] = fma(x[j], a, b);          // DFMA
            else if (OP == 1) x[j] = fmin(x[j] + a, b);   // DADD + DMNMX
            else x[j] = x[j] * a;                         // DMUL
        }
    }
    double s = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) s += x[j];
    if (s == 12345.678) out[0] = s;
}

template <int OP>
double run(int blocks, int threads, int iters) {
    double* out;
    cudaMalloc(&out, 8);
    k_chain<OP><<<blocks, threads>>>(out, 16, 0.999999, 1e-7);
    cudaDeviceSynchronize();
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    k_chain<OP><<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    cudaFree(out);
    const double ops_per_thread = (OP == 1 ? 2.0 : 1.0) * 8.0 * iters;   // instructions, FMA = 1
    return (double)blocks * threads * ops_per_thread / (ms / 1e3);
}

int main() {
    int dev = 0, sms = 0, clk = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
    const int blocks = sms * 8, threads = 256, iters = 1 << 14;
    double best_fma = 0, best_addmin = 0, best_mul = 0;
    for (int r = 0; r < 5; ++r) {
        double v = run<0>(blocks, threads, iters); if (v > best_fma) best_fma = v;
        v = run<1>(blocks, threads, iters); if (v > best_addmin) best_addmin = v;
        v = run<2>(blocks, threads, iters); if (v > best_mul) best_mul = v;
    }
    printf("{\"sms\": %d, \"clock_khz\": %d, \"dfma_lane_ops_per_s\": %.4e, \"dfma_tflops\": %.3f, "
           "\"dadd_dmnmx_lane_ops_per_s\": %.4e, \"dmul_lane_ops_per_s\": %.4e, "
           "\"derived_peak_lane_ops_per_s\": %.4e}\n",
           sms, clk, best_fma, 2 * best_fma / 1e12, best_addmin, best_mul, (double)sms * 64 * 1.965e9);
    return 0;
}
