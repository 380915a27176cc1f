// fp64 issue-rate microbenchmark (DFMA / DADD / DMUL): 8 independent chains per thread,
// enough warps per SM to cover the pipe latency.  Prints thread-instructions per clock per SM
// and TFLOP/s (DFMA = 2 flops) at the clock measured with clock64 over the same kernel.
#include <cstdio>
#include <cuda_runtime.h>

template <int OP>
__global__ void k(double* out, int iters, double a, double b, long long* clk) {
    double x[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-9 + i;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < 16; ++u)
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                if (OP == 0) x[i] = fma(x[i], a, b);
                else if (OP == 1) x[i] = x[i] + b;
                else x[i] = x[i] * a;
            }
    }
    long long t1 = clock64();
    double s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += x[i];
    if (s == 12345.678) out[0] = s;
    if (threadIdx.x == 0 && blockIdx.x == 0) clk[0] = t1 - t0;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* out;
    long long* clk;
    cudaMalloc(&out, 8);
    cudaMalloc(&clk, 8);
    const char* names[3] = {"DFMA", "DADD", "DMUL"};
    for (int op = 0; op < 3; ++op)
        for (int warps : {8, 16, 32}) {
            const int iters = 2000, threads = 32 * warps, blocks = sms;
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0);
            cudaEventCreate(&e1);
            for (int rep = 0; rep < 2; ++rep) {
                cudaEventRecord(e0);
                if (op == 0) k<0><<<blocks, threads>>>(out, iters, 0.999999, 1e-7, clk);
                if (op == 1) k<1><<<blocks, threads>>>(out, iters, 0.999999, 1e-7, clk);
                if (op == 2) k<2><<<blocks, threads>>>(out, iters, 0.999999, 1e-7, clk);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
            }
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            long long c;
            cudaMemcpy(&c, clk, 8, cudaMemcpyDeviceToHost);
            const double ninstr = (double)blocks * threads * iters * 16 * 8;
            const double per_clk_sm = ninstr / sms / (double)c;
            printf("%s warps/SM %2d: %.3f ms, %.1f thread-instr/clk/SM, %.2f T instr/s, clock %.0f MHz, %.1f TFLOP/s\n",
                   names[op], warps, ms, per_clk_sm, ninstr / ms / 1e9, c / (ms * 1e3), ninstr * (op == 0 ? 2 : 1) / ms / 1e9);
        }
    return 0;
}
