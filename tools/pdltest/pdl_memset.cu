// Does a programmatic-dependent launch right after a memset / memcpy wait for it?  (B200 check for
// the PDL use in libmgcg: kernels launched with the attribute must never overtake a copy node.)
#include <cstdio>
#include <cuda_runtime.h>

__global__ void fill(double* a, long long n, double v) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) a[i] = v;
}
__global__ void check(const double* a, long long n, unsigned long long* bad) {
    asm volatile("griddepcontrol.wait;\n" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
    unsigned long long c = 0;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        if (a[i] != 0.0) ++c;
    if (c) atomicAdd(bad, c);
}
static void launch_pdl(const double* a, long long n, unsigned long long* bad, cudaStream_t s) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(148 * 4); cfg.blockDim = dim3(256); cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, check, a, n, bad);
}
int main() {
    const long long n = 1LL << 27;   // 1 GiB of doubles
    double *a, *z; unsigned long long* bad;
    cudaMalloc(&a, n * 8); cudaMalloc(&z, n * 8); cudaMalloc(&bad, 8);
    cudaMemset(z, 0, n * 8);
    cudaStream_t s; cudaStreamCreate(&s);
    unsigned long long tot[4] = {0, 0, 0, 0};
    for (int mode = 0; mode < 4; ++mode) {   // 0 memset stream, 1 memcpy stream, 2 memset graph, 3 memcpy graph
        for (int rep = 0; rep < 20; ++rep) {
            cudaMemsetAsync(bad, 0, 8, s);
            fill<<<148 * 4, 256, 0, s>>>(a, n, 1.0);
            cudaGraphExec_t ge = nullptr;
            if (mode >= 2) cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
            if (mode % 2 == 0) cudaMemsetAsync(a, 0, n * 8, s);
            else cudaMemcpyAsync(a, z, n * 8, cudaMemcpyDeviceToDevice, s);
            launch_pdl(a, n, bad, s);
            if (mode >= 2) {
                cudaGraph_t g; cudaStreamEndCapture(s, &g); cudaGraphInstantiate(&ge, g, 0); cudaGraphDestroy(g);
                cudaGraphLaunch(ge, s);
            }
            unsigned long long h = 0;
            cudaMemcpyAsync(&h, bad, 8, cudaMemcpyDeviceToHost, s);
            cudaStreamSynchronize(s);
            tot[mode] += h;
            if (ge) cudaGraphExecDestroy(ge);
        }
    }
    printf("nonzero seen after memset(stream) %llu memcpy(stream) %llu memset(graph) %llu memcpy(graph) %llu; err=%s\n",
           tot[0], tot[1], tot[2], tot[3], cudaGetErrorString(cudaGetLastError()));
    return 0;
}
