// Minimal TMA + mbarrier check (same PTX helpers as h8t.cu): load one 4-D box of a padded vector
// tensor and one 3-D uint8 box, copy them back out, compare on the host.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstring>
#include <vector>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned sm(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

struct Maps { CUtensorMap A, M; };

template <int MODE>
__global__ void k(const __grid_constant__ Maps tm, double* out, unsigned char* outm, int c0, int j0, int Q, int r) {
    extern __shared__ __align__(128) unsigned char s[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(s + 16384);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(sm(bar)), "r"(1u) : "memory");
        if (MODE >= 1) asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    if (MODE >= 2 && threadIdx.x == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(sm(bar)), "r"(9u * 768u + 9u * 32u) : "memory");
        asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];\n"
                     ::"r"(sm(s)), "l"((unsigned long long)&tm.A), "r"(3 * c0), "r"(j0), "r"(Q), "r"(r), "r"(sm(bar)) : "memory");
        asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];\n"
                     ::"r"(sm(s + 8192)), "l"((unsigned long long)&tm.M), "r"(c0), "r"(j0), "r"(Q), "r"(sm(bar)) : "memory");
    }
    if (MODE >= 2) {
        asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(sm(bar)), "r"(0u) : "memory");
        for (int i = threadIdx.x; i < 9 * 96; i += blockDim.x) out[i] = reinterpret_cast<double*>(s)[i];
        for (int i = threadIdx.x; i < 9 * 32; i += blockDim.x) outm[i] = s[8192 + i];
    }
}

int main() {
    const int n0 = 17, n1 = 9, n2 = 9, R = 3, p2 = 10, m2 = 16;
    const long long vstr = 3LL * n0 * n1 * p2;
    std::vector<double> hv(vstr * R);
    for (size_t i = 0; i < hv.size(); ++i) hv[i] = (double)i;
    std::vector<unsigned char> hm(n0 * n1 * m2);
    for (size_t i = 0; i < hm.size(); ++i) hm[i] = (unsigned char)(i * 7);
    double* dv; unsigned char* dm; double* out; unsigned char* outm;
    cudaMalloc(&dv, hv.size() * 8); cudaMalloc(&dm, hm.size()); cudaMalloc(&out, 9 * 96 * 8); cudaMalloc(&outm, 9 * 32);
    cudaMemcpy(dv, hv.data(), hv.size() * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(dm, hm.data(), hm.size(), cudaMemcpyHostToDevice);
    void* p = nullptr; cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
    auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    Maps tm; memset(&tm, 0, sizeof(tm));
    cuuint64_t dims[4] = {3 * n2, n1, n0, R}, str[3] = {3ull * p2 * 8, 3ull * p2 * n1 * 8, (cuuint64_t)vstr * 8};
    cuuint32_t box[4] = {96, 9, 1, 1}, es[4] = {1, 1, 1, 1};
    CUresult e1 = enc(&tm.A, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, dv, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                      CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    cuuint64_t mdims[3] = {n2, n1, n0}, mstr[2] = {(cuuint64_t)m2, (cuuint64_t)m2 * n1};
    cuuint32_t mbox[3] = {32, 9, 1};
    CUresult e2 = enc(&tm.M, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, dm, mdims, mstr, mbox, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                      CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode %d %d\n", (int)e1, (int)e2);
    cudaFuncSetAttribute(k<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 20000);
    cudaFuncSetAttribute(k<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 20000);
    cudaFuncSetAttribute(k<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 20000);
    k<0><<<1, 128, 20000>>>(tm, out, outm, -1, -1, 3, 1);
    printf("mode0 %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    k<1><<<1, 128, 20000>>>(tm, out, outm, -1, -1, 3, 1);
    printf("mode1 %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    k<2><<<1, 128, 20000>>>(tm, out, outm, -1, -1, 3, 1);
    printf("mode2 %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    std::vector<double> ho(9 * 96);
    std::vector<unsigned char> hom(9 * 32);
    cudaMemcpy(ho.data(), out, ho.size() * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(hom.data(), outm, hom.size(), cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int row = 0; row < 9; ++row)
        for (int x = 0; x < 96; ++x) {
            const int c = -3 + x, j = -1 + row;   // dim0 coordinate 3*c0 + x
            double ref = (c >= 0 && c < 3 * n2 && j >= 0 && j < n1) ? hv[(size_t)1 * vstr + (3LL * j * p2 + c) + 3LL * 3 * n1 * p2] : 0.0;
            if (ho[row * 96 + x] != ref) { if (bad < 5) printf("vec mismatch row %d x %d got %g ref %g\n", row, x, ho[row * 96 + x], ref); ++bad; }
        }
    for (int row = 0; row < 9; ++row)
        for (int x = 0; x < 32; ++x) {
            const int c = -1 + x, j = -1 + row;
            unsigned char ref = (c >= 0 && c < n2 && j >= 0 && j < n1) ? hm[(size_t)(3 * n1 + j) * m2 + c] : 0;
            if (hom[row * 32 + x] != ref) { if (bad < 10) printf("mask mismatch row %d x %d got %d ref %d\n", row, x, hom[row * 32 + x], ref); ++bad; }
        }
    printf("mismatches %d\n", bad);
    return 0;
}
