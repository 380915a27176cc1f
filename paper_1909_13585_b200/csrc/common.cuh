// Shared device-side definitions for the mgcg library (sm_100a, fp64).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#define MGK_FULL 0xffffffffu

// Layout of one multigrid level (structured grid, unit or 2^l-sized elements).
struct LevelGeom {
    int dim;
    int N[3];      // element counts (N[2] = 1 in 2D for convenience of products)
    int nn[3];     // node counts    (nn[2] = 1 in 2D)
    long long nnodes;
    long long ndof;
    long long nelem;
    int p2;          // node row pitch along axis 2 of the vectors (nn[2] compact; even on the padded 3D fine level)
    long long vstr;  // doubles per RHS vector (ndof compact)
};

// Device-side CG control block (per RHS arrays of length MG_MAX_RHS).
struct CgCtl {
    double* alpha;
    double* beta;
    double* rz;       // r.z of the current iteration
    double* rr;       // r.r
    double* bb;       // b.b
    double* pq;       // p.q
    double* tt;       // true residual t.t
    double* xalpha;   // deferred x update alpha (applied by the next CGP kernel or the flush)
    int* xbuf;        // which p buffer holds the p of xalpha (0/1)
    int* active;      // 1 = still iterating
    int* iters;
    int* done;        // 1 = no active RHS
    int* status;      // bit0 breakdown
};

__device__ __forceinline__ double shfl_up1(double v) { return __shfl_up_sync(MGK_FULL, v, 1); }
__device__ __forceinline__ double shfl_dn1(double v) { return __shfl_down_sync(MGK_FULL, v, 1); }

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(MGK_FULL, v, o);
    return v;
}

// ---- programmatic dependent launch (PDL) for the kernels of the CG iteration graphs.
// A kernel launched with launch_k() may start while its predecessor in the stream is finishing:
// its first statement is pdl_begin(), which waits until the predecessor grid has completed and
// its memory is visible (griddepcontrol.wait), then lets the next dependent grid begin launching
// (griddepcontrol.launch_dependents).  Launch latency overlaps the previous kernel's tail; the
// data dependencies are unchanged.  Outside a PDL launch both instructions are no-ops.  Used for
// the 2D iteration (march2, coarse2d) and the small scalar / dense kernels: B200 C1 -5%, C2 -3%;
// the 3D kernels (H8, stencil, transfers, r update) launch without it -- early-resident dependents
// of their large grids cost the 3D configs ~1%.
__device__ __forceinline__ void pdl_begin() {
    asm volatile("griddepcontrol.wait;\n" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
}

bool pdl_enabled();   // MG_PDL (default 1)

template <typename... KArgs, typename... Args>
inline void launch_kp(bool pdl, void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                      Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = (pdl && pdl_enabled()) ? 1 : 0;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

template <typename... KArgs, typename... Args>
inline void launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args... args) {
    launch_kp(true, kern, grid, block, smem, s, args...);
}
