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
