// Fine-level (level 0) operator dispatch and diagonal ("K_e[x_e] = E_kappa(x_e) K_e0";
// SURVEY 8(a) a2/a3).  The operator itself is applied by fused march kernels with Dirichlet
// rows/columns replaced by identity (reading r11):
//   FOP_MATVEC  y = K x
//   FOP_RESID   y = b - K x                            (MG residual, true residual)
//   FOP_JACOBI  y = x + omega D^-1 (b - K x), dot(b,y)  (damped-Jacobi sweep)
//   FOP_CGP     p = z + beta p_in ; q = K p ; dot(p,q)  (CG direction update + matvec)
//   FOP_RESTR3  r = r_in - alpha q ; z1 = omega D^-1 r ; y = r - K z1 ; dot(r,r)
// 2D (Q4): fine2d.cu (march2 kernels on the padded 2D layout); 3D (H8): h8t.cu (TMA plane-ring
// march on the padded 3D layout).  This file keeps the 3D dispatch and the fine diagonal.
#include <cstdlib>

#include "kernels.h"

__constant__ double c_K0[576];

void fine_set_constants(int dim, const double* K0, cudaStream_t s) {
    int nl = dim * (1 << dim);
    cudaMemcpyToSymbolAsync(c_K0, K0, sizeof(double) * nl * nl, 0, cudaMemcpyHostToDevice, s);
}

int fine_items(const LevelGeom& g, int R) {
    if (g.dim == 2) return march2_items(M2_MATVEC, g, nullptr, R);
    return h8t_items(g, R);
}

// 3D only (2D goes through march2_apply); returns dot-partial items per RHS, or -1 if the
// kernel could not be launched (tensor-map encoding failed)
int fine_apply(int op, const FineArgs& a, cudaStream_t s) {
    if (a.g.dim != 3) return -1;
    return h8t_apply(op, a, s);
}

// D = diag(K): sum over adjacent elements E_e K0[(a,k),(a,k)]; 1 at fixed DOFs (identity rows).
template <int DIM>
__global__ void fine_diag_kernel(LevelGeom g, const double* __restrict__ E, const uint8_t* __restrict__ mask,
                                 double* Dinv, double* D) {
    long long node = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (node >= g.nnodes) return;
    int idx[3] = {0, 0, 0};
    long long t = node;
    for (int k = DIM - 1; k >= 0; --k) { idx[k] = (int)(t % g.nn[k]); t /= g.nn[k]; }
    const int NL = DIM * (1 << DIM);
    double acc[DIM];
#pragma unroll
    for (int k = 0; k < DIM; ++k) acc[k] = 0.0;
    for (int a = 0; a < (1 << DIM); ++a) {
        int e[3];
        bool ok = true;
        for (int k = 0; k < DIM; ++k) {
            int bit = (a >> (DIM - 1 - k)) & 1;
            e[k] = idx[k] - bit;
            if (e[k] < 0 || e[k] >= g.N[k]) ok = false;
        }
        if (!ok) continue;
        long long el = e[0];
        for (int k = 1; k < DIM; ++k) el = el * g.N[k] + e[k];
        const double Ev = E[el];
#pragma unroll
        for (int k = 0; k < DIM; ++k) acc[k] += Ev * c_K0[(a * DIM + k) * NL + a * DIM + k];
    }
    const int mb = mask[node];
#pragma unroll
    for (int k = 0; k < DIM; ++k) {
        double dv = ((mb >> k) & 1) ? 1.0 : acc[k];
        if (D) D[DIM * node + k] = dv;
        Dinv[DIM * node + k] = 1.0 / dv;
    }
}

void fine_diag(const LevelGeom& g, const double* E, const uint8_t* mask, double* Dinv, double* D, cudaStream_t s) {
    int th = 256;
    unsigned bl = (unsigned)((g.nnodes + th - 1) / th);
    if (g.dim == 2)
        fine_diag_kernel<2><<<bl, th, 0, s>>>(g, E, mask, Dinv, D);
    else
        fine_diag_kernel<3><<<bl, th, 0, s>>>(g, E, mask, Dinv, D);
}
