// Unit-element stiffness K_e0 as a constexpr function (standard bilinear Q4 in plane
// stress / trilinear H8, exact integration; PAPER.md:99, :111 reading r1):
//   K0[(a,i),(b,j)] = lam S_ij[a,b] + mu S_ji[a,b] + mu delta_ij sum_k S_kk[a,b],
//   S_ij[a,b] = int_{[0,1]^d} dN_a/dx_i dN_b/dx_j  = prod_k (1-D integral on [0,1]).
// With nu a compile-time constant the entries fold to immediates / constant-bank
// operands, so the hot kernels keep no K0 registers.
#pragma once

__host__ __device__ constexpr double s1d(int kind, int a, int b) {
    // kind 0: M[a][b] = int phi_a phi_b; 1: D = int phi_a' phi_b'; 2: C[a][b] = int phi_a' phi_b; 3: C[b][a]
    return kind == 0 ? (a == b ? 1.0 / 3.0 : 1.0 / 6.0)
         : kind == 1 ? (a == b ? 1.0 : -1.0)
         : kind == 2 ? (a == 0 ? -0.5 : 0.5)
                     : (b == 0 ? -0.5 : 0.5);
}

template <int DIM>
__host__ __device__ constexpr double s_ij(int i, int j, int a, int b) {
    double v = 1.0;
    for (int k = 0; k < DIM; ++k) {
        const int ak = (a >> (DIM - 1 - k)) & 1, bk = (b >> (DIM - 1 - k)) & 1;
        const int kind = (k == i && k == j) ? 1 : (k == i ? 2 : (k == j ? 3 : 0));
        v *= s1d(kind, ak, bk);
    }
    return v;
}

template <int DIM>
__host__ __device__ constexpr double k0_entry(double nu, int row, int col) {
    const int a = row / DIM, i = row % DIM, b = col / DIM, j = col % DIM;
    const double mu = 1.0 / (2.0 * (1.0 + nu));
    const double lam = DIM == 2 ? nu / (1.0 - nu * nu) : nu / ((1.0 + nu) * (1.0 - 2.0 * nu));
    double v = lam * s_ij<DIM>(i, j, a, b) + mu * s_ij<DIM>(j, i, a, b);
    if (i == j)
        for (int k = 0; k < DIM; ++k) v += mu * s_ij<DIM>(k, k, a, b);
    return v;
}

// The paper's Poisson ratio ("the Poisson ratio is fixed to nu = 0.3").
#define MG_NU_PAPER 0.3
