// Adjoint right-hand sides and eigenvalue sensitivities:
//
//   mg_adjoint_rhs       b_i = phi_i^T (grad_u G) phi_i              Eq. 5
//   mg_eigen_sensitivity s_ie = dEk_e (k_ie - lam_i kz_ie) + lam_i dEs_e g_ie   Eq. 4 (:126-130)
//                        k = phi_e^T K0 phi_e, g = phi_e^T G0[u_e] phi_e, kz = z_e^T K0 u_e
//
// With G_e0[u_e] = (sum_ij sigma_ij H_ij) kron I_d and sigma = D0 B(c) u_e (reading r15),
// phi_e^T G_e0 phi_e = sum_v sigma_v P_v(phi_e) with P_v = sum_ab H_v[a][b] (phi_a . phi_b)
// (H_v = H_ii for normal, H_ij + H_ji for shear components).  The form is linear in u_e, so its
// gradient is B(c)^T D0 P(phi_e), independent of u: the adjoint RHS is
//   b = F sum_e A_e^T Es_e B(c)^T D0 P(F phi_e)          (F = free-DOF mask)
// computed as w_e = Es_e D0 P(phi_e) per element (3 / 6 numbers) and a node gather of B(c)^T w
// over the 2^d adjacent elements (no atomics).
#include "kernels.h"

__constant__ double c_sK0[576];
__constant__ double c_sD0[36];
__constant__ double c_sH[3 * 3 * 8 * 8];   // H[i][j][a][b]

void sens_set_constants(int dim, const double* K0, double nu, cudaStream_t s) {
    const int nl = dim * (1 << dim);
    cudaMemcpyToSymbolAsync(c_sK0, K0, sizeof(double) * nl * nl, 0, cudaMemcpyHostToDevice, s);
    double D0[36] = {0};
    if (dim == 2) {
        const double c = 1.0 / (1.0 - nu * nu);
        const double m[9] = {c, c * nu, 0, c * nu, c, 0, 0, 0, c * (1 - nu) / 2};
        for (int i = 0; i < 9; ++i) D0[i] = m[i];
    } else {
        const double lam = nu / ((1 + nu) * (1 - 2 * nu)), mu = 1.0 / (2 * (1 + nu));
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j) D0[i * 6 + j] = lam + (i == j ? 2 * mu : 0.0);
        for (int i = 3; i < 6; ++i) D0[i * 6 + i] = mu;
    }
    // H_ij[a][b] = int dN_a/dx_i dN_b/dx_j: products of 1-D integrals M, D, C on [0, 1]
    static double H[3 * 3 * 8 * 8];
    const double M[2][2] = {{1.0 / 3, 1.0 / 6}, {1.0 / 6, 1.0 / 3}};
    const double Dd[2][2] = {{1.0, -1.0}, {-1.0, 1.0}};
    const double C[2][2] = {{-0.5, -0.5}, {0.5, 0.5}};
    const int na = 1 << dim;
    for (int i = 0; i < dim; ++i)
        for (int j = 0; j < dim; ++j)
            for (int a = 0; a < na; ++a)
                for (int b = 0; b < na; ++b) {
                    double v = 1.0;
                    for (int k = 0; k < dim; ++k) {
                        const int ak = (a >> (dim - 1 - k)) & 1, bk = (b >> (dim - 1 - k)) & 1;
                        if (k == i && k == j) v *= Dd[ak][bk];
                        else if (k == i) v *= C[ak][bk];
                        else if (k == j) v *= C[bk][ak];
                        else v *= M[ak][bk];
                    }
                    H[((i * 3 + j) * 8 + a) * 8 + b] = v;
                }
    cudaMemcpyToSymbolAsync(c_sD0, D0, sizeof(D0), 0, cudaMemcpyHostToDevice, s);
    cudaMemcpyToSymbolAsync(c_sH, H, sizeof(H), 0, cudaMemcpyHostToDevice, s);
}

template <int DIM>
struct Voigt {
    static constexpr int NV = DIM == 2 ? 3 : 6;
    // component v -> (i, j)
    __device__ static void ij(int v, int& i, int& j) {
        if (v < DIM) { i = j = v; return; }
        if (DIM == 2) { i = 0; j = 1; return; }
        const int s = v - 3;   // 3: (1,2) 4: (0,2) 5: (0,1)
        i = s == 2 ? 0 : (s == 1 ? 0 : 1);
        j = s == 0 ? 2 : (s == 1 ? 2 : 1);
    }
};

// local element data: node a of element (coords ec) -> global node index
template <int DIM>
__device__ __forceinline__ long long elem_node(const LevelGeom& g, const int* ec, int a) {
    long long nd = 0;
#pragma unroll
    for (int k = 0; k < DIM; ++k) nd = nd * g.nn[k] + ec[k] + ((a >> (DIM - 1 - k)) & 1);
    return nd;
}

// P_v(phi_e) for masked element vector pe[a][k]
template <int DIM>
__device__ __forceinline__ void form_P(const double (*pe)[DIM], double* P) {
    constexpr int NA = 1 << DIM, NV = Voigt<DIM>::NV;
    double dotab[NA][NA];
#pragma unroll
    for (int a = 0; a < NA; ++a)
#pragma unroll
        for (int b = 0; b < NA; ++b) {
            double s = 0.0;
#pragma unroll
            for (int k = 0; k < DIM; ++k) s = fma(pe[a][k], pe[b][k], s);
            dotab[a][b] = s;
        }
#pragma unroll
    for (int v = 0; v < NV; ++v) {
        int i, j;
        Voigt<DIM>::ij(v, i, j);
        double s = 0.0;
#pragma unroll
        for (int a = 0; a < NA; ++a)
#pragma unroll
            for (int b = 0; b < NA; ++b) {
                double h = c_sH[((i * 3 + j) * 8 + a) * 8 + b];
                if (i != j) h += c_sH[((j * 3 + i) * 8 + a) * 8 + b];
                s = fma(h, dotab[a][b], s);
            }
        P[v] = s;
    }
}

// dN_a/dx_j at the centroid: +-(1/2)^(d-1)
template <int DIM>
__device__ __forceinline__ double cgrad(int a, int j) {
    const double h = DIM == 2 ? 0.5 : 0.25;
    return ((a >> (DIM - 1 - j)) & 1) ? h : -h;
}

// w[r][e][v] = Es_e (D0 P(phi_r,e))_v
template <int DIM>
__global__ void adjoint_w_kernel(LevelGeom g, const double* __restrict__ Es, const uint8_t* __restrict__ mask,
                                 const double* __restrict__ phi, int nphi, double* __restrict__ w) {
    constexpr int NA = 1 << DIM, NV = Voigt<DIM>::NV;
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= g.nelem) return;
    int ec[3] = {0, 0, 0};
    long long t = e;
    for (int k = DIM - 1; k >= 0; --k) { ec[k] = (int)(t % g.N[k]); t /= g.N[k]; }
    long long nd[NA];
    int mb[NA];
#pragma unroll
    for (int a = 0; a < NA; ++a) { nd[a] = elem_node<DIM>(g, ec, a); mb[a] = mask[nd[a]]; }
    const double es = Es[e];
    for (int r = 0; r < nphi; ++r) {
        const double* pv = phi + (long long)r * g.ndof;
        double pe[NA][DIM];
#pragma unroll
        for (int a = 0; a < NA; ++a)
#pragma unroll
            for (int k = 0; k < DIM; ++k) pe[a][k] = ((mb[a] >> k) & 1) ? 0.0 : pv[DIM * nd[a] + k];
        double P[NV];
        form_P<DIM>(pe, P);
#pragma unroll
        for (int v = 0; v < NV; ++v) {
            double s = 0.0;
#pragma unroll
            for (int q = 0; q < NV; ++q) s = fma(c_sD0[v * NV + q], P[q], s);
            w[((long long)r * g.nelem + e) * NV + v] = es * s;
        }
    }
}

// b[r][node][k] = free * sum_{e at node} (B(c)^T w_e)[(a, k)]
template <int DIM>
__global__ void adjoint_gather_kernel(LevelGeom g, const uint8_t* __restrict__ mask, const double* __restrict__ w,
                                      int nphi, double* __restrict__ b) {
    constexpr int NA = 1 << DIM, NV = Voigt<DIM>::NV;
    const long long node = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (node >= g.nnodes) return;
    int idx[3] = {0, 0, 0};
    long long t = node;
    for (int k = DIM - 1; k >= 0; --k) { idx[k] = (int)(t % g.nn[k]); t /= g.nn[k]; }
    const int mb = mask[node];
    for (int r = 0; r < nphi; ++r) {
        double acc[DIM];
#pragma unroll
        for (int k = 0; k < DIM; ++k) acc[k] = 0.0;
#pragma unroll
        for (int a = 0; a < NA; ++a) {   // this node is local node a of element idx - bits(a)
            int ec[3];
            bool ok = true;
#pragma unroll
            for (int k = 0; k < DIM; ++k) {
                ec[k] = idx[k] - ((a >> (DIM - 1 - k)) & 1);
                ok = ok && ec[k] >= 0 && ec[k] < g.N[k];
            }
            if (!ok) continue;
            long long e = ec[0];
#pragma unroll
            for (int k = 1; k < DIM; ++k) e = e * g.N[k] + ec[k];
            const double* we = w + ((long long)r * g.nelem + e) * NV;
#pragma unroll
            for (int v = 0; v < NV; ++v) {
                int i, j;
                Voigt<DIM>::ij(v, i, j);
                const double wv = we[v];
                if (i == j) {
                    acc[i] = fma(cgrad<DIM>(a, i), wv, acc[i]);
                } else {   // engineering shear: du_i/dx_j + du_j/dx_i
                    acc[i] = fma(cgrad<DIM>(a, j), wv, acc[i]);
                    acc[j] = fma(cgrad<DIM>(a, i), wv, acc[j]);
                }
            }
        }
        double* bv = b + (long long)r * g.ndof + DIM * node;
#pragma unroll
        for (int k = 0; k < DIM; ++k) bv[k] = ((mb >> k) & 1) ? 0.0 : acc[k];
    }
}

// s[r][e] = dEk_e (phi^T K0 phi - lam_r z^T K0 u) + lam_r dEs_e phi^T G0[u_e] phi
template <int DIM>
__global__ void sens_kernel(LevelGeom g, const double* __restrict__ dEk, const double* __restrict__ dEs,
                            const uint8_t* __restrict__ mask, const double* __restrict__ u,
                            const double* __restrict__ phi, const double* __restrict__ z,
                            const double* __restrict__ lam, int nphi, double* __restrict__ s) {
    constexpr int NA = 1 << DIM, NV = Voigt<DIM>::NV, NL = DIM * NA;
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= g.nelem) return;
    int ec[3] = {0, 0, 0};
    long long t = e;
    for (int k = DIM - 1; k >= 0; --k) { ec[k] = (int)(t % g.N[k]); t /= g.N[k]; }
    long long nd[NA];
    int mb[NA];
#pragma unroll
    for (int a = 0; a < NA; ++a) { nd[a] = elem_node<DIM>(g, ec, a); mb[a] = mask[nd[a]]; }
    // state: sigma0 = D0 B(c) u_e (unmasked u), K0 u_e (masked u)
    double ue[NL], uf[NL];
#pragma unroll
    for (int a = 0; a < NA; ++a)
#pragma unroll
        for (int k = 0; k < DIM; ++k) {
            ue[DIM * a + k] = u[DIM * nd[a] + k];
            uf[DIM * a + k] = ((mb[a] >> k) & 1) ? 0.0 : ue[DIM * a + k];
        }
    double eps[NV];
#pragma unroll
    for (int v = 0; v < NV; ++v) {
        int i, j;
        Voigt<DIM>::ij(v, i, j);
        double sv = 0.0;
#pragma unroll
        for (int a = 0; a < NA; ++a) {
            if (i == j) sv = fma(cgrad<DIM>(a, i), ue[DIM * a + i], sv);
            else sv = fma(cgrad<DIM>(a, j), ue[DIM * a + i], fma(cgrad<DIM>(a, i), ue[DIM * a + j], sv));
        }
        eps[v] = sv;
    }
    double sig[NV];
#pragma unroll
    for (int v = 0; v < NV; ++v) {
        double sv = 0.0;
#pragma unroll
        for (int q = 0; q < NV; ++q) sv = fma(c_sD0[v * NV + q], eps[q], sv);
        sig[v] = sv;
    }
    double Ku[NL];
#pragma unroll
    for (int p = 0; p < NL; ++p) {
        double sv = 0.0;
#pragma unroll
        for (int q = 0; q < NL; ++q) sv = fma(c_sK0[p * NL + q], uf[q], sv);
        Ku[p] = sv;
    }
    const double dk = dEk[e], ds = dEs[e];
    for (int r = 0; r < nphi; ++r) {
        const double* pv = phi + (long long)r * g.ndof;
        const double* zv = z + (long long)r * g.ndof;
        double pe[NA][DIM];
        double kz = 0.0;
#pragma unroll
        for (int a = 0; a < NA; ++a)
#pragma unroll
            for (int k = 0; k < DIM; ++k) {
                const bool fx = (mb[a] >> k) & 1;
                pe[a][k] = fx ? 0.0 : pv[DIM * nd[a] + k];
                kz = fma(fx ? 0.0 : zv[DIM * nd[a] + k], Ku[DIM * a + k], kz);
            }
        double kp = 0.0;
#pragma unroll
        for (int p = 0; p < NL; ++p) {
            double sv = 0.0;
#pragma unroll
            for (int q = 0; q < NL; ++q) sv = fma(c_sK0[p * NL + q], pe[q / DIM][q % DIM], sv);
            kp = fma(pe[p / DIM][p % DIM], sv, kp);
        }
        double P[NV];
        form_P<DIM>(pe, P);
        double gp = 0.0;
#pragma unroll
        for (int v = 0; v < NV; ++v) gp = fma(sig[v], P[v], gp);
        const double l = lam[r];
        s[(long long)r * g.nelem + e] = fma(dk, kp - l * kz, l * ds * gp);
    }
}

void adjoint_rhs_apply(const LevelGeom& g, const double* Es, const uint8_t* mask, const double* phi, int nphi,
                       double* w, double* b, cudaStream_t s) {
    const int th = 128;
    if (g.dim == 2) {
        adjoint_w_kernel<2><<<(unsigned)((g.nelem + th - 1) / th), th, 0, s>>>(g, Es, mask, phi, nphi, w);
        adjoint_gather_kernel<2><<<(unsigned)((g.nnodes + th - 1) / th), th, 0, s>>>(g, mask, w, nphi, b);
    } else {
        adjoint_w_kernel<3><<<(unsigned)((g.nelem + th - 1) / th), th, 0, s>>>(g, Es, mask, phi, nphi, w);
        adjoint_gather_kernel<3><<<(unsigned)((g.nnodes + th - 1) / th), th, 0, s>>>(g, mask, w, nphi, b);
    }
}

void eigen_sensitivity_apply(const LevelGeom& g, const double* dEk, const double* dEs, const uint8_t* mask,
                             const double* u, const double* phi, const double* z, const double* lam, int nphi,
                             double* out, cudaStream_t s) {
    const int th = 128;
    const unsigned bl = (unsigned)((g.nelem + th - 1) / th);
    if (g.dim == 2) sens_kernel<2><<<bl, th, 0, s>>>(g, dEk, dEs, mask, u, phi, z, lam, nphi, out);
    else sens_kernel<3><<<bl, th, 0, s>>>(g, dEk, dEs, mask, u, phi, z, lam, nphi, out);
}
