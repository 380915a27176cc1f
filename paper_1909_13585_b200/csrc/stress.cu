// Stress-stiffness product y = G(u) phi ("G_e = E_sigma(x_e) G_e0[u_e]",
// Eq. 2 :106; used as the RHS G Psi of Eq. 6 :163 and in the residual Eq. 7 :181;
// SURVEY 8(a) a8, reading r15):
//   sigma_e = Es_e D0 B(centroid) u_e                       (stress_sigma)
//   G_e     = (sum_ij sigma_e,ij H_ij) kron I_d,  H_ij[a,b] = int dN_a/dx_i dN_b/dx_j
//   y       = F (sum_e A_e^T G_e A_e) F phi,  F = free-DOF mask  (stress_apply)
// Because G_e = S_e kron I_d, every displacement component sees the same scalar
// 2^d x 2^d element matrix S_e: the apply kernel forms the two rows of S_e it needs
// per element from sigma_e (3 or 6 doubles) and applies them to all d components.
// Layout and march are those of the fine matvec (fine_ops.cu): warp = 30 node
// columns, march along axis 0, phi index fastest in the grid.
#include <algorithm>
#include <cstdint>
#include <cstdlib>

#include "kernels.h"

__constant__ double c_D0[36];          // Voigt constitutive matrix, E = 1
__constant__ double c_H[3 * 3 * 8 * 8];  // H[i][j][a][b]

static constexpr int SCOLS = 30;
static constexpr int SCH2 = 32, SCH3 = 16;

// Closed-form H_ij as products of 1-D integrals over [0,1] with phi0 = 1 - t, phi1 = t:
// M = [[1/3,1/6],[1/6,1/3]], D = [[1,-1],[-1,1]], C[a][b] = int phi_a' phi_b.
static double h1d(int kind, int a, int b) {
    static const double M[2][2] = {{1.0 / 3, 1.0 / 6}, {1.0 / 6, 1.0 / 3}};
    static const double D[2][2] = {{1.0, -1.0}, {-1.0, 1.0}};
    static const double C[2][2] = {{-0.5, -0.5}, {0.5, 0.5}};
    if (kind == 0) return M[a][b];
    if (kind == 1) return D[a][b];
    if (kind == 2) return C[a][b];
    return C[b][a];
}

void stress_set_constants(int dim, double nu, cudaStream_t s) {
    double D0[36] = {0};
    if (dim == 2) {
        double c = 1.0 / (1.0 - nu * nu);
        double m[9] = {c, c * nu, 0, c * nu, c, 0, 0, 0, c * (1 - nu) / 2};
        for (int i = 0; i < 9; ++i) D0[i] = m[i];
    } else {
        double lam = nu / ((1 + nu) * (1 - 2 * nu)), mu = 1.0 / (2 * (1 + nu));
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j) D0[i * 6 + j] = lam + (i == j ? 2 * mu : 0.0);
        for (int i = 3; i < 6; ++i) D0[i * 6 + i] = mu;
    }
    static double H[3 * 3 * 8 * 8];
    int na = 1 << dim;
    for (int i = 0; i < dim; ++i)
        for (int j = 0; j < dim; ++j)
            for (int a = 0; a < na; ++a)
                for (int b = 0; b < na; ++b) {
                    double v = 1.0;
                    for (int k = 0; k < dim; ++k) {
                        int ak = (a >> (dim - 1 - k)) & 1, bk = (b >> (dim - 1 - k)) & 1;
                        int kind = (k == i && k == j) ? 1 : (k == i ? 2 : (k == j ? 3 : 0));
                        v *= h1d(kind, ak, bk);
                    }
                    H[((i * 3 + j) * 8 + a) * 8 + b] = v;
                }
    cudaMemcpyToSymbolAsync(c_D0, D0, sizeof(D0), 0, cudaMemcpyHostToDevice, s);
    cudaMemcpyToSymbolAsync(c_H, H, sizeof(H), 0, cudaMemcpyHostToDevice, s);
}

// sigma (Voigt: 2D [s00, s11, s01]; 3D [s00, s11, s22, s12, s02, s01]) per element, times Es_e.
template <int DIM>
__global__ void sigma_kernel(LevelGeom g, const double* __restrict__ Es, const double* __restrict__ u,
                             double* __restrict__ sig) {
    constexpr int NA = 1 << DIM, NV = DIM == 2 ? 3 : 6;
    long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= g.nelem) return;
    int ei[3] = {0, 0, 0};
    long long t = e;
    for (int k = DIM - 1; k >= 0; --k) { ei[k] = (int)(t % g.N[k]); t /= g.N[k]; }
    double grad[DIM][DIM];   // grad[i][j] = du_i/dx_j at the centroid
#pragma unroll
    for (int i = 0; i < DIM; ++i)
#pragma unroll
        for (int j = 0; j < DIM; ++j) grad[i][j] = 0.0;
    const double hw = DIM == 2 ? 0.5 : 0.25;   // |dN_a/dx_j| at the centroid
#pragma unroll
    for (int a = 0; a < NA; ++a) {
        long long node = 0;
#pragma unroll
        for (int k = 0; k < DIM; ++k) node = node * g.nn[k] + ei[k] + ((a >> (DIM - 1 - k)) & 1);
#pragma unroll
        for (int i = 0; i < DIM; ++i) {
            const double ui = u[DIM * node + i];
#pragma unroll
            for (int j = 0; j < DIM; ++j) {
                const double sgn = ((a >> (DIM - 1 - j)) & 1) ? hw : -hw;
                grad[i][j] = fma(sgn, ui, grad[i][j]);
            }
        }
    }
    double eps[NV];
    if (DIM == 2) {
        eps[0] = grad[0][0]; eps[1] = grad[1][1]; eps[2] = grad[0][1] + grad[1][0];
    } else {
        eps[0] = grad[0][0]; eps[1] = grad[1][1]; eps[2] = grad[2][2];
        eps[3] = grad[1][2] + grad[2][1]; eps[4] = grad[0][2] + grad[2][0]; eps[5] = grad[0][1] + grad[1][0];
    }
    const double es = Es[e];
#pragma unroll
    for (int v = 0; v < NV; ++v) {
        double s = 0.0;
#pragma unroll
        for (int w = 0; w < NV; ++w) s = fma(c_D0[v * NV + w], eps[w], s);
        sig[e * NV + v] = es * s;
    }
}

void stress_sigma(const LevelGeom& g, const double* Es, const double* u, double* sig, cudaStream_t s) {
    int th = 128;
    unsigned bl = (unsigned)((g.nelem + th - 1) / th);
    if (g.dim == 2) sigma_kernel<2><<<bl, th, 0, s>>>(g, Es, u, sig);
    else sigma_kernel<3><<<bl, th, 0, s>>>(g, Es, u, sig);
}

// S_e[a][b] = sum_ij sigma_ij H_ij[a][b] (sigma symmetric)
template <int DIM>
__device__ __forceinline__ double s_entry(const double* sg, int a, int b) {
    constexpr int NV = DIM == 2 ? 3 : 6;
    double v = 0.0;
#pragma unroll
    for (int i = 0; i < DIM; ++i) v = fma(sg[i], c_H[((i * 3 + i) * 8 + a) * 8 + b], v);
    if (DIM == 2) {
        v = fma(sg[2], c_H[((0 * 3 + 1) * 8 + a) * 8 + b] + c_H[((1 * 3 + 0) * 8 + a) * 8 + b], v);
    } else {
        v = fma(sg[3], c_H[((1 * 3 + 2) * 8 + a) * 8 + b] + c_H[((2 * 3 + 1) * 8 + a) * 8 + b], v);
        v = fma(sg[4], c_H[((0 * 3 + 2) * 8 + a) * 8 + b] + c_H[((2 * 3 + 0) * 8 + a) * 8 + b], v);
        v = fma(sg[5], c_H[((0 * 3 + 1) * 8 + a) * 8 + b] + c_H[((1 * 3 + 0) * 8 + a) * 8 + b], v);
    }
    (void)NV;
    return v;
}

template <int DIM>
__global__ void __launch_bounds__(128) stress_apply_kernel(LevelGeom g, const double* __restrict__ sig,
                                                           const uint8_t* __restrict__ mask,
                                                           const double* __restrict__ phi, double* __restrict__ y,
                                                           int nphi, int nct, int nch) {
    constexpr int NV = DIM == 2 ? 3 : 6;
    constexpr int CH = DIM == 2 ? SCH2 : SCH3;
    constexpr int NJ = DIM == 2 ? 1 : 3;      // rows j-1..j+1 in 3D
    constexpr int NE = DIM == 2 ? 1 : 2;      // element rows in 3D
    const int lane = threadIdx.x & 31;
    const long long w = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int n0 = g.nn[0], n1 = g.nn[1];
    const int nlast = g.nn[DIM - 1], Nlast = g.N[DIM - 1];
    const int nrow = DIM == 2 ? 1 : n1;
    const int items = nct * nch * nrow;
    if (w >= (long long)nphi * items) return;
    const int r = (int)(w % nphi);
    const int item = (int)(w / nphi);
    const int ct = item % nct;
    const int j = DIM == 2 ? 0 : (item / nct) % n1;
    const int ch = item / (nct * nrow);
    const int c = ct * SCOLS + lane - 1;
    const bool cin = c >= 0 && c < nlast;
    const bool own = cin && lane >= 1 && lane <= SCOLS;
    const int i0 = ch * CH, i1 = min(i0 + CH, n0);
    const long long vbase = (long long)r * g.ndof;

    double A[NJ][3][DIM], B[NJ][3][DIM];
    int mOwnA = 0, mOwnB = 0;
    double carry[DIM];
#pragma unroll
    for (int k = 0; k < DIM; ++k) carry[k] = 0.0;

    auto node_of = [&](int P, int jj) -> long long {
        return DIM == 2 ? (long long)P * n1 + c : ((long long)P * n1 + jj) * nlast + c;
    };
    auto load_plane = [&](int P, double (&W)[NJ][3][DIM], int& mown) {
#pragma unroll
        for (int dj = 0; dj < NJ; ++dj) {
            const int jj = DIM == 2 ? 0 : j + dj - 1;
            const bool v = cin && P >= 0 && P < n0 && (DIM == 2 || (jj >= 0 && jj < n1));
            double m[DIM];
            int mb = (1 << DIM) - 1;
            if (v) {
                const long long nd = node_of(P, jj);
                mb = mask[nd];
#pragma unroll
                for (int k = 0; k < DIM; ++k) m[k] = ((mb >> k) & 1) ? 0.0 : phi[vbase + DIM * nd + k];
            } else {
#pragma unroll
                for (int k = 0; k < DIM; ++k) m[k] = 0.0;
            }
            if (dj == NJ / 2) mown = mb;
#pragma unroll
            for (int k = 0; k < DIM; ++k) { W[dj][1][k] = m[k]; W[dj][0][k] = shfl_up1(m[k]); W[dj][2][k] = shfl_dn1(m[k]); }
        }
    };

    load_plane(i0 - 1, A, mOwnA);
    for (int L = i0 - 1; L < i1; ++L) {
        load_plane(L + 1, B, mOwnB);
        double sg[NE][2][NV];
#pragma unroll
        for (int ej = 0; ej < NE; ++ej) {
            const int je = DIM == 2 ? 0 : j - 1 + ej;
            const bool ok = L >= 0 && L < g.N[0] && c >= 0 && c < Nlast && (DIM == 2 || (je >= 0 && je < g.N[1]));
            const long long el = DIM == 2 ? (long long)L * g.N[1] + c : ((long long)L * g.N[1] + je) * Nlast + c;
#pragma unroll
            for (int v = 0; v < NV; ++v) {
                const double sv = ok ? sig[el * NV + v] : 0.0;
                const double svl = shfl_up1(sv);
                sg[ej][1][v] = sv;
                sg[ej][0][v] = (c - 1 >= 0) ? svl : 0.0;
            }
        }
        double lo[DIM], hi[DIM];
#pragma unroll
        for (int k = 0; k < DIM; ++k) { lo[k] = carry[k]; hi[k] = 0.0; }
#pragma unroll
        for (int ej = 0; ej < NE; ++ej)
#pragma unroll
            for (int ec = 0; ec < 2; ++ec) {
                const int a1 = 1 - ej, a2 = 1 - ec;
                const int alo = DIM == 2 ? (0 * 2 + a2) : ((0 * 2 + a1) * 2 + a2);
                const int ahi = DIM == 2 ? (1 * 2 + a2) : ((1 * 2 + a1) * 2 + a2);
#pragma unroll
                for (int b = 0; b < (1 << DIM); ++b) {
                    const int b0 = b >> (DIM - 1);
                    const int b1 = DIM == 2 ? 0 : (b >> 1) & 1;
                    const int b2 = b & 1;
                    const double slo = s_entry<DIM>(sg[ej][ec], alo, b);
                    const double shi = s_entry<DIM>(sg[ej][ec], ahi, b);
                    const int rj = DIM == 2 ? 0 : ej + b1;
#pragma unroll
                    for (int k = 0; k < DIM; ++k) {
                        const double xv = b0 ? B[rj][ec + b2][k] : A[rj][ec + b2][k];
                        lo[k] = fma(slo, xv, lo[k]);
                        hi[k] = fma(shi, xv, hi[k]);
                    }
                }
            }
        if (own && L >= i0) {
            const long long o = vbase + DIM * node_of(L, j);
#pragma unroll
            for (int k = 0; k < DIM; ++k) y[o + k] = ((mOwnA >> k) & 1) ? 0.0 : lo[k];
        }
#pragma unroll
        for (int k = 0; k < DIM; ++k) carry[k] = hi[k];
#pragma unroll
        for (int q = 0; q < NJ; ++q)
#pragma unroll
            for (int s = 0; s < 3; ++s)
#pragma unroll
                for (int k = 0; k < DIM; ++k) A[q][s][k] = B[q][s][k];
        mOwnA = mOwnB;
    }
}

// ---------------------------------------------------------------- 2D: sum/difference-basis march
// y = G(u) phi in 2D with the element matrix in the per-axis (m, d) basis (as the Q4 stiffness in
// fine2d.cu): S^ = sum_ij sigma_ij H^_ij has 5 nonzeros (rows / cols of the (m, m) mode are zero).
// A warp owns 30 node columns (lanes 1..30) of one phi and marches along axis 0; the next PD
// planes of phi (one 16-byte load per node), masks and the element stresses (3 per element) are
// prefetched into registers; column neighbours by shuffles, the axis-0 half of each element
// result carried to the next plane.  Reads phi and sigma once, writes y once.
__host__ __device__ constexpr double s2f(int kind, int ta, int tb) {   // 1-D factors in the (m, d) basis
    return kind == 0 ? (ta == tb ? (ta == 0 ? 0.25 : 1.0 / 12.0) : 0.0)
         : kind == 1 ? ((ta == 1 && tb == 1) ? 1.0 : 0.0)
         : kind == 2 ? ((ta == 1 && tb == 0) ? 0.5 : 0.0)
                     : ((ta == 0 && tb == 1) ? 0.5 : 0.0);
}
__host__ __device__ constexpr double s2h(int i, int j, int s, int t) {   // H^_ij[s][t]
    double v = 1.0;
    for (int k = 0; k < 2; ++k) {
        const int ta = (s >> (1 - k)) & 1, tb = (t >> (1 - k)) & 1;
        const int kind = (k == i && k == j) ? 1 : (k == i ? 2 : (k == j ? 3 : 0));
        v *= s2f(kind, ta, tb);
    }
    return v;
}

static constexpr int G2_PD = 3;    // planes prefetched

__global__ void __launch_bounds__(128) stress2_kernel(LevelGeom g, const double* __restrict__ sig,
                                                      const uint8_t* __restrict__ mask, const double* __restrict__ phi,
                                                      double* __restrict__ y, int nphi, int nct, int nch, int hch) {
    const int lane = threadIdx.x & 31;
    const long long w = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (w >= (long long)nphi * nct * nch) return;
    const int r = (int)(w % nphi);
    const int item = (int)(w / nphi);
    const int ct = item % nct, ch = item / nct;
    const int n0 = g.nn[0], n1 = g.nn[1], N0 = g.N[0], N1 = g.N[1];
    const int c = 30 * ct + lane - 1;
    const bool cin = c >= 0 && c < n1;
    const bool own = cin && lane >= 1 && lane <= 30;
    const bool ein = c >= 0 && c < N1 && lane < 31;
    const int i0 = ch * hch, i1 = min(i0 + hch, n0);
    const double2* ph = reinterpret_cast<const double2*>(phi + (long long)r * g.ndof);
    // prefetch ring: phi of node (P, c), its mask, sigma of element (P, c)
    double2 rp[G2_PD];
    int rm[G2_PD];
    double rs[G2_PD][3];
    auto load = [&](int P, int q) {
        const bool v = cin && P >= 0 && P < n0;
        const long long nd = v ? (long long)P * n1 + c : 0;
        rm[q] = v ? mask[nd] : 3;
        rp[q] = v ? __ldg(ph + nd) : make_double2(0.0, 0.0);
        const bool ve = ein && P >= 0 && P < N0;
        const long long el = ve ? (long long)P * N1 + c : 0;
#pragma unroll
        for (int v3 = 0; v3 < 3; ++v3) rs[q][v3] = ve ? __ldg(sig + 3 * el + v3) : 0.0;
    };
#pragma unroll
    for (int q = 0; q < G2_PD; ++q) load(i0 - 1 + q, q);
    double FL[2][2], CY[2][2];   // [comp][t1]: face (m, d along axis 1) of plane L; carry to plane P
    int mL;
    {
        const int m = rm[0];
        const double u0 = (m & 1) ? 0.0 : rp[0].x, u1 = (m & 2) ? 0.0 : rp[0].y;
        const double un0 = __shfl_down_sync(MGK_FULL, u0, 1), un1 = __shfl_down_sync(MGK_FULL, u1, 1);
        FL[0][0] = u0 + un0; FL[0][1] = un0 - u0;
        FL[1][0] = u1 + un1; FL[1][1] = un1 - u1;
        mL = m;
    }
    CY[0][0] = CY[0][1] = CY[1][0] = CY[1][1] = 0.0;
    double sgL[3] = {rs[0][0], rs[0][1], rs[0][2]};
    for (int L = i0 - 1; L < i1; ++L) {
        // rotate the ring: slot (L - i0 + 2) % PD holds plane L + 1
        const int q1 = ((L - i0 + 2) % G2_PD + G2_PD) % G2_PD;
        double2 pP = rp[0];
        int mP = rm[0];
        double sgP[3] = {rs[0][0], rs[0][1], rs[0][2]};
#pragma unroll
        for (int q = 0; q < G2_PD; ++q)
            if (q == q1) { pP = rp[q]; mP = rm[q]; sgP[0] = rs[q][0]; sgP[1] = rs[q][1]; sgP[2] = rs[q][2]; }
        // refill that slot with plane L + 1 + PD... (the slot of plane L is free: load L + PD)
        const int q0 = ((L - i0 + 1) % G2_PD + G2_PD) % G2_PD;
#pragma unroll
        for (int q = 0; q < G2_PD; ++q)
            if (q == q0) load(L + G2_PD, q);
        double FP[2][2];
        {
            const double u0 = (mP & 1) ? 0.0 : pP.x, u1 = (mP & 2) ? 0.0 : pP.y;
            const double un0 = __shfl_down_sync(MGK_FULL, u0, 1), un1 = __shfl_down_sync(MGK_FULL, u1, 1);
            FP[0][0] = u0 + un0; FP[0][1] = un0 - u0;
            FP[1][0] = u1 + un1; FP[1][1] = un1 - u1;
        }
        // element (L, c): S^ from sigma_L, u^ (s = 2 t0 + t1), y^ = S^ u^, per component
        double S[4][4];
#pragma unroll
        for (int a = 1; a < 4; ++a)
#pragma unroll
            for (int b = 1; b < 4; ++b) {
                double v = 0.0;
                bool first = true;
#pragma unroll
                for (int i = 0; i < 2; ++i)
#pragma unroll
                    for (int j = 0; j < 2; ++j) {
                        const double hv = s2h(i, j, a, b);
                        if (hv == 0.0) continue;
                        const double sv = (i == j) ? sgL[i] : sgL[2];
                        v = first ? sv * hv : fma(sv, hv, v);
                        first = false;
                    }
                S[a][b] = v;
            }
        double GL[2][2];
#pragma unroll
        for (int k = 0; k < 2; ++k) {
            double uh[4], yh[4];
            uh[1] = FL[k][1] + FP[k][1];   // (m, d)
            uh[2] = FP[k][0] - FL[k][0];   // (d, m)
            uh[3] = FP[k][1] - FL[k][1];   // (d, d)
#pragma unroll
            for (int a = 1; a < 4; ++a) {
                double v = 0.0;
                bool first = true;
#pragma unroll
                for (int b = 1; b < 4; ++b) {
                    bool nz = false;
#pragma unroll
                    for (int i = 0; i < 2; ++i)
#pragma unroll
                        for (int j = 0; j < 2; ++j) nz = nz || s2h(i, j, a, b) != 0.0;
                    if (!nz) continue;
                    v = first ? S[a][b] * uh[b] : fma(S[a][b], uh[b], v);
                    first = false;
                }
                yh[a] = v;
            }
            // axis 0: plane L gets ym - yd, plane P gets ym + yd (t1 = m: s = 0 / 2, t1 = d: s = 1 / 3)
            GL[k][0] = CY[k][0] - yh[2];
            CY[k][0] = yh[2];
            GL[k][1] = CY[k][1] + (yh[1] - yh[3]);
            CY[k][1] = yh[1] + yh[3];
        }
        // axis 1: node c gets fm - fd, node c + 1 gets fm + fd (from lane - 1)
        if (L >= i0) {
#pragma unroll
            for (int k = 0; k < 2; ++k) {
                const double up = __shfl_up_sync(MGK_FULL, GL[k][0] + GL[k][1], 1);
                const double v = (GL[k][0] - GL[k][1]) + (lane > 0 ? up : 0.0);
                if (own && ((mL >> k) & 1) == 0) y[(long long)r * g.ndof + 2 * ((long long)L * n1 + c) + k] = v;
                else if (own) y[(long long)r * g.ndof + 2 * ((long long)L * n1 + c) + k] = 0.0;
            }
        }
#pragma unroll
        for (int k = 0; k < 2; ++k) { FL[k][0] = FP[k][0]; FL[k][1] = FP[k][1]; }
        sgL[0] = sgP[0]; sgL[1] = sgP[1]; sgL[2] = sgP[2];
        mL = mP;
    }
}

void stress_apply(const LevelGeom& g, const double* sig, const uint8_t* mask, const double* phi, double* y, int nphi,
                  cudaStream_t s) {
    if (g.dim == 2 && ((uintptr_t)phi & 15) == 0 && !getenv("MG_STRESS2_LEGACY")) {
        const int nct = (g.nn[1] + 29) / 30;
        // chunks along axis 0 so the warp count fills whole waves of the resident warps (the
        // occupancy calculator's CTAs per SM x 4 warps x 148 SMs) with the least tail
        static int per_sm = [] {
            int nb = 0;
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, stress2_kernel, 128, 0);
            return std::max(1, nb) * 4;
        }();
        const long long slots = 148LL * per_sm;
        int nch = 1;
        double best = -1.0;
        for (int c = 1; c <= std::max(1, g.nn[0] / 16); ++c) {
            const int h = (g.nn[0] + c - 1) / c;
            const int cc = (g.nn[0] + h - 1) / h;
            const double waves = (double)nct * cc * nphi / slots;
            const double eff = waves / std::ceil(waves) * h / (h + 1.0);
            if (eff > best + 1e-9) { best = eff; nch = cc; }
        }
        const int hch = (g.nn[0] + nch - 1) / nch;
        const long long warps = (long long)nphi * nct * nch;
        stress2_kernel<<<(unsigned)((warps + 3) / 4), 128, 0, s>>>(g, sig, mask, phi, y, nphi, nct, nch, hch);
        return;
    }
    int ncols = g.nn[g.dim - 1];
    int nct = (ncols + SCOLS - 1) / SCOLS;
    int ch = g.dim == 2 ? SCH2 : SCH3;
    int nch = (g.nn[0] + ch - 1) / ch;
    int nrow = g.dim == 2 ? 1 : g.nn[1];
    long long warps = (long long)nphi * nct * nch * nrow;
    unsigned bl = (unsigned)((warps + 3) / 4);
    if (g.dim == 2) stress_apply_kernel<2><<<bl, 128, 0, s>>>(g, sig, mask, phi, y, nphi, nct, nch);
    else stress_apply_kernel<3><<<bl, 128, 0, s>>>(g, sig, mask, phi, y, nphi, nct, nch);
}
