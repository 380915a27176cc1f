// Fine-level matrix-free element-by-element operator K = sum_e E_e A_e^T K0 A_e
// ("K_e[x_e] = E_kappa(x_e) K_e0"), with Dirichlet
// rows/columns replaced by identity (reading r11), fused with its consumers:
//   FOP_MATVEC  y = K x
//   FOP_RESID   y = b - K x                            (MG residual, true residual)
//   FOP_JACOBI  y = x + omega D^-1 (b - K x), dot(b,y)  (damped-Jacobi sweep)
//   FOP_CGP     p = z + beta p_in ; q = K p ; dot(p,q)  (CG direction update + matvec)
//
// Design (B200): node-centric gather, no colouring, no atomics, deterministic.
// One warp owns 30 node columns along the fastest axis (lanes 1..30; lanes 0/31
// are halo) and marches along axis 0 over a chunk of node planes.  Element layer
// L (between node planes L and L+1) contributes to planes L and L+1; the
// contribution to plane L+1 is carried in registers to the next step, so each
// element row-block is computed once per (node, element) pair and x is read once
// per plane.  Neighbours along the fastest axis come from warp shuffles; in 3D the
// warp also reads rows j-1, j+1 (served by L1/L2).  The RHS index is the fastest
// grid dimension so that the R warps working on one tile run together and E_e is
// read from HBM once per tile.
#include <cstdlib>

#include "kernels.h"

__constant__ double c_K0[576];

void fine_set_constants(int dim, const double* K0, cudaStream_t s) {
    int nl = dim * (1 << dim);
    cudaMemcpyToSymbolAsync(c_K0, K0, sizeof(double) * nl * nl, 0, cudaMemcpyHostToDevice, s);
}

static constexpr int COLS_PER_WARP = 30;
static constexpr int CHUNK2 = 32;
static constexpr int CHUNK3 = 16;

int fine_items(const LevelGeom& g, int R) {
    if (g.dim == 2) return march2_items(M2_MATVEC, g, nullptr, R);
    if (!getenv("MG_DENSE_H8")) return h8_items(g, R);
    int ncols = g.nn[g.dim - 1];
    int nct = (ncols + COLS_PER_WARP - 1) / COLS_PER_WARP;
    int chunk = g.dim == 2 ? CHUNK2 : CHUNK3;
    int nch = (g.nn[0] + chunk - 1) / chunk;
    int nj = g.dim == 2 ? 1 : g.nn[1];
    return nct * nch * nj;
}

template <int DIM, int OP>
__device__ __forceinline__ void load_node(const FineArgs& a, long long vbase, long long node, bool valid,
                                          double* raw, double* msk, double beta, int& mbits) {
    if (valid) {
        mbits = a.mask[node];
        const long long o = vbase + (long long)DIM * node;
        if (OP == FOP_CGP) {
#pragma unroll
            for (int k = 0; k < DIM; ++k) raw[k] = a.z[o + k] + beta * a.pin[o + k];
        } else {
            if (DIM == 2) {
                double2 v = *reinterpret_cast<const double2*>(a.x + o);
                raw[0] = v.x; raw[1] = v.y;
            } else {
#pragma unroll
                for (int k = 0; k < DIM; ++k) raw[k] = a.x[o + k];
            }
        }
    } else {
        mbits = (1 << DIM) - 1;
#pragma unroll
        for (int k = 0; k < DIM; ++k) raw[k] = 0.0;
    }
#pragma unroll
    for (int k = 0; k < DIM; ++k) msk[k] = ((mbits >> k) & 1) ? 0.0 : raw[k];
}

// Epilogue at an owned output node.  acc = (K M x) row values, raw = unmasked x.
template <int DIM, int OP>
__device__ __forceinline__ void finish_node(const FineArgs& a, long long vbase, long long node, int mbits,
                                            const double* acc, const double* raw, double& dot, double xal,
                                            bool sdot) {
    const long long o = vbase + (long long)DIM * node;
    double out[DIM];
#pragma unroll
    for (int k = 0; k < DIM; ++k) {
        const double ax = ((mbits >> k) & 1) ? raw[k] : acc[k];
        if (OP == FOP_MATVEC || OP == FOP_CGP) {
            out[k] = ax;
        } else if (OP == FOP_RESID) {
            out[k] = a.b[o + k] - ax;
        } else {  // JACOBI
            const double bk = a.b[o + k];
            out[k] = raw[k] + a.omega * a.Dinv[(long long)DIM * node + k] * (bk - ax);
            if (sdot) dot += bk * out[k];
        }
        if (OP == FOP_CGP) {
            if (sdot) dot += raw[k] * ax;
            if (a.xv) a.xv[o + k] = fma(xal, a.pin[o + k], a.xv[o + k]);   // deferred x += alpha p
        }
    }
    if (DIM == 2) {
        *reinterpret_cast<double2*>(a.y + o) = make_double2(out[0], out[1]);
    } else {
#pragma unroll
        for (int k = 0; k < DIM; ++k) a.y[o + k] = out[k];
    }
}

// ------------------------------------------------------------------ 3D (H8)
template <int OP>
__global__ void __launch_bounds__(128) fine3d_kernel(FineArgs a, int nct, int nch) {
    const int lane = threadIdx.x & 31;
    const long long w = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int n0 = a.g.nn[0], n1 = a.g.nn[1], n2 = a.g.nn[2];
    const int N0 = a.g.N[0], N1 = a.g.N[1], N2 = a.g.N[2];
    const int items = nct * nch * n1;
    if (w >= (long long)a.R * items) return;
    if (a.done && *a.done) return;
    const int r = (int)(w % a.R);
    const int item = (int)(w / a.R);
    if (a.active && !a.active[r]) return;
    const int ct = item % nct;
    const int j = (item / nct) % n1;
    const int ch = item / (nct * n1);
    const int c = ct * COLS_PER_WARP + lane - 1;
    const bool cin = (c >= 0) && (c < n2);
    const bool own = cin && lane >= 1 && lane <= COLS_PER_WARP;
    const int i0 = ch * CHUNK3, i1 = min(i0 + CHUNK3, n0);
    const long long vbase = (long long)r * a.g.ndof;
    const double beta = (OP == FOP_CGP) ? a.beta[r] : 0.0;
    const double xal = (OP == FOP_CGP && a.xv) ? a.xalpha[r] : 0.0;

    double A[3][3][3], B[3][3][3];   // [row j-1..j+1][col c-1..c+1][comp]
    double rawA[3], rawB[3];
    int mA = 7, mB = 7;
    double carry[3] = {0.0, 0.0, 0.0};
    double dot = 0.0;

    auto load_plane = [&](int P, double (&W)[3][3][3], double (&raw)[3], int& mown) {
#pragma unroll
        for (int dj = 0; dj < 3; ++dj) {
            const int jj = j + dj - 1;
            const bool v = cin && P >= 0 && P < n0 && jj >= 0 && jj < n1;
            double rw[3], m[3];
            int mb;
            load_node<3, OP>(a, vbase, ((long long)P * n1 + jj) * n2 + c, v, rw, m, beta, mb);
            if (dj == 1) { raw[0] = rw[0]; raw[1] = rw[1]; raw[2] = rw[2]; mown = mb; }
#pragma unroll
            for (int k = 0; k < 3; ++k) { W[dj][1][k] = m[k]; W[dj][0][k] = shfl_up1(m[k]); W[dj][2][k] = shfl_dn1(m[k]); }
        }
    };

    load_plane(i0 - 1, A, rawA, mA);
    for (int L = i0 - 1; L < i1; ++L) {
        const int P = L + 1;
        load_plane(P, B, rawB, mB);
        if (OP == FOP_CGP && own && P >= i0 && P < i1) {
            const long long o = vbase + 3LL * (((long long)P * n1 + j) * n2 + c);
            a.pout[o] = rawB[0]; a.pout[o + 1] = rawB[1]; a.pout[o + 2] = rawB[2];
        }
        // element moduli of layer L: [ej][ec] -> element (L, j-1+ej, c-1+ec)
        double Ee[2][2];
#pragma unroll
        for (int ej = 0; ej < 2; ++ej) {
            const int je = j - 1 + ej;
            double Ev = 0.0;
            if (L >= 0 && L < N0 && je >= 0 && je < N1 && c >= 0 && c < N2)
                Ev = a.E[((long long)L * N1 + je) * N2 + c];
            Ee[ej][1] = Ev;
            Ee[ej][0] = shfl_up1(Ev);
            if (c - 1 < 0) Ee[ej][0] = 0.0;
        }
        double lo[3] = {carry[0], carry[1], carry[2]}, hi[3] = {0.0, 0.0, 0.0};
#pragma unroll
        for (int ej = 0; ej < 2; ++ej)
#pragma unroll
            for (int ec = 0; ec < 2; ++ec) {
                const int a1 = 1 - ej, a2 = 1 - ec;
                double tl[3] = {0.0, 0.0, 0.0}, th[3] = {0.0, 0.0, 0.0};
#pragma unroll
                for (int b0 = 0; b0 < 2; ++b0)
#pragma unroll
                    for (int b1 = 0; b1 < 2; ++b1)
#pragma unroll
                        for (int b2 = 0; b2 < 2; ++b2)
#pragma unroll
                            for (int k2 = 0; k2 < 3; ++k2) {
                                const double xv = b0 ? B[ej + b1][ec + b2][k2] : A[ej + b1][ec + b2][k2];
                                const int col = ((b0 * 2 + b1) * 2 + b2) * 3 + k2;
#pragma unroll
                                for (int k = 0; k < 3; ++k) {
                                    tl[k] = fma(c_K0[(((0 * 2 + a1) * 2 + a2) * 3 + k) * 24 + col], xv, tl[k]);
                                    th[k] = fma(c_K0[(((1 * 2 + a1) * 2 + a2) * 3 + k) * 24 + col], xv, th[k]);
                                }
                            }
#pragma unroll
                for (int k = 0; k < 3; ++k) {
                    lo[k] = fma(Ee[ej][ec], tl[k], lo[k]);
                    hi[k] = fma(Ee[ej][ec], th[k], hi[k]);
                }
            }
        if (own && L >= i0)
            finish_node<3, OP>(a, vbase, ((long long)L * n1 + j) * n2 + c, mA, lo, rawA, dot, xal,
                               L >= a.so0 && L < a.so1);
        carry[0] = hi[0]; carry[1] = hi[1]; carry[2] = hi[2];
#pragma unroll
        for (int q = 0; q < 3; ++q)
#pragma unroll
            for (int s = 0; s < 3; ++s)
#pragma unroll
                for (int k = 0; k < 3; ++k) A[q][s][k] = B[q][s][k];
        rawA[0] = rawB[0]; rawA[1] = rawB[1]; rawA[2] = rawB[2]; mA = mB;
    }
    if (a.partial) {
        dot = warp_sum(dot);
        if (lane == 0) a.partial[(long long)r * a.pstride + item] = dot;
    }
}

template <int OP>
static void launch_fine(const FineArgs& a, cudaStream_t s) {
    const LevelGeom& g = a.g;
    int ncols = g.nn[g.dim - 1];
    int nct = (ncols + COLS_PER_WARP - 1) / COLS_PER_WARP;
    int chunk = g.dim == 2 ? CHUNK2 : CHUNK3;
    int nch = (g.nn[0] + chunk - 1) / chunk;
    long long warps = (long long)a.R * fine_items(g, a.R);
    int wpb = 4;
    long long blocks = (warps + wpb - 1) / wpb;
    fine3d_kernel<OP><<<(unsigned)blocks, 32 * wpb, 0, s>>>(a, nct, nch);
}

int fine_apply(int op, const FineArgs& a, cudaStream_t s) {
    if (a.g.dim == 3 && !getenv("MG_DENSE_H8")) return h8_apply(op, a, s);
    switch (op) {
        case FOP_MATVEC: launch_fine<FOP_MATVEC>(a, s); break;
        case FOP_RESID: launch_fine<FOP_RESID>(a, s); break;
        case FOP_JACOBI: launch_fine<FOP_JACOBI>(a, s); break;
        default: launch_fine<FOP_CGP>(a, s); break;
    }
    return fine_items(a.g, a.R);
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
