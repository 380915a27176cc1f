// 3D (H8) fine level: matrix-free element-by-element K = sum_e E_e A_e^T K0 A_e (PAPER.md:99
// "K_e = E_kappa(x_e) K_e0"), Dirichlet rows/cols identity (reading r11),
// fused with its consumer in the CG iteration / smoother exactly like the former dense kernel:
//   FOP_MATVEC  y = K x
//   FOP_RESID   y = b - K x
//   FOP_JACOBI  y = x + omega D^-1 (b - K x), dot(b, y)
//   FOP_CGP     p = z + beta p_in ; q = K p ; dot(p, q) ; x += xalpha p_in
//
// Why not dense: 24x24 per element is 576 DFMA per element x RHS, ~4x over the fp64 ridge
// of B200 (the fine matvec moves ~50 B per element x RHS).  Here every element is applied
// once, in the sum/difference basis of the trilinear shape functions: per axis the nodal
// pair (v0, v1) becomes (m = v0 + v1, d = v1 - v0), in which the 1-D mass and stiffness
// matrices are diagonal and the mixed one has a single entry, so the element matrix
// K^ = T^-T K0 T^-1 has 45 nonzeros instead of 576 (SURVEY 7 "Hard parts" 1; closed form
// below, pinned against K0 in tests).  The transform is separable and shared between
// neighbouring elements: edges along axis 2 by a warp shuffle, faces along axis 1 through
// shared memory, the axis-0 stage in registers while marching -- ~171 fp64 instructions per
// element x RHS instead of 576.  The transposed transform scatters the element result back
// to its 8 nodes through the same stages (no atomics, deterministic).
//
// Work decomposition: a CTA is a tile of 8 node rows (axis 1) x 32 node columns (axis 2),
// one warp per row, marching along axis 0 over a chunk of node planes.  Thread (r, lane)
// computes element (j, c) = (row, col) of each layer; owned outputs are rows 1..6 and lanes
// 1..30 of the tile (the outer ring only feeds neighbours).  RHS index is the fastest grid
// coordinate so the R CTAs of a tile run together and share E in L2.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "element.cuh"
#include "kernels.h"

__constant__ double c_Kh[576];

// ---------------------------------------------------------------- K^ in closed form
// 1-D factors in the (m, d) basis (t = 0: m, t = 1: d) of the integrals of element.cuh:
// M^ = diag(1/4, 1/12), D^ = diag(0, 1), C^[d][m] = 1/2 (derivative on the test function),
// C^T[m][d] = 1/2.  K^[(s,i),(t,j)] = lam S^_ij + mu S^_ji + mu delta_ij sum_k S^_kk.
__host__ __device__ constexpr double f1h(int kind, int ta, int tb) {
    return kind == 0 ? (ta == tb ? (ta == 0 ? 0.25 : 1.0 / 12.0) : 0.0)
         : kind == 1 ? ((ta == 1 && tb == 1) ? 1.0 : 0.0)
         : kind == 2 ? ((ta == 1 && tb == 0) ? 0.5 : 0.0)
                     : ((ta == 0 && tb == 1) ? 0.5 : 0.0);
}

__host__ __device__ constexpr double sh3(int i, int j, int s, int t) {
    double v = 1.0;
    for (int k = 0; k < 3; ++k) {
        const int ta = (s >> (2 - k)) & 1, tb = (t >> (2 - k)) & 1;
        const int kind = (k == i && k == j) ? 1 : (k == i ? 2 : (k == j ? 3 : 0));
        v *= f1h(kind, ta, tb);
    }
    return v;
}

__host__ __device__ constexpr double khat(double nu, int row, int col) {
    const int s = row / 3, i = row % 3, t = col / 3, j = col % 3;
    const double mu = 1.0 / (2.0 * (1.0 + nu));
    const double lam = nu / ((1.0 + nu) * (1.0 - 2.0 * nu));
    double v = lam * sh3(i, j, s, t) + mu * sh3(j, i, s, t);
    if (i == j)
        for (int k = 0; k < 3; ++k) v += mu * sh3(k, k, s, t);
    return v;
}

// K^ = T^-T K0 T^-1 for any element matrix K0 (standard at any nu, or the incompatible-mode
// element): per axis T^-1 = (1/2) [[1, -1], [1, 1]].  Its sparsity is that of khat (checked for
// both element types), which the kernel's compile-time skip pattern relies on.
void h8_set_constants(const double* K0, cudaStream_t s) {
    static double Ti[24][24], Kh[576];
    for (int a = 0; a < 8; ++a)       // nodal index a, transformed index t
        for (int t = 0; t < 8; ++t) {
            double v = 1.0;
            for (int k = 0; k < 3; ++k) {
                const int ab = (a >> (2 - k)) & 1, tb = (t >> (2 - k)) & 1;
                v *= 0.5 * ((tb == 0) ? 1.0 : (ab ? 1.0 : -1.0));
            }
            for (int i = 0; i < 3; ++i)
                for (int j = 0; j < 3; ++j) Ti[3 * a + i][3 * t + j] = (i == j) ? v : 0.0;
        }
    for (int r = 0; r < 24; ++r)
        for (int c = 0; c < 24; ++c) {
            double v = 0.0;
            for (int p = 0; p < 24; ++p) {
                if (Ti[p][r] == 0.0) continue;
                for (int q = 0; q < 24; ++q) v += Ti[p][r] * K0[p * 24 + q] * Ti[q][c];
            }
            Kh[r * 24 + c] = v;
        }
    cudaMemcpyToSymbolAsync(c_Kh, Kh, sizeof(Kh), 0, cudaMemcpyHostToDevice, s);
}

// the sparsity pattern is nu-independent; values are immediates for nu = 0.3
template <bool C03>
__device__ __forceinline__ double KH(int r, int c) {
    if (C03) return khat(MG_NU_PAPER, r, c);
    return c_Kh[r * 24 + c];
}

// connected components of the K^ sparsity pattern (rows = cols; the zero rows of the rigid
// translation modes s = 0 are left out): the element result is formed one component at a time
static constexpr int H8_NCOMP = 11;
__device__ constexpr int H8_COMP[H8_NCOMP][3] = {
    {3, 14, -1},
    {4, 8, -1},
    {5, 7, 12},
    {6, 13, -1},
    {9, 16, 20},
    {10, 15, -1},
    {11, 18, -1},
    {17, 19, -1},
    {21, -1, -1},
    {22, -1, -1},
    {23, -1, -1}};

static constexpr int TOWN_C = 30;   // owned columns
static constexpr int HCH = 32;      // node planes per chunk

struct H8Plane {              // per-thread data of one node plane
    double raw[3];            // unmasked operator input (identity rows / dots)
    double aux[3];            // RESID/JACOBI: b ; CGP: unused
    double dinv[3];           // JACOBI
    double xo[3];             // CGP: x (deferred update x += xalpha p_in)
    double E;                 // element (P, j, c)
    int m;                    // fixed bits
};

// TR node rows per CTA (one warp each), TR - 2 owned; MINB CTAs per SM (register cap)
template <int OP, bool C03, int TR, int MINB>
__global__ void __launch_bounds__(32 * TR, MINB) h8_kernel(FineArgs a, int ntc, int ntr, int nch, int hch) {
    pdl_begin();
    constexpr int TOWN_R = TR - 2;
    extern __shared__ double h8_smem[];
    double (*s_fwd)[6][32] = reinterpret_cast<double (*)[6][32]>(h8_smem);             // edge (m, d) x 3 comps, per row
    double (*s_inv)[6][32] = reinterpret_cast<double (*)[6][32]>(h8_smem + TR * 6 * 32); // inverse edges for row + 1
    const int lane = threadIdx.x & 31, row = threadIdx.x >> 5;
    const int nt = ntc * ntr;
    const int bid = blockIdx.x;
    const int R = a.R;
    const int r = bid % R;
    const int tile = bid / R;
    if (tile >= nt * nch) return;
    if (a.done && *a.done) return;
    if (a.active && !a.active[r]) return;
    const int tc = tile % ntc, tr = (tile / ntc) % ntr, ch = tile / nt;
    const int n0 = a.g.nn[0], n1 = a.g.nn[1], n2 = a.g.nn[2];
    const int N0 = a.g.N[0], N1 = a.g.N[1], N2 = a.g.N[2];
    const int j = tr * TOWN_R - 1 + row;
    const int c = tc * TOWN_C - 1 + lane;
    const bool node_ok = j >= 0 && j < n1 && c >= 0 && c < n2;
    const bool elem_jc = j >= 0 && j < N1 && c >= 0 && c < N2 && row < TR - 1 && lane < 31;
    const bool own = node_ok && row >= 1 && row <= TOWN_R && lane >= 1 && lane <= TOWN_C;
    const int i0 = ch * hch, i1 = min(i0 + hch, n0);
    const long long vbase = (long long)r * a.g.ndof;
    const long long col = (long long)j * n2 + c;          // node offset within a plane
    const long long ecol = (long long)j * N2 + c;         // element offset within a layer
    const long long pstride = (long long)n1 * n2, estride = (long long)N1 * N2;
    const double beta = (OP == FOP_CGP) ? a.beta[r] : 0.0;
    const double alpha = (OP == FOP_RESTR3) ? a.alpha[r] : 0.0;
    const double xal = (OP == FOP_CGP && a.xv) ? a.xalpha[r] : 0.0;

    auto load = [&](H8Plane& q, int P) {
        q.E = 0.0;
        if (elem_jc && P >= 0 && P < N0) q.E = a.E[(long long)P * estride + ecol];
        if (!(node_ok && P >= 0 && P < n0)) {
            q.m = 7;
#pragma unroll
            for (int k = 0; k < 3; ++k) q.raw[k] = q.aux[k] = q.dinv[k] = 0.0;
            return;
        }
        const long long nd = (long long)P * pstride + col;
        const long long o = vbase + 3 * nd;
        q.m = a.mask[nd];
        if (OP == FOP_RESTR3) {
            // r = rin - alpha q (kept in aux, stored by the caller loop), input omega D^-1 r
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                const double rv = fma(-alpha, a.q[o + k], a.rin[o + k]);
                q.aux[k] = rv;
                q.raw[k] = a.omega * a.Dinv[3 * nd + k] * rv;
            }
        } else if (OP == FOP_POST3) {
            // input z2 = omega D^-1 b + P ec (trilinear prolongation, coarse-masked)
            const int Ps = P + a.off0;
            const int I0 = Ps >> 1, I1 = (Ps + 1) >> 1, J0 = j >> 1, J1 = (j + 1) >> 1, C0 = c >> 1,
                      C1 = (c + 1) >> 1;
            const int cn1 = a.gc.nn[1], cn2 = a.gc.nn[2];
            const double* ev = a.ec + (long long)r * a.gc.ndof;
            double pe[3] = {0.0, 0.0, 0.0};
#pragma unroll
            for (int s8 = 0; s8 < 8; ++s8) {
                const int I = (s8 & 4) ? I1 : I0, J = (s8 & 2) ? J1 : J0, C = (s8 & 1) ? C1 : C0;
                const long long cn = ((long long)I * cn1 + J) * cn2 + C;
                const int mc = a.maskc[cn];
#pragma unroll
                for (int k = 0; k < 3; ++k) pe[k] += ((mc >> k) & 1) ? 0.0 : ev[3 * cn + k];
            }
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                const double bv = a.b[o + k];
                q.aux[k] = bv;
                q.dinv[k] = a.Dinv[3 * nd + k];
                q.raw[k] = ((q.m >> k) & 1) ? 0.0 : fma(a.omega * q.dinv[k], bv, 0.125 * pe[k]);
            }
        } else if (OP == FOP_CGP) {
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                const double pin = a.pin[o + k];
                q.raw[k] = fma(beta, pin, a.z[o + k]);
                q.aux[k] = pin;
                if (a.xv) q.xo[k] = a.xv[o + k];
            }
        } else if (OP != FOP_RESTR3 && OP != FOP_POST3) {
#pragma unroll
            for (int k = 0; k < 3; ++k) q.raw[k] = a.x[o + k];
        }
        if (OP == FOP_RESID || OP == FOP_JACOBI) {
#pragma unroll
            for (int k = 0; k < 3; ++k) q.aux[k] = a.b[o + k];
        }
        if (OP == FOP_JACOBI) {
#pragma unroll
            for (int k = 0; k < 3; ++k) q.dinv[k] = a.Dinv[3 * nd + k];
        }
    };

    // forward stages of plane P: edges along axis 2 (shuffle), faces along axis 1 (smem)
    auto forward = [&](const H8Plane& q, double (&F)[3][4]) {
        double em[3], ed[3];
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            const double u = ((q.m >> k) & 1) ? 0.0 : q.raw[k];
            const double un = __shfl_down_sync(MGK_FULL, u, 1);
            em[k] = u + un;
            ed[k] = un - u;
            s_fwd[row][k][lane] = em[k];
            s_fwd[row][3 + k][lane] = ed[k];
        }
        __syncthreads();
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            const double em1 = row < TR - 1 ? s_fwd[row + 1][k][lane] : 0.0;
            const double ed1 = row < TR - 1 ? s_fwd[row + 1][3 + k][lane] : 0.0;
            F[k][0] = em[k] + em1;   // (m_j, m_c)
            F[k][1] = ed[k] + ed1;   // (m_j, d_c)
            F[k][2] = em1 - em[k];   // (d_j, m_c)
            F[k][3] = ed1 - ed[k];   // (d_j, d_c)
        }
    };

    double FL[3][4], CY[3][4];
    H8Plane cur, nxt;
    double dot = 0.0;
    // prologue: plane i0-1 (its face; element layer i0-1 is added in the first step)
    load(cur, i0 - 1);
    forward(cur, FL);
#pragma unroll
    for (int k = 0; k < 3; ++k)
#pragma unroll
        for (int f = 0; f < 4; ++f) CY[k][f] = 0.0;
    load(nxt, i0);
    for (int L = i0 - 1; L < i1; ++L) {
        const int P = L + 1;
        H8Plane pl = nxt;                       // plane P
        H8Plane lo = cur;                       // plane L
        if (P + 1 <= i1) load(nxt, P + 1);      // prefetch
        if (OP == FOP_RESTR3 && own && P >= i0 && P < i1) {
            const long long o = vbase + 3 * ((long long)P * pstride + col);
            const bool sd = P >= a.so0 && P < a.so1;
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                a.rout[o + k] = pl.aux[k];
                if (a.z1out) a.z1out[o + k] = pl.raw[k];
                if (sd) dot = fma(pl.aux[k], pl.aux[k], dot);
            }
        }
        if (OP == FOP_CGP && own && P >= i0 && P < i1) {
            const long long o = vbase + 3 * ((long long)P * pstride + col);
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                a.pout[o + k] = pl.raw[k];
                if (a.xv) a.xv[o + k] = fma(xal, pl.aux[k], pl.xo[k]);   // deferred x += alpha p_in
            }
        }
        // (no barrier needed here: every thread passed the previous step's second barrier,
        // so all reads of s_fwd of that step are complete)
        double FP[3][4];
        forward(pl, FP);
        // element (L, j, c): u^ = E * (T u) ; y^ = K^ u^ ; back to the two faces
        double GL[3][4];
        if (row == TR - 1) {   // top halo row: feeds row TR-2's faces only (warp-uniform)
#pragma unroll
            for (int k = 0; k < 3; ++k)
#pragma unroll
                for (int f = 0; f < 4; ++f) GL[k][f] = 0.0;
        } else {
            const double Ee = lo.E;   // E of element layer L, loaded with plane L
            double uh[24], yh[24];
#pragma unroll
            for (int f = 0; f < 4; ++f)
#pragma unroll
                for (int k = 0; k < 3; ++k) {
                    uh[3 * f + k] = Ee * (FL[k][f] + FP[k][f]);          // t0 = m
                    uh[3 * (4 + f) + k] = Ee * (FP[k][f] - FL[k][f]);    // t0 = d
                }
#pragma unroll
            for (int rr = 0; rr < 24; ++rr) {
                double acc = 0.0;
#pragma unroll
                for (int cc = 0; cc < 24; ++cc)
                    if (khat(MG_NU_PAPER, rr, cc) != 0.0) acc = fma(KH<C03>(rr, cc), uh[cc], acc);
                yh[rr] = acc;
            }
#pragma unroll
            for (int f = 0; f < 4; ++f)
#pragma unroll
                for (int k = 0; k < 3; ++k) {
                    const double ym = yh[3 * f + k], yd = yh[3 * (4 + f) + k];
                    GL[k][f] = CY[k][f] + (ym - yd);   // face L total
                    CY[k][f] = ym + yd;                // carried to face P
                }
        }
        // face L -> edges of rows j (own) and j+1 (neighbour) -> nodes
        double eo[3][2];
#pragma unroll
        for (int k = 0; k < 3; ++k)
#pragma unroll
            for (int t2 = 0; t2 < 2; ++t2) {
                const double fm = GL[k][t2], fd = GL[k][2 + t2];
                eo[k][t2] = fm - fd;
                s_inv[row][2 * k + t2][lane] = fm + fd;
            }
        __syncthreads();
        double y[3];
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            const double em = eo[k][0] + (row > 0 ? s_inv[row - 1][2 * k][lane] : 0.0);
            const double ed = eo[k][1] + (row > 0 ? s_inv[row - 1][2 * k + 1][lane] : 0.0);
            const double up = __shfl_up_sync(MGK_FULL, em + ed, 1);   // node c+1 part of lane-1
            y[k] = (em - ed) + up;
        }
        if (own && L >= i0) {
            const long long nd = (long long)L * pstride + col;
            const long long o = vbase + 3 * nd;
            const bool sdot = L >= a.so0 && L < a.so1;
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                const double ax = ((lo.m >> k) & 1) ? lo.raw[k] : y[k];
                double out;
                if (OP == FOP_MATVEC || OP == FOP_CGP) out = ax;
                else if (OP == FOP_RESID || OP == FOP_RESTR3) out = lo.aux[k] - ax;
                else out = fma(a.omega * lo.dinv[k], lo.aux[k] - ax, lo.raw[k]);
                if ((OP == FOP_JACOBI || OP == FOP_POST3) && sdot) dot = fma(lo.aux[k], out, dot);
                if (OP == FOP_CGP && sdot) dot = fma(lo.raw[k], ax, dot);
                a.y[o + k] = out;
            }
        }
#pragma unroll
        for (int k = 0; k < 3; ++k)
#pragma unroll
            for (int f = 0; f < 4; ++f) FL[k][f] = FP[k][f];
        cur = pl;
    }
    if (a.partial) {
        dot = warp_sum(dot);
        __shared__ double s_dot[TR];
        if (lane == 0) s_dot[row] = dot;
        __syncthreads();
        if (threadIdx.x == 0) {
            double t = 0.0;
#pragma unroll
            for (int w = 0; w < TR; ++w) t += s_dot[w];
            a.partial[(long long)r * a.pstride + tile] = t;
        }
    }
}

// ---------------------------------------------------------------- shared-memory plane ring
// Same operator and march as h8_kernel (MATVEC / RESID / JACOBI / CGP), but the per-plane inputs
// are staged by per-thread cp.async (LDGSTS, zero-fill predicates) into a ring of NS planes in
// shared memory and consumed from there, instead of a one-plane register prefetch.  A thread
// keeps in registers only what the march carries (forward faces FL, carried element results CY)
// and the few values of plane L its output needs, so the kernel fits 128 registers: 16 warps per
// SM (2 CTAs of 8 rows, or 1 of 16) with NS planes in flight.
__device__ __forceinline__ void h8_cpa8(void* dst, const void* src, bool pred) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(d), "l"(src), "r"(pred ? 8 : 0));
}
__device__ __forceinline__ void h8_cpa4(void* dst, const void* src, bool pred) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(d), "l"(src), "r"(pred ? 4 : 0));
}
__device__ __forceinline__ void h8_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void h8_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// ring fields (8-byte words per thread and plane)
template <int OP>
struct H8R {
    // vector fields: A = x (MATVEC/RESID/JACOBI), p_in (CGP) or r_in (RESTR3); B = b (RESID/JACOBI),
    // z (CGP) or q (RESTR3); C = D^-1 (JACOBI/RESTR3) or x (CGP, deferred update)
    static constexpr bool HB = OP != FOP_MATVEC;
    static constexpr bool HC = OP == FOP_JACOBI || OP == FOP_CGP || OP == FOP_RESTR3;
    static constexpr int FA = 0, FB = 3, FC = HB ? 6 : 3;
    static constexpr int FE = FC + (HC ? 3 : 0), FM = FE + 1, NW = FM + 1;
};

// KEEP: plane L's ring slot is kept until its output is written (output terms read from shared
// memory instead of registers; one plane less in flight)
template <int OP, bool C03, int TR, int MINB, int NS, bool KEEP>
__global__ void __launch_bounds__(32 * TR, MINB) h8r_kernel(FineArgs a, int ntc, int ntr, int nch, int hch) {
    pdl_begin();
    using F = H8R<OP>;
    constexpr int TOWN_R = TR - 2, NT = 32 * TR;
    extern __shared__ double h8_smem[];
    double (*s_fwd)[6][32] = reinterpret_cast<double (*)[6][32]>(h8_smem);
    double (*s_inv)[6][32] = reinterpret_cast<double (*)[6][32]>(h8_smem + TR * 6 * 32);
    double* ring = h8_smem + 2 * TR * 6 * 32;   // [NS][NW][NT]
    const int lane = threadIdx.x & 31, row = threadIdx.x >> 5, tid = threadIdx.x;
    const int nt = ntc * ntr;
    const int bid = blockIdx.x;
    const int R = a.R;
    const int r = bid % R;
    const int tile = bid / R;
    if (tile >= nt * nch) return;
    if (a.done && *a.done) return;
    if (a.active && !a.active[r]) return;
    const int tc = tile % ntc, tr = (tile / ntc) % ntr, ch = tile / nt;
    const int n0 = a.g.nn[0], n1 = a.g.nn[1], n2 = a.g.nn[2];
    const int N0 = a.g.N[0], N1 = a.g.N[1], N2 = a.g.N[2];
    const int j = tr * TOWN_R - 1 + row;
    const int c = tc * TOWN_C - 1 + lane;
    const bool node_ok = j >= 0 && j < n1 && c >= 0 && c < n2;
    const bool elem_jc = j >= 0 && j < N1 && c >= 0 && c < N2 && row < TR - 1 && lane < 31;
    const bool own = node_ok && row >= 1 && row <= TOWN_R && lane >= 1 && lane <= TOWN_C;
    const int i0 = ch * hch, i1 = min(i0 + hch, n0);
    const long long vbase = (long long)r * a.g.ndof;
    const long long col = (long long)j * n2 + c;
    const long long ecol = (long long)j * N2 + c;
    const long long pstride = (long long)n1 * n2, estride = (long long)N1 * N2;
    const double beta = (OP == FOP_CGP) ? a.beta[r] : 0.0;
    const double xal = (OP == FOP_CGP && a.xv) ? a.xalpha[r] : 0.0;
    const double alpha = (OP == FOP_RESTR3) ? a.alpha[r] : 0.0;
    const double* vA = (OP == FOP_CGP) ? a.pin : (OP == FOP_RESTR3 ? a.rin : a.x);
    const double* vB = (OP == FOP_CGP) ? a.z : (OP == FOP_RESTR3 ? a.q : a.b);
    const double* vC = (OP == FOP_CGP) ? a.xv : a.Dinv;
    const bool hasC = F::HC && (OP != FOP_CGP || a.xv);

    double dot = 0.0;
    auto slot = [&](int Q, int f) -> double* { return ring + ((long long)(((Q - i0 + 1) % NS) * F::NW + f)) * NT + tid; };
    auto issue = [&](int Q) {
        if (Q <= i1) {
            const bool nok = node_ok && Q >= 0 && Q < n0;
            const bool eok = elem_jc && Q >= 0 && Q < N0;
            const long long nd = nok ? (long long)Q * pstride + col : 0;
            const long long o = vbase + 3 * nd;
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                h8_cpa8(slot(Q, F::FA + k), vA + o + k, nok);
                if (F::HB) h8_cpa8(slot(Q, F::FB + k), vB + o + k, nok);
                if (F::HC && hasC) h8_cpa8(slot(Q, F::FC + k), vC + (OP == FOP_CGP ? o : 3 * nd) + k, nok);
            }
            h8_cpa8(slot(Q, F::FE), a.E + (eok ? (long long)Q * estride + ecol : 0), eok);
            h8_cpa4(slot(Q, F::FM), reinterpret_cast<const uint8_t*>((uintptr_t)(a.mask + nd) & ~(uintptr_t)3), nok);
        }
        h8_commit();
    };
    // plane values a thread needs after its plane's step: operator input, output terms, E, mask
    struct Lo {
        double raw[3], aux[3], dinv[3], E;
        int m;
    };
    // read plane Q from the ring (after the wait); CGP stores p and the deferred x update here
    auto take = [&](int Q, Lo& q) {
        const int nd4 = (int)(((long long)Q * pstride + col) & 3);
        const unsigned mw = *reinterpret_cast<const unsigned*>(slot(Q, F::FM));
        q.m = (node_ok && Q >= 0 && Q < n0) ? (int)((mw >> (8 * nd4)) & 0xffu) : 7;
        q.E = *slot(Q, F::FE);
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            const double va = *slot(Q, F::FA + k);
            if (OP == FOP_CGP) {
                q.raw[k] = fma(beta, va, *slot(Q, F::FB + k));
            } else if (OP == FOP_RESTR3) {
                // r = r_in - alpha q ; operator input omega D^-1 r
                const double rv = fma(-alpha, *slot(Q, F::FB + k), va);
                if (!KEEP) q.aux[k] = rv;
                q.raw[k] = a.omega * *slot(Q, F::FC + k) * rv;
                if (own && Q >= i0 && Q < i1) {
                    a.rout[vbase + 3 * ((long long)Q * pstride + col) + k] = rv;
                    if (a.z1out) a.z1out[vbase + 3 * ((long long)Q * pstride + col) + k] = q.raw[k];
                    if (Q >= a.so0 && Q < a.so1) dot = fma(rv, rv, dot);
                }
            } else {
                q.raw[k] = va;
                if (F::HB && !KEEP) q.aux[k] = *slot(Q, F::FB + k);
                if (OP == FOP_JACOBI && !KEEP) q.dinv[k] = *slot(Q, F::FC + k);
            }
        }
        if (OP == FOP_CGP && own && Q >= i0 && Q < i1) {
            const long long o = vbase + 3 * ((long long)Q * pstride + col);
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                a.pout[o + k] = q.raw[k];
                if (a.xv) a.xv[o + k] = fma(xal, *slot(Q, F::FA + k), *slot(Q, F::FC + k));
            }
        }
    };
    auto forward = [&](const Lo& q, double (&Fo)[3][4]) {
        double em[3], ed[3];
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            const double u = ((q.m >> k) & 1) ? 0.0 : q.raw[k];
            const double un = __shfl_down_sync(MGK_FULL, u, 1);
            em[k] = u + un;
            ed[k] = un - u;
            s_fwd[row][k][lane] = em[k];
            s_fwd[row][3 + k][lane] = ed[k];
        }
        __syncthreads();
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            const double em1 = row < TR - 1 ? s_fwd[row + 1][k][lane] : 0.0;
            const double ed1 = row < TR - 1 ? s_fwd[row + 1][3 + k][lane] : 0.0;
            Fo[k][0] = em[k] + em1;
            Fo[k][1] = ed[k] + ed1;
            Fo[k][2] = em1 - em[k];
            Fo[k][3] = ed1 - ed[k];
        }
    };

    double FL[3][4], CY[3][4];
    Lo lo;
#pragma unroll
    for (int q = 0; q < NS; ++q) issue(i0 - 1 + q);
    h8_wait<NS - 1>();
    take(i0 - 1, lo);
    if (!KEEP) issue(i0 - 1 + NS);
    forward(lo, FL);
#pragma unroll
    for (int k = 0; k < 3; ++k)
#pragma unroll
        for (int f = 0; f < 4; ++f) CY[k][f] = 0.0;
    for (int L = i0 - 1; L < i1; ++L) {
        const int P = L + 1;
        if (KEEP) h8_wait<NS - 2>();
        else h8_wait<NS - 1>();
        Lo pl;
        take(P, pl);
        if (!KEEP) issue(P + NS);   // the slot just read (own slots only: no barrier)
        double FP[3][4];
        forward(pl, FP);
        double GL[3][4];
        if (row == TR - 1) {
#pragma unroll
            for (int k = 0; k < 3; ++k)
#pragma unroll
                for (int f = 0; f < 4; ++f) GL[k][f] = 0.0;
        } else {
            const double Ee = lo.E;
            // GL = CY + (y_m - y_d), CY = y_m + y_d, accumulated component by component
#pragma unroll
            for (int k = 0; k < 3; ++k)
#pragma unroll
                for (int f = 0; f < 4; ++f) {
                    GL[k][f] = CY[k][f];
                    CY[k][f] = 0.0;
                }
#pragma unroll
            for (int ci = 0; ci < H8_NCOMP; ++ci) {
                double u[3];
#pragma unroll
                for (int q = 0; q < 3; ++q) {
                    const int cc = H8_COMP[ci][q];
                    if (cc < 0) continue;
                    const int sc = cc / 3, kc = cc % 3, fc = sc & 3;
                    u[q] = Ee * (sc < 4 ? FL[kc][fc] + FP[kc][fc] : FP[kc][fc] - FL[kc][fc]);
                }
#pragma unroll
                for (int q = 0; q < 3; ++q) {
                    const int rr = H8_COMP[ci][q];
                    if (rr < 0) continue;
                    double acc = 0.0;
#pragma unroll
                    for (int q2 = 0; q2 < 3; ++q2) {
                        const int cc = H8_COMP[ci][q2];
                        if (cc >= 0 && khat(MG_NU_PAPER, rr, cc) != 0.0) acc = fma(KH<C03>(rr, cc), u[q2], acc);
                    }
                    const int sr = rr / 3, kr = rr % 3, fr = sr & 3;
                    GL[kr][fr] += sr < 4 ? acc : -acc;
                    CY[kr][fr] += acc;
                }
            }
        }
        double eo[3][2];
#pragma unroll
        for (int k = 0; k < 3; ++k)
#pragma unroll
            for (int t2 = 0; t2 < 2; ++t2) {
                const double fm = GL[k][t2], fd = GL[k][2 + t2];
                eo[k][t2] = fm - fd;
                s_inv[row][2 * k + t2][lane] = fm + fd;
            }
        __syncthreads();
        double y[3];
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            const double em = eo[k][0] + (row > 0 ? s_inv[row - 1][2 * k][lane] : 0.0);
            const double ed = eo[k][1] + (row > 0 ? s_inv[row - 1][2 * k + 1][lane] : 0.0);
            const double up = __shfl_up_sync(MGK_FULL, em + ed, 1);
            y[k] = (em - ed) + up;
        }
        if (own && L >= i0) {
            const long long o = vbase + 3 * ((long long)L * pstride + col);
            const bool sdot = L >= a.so0 && L < a.so1;
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                const double ax = ((lo.m >> k) & 1) ? lo.raw[k] : y[k];
                const double bk = (KEEP && OP == FOP_RESTR3) ? fma(-alpha, *slot(L, F::FB + k), *slot(L, F::FA + k))
                                : (KEEP && F::HB)              ? *slot(L, F::FB + k)
                                                               : lo.aux[k];
                const double dk = (KEEP && OP == FOP_JACOBI) ? *slot(L, F::FC + k) : lo.dinv[k];
                double out;
                if (OP == FOP_MATVEC || OP == FOP_CGP) out = ax;
                else if (OP == FOP_RESID || OP == FOP_RESTR3) out = bk - ax;
                else out = fma(a.omega * dk, bk - ax, lo.raw[k]);
                if (OP == FOP_JACOBI && sdot) dot = fma(bk, out, dot);
                if (OP == FOP_CGP && sdot) dot = fma(lo.raw[k], ax, dot);
                a.y[o + k] = out;
            }
        }
#pragma unroll
        for (int k = 0; k < 3; ++k)
#pragma unroll
            for (int f = 0; f < 4; ++f) FL[k][f] = FP[k][f];
        lo = pl;
        if (KEEP) issue(L + NS);   // plane L's slot is free now
    }
    h8_wait<0>();
    if (a.partial) {
        dot = warp_sum(dot);
        __shared__ double s_dot[TR];
        if (lane == 0) s_dot[row] = dot;
        __syncthreads();
        if (threadIdx.x == 0) {
            double t = 0.0;
#pragma unroll
            for (int w = 0; w < TR; ++w) t += s_dot[w];
            a.partial[(long long)r * a.pstride + tile] = t;
        }
    }
}

// variant: 0 = 8 rows x 1 CTA/SM, 1 = 16 rows x 1 CTA/SM (128-register cap), 2 = 8 rows x
// 2 CTAs/SM (128-register cap), 3 = plane ring, 8 rows x 2 CTAs/SM, 4 = plane ring, 16 rows x
// 1 CTA/SM (MATVEC / RESID / JACOBI / CGP only); MG_H8_VARIANT overrides the per-op default.
static int h8_variant(int op) {
    static int v = [] {
        const char* e = getenv("MG_H8_VARIANT");
        return e ? atoi(e) : -1;
    }();
    // MG_H8_VARIANTS="v_matvec,v_resid,v_jacobi,v_cgp,v_restr3"
    static int vo[5] = {-1, -1, -1, -1, -1};
    static bool vo_init = [] {
        const char* e = getenv("MG_H8_VARIANTS");
        if (e) sscanf(e, "%d,%d,%d,%d,%d", &vo[0], &vo[1], &vo[2], &vo[3], &vo[4]);
        return true;
    }();
    (void)vo_init;
    if (op <= FOP_RESTR3 && vo[op] == 9) return op == FOP_CGP ? 1 : 0;
    if (op <= FOP_RESTR3 && vo[op] >= 0) return (vo[op] >= 3 && op > FOP_RESTR3) ? 0 : vo[op];
    if (v == 9) return op == FOP_CGP ? 1 : 0;   // register-prefetch kernel, former per-op default
    if (v >= 0) return (v >= 3 && op > FOP_RESTR3) ? 0 : v;
    // B200 A/B (C4/C5): ring kernel for MATVEC (3), RESID / CGP / RESTR3 (5, KEEP); JACOBI and
    // POST3 stay on the register-prefetch kernel
    switch (op) {
        case FOP_MATVEC: return 3;
        case FOP_RESID: return 5;
        case FOP_CGP: return 5;
        case FOP_RESTR3: return 5;
        default: return 0;
    }
}
static int h8_rows(int op) { return (h8_variant(op) == 1 || h8_variant(op) == 4) ? 16 : 8; }
static int h8_slots(int op) {
    const int v = h8_variant(op);
    return 148 * ((v == 2 || v == 3 || v == 5) ? 2 : 1);
}

// Chunking along axis 0: between HCH/2 and 2 HCH planes per chunk, picked so that the CTA
// count fills the resident slots (148 SMs x CTAs per SM) with the smallest tail wave.
static void h8_chunks(int op, const LevelGeom& g, int R, int* nch_out, int* hch_out) {
    const int town_r = h8_rows(op) - 2;
    const int ntc = (g.nn[2] + TOWN_C - 1) / TOWN_C;
    const int ntr = (g.nn[1] + town_r - 1) / town_r;
    const long long slots = h8_slots(op);
    const int n0 = g.nn[0];
    int best = (n0 + HCH - 1) / HCH;
    double best_eff = -1.0;
    for (int nch = std::max(1, n0 / (2 * HCH)); nch <= std::max(1, 2 * n0 / HCH); ++nch) {
        const int hch = (n0 + nch - 1) / nch;
        const int nc = (n0 + hch - 1) / hch;
        const long long ctas = (long long)ntc * ntr * nc * R;
        const double waves = (double)ctas / slots;
        const double fill = waves / std::ceil(waves);
        const double eff = fill * hch / (hch + 1.0);   // + one prologue plane per chunk
        if (eff > best_eff + 1e-9) { best_eff = eff; best = nc; }
    }
    *nch_out = best;
    *hch_out = (n0 + best - 1) / best;
}

static int h8_items_op(int op, const LevelGeom& g, int R) {
    const int town_r = h8_rows(op) - 2;
    const int ntc = (g.nn[2] + TOWN_C - 1) / TOWN_C;
    const int ntr = (g.nn[1] + town_r - 1) / town_r;
    int nch, hch;
    h8_chunks(op, g, R, &nch, &hch);
    return ntc * ntr * nch;
}

// partial items: the largest over the ops (buffers are sized with this)
int h8_items(const LevelGeom& g, int R) {
    int m = 0;
    for (int op = 0; op <= FOP_POST3; ++op) m = std::max(m, h8_items_op(op, g, R));
    return m;
}

template <int OP, int TR, int MINB>
static void launch_h8_v(const FineArgs& a, int ntc, int ntr, int nch, int hch, unsigned nb, cudaStream_t s) {
    const size_t smem = sizeof(double) * 2 * TR * 6 * 32;
    static bool attr = [&] {
        cudaFuncSetAttribute(h8_kernel<OP, true, TR, MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaFuncSetAttribute(h8_kernel<OP, false, TR, MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        return true;
    }();
    (void)attr;
    if (a.nu_paper) launch_kp(false, h8_kernel<OP, true, TR, MINB>, dim3(nb), dim3(32 * TR), smem, s, a, ntc, ntr, nch, hch);
    else launch_kp(false, h8_kernel<OP, false, TR, MINB>, dim3(nb), dim3(32 * TR), smem, s, a, ntc, ntr, nch, hch);
}

static constexpr int H8_NS = 3;

template <int OP, int TR, int MINB, bool KEEP>
static void launch_h8r(const FineArgs& a, int ntc, int ntr, int nch, int hch, unsigned nb, cudaStream_t s) {
    if constexpr (OP <= FOP_RESTR3) {
        const size_t smem = sizeof(double) * (2 * TR * 6 * 32 + (size_t)H8_NS * H8R<OP>::NW * 32 * TR);
        static bool attr = [&] {
            cudaFuncSetAttribute(h8r_kernel<OP, true, TR, MINB, H8_NS, KEEP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem);
            cudaFuncSetAttribute(h8r_kernel<OP, false, TR, MINB, H8_NS, KEEP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem);
            return true;
        }();
        (void)attr;
        if (a.nu_paper) launch_kp(false, h8r_kernel<OP, true, TR, MINB, H8_NS, KEEP>, dim3(nb), dim3(32 * TR), smem, s, a, ntc, ntr, nch, hch);
        else launch_kp(false, h8r_kernel<OP, false, TR, MINB, H8_NS, KEEP>, dim3(nb), dim3(32 * TR), smem, s, a, ntc, ntr, nch, hch);
    }
}

template <int OP>
static void launch_h8(const FineArgs& a, cudaStream_t s) {
    const LevelGeom& g = a.g;
    const int town_r = h8_rows(OP) - 2;
    const int ntc = (g.nn[2] + TOWN_C - 1) / TOWN_C;
    const int ntr = (g.nn[1] + town_r - 1) / town_r;
    int nch, hch;
    h8_chunks(OP, g, a.R, &nch, &hch);
    const unsigned nb = (unsigned)((long long)ntc * ntr * nch * a.R);
    switch (h8_variant(OP)) {
        case 1: launch_h8_v<OP, 16, 1>(a, ntc, ntr, nch, hch, nb, s); break;
        case 2: launch_h8_v<OP, 8, 2>(a, ntc, ntr, nch, hch, nb, s); break;
        case 3: launch_h8r<OP, 8, 2, false>(a, ntc, ntr, nch, hch, nb, s); break;
        case 4: launch_h8r<OP, 16, 1, false>(a, ntc, ntr, nch, hch, nb, s); break;
        case 5: launch_h8r<OP, 8, 2, true>(a, ntc, ntr, nch, hch, nb, s); break;
        default: launch_h8_v<OP, 8, 1>(a, ntc, ntr, nch, hch, nb, s); break;
    }
}

int h8_apply(int op, const FineArgs& a, cudaStream_t s) {
    switch (op) {
        case FOP_MATVEC: launch_h8<FOP_MATVEC>(a, s); break;
        case FOP_RESID: launch_h8<FOP_RESID>(a, s); break;
        case FOP_JACOBI: launch_h8<FOP_JACOBI>(a, s); break;
        case FOP_RESTR3: launch_h8<FOP_RESTR3>(a, s); break;
        case FOP_POST3: launch_h8<FOP_POST3>(a, s); break;
        default: launch_h8<FOP_CGP>(a, s); break;
    }
    return h8_items_op(op, a.g, a.R);
}
