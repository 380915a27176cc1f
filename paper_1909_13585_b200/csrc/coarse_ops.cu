// Coarse levels: Galerkin operators K^{l+1} = P^T K^l P (Alg. 2 l.5
// :705), stored as assembled 3^d-point block stencils, and the
// stencil-based smoothing / residual kernels of the V-cycle.
//
// Galerkin is computed exactly by coarse-element agglomeration:
//   K_E = M_E ( sum_{children c of E} Q_c^T (M_c K_c M_c) Q_c ) M_E
// where Q_c interpolates the coarse element's nodal DOFs to child c's nodal DOFs
// (tensor product of the 1-D weights {1, 1/2, 0}) and M are the 0/1 free-DOF masks
// (reading r11: P is masked on both sides).  The level's operator is then
//   A = sum_E A_E^T K_E A_E + (I - M)
// assembled into a per-node stencil of 3^d blocks (d x d); a coarse DOF whose
// Galerkin diagonal is exactly 0 (P column zero on the free fine DOFs) is marked
// fixed, which leaves the preconditioner unchanged.
#include <cstdlib>

#include "kernels.h"

__constant__ double c_K0g[576];
__constant__ double c_Q[8 * 8 * 8];   // [child][fine local node a][coarse local node b]
__constant__ double c_Hg[3 * 3 * 8 * 8];   // H_ij[a][b] = int dN_a/dx_i dN_b/dx_j (G element matrices)

void galerkin_set_constants(int dim, const double* K0, cudaStream_t s) {
    int nl = dim * (1 << dim);
    cudaMemcpyToSymbolAsync(c_K0g, K0, sizeof(double) * nl * nl, 0, cudaMemcpyHostToDevice, s);
    // Q[c][a][b] = prod_k w(c_k + a_k, b_k), w(pos, b) = 1 if pos == 2b, 1/2 if pos == 1, else 0
    static double Q[512];
    int na = 1 << dim;
    for (int c = 0; c < na; ++c)
        for (int a = 0; a < na; ++a)
            for (int b = 0; b < na; ++b) {
                double v = 1.0;
                for (int k = 0; k < dim; ++k) {
                    int sh = dim - 1 - k;
                    int pos = ((c >> sh) & 1) + ((a >> sh) & 1);
                    int bb = (b >> sh) & 1;
                    double w = (pos == 1) ? 0.5 : (pos == 2 * bb ? 1.0 : 0.0);
                    v *= w;
                }
                Q[(c * na + a) * na + b] = v;
            }
    cudaMemcpyToSymbolAsync(c_Q, Q, sizeof(double) * na * na * na, 0, cudaMemcpyHostToDevice, s);
    static double H[3 * 3 * 8 * 8];
    const double M1[2][2] = {{1.0 / 3, 1.0 / 6}, {1.0 / 6, 1.0 / 3}};
    const double D1[2][2] = {{1.0, -1.0}, {-1.0, 1.0}};
    const double C1[2][2] = {{-0.5, -0.5}, {0.5, 0.5}};
    for (int i = 0; i < dim; ++i)
        for (int j = 0; j < dim; ++j)
            for (int a = 0; a < na; ++a)
                for (int b = 0; b < na; ++b) {
                    double v = 1.0;
                    for (int k = 0; k < dim; ++k) {
                        const int ak = (a >> (dim - 1 - k)) & 1, bk = (b >> (dim - 1 - k)) & 1;
                        if (k == i && k == j) v *= D1[ak][bk];
                        else if (k == i) v *= C1[ak][bk];
                        else if (k == j) v *= C1[bk][ak];
                        else v *= M1[ak][bk];
                    }
                    H[((i * 3 + j) * 8 + a) * 8 + b] = v;
                }
    cudaMemcpyToSymbolAsync(c_Hg, H, sizeof(H), 0, cudaMemcpyHostToDevice, s);
}

__device__ __forceinline__ void node_coords(const LevelGeom& g, long long node, int* idx) {
    long long t = node;
    for (int k = g.dim - 1; k >= 0; --k) { idx[k] = (int)(t % g.nn[k]); t /= g.nn[k]; }
}

// ---------------------------------------------------------------- element matrices
// Level-0 element matrices E_e M K0 M (only needed when levels == 1).
template <int DIM>
__global__ void elements_from_E_kernel(LevelGeom g, const double* __restrict__ E, const uint8_t* __restrict__ mask,
                                       double* elm) {
    constexpr int NA = 1 << DIM, NL = DIM * NA;
    long long e = blockIdx.x;
    int t = threadIdx.x;  // NL*NL threads
    int row = t / NL, col = t % NL;
    int ei[3] = {0, 0, 0};
    long long tt = e;
    for (int k = DIM - 1; k >= 0; --k) { ei[k] = (int)(tt % g.N[k]); tt /= g.N[k]; }
    auto local_free = [&](int ld) {
        int a = ld / DIM, comp = ld % DIM;
        long long node = 0;
        for (int k = 0; k < DIM; ++k) node = node * g.nn[k] + ei[k] + ((a >> (DIM - 1 - k)) & 1);
        return ((mask[node] >> comp) & 1) ? 0.0 : 1.0;
    };
    elm[e * NL * NL + t] = E[e] * c_K0g[row * NL + col] * local_free(row) * local_free(col);
}

void elements_from_E(const LevelGeom& g, const double* E, const uint8_t* mask, double* elm, cudaStream_t s) {
    if (g.dim == 2)
        elements_from_E_kernel<2><<<(unsigned)g.nelem, 64, 0, s>>>(g, E, mask, elm);
    else
        elements_from_E_kernel<3><<<(unsigned)g.nelem, 576, 0, s>>>(g, E, mask, elm);
}

// One CTA per coarse element; thread (row, col) owns one entry of K_E.
// Level 1 from E: when none of the 3^d fine nodes of the coarse element is fixed, every
// child matrix is E_c K0 and K_E = sum_c E_c M_c with the constant M_c = Q_c^T K0 Q_c
// (c_M, set once per handle) -- one FMA per child instead of two small matrix products.
// SRC: 0 = child element matrices elm_f (levels >= 2), 1 = E_e K0 (K, level 1), 2 = the stress
// stiffness Es_e (sigma_e : H) kron I_d from per-element Voigt stresses in E (G, level 1; NEXT-2)
// NT threads per coarse element, EPT = NL^2 / NT matrix entries per thread (3D: 192 threads x 3
// entries, so ~8 elements are in flight per SM instead of 3 -- the per-element mask check and
// child loads are latency, not bandwidth).
template <int DIM, int SRC, int NT>
__global__ void __launch_bounds__(NT) galerkin_kernel(LevelGeom gc, LevelGeom gf, const double* __restrict__ E,
                                                      const double* __restrict__ elm_f,
                                                      const uint8_t* __restrict__ mask_f,
                                                      const uint8_t* __restrict__ mask_c, double* __restrict__ elm_c,
                                                      int off0, const double* __restrict__ Mc,
                                                      const int* __restrict__ list) {
    constexpr int NA = 1 << DIM, NL = DIM * NA;
    constexpr int EPT = NL * NL / NT;
    static_assert(EPT * NT == NL * NL, "NT divides NL^2");
    __shared__ double Kc[NL * NL];
    __shared__ double T[NL * NL];
    __shared__ double fr[NL];
    __shared__ double frc[NL];   // coarse free-DOF factors of the current element
    // the prolongation stencils in shared memory: the lanes of a warp index different columns b2, which
    // the constant cache would serve one address at a time
    __shared__ double Qs[NA * NA * NA];
    const int t0 = threadIdx.x;
    for (int e = t0; e < NA * NA * NA; e += NT) Qs[e] = c_Q[e];
    __syncthreads();
    // grid-stride over coarse elements (list: count, then the element indices)
    const long long ne = list ? (long long)list[0] : gc.nelem;
    for (long long ie = blockIdx.x; ie < ne; ie += gridDim.x) {
    const long long Ec = list ? (long long)list[1 + ie] : ie;
    int ci[3] = {0, 0, 0};
    long long tt = Ec;
    for (int k = DIM - 1; k >= 0; --k) { ci[k] = (int)(tt % gc.N[k]); tt /= gc.N[k]; }
    // slab ghost element layer (children not local): filled by the halo exchange instead
    if (ci[0] < off0) continue;
    double acc[EPT];
#pragma unroll
    for (int u = 0; u < EPT; ++u) acc[u] = 0.0;
    if (t0 < NL) {   // read after the barriers below
        const int a = t0 / DIM, comp = t0 % DIM;
        long long node = 0;
        for (int k = 0; k < DIM; ++k) node = node * gc.nn[k] + ci[k] + ((a >> (DIM - 1 - k)) & 1);
        frc[t0] = ((mask_c[node] >> comp) & 1) ? 0.0 : 1.0;
    }
    bool fast = false;
    constexpr bool FROM_E = SRC == 1;
    if (FROM_E && Mc) {
        constexpr int NF = DIM == 2 ? 9 : 27;   // fine nodes of the coarse element
        static_assert(NF <= NT, "one fine node per thread");
        int fixed_here = 0;
        if (t0 < NF) {
            int q = t0, node = 0;
            int fc[3];
            for (int k = DIM - 1; k >= 0; --k) { fc[k] = 2 * ci[k] + q % 3 - (k == 0 ? off0 : 0); q /= 3; }
            bool inside = true;
            for (int k = 0; k < DIM; ++k) inside = inside && fc[k] >= 0 && fc[k] < gf.nn[k];
            if (inside) {
                for (int k = 0; k < DIM; ++k) node = node * gf.nn[k] + fc[k];
                fixed_here = mask_f[node] != 0;
            } else {
                fixed_here = 1;
            }
        }
        fast = !__syncthreads_or(fixed_here);
    }
    if (fast) {
        double ev[NA];
#pragma unroll
        for (int ch = 0; ch < NA; ++ch) {
            long long fe = 0;
            for (int k = 0; k < DIM; ++k)
                fe = fe * gf.N[k] + 2 * ci[k] + ((ch >> (DIM - 1 - k)) & 1) - (k == 0 ? off0 : 0);
            ev[ch] = E[fe];
        }
#pragma unroll
        for (int ch = 0; ch < NA; ++ch)
#pragma unroll
            for (int u = 0; u < EPT; ++u) acc[u] = fma(ev[ch], Mc[ch * NL * NL + t0 + u * NT], acc[u]);
    } else
    for (int ch = 0; ch < NA; ++ch) {
        int fi[3];
        for (int k = 0; k < DIM; ++k) fi[k] = 2 * ci[k] + ((ch >> (DIM - 1 - k)) & 1) - (k == 0 ? off0 : 0);
        long long fe = fi[0];
        for (int k = 1; k < DIM; ++k) fe = fe * gf.N[k] + fi[k];
        if (SRC == 1 || SRC == 2) {
            if (t0 < NL) {
                int a = t0 / DIM, comp = t0 % DIM;
                long long node = 0;
                for (int k = 0; k < DIM; ++k) node = node * gf.nn[k] + fi[k] + ((a >> (DIM - 1 - k)) & 1);
                fr[t0] = ((mask_f[node] >> comp) & 1) ? 0.0 : 1.0;
            }
            __syncthreads();
#pragma unroll
            for (int u = 0; u < EPT; ++u) {
                const int t = t0 + u * NT, row = t / NL, col = t % NL;
                if (SRC == 1) {
                    Kc[t] = E[fe] * c_K0g[t] * fr[row] * fr[col];
                } else {
                    constexpr int NV = DIM == 2 ? 3 : 6;
                    const int a = row / DIM, b = col / DIM;
                    double v = 0.0;
                    if (row % DIM == col % DIM) {
                        const double* sg = E + fe * NV;
                        for (int i = 0; i < DIM; ++i) v += sg[i] * c_Hg[((i * 3 + i) * 8 + a) * 8 + b];
                        for (int q = 0; q < NV - DIM; ++q) {
                            const int i = DIM == 2 ? 0 : (q == 0 ? 1 : 0), j = DIM == 2 ? 1 : (q == 2 ? 1 : 2);
                            v += sg[DIM + q] * (c_Hg[((i * 3 + j) * 8 + a) * 8 + b] + c_Hg[((j * 3 + i) * 8 + a) * 8 + b]);
                        }
                    }
                    Kc[t] = v * fr[row] * fr[col];
                }
            }
        } else {
#pragma unroll
            for (int u = 0; u < EPT; ++u) Kc[t0 + u * NT] = elm_f[fe * NL * NL + t0 + u * NT];   // masked at l-1
        }
        __syncthreads();
        // T[(a,k),(b2,k2)] = sum_a2 Kc[(a,k),(a2,k2)] Q[a2][b2]
#pragma unroll
        for (int u = 0; u < EPT; ++u) {
            const int t = t0 + u * NT, row = t / NL, col = t % NL;
            const int b2 = col / DIM, k2 = col % DIM;
            double sacc = 0.0;
#pragma unroll
            for (int a2 = 0; a2 < NA; ++a2) sacc = fma(Kc[row * NL + a2 * DIM + k2], Qs[(ch * NA + a2) * NA + b2], sacc);
            T[t] = sacc;
        }
        __syncthreads();
#pragma unroll
        for (int u = 0; u < EPT; ++u) {
            const int t = t0 + u * NT, row = t / NL, col = t % NL;
            const int b = row / DIM, k = row % DIM;
#pragma unroll
            for (int a = 0; a < NA; ++a) acc[u] = fma(Qs[(ch * NA + a) * NA + b], T[(a * DIM + k) * NL + col], acc[u]);
        }
        __syncthreads();
    }
    // coarse masks
    if (!FROM_E || !Mc || !fast) __syncthreads();   // fast path: frc visible through __syncthreads_or
#pragma unroll
    for (int u = 0; u < EPT; ++u) {
        const int t = t0 + u * NT, row = t / NL, col = t % NL;
        elm_c[Ec * NL * NL + t] = acc[u] * frc[row] * frc[col];
    }
    __syncthreads();   // shared Kc / T / fr are rewritten for the next element
    }
}

// 3D level 1 from E: a warp per coarse element.  Elements whose 27 fine nodes are all free have
// K_E = sum_c E_c M_c (M_c = Q_c' K0 Q_c, staged in shared memory), formed entry by entry in the
// children order of galerkin_kernel's fast path (bitwise the same matrices) and scaled by the coarse
// free-DOF factors; the others are appended to `list` (list[0] = count) for galerkin_kernel.  No
// CTA barrier per element: 8 warps per CTA keep 8 elements in flight each.
static constexpr int GALW_WARPS = 8, GALW_EPW = 4;
__global__ void __launch_bounds__(32 * GALW_WARPS) galerkin_warp3_kernel(LevelGeom gc, LevelGeom gf,
                                                                         const double* __restrict__ E,
                                                                         const uint8_t* __restrict__ mask_f,
                                                                         const uint8_t* __restrict__ mask_c,
                                                                         double* __restrict__ elm_c, int off0,
                                                                         const double* __restrict__ Mc, int* list) {
    constexpr int NL = 24, NE = NL * NL;
    extern __shared__ double Ms[];   // [8][576]
    for (int e = threadIdx.x; e < 8 * NE; e += blockDim.x) Ms[e] = Mc[e];
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    // GALW_EPW consecutive elements per warp iteration: every M_c entry read from shared memory
    // serves all of them (the kernel is bound by those reads otherwise)
    const long long stride = (long long)gridDim.x * GALW_WARPS * GALW_EPW;
    for (long long E0 = ((long long)blockIdx.x * GALW_WARPS + warp) * GALW_EPW; E0 < gc.nelem; E0 += stride) {
        bool fast[GALW_EPW];
        double fr[GALW_EPW], evc[GALW_EPW][8];
#pragma unroll
        for (int q = 0; q < GALW_EPW; ++q) {
            const long long Ec = E0 + q;
            fast[q] = false;
            fr[q] = 0.0;
#pragma unroll
            for (int ch = 0; ch < 8; ++ch) evc[q][ch] = 0.0;
            if (Ec >= gc.nelem) continue;   // warp-uniform
            int ci[3];
            long long tt = Ec;
            for (int k = 2; k >= 0; --k) { ci[k] = (int)(tt % gc.N[k]); tt /= gc.N[k]; }
            if (ci[0] < off0) continue;   // slab ghost element layer: filled by the halo exchange
            int fixed_here = 0;
            if (lane < 27) {
                int qq = lane, fc[3];
                for (int k = 2; k >= 0; --k) { fc[k] = 2 * ci[k] + qq % 3 - (k == 0 ? off0 : 0); qq /= 3; }
                const bool inside = fc[0] >= 0 && fc[0] < gf.nn[0] && fc[1] < gf.nn[1] && fc[2] < gf.nn[2];
                fixed_here = inside ? mask_f[((long long)fc[0] * gf.nn[1] + fc[1]) * gf.nn[2] + fc[2]] != 0 : 1;
            }
            if (__any_sync(0xffffffffu, fixed_here)) {
                if (lane == 0) list[1 + atomicAdd(list, 1)] = (int)Ec;
                continue;
            }
            fast[q] = true;
            if (lane < NL) {   // coarse free-DOF factor of local DOF lane
                const int a = lane / 3, comp = lane % 3;
                const long long node = ((long long)(ci[0] + (a >> 2)) * gc.nn[1] + ci[1] + ((a >> 1) & 1)) * gc.nn[2] + ci[2] + (a & 1);
                fr[q] = ((mask_c[node] >> comp) & 1) ? 0.0 : 1.0;
            }
            double ev = 0.0;
            if (lane < 8) {    // child lane's modulus
                const long long fe = ((long long)(2 * ci[0] + (lane >> 2) - off0) * gf.N[1] + 2 * ci[1] + ((lane >> 1) & 1)) * gf.N[2] +
                                     2 * ci[2] + (lane & 1);
                ev = E[fe];
            }
#pragma unroll
            for (int ch = 0; ch < 8; ++ch) evc[q][ch] = __shfl_sync(0xffffffffu, ev, ch);
        }
#pragma unroll 2
        for (int u = 0; u < NE / 32; ++u) {
            const int t = lane + 32 * u, row = t / NL, col = t % NL;
            double acc[GALW_EPW];
#pragma unroll
            for (int q = 0; q < GALW_EPW; ++q) acc[q] = 0.0;
#pragma unroll
            for (int ch = 0; ch < 8; ++ch) {
                const double mv = Ms[ch * NE + t];
#pragma unroll
                for (int q = 0; q < GALW_EPW; ++q) acc[q] = fma(evc[q][ch], mv, acc[q]);
            }
#pragma unroll
            for (int q = 0; q < GALW_EPW; ++q) {
                const double frow = __shfl_sync(0xffffffffu, fr[q], row), fcol = __shfl_sync(0xffffffffu, fr[q], col);
                if (fast[q]) elm_c[(E0 + q) * NE + t] = acc[q] * frow * fcol;
            }
        }
    }
}

#ifndef MG_GAL3_NT
#define MG_GAL3_NT 192   // B200 A/B (C4/C5 setup): 192 < 64 < 576 (ms)
#endif
static constexpr int GAL3_NT = MG_GAL3_NT;   // threads per coarse element (3D)

static unsigned galerkin_grid(const LevelGeom& gc) {
    const long long cap = 148LL * 32;
    return (unsigned)(gc.nelem < cap ? gc.nelem : cap);
}

void galerkin_elements(const LevelGeom& gc, const LevelGeom& gf, const double* E, const double* elm_f,
                       const uint8_t* mask_f, const uint8_t* mask_c, double* elm_c, cudaStream_t s, int off0,
                       const double* Mc, int* slow_ws) {
    unsigned bl = galerkin_grid(gc);
    if (gc.dim == 3 && E && Mc && slow_ws) {
        const size_t sm = sizeof(double) * 8 * 576;
        static bool at = (cudaFuncSetAttribute(galerkin_warp3_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm), true);
        (void)at;
        cudaMemsetAsync(slow_ws, 0, sizeof(int), s);
        const long long nb = (gc.nelem + GALW_WARPS * GALW_EPW - 1) / (GALW_WARPS * GALW_EPW);
        const unsigned gw = (unsigned)(nb < 148LL * 48 ? nb : 148LL * 48);
        galerkin_warp3_kernel<<<gw, 32 * GALW_WARPS, sm, s>>>(gc, gf, E, mask_f, mask_c, elm_c, off0, Mc, slow_ws);
        galerkin_kernel<3, 1, GAL3_NT><<<bl, GAL3_NT, 0, s>>>(gc, gf, E, elm_f, mask_f, mask_c, elm_c, off0, Mc, slow_ws);
        return;
    }
    if (gc.dim == 2) {
        if (E) galerkin_kernel<2, 1, 64><<<bl, 64, 0, s>>>(gc, gf, E, elm_f, mask_f, mask_c, elm_c, off0, Mc, nullptr);
        else galerkin_kernel<2, 0, 64><<<bl, 64, 0, s>>>(gc, gf, E, elm_f, mask_f, mask_c, elm_c, off0, nullptr, nullptr);
    } else {
        if (E) galerkin_kernel<3, 1, GAL3_NT><<<bl, GAL3_NT, 0, s>>>(gc, gf, E, elm_f, mask_f, mask_c, elm_c, off0, Mc, nullptr);
        else galerkin_kernel<3, 0, GAL3_NT><<<bl, GAL3_NT, 0, s>>>(gc, gf, E, elm_f, mask_f, mask_c, elm_c, off0, nullptr, nullptr);
    }
}

// level-1 Galerkin element matrices of G from the fine per-element Voigt stresses (Es included)
void galerkin_elements_G(const LevelGeom& gc, const LevelGeom& gf, const double* sig, const uint8_t* mask_f,
                         const uint8_t* mask_c, double* elm_c, cudaStream_t s) {
    unsigned bl = galerkin_grid(gc);
    if (gc.dim == 2) galerkin_kernel<2, 2, 64><<<bl, 64, 0, s>>>(gc, gf, sig, nullptr, mask_f, mask_c, elm_c, 0, nullptr, nullptr);
    else galerkin_kernel<3, 2, GAL3_NT><<<bl, GAL3_NT, 0, s>>>(gc, gf, sig, nullptr, mask_f, mask_c, elm_c, 0, nullptr, nullptr);
}

// M_c = Q_c^T K0 Q_c for the 2^d children (host, once per handle); layout [child][NL*NL]
void galerkin_child_matrices(int dim, const double* K0, double* Mc_host) {
    const int na = 1 << dim, nl = dim * na;
    for (int c = 0; c < na; ++c)
        for (int r = 0; r < nl; ++r)
            for (int q = 0; q < nl; ++q) {
                const int b = r / dim, i = r % dim, b2 = q / dim, j = q % dim;
                double v = 0.0;
                for (int a = 0; a < na; ++a)
                    for (int a2 = 0; a2 < na; ++a2) {
                        double w1 = 1.0, w2 = 1.0;
                        for (int k = 0; k < dim; ++k) {
                            const int sh = dim - 1 - k;
                            const int p1 = ((c >> sh) & 1) + ((a >> sh) & 1), p2 = ((c >> sh) & 1) + ((a2 >> sh) & 1);
                            w1 *= (p1 == 1) ? 0.5 : (p1 == 2 * ((b >> sh) & 1) ? 1.0 : 0.0);
                            w2 *= (p2 == 1) ? 0.5 : (p2 == 2 * ((b2 >> sh) & 1) ? 1.0 : 0.0);
                        }
                        if (w1 != 0.0 && w2 != 0.0) v += w1 * K0[(a * dim + i) * nl + a2 * dim + j] * w2;
                    }
                Mc_host[(c * nl + r) * nl + q] = v;
            }
}

// ---------------------------------------------------------------- stencil assembly
// st[(s*DIM + k)*DIM + k2][node] = sum over elements containing node (local a) and
// node+delta_s (local b = a + delta_s) of elm[E][(a,k),(b,k2)]; identity at fixed DOFs.
template <int DIM>
__global__ void stencil_kernel(LevelGeom g, const double* __restrict__ elm, const uint8_t* __restrict__ mask,
                               double* __restrict__ st, int ident) {
    constexpr int NA = 1 << DIM, NL = DIM * NA;
    constexpr int NS = DIM == 2 ? 9 : 27;
    long long node = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const int s = blockIdx.y;
    if (node >= g.nnodes) return;
    int idx[3] = {0, 0, 0};
    node_coords(g, node, idx);
    int dlt[3];
    {
        int ss = s;
        for (int k = DIM - 1; k >= 0; --k) { dlt[k] = ss % 3 - 1; ss /= 3; }
    }
    double acc[DIM * DIM];
#pragma unroll
    for (int q = 0; q < DIM * DIM; ++q) acc[q] = 0.0;
    for (int a = 0; a < NA; ++a) {
        int b = 0;
        bool ok = true;
        long long el = 0;
        for (int k = 0; k < DIM; ++k) {
            int ab = (a >> (DIM - 1 - k)) & 1;
            int bb = ab + dlt[k];
            if (bb < 0 || bb > 1) ok = false;
            b = b * 2 + (bb & 1);
            int ek = idx[k] - ab;
            if (ek < 0 || ek >= g.N[k]) ok = false;
            el = el * g.N[k] + ek;
        }
        if (!ok) continue;
        const double* m = elm + el * NL * NL;
#pragma unroll
        for (int k = 0; k < DIM; ++k)
#pragma unroll
            for (int k2 = 0; k2 < DIM; ++k2) acc[k * DIM + k2] += m[(a * DIM + k) * NL + b * DIM + k2];
    }
    const int mb = mask[node];
    const bool center = (s == NS / 2);
#pragma unroll
    for (int k = 0; k < DIM; ++k)
#pragma unroll
        for (int k2 = 0; k2 < DIM; ++k2) {
            double v = acc[k * DIM + k2];
            if (ident && center && k == k2 && ((mb >> k) & 1)) v = 1.0;
            st[((long long)(s * DIM + k) * DIM + k2) * g.nnodes + node] = v;
        }
}

// 3D: a CTA per 16 consecutive nodes, thread (node, s) with s fastest, so the threads reading one
// element matrix (its node-a rows, one 3-column block per neighbour s) touch contiguous 192-byte row
// segments and every element entry leaves HBM once; the 243 x 32 results go through shared memory
// so the stencil arrays are written as coalesced 128-byte rows.  Same sums in the same order as
// stencil_kernel (bitwise equal).
__global__ void __launch_bounds__(432) stencil3_tile_kernel(LevelGeom g, const double* __restrict__ elm,
                                                            const uint8_t* __restrict__ mask, double* __restrict__ st,
                                                            int ident) {
    constexpr int NA = 8, NL = 24, NS = 27;
    __shared__ double tile[NS * 9][17];
    const int nl = threadIdx.x / NS, s = threadIdx.x % NS;
    const long long node = (long long)blockIdx.x * 16 + nl;
    double acc[9];
#pragma unroll
    for (int q = 0; q < 9; ++q) acc[q] = 0.0;
    if (node < g.nnodes) {
        const int i2 = (int)(node % g.nn[2]);
        const long long t = node / g.nn[2];
        const int idx[3] = {(int)(t / g.nn[1]), (int)(t % g.nn[1]), i2};
        const int dlt[3] = {s / 9 - 1, (s / 3) % 3 - 1, s % 3 - 1};
        for (int a = 0; a < NA; ++a) {
            int b = 0;
            bool ok = true;
            long long el = 0;
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                const int ab = (a >> (2 - k)) & 1;
                const int bb = ab + dlt[k];
                if (bb < 0 || bb > 1) ok = false;
                b = b * 2 + (bb & 1);
                const int ek = idx[k] - ab;
                if (ek < 0 || ek >= g.N[k]) ok = false;
                el = el * g.N[k] + ek;
            }
            if (!ok) continue;
            const double* m = elm + el * NL * NL;
#pragma unroll
            for (int k = 0; k < 3; ++k)
#pragma unroll
                for (int k2 = 0; k2 < 3; ++k2) acc[k * 3 + k2] += m[(a * 3 + k) * NL + b * 3 + k2];
        }
        const int mb = mask[node];
        if (ident && s == NS / 2)
#pragma unroll
            for (int k = 0; k < 3; ++k)
                if ((mb >> k) & 1) acc[k * 3 + k] = 1.0;
    }
#pragma unroll
    for (int e = 0; e < 9; ++e) tile[s * 9 + e][nl] = acc[e];
    __syncthreads();
    const long long n0 = (long long)blockIdx.x * 16;
    for (int q = threadIdx.x; q < NS * 9 * 16; q += blockDim.x) {
        const int arr = q >> 4, j = q & 15;
        if (n0 + j < g.nnodes) st[(long long)arr * g.nnodes + n0 + j] = tile[arr][j];
    }
}

void stencil_from_elements(const LevelGeom& g, const double* elm, uint8_t* mask, double* st, cudaStream_t s,
                           bool identity_fixed) {
    int th = 128;
    dim3 grid((unsigned)((g.nnodes + th - 1) / th), g.dim == 2 ? 9 : 27);
    static const bool tiled = !getenv("MG_STENCIL_TILE") || atoi(getenv("MG_STENCIL_TILE")) != 0;
    if (g.dim == 2)
        stencil_kernel<2><<<grid, th, 0, s>>>(g, elm, mask, st, identity_fixed ? 1 : 0);
    else if (tiled)
        stencil3_tile_kernel<<<(unsigned)((g.nnodes + 15) / 16), 432, 0, s>>>(g, elm, mask, st, identity_fixed ? 1 : 0);
    else
        stencil_kernel<3><<<grid, th, 0, s>>>(g, elm, mask, st, identity_fixed ? 1 : 0);
}

// Diagonal from the stencil centre; free DOFs with zero Galerkin diagonal become fixed.
template <int DIM>
__global__ void stencil_diag_kernel(LevelGeom g, uint8_t* mask, double* st, double* Dinv, double* D) {
    constexpr int NS = DIM == 2 ? 9 : 27;
    long long node = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (node >= g.nnodes) return;
    int mb = mask[node];
    for (int k = 0; k < DIM; ++k) {
        double* dp = st + ((long long)((NS / 2) * DIM + k) * DIM + k) * g.nnodes + node;
        double dv = *dp;
        if (!((mb >> k) & 1) && !(dv > 0.0)) {
            mb |= 1 << k;
            *dp = 1.0;
            dv = 1.0;
        }
        if (D) D[DIM * node + k] = dv;
        Dinv[DIM * node + k] = 1.0 / dv;
    }
    mask[node] = (uint8_t)mb;
}

void stencil_diag(const LevelGeom& g, const double* /*st*/, uint8_t* mask, double* st_rw, double* Dinv, double* D,
                  cudaStream_t s) {
    int th = 256;
    unsigned bl = (unsigned)((g.nnodes + th - 1) / th);
    if (g.dim == 2)
        stencil_diag_kernel<2><<<bl, th, 0, s>>>(g, mask, st_rw, Dinv, D);
    else
        stencil_diag_kernel<3><<<bl, th, 0, s>>>(g, mask, st_rw, Dinv, D);
}

// ---------------------------------------------------------------- stencil operator kernels
// Thread per node; all R vectors (chunks of RB) accumulated in registers so the
// stencil (3^d d^2 doubles per node) is read once per chunk.  The 3^d neighbour loop is
// unrolled (compile-time offsets, no local-memory index arrays).
template <int DIM, int OP, int RB, bool SYMH>
__global__ void __launch_bounds__(128) coarse_kernel(CoarseArgs a, int r0, int xs) {
    pdl_begin();
    constexpr int NS = DIM == 2 ? 9 : 27;
    // RHS groups spread over grid.y (small levels), or over xs consecutive blocks (blockIdx.x % xs),
    // so the groups of a node block run side by side and all but one read the stencil from L2
    r0 += (xs ? (int)(blockIdx.x % xs) : (int)blockIdx.y) * RB;
    long long node = (long long)(xs ? blockIdx.x / xs : blockIdx.x) * blockDim.x + threadIdx.x;
    if (node >= a.g.nnodes) return;
    if (a.done && *a.done) return;
    const int n1 = a.g.nn[1], n2 = DIM == 3 ? a.g.nn[2] : 1;
    int i0, i1, i2 = 0;
    if (DIM == 3) {
        i2 = (int)(node % n2);
        const long long t = node / n2;
        i1 = (int)(t % n1);
        i0 = (int)(t / n1);
    } else {
        i1 = (int)(node % n1);
        i0 = (int)(node / n1);
    }
    const int nr = min(RB, a.R - r0);
    bool act[RB];
#pragma unroll
    for (int q = 0; q < RB; ++q) act[q] = (q < nr) && (!a.active || a.active[r0 + q]);
    double acc[RB][DIM];
#pragma unroll
    for (int q = 0; q < RB; ++q)
#pragma unroll
        for (int k = 0; k < DIM; ++k) acc[q][k] = 0.0;
    const long long nn = a.g.nnodes;
#pragma unroll
    for (int s = 0; s < NS; ++s) {
        const int d0 = DIM == 3 ? s / 9 - 1 : s / 3 - 1;
        const int d1 = DIM == 3 ? (s / 3) % 3 - 1 : s % 3 - 1;
        const int d2 = DIM == 3 ? s % 3 - 1 : 0;
        const bool ok = i0 + d0 >= 0 && i0 + d0 < a.g.nn[0] && i1 + d1 >= 0 && i1 + d1 < n1 &&
                        (DIM == 2 || (i2 + d2 >= 0 && i2 + d2 < n2));
        if (!ok) continue;
        const long long q = node + ((long long)d0 * n1 + d1) * n2 + d2;
        double blk[DIM * DIM];
        if (SYMH && s < NS / 2) {
            // lower half from the transposed upper block stored at the neighbour: A(i, q) = A(q, i)^T
            // (the coarse operator is symmetric, P' K P); that block was (or will be) read by node q
            // itself shortly, so the lower half of the stencil never leaves HBM
#pragma unroll
            for (int k = 0; k < DIM; ++k)
#pragma unroll
                for (int k2 = 0; k2 < DIM; ++k2)
                    blk[k * DIM + k2] = __ldg(a.st + (long long)((NS - 1 - s) * DIM * DIM + k2 * DIM + k) * nn + q);
        } else {
#pragma unroll
            for (int e = 0; e < DIM * DIM; ++e) blk[e] = __ldcs(a.st + (long long)(s * DIM * DIM + e) * nn + node);   // streamed once: keep L1 for x
        }
#pragma unroll
        for (int rr = 0; rr < RB; ++rr) {
            if (!act[rr]) continue;
            const double* xv = a.x + (long long)(r0 + rr) * a.g.ndof + (long long)DIM * q;
            double xq[DIM];
#pragma unroll
            for (int k2 = 0; k2 < DIM; ++k2) xq[k2] = xv[k2];
#pragma unroll
            for (int k = 0; k < DIM; ++k)
#pragma unroll
                for (int k2 = 0; k2 < DIM; ++k2) acc[rr][k] = fma(blk[k * DIM + k2], xq[k2], acc[rr][k]);
        }
    }
#pragma unroll
    for (int rr = 0; rr < RB; ++rr) {
        if (!act[rr]) continue;
        const long long o = (long long)(r0 + rr) * a.g.ndof + (long long)DIM * node;
#pragma unroll
        for (int k = 0; k < DIM; ++k) {
            double v;
            if (OP == COP_MATVEC) v = acc[rr][k];
            else if (OP == COP_RESID) v = a.b[o + k] - acc[rr][k];
            else v = a.x[o + k] + a.omega * a.Dinv[(long long)DIM * node + k] * (a.b[o + k] - acc[rr][k]);
            a.y[o + k] = v;
        }
    }
}

// Small levels: one warp per (32 nodes, output component k) -- a CTA is DIM warps over the same
// 32 nodes -- and all RB right-hand sides per thread.  Each thread reads its row k of the node's
// 3^d blocks once (the stencil leaves HBM once instead of once per RHS) and the neighbour
// vectors from L1; DIM x more threads than node-per-thread at the same stencil traffic.
template <int DIM, int OP, int RB>
__global__ void __launch_bounds__(32 * DIM) coarse_comp_kernel(CoarseArgs a, int r0) {
    pdl_begin();
    constexpr int NS = DIM == 2 ? 9 : 27;
    const int k = threadIdx.x >> 5;
    const long long node = (long long)blockIdx.x * 32 + (threadIdx.x & 31);
    if (node >= a.g.nnodes) return;
    if (a.done && *a.done) return;
    const int n1 = a.g.nn[1], n2 = DIM == 3 ? a.g.nn[2] : 1;
    int i0, i1, i2 = 0;
    if (DIM == 3) {
        i2 = (int)(node % n2);
        const long long t = node / n2;
        i1 = (int)(t % n1);
        i0 = (int)(t / n1);
    } else {
        i1 = (int)(node % n1);
        i0 = (int)(node / n1);
    }
    const int nr = min(RB, a.R - r0);
    bool act[RB];
#pragma unroll
    for (int q = 0; q < RB; ++q) act[q] = (q < nr) && (!a.active || a.active[r0 + q]);
    double acc[RB];
#pragma unroll
    for (int q = 0; q < RB; ++q) acc[q] = 0.0;
    const long long nn = a.g.nnodes;
#pragma unroll
    for (int s = 0; s < NS; ++s) {
        const int d0 = DIM == 3 ? s / 9 - 1 : s / 3 - 1;
        const int d1 = DIM == 3 ? (s / 3) % 3 - 1 : s % 3 - 1;
        const int d2 = DIM == 3 ? s % 3 - 1 : 0;
        const bool ok = i0 + d0 >= 0 && i0 + d0 < a.g.nn[0] && i1 + d1 >= 0 && i1 + d1 < n1 &&
                        (DIM == 2 || (i2 + d2 >= 0 && i2 + d2 < n2));
        if (!ok) continue;
        const long long q = node + ((long long)d0 * n1 + d1) * n2 + d2;
        double blk[DIM];
#pragma unroll
        for (int k2 = 0; k2 < DIM; ++k2) blk[k2] = __ldcs(a.st + (long long)((s * DIM + k) * DIM + k2) * nn + node);
#pragma unroll
        for (int rr = 0; rr < RB; ++rr) {
            if (!act[rr]) continue;
            const double* xv = a.x + (long long)(r0 + rr) * a.g.ndof + (long long)DIM * q;
#pragma unroll
            for (int k2 = 0; k2 < DIM; ++k2) acc[rr] = fma(blk[k2], __ldg(xv + k2), acc[rr]);
        }
    }
#pragma unroll
    for (int rr = 0; rr < RB; ++rr) {
        if (!act[rr]) continue;
        const long long o = (long long)(r0 + rr) * a.g.ndof + (long long)DIM * node + k;
        double v;
        if (OP == COP_MATVEC) v = acc[rr];
        else if (OP == COP_RESID) v = a.b[o] - acc[rr];
        else v = a.x[o] + a.omega * a.Dinv[(long long)DIM * node + k] * (a.b[o] - acc[rr]);
        a.y[o] = v;
    }
}

// Small levels (latency-bound): a CTA takes 32 nodes; warp (k, p) = output component k and the
// neighbour plane d0 = p - 1 (9 offsets), all RB right-hand sides per thread, branch-free loads (an
// out-of-grid neighbour reads the node itself against the zero stencil block) so a thread's loads are
// all in flight at once; the three plane partials are summed in shared memory in a fixed order.
template <int OP, int RB, int SP>
__global__ void __launch_bounds__(96 * SP) coarse_split_kernel(CoarseArgs a, int r0) {
    pdl_begin();
    // SP = 3: warp (k, p) with p = the neighbour plane d0 (9 offsets each); SP = 9: p = (d0, d1)
    // (3 offsets each) -- more loads in flight for the smallest levels
    extern __shared__ double part[];   // [3 k][SP p][RB][32 lanes]
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, k = w / SP, p = w % SP;
    const long long node0 = (long long)blockIdx.x * 32 + lane;
    if (a.done && *a.done) return;
    const bool valid = node0 < a.g.nnodes;
    const long long node = valid ? node0 : 0;
    const int n1 = a.g.nn[1], n2 = a.g.nn[2];
    const int i2 = (int)(node % n2);
    const long long t = node / n2;
    const int i1 = (int)(t % n1), i0 = (int)(t / n1);
    const int nr = min(RB, a.R - r0);
    const long long nn = a.g.nnodes;
    double acc[RB];
#pragma unroll
    for (int q = 0; q < RB; ++q) acc[q] = 0.0;
    constexpr int NO = 27 / SP;   // offsets per thread
#pragma unroll
    for (int so = 0; so < NO; ++so) {
        const int s = p * NO + so;
        const int d0 = s / 9 - 1, d1 = (s / 3) % 3 - 1, d2 = s % 3 - 1;
        const bool ok = i0 + d0 >= 0 && i0 + d0 < a.g.nn[0] && i1 + d1 >= 0 && i1 + d1 < n1 && i2 + d2 >= 0 && i2 + d2 < n2;
        const long long q = ok ? node + ((long long)d0 * n1 + d1) * n2 + d2 : node;
        double blk[3];
#pragma unroll
        for (int k2 = 0; k2 < 3; ++k2) blk[k2] = __ldg(a.st + (long long)((s * 3 + k) * 3 + k2) * nn + node);
#pragma unroll
        for (int rr = 0; rr < RB; ++rr) {
            if (rr >= nr) continue;   // uniform
            const double* xv = a.x + (long long)(r0 + rr) * a.g.ndof + 3 * q;
#pragma unroll
            for (int k2 = 0; k2 < 3; ++k2) acc[rr] = fma(blk[k2], __ldg(xv + k2), acc[rr]);
        }
    }
#pragma unroll
    for (int rr = 0; rr < RB; ++rr) part[((k * SP + p) * RB + rr) * 32 + lane] = acc[rr];
    __syncthreads();
    if (p != 0 || !valid) return;
#pragma unroll
    for (int rr = 0; rr < RB; ++rr) {
        if (rr >= nr || (a.active && !a.active[r0 + rr])) continue;
        double v3 = part[((k * SP + 0) * RB + rr) * 32 + lane];
#pragma unroll
        for (int pp = 1; pp < SP; ++pp) v3 += part[((k * SP + pp) * RB + rr) * 32 + lane];
        const long long o = (long long)(r0 + rr) * a.g.ndof + 3 * node + k;
        double v;
        if (OP == COP_MATVEC) v = v3;
        else if (OP == COP_RESID) v = a.b[o] - v3;
        else v = a.x[o] + a.omega * a.Dinv[3 * node + k] * (a.b[o] - v3);
        a.y[o] = v;
    }
}

template <int OP, int SP>
static void launch_coarse_split_sp(const CoarseArgs& a, cudaStream_t s) {
    const unsigned bc = (unsigned)((a.g.nnodes + 31) / 32);
    for (int r0 = 0; r0 < a.R; r0 += 8) {
        const int rb = a.R - r0 > 4 ? 8 : (a.R - r0 > 1 ? 4 : 1);
        const size_t sm = sizeof(double) * 3 * SP * rb * 32;
        if (rb == 8) {
            static bool at = (cudaFuncSetAttribute(coarse_split_kernel<OP, 8, SP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm), true);
            (void)at;
            launch_kp(false, coarse_split_kernel<OP, 8, SP>, dim3(bc), dim3(96 * SP), sm, s, a, r0);
        } else if (rb == 4) {
            launch_kp(false, coarse_split_kernel<OP, 4, SP>, dim3(bc), dim3(96 * SP), sm, s, a, r0);
        } else {
            launch_kp(false, coarse_split_kernel<OP, 1, SP>, dim3(bc), dim3(96 * SP), sm, s, a, r0);
        }
    }
}

// MG_COARSE_SPLIT9: levels below this many nodes (default 40000, i.e. every split level) split the
// offsets 9 ways (B200 C4: 17.15 ms/step with 3 ways, 16.35 with 9)
template <int OP>
static void launch_coarse_split(const CoarseArgs& a, cudaStream_t s) {
    static const long long s9 = getenv("MG_COARSE_SPLIT9") ? atoll(getenv("MG_COARSE_SPLIT9")) : 40000;
    if (a.g.nnodes < s9) launch_coarse_split_sp<OP, 9>(a, s);
    else launch_coarse_split_sp<OP, 3>(a, s);
}

template <int DIM, int OP, bool SYMH>
static void launch_coarse_large(const CoarseArgs& a, unsigned bl, int th, cudaStream_t s) {
    for (int r0 = 0; r0 < a.R;) {
        int rem = a.R - r0;
        if (rem > 8) {
            launch_kp(false, coarse_kernel<DIM, OP, 16, SYMH>, dim3(bl), dim3(th), 0, s, a, r0, 0);
            r0 += 16;
        } else if (rem > 4) {
            // MG_COARSE_XSPLIT = 2 (default): two RHS groups of 4 per node block, 4: four of 2, 0: all 8
            // per thread (fewer accumulators per thread: more resident warps; B200 C5 solve -0.5 ms)
            static const int xsplit = getenv("MG_COARSE_XSPLIT") ? atoi(getenv("MG_COARSE_XSPLIT")) : 2;
            if (xsplit == 4) launch_kp(false, coarse_kernel<DIM, OP, 2, SYMH>, dim3(4 * bl), dim3(th), 0, s, a, r0, 4);
            else if (xsplit == 2) launch_kp(false, coarse_kernel<DIM, OP, 4, SYMH>, dim3(2 * bl), dim3(th), 0, s, a, r0, 2);
            else launch_kp(false, coarse_kernel<DIM, OP, 8, SYMH>, dim3(bl), dim3(th), 0, s, a, r0, 0);
            r0 += 8;
        } else if (rem > 1) {
            launch_kp(false, coarse_kernel<DIM, OP, 4, SYMH>, dim3(bl), dim3(th), 0, s, a, r0, 0);
            r0 += 4;
        } else {
            launch_kp(false, coarse_kernel<DIM, OP, 1, SYMH>, dim3(bl), dim3(th), 0, s, a, r0, 0);
            r0 += 1;
        }
    }
}

template <int DIM, int OP>
static void launch_coarse_dim(const CoarseArgs& a, cudaStream_t s) {
    int th = 128;
    unsigned bl = (unsigned)((a.g.nnodes + th - 1) / th);
    // 3D levels below MG_COARSE_SPLIT nodes (default 40000): plane-split kernel
    static const long long split = getenv("MG_COARSE_SPLIT") ? atoll(getenv("MG_COARSE_SPLIT")) : 40000;
    if (DIM == 3 && a.g.nnodes < split) {
        launch_coarse_split<OP>(a, s);
        return;
    }
    if (bl < 2 * 148) {   // small level: warp per (32 nodes, component), all RHS per thread
        static const bool comp = !getenv("MG_COARSE_COMP") || atoi(getenv("MG_COARSE_COMP")) != 0;
        if (!comp) {   // former path: one RHS per thread, RHS over grid.y (stencil from L2)
            launch_kp(false, coarse_kernel<DIM, OP, 1, false>, dim3(dim3(bl, a.R)), dim3(th), 0, s, a, 0, 0);
            return;
        }
        const unsigned bc = (unsigned)((a.g.nnodes + 31) / 32);
        for (int r0 = 0; r0 < a.R; r0 += 8) {
            if (a.R - r0 > 4) launch_kp(false, coarse_comp_kernel<DIM, OP, 8>, dim3(bc), dim3(32 * DIM), 0, s, a, r0);
            else if (a.R - r0 > 1) launch_kp(false, coarse_comp_kernel<DIM, OP, 4>, dim3(bc), dim3(32 * DIM), 0, s, a, r0);
            else launch_kp(false, coarse_comp_kernel<DIM, OP, 1>, dim3(bc), dim3(32 * DIM), 0, s, a, r0);
        }
        return;
    }
    // large levels read the upper half of the stencil only (MG_COARSE_SYMH=0: the whole stencil)
    static const bool symh = !getenv("MG_COARSE_SYMH") || atoi(getenv("MG_COARSE_SYMH")) != 0;
    if (symh) launch_coarse_large<DIM, OP, true>(a, bl, th, s);
    else launch_coarse_large<DIM, OP, false>(a, bl, th, s);
}

void coarse_apply(int op, const CoarseArgs& a, cudaStream_t s) {
    if (a.g.dim == 2) {
        if (op == COP_MATVEC) launch_coarse_dim<2, COP_MATVEC>(a, s);
        else if (op == COP_RESID) launch_coarse_dim<2, COP_RESID>(a, s);
        else launch_coarse_dim<2, COP_JACOBI>(a, s);
    } else {
        if (op == COP_MATVEC) launch_coarse_dim<3, COP_MATVEC>(a, s);
        else if (op == COP_RESID) launch_coarse_dim<3, COP_RESID>(a, s);
        else launch_coarse_dim<3, COP_JACOBI>(a, s);
    }
}
