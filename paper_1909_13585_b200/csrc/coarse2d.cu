// 2D coarse levels of the V(1,1) cycle fused into two kernels per level (
// smoother reading r13, Galerkin operator PAPER.md:155, transfers PAPER.md:146):
//
//   down  (level l -> l+1):  z1 = omega D^-1 r ;  w = r - A z1 ;  r_{l+1} = P^T w
//   up    (level l)       :  z2 = omega D^-1 r + P e_{l+1} ;  z = z2 + omega D^-1 (r - A z2)
//
// which is exactly the unfused sequence jacobi0 -> residual -> restrict -> (coarser levels)
// -> prolong-add -> damped-Jacobi sweep, but reads r and the stencil once per kernel and
// never stores z1, w or z2: per level ~3.3 R-vectors + 2 stencil reads instead of ~11.5
// R-vectors + 2 stencil reads.
//
// A CTA is a 16 x 32 tile of level-l nodes (one thread per node, rows along axis 0); each
// thread keeps its node's 3x3-block stencil (36 doubles) in registers and the CTA loops over
// all R right-hand sides, so the stencil is read once per kernel.  Neighbour values (z1, w,
// z2, e) go through shared memory.  Slabs: off0 shifts axis-0 parities (coarse plane I is
// fine plane 2I - off0); restriction sources are the slab-owned fine planes [fo0, fo1) only.
#include <algorithm>

#include "kernels.h"

#ifndef MG_C2D_TJ
#define MG_C2D_TJ 32   // thread tile 16 x TJ level-l nodes (TJ = 32: 1 CTA/SM, 16: 2 CTAs/SM)
#endif
static constexpr int CT_I = 16, CT_J = MG_C2D_TJ;   // thread tile (level-l nodes)
static constexpr int C2D_MINB = CT_J == 32 ? 1 : 2;
static constexpr int NSR = 3;                // right-hand sides in flight (cp.async ring)

__device__ __forceinline__ void cpa16c(void* dst, const void* src, bool pred) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(d), "l"(src), "r"(pred ? 16 : 0));
}
__device__ __forceinline__ void cpa_commit_c() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cpa_wait_c() { asm volatile("cp.async.wait_group %0;\n" ::"n"(NSR - 1)); }
__device__ __forceinline__ void cpa_wait_all_c() { asm volatile("cp.async.wait_group 0;\n" ::); }
static constexpr int DN_CI = CT_I / 2 - 2, DN_CJ = CT_J / 2 - 2;  // coarse nodes owned by a down CTA
static constexpr int UP_OI = CT_I - 2, UP_OJ = CT_J - 2;          // level-l nodes owned by an up CTA

__device__ __forceinline__ void load_stencil(const double* __restrict__ st, long long nn, long long node, bool ok,
                                             double (&A)[36]) {
#pragma unroll
    for (int e = 0; e < 36; ++e) A[e] = ok ? st[(long long)e * nn + node] : 0.0;
}

// y = sum_s A_s x(nbr_s) for this node, neighbours from a shared tile of 2-vectors
__device__ __forceinline__ void apply_stencil(const double (&A)[36], const double2 (*tile)[CT_J], int ti, int tj,
                                              double& yx, double& yy) {
    yx = 0.0;
    yy = 0.0;
#pragma unroll
    for (int s = 0; s < 9; ++s) {
        const double2 v = tile[ti + s / 3 - 1][tj + s % 3 - 1];
        yx = fma(A[4 * s + 0], v.x, yx);
        yx = fma(A[4 * s + 1], v.y, yx);
        yy = fma(A[4 * s + 2], v.x, yy);
        yy = fma(A[4 * s + 3], v.y, yy);
    }
}

__global__ void __launch_bounds__(CT_I * CT_J, C2D_MINB) coarse2d_down_kernel(LevelGeom g, LevelGeom gc,
                                                                       const double* __restrict__ st,
                                                                       const double* __restrict__ Dinv,
                                                                       const uint8_t* __restrict__ mask,
                                                                       const uint8_t* __restrict__ maskc,
                                                                       const double* __restrict__ r, double* rc,
                                                                       int R, double omega, int off0, int fo0, int fo1,
                                                                       int nbj, int rg, const int* active,
                                                                       const int* done) {
    pdl_begin();
    __shared__ double2 s_z[CT_I][CT_J];
    __shared__ double2 s_w[CT_I][CT_J];
    __shared__ double2 s_r[NSR][CT_I * CT_J];   // r of the next RHS, per thread
    if (done && *done) return;
    const int ti = threadIdx.x / CT_J, tj = threadIdx.x % CT_J;
    const int bI = blockIdx.x / nbj, bJ = blockIdx.x % nbj;
    const int I0 = bI * DN_CI, J0 = bJ * DN_CJ;
    const int k0 = blockIdx.y * rg, k1 = min(R, k0 + rg);   // this CTA's right-hand sides
    const int fi = 2 * I0 - off0 - 2 + ti, fj = 2 * J0 - 2 + tj;
    const int n0 = g.nn[0], n1 = g.nn[1];
    const bool ok = fi >= 0 && fi < n0 && fj >= 0 && fj < n1;
    const long long node = (long long)fi * n1 + fj;
    const bool wreg = ti >= 1 && ti < CT_I - 1 && tj >= 1 && tj < CT_J - 1;
    double A[36];
    load_stencil(st, g.nnodes, node, ok && wreg, A);   // the halo ring only supplies z1
    const int m = ok ? mask[node] : 3;
    const double dx = ok ? Dinv[2 * node] : 0.0, dy = ok ? Dinv[2 * node + 1] : 0.0;
    // restriction source: slab-owned, free fine DOFs
    const bool src = ok && fi >= fo0 && fi < fo1;
    // coarse owner: ti = 2 + 2a, tj = 2 + 2b
    const bool cown = ti >= 2 && ti <= 2 * DN_CI && !(ti & 1) && tj >= 2 && tj <= 2 * DN_CJ && !(tj & 1);
    const int Ic = I0 + (ti - 2) / 2, Jc = J0 + (tj - 2) / 2;
    const bool cok = cown && Ic < gc.nn[0] && Jc < gc.nn[1];
    const long long cnode = (long long)Ic * gc.nn[1] + Jc;
    const int mc = cok ? maskc[cnode] : 3;
    // software pipeline over the RHS: r of the next NSR - 1 RHS is in flight (cp.async ring, one
    // commit group per RHS; a thread reads only its own slots)
    const int tid = threadIdx.x;
    const double* rnode = r + 2 * node;
#pragma unroll
    for (int q = 0; q < NSR; ++q) {
        if (k0 + q < k1) cpa16c(&s_r[q][tid], rnode + (long long)(k0 + q) * g.ndof, ok);
        cpa_commit_c();
    }
    for (int k = k0; k < k1; ++k) {
        const int st = (k - k0) % NSR;
        cpa_wait_c();
        const double2 rv = s_r[st][tid];
        const double rx = rv.x, ry = rv.y;
        if (k + NSR < k1) cpa16c(&s_r[st][tid], rnode + (long long)(k + NSR) * g.ndof, ok);
        cpa_commit_c();
        if (active && !active[k]) continue;
        s_z[ti][tj] = make_double2(omega * dx * rx, omega * dy * ry);
        __syncthreads();
        if (wreg) {
            double ax, ay;
            apply_stencil(A, s_z, ti, tj, ax, ay);
            const double wx = (src && !(m & 1)) ? rx - ax : 0.0;
            const double wy = (src && !(m & 2)) ? ry - ay : 0.0;
            s_w[ti][tj] = make_double2(wx, wy);
        }
        __syncthreads();
        if (cok) {
            double cx = 0.0, cy = 0.0;
#pragma unroll
            for (int s = 0; s < 9; ++s) {
                const int di = s / 3 - 1, dj = s % 3 - 1;
                const double wt = (di ? 0.5 : 1.0) * (dj ? 0.5 : 1.0);
                const double2 v = s_w[ti + di][tj + dj];
                cx = fma(wt, v.x, cx);
                cy = fma(wt, v.y, cy);
            }
            double* cv = rc + (long long)k * gc.ndof + 2 * cnode;
            *reinterpret_cast<double2*>(cv) = make_double2((mc & 1) ? 0.0 : cx, (mc & 2) ? 0.0 : cy);
        }
        // next RHS overwrites s_z only after every thread has passed the second barrier,
        // i.e. finished reading s_z; s_w is rewritten after the next first barrier
    }
    cpa_wait_all_c();
}

__global__ void __launch_bounds__(CT_I * CT_J, C2D_MINB) coarse2d_up_kernel(LevelGeom g, LevelGeom gc,
                                                                     const double* __restrict__ st,
                                                                     const double* __restrict__ Dinv,
                                                                     const uint8_t* __restrict__ mask,
                                                                     const uint8_t* __restrict__ maskc,
                                                                     const double* __restrict__ r,
                                                                     const double* __restrict__ ec, double* z, int R,
                                                                     double omega, int off0, int nbj, int rg,
                                                                     const int* active, const int* done) {
    pdl_begin();
    constexpr int CI = CT_I / 2 + 2, CJ = CT_J / 2 + 2;
    __shared__ double2 s_z[CT_I][CT_J];
    __shared__ double2 s_e[CI][CJ];
    __shared__ double2 s_r[NSR][CT_I * CT_J];   // r of the next RHS, per thread
    __shared__ double2 s_en[NSR][CI * CJ];      // coarse tile entry of the next RHS
    if (done && *done) return;
    const int ti = threadIdx.x / CT_J, tj = threadIdx.x % CT_J;
    const int bI = blockIdx.x / nbj, bJ = blockIdx.x % nbj;
    const int fi0 = bI * UP_OI - 1, fj0 = bJ * UP_OJ - 1;
    const int k0 = blockIdx.y * rg, k1 = min(R, k0 + rg);   // this CTA's right-hand sides
    const int fi = fi0 + ti, fj = fj0 + tj;
    const int n0 = g.nn[0], n1 = g.nn[1];
    const bool ok = fi >= 0 && fi < n0 && fj >= 0 && fj < n1;
    const long long node = (long long)fi * n1 + fj;
    const bool own = ok && ti >= 1 && ti < CT_I - 1 && tj >= 1 && tj < CT_J - 1;
    double A[36];
    load_stencil(st, g.nnodes, node, own, A);   // the halo ring only supplies z2
    const int m = ok ? mask[node] : 3;
    const double dx = ok ? Dinv[2 * node] : 0.0, dy = ok ? Dinv[2 * node + 1] : 0.0;
    // coarse tile: shifted fine index fs = f + off0 maps to coarse fs >> 1 (floor) .. (fs + 1) >> 1
    const int ci0 = (fi0 + off0) >> 1, cj0 = fj0 >> 1;
    const int fsi = fi + off0;
    const int li0 = (fsi >> 1) - ci0, li1 = ((fsi + 1) >> 1) - ci0;
    const int lj0 = (fj >> 1) - cj0, lj1 = ((fj + 1) >> 1) - cj0;
    static_assert(CI * CJ <= CT_I * CT_J, "one coarse tile entry per thread");
    // this thread's coarse tile entry (if any)
    const int ea = threadIdx.x / CJ, eb = threadIdx.x % CJ;
    const int eI = ci0 + ea, eJ = cj0 + eb;
    const bool eok = threadIdx.x < CI * CJ && eI >= 0 && eI < gc.nn[0] && eJ >= 0 && eJ < gc.nn[1];
    const long long ecn = eok ? (long long)eI * gc.nn[1] + eJ : 0;
    const int emc = eok ? maskc[ecn] : 3;
    // software pipeline over the RHS: e and r of the next NSR - 1 RHS are in flight (cp.async ring)
    const int tid = threadIdx.x;
    const bool has_e = tid < CI * CJ;
    const double* rnode = r + 2 * node;
    const double* enode = ec + 2 * ecn;
#pragma unroll
    for (int q = 0; q < NSR; ++q) {
        if (k0 + q < k1) {
            cpa16c(&s_r[q][tid], rnode + (long long)(k0 + q) * g.ndof, ok);
            if (has_e) cpa16c(&s_en[q][tid], enode + (long long)(k0 + q) * gc.ndof, eok);
        }
        cpa_commit_c();
    }
    for (int k = k0; k < k1; ++k) {
        const int st = (k - k0) % NSR;
        cpa_wait_c();
        const double2 rv = s_r[st][tid];
        const double2 ev = has_e ? s_en[st][tid] : make_double2(0.0, 0.0);
        const double rx = rv.x, ry = rv.y;
        if (k + NSR < k1) {
            cpa16c(&s_r[st][tid], rnode + (long long)(k + NSR) * g.ndof, ok);
            if (has_e) cpa16c(&s_en[st][tid], enode + (long long)(k + NSR) * gc.ndof, eok);
        }
        cpa_commit_c();
        if (active && !active[k]) continue;
        if (threadIdx.x < CI * CJ)
            s_e[ea][eb] = make_double2((emc & 1) ? 0.0 : ev.x, (emc & 2) ? 0.0 : ev.y);
        __syncthreads();
        double zx = 0.0, zy = 0.0;
        if (ok) {
            const double2 a00 = s_e[li0][lj0], a01 = s_e[li0][lj1], a10 = s_e[li1][lj0], a11 = s_e[li1][lj1];
            const double px = 0.5 * (0.5 * (a00.x + a01.x) + 0.5 * (a10.x + a11.x));
            const double py = 0.5 * (0.5 * (a00.y + a01.y) + 0.5 * (a10.y + a11.y));
            zx = (m & 1) ? 0.0 : fma(omega * dx, rx, px);
            zy = (m & 2) ? 0.0 : fma(omega * dy, ry, py);
        }
        s_z[ti][tj] = make_double2(zx, zy);
        __syncthreads();
        if (own) {
            double ax, ay;
            apply_stencil(A, s_z, ti, tj, ax, ay);
            const double ox = fma(omega * dx, rx - ax, zx), oy = fma(omega * dy, ry - ay, zy);
            *reinterpret_cast<double2*>(z + (long long)k * g.ndof + 2 * node) = make_double2(ox, oy);
        }
        // s_e is rewritten by the next RHS only after every thread passed the second barrier
        // (all s_e reads done); s_z only after the next first barrier (all s_z reads done)
    }
    cpa_wait_all_c();
}

// RHS per CTA: all of them on large levels (stencil read once); on small levels the RHS are
// spread over CTAs so the grid still covers the SMs (the stencil then comes from L2)
static int rhs_group(int tiles, int R) {
    const int want = 2 * 148;
    if (tiles >= want) return R;
    const int groups = std::min(R, (want + tiles - 1) / tiles);
    return (R + groups - 1) / groups;
}

void coarse2d_down(const LevelGeom& g, const LevelGeom& gc, const double* st, const double* Dinv,
                   const uint8_t* mask, const uint8_t* maskc, const double* r, double* rc, int R, double omega,
                   int off0, int fo0, int fo1, const int* active, const int* done, cudaStream_t s) {
    const int nbi = (gc.nn[0] + DN_CI - 1) / DN_CI, nbj = (gc.nn[1] + DN_CJ - 1) / DN_CJ;
    const int rg = rhs_group(nbi * nbj, R);
    dim3 grid(nbi * nbj, (R + rg - 1) / rg);
    launch_k(coarse2d_down_kernel, dim3(grid), dim3(CT_I * CT_J), 0, s, g, gc, st, Dinv, mask, maskc, r, rc, R, omega, off0, fo0, fo1,
                                                    nbj, rg, active, done);
}

void coarse2d_up(const LevelGeom& g, const LevelGeom& gc, const double* st, const double* Dinv, const uint8_t* mask,
                 const uint8_t* maskc, const double* r, const double* ec, double* z, int R, double omega, int off0,
                 const int* active, const int* done, cudaStream_t s) {
    const int nbi = (g.nn[0] + UP_OI - 1) / UP_OI, nbj = (g.nn[1] + UP_OJ - 1) / UP_OJ;
    const int rg = rhs_group(nbi * nbj, R);
    dim3 grid(nbi * nbj, (R + rg - 1) / rg);
    launch_k(coarse2d_up_kernel, dim3(grid), dim3(CT_I * CT_J), 0, s, g, gc, st, Dinv, mask, maskc, r, ec, z, R, omega, off0, nbj, rg,
                                                  active, done);
}
