// Grid transfers between consecutive levels (PAPER.md:146 I^j_{j+1}, I^{j+1}_j;
// Alg. 2 l.9 :715).
// P = bilinear / trilinear nodal interpolation (tensor product of the 1-D stencil
// [1/2, 1, 1/2]), restriction R = P^T, both masked by the free-DOF masks of the
// two levels (reading r11: P_m = M_f P M_c).
#include <cstdlib>

#include <cstdint>
#include <cstdlib>

#include "kernels.h"

// coarse(I,k) = free_c(I,k) * sum_{delta in {-1,0,1}^d} w(delta) free_f(2I+delta,k) fine(2I+delta,k)
// Slabs: fine local plane f is coincident with coarse local plane I when f = 2I - off0, and only
// fine planes in [fo0, fo1) (slab-owned) contribute; the coarse ghost plane above then holds a
// partial sum that the owner adds in (reverse halo exchange).  The 3^d neighbour loop is
// unrolled with compile-time weights (no per-thread index arrays).
template <int DIM>
__global__ void restrict_kernel(LevelGeom gf, LevelGeom gc, const uint8_t* __restrict__ mf,
                                const uint8_t* __restrict__ mc, const double* __restrict__ fine,
                                double* __restrict__ coarse, int R, const int* active, const int* done, int off0,
                                int fo0, int fo1) {
    pdl_begin();
    constexpr int NS = DIM == 2 ? 9 : 27;
    long long I = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (I >= gc.nnodes) return;
    if (done && *done) return;
    int ci[3] = {0, 0, 0};
    {
        long long t = I;
        if (DIM == 3) { ci[2] = (int)(t % gc.nn[2]); t /= gc.nn[2]; }
        ci[1] = (int)(t % gc.nn[1]);
        ci[0] = (int)(t / gc.nn[1]);
    }
    const int f0 = 2 * ci[0] - off0, f1 = 2 * ci[1], f2 = DIM == 3 ? 2 * ci[2] : 0;
    const int n1 = gf.nn[1], n2 = DIM == 3 ? gf.nn[2] : 1;
    const int p2 = DIM == 3 ? gf.p2 : 1;   // vector row pitch (padded 3D fine level) vs mask pitch n2
    const long long fbase = ((long long)f0 * n1 + f1) * n2 + f2;
    const long long vfbase = ((long long)f0 * n1 + f1) * p2 + f2;
    const int mcb = mc[I];
    {   // one RHS per thread (grid.y): enough independent loads in flight on small levels
        const int r = blockIdx.y;
        if (active && !active[r]) return;
        const double* fv = fine + (long long)r * gf.vstr;
        double acc[DIM];
#pragma unroll
        for (int k = 0; k < DIM; ++k) acc[k] = 0.0;
#pragma unroll
        for (int s = 0; s < NS; ++s) {
            const int d0 = DIM == 3 ? s / 9 - 1 : s / 3 - 1;
            const int d1 = DIM == 3 ? (s / 3) % 3 - 1 : s % 3 - 1;
            const int d2 = DIM == 3 ? s % 3 - 1 : 0;
            const double w = (d0 ? 0.5 : 1.0) * (d1 ? 0.5 : 1.0) * (d2 ? 0.5 : 1.0);
            const int g0 = f0 + d0;
            const bool ok = g0 >= 0 && g0 < gf.nn[0] && g0 >= fo0 && g0 < fo1 && f1 + d1 >= 0 && f1 + d1 < n1 &&
                            (DIM == 2 || (f2 + d2 >= 0 && f2 + d2 < n2));
            if (!ok) continue;
            const long long q = fbase + ((long long)d0 * n1 + d1) * n2 + d2;
            const long long qv = vfbase + ((long long)d0 * n1 + d1) * p2 + d2;
            const int fm = mf[q];
#pragma unroll
            for (int k = 0; k < DIM; ++k)
                if (!((fm >> k) & 1)) acc[k] = fma(w, fv[DIM * qv + k], acc[k]);
        }
        double* cv = coarse + (long long)r * gc.ndof + DIM * I;
#pragma unroll
        for (int k = 0; k < DIM; ++k) cv[k] = ((mcb >> k) & 1) ? 0.0 : acc[k];
    }
}

void restrict_apply(const LevelGeom& gf, const LevelGeom& gc, const uint8_t* mf, const uint8_t* mc,
                    const double* fine, double* coarse, int R, const int* active, const int* done, cudaStream_t s,
                    int off0, int fo0, int fo1) {
    if (fo1 < 0) fo1 = gf.nn[0];
    int th = 128;
    dim3 bl((unsigned)((gc.nnodes + th - 1) / th), R);
    if (gf.dim == 2)
        launch_kp(false, restrict_kernel<2>, dim3(bl), dim3(th), 0, s, gf, gc, mf, mc, fine, coarse, R, active, done, off0, fo0, fo1);
    else
        launch_kp(false, restrict_kernel<3>, dim3(bl), dim3(th), 0, s, gf, gc, mf, mc, fine, coarse, R, active, done, off0, fo0, fo1);
}

// fine(i,k) (+)= free_f(i,k) * sum_I w free_c(I,k) coarse(I,k): along each axis an even
// fine index takes the coincident coarse node (w = 1), an odd one the two neighbours (1/2 each).
template <int DIM>
__global__ void prolong_kernel(LevelGeom gf, LevelGeom gc, const uint8_t* __restrict__ mf,
                               const uint8_t* __restrict__ mc, const double* __restrict__ coarse,
                               double* __restrict__ fine, int R, const int* active, const int* done, bool accumulate,
                               int off0) {
    pdl_begin();
    long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= gf.nnodes) return;
    if (done && *done) return;
    int fi[3] = {0, 0, 0};
    long long t = i;
    for (int k = DIM - 1; k >= 0; --k) { fi[k] = (int)(t % gf.nn[k]); t /= gf.nn[k]; }
    // vector index of fine node i (row pitch p2 on the padded 3D fine level; masks stay compact)
    const long long iv = DIM == 3 ? ((long long)fi[0] * gf.nn[1] + fi[1]) * gf.p2 + fi[2] : i;
    fi[0] += off0;   // shifted so that coarse plane I is coincident with fi[0] = 2I
    const int mfb = mf[i];
    constexpr int NC = 1 << DIM;
    long long cn[NC];
    double wgt[NC];
    int cm[NC];
#pragma unroll
    for (int s = 0; s < NC; ++s) {
        long long q = 0;
        double w = 1.0;
        bool ok = true;
        for (int k = 0; k < DIM; ++k) {
            int bit = (s >> (DIM - 1 - k)) & 1;
            int c;
            if (fi[k] & 1) { c = (fi[k] >> 1) + bit; w *= 0.5; }
            else { if (bit) { ok = false; } c = fi[k] >> 1; }
            q = q * gc.nn[k] + c;
        }
        cn[s] = ok ? q : 0; wgt[s] = ok ? w : 0.0; cm[s] = ok ? mc[q] : 0xff;
    }
    // RHS group of this thread: grid.y = R on small levels, all RHS per thread on large ones
    const int rg = (R + gridDim.y - 1) / gridDim.y;
    const int rb = blockIdx.y * rg, re = min(R, rb + rg);
    for (int r = rb; r < re; ++r) {
        if (active && !active[r]) continue;
        const double* cv = coarse + (long long)r * gc.ndof;
        double acc[DIM];
#pragma unroll
        for (int k = 0; k < DIM; ++k) acc[k] = 0.0;
#pragma unroll
        for (int s = 0; s < NC; ++s)
#pragma unroll
            for (int k = 0; k < DIM; ++k)
                if (!((cm[s] >> k) & 1)) acc[k] = fma(wgt[s], cv[DIM * cn[s] + k], acc[k]);
        double* fv = fine + (long long)r * gf.vstr + DIM * iv;
#pragma unroll
        for (int k = 0; k < DIM; ++k) {
            double v = ((mfb >> k) & 1) ? 0.0 : acc[k];
            fv[k] = accumulate ? fv[k] + v : v;
        }
    }
}

void prolong_add(const LevelGeom& gf, const LevelGeom& gc, const uint8_t* mf, const uint8_t* mc,
                 const double* coarse, double* fine, int R, const int* active, const int* done, bool accumulate,
                 cudaStream_t s, int off0) {
    int th = 128;
    const long long blocks = (gf.nnodes + th - 1) / th;
    // RHS over grid.y (one RHS per thread) unless the level is large; MG_PROLONG_SPLIT=1 always splits
    static const int split = getenv("MG_PROLONG_SPLIT") ? atoi(getenv("MG_PROLONG_SPLIT")) : 0;
    dim3 bl((unsigned)blocks, (blocks >= 148 * 16 && !split) ? 1 : R);
    if (gf.dim == 2)
        launch_kp(false, prolong_kernel<2>, dim3(bl), dim3(th), 0, s, gf, gc, mf, mc, coarse, fine, R, active, done, accumulate, off0);
    else
        launch_kp(false, prolong_kernel<3>, dim3(bl), dim3(th), 0, s, gf, gc, mf, mc, coarse, fine, R, active, done, accumulate, off0);
}
