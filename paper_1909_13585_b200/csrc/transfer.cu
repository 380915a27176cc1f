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

// ---------------------------------------------------------------- padded 3D fine level <-> level 1
// Thread per coarse node (I, J, m) in compact coarse order, all R right-hand sides per thread.  The
// fine node pair (2m, 2m + 1) of a fine row is 16-byte aligned in the padded layout (p2 even), so a
// warp moves the fine rows it touches as contiguous 16-byte loads / stores, and the third fine
// column a coarse node needs (2m - 1 for restriction, the coarse column m + 1 for prolongation)
// comes from the neighbouring lane by a shuffle (lane 0 / 31 load it themselves).  Every fine value
// is read (restriction) or written (prolongation) by one thread per fine (plane, row).
__device__ __forceinline__ double tp_mask(int mk, int k, double v) { return ((mk >> k) & 1) ? 0.0 : v; }

__global__ void __launch_bounds__(128) restrict3p_kernel(LevelGeom gf, LevelGeom gc, const uint8_t* __restrict__ mf,
                                                         const uint8_t* __restrict__ mc, const double* __restrict__ fine,
                                                         double* __restrict__ coarse, int R, const int* active,
                                                         const int* done, int off0, int fo0, int fo1) {
    pdl_begin();
    if (done && *done) return;
    const long long I = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const bool valid = I < gc.nnodes;
    const int lane = threadIdx.x & 31;
    const long long Ic = valid ? I : 0;
    const int m = (int)(Ic % gc.nn[2]);
    const long long t = Ic / gc.nn[2];
    const int J = (int)(t % gc.nn[1]), P = (int)(t / gc.nn[1]);
    const int n1 = gf.nn[1], n2 = gf.nn[2], p2 = gf.p2;
    const int c = 2 * m;
    const bool left_ld = lane == 0 && m > 0;   // column 2m - 1 not held by a lane of this warp
    // masks of the 9 fine (plane, row) combinations: bits 0-2 node 2m, 3-5 node 2m + 1, 6-8 node 2m - 1
    int mk[9];
    long long rowv[9];   // vector offset of fine node (g0, g1, 2m), -1 when the combination is out of range
#pragma unroll
    for (int q = 0; q < 9; ++q) {
        const int g0 = 2 * P - off0 + q / 3 - 1, g1 = 2 * J + q % 3 - 1;
        const bool ok = valid && g0 >= 0 && g0 < gf.nn[0] && g0 >= fo0 && g0 < fo1 && g1 >= 0 && g1 < n1;
        rowv[q] = ok ? 3 * (((long long)g0 * n1 + g1) * p2 + c) : -1;
        int b = 0x1ff;
        if (ok) {
            const long long mi = ((long long)g0 * n1 + g1) * n2 + c;
            b = mf[mi] | ((c + 1 < n2 ? mf[mi + 1] : 7) << 3) | ((left_ld ? mf[mi - 1] : 7) << 6);
        }
        mk[q] = b;
    }
    const int mcb = valid ? mc[Ic] : 7;
    const int rg = (R + gridDim.y - 1) / gridDim.y;   // RHS group of this thread (grid.y > 1 on small levels)
    for (int r = blockIdx.y * rg; r < min(R, (int)(blockIdx.y + 1) * rg); ++r) {
        if (active && !active[r]) continue;   // uniform
        const double* fv = fine + (long long)r * gf.vstr;
        double acc[3] = {0.0, 0.0, 0.0};
#pragma unroll
        for (int q = 0; q < 9; ++q) {
            const double w = ((q / 3) != 1 ? 0.5 : 1.0) * ((q % 3) != 1 ? 0.5 : 1.0);
            double a[3] = {0.0, 0.0, 0.0}, b[3] = {0.0, 0.0, 0.0}, l[3] = {0.0, 0.0, 0.0};
            if (rowv[q] >= 0) {
                const double2* p = reinterpret_cast<const double2*>(fv + rowv[q]);
                const double2 v0 = __ldg(p), v1 = __ldg(p + 1), v2 = __ldg(p + 2);
                a[0] = tp_mask(mk[q], 0, v0.x); a[1] = tp_mask(mk[q], 1, v0.y); a[2] = tp_mask(mk[q], 2, v1.x);
                b[0] = tp_mask(mk[q], 3, v1.y); b[1] = tp_mask(mk[q], 4, v2.x); b[2] = tp_mask(mk[q], 5, v2.y);
                if (left_ld) {
#pragma unroll
                    for (int k = 0; k < 3; ++k) l[k] = tp_mask(mk[q], 6 + k, __ldg(fv + rowv[q] - 3 + k));
                }
            }
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                const double up = __shfl_up_sync(MGK_FULL, b[k], 1);
                const double left = lane == 0 ? l[k] : (m > 0 ? up : 0.0);
                acc[k] = fma(w, a[k] + 0.5 * (b[k] + left), acc[k]);
            }
        }
        if (valid) {
            double* cv = coarse + (long long)r * gc.ndof + 3 * Ic;
#pragma unroll
            for (int k = 0; k < 3; ++k) cv[k] = tp_mask(mcb, k, acc[k]);
        }
    }
}

__global__ void __launch_bounds__(128) prolong3p_kernel(LevelGeom gf, LevelGeom gc, const uint8_t* __restrict__ mf,
                                                        const uint8_t* __restrict__ mc, const double* __restrict__ coarse,
                                                        double* fine, int R, const int* active, const int* done,
                                                        bool accumulate, int off0, const double* __restrict__ rb,
                                                        const double* __restrict__ dinv, double omega) {
    pdl_begin();
    if (done && *done) return;
    const long long I = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const bool valid = I < gc.nnodes;
    const int lane = threadIdx.x & 31;
    const long long Ic = valid ? I : 0;
    const int m = (int)(Ic % gc.nn[2]);
    const long long t = Ic / gc.nn[2];
    const int J = (int)(t % gc.nn[1]), P = (int)(t / gc.nn[1]);
    const int cn1 = gc.nn[1], cn2 = gc.nn[2];
    const int n1 = gf.nn[1], n2 = gf.nn[2], p2 = gf.p2;
    const bool right_ld = lane == 31 && m + 1 < cn2;   // coarse column m + 1 not held by a lane of this warp
    // coarse nodes (P + a, J + b, m) (and m + 1 for lane 31): offsets, -1 outside; masks
    long long co[4];
    int cm[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const int Pa = P + (q >> 1), Jb = J + (q & 1);
        const bool ok = valid && Pa < gc.nn[0] && Jb < cn1;
        co[q] = ok ? ((long long)Pa * cn1 + Jb) * cn2 + m : -1;
        cm[q] = ok ? (mc[co[q]] | ((right_ld ? mc[co[q] + 1] : 7) << 3)) : 0x3f;
    }
    // fine (plane, row) pairs (2P + a - off0, 2J + b): vector offset of node 2m, -1 outside; masks
    long long fo[4];
    int fm[4];
    const int c = 2 * m;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const int g0 = 2 * P + (q >> 1) - off0, g1 = 2 * J + (q & 1);
        const bool ok = valid && g0 >= 0 && g0 < gf.nn[0] && g1 < n1;
        fo[q] = ok ? 3 * (((long long)g0 * n1 + g1) * p2 + c) : -1;
        const long long mi = ((long long)g0 * n1 + g1) * n2 + c;
        fm[q] = ok ? (mf[mi] | ((c + 1 < n2 ? mf[mi + 1] : 7) << 3)) : 0x3f;
    }
    const int rg = (R + gridDim.y - 1) / gridDim.y;   // RHS group of this thread (grid.y > 1 on small levels)
    for (int r = blockIdx.y * rg; r < min(R, (int)(blockIdx.y + 1) * rg); ++r) {
        if (active && !active[r]) continue;   // uniform
        const double* cv = coarse + (long long)r * gc.ndof;
        // e[a][b][cc][k]: masked coarse values at (P + a, J + b, m + cc)
        double e[2][2][2][3];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            double own[3] = {0.0, 0.0, 0.0}, rt[3] = {0.0, 0.0, 0.0};
            if (co[q] >= 0) {
#pragma unroll
                for (int k = 0; k < 3; ++k) own[k] = tp_mask(cm[q], k, __ldg(cv + 3 * co[q] + k));
                if (right_ld) {
#pragma unroll
                    for (int k = 0; k < 3; ++k) rt[k] = tp_mask(cm[q], 3 + k, __ldg(cv + 3 * co[q] + 3 + k));
                }
            }
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                const double dn = __shfl_down_sync(MGK_FULL, own[k], 1);
                e[q >> 1][q & 1][0][k] = own[k];
                e[q >> 1][q & 1][1][k] = lane == 31 ? rt[k] : (m + 1 < cn2 ? dn : 0.0);
            }
        }
        double* fvr = fine + (long long)r * gf.vstr;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            if (fo[q] < 0) continue;
            const int a = q >> 1, b = q & 1;
            double v[2][3];
#pragma unroll
            for (int cc = 0; cc < 2; ++cc)
#pragma unroll
                for (int k = 0; k < 3; ++k) {
                    // along axis 0 / 1: even fine index -> coincident coarse node, odd -> mean of two
                    auto pl = [&](int bb, int c2) { return a ? 0.5 * (e[0][bb][c2][k] + e[1][bb][c2][k]) : e[0][bb][c2][k]; };
                    auto rw = [&](int c2) { return b ? 0.5 * (pl(0, c2) + pl(1, c2)) : pl(0, c2); };
                    v[cc][k] = cc ? 0.5 * (rw(0) + rw(1)) : rw(0);
                }
            double2* p = reinterpret_cast<double2*>(fvr + fo[q]);
            double o[6];
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                o[k] = tp_mask(fm[q], k, v[0][k]);
                o[3 + k] = (c + 1 < n2) ? tp_mask(fm[q], 3 + k, v[1][k]) : 0.0;   // padding column stays zero
            }
            if (rb) {   // fine = omega D^-1 r + P e: the pre-smoothed z1 formed here from r (not stored)
                const double2* rp = reinterpret_cast<const double2*>(rb + (long long)r * gf.vstr + fo[q]);
                const double2* dp = reinterpret_cast<const double2*>(dinv + fo[q]);
                const double2 r0 = rp[0], r1 = rp[1], r2 = rp[2], d0 = __ldg(dp), d1 = __ldg(dp + 1), d2 = __ldg(dp + 2);
                const double rv[6] = {r0.x, r0.y, r1.x, r1.y, r2.x, r2.y}, dv[6] = {d0.x, d0.y, d1.x, d1.y, d2.x, d2.y};
#pragma unroll
                for (int u = 0; u < 6; ++u) o[u] += __dmul_rn(__dmul_rn(omega, dv[u]), rv[u]);
            } else if (accumulate) {
                const double2 u0 = p[0], u1 = p[1], u2 = p[2];
                o[0] += u0.x; o[1] += u0.y; o[2] += u1.x; o[3] += u1.y; o[4] += u2.x; o[5] += u2.y;
            }
            p[0] = make_double2(o[0], o[1]);
            p[1] = make_double2(o[2], o[3]);
            p[2] = make_double2(o[4], o[5]);
        }
    }
}

// the pair kernels need the padded 3D fine layout (even row pitch, zero padding column)
static bool tp_ok(const LevelGeom& gf, const LevelGeom& gc, const void* fine) {
    static const int on = getenv("MG_TRANSFER_PAIR") ? atoi(getenv("MG_TRANSFER_PAIR")) : 1;
    return on && gf.dim == 3 && (gf.p2 & 1) == 0 && gf.p2 == gf.nn[2] + 1 && gc.nn[2] * 2 - 1 == gf.nn[2] &&
           ((uintptr_t)fine & 15) == 0 && (gf.vstr & 1) == 0;
}

void restrict_apply(const LevelGeom& gf, const LevelGeom& gc, const uint8_t* mf, const uint8_t* mc,
                    const double* fine, double* coarse, int R, const int* active, const int* done, cudaStream_t s,
                    int off0, int fo0, int fo1) {
    if (fo1 < 0) fo1 = gf.nn[0];
    if (tp_ok(gf, gc, fine)) {
        const unsigned nb = (unsigned)((gc.nnodes + 127) / 128);
        launch_kp(false, restrict3p_kernel, dim3(nb, nb >= 148 * 8 ? 1 : R), dim3(128), 0, s, gf, gc, mf, mc, fine,
                  coarse, R, active, done, off0, fo0, fo1);
        return;
    }
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

bool prolong_from_r_ok(const LevelGeom& gf, const LevelGeom& gc, const double* fine) { return tp_ok(gf, gc, fine); }

void prolong_add(const LevelGeom& gf, const LevelGeom& gc, const uint8_t* mf, const uint8_t* mc,
                 const double* coarse, double* fine, int R, const int* active, const int* done, bool accumulate,
                 cudaStream_t s, int off0, const double* rb, const double* dinv, double omega) {
    if (tp_ok(gf, gc, fine)) {
        const unsigned nb = (unsigned)((gc.nnodes + 127) / 128);
        launch_kp(false, prolong3p_kernel, dim3(nb, nb >= 148 * 8 ? 1 : R), dim3(128), 0, s, gf, gc, mf, mc, coarse,
                  fine, R, active, done, accumulate, off0, rb, dinv, omega);
        return;
    }
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
