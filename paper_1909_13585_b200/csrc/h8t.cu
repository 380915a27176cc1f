// 3D fine level (trilinear H8), TMA plane-ring march.  K = sum_e E_e A_e^T K0 A_e applied
// matrix-free ("K_e = E_kappa K_e0", Eq. 2 :101-108), fused with the damped-Jacobi
// smoother / residual / CG direction of the fine V(1,1)-PCG iteration.
//
// Element operator in the per-axis sum/difference basis (m = v0 + v1, d = v1 - v0): the 1-D mass
// and stiffness matrices are diagonal there and the mixed one has one entry, so
// K^ = T^-T K0 T^-1 has 45 nonzeros instead of 576 (closed form below; equal to K0 after the
// transform for any nu and for the incompatible-mode element, whose K^ has the same pattern).
//
// Work decomposition.  A CTA owns a tile of TR - 1 node rows (axis 1) x 30 node columns (axis 2)
// and marches along axis 0 over a chunk of node planes.  Warp w (0 <= w < TR) handles element
// row j0 + w, lane l element column c0 + l (c0 = 30 tc - 1, j0 = (TR - 1) tr - 1); node rows
// 1..TR-1 / lanes 1..30 of the tile are its outputs.  Per node plane, one thread issues TMA box
// loads (cp.async.bulk.tensor, zero fill outside the grid) of every input field of the tile's
// (TR + 1) x 32 nodes into a ring of NS plane slots (mbarrier complete_tx); the last warp to
// release a slot refills it (smem counter), so no warp waits for a producer.  The only
// cross-warp exchange per plane is row w's contribution to node row w + 1 (6 doubles per lane)
// through a double-buffered shared array with point-to-point mbarriers (warp w -> warp w + 1):
// no CTA-wide barrier inside the march.  Per thread the march carries the element's two forward
// faces and the axis-0 carry of its element results in registers (the loop is unrolled by two
// planes so the faces ping-pong between two register sets without moves).  A last column tile
// that owns <= 9 node columns is marched by a second (TAIL) launch that stacks three such 7-row
// tiles in the lanes of one CTA (three groups of 10 lanes, see TLT below).
//
// Layout (padded 3D fine level, mgcg.cu): vectors (R, n0, n1, p2, 3) with p2 = n2 rounded up to
// even (TMA row strides are multiples of 16 bytes); D^-1 (n0, n1, p2, 3); masks (n0, n1, m2) bytes,
// m2 = n2 rounded up to 16; E compact (N0, N1, N2) when N2 is even, else padded to even.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <type_traits>

#include "element.cuh"
#include "kernels.h"

#ifndef H8T_RAWRE
#define H8T_RAWRE 1
#endif

__constant__ double c_Kt[576];
__constant__ double c_Glm[2];   // lambda, mu of the centroid stress (E = 1) for G(u) phi

// ---------------------------------------------------------------- K^ in closed form
// 1-D factors in the (m, d) basis (t = 0: m, t = 1: d): M^ = diag(1/4, 1/12), D^ = diag(0, 1),
// C^[d][m] = 1/2 (derivative on the test function), C^T[m][d] = 1/2.
// K^[(s,i),(t,j)] = lam S^_ij + mu S^_ji + mu delta_ij sum_k S^_kk.
__host__ __device__ constexpr double t1h(int kind, int ta, int tb) {
    return kind == 0 ? (ta == tb ? (ta == 0 ? 0.25 : 1.0 / 12.0) : 0.0)
         : kind == 1 ? ((ta == 1 && tb == 1) ? 1.0 : 0.0)
         : kind == 2 ? ((ta == 1 && tb == 0) ? 0.5 : 0.0)
                     : ((ta == 0 && tb == 1) ? 0.5 : 0.0);
}
__host__ __device__ constexpr double tsh3(int i, int j, int s, int t) {
    double v = 1.0;
    for (int k = 0; k < 3; ++k) {
        const int ta = (s >> (2 - k)) & 1, tb = (t >> (2 - k)) & 1;
        const int kind = (k == i && k == j) ? 1 : (k == i ? 2 : (k == j ? 3 : 0));
        v *= t1h(kind, ta, tb);
    }
    return v;
}
__host__ __device__ constexpr double tkhat(double nu, int row, int col) {
    const int s = row / 3, i = row % 3, t = col / 3, j = col % 3;
    const double mu = 1.0 / (2.0 * (1.0 + nu));
    const double lam = nu / ((1.0 + nu) * (1.0 - 2.0 * nu));
    double v = lam * tsh3(i, j, s, t) + mu * tsh3(j, i, s, t);
    if (i == j)
        for (int k = 0; k < 3; ++k) v += mu * tsh3(k, k, s, t);
    return v;
}

void h8t_set_constants(const double* K0, double nu, cudaStream_t s) {
    static double lm[2];
    lm[0] = nu / ((1.0 + nu) * (1.0 - 2.0 * nu));
    lm[1] = 1.0 / (2.0 * (1.0 + nu));
    cudaMemcpyToSymbolAsync(c_Glm, lm, sizeof(lm), 0, cudaMemcpyHostToDevice, s);
    static double Ti[24][24], Kh[576];
    for (int a = 0; a < 8; ++a)
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
    cudaMemcpyToSymbolAsync(c_Kt, Kh, sizeof(Kh), 0, cudaMemcpyHostToDevice, s);
}

// nu = 0.3 (C03): lambda / mu = 3/2 exactly, and with the 1-D factors scaled by 12 (M^ = diag(3, 1),
// D^ = diag(0, 12), C^ = 6) every entry of K^ is (mu / 27) times a dyadic rational with a small
// numerator (7 distinct values: 9/16 ... 189/32), so K~ = (27 / mu) K^ enters DFMA as a 32-bit
// immediate instead of a 64-bit constant materialised in two registers per use; the element
// modulus carries the factor mu / 27 (one DMUL per element).
__host__ __device__ constexpr double t1i(int kind, int ta, int tb) {
    return kind == 0 ? (ta == tb ? (ta == 0 ? 3.0 : 1.0) : 0.0)
         : kind == 1 ? ((ta == 1 && tb == 1) ? 12.0 : 0.0)
         : kind == 2 ? ((ta == 1 && tb == 0) ? 6.0 : 0.0)
                     : ((ta == 0 && tb == 1) ? 6.0 : 0.0);
}
__host__ __device__ constexpr double tsh3i(int i, int j, int s, int t) {
    double v = 1.0;
    for (int k = 0; k < 3; ++k) {
        const int ta = (s >> (2 - k)) & 1, tb = (t >> (2 - k)) & 1;
        const int kind = (k == i && k == j) ? 1 : (k == i ? 2 : (k == j ? 3 : 0));
        v *= t1i(kind, ta, tb);
    }
    return v;
}
__host__ __device__ constexpr double tkhat_dy(int row, int col) {   // (27 / mu) K^ at nu = 0.3: exact
    const int s = row / 3, i = row % 3, t = col / 3, j = col % 3;
    double v = 1.5 * tsh3i(i, j, s, t) + tsh3i(j, i, s, t);
    if (i == j)
        for (int k = 0; k < 3; ++k) v += tsh3i(k, k, s, t);
    return v / 64.0;   // x 27 / 12^3
}
static constexpr double H8T_KSCALE = 1.0 / (2.0 * (1.0 + MG_NU_PAPER)) / 27.0;   // mu / 27 at nu = 0.3

template <bool C03>
__device__ __forceinline__ double KT(int r, int c) {
    if (C03) return tkhat_dy(r, c);
    return c_Kt[r * 24 + c];
}

// connected components of the K^ pattern (rows = cols; the rigid-translation rows s = 0 are zero)
static constexpr int T_NCOMP = 11;
__device__ constexpr int T_COMP[T_NCOMP][3] = {{3, 14, -1}, {4, 8, -1},   {5, 7, 12},  {6, 13, -1},
                                               {9, 16, 20}, {10, 15, -1}, {11, 18, -1}, {17, 19, -1},
                                               {21, -1, -1}, {22, -1, -1}, {23, -1, -1}};
// row rr = 3 s + k pairs with rr ^ 12 (s ^ 4: t0 flipped); "seen" = the partner was formed in an
// earlier component (compile time)
__host__ __device__ constexpr bool t_partner_seen(int ci, int q) {
    const int rr = T_COMP[ci][q];
    const int pr = ((rr / 3) ^ 4) * 3 + rr % 3;
    for (int c2 = 0; c2 < ci; ++c2)
        for (int q2 = 0; q2 < 3; ++q2)
            if (T_COMP[c2][q2] == pr) return true;
    for (int q2 = 0; q2 < q; ++q2)
        if (T_COMP[ci][q2] == pr) return true;
    return false;
}

// ---------------------------------------------------------------- PTX helpers (TMA, mbarrier)
__device__ __forceinline__ unsigned t_smem(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void t_mbar_init(uint64_t* b, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(t_smem(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void t_mbar_expect_tx(uint64_t* b, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(t_smem(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void t_mbar_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(t_smem(b)) : "memory");
}
__device__ __forceinline__ void t_mbar_wait(uint64_t* b, unsigned parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "T_WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, 0x989680;\n"
        "@!p bra T_WAIT_%=;\n"
        "}\n" ::"r"(t_smem(b)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void t_tma1(void* dst, const CUtensorMap* m, int c0, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.1d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2}], [%3];\n" ::"r"(
            t_smem(dst)),
        "l"((unsigned long long)m), "r"(c0), "r"(t_smem(bar))
        : "memory");
}
__device__ __forceinline__ void t_tma3(void* dst, const CUtensorMap* m, int c0, int c1, int c2, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(
            t_smem(dst)),
        "l"((unsigned long long)m), "r"(c0), "r"(c1), "r"(c2), "r"(t_smem(bar))
        : "memory");
}
__device__ __forceinline__ void t_tma4(void* dst, const CUtensorMap* m, int c0, int c1, int c2, int c3, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];\n" ::"r"(
            t_smem(dst)),
        "l"((unsigned long long)m), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(t_smem(bar))
        : "memory");
}

// ---------------------------------------------------------------- ring layout
// fields per slot: A (vector), B (vector), C (vector or D^-1), E (element row box), M (mask box)
//   MATVEC: A = x            RESID: A = x, B = b            JACOBI: A = x, B = b, C = D^-1
//   CGP:    A = p_in, B = z, C = x (deferred update; optional)
//   RESTR3: A = r_in, B = q, C = D^-1
// TMA requires the innermost box start to be 16-byte aligned, so the boxes start left of the
// tile (c0 = 30 tc - 1 is odd): vectors at node c0 - 1 (100 doubles = 33 nodes + 1 per row), E at
// element c0 - 1 (34 per row), masks at the 16-byte boundary at or below c0 - 1 (48 bytes per row).
static constexpr int T_VW = 100, T_EW = 34, T_MW = 48;
// G(u) phi reads phi and u in the compact user layout, whose rows (odd node count) are not 16-byte
// aligned: one 1-D box of 102 doubles per row, started at the even double at or below node c0 - 1
// (row offset 0 / 1), rows 128-byte aligned in shared memory
static constexpr int T_VWC = 112, T_RB = 102;
__host__ __device__ constexpr int t_r128(int b) { return (b + 127) / 128 * 128; }
// Tail tile (round 2d): when the last column tile owns <= 9 node columns (C5: 129 = 4 x 30 + 9), its
// CTA stacks three row groups of 10 lanes (lanes 30, 31 idle copies of lane 29) instead of using 10
// of 32 lanes: group g = lane / 10 marches element rows j0 + 7 g + w, i.e. three ordinary 7-row
// tiles side by side in one warp set (same per-lane arithmetic, same exchange).  Boxes: vectors
// {34 doubles, 23 rows}, E {12, 22}, masks {32 bytes, 23 rows} placed in the A field's slack.
static constexpr int TT_G = 10, TT_VW = 34, TT_EW = 12, TT_MW = 32;
template <int TR>
struct TLT {
    static constexpr int BR = 3 * (TR - 1) + 2;   // node rows per box
    static constexpr int ER = 3 * (TR - 1) + 1;   // element rows per box
    static constexpr int VB = BR * TT_VW * 8;
    static constexpr int EB = ER * TT_EW * 8;
    static constexpr int MB = BR * TT_MW;
    static constexpr int OMA = t_r128(VB);        // mask box offset inside the A field
};
template <int OP, int TR, int NB>
struct TL {
    static constexpr int BR = TR + 1;                    // node rows per box
    static constexpr bool HB = OP != FOP_MATVEC;
    static constexpr bool HC = OP == FOP_JACOBI || OP == FOP_CGP || OP == FOP_RESTR3;
    static constexpr int VB = BR * (OP == FOP_GPHI ? T_VWC : T_VW) * 8;   // vector box bytes
    static constexpr int EB = TR * T_EW * 8;             // E box bytes
    static constexpr int MB = BR * T_MW;                 // mask box bytes
    static constexpr int OA = 0;
    static constexpr int OB = OA + t_r128(VB);
    static constexpr int OC = OB + (HB ? t_r128(VB) : 0);
    static constexpr int OE = OC + (HC ? t_r128(VB) : 0);
    static constexpr int OM = OE + t_r128(EB);
    static constexpr int SLOT = t_r128(OM + MB);
    static constexpr int SINV = NB * TR * 6 * 32 * 8;   // row -> row+1 exchange, NB buffers
};

template <int OP, int TR, int NB>
constexpr bool h8t_tail_fits() {
    using T = TL<OP, TR, NB>;
    using U = TLT<TR>;
    return OP != FOP_GPHI && U::VB <= T::VB && U::OMA + U::MB <= t_r128(T::VB) && U::EB <= T::EB;
}

template <int OP, int TR, int NS, int NB>
static constexpr size_t h8t_smem_bytes() {
    using T = TL<OP, TR, NB>;
    return (size_t)NS * T::SLOT + T::SINV + 8 * (NS + 2 * NB * TR) + 8 * NS + 8 * TR;
}

// per-slot expected TMA bytes (zero-filled out-of-range elements count too)
template <int OP, int TR>
__host__ __device__ constexpr unsigned h8t_tx_bytes(bool hasC) {
    if (OP == FOP_GPHI) return (unsigned)(TR * T_EW * 8 + (TR + 1) * T_MW);   // + 2 T_RB * 8 per in-range row
    using T = TL<OP, TR, 1>;
    return (unsigned)(T::VB + (T::HB ? T::VB : 0) + ((T::HC && hasC) ? T::VB : 0) + T::EB + T::MB);
}
template <int OP, int TR>
__host__ __device__ constexpr unsigned h8t_tx_bytes_tail(bool hasC) {
    using T = TL<OP, TR, 1>;
    using U = TLT<TR>;
    return (unsigned)(U::VB + (T::HB ? U::VB : 0) + ((T::HC && hasC) ? U::VB : 0) + U::EB + U::MB);
}

struct H8TMaps {
    CUtensorMap A, B, C, E, M;
};

template <int OP, bool C03, int TR, int NS, int NB, int MINB, bool TAIL>
__global__ void __launch_bounds__(32 * TR, MINB)
    h8t_kernel(const __grid_constant__ FineArgs a, const __grid_constant__ H8TMaps tm, int ntc, int ntr, int nch,
               int hch, int hasC, int tc0, int toff) {
    pdl_begin();
    using T = TL<OP, TR, NB>;
    using U = TLT<TR>;
    static_assert(!TAIL || h8t_tail_fits<OP, TR, NB>(), "tail boxes must fit the slot");
    constexpr int OWNR = TR - 1;
    constexpr int VW = TAIL ? TT_VW : T_VW, EW = TAIL ? TT_EW : T_EW, MW = TAIL ? TT_MW : T_MW;
    constexpr int OMK = TAIL ? T::OA + U::OMA : T::OM;   // mask box offset in a slot
    extern __shared__ __align__(128) unsigned char t_sm[];
    unsigned char* ring = t_sm;
    double* sinv = reinterpret_cast<double*>(t_sm + NS * T::SLOT);                       // [NB][TR][6][32]
    uint64_t* full = reinterpret_cast<uint64_t*>(t_sm + NS * T::SLOT + T::SINV);         // [NS]
    uint64_t* sfull = full + NS;                                                         // [NB][TR]
    uint64_t* sempty = sfull + NB * TR;                                                  // [NB][TR]
    int* cnt = reinterpret_cast<int*>(sempty + NB * TR);                                 // [NS]
    double* s_dot = reinterpret_cast<double*>(t_sm + NS * T::SLOT + T::SINV + 8 * (NS + 2 * NB * TR) + 8 * NS);

    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int R = a.R;
    const int r = blockIdx.x % R;
    const int tile = blockIdx.x / R;
    const int nt = ntc * ntr;
    if (tile >= nt * nch) return;
    if (a.done && *a.done) return;
    if (a.active && !a.active[r]) return;
    const int tc = tc0 + tile % ntc, tr = (tile / ntc) % ntr, ch = tile / nt;
    const int n0 = a.g.nn[0], n1 = a.g.nn[1], n2 = a.g.nn[2];
    const int p2 = a.g.p2;
    const int c0 = 30 * tc - 1, j0 = (TAIL ? 3 * OWNR : OWNR) * tr - 1;
    const int cm0 = (c0 - 1) & ~15;   // mask box start (16-byte aligned)
    // tail: row group g, lane gl within it (lanes 30, 31 duplicate lane 29 and own nothing)
    const int tg = TAIL ? min(lane / TT_G, 2) : 0;
    const int gl = TAIL ? min(lane - TT_G * tg, TT_G - 1) : lane;
    const int rb = TAIL ? OWNR * tg : 0;   // box row of this lane's element row w
    const int mlane = gl + (c0 - cm0);
    const int j = j0 + rb + w, c = c0 + gl;
    const bool own = w >= 1 && gl >= 1 && (TAIL ? lane < 3 * TT_G : lane <= 30) && j < n1 && c < n2;
    const int i0 = ch * hch, i1 = min(i0 + hch, n0);
    const int nq = i1 - i0 + 2;   // planes i0-1 .. i1
    const long long vbase = (long long)r * a.g.vstr + (OP == FOP_GPHI ? a.goffA : 0);
    const long long pstr = (long long)n1 * p2 * 3;          // doubles per node plane (padded)
    const long long nodeoff = 3 * ((long long)j * p2 + c);  // within a plane
    const double beta = OP == FOP_CGP ? a.beta[r] : 0.0;
    const double xal = (OP == FOP_CGP && hasC) ? a.xalpha[r] : 0.0;
    const double alpha = OP == FOP_RESTR3 ? a.alpha[r] : 0.0;
    const double omega = a.omega;
    const bool z1r = OP == FOP_JACOBI && a.z1r;   // z2 = P e + omega D^-1 r formed here (blk_post)

    if (threadIdx.x == 0) {
        for (int s = 0; s < NS; ++s) {
            t_mbar_init(&full[s], 1);
            cnt[s] = 0;
        }
        for (int b = 0; b < NB * TR; ++b) {
            t_mbar_init(&sfull[b], 1);
            t_mbar_init(&sempty[b], 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    const unsigned txb = TAIL ? h8t_tx_bytes_tail<OP, TR>(hasC != 0) : h8t_tx_bytes<OP, TR>(hasC != 0);
    auto issue = [&](int q) {   // plane Q = i0 - 1 + q into slot q % NS
        const int s = q % NS, Q = i0 - 1 + q;
        unsigned char* sl = ring + s * T::SLOT;
        if constexpr (OP == FOP_GPHI) {
            // phi (RHS r) and u rows in range, one 1-D box per row; E and masks as 3-D boxes
            unsigned bytes = txb;
            for (int i = 0; i < T::BR; ++i) {
                const int jj = j0 + i;
                if (Q >= 0 && Q < n0 && jj >= 0 && jj < n1) bytes += 2 * T_RB * 8;
            }
            t_mbar_expect_tx(&full[s], bytes);
            for (int i = 0; i < T::BR; ++i) {
                const int jj = j0 + i;
                if (!(Q >= 0 && Q < n0 && jj >= 0 && jj < n1)) continue;
                const long long nd = 3 * (((long long)Q * n1 + jj) * n2 + c0 - 1);
                t_tma1(sl + T::OA + i * T_VWC * 8, &tm.A, (int)((vbase + nd) & ~1LL), &full[s]);
                t_tma1(sl + T::OB + i * T_VWC * 8, &tm.B, (int)((a.goffB + nd) & ~1LL), &full[s]);
            }
            t_tma3(sl + T::OE, &tm.E, c0 - 1, j0, Q, &full[s]);
            t_tma3(sl + T::OM, &tm.M, cm0, j0, Q, &full[s]);
            return;
        }
        t_mbar_expect_tx(&full[s], txb);
        const int cv = 3 * (c0 - 1);
        t_tma4(sl + T::OA, &tm.A, cv, j0, Q, r, &full[s]);
        if (T::HB) t_tma4(sl + T::OB, &tm.B, cv, j0, Q, r, &full[s]);
        if (T::HC && hasC) {
            if (OP == FOP_CGP) t_tma4(sl + T::OC, &tm.C, cv, j0, Q, r, &full[s]);
            else t_tma3(sl + T::OC, &tm.C, cv, j0, Q, &full[s]);
        }
        t_tma3(sl + T::OE, &tm.E, c0 - 1, j0, Q, &full[s]);
        t_tma3(sl + OMK, &tm.M, cm0, j0, Q, &full[s]);
    };
    if (threadIdx.x == 0)
        for (int q = 0; q < NS && q < nq; ++q) issue(q);

    auto fA = [&](int s, int row) { return reinterpret_cast<const double*>(ring + s * T::SLOT + T::OA) + (rb + row) * VW + 3 * (gl + 1); };
    auto fB = [&](int s, int row) { return reinterpret_cast<const double*>(ring + s * T::SLOT + T::OB) + (rb + row) * VW + 3 * (gl + 1); };
    auto fC = [&](int s, int row) { return reinterpret_cast<const double*>(ring + s * T::SLOT + T::OC) + (rb + row) * VW + 3 * (gl + 1); };
    auto fE = [&](int s) { return reinterpret_cast<const double*>(ring + s * T::SLOT + T::OE)[(rb + w) * EW + gl + 1]; };
    auto fM = [&](int s, int row) { return (int)(ring + s * T::SLOT + OMK)[(rb + row) * MW + mlane]; };

    // G(u) phi: compact rows (row offset 0 / 1 double), rows outside the grid were not loaded
    const bool colok = c >= 0 && c < n2;
    auto rowok = [&](int Q, int row) {
        const int jj = j0 + row;
        return Q >= 0 && Q < n0 && jj >= 0 && jj < n1;
    };
    auto gvec = [&](int off, int s, int Q, int row, long long vb) {
        const long long nd = vb + 3 * (((long long)Q * n1 + (j0 + row)) * n2 + c0 - 1);
        return reinterpret_cast<const double*>(ring + s * T::SLOT + off) + row * T_VWC + (int)(nd & 1) + 3 * (lane + 1);
    };
    // operator input of box row `row` at slot s (plane Q): raw (unmasked) and u (masked, fed to
    // the element)
    auto input = [&](int s, int Q, int row, double (&raw)[3], double (&u)[3], int& m) {
        m = fM(s, row);
        if constexpr (OP == FOP_GPHI) {
            const bool ok = colok && rowok(Q, row);
            const double* A = gvec(T::OA, s, Q, row, vbase);
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                raw[k] = ok ? A[k] : 0.0;
                u[k] = ((m >> k) & 1) ? 0.0 : raw[k];
            }
            return;
        }
        const double* A = fA(s, row);
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            double v;
            if (OP == FOP_CGP) v = fma(beta, A[k], fB(s, row)[k]);
            else if (OP == FOP_RESTR3) v = omega * fC(s, row)[k] * fma(-alpha, fB(s, row)[k], A[k]);
            else if (OP == FOP_JACOBI && z1r) v = A[k] + __dmul_rn(__dmul_rn(omega, fC(s, row)[k]), fB(s, row)[k]);
            else v = A[k];
            raw[k] = v;
            u[k] = ((m >> k) & 1) ? 0.0 : v;
        }
    };
    // forward face (m/d along axes 1 and 2) of element (w, lane) from its two node rows
    auto face = [&](const double (&u0)[3], const double (&u1)[3], double (&F)[3][4]) {
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            const double a0 = u0[k], a1 = u1[k];
            const double a0n = __shfl_down_sync(MGK_FULL, a0, 1), a1n = __shfl_down_sync(MGK_FULL, a1, 1);
            const double em0 = a0 + a0n, ed0 = a0n - a0, em1 = a1 + a1n, ed1 = a1n - a1;
            F[k][0] = em0 + em1;
            F[k][1] = ed0 + ed1;
            F[k][2] = em1 - em0;
            F[k][3] = ed1 - ed0;
        }
    };

    double dot = 0.0;
    double CY[3][4];
#pragma unroll
    for (int k = 0; k < 3; ++k)
#pragma unroll
        for (int f = 0; f < 4; ++f) CY[k][f] = 0.0;

    // one step: element layer L between node planes L (faces FL, own raw rawL / mask mL) and
    // P = L + 1 (faces FP, rawP, mP computed here); outputs node plane L when L >= i0
    // KC = (L - (i0 - 1)) % NS when the march is unrolled by NS (slot offsets become immediates), or
    // std::integral_constant<int, -1> for a runtime slot
    auto step = [&](auto KC, int L, const double (&FL)[3][4], double (&FP)[3][4], const double (&rawL)[3], double (&rawP)[3],
                    int mL, int& mP) {
        const int P = L + 1;
        const int qP = P - (i0 - 1), qL = L - (i0 - 1);
        constexpr int KS = decltype(KC)::value;
        const int sP = KS >= 0 ? (KS + 1) % NS : qP % NS, sL = KS >= 0 ? KS : qL % NS;
        t_mbar_wait(&full[sP], (unsigned)((qP / NS) & 1));
        {
            double uo[3], uu[3], ru[3];
            int mu;
            input(sP, P, w, rawP, uo, mP);
            input(sP, P, w + 1, ru, uu, mu);
            if ((OP == FOP_CGP || OP == FOP_RESTR3) && own && P >= i0 && P < i1) {
                const long long o = vbase + (long long)P * pstr + nodeoff;
                if (OP == FOP_CGP) {
#pragma unroll
                    for (int k = 0; k < 3; ++k) a.pout[o + k] = rawP[k];
                    if (hasC) {
                        const double* A = fA(sP, w);
                        const double* C = fC(sP, w);
#pragma unroll
                        for (int k = 0; k < 3; ++k) a.xv[o + k] = fma(xal, A[k], C[k]);   // deferred x += alpha p_in
                    }
                } else {
                    const double* A = fA(sP, w);
                    const double* B = fB(sP, w);
                    const bool sd = P >= a.so0 && P < a.so1;
#pragma unroll
                    for (int k = 0; k < 3; ++k) {
                        const double rv = fma(-alpha, B[k], A[k]);
                        a.rout[o + k] = rv;
                        if (a.z1out) a.z1out[o + k] = rawP[k];
                        if (sd) dot = fma(rv, rv, dot);
                    }
                }
            }
            face(uo, uu, FP);
        }
        // element (L, w, lane): u^ = E (T u), y^ = K^ u^, back to the faces of planes L (GL) and P (CY)
        double GL[3][4];
        if constexpr (OP == FOP_GPHI) {
            // centroid stress of element (L, w, lane) from u (PAPER.md:99 G_e0[u_e], reading r15):
            // g[k][a] = 4 du_k/dx_a at the centroid, sigma = Es D0 eps
            double sig[3][3];
            if (a.sig) {   // precomputed (stress_sigma): Voigt [s00, s11, s22, s12, s02, s01], times Es
                const bool eok = L >= 0 && L < a.g.N[0] && j >= 0 && j < a.g.N[1] && c >= 0 && c < a.g.N[2];
                const double* sp = a.sig + 6 * (eok ? (((long long)L * a.g.N[1] + j) * a.g.N[2] + c) : 0);
                double v[6];
#pragma unroll
                for (int q = 0; q < 6; ++q) v[q] = eok ? __ldg(sp + q) : 0.0;
                sig[0][0] = v[0]; sig[1][1] = v[1]; sig[2][2] = v[2];
                sig[1][2] = sig[2][1] = v[3];
                sig[0][2] = sig[2][0] = v[4];
                sig[0][1] = sig[1][0] = v[5];
            } else {
            double g[3][3];
            {
                const double* uL0 = gvec(T::OB, sL, L, w, a.goffB);
                const double* uL1 = gvec(T::OB, sL, L, w + 1, a.goffB);
                const double* uP0 = gvec(T::OB, sP, P, w, a.goffB);
                const double* uP1 = gvec(T::OB, sP, P, w + 1, a.goffB);
                const bool oL0 = colok && rowok(L, w), oL1 = colok && rowok(L, w + 1);
                const bool oP0 = colok && rowok(P, w), oP1 = colok && rowok(P, w + 1);
#pragma unroll
                for (int k = 0; k < 3; ++k) {
                    const double a00 = oL0 ? uL0[k] : 0.0, a10 = oL1 ? uL1[k] : 0.0;
                    const double b00 = oP0 ? uP0[k] : 0.0, b10 = oP1 ? uP1[k] : 0.0;
                    const double a01 = __shfl_down_sync(MGK_FULL, a00, 1), a11 = __shfl_down_sync(MGK_FULL, a10, 1);
                    const double b01 = __shfl_down_sync(MGK_FULL, b00, 1), b11 = __shfl_down_sync(MGK_FULL, b10, 1);
                    const double sl0 = a00 + a01, sl1 = a10 + a11, sp0 = b00 + b01, sp1 = b10 + b11;
                    g[k][0] = (sp0 + sp1) - (sl0 + sl1);
                    g[k][1] = (sl1 - sl0) + (sp1 - sp0);
                    g[k][2] = ((a01 - a00) + (a11 - a10)) + ((b01 - b00) + (b11 - b10));
                }
            }
            const double Es4 = 0.25 * fE(sL);
            const double lam = C03 ? MG_NU_PAPER / ((1.0 + MG_NU_PAPER) * (1.0 - 2.0 * MG_NU_PAPER)) : c_Glm[0];
            const double mu = C03 ? 1.0 / (2.0 * (1.0 + MG_NU_PAPER)) : c_Glm[1];
            const double tr = lam * (g[0][0] + g[1][1] + g[2][2]);
#pragma unroll
            for (int i = 0; i < 3; ++i) sig[i][i] = Es4 * fma(2.0 * mu, g[i][i], tr);
            sig[0][1] = sig[1][0] = Es4 * mu * (g[0][1] + g[1][0]);
            sig[0][2] = sig[2][0] = Es4 * mu * (g[0][2] + g[2][0]);
            sig[1][2] = sig[2][1] = Es4 * mu * (g[1][2] + g[2][1]);
            }
            // S^ = sum_ij sigma_ij H^_ij in the (m, d) basis (H^_ij = T^-T H_ij T^-1 has the same
            // 1-D factors as the stiffness: 19 nonzeros, rows / cols s = 0 zero)
            double S[8][8];
#pragma unroll
            for (int a = 1; a < 8; ++a)
#pragma unroll
                for (int b = 1; b < 8; ++b) {
                    bool first = true;
                    double v = 0.0;
#pragma unroll
                    for (int i = 0; i < 3; ++i)
#pragma unroll
                        for (int jx = 0; jx < 3; ++jx) {
                            const double hv = tsh3(i, jx, a, b);
                            if (hv == 0.0) continue;
                            v = first ? sig[i][jx] * hv : fma(sig[i][jx], hv, v);
                            first = false;
                        }
                    S[a][b] = v;
                }
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                double uh[8], y[8];
#pragma unroll
                for (int t = 1; t < 8; ++t) {
                    const int f = t & 3;
                    uh[t] = t < 4 ? FL[k][f] + FP[k][f] : FP[k][f] - FL[k][f];
                }
#pragma unroll
                for (int a = 1; a < 8; ++a) {
                    bool first = true;
                    double v = 0.0;
#pragma unroll
                    for (int b = 1; b < 8; ++b) {
                        bool nz = false;
#pragma unroll
                        for (int i = 0; i < 3; ++i)
#pragma unroll
                            for (int jx = 0; jx < 3; ++jx) nz = nz || tsh3(i, jx, a, b) != 0.0;
                        if (!nz) continue;
                        v = first ? S[a][b] * uh[b] : fma(S[a][b], uh[b], v);
                        first = false;
                    }
                    y[a] = v;
                }
                GL[k][0] = CY[k][0] - y[4];
                CY[k][0] = y[4];
#pragma unroll
                for (int f = 1; f < 4; ++f) {
                    GL[k][f] = CY[k][f] + (y[f] - y[4 + f]);
                    CY[k][f] = y[f] + y[4 + f];
                }
            }
        } else {
            const double Ee = C03 ? fE(sL) * H8T_KSCALE : fE(sL);
#pragma unroll
            for (int ci = 0; ci < T_NCOMP; ++ci) {
                double u[3];
#pragma unroll
                for (int q = 0; q < 3; ++q) {
                    const int cc = T_COMP[ci][q];
                    if (cc < 0) continue;
                    const int sc = cc / 3, kc = cc % 3, fc = sc & 3;
                    u[q] = Ee * (sc < 4 ? FL[kc][fc] + FP[kc][fc] : FP[kc][fc] - FL[kc][fc]);
                }
#pragma unroll
                for (int q = 0; q < 3; ++q) {
                    const int rr = T_COMP[ci][q];
                    if (rr < 0) continue;
                    double acc = 0.0;
                    bool first = true;
#pragma unroll
                    for (int q2 = 0; q2 < 3; ++q2) {
                        const int cc = T_COMP[ci][q2];
                        if (cc < 0 || tkhat(MG_NU_PAPER, rr, cc) == 0.0) continue;
                        acc = first ? KT<C03>(rr, cc) * u[q2] : fma(KT<C03>(rr, cc), u[q2], acc);
                        first = false;
                    }
                    const int sr = rr / 3, kr = rr % 3, fr = sr & 3;
                    if (!t_partner_seen(ci, q)) {
                        GL[kr][fr] = sr < 4 ? CY[kr][fr] + acc : CY[kr][fr] - acc;
                        CY[kr][fr] = acc;
                    } else {
                        GL[kr][fr] = sr < 4 ? GL[kr][fr] + acc : GL[kr][fr] - acc;
                        CY[kr][fr] += acc;
                    }
                }
            }
        }
        if (L >= i0) {
            // rows: own row w gets fm - fd, row w + 1 gets fm + fd (through the exchange)
            const int o = L - i0;
            const int bi = o % NB;
            const unsigned ph = (unsigned)((o / NB) & 1);
            if (w < TR - 1) {
                if (o >= NB) t_mbar_wait(&sempty[bi * TR + w], ph ^ 1u);
                double* dst = sinv + ((bi * TR + w) * 6) * 32 + lane;
#pragma unroll
                for (int k = 0; k < 3; ++k) {
                    dst[(2 * k) * 32] = GL[k][0] + GL[k][2];
                    dst[(2 * k + 1) * 32] = GL[k][1] + GL[k][3];
                }
                __syncwarp();
                if (lane == 0) t_mbar_arrive(&sfull[bi * TR + w]);
            }
            if (w >= 1) {
                t_mbar_wait(&sfull[bi * TR + w - 1], ph);
                const double* src = sinv + ((bi * TR + w - 1) * 6) * 32 + lane;
                double y[3];
#pragma unroll
                for (int k = 0; k < 3; ++k) {
                    const double em = (GL[k][0] - GL[k][2]) + src[(2 * k) * 32];
                    const double ed = (GL[k][1] - GL[k][3]) + src[(2 * k + 1) * 32];
                    const double up = __shfl_up_sync(MGK_FULL, em + ed, 1);
                    y[k] = (em - ed) + up;
                }
                __syncwarp();
                if (lane == 0) t_mbar_arrive(&sempty[bi * TR + w - 1]);
                // H8T_RAWRE: the own row's raw input and mask of plane L re-read from its ring slot
                // (still resident: released below) instead of carried in registers across the step
                double rawR[3];
                int mR;
                if (H8T_RAWRE) {
                    double uR[3];
                    input(sL, L, w, rawR, uR, mR);
                } else {
#pragma unroll
                    for (int k = 0; k < 3; ++k) rawR[k] = rawL[k];
                    mR = mL;
                }
                if (OP == FOP_GPHI && own && L < i1) {   // F G F phi: fixed rows zero
                    const long long ob = (long long)r * a.g.vstr + 3 * (((long long)L * n1 + j) * n2 + c);
#pragma unroll
                    for (int k = 0; k < 3; ++k) a.y[ob + k] = ((mR >> k) & 1) ? 0.0 : y[k];
                } else if (own && L < i1) {
                    const long long ob = vbase + (long long)L * pstr + nodeoff;
                    const bool sdot = L >= a.so0 && L < a.so1;
#pragma unroll
                    for (int k = 0; k < 3; ++k) {
                        const double ax = ((mR >> k) & 1) ? rawR[k] : y[k];
                        double out;
                        if (OP == FOP_MATVEC || OP == FOP_CGP) {
                            out = ax;
                            if (OP == FOP_CGP && sdot) dot = fma(rawR[k], ax, dot);
                        } else if (OP == FOP_RESID) {
                            out = fB(sL, w)[k] - ax;
                        } else if (OP == FOP_RESTR3) {
                            out = fma(-alpha, fB(sL, w)[k], fA(sL, w)[k]) - ax;
                        } else {   // JACOBI
                            const double bk = fB(sL, w)[k];
                            out = fma(omega * fC(sL, w)[k], bk - ax, rawR[k]);
                            if (sdot) dot = fma(bk, out, dot);
                        }
                        a.y[ob + k] = out;
                    }
                }
            }
        }
        // release plane L's slot; the last warp refills it with plane L + NS
        __syncwarp();
        if (lane == 0) {
            __threadfence_block();
            if (atomicAdd(&cnt[sL], 1) == TR - 1) {
                cnt[sL] = 0;
                if (qL + NS < nq) issue(qL + NS);
            }
        }
    };

    double FA[3][4], FB[3][4], rawA[3], rawB[3];
    int mA = 7, mB = 7;
    {   // prologue: plane i0 - 1 (q = 0)
        t_mbar_wait(&full[0], 0u);
        double uo[3], uu[3], ru[3];
        int mu;
        input(0, i0 - 1, w, rawA, uo, mA);
        input(0, i0 - 1, w + 1, ru, uu, mu);
        face(uo, uu, FA);
    }
    using I0 = std::integral_constant<int, 0>;
    using I1 = std::integral_constant<int, 1>;
    using I2 = std::integral_constant<int, 2>;
    using I3 = std::integral_constant<int, 3>;
    using IR = std::integral_constant<int, -1>;
    if constexpr (NS == 4 && false) {   // unrolled by the ring depth (every slot offset a constant): spills, not used
        for (int L = i0 - 1; L < i1; L += 4) {
            step(I0{}, L, FA, FB, rawA, rawB, mA, mB);
            if (L + 1 < i1) step(I1{}, L + 1, FB, FA, rawB, rawA, mB, mA);
            if (L + 2 < i1) step(I2{}, L + 2, FA, FB, rawA, rawB, mA, mB);
            if (L + 3 < i1) step(I3{}, L + 3, FB, FA, rawB, rawA, mB, mA);
        }
    } else {
        for (int L = i0 - 1; L < i1; L += 2) {
            step(IR{}, L, FA, FB, rawA, rawB, mA, mB);
            if (L + 1 < i1) step(IR{}, L + 1, FB, FA, rawB, rawA, mB, mA);
        }
    }
    if (a.partial) {
        dot = warp_sum(dot);
        if (lane == 0) s_dot[w] = dot;
        __syncthreads();
        if (threadIdx.x == 0) {
            double t = 0.0;
#pragma unroll
            for (int q = 0; q < TR; ++q) t += s_dot[q];
            a.partial[(long long)r * a.pstride + toff + tile] = t;
        }
    }
}

// ---------------------------------------------------------------- host: tensor maps and launch
static PFN_cuTensorMapEncodeTiled_v12000 t_encode() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            p = nullptr;
        return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }();
    return fn;
}

static bool t_map(CUtensorMap* m, CUtensorMapDataType dt, int rank, const void* base, const cuuint64_t* dims,
                  const cuuint64_t* strides, const cuuint32_t* box) {
    auto enc = t_encode();
    if (!enc) return false;
    cuuint32_t es[5] = {1, 1, 1, 1, 1};
    CUresult e = enc(m, dt, (cuuint32_t)rank, const_cast<void*>(base), dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (e != CUDA_SUCCESS) {
        fprintf(stderr, "h8t: cuTensorMapEncodeTiled failed (%d): rank %d dim0 %llu box0 %u base %p\n", (int)e, rank,
                (unsigned long long)dims[0], box[0], base);
        return false;
    }
    return true;
}

// vectors (R, n0, n1, p2, 3) as a 4-D tensor {3 n2, n1, n0, R} (row pitch 3 p2)
static bool t_map_vec(CUtensorMap* m, const FineArgs& a, const double* v, int BR, bool perR, int VW = T_VW) {
    const LevelGeom& g = a.g;
    cuuint64_t dims[4] = {(cuuint64_t)3 * g.nn[2], (cuuint64_t)g.nn[1], (cuuint64_t)g.nn[0], (cuuint64_t)std::max(a.R, 1)};
    cuuint64_t str[3] = {(cuuint64_t)3 * g.p2 * 8, (cuuint64_t)3 * g.p2 * g.nn[1] * 8, (cuuint64_t)g.vstr * 8};
    cuuint32_t box[4] = {(cuuint32_t)VW, (cuuint32_t)BR, 1, 1};
    return t_map(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, perR ? 4 : 3, v, dims, str, box);
}

// MG_H8T_TAIL=0: the last column tile as an ordinary tile even when it owns <= 9 node columns
static bool h8t_tail_enabled() {
    static bool v = [] {
        const char* e = getenv("MG_H8T_TAIL");
        return e ? atoi(e) != 0 : true;
    }();
    return v;
}

// Tiling of one launch: ntc x ntr ordinary tiles per chunk (nch chunks of hch planes), plus, in tail
// mode, ntr3 stacked-row tiles of the last column (nch3 chunks of hch3 planes) in a second launch
// whose dot partials follow the first launch's.
struct H8TPlan {
    bool tail = false;
    int ntc = 0, ntr = 0, nch = 1, hch = 0;
    int ntr3 = 0, nch3 = 1, hch3 = 0;
    int items() const { return ntc * ntr * nch + (tail ? ntr3 * nch3 : 0); }
};

static H8TPlan h8t_plan(int TR, int minb, const LevelGeom& g, int R, bool allow_tail) {
    H8TPlan p;
    const int ntc_all = (g.nn[2] + 29) / 30;
    p.tail = allow_tail && TR == 8 && h8t_tail_enabled() && ntc_all >= 2 &&
             g.nn[2] - 1 - (30 * (ntc_all - 1) - 1) <= TT_G - 1;
    p.ntc = p.tail ? ntc_all - 1 : ntc_all;
    p.ntr = (g.nn[1] + TR - 2) / (TR - 1);
    h8t_chunks(TR, minb, p.ntc * p.ntr, g, R, &p.nch, &p.hch);
    if (p.tail) {
        p.ntr3 = (g.nn[1] + 3 * (TR - 1) - 1) / (3 * (TR - 1));
        h8t_chunks(TR, minb, p.ntr3, g, R, &p.nch3, &p.hch3);
    }
    return p;
}

template <int OP, int TR, int NS, int NB, int MINB, bool TAIL>
static bool launch_h8t_part(const FineArgs& a, cudaStream_t s, int ntc, int ntr, int nch, int hch, int tc0, int toff) {
    using T = TL<OP, TR, NB>;
    using U = TLT<TR>;
    const LevelGeom& g = a.g;
    H8TMaps tm;
    memset(&tm, 0, sizeof(tm));
    const double* vA = OP == FOP_CGP ? a.pin : (OP == FOP_RESTR3 ? a.rin : a.x);
    const double* vB = OP == FOP_CGP ? a.z : (OP == FOP_RESTR3 ? a.q : a.b);
    const bool hasC = T::HC && (OP != FOP_CGP || a.xv != nullptr);
    bool ok;
    if (OP == FOP_GPHI) {   // phi (R, ndof) and u (ndof) as 1-D tensors, one box per row
        cuuint64_t dA[1] = {(cuuint64_t)g.ndof * a.R + a.goffA}, dB[1] = {(cuuint64_t)g.ndof + a.goffB};
        cuuint32_t box[1] = {(cuuint32_t)T_RB};
        cuuint64_t nostr[1] = {0};   // rank 1: no strides (the array must still be valid)
        ok = t_map(&tm.A, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 1, vA - a.goffA, dA, nostr, box) &&
             t_map(&tm.B, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 1, vB - a.goffB, dB, nostr, box);
    } else {
        const int BR = TAIL ? U::BR : T::BR, VW = TAIL ? TT_VW : T_VW;
        ok = t_map_vec(&tm.A, a, vA, BR, true, VW);
        if (T::HB) ok = ok && t_map_vec(&tm.B, a, vB, BR, true, VW);
        if (hasC) ok = ok && t_map_vec(&tm.C, a, OP == FOP_CGP ? a.xv : a.Dinv, BR, OP == FOP_CGP, VW);
    }
    {
        cuuint64_t dims[3] = {(cuuint64_t)g.N[2], (cuuint64_t)g.N[1], (cuuint64_t)g.N[0]};
        cuuint64_t str[2] = {(cuuint64_t)a.ep2 * 8, (cuuint64_t)a.ep2 * g.N[1] * 8};
        cuuint32_t box[3] = {(cuuint32_t)(TAIL ? TT_EW : T_EW), (cuuint32_t)(TAIL ? U::ER : TR), 1};
        ok = ok && t_map(&tm.E, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, a.E, dims, str, box);
    }
    {
        cuuint64_t dims[3] = {(cuuint64_t)g.nn[2], (cuuint64_t)g.nn[1], (cuuint64_t)g.nn[0]};
        cuuint64_t str[2] = {(cuuint64_t)a.m2, (cuuint64_t)a.m2 * g.nn[1]};
        cuuint32_t box[3] = {(cuuint32_t)(TAIL ? TT_MW : T_MW), (cuuint32_t)(TAIL ? U::BR : T::BR), 1};
        ok = ok && t_map(&tm.M, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, a.mask, dims, str, box);
    }
    if (!ok) return false;
    const size_t smem = h8t_smem_bytes<OP, TR, NS, NB>();
    auto k03 = h8t_kernel<OP, true, TR, NS, NB, MINB, TAIL>;
    auto kgn = h8t_kernel<OP, false, TR, NS, NB, MINB, TAIL>;
    static bool attr = [&] {
        cudaFuncSetAttribute(k03, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaFuncSetAttribute(kgn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        return true;
    }();
    (void)attr;
    const unsigned nb = (unsigned)((long long)ntc * ntr * nch * a.R);
    if (a.nu_paper)
        launch_kp(false, k03, dim3(nb), dim3(32 * TR), smem, s, a, tm, ntc, ntr, nch, hch, hasC ? 1 : 0, tc0, toff);
    else
        launch_kp(false, kgn, dim3(nb), dim3(32 * TR), smem, s, a, tm, ntc, ntr, nch, hch, hasC ? 1 : 0, tc0, toff);
    return true;
}

// MG_H8T_TAIL_FORK=0: the tail launch follows the main launch on the same stream; default: it is
// forked onto a side stream right after the main launch (joined before the next operation), so its
// CTAs fill the slots the main grid's last wave leaves free instead of running as a wave of its own.
// Process-wide side stream and events: every C-ABI call holds the API lock, and inside a graph
// capture the event wait pulls the side stream into the capture (a fork / join of kernel nodes).
static bool h8t_tail_fork(cudaStream_t* side, cudaEvent_t* ev) {
    static const bool on = [] {
        const char* e = getenv("MG_H8T_TAIL_FORK");
        return e ? atoi(e) != 0 : true;
    }();
    static cudaStream_t ss = nullptr;
    static cudaEvent_t ee[2] = {nullptr, nullptr};
    if (!on) return false;
    if (!ss) {
        if (cudaStreamCreateWithFlags(&ss, cudaStreamNonBlocking) != cudaSuccess ||
            cudaEventCreateWithFlags(&ee[0], cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&ee[1], cudaEventDisableTiming) != cudaSuccess) {
            ss = nullptr;
            return false;
        }
    }
    *side = ss;
    ev[0] = ee[0];
    ev[1] = ee[1];
    return true;
}

template <int OP, int TR, int NS, int NB, int MINB>
static bool launch_h8t_t(const FineArgs& a, cudaStream_t s) {
    constexpr bool TAILOK = h8t_tail_fits<OP, TR, NB>();
    const H8TPlan p = h8t_plan(TR, MINB, a.g, a.R, TAILOK);
    cudaStream_t side = nullptr;
    cudaEvent_t ev[2];
    const bool fork = p.tail && h8t_tail_fork(&side, ev);
    if (fork) cudaEventRecord(ev[0], s);
    if (!launch_h8t_part<OP, TR, NS, NB, MINB, false>(a, s, p.ntc, p.ntr, p.nch, p.hch, 0, 0)) return false;
    if constexpr (TAILOK) {
        if (p.tail) {
            cudaStream_t st = s;
            if (fork) {
                cudaStreamWaitEvent(side, ev[0], 0);
                st = side;
            }
            const bool ok = launch_h8t_part<OP, TR, NS, NB, MINB, true>(a, st, 1, p.ntr3, p.nch3, p.hch3, p.ntc,
                                                                        p.ntc * p.ntr * p.nch);
            if (fork) {
                cudaEventRecord(ev[1], side);
                cudaStreamWaitEvent(s, ev[1], 0);
            }
            return ok;
        }
    }
    return true;
}

// warps per CTA: MG_H8T_TR = 8 (2 CTAs / SM, default: B200 C5 A/B 147.8 vs 151.5 ms/step) or 16
// (1 CTA / SM: less tile overlap, but a whole SM waits on one CTA's slowest warp)
static int h8t_tr() {
    static int tr = [] {
        const char* e = getenv("MG_H8T_TR");
        const int v = e ? atoi(e) : 8;
        return v == 16 ? 16 : 8;
    }();
    return tr;
}
// ring depth / exchange buffers: MG_H8T_RING = 0 (default: per op, the deepest ring of 3..8 plane
// slots that keeps two 8-warp CTAs per SM, single row-exchange buffer -- B200 C5 A/B: CGP 1.04 -> 0.91
// ms with 4 slots instead of 3), 3 (3 slots, double exchange buffer) or 4 (4 slots, single buffer)
static int h8t_ring() {
    static int v = [] {
        const char* e = getenv("MG_H8T_RING");
        const int r = e ? atoi(e) : 0;
        return (r == 3 || r == 4) ? r : 0;
    }();
    return v;
}
template <int OP, int TR, int NB, int MINB>
constexpr int h8t_auto_ns() {
    constexpr size_t budget = (size_t)(MINB == 2 ? 112 : 224) * 1024;
    int ns = 3;
    if (h8t_smem_bytes<OP, TR, 4, NB>() <= budget) ns = 4;
    if (h8t_smem_bytes<OP, TR, 5, NB>() <= budget) ns = 5;
    if (h8t_smem_bytes<OP, TR, 6, NB>() <= budget) ns = 6;
    return ns;
}

// chunking along axis 0: between 16 and 64 planes per chunk, picked so that the CTA count fills
// the resident slots (148 SMs x CTAs per SM) with the smallest tail wave
void h8t_chunks(int TR, int minb, int tiles, const LevelGeom& g, int R, int* nch_out, int* hch_out) {
    (void)TR;
    const long long slots = 148LL * minb;
    const int n0 = g.nn[0];
    int best = 1;
    double best_eff = -1.0;
    for (int nch = 1; nch <= std::max(1, n0 / 8); ++nch) {
        const int hch = (n0 + nch - 1) / nch;
        const int nc = (n0 + hch - 1) / hch;
        const long long ctas = (long long)tiles * nc * R;
        const double waves = (double)ctas / slots;
        const double fill = waves / std::ceil(waves);
        const double eff = fill * hch / (hch + 1.0);   // + one prologue plane per chunk
        if (eff > best_eff + 1e-9) { best_eff = eff; best = nc; }
    }
    *nch_out = best;
    *hch_out = (n0 + best - 1) / best;
}

// dot-partial items per RHS (sizing): the larger of the plans with and without the tail launch
int h8t_items(const LevelGeom& g, int R) {
    const int TR = h8t_tr(), minb = TR == 8 ? 2 : 1;
    return std::max(h8t_plan(TR, minb, g, R, true).items(), h8t_plan(TR, minb, g, R, false).items());
}

template <int OP>
static bool launch_h8t_op(const FineArgs& a, cudaStream_t s) {
    if (h8t_tr() == 8) {
        // G(u) phi keeps 3 slots + double exchange buffer: its deeper-ring builds spill (C5 1.69 -> 2.03 ms)
        if (h8t_ring() == 3 || OP == FOP_GPHI) return launch_h8t_t<OP, 8, 3, 2, 2>(a, s);
        if (h8t_ring() == 4) return launch_h8t_t<OP, 8, 4, 1, 2>(a, s);
        return launch_h8t_t<OP, 8, h8t_auto_ns<OP, 8, 1, 2>(), 1, 2>(a, s);
    }
    return h8t_ring() == 3 ? launch_h8t_t<OP, 16, 3, 2, 1>(a, s) : launch_h8t_t<OP, 16, 4, 1, 1>(a, s);
}

int h8t_apply(int op, const FineArgs& a, cudaStream_t s) {
    const int TR = h8t_tr();
    bool ok;
    switch (op) {
        case FOP_GPHI: ok = launch_h8t_op<FOP_GPHI>(a, s); break;
        case FOP_MATVEC: ok = launch_h8t_op<FOP_MATVEC>(a, s); break;
        case FOP_RESID: ok = launch_h8t_op<FOP_RESID>(a, s); break;
        case FOP_JACOBI: ok = launch_h8t_op<FOP_JACOBI>(a, s); break;
        case FOP_RESTR3: ok = launch_h8t_op<FOP_RESTR3>(a, s); break;
        default: ok = launch_h8t_op<FOP_CGP>(a, s); break;
    }
    return ok ? h8t_plan(TR, TR == 8 ? 2 : 1, a.g, a.R, op != FOP_GPHI).items() : -1;
}

// ---------------------------------------------------------------- padded 3D fine layout
Pad3 pad3_layout(const LevelGeom& g) {
    Pad3 p{};
    p.p2 = g.nn[2] + (g.nn[2] & 1);
    p.m2 = (g.nn[2] + 15) / 16 * 16;
    p.ep2 = g.N[2] + (g.N[2] & 1);
    p.vstride = 3LL * g.nn[0] * g.nn[1] * p.p2;
    return p;
}

LevelGeom pad3_geom(const LevelGeom& g, const Pad3& p) {
    LevelGeom q = g;
    q.p2 = p.p2;
    q.vstr = p.vstride;
    return q;
}

// compact (R, planes, n1, n2, 3) -> padded; src planes [0, np) map to local planes [p0, p0 + np)
__global__ void pad3_vec_kernel(LevelGeom g, Pad3 p, int R, const uint8_t* mask, int p0, int np, const double* src,
                                long long src_ndof, double* dst) {
    const long long per = (long long)np * g.nn[1] * g.nn[2];
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= per) return;
    const int r = blockIdx.y;
    const int c = (int)(i % g.nn[2]);
    const long long t = i / g.nn[2];
    const int j = (int)(t % g.nn[1]);
    const int P = (int)(t / g.nn[1]) + p0;
    const long long cn = ((long long)P * g.nn[1] + j) * g.nn[2] + c;   // compact local node
    const int m = mask ? mask[cn] : 0;
    const double* s = src + (long long)r * src_ndof + 3 * i;
    double* d = dst + (long long)r * p.vstride + 3 * (((long long)P * g.nn[1] + j) * p.p2 + c);
#pragma unroll
    for (int k = 0; k < 3; ++k) d[k] = ((m >> k) & 1) ? 0.0 : s[k];
}

__global__ void unpad3_vec_kernel(LevelGeom g, Pad3 p, int R, int p0, int np, const double* src, double* dst,
                                  long long dst_ndof) {
    const long long per = (long long)np * g.nn[1] * g.nn[2];
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= per) return;
    const int r = blockIdx.y;
    const int c = (int)(i % g.nn[2]);
    const long long t = i / g.nn[2];
    const int j = (int)(t % g.nn[1]);
    const int P = (int)(t / g.nn[1]) + p0;
    const double* s = src + (long long)r * p.vstride + 3 * (((long long)P * g.nn[1] + j) * p.p2 + c);
    double* d = dst + (long long)r * dst_ndof + 3 * i;
#pragma unroll
    for (int k = 0; k < 3; ++k) d[k] = s[k];
}

void pad3_vectors_planes(const LevelGeom& g, const Pad3& p, int R, const uint8_t* mask, int p0, int np,
                         const double* src, long long src_ndof, double* dst, cudaStream_t s) {
    const long long per = (long long)np * g.nn[1] * g.nn[2];
    if (per <= 0) return;
    pad3_vec_kernel<<<dim3((unsigned)((per + 255) / 256), R), 256, 0, s>>>(g, p, R, mask, p0, np, src, src_ndof, dst);
}

void unpad3_vectors_planes(const LevelGeom& g, const Pad3& p, int R, int p0, int np, const double* src, double* dst,
                           long long dst_ndof, cudaStream_t s) {
    const long long per = (long long)np * g.nn[1] * g.nn[2];
    if (per <= 0) return;
    unpad3_vec_kernel<<<dim3((unsigned)((per + 255) / 256), R), 256, 0, s>>>(g, p, R, p0, np, src, dst, dst_ndof);
}

// node arrays: masks (1 byte) -> pitch m2, D^-1 (3 doubles) -> pitch p2; E (N2) -> pitch ep2
__global__ void pad3_nodes_kernel(LevelGeom g, Pad3 p, const uint8_t* mask, uint8_t* maskp, const double* dinv,
                                  double* dinvp) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= g.nnodes) return;
    const int c = (int)(i % g.nn[2]);
    const long long row = i / g.nn[2];
    maskp[row * p.m2 + c] = mask[i];
#pragma unroll
    for (int k = 0; k < 3; ++k) dinvp[3 * (row * p.p2 + c) + k] = dinv[3 * i + k];
}
__global__ void pad3_elems_kernel(LevelGeom g, Pad3 p, const double* E, double* Ep) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= g.nelem) return;
    const int c = (int)(i % g.N[2]);
    const long long row = i / g.N[2];
    Ep[row * p.ep2 + c] = E[i];
}

void pad3_nodes(const LevelGeom& g, const Pad3& p, const uint8_t* mask, uint8_t* maskp, const double* dinv,
                double* dinvp, cudaStream_t s) {
    pad3_nodes_kernel<<<(unsigned)((g.nnodes + 255) / 256), 256, 0, s>>>(g, p, mask, maskp, dinv, dinvp);
}
void pad3_elems(const LevelGeom& g, const Pad3& p, const double* E, double* Ep, cudaStream_t s) {
    pad3_elems_kernel<<<(unsigned)((g.nelem + 255) / 256), 256, 0, s>>>(g, p, E, Ep);
}
