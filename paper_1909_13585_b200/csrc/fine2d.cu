// 2D (Q4) fine level: matrix-free element-by-element K
// fused with its producers/consumers in the CG iteration and the V(1,1) cycle:
//
//   M2_CGP       p = z + beta p_in ; q = K p ; dot(p,q) ; x += alpha_prev p_in   (a7 + a2)
//   M2_RESTRICT  r = r_in - alpha q ; dot(r,r) ; z1 = omega D^-1 r ;
//                t = r - K z1 ; r_c = P^T t                                      (a7 + a3 + a2 + a4)
//   M2_POST      z2 = omega D^-1 r + P e_c ; z = z2 + omega D^-1 (r - K z2) ; dot(r,z)  (a4 + a3 + a2)
//   M2_MATVEC / M2_RESID / M2_JACOBI   plain y = K x, y = b - K x, damped-Jacobi sweep.
//
// so one CG iteration reads/writes 11 fine R-vectors instead of 20.
// Fixed DOFs: K's rows/cols are identity (reading r11); D = diag(K) is formed on the
// fly from the 4 adjacent E_e (all diagonal entries of the isotropic K0 are equal).
//
// Work decomposition (B200): a warp owns a strip of node columns along axis 1 (30,
// or 28 for the restriction so every coarse node is complete inside one warp), lanes
// = columns, and marches along axis 0 over a chunk of node planes.  Plane data
// (vectors, E_e, masks, coarse rows) is staged by TMA bulk copies (cp.async.bulk,
// issued by lane 0) into a per-warp NS-stage shared-memory ring guarded by
// mbarriers, so each warp keeps NS planes in flight without spending registers.
// Each step exchanges column neighbours by warp shuffles, adds the contribution of
// one element layer to the two node planes it touches, and finishes the lower plane.  No atomics, no colouring: deterministic.  The RHS
// index is the fastest grid coordinate so the R warps of a tile share E_e in L2.
// K0 entries for nu = 0.3 are compile-time constants (element.cuh).
#include "element.cuh"
#include "kernels.h"

__constant__ double c_K2[64];

void fine2d_set_constants(const double* K0, cudaStream_t s) {
    cudaMemcpyToSymbolAsync(c_K2, K0, sizeof(double) * 64, 0, cudaMemcpyHostToDevice, s);
}

template <bool C03>
__device__ __forceinline__ double K2(int r, int c) {
    if (C03) return k0_entry<2>(MG_NU_PAPER, r, c);
    return c_K2[r * 8 + c];
}

static constexpr int NS = 4;      // smem pipeline stages per warp (node planes in flight)
static constexpr int CH = 64;     // node planes per chunk
static constexpr int CCH = 32;    // coarse rows per chunk (M2_RESTRICT)
static constexpr int WPB = 2;     // warps per CTA (independent; no CTA-wide sync)

__device__ __forceinline__ double2 ld2(const double* p) { return *reinterpret_cast<const double2*>(p); }
__device__ __forceinline__ void st2(double* p, double a, double b) { *reinterpret_cast<double2*>(p) = make_double2(a, b); }

// ---------------------------------------------------------------- TMA bulk-copy / mbarrier helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, int count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
    asm volatile(
        "{\n .reg .pred p;\n"
        "WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
        "r"(phase)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// Stage layout (bytes) for RB right-hand sides: NV vectors x RB RHS x 32 nodes x 16 B, then
// E (elements c_first-1 .. c_first+31 from a 16-B aligned start), the node masks, and for
// POST the coarse correction rows (RB x 17 nodes) + coarse mask, for RESTRICT the coarse mask.
template <int OP, int RB>
struct Stage {
    static constexpr int NV = OP == M2_CGP ? 3 : ((OP == M2_MATVEC || OP == M2_POST) ? 1 : 2);
    static constexpr bool HAS_C = OP == M2_POST;
    static constexpr bool HAS_CM = OP == M2_POST || OP == M2_RESTRICT;
    static constexpr int EOFF = NV * RB * 512;
    static constexpr int MOFF = EOFF + 288;
    static constexpr int COFF = MOFF + 48;
    static constexpr int CMOFF = COFF + (HAS_C ? RB * 288 : 0);
    static constexpr int BYTES = CMOFF + (HAS_CM ? 48 : 0);
    static constexpr int NCOPY = NV * RB + 2 + (HAS_C ? RB : 0) + (HAS_CM ? 1 : 0);
};

struct WarpGeom {
    int c_first;        // node column of lane 0
    int vlo, vhi;       // copied node columns [vlo, vhi)
    int clo, chi;       // copied element columns [clo, chi)
    int jbase, jl, jh;  // coarse node columns: smem origin c_first>>1, copied [jl, jh]
};

template <int OP>
__device__ __forceinline__ int coarse_row(const March2Args& a, int P) {
    int crow = -1;
    if (OP == M2_POST) crow = (P & 1) ? (P + 1) >> 1 : -1;
    if (OP == M2_RESTRICT) crow = P >= 1 ? (P - 1) >> 1 : -1;
    return (crow >= 0 && crow < a.gc.nn[0]) ? crow : -1;
}

// Issue the bulk copies of plane P into a stage: lane 0 registers the byte count on the
// stage's mbarrier, then lane t issues copy t (vectors of RHS q, E, masks, coarse rows).
template <int OP, int RB>
__device__ __forceinline__ void issue_plane(const March2Args& a, const WarpGeom& wg, char* st, uint64_t* bar, int P,
                                            long long r0, int nr, unsigned actmask, int lane) {
    using S = Stage<OP, RB>;
    const int n0 = a.g.nn[0], n1 = a.g.nn[1], N0 = a.g.N[0], N1 = a.g.N[1];
    uint32_t vbytes = 0, ebytes = 0, mbytes = 0, cbytes = 0, cmbytes = 0;
    int e_al = 0, m_al = 0, cm_al = 0;
    const int crow = coarse_row<OP>(a, P);
    if (P >= 0 && P < n0 && wg.vlo < wg.vhi) {
        vbytes = 16u * (wg.vhi - wg.vlo);
        m_al = (P * n1 + wg.vlo) & ~15;
        mbytes = (uint32_t)(((P * n1 + wg.vhi + 15) & ~15) - m_al);
    }
    if (P >= 0 && P < N0 && wg.clo < wg.chi) {
        e_al = (8 * (P * N1 + wg.clo)) & ~15;
        ebytes = (uint32_t)(((8 * (P * N1 + wg.chi) + 15) & ~15) - e_al);
    }
    if (S::HAS_CM && crow >= 0 && wg.jl <= wg.jh) {
        const int nc1 = a.gc.nn[1];
        if (S::HAS_C) cbytes = 16u * (wg.jh - wg.jl + 1);
        cm_al = (crow * nc1 + wg.jl) & ~15;
        cmbytes = (uint32_t)(((crow * nc1 + wg.jh + 1 + 15) & ~15) - cm_al);
    }
    const int nact = __popc(actmask);
    if (lane == 0) mbar_expect_tx(bar, S::NV * nact * vbytes + ebytes + mbytes + nact * cbytes + cmbytes);
    __syncwarp();
    const int t = lane;
    if (t < S::NV * RB) {
        const int v = t / RB, q = t % RB;
        if (q < nr && ((actmask >> q) & 1) && vbytes) {
            const double* base = v == 0 ? a.x : (v == 1 ? a.x2 : a.xv);
            const long long off = (r0 + q) * a.g.ndof + 2LL * (P * n1 + wg.vlo);
            bulk_g2s(st + (v * RB + q) * 512 + 16 * (wg.vlo - wg.c_first), base + off, vbytes, bar);
        }
    } else if (t == S::NV * RB) {
        if (ebytes) bulk_g2s(st + S::EOFF, reinterpret_cast<const char*>(a.E) + e_al, ebytes, bar);
    } else if (t == S::NV * RB + 1) {
        if (mbytes) bulk_g2s(st + S::MOFF, a.mask + m_al, mbytes, bar);
    } else if (S::HAS_C && t < S::NV * RB + 2 + RB) {
        const int q = t - (S::NV * RB + 2);
        if (q < nr && ((actmask >> q) & 1) && cbytes) {
            const long long off = (r0 + q) * a.gc.ndof + 2LL * (crow * a.gc.nn[1] + wg.jl);
            bulk_g2s(st + S::COFF + q * 288 + 16 * (wg.jl - wg.jbase), a.ec + off, cbytes, bar);
        }
    } else if (S::HAS_CM && t == S::NCOPY - 1) {
        if (cmbytes) bulk_g2s(st + S::CMOFF, a.maskc + cm_al, cmbytes, bar);
    }
}

struct LaneGeom {
    int c, lane;
    bool cin, own_col, ce, cel;
    int eoff_c;   // 8 (c - clo)
    int vo;       // 16 lane
};

// Per-RHS registers carried between planes.
template <int RB>
struct RhsState {
    double w[RB][6];     // masked matvec input of the current plane at columns c-1, c, c+1 (x, y)
    double u[RB][2];     // unmasked own input
    double k[RB][2];     // b (RESID/JACOBI), p_in (CGP), r (RESTRICT/POST)
    double k2[RB][2];    // x (CGP)
    double car[RB][2];   // contribution of the element layer below to the next plane
    double dot[RB];
    double acc[RB][2];   // RESTRICT: running coarse sums
    double cev[RB][4];   // POST: coarse correction of the last even plane (J0 x,y, J1 x,y)
};

template <int OP, bool C03, int RB>
__global__ void __launch_bounds__(32 * WPB) march2_kernel(March2Args a, int nct, int nch, int nrc) {
    using S = Stage<OP, RB>;
    constexpr int CS = (OP == M2_RESTRICT) ? 28 : 30;
    constexpr int LOFF = (OP == M2_RESTRICT) ? 2 : 1;
    extern __shared__ __align__(128) char smem_raw[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    char* wsm = smem_raw + wid * (NS * S::BYTES + NS * 8);
    uint64_t* bars = reinterpret_cast<uint64_t*>(wsm + NS * S::BYTES);
    const long long w = (long long)blockIdx.x * WPB + wid;
    const int items = nct * nch;
    if (w >= (long long)nrc * items) return;
    if (a.done && *a.done) return;
    const int rc = (int)(w % nrc);
    const int item = (int)(w / nrc);
    const int r0 = (rc * a.R) / nrc, r1 = ((rc + 1) * a.R) / nrc, nr = r1 - r0;
    unsigned actmask = 0;
#pragma unroll
    for (int q = 0; q < RB; ++q)
        if (q < nr && (!a.active || a.active[r0 + q])) actmask |= 1u << q;
    if (!actmask) return;
    const int ct = item % nct, ch = item / nct;
    const int n0 = a.g.nn[0], n1 = a.g.nn[1], N0 = a.g.N[0], N1 = a.g.N[1];
    WarpGeom wg;
    wg.c_first = ct * CS - LOFF;
    wg.vlo = max(wg.c_first, 0);
    wg.vhi = min(wg.c_first + 32, n1);
    wg.clo = max(wg.c_first - 1, 0);
    wg.chi = min(wg.c_first + 32, N1);
    wg.jbase = wg.c_first >> 1;
    wg.jl = max(wg.c_first >> 1, 0);
    wg.jh = (OP == M2_POST || OP == M2_RESTRICT) ? min((wg.c_first + 32) >> 1, a.gc.nn[1] - 1) : 0;
    LaneGeom lg;
    lg.lane = lane;
    lg.c = wg.c_first + lane;
    lg.cin = lg.c >= 0 && lg.c < n1;
    lg.own_col = lg.cin && lane >= LOFF && lane < LOFF + CS;
    lg.ce = lg.cin && lg.c < N1;
    lg.cel = lg.cin && lg.c >= 1 && lg.c - 1 < N1;
    lg.eoff_c = 8 * (lg.c - wg.clo);
    lg.vo = 16 * lane;
    const int c = lg.c;
    int i0, i1, own0, own1, I0 = 0, I1 = 0;
    if (OP == M2_RESTRICT) {
        const int nc0 = a.gc.nn[0];
        I0 = ch * CCH;
        I1 = min(I0 + CCH, nc0);
        i0 = max(0, 2 * I0 - 1);
        i1 = min(2 * I1, n0);
        own0 = 2 * I0;
        own1 = i1;
    } else {
        i0 = ch * CH;
        i1 = min(i0 + CH, n0);
        own0 = i0;
        own1 = i1;
    }
    const double omega = a.omega;
    const double k0d = K2<C03>(0, 0);
    const int nplanes = i1 - i0 + 2;     // planes i0-1 .. i1
    double coef[RB];                     // beta (CGP) / alpha (RESTRICT) per RHS
    double xal[RB];                      // xalpha (CGP)
#pragma unroll
    for (int q = 0; q < RB; ++q) {
        const int rr = min(r0 + q, a.R - 1);
        coef[q] = OP == M2_CGP ? a.beta[rr] : (OP == M2_RESTRICT ? a.alpha[rr] : 0.0);
        xal[q] = OP == M2_CGP ? a.xalpha[rr] : 0.0;
    }

    if (lane == 0) {
        for (int s = 0; s < NS; ++s) mbar_init(&bars[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        fence_proxy_async();
    }
    __syncwarp();
    for (int k = 0; k < NS && k < nplanes; ++k)
        issue_plane<OP, RB>(a, wg, wsm + k * S::BYTES, &bars[k], i0 - 1 + k, r0, nr, actmask, lane);

    RhsState<RB> rs;
#pragma unroll
    for (int q = 0; q < RB; ++q) {
#pragma unroll
        for (int j = 0; j < 6; ++j) rs.w[q][j] = 0.0;
        rs.u[q][0] = rs.u[q][1] = rs.k[q][0] = rs.k[q][1] = rs.k2[q][0] = rs.k2[q][1] = 0.0;
        rs.car[q][0] = rs.car[q][1] = 0.0;
        rs.dot[q] = 0.0;
        rs.acc[q][0] = rs.acc[q][1] = 0.0;
#pragma unroll
        for (int j = 0; j < 4; ++j) rs.cev[q][j] = 0.0;
    }
    // plane-shared state of the current plane
    int mA = 3;
    double DA = 1.0, eA = 0.0, elA = 0.0;
    {   // E of layer i0-2 (diagonal of the first plane): direct loads, once per chunk
        const int Lp = i0 - 2;
        if (Lp >= 0 && Lp < N0) {
            if (lg.ce) eA = a.E[Lp * N1 + c];
            if (lg.cel) elA = a.E[Lp * N1 + c - 1];
        }
    }
    if (OP == M2_POST) {   // coarse row floor(P0/2) of the first plane, per RHS (direct loads, once)
        const int rlo = (i0 - 1) >> 1;
        if (lg.cin && rlo >= 0) {
            const int nc1 = a.gc.nn[1];
            const int J0 = c >> 1, J1 = (c + 1) >> 1;
            const int row = rlo * nc1;
            const int m0 = a.maskc[row + J0], m1 = a.maskc[row + J1];
#pragma unroll
            for (int q = 0; q < RB; ++q) {
                if (!((actmask >> q) & 1)) continue;
                const double* ecb = a.ec + (long long)(r0 + q) * a.gc.ndof;
                const double2 e0 = ld2(ecb + 2 * (row + J0));
                const double2 e1 = ld2(ecb + 2 * (row + J1));
                rs.cev[q][0] = (m0 & 1) ? 0.0 : e0.x; rs.cev[q][1] = (m0 & 2) ? 0.0 : e0.y;
                rs.cev[q][2] = (m1 & 1) ? 0.0 : e1.x; rs.cev[q][3] = (m1 & 2) ? 0.0 : e1.y;
            }
        }
    }

    for (int k = 0; k < nplanes; ++k) {
        const int stg = k % NS;
        const int P = i0 - 1 + k;
        mbar_wait(&bars[stg], (uint32_t)((k / NS) & 1));
        const char* st = wsm + stg * S::BYTES;
        // ---- plane-shared values: mask, E, diagonal, coarse masks
        const bool pv = P >= 0 && P < n0;
        int m = 3;
        double e = 0.0, el = 0.0;
        if (pv && lg.cin) m = *reinterpret_cast<const uint8_t*>(st + S::MOFF + ((P * n1 + wg.vlo) & 15) + (c - wg.vlo));
        if (P >= 0 && P < N0) {
            const int eo = ((8 * (P * N1 + wg.clo)) & 15) + lg.eoff_c;
            if (lg.ce) e = *reinterpret_cast<const double*>(st + S::EOFF + eo);
            if (lg.cel) el = *reinterpret_cast<const double*>(st + S::EOFF + eo - 8);
        }
        const double D = k0d * ((elA + eA) + (el + e));
        const double id = D > 0.0 ? omega / D : 0.0;
        const bool fx = m & 1, fy = m & 2;
        const bool own_plane = P >= own0 && P < own1;
        int cm = 3, cm0 = 3, cm1 = 3, cmf = 0;
        const int crow = S::HAS_CM ? coarse_row<OP>(a, P) : -1;
        if (S::HAS_CM && crow >= 0 && lg.cin) {
            cmf = (crow * a.gc.nn[1] + wg.jl) & 15;
            if (S::HAS_C) {
                cm0 = *reinterpret_cast<const uint8_t*>(st + S::CMOFF + cmf + ((c >> 1) - wg.jl));
                cm1 = *reinterpret_cast<const uint8_t*>(st + S::CMOFF + cmf + (((c + 1) >> 1) - wg.jl));
            } else if (!(c & 1)) {
                cm = *reinterpret_cast<const uint8_t*>(st + S::CMOFF + cmf + ((c >> 1) - wg.jl));
            }
        }
        const int L = P - 1;
        const bool fin = k > 0 && L >= i0;
        const bool own = lg.own_col && L >= own0 && L < own1;
        // ---- per RHS
#pragma unroll
        for (int q = 0; q < RB; ++q) {
            if (!((actmask >> q) & 1)) continue;
            const long long vb = (long long)(r0 + q) * a.g.ndof;
            double v0x = 0, v0y = 0, v1x = 0, v1y = 0, xx = 0, xy = 0;
            if (pv && lg.cin) {
                const double2 x0 = *reinterpret_cast<const double2*>(st + (0 * RB + q) * 512 + lg.vo);
                v0x = x0.x; v0y = x0.y;
                if (S::NV >= 2) {
                    const double2 x1 = *reinterpret_cast<const double2*>(st + (1 * RB + q) * 512 + lg.vo);
                    v1x = x1.x; v1y = x1.y;
                }
                if (S::NV >= 3) {
                    const double2 x2 = *reinterpret_cast<const double2*>(st + (2 * RB + q) * 512 + lg.vo);
                    xx = x2.x; xy = x2.y;
                }
            }
            double ux, uy, kx, ky;
            if (OP == M2_CGP) {
                ux = fma(coef[q], v1x, v0x);
                uy = fma(coef[q], v1y, v0y);
                if (lg.own_col && own_plane) st2(a.y2 + vb + 2 * (P * n1 + c), ux, uy);
                kx = v1x; ky = v1y;
            } else if (OP == M2_RESTRICT) {
                const double rx = fma(-coef[q], v1x, v0x), ry = fma(-coef[q], v1y, v0y);
                if (lg.own_col && own_plane) {
                    st2(a.y2 + vb + 2 * (P * n1 + c), rx, ry);
                    rs.dot[q] = fma(rx, rx, rs.dot[q]);
                    rs.dot[q] = fma(ry, ry, rs.dot[q]);
                }
                kx = rx; ky = ry;
                ux = fx ? 0.0 : id * rx;
                uy = fy ? 0.0 : id * ry;
            } else if (OP == M2_POST) {
                double cx0 = 0, cy0 = 0, cx1 = 0, cy1 = 0;
                if (crow >= 0 && lg.cin) {
                    const char* cp = st + S::COFF + q * 288;
                    const double2 e0 = *reinterpret_cast<const double2*>(cp + 16 * ((c >> 1) - wg.jbase));
                    const double2 e1 = *reinterpret_cast<const double2*>(cp + 16 * (((c + 1) >> 1) - wg.jbase));
                    cx0 = (cm0 & 1) ? 0.0 : e0.x; cy0 = (cm0 & 2) ? 0.0 : e0.y;
                    cx1 = (cm1 & 1) ? 0.0 : e1.x; cy1 = (cm1 & 2) ? 0.0 : e1.y;
                }
                double px, py;
                const bool codd = c & 1;
                if (P & 1) {
                    const double lx = codd ? 0.5 * (rs.cev[q][0] + rs.cev[q][2]) : rs.cev[q][0];
                    const double ly = codd ? 0.5 * (rs.cev[q][1] + rs.cev[q][3]) : rs.cev[q][1];
                    const double hx = codd ? 0.5 * (cx0 + cx1) : cx0, hy = codd ? 0.5 * (cy0 + cy1) : cy0;
                    px = 0.5 * (lx + hx);
                    py = 0.5 * (ly + hy);
                    rs.cev[q][0] = cx0; rs.cev[q][1] = cy0; rs.cev[q][2] = cx1; rs.cev[q][3] = cy1;
                } else {
                    px = codd ? 0.5 * (rs.cev[q][0] + rs.cev[q][2]) : rs.cev[q][0];
                    py = codd ? 0.5 * (rs.cev[q][1] + rs.cev[q][3]) : rs.cev[q][1];
                }
                ux = fx ? 0.0 : fma(id, v0x, px);
                uy = fy ? 0.0 : fma(id, v0y, py);
                kx = v0x; ky = v0y;
            } else {
                ux = v0x; uy = v0y;
                kx = v1x; ky = v1y;
            }
            const double mx = fx ? 0.0 : ux, my = fy ? 0.0 : uy;
            double nw[6];
            nw[2] = mx; nw[3] = my;
            nw[0] = shfl_up1(mx); nw[1] = shfl_up1(my);
            nw[4] = shfl_dn1(mx); nw[5] = shfl_dn1(my);
            if (k > 0) {
                // element layer L between the current plane (rs.w) and plane P (nw)
                double lox = rs.car[q][0], loy = rs.car[q][1], hix = 0.0, hiy = 0.0;
#pragma unroll
                for (int ee = 0; ee < 2; ++ee) {
                    const double Ee = ee ? eA : elA;
                    const int a1 = 1 - ee;
                    double tlx = 0, tly = 0, thx = 0, thy = 0;
#pragma unroll
                    for (int b0 = 0; b0 < 2; ++b0)
#pragma unroll
                        for (int b1 = 0; b1 < 2; ++b1)
#pragma unroll
                            for (int k2 = 0; k2 < 2; ++k2) {
                                const int qq = ee + b1;
                                const double xv = b0 ? nw[2 * qq + k2] : rs.w[q][2 * qq + k2];
                                const int col = (b0 * 2 + b1) * 2 + k2;
                                const int rl = (0 * 2 + a1) * 2, rh = (1 * 2 + a1) * 2;
                                if (!C03 || K2<C03>(rl + 0, col) != 0.0) tlx = fma(K2<C03>(rl + 0, col), xv, tlx);
                                if (!C03 || K2<C03>(rl + 1, col) != 0.0) tly = fma(K2<C03>(rl + 1, col), xv, tly);
                                if (!C03 || K2<C03>(rh + 0, col) != 0.0) thx = fma(K2<C03>(rh + 0, col), xv, thx);
                                if (!C03 || K2<C03>(rh + 1, col) != 0.0) thy = fma(K2<C03>(rh + 1, col), xv, thy);
                            }
                    lox = fma(Ee, tlx, lox); loy = fma(Ee, tly, loy);
                    hix = fma(Ee, thx, hix); hiy = fma(Ee, thy, hiy);
                }
                rs.car[q][0] = hix; rs.car[q][1] = hiy;
                if (fin) {
                    const double Axx = (mA & 1) ? rs.u[q][0] : lox, Axy = (mA & 2) ? rs.u[q][1] : loy;
                    const int o = 2 * (L * n1 + c);
                    if (OP == M2_MATVEC) {
                        if (own) st2(a.y + vb + o, Axx, Axy);
                    } else if (OP == M2_RESID) {
                        if (own) st2(a.y + vb + o, rs.k[q][0] - Axx, rs.k[q][1] - Axy);
                    } else if (OP == M2_JACOBI || OP == M2_POST) {
                        const double idA = omega / DA;
                        const double zx = fma((mA & 1) ? omega : idA, rs.k[q][0] - Axx, rs.u[q][0]);
                        const double zy = fma((mA & 2) ? omega : idA, rs.k[q][1] - Axy, rs.u[q][1]);
                        if (own) {
                            st2(a.y + vb + o, zx, zy);
                            rs.dot[q] = fma(rs.k[q][0], zx, rs.dot[q]);
                            rs.dot[q] = fma(rs.k[q][1], zy, rs.dot[q]);
                        }
                    } else if (OP == M2_CGP) {
                        if (own) {
                            st2(a.y + vb + o, Axx, Axy);
                            rs.dot[q] = fma(rs.u[q][0], Axx, rs.dot[q]);
                            rs.dot[q] = fma(rs.u[q][1], Axy, rs.dot[q]);
                            st2(a.xv + vb + o, fma(xal[q], rs.k[q][0], rs.k2[q][0]), fma(xal[q], rs.k[q][1], rs.k2[q][1]));
                        }
                    } else if (OP == M2_RESTRICT) {
                        const bool tv = lg.cin && lane >= 1 && lane <= 30;
                        const double tx = (tv && !(mA & 1)) ? rs.k[q][0] - Axx : 0.0;
                        const double ty = (tv && !(mA & 2)) ? rs.k[q][1] - Axy : 0.0;
                        const double tlx = shfl_up1(tx), tly = shfl_up1(ty);
                        const double trx = shfl_dn1(tx), try_ = shfl_dn1(ty);
                        const double hx = fma(0.5, tlx + trx, tx), hy = fma(0.5, tly + try_, ty);
                        const bool cown = lg.cin && !(c & 1) && lane >= 2 && lane <= 28;
                        const int nc1 = a.gc.nn[1];
                        const long long cb = (long long)(r0 + q) * a.gc.ndof;
                        if (L & 1) {
                            rs.acc[q][0] = fma(0.5, hx, rs.acc[q][0]);
                            rs.acc[q][1] = fma(0.5, hy, rs.acc[q][1]);
                            const int I = (L - 1) >> 1;
                            if (cown && I >= I0 && I < I1)
                                st2(a.coarse + cb + 2 * (I * nc1 + (c >> 1)), (cm & 1) ? 0.0 : rs.acc[q][0],
                                    (cm & 2) ? 0.0 : rs.acc[q][1]);
                            rs.acc[q][0] = 0.5 * hx;
                            rs.acc[q][1] = 0.5 * hy;
                        } else {
                            rs.acc[q][0] += hx;
                            rs.acc[q][1] += hy;
                            const int I = L >> 1;
                            if (L == n0 - 1 && cown && I >= I0 && I < I1)
                                st2(a.coarse + cb + 2 * (I * nc1 + (c >> 1)), (cm & 1) ? 0.0 : rs.acc[q][0],
                                    (cm & 2) ? 0.0 : rs.acc[q][1]);
                        }
                    }
                }
            }
            // ---- shift plane P -> current
#pragma unroll
            for (int j = 0; j < 6; ++j) rs.w[q][j] = nw[j];
            rs.u[q][0] = ux; rs.u[q][1] = uy;
            rs.k[q][0] = kx; rs.k[q][1] = ky;
            if (OP == M2_CGP) { rs.k2[q][0] = xx; rs.k2[q][1] = xy; }
        }
        mA = m; DA = D; eA = e; elA = el;
        __syncwarp();
        if (k + NS < nplanes) {
            if (lane == 0) fence_proxy_async();
            issue_plane<OP, RB>(a, wg, wsm + stg * S::BYTES, &bars[stg], P + NS, r0, nr, actmask, lane);
        }
    }
    if (a.partial) {
#pragma unroll
        for (int q = 0; q < RB; ++q) {
            if (!((actmask >> q) & 1)) continue;
            const double d = warp_sum(rs.dot[q]);
            if (lane == 0) a.partial[(long long)(r0 + q) * items + item] = d;
        }
    }
}

int march2_items(int op, const LevelGeom& g, const LevelGeom* gc) {
    if (op == M2_RESTRICT) {
        const int nct = (g.nn[1] + 27) / 28;
        const int nch = (gc->nn[0] + CCH - 1) / CCH;
        return nct * nch;
    }
    const int nct = (g.nn[1] + 29) / 30;
    const int nch = (g.nn[0] + CH - 1) / CH;
    return nct * nch;
}

template <int OP, int RB>
static void launch2_rb(const March2Args& a, bool c03, int nct, int nch, cudaStream_t s) {
    const int nrc = (a.R + RB - 1) / RB;
    const long long warps = (long long)nrc * nct * nch;
    const unsigned blocks = (unsigned)((warps + WPB - 1) / WPB);
    const int smem = WPB * NS * (Stage<OP, RB>::BYTES + 8);
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(march2_kernel<OP, true, RB>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        cudaFuncSetAttribute(march2_kernel<OP, false, RB>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        attr = true;
    }
    if (c03) march2_kernel<OP, true, RB><<<blocks, 32 * WPB, smem, s>>>(a, nct, nch, nrc);
    else march2_kernel<OP, false, RB><<<blocks, 32 * WPB, smem, s>>>(a, nct, nch, nrc);
}

template <int OP>
static void launch2(const March2Args& a, bool c03, cudaStream_t s) {
    int nct, nch;
    if (OP == M2_RESTRICT) {
        nct = (a.g.nn[1] + 27) / 28;
        nch = (a.gc.nn[0] + CCH - 1) / CCH;
    } else {
        nct = (a.g.nn[1] + 29) / 30;
        nch = (a.g.nn[0] + CH - 1) / CH;
    }
    launch2_rb<OP, 1>(a, c03, nct, nch, s);   // RHS blocking (RB > 1) measured slower: register bound
}

int march2_apply(int op, const March2Args& a, bool c03, cudaStream_t s) {
    switch (op) {
        case M2_MATVEC: launch2<M2_MATVEC>(a, c03, s); break;
        case M2_RESID: launch2<M2_RESID>(a, c03, s); break;
        case M2_JACOBI: launch2<M2_JACOBI>(a, c03, s); break;
        case M2_CGP: launch2<M2_CGP>(a, c03, s); break;
        case M2_RESTRICT: launch2<M2_RESTRICT>(a, c03, s); break;
        default: launch2<M2_POST>(a, c03, s); break;
    }
    return march2_items(op, a.g, &a.gc);
}
