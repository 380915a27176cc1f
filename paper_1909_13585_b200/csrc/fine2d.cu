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
// (vectors, E_e, masks, coarse rows) is staged by per-lane cp.async (LDGSTS, zero-fill
// predicates) into a per-warp shared-memory ring of NSTAGE planes, one commit group per
// plane (MG_ASYNC_RING; a register prefetch ring is the fallback); the ghost-padded layout
// makes every load unconditional.  Each step exchanges column neighbours by warp shuffles,
// adds the contribution of one element layer to the two node planes it touches, and
// finishes the lower plane.  No atomics, no colouring: deterministic.  The RHS index is
// the fastest grid coordinate so the R warps of a tile share E_e in L2.
// K0 entries for nu = 0.3 are compile-time constants (element.cuh).
#include "element.cuh"
#include <algorithm>

#include "kernels.h"

__constant__ double c_K2[64];
__constant__ double c_Kh2[64];

#ifndef MG_2D_TRANSFORM
#define MG_2D_TRANSFORM 1   // element operator in the sum/difference basis (10 nonzeros, see below)
#endif

// K^ = T^-T K0 T^-1 in the per-axis (m = v0 + v1, d = v1 - v0) basis (see h8t.cu): closed form from
// the 1-D factors M^ = diag(1/4, 1/12), D^ = diag(0, 1), C^[d][m] = C^T[m][d] = 1/2; plane stress.
__host__ __device__ constexpr double f1h2(int kind, int ta, int tb) {
    return kind == 0 ? (ta == tb ? (ta == 0 ? 0.25 : 1.0 / 12.0) : 0.0)
         : kind == 1 ? ((ta == 1 && tb == 1) ? 1.0 : 0.0)
         : kind == 2 ? ((ta == 1 && tb == 0) ? 0.5 : 0.0)
                     : ((ta == 0 && tb == 1) ? 0.5 : 0.0);
}
__host__ __device__ constexpr double sh2(int i, int j, int s, int t) {
    double v = 1.0;
    for (int k = 0; k < 2; ++k) {
        const int ta = (s >> (1 - k)) & 1, tb = (t >> (1 - k)) & 1;
        const int kind = (k == i && k == j) ? 1 : (k == i ? 2 : (k == j ? 3 : 0));
        v *= f1h2(kind, ta, tb);
    }
    return v;
}
__host__ __device__ constexpr double khat2(double nu, int row, int col) {
    const int s = row / 2, i = row % 2, t = col / 2, j = col % 2;
    const double mu = 1.0 / (2.0 * (1.0 + nu));
    const double lam = nu / (1.0 - nu * nu);
    double v = lam * sh2(i, j, s, t) + mu * sh2(j, i, s, t);
    if (i == j)
        for (int k = 0; k < 2; ++k) v += mu * sh2(k, k, s, t);
    return v;
}

void fine2d_set_constants(const double* K0, cudaStream_t s) {
    cudaMemcpyToSymbolAsync(c_K2, K0, sizeof(double) * 64, 0, cudaMemcpyHostToDevice, s);
    // K^ from K0 (any element / nu): per axis T^-1 = (1/2) [[1, -1], [1, 1]]
    static double Ti[8][8], Kh[64];
    for (int a = 0; a < 4; ++a)
        for (int t = 0; t < 4; ++t) {
            double v = 1.0;
            for (int k = 0; k < 2; ++k) {
                const int ab = (a >> (1 - k)) & 1, tb = (t >> (1 - k)) & 1;
                v *= 0.5 * ((tb == 0) ? 1.0 : (ab ? 1.0 : -1.0));
            }
            for (int i = 0; i < 2; ++i)
                for (int j = 0; j < 2; ++j) Ti[2 * a + i][2 * t + j] = (i == j) ? v : 0.0;
        }
    for (int r = 0; r < 8; ++r)
        for (int c = 0; c < 8; ++c) {
            double v = 0.0;
            for (int p = 0; p < 8; ++p)
                for (int q = 0; q < 8; ++q) v += Ti[p][r] * K0[p * 8 + q] * Ti[q][c];
            Kh[r * 8 + c] = v;
        }
    cudaMemcpyToSymbolAsync(c_Kh2, Kh, sizeof(Kh), 0, cudaMemcpyHostToDevice, s);
}

template <bool C03>
__device__ __forceinline__ double K2(int r, int c) {
    if (C03) return k0_entry<2>(MG_NU_PAPER, r, c);
    return c_K2[r * 8 + c];
}
// transformed element matrix: the sparsity (10 nonzeros) is that of the standard element at
// nu = 0.3, shared by every nu and by the incompatible-mode element
template <bool C03>
__device__ __forceinline__ double KH2(int r, int c) {
    if (C03) return khat2(MG_NU_PAPER, r, c);
    return c_Kh2[r * 8 + c];
}

// register prefetch depth (node planes in flight per warp) and CTAs per SM (register cap)
// per kernel: tuned on B200 with ncu / bench A/B
#ifndef MG_PD_CGP
#define MG_PD_CGP 2
#endif
#ifndef MG_PD_RESTRICT
#define MG_PD_RESTRICT 1
#endif
#ifndef MG_PD_POST
#define MG_PD_POST 1
#endif
#ifndef MG_MB_CGP
#define MG_MB_CGP 3
#endif
#ifndef MG_MB_RESTRICT
#define MG_MB_RESTRICT 4
#endif
#ifndef MG_MB_POST
#define MG_MB_POST 4
#endif
static constexpr int prefetch_depth(int op) {
    return op == M2_POST ? MG_PD_POST : op == M2_RESTRICT ? MG_PD_RESTRICT : op == M2_CGP ? MG_PD_CGP : 2;
}
static constexpr int CH_MAX = 64; // node planes per chunk (halved on small grids, see march2_chunk)
static constexpr int WPB = 4;     // warps per CTA (independent)
// cap at 170 registers so 3 CTAs (12 warps) fit per SM (POST would otherwise take 185)
static constexpr int march_minb(int op) {
    return op == M2_POST ? MG_MB_POST : op == M2_RESTRICT ? MG_MB_RESTRICT : op == M2_CGP ? MG_MB_CGP : 3;
}


__device__ __forceinline__ double2 ld2(const double* p) { return *reinterpret_cast<const double2*>(p); }
__device__ __forceinline__ double2 ldg2(const double* p) { return __ldg(reinterpret_cast<const double2*>(p)); }
__device__ __forceinline__ void st2(double* p, double a, double b) { *reinterpret_cast<double2*>(p) = make_double2(a, b); }

// ---------------------------------------------------------------- padded layout
Pad2 pad2_layout(const LevelGeom& g) {
    Pad2 p{};
    const int n0 = g.nn[0], n1 = g.nn[1], N0 = g.N[0], N1 = g.N[1];
    p.pitch = (n1 + 2 + 3) & ~3;                 // multiple of 4: a lane's mask byte offset is fixed
    p.org = 16 + p.pitch + 5;                    // front slack (lanes reach column -3 of row -1); org % 4 == 1
    p.nodes = p.org + (long long)(n0 + 1) * p.pitch + 64;
    p.pitchE = N1 + 2;
    p.orgE = 16 + p.pitchE + 4;
    p.elems = p.orgE + (long long)(N0 + 1) * p.pitchE + 64;
    p.vstride = (2 * p.nodes + 3) & ~3LL;
    return p;
}

__global__ void pad_nodes_u8_kernel(int n0, int n1, Pad2 p, const uint8_t* src, uint8_t* dst, uint8_t fill) {
    long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= p.nodes) return;
    const long long q = i - p.org;
    long long row = q >= 0 ? q / p.pitch : -1 - ((-q - 1) / p.pitch);
    const long long col = q - row * p.pitch;
    uint8_t v = fill;
    if (row >= 0 && row < n0 && col >= 0 && col < n1) v = src[row * n1 + col];
    dst[i] = v;
}

__global__ void pad_nodes_f64_kernel(int n0, int n1, Pad2 p, const double* src, double* dst) {
    long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= p.nodes) return;
    const long long q = i - p.org;
    long long row = q >= 0 ? q / p.pitch : -1 - ((-q - 1) / p.pitch);
    const long long col = q - row * p.pitch;
    double a = 0.0, b = 0.0;
    if (row >= 0 && row < n0 && col >= 0 && col < n1) {
        a = src[2 * (row * n1 + col)];
        b = src[2 * (row * n1 + col) + 1];
    }
    dst[2 * i] = a;
    dst[2 * i + 1] = b;
}

__global__ void pad_elems_kernel(int N0, int N1, Pad2 p, const double* src, double* dst) {
    long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= p.elems) return;
    const long long q = i - p.orgE;
    long long row = q >= 0 ? q / p.pitchE : -1 - ((-q - 1) / p.pitchE);
    const long long col = q - row * p.pitchE;
    double v = 0.0;
    if (row >= 0 && row < N0 && col >= 0 && col < N1) v = src[row * N1 + col];
    dst[i] = v;
}

// compact (R, src_ndof) planes [0, nplanes) -> padded local planes [p0, p0 + nplanes), masked at
// fixed DOFs (mask: compact local node masks or NULL)
__global__ void pad_vectors_kernel(int nplanes, int p0, int n1, Pad2 p, const uint8_t* mask, const double* src,
                                   double* dst, long long src_ndof) {
    const int r = blockIdx.y;
    const long long nodes = (long long)nplanes * n1;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < nodes; i += (long long)gridDim.x * blockDim.x) {
        const long long row = i / n1 + p0, col = i - (i / n1) * n1;
        const int m = mask ? mask[row * n1 + col] : 0;
        const double2 v = ld2(src + r * src_ndof + 2 * i);
        st2(dst + r * p.vstride + 2 * (p.org + row * p.pitch + col), (m & 1) ? 0.0 : v.x, (m & 2) ? 0.0 : v.y);
    }
}

__global__ void unpad_vectors_kernel(int nplanes, int p0, int n1, Pad2 p, const double* src, double* dst,
                                     long long dst_ndof) {
    const int r = blockIdx.y;
    const long long nodes = (long long)nplanes * n1;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < nodes; i += (long long)gridDim.x * blockDim.x) {
        const long long row = i / n1 + p0, col = i - (i / n1) * n1;
        const double2 v = ld2(src + r * p.vstride + 2 * (p.org + row * p.pitch + col));
        st2(dst + r * dst_ndof + 2 * i, v.x, v.y);
    }
}

static unsigned blocks_for(long long n) { return (unsigned)((n + 255) / 256); }

void pad2_nodes_u8(const LevelGeom& g, const Pad2& p, const uint8_t* src, uint8_t* dst, uint8_t fill, cudaStream_t s) {
    pad_nodes_u8_kernel<<<blocks_for(p.nodes), 256, 0, s>>>(g.nn[0], g.nn[1], p, src, dst, fill);
}
void pad2_nodes_f64(const LevelGeom& g, const Pad2& p, const double* src, double* dst, cudaStream_t s) {
    pad_nodes_f64_kernel<<<blocks_for(p.nodes), 256, 0, s>>>(g.nn[0], g.nn[1], p, src, dst);
}
void pad2_elems(const LevelGeom& g, const Pad2& p, const double* src, double* dst, cudaStream_t s) {
    pad_elems_kernel<<<blocks_for(p.elems), 256, 0, s>>>(g.N[0], g.N[1], p, src, dst);
}
void pad2_vectors(const LevelGeom& g, const Pad2& p, int R, const uint8_t* mask, const double* src, double* dst,
                  cudaStream_t s) {
    pad2_vectors_planes(g, p, R, mask, 0, g.nn[0], src, g.ndof, dst, s);
}
void unpad2_vectors(const LevelGeom& g, const Pad2& p, int R, const double* src, double* dst, cudaStream_t s) {
    unpad2_vectors_planes(g, p, R, 0, g.nn[0], src, dst, g.ndof, s);
}
void pad2_vectors_planes(const LevelGeom& g, const Pad2& p, int R, const uint8_t* mask, int p0, int nplanes,
                         const double* src, long long src_ndof, double* dst, cudaStream_t s) {
    dim3 grid((unsigned)std::min<long long>(blocks_for((long long)nplanes * g.nn[1]), 1184), R);
    pad_vectors_kernel<<<grid, 256, 0, s>>>(nplanes, p0, g.nn[1], p, mask, src, dst, src_ndof);
}
void unpad2_vectors_planes(const LevelGeom& g, const Pad2& p, int R, int p0, int nplanes, const double* src,
                           double* dst, long long dst_ndof, cudaStream_t s) {
    dim3 grid((unsigned)std::min<long long>(blocks_for((long long)nplanes * g.nn[1]), 1184), R);
    unpad_vectors_kernel<<<grid, 256, 0, s>>>(nplanes, p0, g.nn[1], p, src, dst, dst_ndof);
}

// ---------------------------------------------------------------- march kernels
struct Slot {
    double v0x, v0y, v1x, v1y, xx, xy;   // vectors at (P, c)
    double e, el;                        // E(P, c), E(P, c-1)
    double dx, dy;                       // D^-1 at (P, c)   (RESTRICT / POST / JACOBI)
    int m;                               // fixed bits at (P, c)
    double cx0, cy0, cx1, cy1;           // POST: coarse row (P+1)/2 at J0, J1 (odd P), coarse-masked
    int cm;                              // RESTRICT: coarse mask of row (P-1)>>1 at J = c/2
};

template <int OP>
struct Ops {
    static constexpr bool V1 = OP == M2_CGP || OP == M2_RESTRICT || OP == M2_RESID || OP == M2_JACOBI;
    static constexpr bool XV = OP == M2_CGP;
    static constexpr bool DI = OP == M2_RESTRICT || OP == M2_POST || OP == M2_JACOBI;
};

#ifndef MG_ASYNC_RING
#define MG_ASYNC_RING 1   // POST / RESTRICT: cp.async shared-memory prefetch ring (see below)
#endif
#ifndef MG_2D_UNROLL
#define MG_2D_UNROLL 3    // async ring loop unrolled by NSTAGE: bit 0 CGP, bit 1 RESTRICT, bit 2 POST (B200 A/B: POST slower)
#endif
#ifndef MG_ASYNC_CGP
#define MG_ASYNC_CGP 1    // CGP through the same ring
#endif
#ifndef MG_NSTAGE
#define MG_NSTAGE 4
#endif
static constexpr int NSTAGE = MG_NSTAGE;   // planes in flight per warp in the async ring

// cp.async (LDGSTS): per-lane asynchronous global -> shared copies; a false predicate zero-fills
__device__ __forceinline__ void cpa16(void* dst, const void* src, bool pred) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(d), "l"(src), "r"(pred ? 16 : 0));
}
__device__ __forceinline__ void cpa8(void* dst, const void* src, bool pred) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(d), "l"(src), "r"(pred ? 8 : 0));
}
__device__ __forceinline__ void cpa4(void* dst, const void* src, bool pred) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(d), "l"(src), "r"(pred ? 4 : 0));
}
__device__ __forceinline__ void cpa_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cpa_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// Per-warp ring of NSTAGE planes (struct of arrays over the 32 lanes); unused fields have size 1.
template <int OP>
struct ARing {
    static constexpr bool POST = OP == M2_POST, RESTR = OP == M2_RESTRICT, CGP = OP == M2_CGP;
    double2 v0[NSTAGE][32];
    double2 v1[(RESTR || CGP) ? NSTAGE : 1][32];
    double2 xv[CGP ? NSTAGE : 1][32];
    double2 d[CGP ? 1 : NSTAGE][32];
    double e[NSTAGE][32];
    unsigned m[NSTAGE][32];                 // aligned 4-byte word holding the mask byte
    double2 c0[POST ? NSTAGE : 1][32];       // coarse node J0 = c >> 1 (J1's value comes from lane + 1)
    unsigned cm0[CGP ? 1 : NSTAGE][32];
};

// SLAB = false: single slab (off0 = 0, every plane owned) -- the slab checks compile away
template <int OP, bool C03, bool SLAB>
__global__ void __launch_bounds__(32 * WPB, march_minb(OP)) march2_kernel(March2Args a, int nct, int nch, int chl) {
    pdl_begin();
    constexpr int CS = (OP == M2_RESTRICT) ? 28 : 30;      // owned columns per warp
    // lane of the first owned column; lane 0 sits at an odd column for every op, which with
    // pad2_layout's odd org and pitch % 4 == 0 makes each warp's 512-byte plane row 32-byte aligned
    constexpr int LOFF = (OP == M2_RESTRICT) ? 3 : 1;
    const int lane = threadIdx.x & 31;
    const long long w = (long long)blockIdx.x * WPB + (threadIdx.x >> 5);
    const int items = nct * nch;
    if (w >= (long long)a.R * items) return;
    if (a.done && *a.done) return;
    const int r = (int)(w % a.R);
    const int item = (int)(w / a.R);
    if (a.active && !a.active[r]) return;
    const int ct = item % nct, ch = item / nct;
    const int n0 = a.g.nn[0], n1 = a.g.nn[1];
    const int c = ct * CS + lane - LOFF;
    const bool cin = c >= 0 && c < n1;
    const bool own_col = cin && lane >= LOFF && lane < LOFF + CS;
    // off0 = 1 when the slab's local plane 0 is a ghost plane at an odd global index:
    // coarse row I is coincident with local fine plane 2I - off0 (parities use P + off0).
    const int off0 = SLAB ? a.off0 : 0;
    int i0, i1, own0, own1, I0 = 0, I1 = 0;
    if (OP == M2_RESTRICT) {
        const int nc0 = a.gc.nn[0];
        I0 = ch * (chl / 2);
        I1 = min(I0 + chl / 2, nc0);
        i0 = max(0, 2 * I0 - 1 - off0);
        i1 = min(2 * I1 - off0, n0);
        own0 = max(0, 2 * I0 - off0);
        own1 = i1;
    } else {
        i0 = ch * chl;
        i1 = min(i0 + chl, n0);
        own0 = i0;
        own1 = i1;
    }
    const Pad2& pd = a.pd;
    const long long vb = (long long)r * pd.vstride;
    const long long vbc = (OP == M2_RESTRICT || OP == M2_POST) ? (long long)r * a.gc.ndof : 0;
    const double* x0b = a.x + vb;
    const double* x1b = Ops<OP>::V1 ? a.x2 + vb : nullptr;
    double* xvb = Ops<OP>::XV ? a.xv + vb : nullptr;
    double* yb = (OP != M2_RESTRICT) ? a.y + vb : nullptr;
    double* y2b = (OP == M2_CGP || OP == M2_RESTRICT) ? a.y2 + vb : nullptr;
    const double beta = (OP == M2_CGP) ? a.beta[r] : 0.0;
    const double alpha = (OP == M2_RESTRICT) ? a.alpha[r] : 0.0;
    const double xalpha = (OP == M2_CGP) ? a.xalpha[r] : 0.0;
    const double omega = a.omega;
    const int nc1 = (OP == M2_RESTRICT || OP == M2_POST) ? a.gc.nn[1] : 0;
    const int J0 = c >> 1, J1 = (c + 1) >> 1;

    // padded offsets of plane P at this lane's column: node org + P*pitch + c, element orgE + P*pitchE + c
    auto load = [&](Slot& s, int P) {
        const long long no = pd.org + (long long)P * pd.pitch + c;
        const long long eo = pd.orgE + (long long)P * pd.pitchE + c;
        const double2 v0 = ldg2(x0b + 2 * no);
        s.v0x = v0.x; s.v0y = v0.y;
        if (Ops<OP>::V1) { const double2 v1 = ldg2(x1b + 2 * no); s.v1x = v1.x; s.v1y = v1.y; }
        if (Ops<OP>::XV) { const double2 v2 = ld2(xvb + 2 * no); s.xx = v2.x; s.xy = v2.y; }
        if (Ops<OP>::DI) { const double2 d = ldg2(a.Dinv + 2 * no); s.dx = d.x; s.dy = d.y; }
        s.e = __ldg(a.E + eo);
#if !MG_2D_TRANSFORM
        s.el = __ldg(a.E + eo - 1);
#endif
        s.m = __ldg(a.mask + no);
        if (OP == M2_POST) {
            s.cx0 = s.cy0 = s.cx1 = s.cy1 = 0.0;
            const int Ps = P + off0;
            const int I = (Ps + 1) >> 1;
            if ((Ps & 1) && cin && I < a.gc.nn[0]) {
                const long long row = (long long)I * nc1;
                const int m0 = a.maskc[row + J0], m1 = a.maskc[row + J1];
                const double2 e0 = ld2(a.ec + vbc + 2 * (row + J0));
                const double2 e1 = ld2(a.ec + vbc + 2 * (row + J1));
                s.cx0 = (m0 & 1) ? 0.0 : e0.x; s.cy0 = (m0 & 2) ? 0.0 : e0.y;
                s.cx1 = (m1 & 1) ? 0.0 : e1.x; s.cy1 = (m1 & 2) ? 0.0 : e1.y;
            }
        }
        if (OP == M2_RESTRICT) {
            s.cm = 3;
            const int Ps = P + off0;
            const int I = (Ps - 1) >> 1;
            if (Ps >= 1 && cin && !(c & 1) && I < a.gc.nn[0]) s.cm = a.maskc[(long long)I * nc1 + J0];
        }
    };

    // async ring (POST / RESTRICT): issue(P) copies plane P's lane data into stage st; fetch(s, P)
    // rebuilds the same Slot as load() from shared memory (after cpa_wait)
    constexpr bool ASYNC = MG_ASYNC_RING && (OP == M2_POST || OP == M2_RESTRICT || (MG_ASYNC_CGP && OP == M2_CGP));
    __shared__ ARing<OP> ring_sm[ASYNC ? WPB : 1];
    ARing<OP>& AR = ring_sm[ASYNC ? (threadIdx.x >> 5) : 0];
    auto issue = [&](int P, int st) {
        const long long no = pd.org + (long long)P * pd.pitch + c;
        const long long eo = pd.orgE + (long long)P * pd.pitchE + c;
        cpa16(&AR.v0[st][lane], x0b + 2 * no, true);
        if (OP == M2_RESTRICT || OP == M2_CGP) cpa16(&AR.v1[st][lane], x1b + 2 * no, true);
        if (OP == M2_CGP) cpa16(&AR.xv[st][lane], xvb + 2 * no, true);
        if (OP != M2_CGP) cpa16(&AR.d[st][lane], a.Dinv + 2 * no, true);
        cpa8(&AR.e[st][lane], a.E + eo, true);
        cpa4(&AR.m[st][lane], reinterpret_cast<const uint8_t*>((uintptr_t)(a.mask + no) & ~(uintptr_t)3), true);
        const int Ps = P + off0;
        if (OP == M2_POST) {
            const int I = (Ps + 1) >> 1;
            const bool pr = (Ps & 1) && cin && I < a.gc.nn[0];
            const long long row = (long long)(pr ? I : 0) * nc1;
            const long long j0 = pr ? J0 : 0;
            cpa16(&AR.c0[st][lane], a.ec + vbc + 2 * (row + j0), pr);
            cpa4(&AR.cm0[st][lane], reinterpret_cast<const uint8_t*>((uintptr_t)(a.maskc + row + j0) & ~(uintptr_t)3), pr);
        }
        if (OP == M2_RESTRICT) {
            const int I = (Ps - 1) >> 1;
            const bool pr = Ps >= 1 && cin && !(c & 1) && I < a.gc.nn[0];
            const long long ci = pr ? (long long)I * nc1 + J0 : 0;
            cpa4(&AR.cm0[st][lane], reinterpret_cast<const uint8_t*>((uintptr_t)(a.maskc + ci) & ~(uintptr_t)3), pr);
        }
    };
    const int msh = 8 * (int)((unsigned)(pd.org + c) & 3u);   // pitch % 4 == 0 (pad2_layout)
    // byte i of a mask array (4-byte aligned base) from the aligned word holding it
    auto byte_of = [](unsigned word, unsigned i) { return (int)((word >> (8 * (i & 3u))) & 0xffu); };
    auto fetch = [&](Slot& s, int P, int st) {
        const double2 v0 = AR.v0[st][lane];
        s.v0x = v0.x; s.v0y = v0.y;
        if (OP == M2_RESTRICT || OP == M2_CGP) { const double2 v1 = AR.v1[st][lane]; s.v1x = v1.x; s.v1y = v1.y; }
        if (OP == M2_CGP) { const double2 x2 = AR.xv[st][lane]; s.xx = x2.x; s.xy = x2.y; }
        if (OP != M2_CGP) { const double2 d = AR.d[st][lane]; s.dx = d.x; s.dy = d.y; }
        s.e = AR.e[st][lane];
        s.m = (int)((AR.m[st][lane] >> msh) & 0xffu);
        const int Ps = P + off0;
        if (OP == M2_POST) {
            const int I = (Ps + 1) >> 1;
            const bool pr = (Ps & 1) && cin && I < a.gc.nn[0];
            s.cx0 = s.cy0 = 0.0;
            if (pr) {
                const int m0 = byte_of(AR.cm0[st][lane], (unsigned)I * (unsigned)nc1 + J0);
                const double2 e0 = AR.c0[st][lane];
                s.cx0 = (m0 & 1) ? 0.0 : e0.x; s.cy0 = (m0 & 2) ? 0.0 : e0.y;
            }
            // J1 = (c + 1) >> 1 is lane + 1's J0 when c is odd (c + 1 <= N1 is inside), else J0
            const double nx = shfl_dn1(s.cx0), ny = shfl_dn1(s.cy0);
            s.cx1 = (c & 1) ? nx : s.cx0;
            s.cy1 = (c & 1) ? ny : s.cy0;
        }
        if (OP == M2_RESTRICT) {
            const int I = (Ps - 1) >> 1;
            const bool pr = Ps >= 1 && cin && !(c & 1) && I < a.gc.nn[0];
            s.cm = pr ? byte_of(AR.cm0[st][lane], (unsigned)I * (unsigned)nc1 + J0) : 3;
        }
    };

    // plane state
#if MG_2D_TRANSFORM
    double eAmx, eAdx, eAmy, eAdy;              // edge (c, c+1) of plane L in the (m, d) basis
    double cymx = 0.0, cydx = 0.0, cymy = 0.0, cydy = 0.0;   // element layer L-1's plane-L edge part
#else
    double A0x, A0y, A1x, A1y, A2x, A2y;      // masked input at c-1, c, c+1 of plane L
#endif
    double urx, ury, auxx = 0, auxy = 0, aux2x = 0, aux2y = 0, dax = 1, day = 1;
#if MG_2D_TRANSFORM
    double ex;                                // E of layer L at c
#else
    double ex, exl;                           // E of layer L at c, c-1
    double carx = 0.0, cary = 0.0;
#endif
    int mA;
    double cev[4] = {0.0, 0.0, 0.0, 0.0};     // POST: coarse row of the last even plane
    double dot = 0.0, accx = 0.0, accy = 0.0;
    if (OP == M2_POST) {
        const int rlo = (i0 - 1 + off0) >> 1;
        if (cin && rlo >= 0) {
            const long long row = (long long)rlo * nc1;
            const int m0 = a.maskc[row + J0], m1 = a.maskc[row + J1];
            const double2 e0 = ld2(a.ec + vbc + 2 * (row + J0));
            const double2 e1 = ld2(a.ec + vbc + 2 * (row + J1));
            cev[0] = (m0 & 1) ? 0.0 : e0.x; cev[1] = (m0 & 2) ? 0.0 : e0.y;
            cev[2] = (m1 & 1) ? 0.0 : e1.x; cev[3] = (m1 & 2) ? 0.0 : e1.y;
        }
    }

    // derive the matvec input (u) of plane P from its slot; keeps the op's per-plane values
    auto derive = [&](const Slot& s, int P, double& ux, double& uy, double& kx, double& ky, double& k2x,
                      double& k2y) {
        const bool fx = s.m & 1, fy = s.m & 2;
        const bool own_plane = P >= own0 && P < own1;
        const bool slab_plane = !SLAB || (P >= a.so0 && P < a.so1);   // dots: slab-owned planes only
        if (OP == M2_CGP) {
            ux = fma(beta, s.v1x, s.v0x);
            uy = fma(beta, s.v1y, s.v0y);
            if (own_col && own_plane) st2(y2b + 2 * (pd.org + (long long)P * pd.pitch + c), ux, uy);
            kx = s.v1x; ky = s.v1y;
            k2x = s.xx; k2y = s.xy;
        } else if (OP == M2_RESTRICT) {
            const double rx = fma(-alpha, s.v1x, s.v0x), ry = fma(-alpha, s.v1y, s.v0y);
            if (own_col && own_plane) {
                st2(y2b + 2 * (pd.org + (long long)P * pd.pitch + c), rx, ry);
                if (slab_plane) {
                    dot = fma(rx, rx, dot);
                    dot = fma(ry, ry, dot);
                }
            }
            kx = rx; ky = ry;
            ux = fx ? 0.0 : omega * s.dx * rx;
            uy = fy ? 0.0 : omega * s.dy * ry;
            k2x = (double)s.cm;
        } else if (OP == M2_POST) {
            double px, py;
            const bool codd = c & 1;
            if ((P + off0) & 1) {
                const double lx = codd ? 0.5 * (cev[0] + cev[2]) : cev[0], ly = codd ? 0.5 * (cev[1] + cev[3]) : cev[1];
                const double hx = codd ? 0.5 * (s.cx0 + s.cx1) : s.cx0, hy = codd ? 0.5 * (s.cy0 + s.cy1) : s.cy0;
                px = 0.5 * (lx + hx);
                py = 0.5 * (ly + hy);
                cev[0] = s.cx0; cev[1] = s.cy0; cev[2] = s.cx1; cev[3] = s.cy1;
            } else {
                px = codd ? 0.5 * (cev[0] + cev[2]) : cev[0];
                py = codd ? 0.5 * (cev[1] + cev[3]) : cev[1];
            }
            ux = fx ? 0.0 : fma(omega * s.dx, s.v0x, px);
            uy = fy ? 0.0 : fma(omega * s.dy, s.v0y, py);
            kx = s.v0x; ky = s.v0y;
            k2x = k2y = 0.0;
        } else {
            ux = s.v0x; uy = s.v0y;
            kx = s.v1x; ky = s.v1y;
            k2x = k2y = 0.0;
        }
    };

    // ---- one march step: element layer L, finishing node plane L, with plane P = L + 1's slot
    auto prologue = [&](const Slot& s0) {
        double ux, uy;
        derive(s0, i0 - 1, ux, uy, auxx, auxy, aux2x, aux2y);
        mA = s0.m;
        urx = ux; ury = uy;
        dax = s0.dx; day = s0.dy;
        const double mx = (mA & 1) ? 0.0 : ux, my = (mA & 2) ? 0.0 : uy;
#if MG_2D_TRANSFORM
        const double nx0 = shfl_dn1(mx), ny0 = shfl_dn1(my);
        eAmx = mx + nx0; eAdx = nx0 - mx; eAmy = my + ny0; eAdy = ny0 - my;
        ex = s0.e;
#else
        A1x = mx; A1y = my;
        A0x = shfl_up1(mx); A0y = shfl_up1(my);
        A2x = shfl_dn1(mx); A2y = shfl_dn1(my);
        ex = s0.e; exl = s0.el;
#endif
    };
    auto step = [&](const Slot& s, int L) {
            const int P = L + 1;
        double ux, uy, kx, ky, k2x, k2y;
        derive(s, P, ux, uy, kx, ky, k2x, k2y);
        const double mx = (s.m & 1) ? 0.0 : ux, my = (s.m & 2) ? 0.0 : uy;
#if !MG_2D_TRANSFORM
        const double B1x = mx, B1y = my;
        const double B0x = shfl_up1(mx), B0y = shfl_up1(my);
        const double B2x = shfl_dn1(mx), B2y = shfl_dn1(my);
#endif
#if MG_2D_TRANSFORM
        // element (L, c) in the sum/difference basis: edge (c, c+1) of plane L+1 by a shuffle,
        // the axis-0 combination with the carried edge of plane L, K^ (10 nonzeros), and back:
        // the edge of plane L is completed with the carry, its node-c+1 half shuffled up.
        double lox, loy;
        {
            const double nxB = shfl_dn1(mx), nyB = shfl_dn1(my);
            const double eBmx = mx + nxB, eBdx = nxB - mx, eBmy = my + nyB, eBdy = nyB - my;
            // uh[2 s + k], s = 2 t0 + t1 (t0: axis 0, t1: axis 1), scaled by E(L, c)
            double uh[8];
            uh[0] = 0.0; uh[1] = 0.0;                             // translations (zero rows/cols)
            uh[2] = ex * (eAdx + eBdx); uh[3] = ex * (eAdy + eBdy);   // s = 1: (m, d)
            uh[4] = ex * (eBmx - eAmx); uh[5] = ex * (eBmy - eAmy);   // s = 2: (d, m)
            uh[6] = ex * (eBdx - eAdx); uh[7] = ex * (eBdy - eAdy);   // s = 3: (d, d)
            double yh[8];
#pragma unroll
            for (int r = 0; r < 8; ++r) {
                double acc = 0.0;
#pragma unroll
                for (int q = 2; q < 8; ++q)
                    if (khat2(MG_NU_PAPER, r, q) != 0.0) acc = fma(KH2<C03>(r, q), uh[q], acc);
                yh[r] = acc;
            }
            // lower edge (plane L) = s(0,t1) - s(1,t1) ; upper (plane L+1) = sum
            const double gmx = cymx + (yh[0] - yh[4]), gmy = cymy + (yh[1] - yh[5]);
            const double gdx = cydx + (yh[2] - yh[6]), gdy = cydy + (yh[3] - yh[7]);
            cymx = yh[0] + yh[4]; cymy = yh[1] + yh[5];
            cydx = yh[2] + yh[6]; cydy = yh[3] + yh[7];
            const double upx = shfl_up1(gmx + gdx), upy = shfl_up1(gmy + gdy);
            lox = (gmx - gdx) + upx;
            loy = (gmy - gdy) + upy;
            eAmx = eBmx; eAdx = eBdx; eAmy = eBmy; eAdy = eBdy;
        }
#else
        // element layer L: e=0 -> element column c-1, e=1 -> column c
        double lox = carx, loy = cary, hix = 0.0, hiy = 0.0;
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            const double Ee = e ? ex : exl;
            const int a1 = 1 - e;
            double tlx = 0, tly = 0, thx = 0, thy = 0;
#pragma unroll
            for (int b0 = 0; b0 < 2; ++b0)
#pragma unroll
                for (int b1 = 0; b1 < 2; ++b1)
#pragma unroll
                    for (int k2 = 0; k2 < 2; ++k2) {
                        const int q = e + b1;
                        const double xv = b0 ? (q == 0 ? (k2 ? B0y : B0x) : q == 1 ? (k2 ? B1y : B1x) : (k2 ? B2y : B2x))
                                             : (q == 0 ? (k2 ? A0y : A0x) : q == 1 ? (k2 ? A1y : A1x) : (k2 ? A2y : A2x));
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
#endif
        // ---- finish node plane L
        if (L >= i0) {
            const double Axx = (mA & 1) ? urx : lox, Axy = (mA & 2) ? ury : loy;
            const bool own = own_col && L >= own0 && L < own1;
            const bool sdot = own && (!SLAB || (L >= a.so0 && L < a.so1));   // slab-owned: counts in dots
            const long long o = 2 * (pd.org + (long long)L * pd.pitch + c);
            if (OP == M2_MATVEC) {
                if (own) st2(yb + o, Axx, Axy);
            } else if (OP == M2_RESID) {
                if (own) st2(yb + o, auxx - Axx, auxy - Axy);
            } else if (OP == M2_JACOBI || OP == M2_POST) {
                const double zx = fma(omega * dax, auxx - Axx, urx);
                const double zy = fma(omega * day, auxy - Axy, ury);
                if (own) {
                    st2(yb + o, zx, zy);
                    if (sdot) {
                        dot = fma(auxx, zx, dot);
                        dot = fma(auxy, zy, dot);
                    }
                }
            } else if (OP == M2_CGP) {
                if (own) {
                    st2(yb + o, Axx, Axy);
                    if (sdot) {
                        dot = fma(urx, Axx, dot);
                        dot = fma(ury, Axy, dot);
                    }
                    st2(xvb + o, fma(xalpha, auxx, aux2x), fma(xalpha, auxy, aux2y));
                }
            } else if (OP == M2_RESTRICT) {
                // t = r - K z1 (lanes 1..30 valid), then P^T: columns by shuffles, planes by carry
                // t counts only on slab-owned planes: the coarse ghost row above gets a
                // partial sum that the upper neighbour adds in (reverse halo exchange)
                const bool tv = cin && lane >= 1 && lane <= 30 && (!SLAB || (L >= a.so0 && L < a.so1));
                const double tx = (tv && !(mA & 1)) ? auxx - Axx : 0.0;
                const double ty = (tv && !(mA & 2)) ? auxy - Axy : 0.0;
                const double tlx = shfl_up1(tx), tly = shfl_up1(ty);
                const double trx = shfl_dn1(tx), try_ = shfl_dn1(ty);
                const double hx = fma(0.5, tlx + trx, tx), hy = fma(0.5, tly + try_, ty);
                const bool cown = cin && !(c & 1) && lane >= LOFF && lane <= LOFF + CS - 2;
                const int cm = (int)k2x;     // coarse mask of row (P-1)>>1 = the row output below
                const int Ls = L + off0;
                if (Ls & 1) {
                    accx = fma(0.5, hx, accx); accy = fma(0.5, hy, accy);
                    const int I = (Ls - 1) >> 1;
                    if (cown && I >= I0 && I < I1)
                        st2(a.coarse + vbc + 2 * ((long long)I * nc1 + J0), (cm & 1) ? 0.0 : accx,
                            (cm & 2) ? 0.0 : accy);
                    accx = 0.5 * hx; accy = 0.5 * hy;
                } else {
                    accx += hx; accy += hy;
                    const int I = Ls >> 1;
                    if (L == n0 - 1 && cown && I >= I0 && I < I1)
                        st2(a.coarse + vbc + 2 * ((long long)I * nc1 + J0), (cm & 1) ? 0.0 : accx,
                            (cm & 2) ? 0.0 : accy);
                }
            }
        }
        // ---- shift plane L+1 -> L
#if !MG_2D_TRANSFORM
        carx = hix; cary = hiy;
        A0x = B0x; A0y = B0y; A1x = B1x; A1y = B1y; A2x = B2x; A2y = B2y;
#endif
        urx = ux; ury = uy; mA = s.m;
        auxx = kx; auxy = ky; aux2x = k2x; aux2y = k2y;
        dax = s.dx; day = s.dy;
#if MG_2D_TRANSFORM
        ex = s.e;
#else
        ex = s.e; exl = s.el;
#endif
    };

    if constexpr (!ASYNC) {
        // register prefetch ring of PD planes
        constexpr int PD = prefetch_depth(OP);
        Slot ring[PD];
        Slot s0;
        load(s0, i0 - 1);
#pragma unroll
        for (int u = 0; u < PD; ++u) load(ring[u], min(i0 + u, i1));
        prologue(s0);
        for (int L0 = i0 - 1; L0 < i1; L0 += PD) {
#pragma unroll
            for (int u = 0; u < PD; ++u) {
                const int L = L0 + u;
                if (L >= i1) break;
                const Slot s = ring[u];
                if (L + 1 + PD <= i1) load(ring[u], L + 1 + PD);
                step(s, L);
            }
        }
    } else {
        // cp.async ring: NSTAGE planes in flight, one commit group per plane (empty groups keep
        // the count uniform), plane p in stage (p - i0 + 1) % NSTAGE
        auto stage = [&](int p) { return (int)((unsigned)(p - i0 + 1) % NSTAGE); };
#pragma unroll
        for (int k = 0; k < NSTAGE; ++k) {
            issue(min(i0 - 1 + k, i1), k);
            cpa_commit();
        }
        cpa_wait<NSTAGE - 1>();
        Slot s0;
        fetch(s0, i0 - 1, 0);
        prologue(s0);
        constexpr bool UNR = (MG_2D_UNROLL >> (OP == M2_CGP ? 0 : OP == M2_RESTRICT ? 1 : 2)) & 1;
        if constexpr (UNR) {
        // unrolled by NSTAGE: stage indices are compile-time and the plane-state shift becomes
        // register renaming (no moves)
        for (int L0 = i0 - 1; L0 < i1; L0 += NSTAGE) {
#pragma unroll
            for (int u = 0; u < NSTAGE; ++u) {
                const int L = L0 + u;
                if (L >= i1) break;
                const int P = L + 1;
                const int pn = P + NSTAGE - 1;
                if (pn <= i1) issue(pn, u);
                cpa_commit();
                cpa_wait<NSTAGE - 1>();
                Slot s;
                fetch(s, P, (u + 1) % NSTAGE);
                step(s, L);
            }
        }
        } else {
        for (int L = i0 - 1; L < i1; ++L) {
            const int P = L + 1;
            const int pn = P + NSTAGE - 1;
            if (pn <= i1) issue(pn, stage(pn));
            cpa_commit();
            cpa_wait<NSTAGE - 1>();
            Slot s;
            fetch(s, P, stage(P));
            step(s, L);
        }
        }
        cpa_wait<0>();
    }
    if (a.partial) {
        dot = warp_sum(dot);
        if (lane == 0) a.partial[(long long)r * a.pstride + item] = dot;
    }
}

// Chunk length along axis 0 (planes; RESTRICT: coarse rows = chl / 2): CH_MAX unless the
// grid then has too few warps to fill the SMs (small levels / configs), down to 4 planes.
static int march2_chunk(int op, const LevelGeom& g, const LevelGeom* gc, int R, int* nct_out, int* nch_out) {
    const int nct = op == M2_RESTRICT ? (g.nn[1] + 27) / 28 : (g.nn[1] + 29) / 30;
    const long long want = 3LL * 148 * WPB;   // resident warps at 3 CTAs / SM
    int chl = CH_MAX, nch = 0;
    for (;;) {
        nch = op == M2_RESTRICT ? (gc->nn[0] + chl / 2 - 1) / (chl / 2) : (g.nn[0] + chl - 1) / chl;
        if (chl <= 4 || (long long)R * nct * nch >= want) break;
        chl /= 2;
    }
    *nct_out = nct;
    *nch_out = nch;
    return chl;
}

int march2_items(int op, const LevelGeom& g, const LevelGeom* gc, int R) {
    int nct, nch;
    march2_chunk(op, g, gc, R, &nct, &nch);
    return nct * nch;
}

template <int OP>
static void launch2(const March2Args& a, bool c03, cudaStream_t s) {
    int nct, nch;
    const int chl = march2_chunk(OP, a.g, &a.gc, a.R, &nct, &nch);
    const long long warps = (long long)a.R * nct * nch;
    const unsigned blocks = (unsigned)((warps + WPB - 1) / WPB);
    const bool slab = a.off0 != 0 || a.so0 != 0 || a.so1 != a.g.nn[0];
    if (slab) {
        if (c03) launch_k(march2_kernel<OP, true, true>, dim3(blocks), dim3(32 * WPB), 0, s, a, nct, nch, chl);
        else launch_k(march2_kernel<OP, false, true>, dim3(blocks), dim3(32 * WPB), 0, s, a, nct, nch, chl);
    } else {
        if (c03) launch_k(march2_kernel<OP, true, false>, dim3(blocks), dim3(32 * WPB), 0, s, a, nct, nch, chl);
        else launch_k(march2_kernel<OP, false, false>, dim3(blocks), dim3(32 * WPB), 0, s, a, nct, nch, chl);
    }
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
    return march2_items(op, a.g, &a.gc, a.R);
}
