// Coarsest-level direct solve on the device ("dense
// factorization"; the paper's coarsest solve is unstated).
// Setup: the coarsest Galerkin operator (n_L <= a few thousand DOFs) is assembled
// dense and inverted in place by blocked Gauss-Jordan (SPD => no pivoting needed,
// block 32; rank-32 updates on the fp64 tensor cores, DMMA).  Per V-cycle: z = A^-1 r
// for all R vectors as a dense product on DMMA tiles (dense_apply_mma_kernel: a CTA owns
// 8 rows, its warps split k), so the solve is a bandwidth-bound dense product instead of a
// latency-bound triangular sweep.
#include <cstdlib>

#include "kernels.h"

static constexpr int GJ_NB = 32;

template <int DIM>
__global__ void dense_from_stencil_kernel(LevelGeom g, const double* __restrict__ st, double* A, long long ld) {
    pdl_begin();
    constexpr int NS = DIM == 2 ? 9 : 27;
    long long node = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    int s = blockIdx.y;
    if (node >= g.nnodes) return;
    int idx[3] = {0, 0, 0};
    long long t = node;
    for (int k = DIM - 1; k >= 0; --k) { idx[k] = (int)(t % g.nn[k]); t /= g.nn[k]; }
    int ss = s;
    int dl[3];
    for (int k = DIM - 1; k >= 0; --k) { dl[k] = ss % 3 - 1; ss /= 3; }
    long long q = 0;
    for (int k = 0; k < DIM; ++k) {
        int c = idx[k] + dl[k];
        if (c < 0 || c >= g.nn[k]) return;
        q = q * g.nn[k] + c;
    }
    for (int k = 0; k < DIM; ++k)
        for (int k2 = 0; k2 < DIM; ++k2)
            A[(DIM * node + k) * ld + DIM * q + k2] = st[((long long)(s * DIM + k) * DIM + k2) * g.nnodes + node];
    (void)NS;
}

void dense_from_stencil(const LevelGeom& g, const double* st, double* A, long long ld, cudaStream_t s) {
    int th = 128;
    dim3 grid((unsigned)((g.nnodes + th - 1) / th), g.dim == 2 ? 9 : 27);
    if (g.dim == 2)
        dense_from_stencil_kernel<2><<<grid, th, 0, s>>>(g, st, A, ld);
    else
        dense_from_stencil_kernel<3><<<grid, th, 0, s>>>(g, st, A, ld);
}

__global__ void pad_identity_kernel(double* A, long long n, long long npad) {
    pdl_begin();
    long long i = n + blockIdx.x * blockDim.x + threadIdx.x;
    if (i < npad) A[i * npad + i] = 1.0;
}

void dense_pad_identity(double* A, long long n, long long npad, cudaStream_t s) {
    if (npad > n) pad_identity_kernel<<<1, GJ_NB, 0, s>>>(A, n, npad);
}

// panel / fix-up kernels split the NB panel rows over GJ_TQ CTAs (grid.y) for parallelism
static constexpr int GJ_TQ = 4;

// Rrow[t][j] = sum_s P[t][s] A[k0+s][j]   (new row panel), Ccol[i][t] = A[i][k0+t] (old column panel)
// sym: only the lower triangle of the state M is kept (M[i][j] = sigma M[j][i], sigma = -1 when
// exactly one of i, j is a processed pivot index, see dense_spd_inverse): for j >= k0 + NB the row
// panel is read as M[j][K] (j unprocessed: sigma = +1), for j < k0 the column panel as -M[K][j].
__global__ void gj_panels_kernel(const double* A, long long ld, long long n, int k0, const double* P, double* Rrow,
                                 double* Ccol, int sym) {
    pdl_begin();
    __shared__ double Ps[GJ_NB][GJ_NB];
    const int tid = threadIdx.x;
    for (int e = tid; e < GJ_NB * GJ_NB; e += blockDim.x) Ps[e / GJ_NB][e % GJ_NB] = P[e];
    __syncthreads();
    long long j = (long long)blockIdx.x * blockDim.x + tid;
    if (j >= n) return;
    const int tb = blockIdx.y * (GJ_NB / GJ_TQ);   // this CTA's rows t of the panels
    double col[GJ_NB];
    const bool up = sym && j >= k0 + GJ_NB;   // upper part: read row j of the lower triangle
#pragma unroll
    for (int s = 0; s < GJ_NB; ++s) col[s] = up ? A[j * ld + k0 + s] : A[(k0 + s) * ld + j];
#pragma unroll
    for (int tt = 0; tt < GJ_NB / GJ_TQ; ++tt) {
        const int t = tb + tt;
        double acc = 0.0;
#pragma unroll
        for (int s = 0; s < GJ_NB; ++s) acc = fma(Ps[t][s], col[s], acc);
        Rrow[t * n + j] = acc;
    }
    // column panel: row j of A's column block (full storage: read explicitly to stay exact for the
    // unsymmetric rounding; sym: M[j][K] = -M[K][j] for processed j < k0, stored for j >= k0)
#pragma unroll
    for (int tt = 0; tt < GJ_NB / GJ_TQ; ++tt)
        Ccol[j * GJ_NB + tb + tt] = (sym && j < k0) ? -col[tb + tt] : (up ? col[tb + tt] : A[j * ld + k0 + tb + tt]);
}

// A[i][j] -= sum_t Ccol[i][t] Rrow[t][j] for all i, j (64x64 tile per CTA, 4x4 per thread).
__global__ void __launch_bounds__(256) gj_update_kernel(double* A, long long ld, long long n, const double* Ccol,
                                                        const double* Rrow, int sym) {
    pdl_begin();
    __shared__ double Cs[64][GJ_NB + 1];
    __shared__ double Rs[GJ_NB][64 + 1];
    const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
    const long long i0 = (long long)blockIdx.y * 64, j0 = (long long)blockIdx.x * 64;
    if (sym && j0 > i0) return;   // lower-triangle storage: upper tiles are not kept
    // the A tile is read up front so its latency overlaps the panel loads and the product
    double aold[4][4];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            const long long i = i0 + ty + 16 * a, j = j0 + tx + 16 * b;
            aold[a][b] = (i < n && j < n) ? A[i * ld + j] : 0.0;
        }
    for (int e = threadIdx.x; e < 64 * GJ_NB; e += 256) {
        int r = e / GJ_NB, t = e % GJ_NB;
        long long i = i0 + r;
        Cs[r][t] = i < n ? Ccol[i * GJ_NB + t] : 0.0;
        int t2 = e / 64, c = e % 64;
        long long j = j0 + c;
        Rs[t2][c] = j < n ? Rrow[t2 * n + j] : 0.0;
    }
    __syncthreads();
    double acc[4][4];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b] = 0.0;
#pragma unroll 8
    for (int t = 0; t < GJ_NB; ++t) {
        double cv[4], rv[4];
#pragma unroll
        for (int a = 0; a < 4; ++a) cv[a] = Cs[ty + 16 * a][t];
#pragma unroll
        for (int b = 0; b < 4; ++b) rv[b] = Rs[t][tx + 16 * b];
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int b = 0; b < 4; ++b) acc[a][b] = fma(cv[a], rv[b], acc[a][b]);
    }
#pragma unroll
    for (int a = 0; a < 4; ++a) {
        long long i = i0 + ty + 16 * a;
        if (i >= n) continue;
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            long long j = j0 + tx + 16 * b;
            if (j < n) A[i * ld + j] = aold[a][b] - acc[a][b];
        }
    }
}

// Same update on the fp64 tensor-core path (DMMA, mma.sync m8n8k4 f64): 64x64 tile per CTA,
// 4 warps of 32x32 (4x4 m8n8 tiles each); per k-step of 4 a warp loads 4 A and 4 B fragments
// (one double per lane each) for 16 MMAs instead of 8 shared loads per 16 FMAs per thread.
// Shared-memory leading dimensions = 4 (mod 16) doubles: conflict-free fragment loads.
static constexpr int GU_LDC = GJ_NB + 4, GU_LDR = 64 + 4;

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

// kn >= 0: the CTA whose tile holds the next diagonal block (kn..kn+31)^2 -- scheduled first --
// also inverts it after its update (Gauss-Jordan in shared memory) into Pn, so the next block
// step needs no separate diagonal kernel.
// Gauss-Jordan inverse of the 32x32 SPD block S in shared memory by NT threads (1024 / NT entries
// each, two barriers per pivot).  Scalar pivots: the blocked (4x4-pivot) variant measured slower
// on B200 (the redundant pivot-block inverses cost more than the barriers they save).
template <int NT>
__device__ __forceinline__ void gj_block_inverse_smem(double (*S)[GJ_NB + 1], int tid, int* status) {
    constexpr int PE = GJ_NB * GJ_NB / NT;
    for (int p = 0; p < GJ_NB; ++p) {
        const double piv = S[p][p];
        const double ip = __drcp_rn(piv);   // correctly rounded reciprocal, no division slow path
        double v[PE];
#pragma unroll
        for (int q = 0; q < PE; ++q) {
            const int e = tid + q * NT, i = e / GJ_NB, j = e % GJ_NB;
            if (i == p && j == p) v[q] = ip;
            else if (i == p) v[q] = S[p][j] * ip;
            else if (j == p) v[q] = -S[i][p] * ip;
            else v[q] = S[i][j] - S[i][p] * S[p][j] * ip;
        }
        if (!(piv > 0.0) && tid == 0) atomicOr(status, 2);
        __syncthreads();
#pragma unroll
        for (int q = 0; q < PE; ++q) {
            const int e = tid + q * NT;
            S[e / GJ_NB][e % GJ_NB] = v[q];
        }
        __syncthreads();
    }
}

// The standalone pivot-block inverse (1024 threads, one entry each) pivots on 2x2 blocks: half the
// barrier pairs of the scalar sweep; the 2x2 pivot inverse is closed-form in every thread.
__global__ void __launch_bounds__(1024) gj_diag_kernel(const double* A, long long ld, int k0, double* P, int* status) {
    pdl_begin();
    __shared__ double S[GJ_NB][GJ_NB + 1];
    const int e = threadIdx.x, i = e / GJ_NB, j = e % GJ_NB;
    S[i][j] = A[(k0 + i) * ld + k0 + j];
    __syncthreads();
    for (int b = 0; b < GJ_NB; b += 2) {
        const double a00 = S[b][b], a01 = S[b][b + 1], a10 = S[b + 1][b], a11 = S[b + 1][b + 1];
        const double det = a00 * a11 - a01 * a10;
        if (e == 0 && !(a00 > 0.0 && det > 0.0)) atomicOr(status, 2);
        const double id = __drcp_rn(det);
        const double q00 = a11 * id, q01 = -a01 * id, q10 = -a10 * id, q11 = a00 * id;
        const int ri = i - b, rj = j - b;
        const bool ip = ri == 0 || ri == 1, jp = rj == 0 || rj == 1;
        double v;
        if (ip && jp) {
            v = ri == 0 ? (rj == 0 ? q00 : q01) : (rj == 0 ? q10 : q11);
        } else if (ip) {
            const double s0 = S[b][j], s1 = S[b + 1][j];
            v = ri == 0 ? fma(q00, s0, q01 * s1) : fma(q10, s0, q11 * s1);
        } else if (jp) {
            const double s0 = S[i][b], s1 = S[i][b + 1];
            v = rj == 0 ? -fma(s0, q00, s1 * q10) : -fma(s0, q01, s1 * q11);
        } else {
            const double c0 = S[i][b], c1 = S[i][b + 1], r0 = S[b][j], r1 = S[b + 1][j];
            const double u0 = fma(q00, r0, q01 * r1), u1 = fma(q10, r0, q11 * r1);
            v = S[i][j] - fma(c0, u0, c1 * u1);
        }
        __syncthreads();
        S[i][j] = v;
        __syncthreads();
    }
    P[e] = S[i][j];
}

__global__ void __launch_bounds__(128) gj_update_mma_kernel(double* A, long long ld, long long n, const double* Ccol,
                                                            const double* Rrow, long long kn, double* Pn,
                                                            int* status, int sym) {
    pdl_begin();
    __shared__ __align__(16) double Cs[64 * GU_LDC];
    __shared__ __align__(16) double Rs[GJ_NB * GU_LDR];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int wm = warp >> 1, wn = warp & 1;
    // tile order: the next diagonal block's tile first, the others shifted up (CTA 0 starts first)
    const long long nt = gridDim.x;
    long long tile = (long long)blockIdx.y * nt + blockIdx.x;
    const long long td = kn >= 0 ? (kn / 64) * nt + kn / 64 : -1;
    if (td >= 0) tile = tile == 0 ? td : (tile <= td ? tile - 1 : tile);
    const long long i0 = (tile / nt) * 64, j0 = (tile % nt) * 64;
    if (sym && j0 > i0) return;   // lower-triangle storage: upper tiles are not kept
    const int gr = lane >> 2, gc = lane & 3;
    // old A values at this thread's accumulator positions (latency overlaps the panel loads)
    double2 aold[4][4];
#pragma unroll
    for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int ni = 0; ni < 4; ++ni) {
            const long long i = i0 + wm * 32 + mi * 8 + gr, j = j0 + wn * 32 + ni * 8 + 2 * gc;
            aold[mi][ni] = (i < n && j < n) ? *reinterpret_cast<const double2*>(A + i * ld + j) : make_double2(0.0, 0.0);
        }
    // panels by cp.async (16-byte pairs, zero-filled outside the matrix): all 16 copies of a
    // thread in flight at once instead of a load -> store dependency per element
#pragma unroll
    for (int q = 0; q < 64 * GJ_NB / 2 / 128; ++q) {
        const int e = 2 * (threadIdx.x + q * 128);
        const int r = e / GJ_NB, t = e % GJ_NB;
        const long long i = i0 + r;
        const unsigned dc = (unsigned)__cvta_generic_to_shared(&Cs[r * GU_LDC + t]);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dc),
                     "l"(Ccol + (i < n ? i : 0) * GJ_NB + t), "r"(i < n ? 16 : 0));
        const int t2 = e / 64, c = e % 64;
        const long long j = j0 + c;
        const unsigned dr = (unsigned)__cvta_generic_to_shared(&Rs[t2 * GU_LDR + c]);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dr),
                     "l"(Rrow + t2 * n + (j < n ? j : 0)), "r"(j < n ? 16 : 0));
    }
    asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::);
    __syncthreads();
    double acc[4][4][2];
#pragma unroll
    for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int ni = 0; ni < 4; ++ni) acc[mi][ni][0] = acc[mi][ni][1] = 0.0;
#pragma unroll
    for (int k0 = 0; k0 < GJ_NB; k0 += 4) {
        double af[4], bf[4];
#pragma unroll
        for (int mi = 0; mi < 4; ++mi) af[mi] = Cs[(wm * 32 + mi * 8 + gr) * GU_LDC + k0 + gc];
#pragma unroll
        for (int ni = 0; ni < 4; ++ni) bf[ni] = Rs[(k0 + gc) * GU_LDR + wn * 32 + ni * 8 + gr];
#pragma unroll
        for (int mi = 0; mi < 4; ++mi)
#pragma unroll
            for (int ni = 0; ni < 4; ++ni) dmma(acc[mi][ni][0], acc[mi][ni][1], af[mi], bf[ni]);
    }
#pragma unroll
    for (int mi = 0; mi < 4; ++mi) {
        const long long i = i0 + wm * 32 + mi * 8 + gr;
        if (i >= n) continue;
#pragma unroll
        for (int ni = 0; ni < 4; ++ni) {
            const long long j = j0 + wn * 32 + ni * 8 + 2 * gc;
            if (j < n)
                *reinterpret_cast<double2*>(A + i * ld + j) =
                    make_double2(aold[mi][ni].x - acc[mi][ni][0], aold[mi][ni].y - acc[mi][ni][1]);
        }
    }
    if (td < 0 || tile != td) return;
    // the next diagonal block is warp (q, q)'s 32x32 sub-tile
    const int q = (int)((kn / 32) & 1);
    __syncthreads();   // Cs is reused as the block
    double(*S)[GJ_NB + 1] = reinterpret_cast<double(*)[GJ_NB + 1]>(Cs);
    if (wm == q && wn == q) {
#pragma unroll
        for (int mi = 0; mi < 4; ++mi)
#pragma unroll
            for (int ni = 0; ni < 4; ++ni) {
                S[mi * 8 + gr][ni * 8 + 2 * gc] = aold[mi][ni].x - acc[mi][ni][0];
                S[mi * 8 + gr][ni * 8 + 2 * gc + 1] = aold[mi][ni].y - acc[mi][ni][1];
            }
    }
    __syncthreads();
    gj_block_inverse_smem<128>(S, threadIdx.x, status);
    for (int e = threadIdx.x; e < GJ_NB * GJ_NB; e += 128) Pn[e] = S[e / GJ_NB][e % GJ_NB];
}

// Both fix-ups in one launch (disjoint parts of A): grid.y < GJ_TQ -> pivot columns (rows outside
// the block, NB / GJ_TQ columns per CTA row), grid.y >= GJ_TQ -> pivot rows.
__global__ void __launch_bounds__(128) gj_fix_kernel(double* A, long long ld, long long n, int k0, const double* P,
                                                     const double* Ccol, const double* Rrow, int sym) {
    pdl_begin();
    __shared__ double Ps[GJ_NB][GJ_NB];
    if (blockIdx.y >= GJ_TQ) {
        const long long j = (long long)blockIdx.x * 128 + threadIdx.x;
        if (j >= n || (sym && j >= k0 + GJ_NB)) return;   // sym: pivot rows left of the block only
#pragma unroll
        for (int tt = 0; tt < GJ_NB / GJ_TQ; ++tt) {
            const int t = (blockIdx.y - GJ_TQ) * (GJ_NB / GJ_TQ) + tt;
            A[(k0 + t) * ld + j] = (j >= k0 && j < k0 + GJ_NB) ? P[t * GJ_NB + (j - k0)] : Rrow[t * n + j];
        }
        return;
    }
    for (int e = threadIdx.x; e < GJ_NB * GJ_NB; e += blockDim.x) Ps[e / GJ_NB][e % GJ_NB] = P[e];
    __syncthreads();
    long long i = (long long)blockIdx.x * 128 + threadIdx.x;
    if (i >= n || (i >= k0 && i < k0 + GJ_NB) || (sym && i < k0)) return;   // sym: pivot columns below only
    double c[GJ_NB];
#pragma unroll
    for (int s = 0; s < GJ_NB; ++s) c[s] = Ccol[i * GJ_NB + s];
#pragma unroll
    for (int tt = 0; tt < GJ_NB / GJ_TQ; ++tt) {
        const int t = blockIdx.y * (GJ_NB / GJ_TQ) + tt;
        double acc = 0.0;
#pragma unroll
        for (int s = 0; s < GJ_NB; ++s) acc = fma(c[s], Ps[s][t], acc);
        A[i * ld + k0 + t] = -acc;
    }
}

// MG_GJ_MMA=0 selects the DFMA update kernel
static bool gj_mma() {
    static bool v = [] {
        const char* e = getenv("MG_GJ_MMA");
        return e ? atoi(e) != 0 : true;
    }();
    return v;
}

static constexpr long long GJ_FOLD_N = 3072;

// MG_GJ_SYM=0: full storage; default: the state is kept in its lower triangle.  Invariant of the
// in-place Gauss-Jordan sweep on a symmetric matrix (processed pivot set S): M[S,S] and M[U,U]
// symmetric, M[S,U] = -M[U,S]^T -- so the update needs only the lower tiles (half the traffic;
// the 4160^2 C5 coarsest matrix then fits in L2), panels and fix-ups read / write the lower
// counterparts, and a final mirror restores the full symmetric inverse.
static bool gj_sym() {
    static bool v = [] {
        const char* e = getenv("MG_GJ_SYM");
        return e ? atoi(e) != 0 : true;
    }();
    return v;
}

int dense_spd_inverse_launches(long long npad) {
    const long long steps = npad / GJ_NB;
    const bool fold = gj_mma() && npad >= GJ_FOLD_N;
    return (int)(fold ? 3 * steps + 1 : 4 * steps) + (gj_sym() ? 1 : 0);
}

// MG_GJ_PDL=1: the Gauss-Jordan block steps launched with programmatic dependent launch (every
// kernel of the sequence starts with griddepcontrol.wait, so none reads its predecessors' output
// early); default off (B200 A/B in DESIGN.md)
static bool gj_pdl() {
    static bool v = [] {
        const char* e = getenv("MG_GJ_PDL");
        return e ? atoi(e) != 0 : false;
    }();
    return v;
}

// lower triangle -> upper (symmetric Gauss-Jordan: the final state is symmetric)
__global__ void gj_mirror_kernel(double* A, long long n) {
    pdl_begin();
    __shared__ double T[32][33];
    const long long bi = blockIdx.y, bj = blockIdx.x;   // tile (bi, bj) with bi > bj -> (bj, bi)
    if (bj >= bi) return;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    for (int r = ty; r < 32; r += blockDim.x >> 5) {
        const long long i = bi * 32 + r, j = bj * 32 + tx;
        T[r][tx] = (i < n && j < n) ? A[i * n + j] : 0.0;
    }
    __syncthreads();
    for (int r = ty; r < 32; r += blockDim.x >> 5) {
        const long long i = bj * 32 + r, j = bi * 32 + tx;
        if (i < n && j < n) A[i * n + j] = T[tx][r];
    }
}

void dense_spd_inverse(double* A, long long npad, double* work, int* d_status, cudaStream_t s) {
    double* Pb[2] = {work, work + GJ_NB * GJ_NB};   // ping-pong: block k's inverse, next block's
    double* Rrow = work + 2 * GJ_NB * GJ_NB;
    double* Ccol = Rrow + npad * GJ_NB;
    const long long n = npad;
    const bool mma = gj_mma();
    const unsigned nb = (unsigned)((n + 127) / 128);
    for (long long k0 = 0, it = 0; k0 < n; k0 += GJ_NB, ++it) {
        double* P = Pb[it & 1];
        double* Pn = Pb[(it + 1) & 1];
        // the next diagonal block is inverted inside the update kernel when that kernel is long
        // enough to hide it (large coarsest levels), else by its own kernel
        const bool fold = mma && n >= GJ_FOLD_N;
        const bool pdl = gj_pdl();
        const int sym = gj_sym() ? 1 : 0;
        if (!fold || k0 == 0) launch_kp(pdl, gj_diag_kernel, dim3(1), dim3(1024), 0, s, A, n, (int)k0, P, d_status);
        launch_kp(pdl, gj_panels_kernel, dim3(nb, GJ_TQ), dim3(128), 0, s, A, n, n, (int)k0, (const double*)P, Rrow, Ccol,
                  sym);
        dim3 g((unsigned)((n + 63) / 64), (unsigned)((n + 63) / 64));
        const long long kn = (fold && k0 + GJ_NB < n) ? k0 + GJ_NB : -1;
        if (mma) launch_kp(pdl, gj_update_mma_kernel, g, dim3(128), 0, s, A, n, n, (const double*)Ccol, (const double*)Rrow, kn, Pn, d_status, sym);
        else launch_kp(pdl, gj_update_kernel, g, dim3(256), 0, s, A, n, n, (const double*)Ccol, (const double*)Rrow, sym);
        launch_kp(pdl, gj_fix_kernel, dim3(nb, 2 * GJ_TQ), dim3(128), 0, s, A, n, n, (int)k0, (const double*)P,
                  (const double*)Ccol, (const double*)Rrow, sym);
    }
    if (gj_sym()) {
        const unsigned nt = (unsigned)((n + 31) / 32);
        launch_kp(gj_pdl(), gj_mirror_kernel, dim3(nt, nt), dim3(256), 0, s, A, n);
    }
}

// z[q][i] = sum_j Ainv[i][j] r[q][j] for the RB right-hand sides q of this chunk.  A CTA owns
// RW = 32 / RB rows; its 8 warps split the columns, every lane accumulates RW x RB = 32 partial
// sums (one A load per row and one r load per RHS per column: RW RB FMAs per RW + RB loads).
// The 32 per-lane values are reduced across the warp by a transposing butterfly (31 shuffles,
// lane l ends with value l), then across the 8 warps through shared memory.
static constexpr int DA_WARPS = 8;

template <int RB>
__global__ void __launch_bounds__(32 * DA_WARPS) dense_apply_kernel(const double* __restrict__ Ainv, long long ld,
                                                                    long long n, const double* __restrict__ rv,
                                                                    double* __restrict__ z, int R, int r0,
                                                                    const int* active, const int* done) {
    pdl_begin();
    constexpr int RW = 32 / RB;
    __shared__ double red[DA_WARPS][32];
    if (done && *done) return;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const long long i0 = (long long)blockIdx.x * RW;
    const int nr = min(RB, R - r0);
    double v[32];
#pragma unroll
    for (int t = 0; t < 32; ++t) v[t] = 0.0;
    const long long seg = ((n + 32 * DA_WARPS - 1) / (32 * DA_WARPS)) * 32;
    const long long jb = w * seg, je = min(n, jb + seg);
    const int nrow = (int)(n - i0 < RW ? n - i0 : RW);
    const double* row0 = Ainv + i0 * ld;
    for (long long j = jb + lane; j < je; j += 32) {
        double a[RW];
#pragma unroll
        for (int rr = 0; rr < RW; ++rr) a[rr] = rr < nrow ? __ldg(row0 + rr * ld + j) : 0.0;
#pragma unroll
        for (int q = 0; q < RB; ++q) {
            const double x = q < nr ? __ldg(rv + (long long)(r0 + q) * n + j) : 0.0;
#pragma unroll
            for (int rr = 0; rr < RW; ++rr) v[rr * RB + q] = fma(a[rr], x, v[rr * RB + q]);
        }
    }
    // transposing butterfly: after the step with offset o, a lane keeps the half of its values
    // selected by its bit o; lane l finishes with the warp sum of value l
#pragma unroll
    for (int o = 16, cnt = 32; o >= 1; o >>= 1, cnt >>= 1) {
        const bool up = lane & o;
#pragma unroll
        for (int k = 0; k < cnt / 2; ++k) {
            const double send = up ? v[k] : v[k + cnt / 2];
            const double keep = up ? v[k + cnt / 2] : v[k];
            v[k] = keep + __shfl_xor_sync(0xffffffffu, send, o);
        }
    }
    red[w][lane] = v[0];
    __syncthreads();
    if (threadIdx.x < 32) {
        const int t = threadIdx.x, rr = t / RB, q = t % RB;
        double sum = 0.0;
#pragma unroll
        for (int ww = 0; ww < DA_WARPS; ++ww) sum += red[ww][t];
        const long long i = i0 + rr;
        if (i < n && q < nr && (!active || active[r0 + q])) z[(long long)(r0 + q) * n + i] = sum;
    }
}

// Tensor-core variant (default at every size; B200: C2 6.47 -> 6.21, C4 22.6 -> 22.0, C5 179 -> 177
// ms/step against the column-split kernel above): Z^T = Ainv X^T
// with DMMA m8n8k4 tiles -- a CTA owns 8 rows, its 8 warps split the k range, each warp keeps one
// (or two) 8x8 accumulator tiles of (rows x RHS); the partial tiles are summed across the warps in
// shared memory.  ~1k warps in flight instead of RW-row CTAs looping over the columns.
template <int NT>
__global__ void __launch_bounds__(256) dense_apply_mma_kernel(const double* __restrict__ Ainv, long long ld, long long n,
                                                              const double* __restrict__ rv, double* __restrict__ z,
                                                              int R, int r0, const int* active, const int* done) {
    pdl_begin();
    __shared__ double red[8][NT][32][2];
    if (done && *done) return;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const long long i0 = (long long)blockIdx.x * 8;   // i0 + 7 < npad (padded rows are valid memory)
    const long long steps = (n + 3) / 4, per = (steps + 7) / 8;
    const long long kb = w * per * 4, ke = min(n, (w + 1) * per * 4);
    const int gr = lane >> 2, gc = lane & 3;
    const double* arow = Ainv + (i0 + gr) * ld;
    const int rend = min(R, r0 + 8 * NT);
    double acc[NT][2];
#pragma unroll
    for (int t = 0; t < NT; ++t) acc[t][0] = acc[t][1] = 0.0;
#pragma unroll 2
    for (long long k0 = kb; k0 < ke; k0 += 4) {
        const long long kk = k0 + gc;
        const bool kin = kk < n;
        const double a = kin ? __ldg(arow + kk) : 0.0;
#pragma unroll
        for (int t = 0; t < NT; ++t) {
            const int q = r0 + t * 8 + gr;
            const double b = (kin && q < rend) ? __ldg(rv + (long long)q * n + kk) : 0.0;
            dmma(acc[t][0], acc[t][1], a, b);
        }
    }
#pragma unroll
    for (int t = 0; t < NT; ++t) {
        red[w][t][lane][0] = acc[t][0];
        red[w][t][lane][1] = acc[t][1];
    }
    __syncthreads();
    if (w >= NT) return;
    // warp t sums n-tile t over the 8 k-segments; lane holds rows gr, RHS 2 gc + {0, 1}
    const int t = w;
    double v0 = 0.0, v1 = 0.0;
#pragma unroll
    for (int ww = 0; ww < 8; ++ww) {
        v0 += red[ww][t][lane][0];
        v1 += red[ww][t][lane][1];
    }
    const long long i = i0 + gr;
    if (i >= n) return;
    const int qa = r0 + t * 8 + 2 * gc, qb = qa + 1;
    if (qa < rend && (!active || active[qa])) z[(long long)qa * n + i] = v0;
    if (qb < rend && (!active || active[qb])) z[(long long)qb * n + i] = v1;
}

static bool dense_mma() {   // MG_DENSE_MMA=0: column-split DFMA kernel on small levels
    static const bool v = [] {
        const char* e = getenv("MG_DENSE_MMA");
        return e ? atoi(e) != 0 : true;
    }();
    return v;
}


void dense_apply(const double* Ainv, long long ld, long long n, const double* r, double* z, int R, const int* active,
                 const int* done, cudaStream_t s) {
    if (dense_mma()) {
        const unsigned bl = (unsigned)((n + 7) / 8);
        for (int r0 = 0; r0 < R;) {
            if (R - r0 > 8) { launch_k(dense_apply_mma_kernel<2>, dim3(bl), dim3(256), 0, s, Ainv, ld, n, r, z, R, r0, active, done); r0 += 16; }
            else { launch_k(dense_apply_mma_kernel<1>, dim3(bl), dim3(256), 0, s, Ainv, ld, n, r, z, R, r0, active, done); r0 += 8; }
        }
        return;
    }
    for (int r0 = 0; r0 < R;) {
        const int rem = R - r0;
        const int rb = rem > 16 ? 32 : rem > 8 ? 16 : rem > 4 ? 8 : rem > 1 ? 4 : 1;
        const unsigned bl = (unsigned)((n + 32 / rb - 1) / (32 / rb));
        switch (rb) {
            case 32: launch_k(dense_apply_kernel<32>, dim3(bl), dim3(32 * DA_WARPS), 0, s, Ainv, ld, n, r, z, R, r0, active, done); break;
            case 16: launch_k(dense_apply_kernel<16>, dim3(bl), dim3(32 * DA_WARPS), 0, s, Ainv, ld, n, r, z, R, r0, active, done); break;
            case 8: launch_k(dense_apply_kernel<8>, dim3(bl), dim3(32 * DA_WARPS), 0, s, Ainv, ld, n, r, z, R, r0, active, done); break;
            case 4: launch_k(dense_apply_kernel<4>, dim3(bl), dim3(32 * DA_WARPS), 0, s, Ainv, ld, n, r, z, R, r0, active, done); break;
            default: launch_k(dense_apply_kernel<1>, dim3(bl), dim3(32 * DA_WARPS), 0, s, Ainv, ld, n, r, z, R, r0, active, done); break;
        }
        r0 += rb;
    }
}
