// Coarsest-level direct solve on the device ("dense
// factorization"; the paper's coarsest solve is unstated).
// Setup: the coarsest Galerkin operator (n_L <= a few thousand DOFs) is assembled
// dense and inverted in place by blocked Gauss-Jordan (SPD => no pivoting needed,
// block 32).  Per V-cycle: z = A^-1 r for all R vectors, one warp per row, so the
// solve is a bandwidth-bound dense product instead of a latency-bound triangular
// sweep.
#include "kernels.h"

static constexpr int GJ_NB = 32;

template <int DIM>
__global__ void dense_from_stencil_kernel(LevelGeom g, const double* __restrict__ st, double* A, long long ld) {
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
    long long i = n + blockIdx.x * blockDim.x + threadIdx.x;
    if (i < npad) A[i * npad + i] = 1.0;
}

void dense_pad_identity(double* A, long long n, long long npad, cudaStream_t s) {
    if (npad > n) pad_identity_kernel<<<1, GJ_NB, 0, s>>>(A, n, npad);
}

// In-place Gauss-Jordan inverse of the NB x NB diagonal block k (one CTA, NB*NB threads).
__global__ void gj_diag_kernel(double* A, long long ld, int k0, double* P, int* status) {
    __shared__ double S[GJ_NB][GJ_NB + 1];
    const int i = threadIdx.y, j = threadIdx.x;
    S[i][j] = A[(k0 + i) * ld + k0 + j];
    __syncthreads();
    for (int p = 0; p < GJ_NB; ++p) {
        const double piv = S[p][p];
        const double sip = S[i][p], spj = S[p][j], sij = S[i][j];
        __syncthreads();
        if (!(piv > 0.0)) {
            if (i == 0 && j == 0) atomicOr(status, 2);
        }
        const double ip = 1.0 / piv;
        double v;
        if (i == p && j == p) v = ip;
        else if (i == p) v = spj * ip;
        else if (j == p) v = -sip * ip;
        else v = sij - sip * spj * ip;
        S[i][j] = v;
        __syncthreads();
    }
    P[i * GJ_NB + j] = S[i][j];
}

// Rrow[t][j] = sum_s P[t][s] A[k0+s][j]   (new row panel), Ccol[i][t] = A[i][k0+t] (old column panel)
__global__ void gj_panels_kernel(const double* A, long long ld, long long n, int k0, const double* P, double* Rrow,
                                 double* Ccol) {
    __shared__ double Ps[GJ_NB][GJ_NB];
    const int tid = threadIdx.x;
    for (int e = tid; e < GJ_NB * GJ_NB; e += blockDim.x) Ps[e / GJ_NB][e % GJ_NB] = P[e];
    __syncthreads();
    long long j = (long long)blockIdx.x * blockDim.x + tid;
    if (j >= n) return;
    double col[GJ_NB];
#pragma unroll
    for (int s = 0; s < GJ_NB; ++s) col[s] = A[(k0 + s) * ld + j];
#pragma unroll 4
    for (int t = 0; t < GJ_NB; ++t) {
        double acc = 0.0;
#pragma unroll
        for (int s = 0; s < GJ_NB; ++s) acc = fma(Ps[t][s], col[s], acc);
        Rrow[t * n + j] = acc;
    }
    // column panel: row j of A's column block (A symmetric in exact arithmetic, but
    // read the column explicitly to stay exact for the unsymmetric rounding)
#pragma unroll
    for (int t = 0; t < GJ_NB; ++t) Ccol[j * GJ_NB + t] = A[j * ld + k0 + t];
}

// A[i][j] -= sum_t Ccol[i][t] Rrow[t][j] for all i, j (64x64 tile per CTA, 4x4 per thread).
__global__ void __launch_bounds__(256) gj_update_kernel(double* A, long long ld, long long n, const double* Ccol,
                                                        const double* Rrow) {
    __shared__ double Cs[64][GJ_NB + 1];
    __shared__ double Rs[GJ_NB][64 + 1];
    const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
    const long long i0 = (long long)blockIdx.y * 64, j0 = (long long)blockIdx.x * 64;
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

// Overwrite the pivot column panel: A[i][k] = -Ccol[i] P for rows i outside the pivot block.
__global__ void gj_fix_cols_kernel(double* A, long long ld, long long n, int k0, const double* P, const double* Ccol) {
    __shared__ double Ps[GJ_NB][GJ_NB];
    for (int e = threadIdx.x; e < GJ_NB * GJ_NB; e += blockDim.x) Ps[e / GJ_NB][e % GJ_NB] = P[e];
    __syncthreads();
    long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n || (i >= k0 && i < k0 + GJ_NB)) return;
    double c[GJ_NB];
#pragma unroll
    for (int s = 0; s < GJ_NB; ++s) c[s] = Ccol[i * GJ_NB + s];
#pragma unroll 4
    for (int t = 0; t < GJ_NB; ++t) {
        double acc = 0.0;
#pragma unroll
        for (int s = 0; s < GJ_NB; ++s) acc = fma(c[s], Ps[s][t], acc);
        A[i * ld + k0 + t] = -acc;
    }
}

// Overwrite the pivot row panel: A[k][j] = Rrow (j outside the block), A[k][k] = P.
__global__ void gj_fix_rows_kernel(double* A, long long ld, long long n, int k0, const double* P, const double* Rrow) {
    const long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const int t = blockIdx.y;
    if (j >= n) return;
    A[(k0 + t) * ld + j] = (j >= k0 && j < k0 + GJ_NB) ? P[t * GJ_NB + (j - k0)] : Rrow[t * n + j];
}

void dense_spd_inverse(double* A, long long npad, double* work, int* d_status, cudaStream_t s) {
    double* P = work;
    double* Rrow = work + GJ_NB * GJ_NB;
    double* Ccol = Rrow + npad * GJ_NB;
    const long long n = npad;
    for (long long k0 = 0; k0 < n; k0 += GJ_NB) {
        gj_diag_kernel<<<1, dim3(GJ_NB, GJ_NB), 0, s>>>(A, n, (int)k0, P, d_status);
        gj_panels_kernel<<<(unsigned)((n + 127) / 128), 128, 0, s>>>(A, n, n, (int)k0, P, Rrow, Ccol);
        dim3 g((unsigned)((n + 63) / 64), (unsigned)((n + 63) / 64));
        gj_update_kernel<<<g, 256, 0, s>>>(A, n, n, Ccol, Rrow);
        gj_fix_cols_kernel<<<(unsigned)((n + 127) / 128), 128, 0, s>>>(A, n, n, (int)k0, P, Ccol);
        gj_fix_rows_kernel<<<dim3((unsigned)((n + 255) / 256), GJ_NB), 256, 0, s>>>(A, n, n, (int)k0, P, Rrow);
    }
}

// z[r][i] = sum_j Ainv[i][j] rvec[r][j]: 4 rows per CTA (one warp each), the RB right-hand
// sides staged through shared memory in column chunks so every Ainv row is streamed once and
// the vectors come from shared memory (Ainv and the vectors are L2-resident, n_L <= ~4k).
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

void dense_apply(const double* Ainv, long long ld, long long n, const double* r, double* z, int R, const int* active,
                 const int* done, cudaStream_t s) {
    for (int r0 = 0; r0 < R;) {
        const int rem = R - r0;
        const int rb = rem > 16 ? 32 : rem > 8 ? 16 : rem > 4 ? 8 : rem > 1 ? 4 : 1;
        const unsigned bl = (unsigned)((n + 32 / rb - 1) / (32 / rb));
        switch (rb) {
            case 32: dense_apply_kernel<32><<<bl, 32 * DA_WARPS, 0, s>>>(Ainv, ld, n, r, z, R, r0, active, done); break;
            case 16: dense_apply_kernel<16><<<bl, 32 * DA_WARPS, 0, s>>>(Ainv, ld, n, r, z, R, r0, active, done); break;
            case 8: dense_apply_kernel<8><<<bl, 32 * DA_WARPS, 0, s>>>(Ainv, ld, n, r, z, R, r0, active, done); break;
            case 4: dense_apply_kernel<4><<<bl, 32 * DA_WARPS, 0, s>>>(Ainv, ld, n, r, z, R, r0, active, done); break;
            default: dense_apply_kernel<1><<<bl, 32 * DA_WARPS, 0, s>>>(Ainv, ld, n, r, z, R, r0, active, done); break;
        }
        r0 += rb;
    }
}
