// Block PCG kernels (mgBPCG, "block version of the
// mgPCG", Alg. 2 l.15 :732; O'Leary's block conjugate gradients):
//   gram         G = A^T B for two blocks of R vectors (partials per row chunk + fixed-order sum)
//   block_coef   C = Gamma^+ Rho with a pivoted Cholesky of the SPD R x R Gamma; directions whose
//                pivot falls below a relative threshold are dropped (deflation of dependent or
//                converged columns)
//   block_axpy   Y_j = base_j + sign * sum_k X_k C[k][j]  (all R outputs of a row per thread)
#include "kernels.h"

static constexpr int GR_THREADS = 256;

static int gram_chunk(int R) {   // rows per CTA so that 2 R chunk doubles fit in 64 KB
    int ch = 4096 / R;
    ch = ch >= 256 ? 256 : (ch >= 128 ? 128 : 64);
    return ch;
}

// partial[(i * R + j) * nblk + blk] = sum over the CTA's rows of A_i B_j
__global__ void __launch_bounds__(GR_THREADS) gram_kernel(long long n, long long stride, int R, int ch,
                                                          const double* __restrict__ A, const double* __restrict__ B,
                                                          double* partial) {
    extern __shared__ double sm[];
    double* sA = sm;
    double* sB = sm + (long long)R * ch;
    const long long r0 = (long long)blockIdx.x * ch;
    const int len = (int)(n - r0 < ch ? n - r0 : ch);
    for (int e = threadIdx.x; e < R * ch; e += GR_THREADS) {
        const int k = e / ch, t = e % ch;
        sA[e] = t < len ? A[(long long)k * stride + r0 + t] : 0.0;
        sB[e] = t < len ? B[(long long)k * stride + r0 + t] : 0.0;
    }
    __syncthreads();
    for (int p = threadIdx.x; p < R * R; p += GR_THREADS) {
        const int i = p / R, j = p % R;
        const double* a = sA + (long long)i * ch;
        const double* b = sB + (long long)j * ch;
        double s = 0.0;
        for (int t = 0; t < len; ++t) s = fma(a[t], b[t], s);
        partial[(long long)p * gridDim.x + blockIdx.x] = s;
    }
}

__global__ void gram_reduce_kernel(int R, int nblk, const double* __restrict__ partial, double* G) {
    const int lane = threadIdx.x & 31;
    for (int p = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); p < R * R; p += gridDim.x * (blockDim.x >> 5)) {
        double s = 0.0;
        for (int b = lane; b < nblk; b += 32) s += partial[(long long)p * nblk + b];
        s = warp_sum(s);
        if (lane == 0) G[p] = s;
    }
}

int gram_blocks(long long n, int R) { return (int)((n + gram_chunk(R) - 1) / gram_chunk(R)); }

void gram(long long n, long long stride, int R, const double* A, const double* B, double* partial, double* G,
          cudaStream_t s) {
    const int ch = gram_chunk(R);
    const int nblk = (int)((n + ch - 1) / ch);
    const size_t smem = sizeof(double) * 2 * R * ch;
    static bool attr = [] {
        cudaFuncSetAttribute(gram_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
        return true;
    }();
    (void)attr;
    gram_kernel<<<nblk, GR_THREADS, smem, s>>>(n, stride, R, ch, A, B, partial);
    gram_reduce_kernel<<<(R * R + 7) / 8, 256, 0, s>>>(R, nblk, partial, G);
}

// One CTA.  Pivoted Cholesky Gamma[piv][piv] = L L^T over the pivots whose remaining diagonal
// stays above thr * max(diag); C = Gamma^+ Rho on those rows, 0 on the dropped ones.
// rank_out (device int) receives the rank.
__global__ void block_coef_kernel(int R, const double* __restrict__ Gam, const double* __restrict__ Rho, double* C,
                                  double thr, int* rank_out) {
    __shared__ double A[64][65];
    __shared__ int piv[64];
    __shared__ int rank;
    const int tid = threadIdx.x;
    for (int e = tid; e < R * R; e += blockDim.x) A[e / R][e % R] = Gam[e];
    __syncthreads();
    if (tid == 0) {
        double dmax = 0.0;
        for (int i = 0; i < R; ++i) dmax = fmax(dmax, A[i][i]);
        int used[64];
        for (int i = 0; i < R; ++i) used[i] = 0;
        int r = 0;
        // right-looking pivoted Cholesky (R <= 64: serial is a few microseconds)
        for (int k = 0; k < R; ++k) {
            int best = -1;
            double bv = 0.0;
            for (int i = 0; i < R; ++i)
                if (!used[i] && A[i][i] > bv) { bv = A[i][i]; best = i; }
            if (best < 0 || !(bv > thr * dmax)) break;
            used[best] = 1;
            piv[r] = best;
            const double l = sqrt(bv);
            A[best][best] = l;
            for (int i = 0; i < R; ++i)
                if (!used[i]) A[i][best] /= l;
            for (int i = 0; i < R; ++i) {
                if (used[i]) continue;
                for (int j = 0; j <= i; ++j)
                    if (!used[j]) {
                        A[i][j] -= A[i][best] * A[j][best];
                        A[j][i] = A[i][j];
                    }
            }
            ++r;
        }
        rank = r;
        *rank_out = r;
    }
    __syncthreads();
    const int r = rank;
    // solve for every RHS column c: L y = Rho[piv][c], L^T x = y (L stored at A[piv[i]][piv[j]], i >= j)
    for (int c = tid; c < R; c += blockDim.x) {
        double y[64];
        for (int i = 0; i < r; ++i) {
            double v = Rho[piv[i] * R + c];
            for (int j = 0; j < i; ++j) v -= A[piv[i]][piv[j]] * y[j];
            y[i] = v / A[piv[i]][piv[i]];
        }
        for (int i = r - 1; i >= 0; --i) {
            double v = y[i];
            for (int j = i + 1; j < r; ++j) v -= A[piv[j]][piv[i]] * y[j];
            y[i] = v / A[piv[i]][piv[i]];
        }
        for (int i = 0; i < R; ++i) C[i * R + c] = 0.0;
        for (int i = 0; i < r; ++i) C[piv[i] * R + c] = y[i];
    }
}

void block_coef(int R, const double* Gam, const double* Rho, double* C, double thr, int* rank, cudaStream_t s) {
    block_coef_kernel<<<1, 64, 0, s>>>(R, Gam, Rho, C, thr, rank);
}

// Y[j][i] = (base ? base[j][i] : Y[j][i]) + sign * sum_k X[k][i] C[k][j]; every row's X values are
// read before its Y values are written, so Y may alias X
template <int RB>
__global__ void block_axpy_kernel(long long n, long long stride, int R, const double* __restrict__ X,
                                  const double* __restrict__ C, const double* base, double* Y, double sign) {
    __shared__ double Cs[RB * RB];
    for (int e = threadIdx.x; e < RB * RB; e += blockDim.x) {
        const int k = e / RB, j = e % RB;
        Cs[e] = (k < R && j < R) ? C[k * R + j] : 0.0;
    }
    __syncthreads();
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        double xv[RB];
#pragma unroll
        for (int k = 0; k < RB; ++k) xv[k] = k < R ? X[(long long)k * stride + i] : 0.0;
#pragma unroll
        for (int j = 0; j < RB; ++j) {
            if (j >= R) break;
            double s = 0.0;
#pragma unroll
            for (int k = 0; k < RB; ++k) s = fma(xv[k], Cs[k * RB + j], s);
            const long long o = (long long)j * stride + i;
            Y[o] = fma(sign, s, base ? base[o] : Y[o]);
        }
    }
}

// R > 16: the row's X values are staged in shared memory instead of registers (no spills; Y may
// still alias X: a thread reads its whole row before writing it)
static constexpr int BAX_T = 128;
__global__ void __launch_bounds__(BAX_T) block_axpy_smem_kernel(long long n, long long stride, int R,
                                                                const double* __restrict__ X,
                                                                const double* __restrict__ C, const double* base,
                                                                double* Y, double sign) {
    extern __shared__ double bax_sm[];
    double* Cs = bax_sm;               // R x R
    double* xs = bax_sm + R * R;       // R x BAX_T
    for (int e = threadIdx.x; e < R * R; e += blockDim.x) Cs[e] = C[e];
    __syncthreads();
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        for (int k = 0; k < R; ++k) xs[k * BAX_T + threadIdx.x] = X[(long long)k * stride + i];
        for (int j = 0; j < R; ++j) {
            double s0 = 0.0, s1 = 0.0;
            int k = 0;
            for (; k + 1 < R; k += 2) {
                s0 = fma(xs[k * BAX_T + threadIdx.x], Cs[k * R + j], s0);
                s1 = fma(xs[(k + 1) * BAX_T + threadIdx.x], Cs[(k + 1) * R + j], s1);
            }
            if (k < R) s0 = fma(xs[k * BAX_T + threadIdx.x], Cs[k * R + j], s0);
            const long long o = (long long)j * stride + i;
            Y[o] = fma(sign, s0 + s1, base ? base[o] : Y[o]);
        }
    }
}

void block_axpy(long long n, long long stride, int R, const double* X, const double* C, const double* base, double* Y,
                double sign, cudaStream_t s) {
    long long bl = (n + 255) / 256;
    if (bl > 148 * 8) bl = 148 * 8;
    if (R <= 8) block_axpy_kernel<8><<<(unsigned)bl, 256, 0, s>>>(n, stride, R, X, C, base, Y, sign);
    else if (R <= 16) block_axpy_kernel<16><<<(unsigned)bl, 256, 0, s>>>(n, stride, R, X, C, base, Y, sign);
    else {
        const size_t smem = sizeof(double) * ((size_t)R * R + (size_t)R * BAX_T);
        static bool attr = [] {
            cudaFuncSetAttribute(block_axpy_smem_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
            return true;
        }();
        (void)attr;
        long long b2 = (n + BAX_T - 1) / BAX_T;
        if (b2 > 148 * 4) b2 = 148 * 4;
        block_axpy_smem_kernel<<<(unsigned)b2, BAX_T, smem, s>>>(n, stride, R, X, C, base, Y, sign);
    }
}

// per-column convergence of the block solve: rr[k] <= tol^2 bb[k] for all k -> *done = 1;
// iters[k] += 1 for columns not yet converged before this iteration
__global__ void block_conv_kernel(int R, const double* __restrict__ partial, int items, double tol, CgCtl c) {
    __shared__ int all;
    if (threadIdx.x == 0) all = 1;
    __syncthreads();
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int r = w; r < R; r += blockDim.x >> 5) {
        double v = 0.0;
        for (int i = lane; i < items; i += 32) v += partial[(long long)r * items + i];
        v = warp_sum(v);
        if (lane == 0) {
            if (c.active[r]) c.iters[r] += 1;
            c.rr[r] = v;
            const bool conv = v <= tol * tol * c.bb[r];
            c.active[r] = conv ? 0 : 1;
            if (!conv) atomicAnd(&all, 0);
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) *c.done = all;
}

void block_conv(int R, const double* partial, int items, double tol, CgCtl c, cudaStream_t s) {
    block_conv_kernel<<<1, 512, 0, s>>>(R, partial, items, tol, c);
}

// ---------------------------------------------------------------- NEXT-2 mode post-processing
// Phi_i *= s_i (K normalisation) and, if y1, the Eq. 7 residual of the first pair
// y1 = s_0 (K phi_0 + lambda_1 G phi_0) = (K + lambda~_1 G) phi~_1.
__global__ void modes_finish_kernel(long long n, int q, double* Phi, const double* KPhi, const double* GPhi,
                                    const double* sc, double lam1, double* y1) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    for (int k = 0; k < q; ++k) Phi[(long long)k * n + i] *= sc[k];
    if (y1) y1[i] = sc[0] * fma(lam1, GPhi[i], KPhi[i]);
}

void modes_finish(long long n, int q, double* Phi, const double* KPhi, const double* GPhi, const double* sc,
                  double lam1, double* y1, cudaStream_t s) {
    modes_finish_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(n, q, Phi, KPhi, GPhi, sc, lam1, y1);
}
