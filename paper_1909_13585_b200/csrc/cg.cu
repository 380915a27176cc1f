// Batched preconditioned CG vector kernels (mgPCG PAPER.md:758,
// multi-RHS :760-761).  Per RHS k:
//   alpha_k = (r.z)_k / (p.q)_k ; x += alpha p ; r -= alpha q ; stop when
//   ||r_k|| <= tol ||b_k|| ; beta_k = (r.z)_new / (r.z)_old ; p = z + beta p.
// Dot products: per-warp shuffle reductions written to a partial array, then
// summed in a fixed order by `cg_scalars` (deterministic, no atomics).
#include <cstdlib>

#include "kernels.h"

bool pdl_enabled() {
    static const bool on = [] {
        const char* e = getenv("MG_PDL");
        return e ? atoi(e) != 0 : true;
    }();
    return on;
}

#define MG_MAX_RHS_DEV 64

static constexpr int VEC_THREADS = 256;

int vec_blocks(long long n) {
    long long b = (n + VEC_THREADS * 4 - 1) / (VEC_THREADS * 4);
    if (b > 1184) b = 1184;   // 8 x 148 SMs
    if (b < 1) b = 1;
    return (int)b;
}

__device__ __forceinline__ void block_partial(double v, double* partial, long long slot) {
    __shared__ double red[VEC_THREADS / 32];
    v = warp_sum(v);
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) red[wid] = v;
    __syncthreads();
    if (wid == 0) {
        double s = lane < (VEC_THREADS / 32) ? red[lane] : 0.0;
        s = warp_sum(s);
        if (lane == 0) partial[slot] = s;
    }
}

// z = omega Dinv r
__global__ void jacobi0_kernel(long long n, const double* __restrict__ r, const double* __restrict__ Dinv,
                               double omega, double* __restrict__ z, const int* active, const int* done) {
    pdl_begin();
    const int rr = blockIdx.y;
    if (done && *done) return;
    if (active && !active[rr]) return;
    const long long o = (long long)rr * n;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        z[o + i] = omega * Dinv[i] * r[o + i];
}

void cg_pointwise_jacobi(long long n, int R, const double* r, const double* Dinv, double omega, double* z,
                         const int* active, const int* done, cudaStream_t s) {
    dim3 g(vec_blocks(n), R);
    launch_kp(false, jacobi0_kernel, dim3(g), dim3(VEC_THREADS), 0, s, n, r, Dinv, omega, z, active, done);
}

// partial[rr * pstride + block] = sum over i in [d0, d1) of a[rr][i] b[rr][i]  (vectors of stride n)
__global__ void __launch_bounds__(VEC_THREADS) dot_kernel(long long n, long long d0, long long d1,
                                                          const double* __restrict__ a,
                                                          const double* __restrict__ b, double* partial,
                                                          long long pstride, const int* active, const int* done) {
    const int rr = blockIdx.y;
    if (done && *done) return;
    if (active && !active[rr]) return;
    const long long o = (long long)rr * n;
    double acc = 0.0;
    for (long long i = d0 + (long long)blockIdx.x * blockDim.x + threadIdx.x; i < d1;
         i += (long long)gridDim.x * blockDim.x)
        acc = fma(a[o + i], b[o + i], acc);
    block_partial(acc, partial, (long long)rr * pstride + blockIdx.x);
}

void vec_dot(long long n, int R, const double* a, const double* b, double* partial, const int* active,
             const int* done, cudaStream_t s) {
    vec_dot_range(n, 0, n, R, a, b, partial, vec_blocks(n), active, done, s);
}

int vec_dot_range(long long n, long long d0, long long d1, int R, const double* a, const double* b, double* partial,
                  long long pstride, const int* active, const int* done, cudaStream_t s) {
    const int nb = vec_blocks(d1 - d0);
    dim3 g(nb, R);
    dot_kernel<<<g, VEC_THREADS, 0, s>>>(n, d0, d1, a, b, partial, pstride, active, done);
    return nb;
}

// dst = src masked to zero at fixed DOFs
__global__ void mask_copy_kernel(long long nnodes, int dim, const uint8_t* __restrict__ mask,
                                 const double* __restrict__ src, double* __restrict__ dst) {
    const int rr = blockIdx.y;
    const long long n = nnodes * dim, o = (long long)rr * n;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const long long node = i / dim;
        const int k = (int)(i - node * dim);
        dst[o + i] = ((mask[node] >> k) & 1) ? 0.0 : src[o + i];
    }
}

void vec_mask_copy(long long nnodes, int dim, int R, const uint8_t* mask, const double* src, double* dst,
                   cudaStream_t s) {
    dim3 g(vec_blocks(nnodes * dim), R);
    mask_copy_kernel<<<g, VEC_THREADS, 0, s>>>(nnodes, dim, mask, src, dst);
}

// r = t for RHS flagged in `restart` (true-residual restart)
__global__ void restart_copy_kernel(long long n, const double* __restrict__ t, double* __restrict__ r,
                                    const int* restart) {
    const int rr = blockIdx.y;
    if (!restart[rr]) return;
    const long long o = (long long)rr * n;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        r[o + i] = t[o + i];
}

void vec_axpy_masked_restart(long long n, int R, const double* t, double* r, const int* restart, cudaStream_t s) {
    dim3 g(vec_blocks(n), R);
    restart_copy_kernel<<<g, VEC_THREADS, 0, s>>>(n, t, r, restart);
}

// One CTA: warp w sums the partials of RHS w, w+16, ... in a fixed order, then
// the scalar CG logic runs per RHS.
__global__ void __launch_bounds__(512) scalars_kernel(int mode, int R, const double* __restrict__ partial, int items,
                                                      long long pstride, CgCtl c, double tol, int aux) {
    pdl_begin();
    __shared__ int any_active;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (threadIdx.x == 0) any_active = 0;
    if (mode != SM_INIT && mode != SM_BB && mode != SM_TRUE && *c.done) return;
    __syncthreads();
    for (int r = wid; r < R; r += blockDim.x >> 5) {
        const bool act = c.active[r] != 0;
        double v = 0.0;
        if (mode == SM_BB || mode == SM_TRUE || act) {
            // four independent chains (fixed order: deterministic, independent of R)
            const double* pr = partial + (long long)r * pstride;
            double v1 = 0.0, v2 = 0.0, v3 = 0.0;
            int i = lane;
            for (; i + 96 < items; i += 128) {
                v += pr[i];
                v1 += pr[i + 32];
                v2 += pr[i + 64];
                v3 += pr[i + 96];
            }
            for (; i < items; i += 32) v += pr[i];
            v = warp_sum((v + v1) + (v2 + v3));
        }
        if (lane == 0) {
            switch (mode) {
                case SM_BB:   // v = b.b ; (re)activate RHS with nonzero b
                    c.bb[r] = v;
                    c.active[r] = v > 0.0 ? 1 : 0;
                    c.iters[r] = 0;
                    c.beta[r] = 0.0;
                    c.alpha[r] = 0.0;
                    c.xalpha[r] = 0.0;
                    c.rr[r] = v;
                    break;
                case SM_RZ0:  // initial r.z
                    if (act) { c.rz[r] = v; c.beta[r] = 0.0; }
                    break;
                case SM_ALPHA:
                    if (act) {
                        c.pq[r] = v;
                        if (!(v > 0.0)) {   // breakdown: operator or preconditioner not SPD
                            c.alpha[r] = 0.0;
                            c.active[r] = 0;
                            atomicOr(c.status, 1);
                        } else {
                            c.alpha[r] = c.rz[r] / v;
                        }
                        c.xalpha[r] = c.alpha[r];   // x += alpha p applied later (deferred)
                        c.xbuf[r] = aux;
                    }
                    break;
                case SM_CONV:
                    if (act) {
                        c.rr[r] = v;
                        c.iters[r] += 1;
                        if (v <= tol * tol * c.bb[r]) c.active[r] = 0;
                    }
                    break;
                case SM_BETA:
                    if (act) {
                        c.beta[r] = v / c.rz[r];
                        c.rz[r] = v;
                    }
                    break;
                case SM_TRUE:
                    c.tt[r] = v;
                    c.xalpha[r] = 0.0;
                    break;
                default:
                    break;
            }
            if (c.active[r]) atomicOr(&any_active, 1);
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) *c.done = any_active ? 0 : 1;
}

void cg_scalars(int mode, int R, const double* partial, int items, CgCtl c, double tol, cudaStream_t s, int aux,
                long long pstride) {
    launch_k(scalars_kernel, dim3(1), dim3(512), 0, s, mode, R, partial, items, pstride < 0 ? items : pstride, c, tol, aux);
}

// sums[r] = sum_i partial[r * pstride + i], i < items (fixed order; multi-rank dots are then
// all-reduced and fed to cg_scalars with items = 1)
__global__ void reduce_partials_kernel(int R, const double* __restrict__ partial, int items, long long pstride,
                                       double* sums) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (int r = wid; r < R; r += blockDim.x >> 5) {
        double v = 0.0;
        for (int i = lane; i < items; i += 32) v += partial[(long long)r * pstride + i];
        v = warp_sum(v);
        if (lane == 0) sums[r] = v;
    }
}

void reduce_partials(int R, const double* partial, int items, long long pstride, double* sums, cudaStream_t s) {
    reduce_partials_kernel<<<1, 512, 0, s>>>(R, partial, items, pstride, sums);
}

// r_out = r_in - alpha q ; partial r.r ; z1 = omega Dinv r_out
__global__ void __launch_bounds__(VEC_THREADS) rupdate_kernel(long long n, const double* __restrict__ alpha,
                                                              const double* __restrict__ rin,
                                                              const double* __restrict__ q, double* __restrict__ rout,
                                                              const double* __restrict__ Dinv, double omega,
                                                              double* __restrict__ z1, double* partial,
                                                              long long pstride, long long d0, long long d1,
                                                              const int* active, const int* done) {
    pdl_begin();
    const int rr = blockIdx.y;
    if (done && *done) return;
    if (active && !active[rr]) return;
    const double al = alpha[rr];
    const long long o = (long long)rr * n;
    double acc = 0.0;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const double v = fma(-al, q[o + i], rin[o + i]);
        rout[o + i] = v;
        if (i >= d0 && i < d1) acc = fma(v, v, acc);
        if (z1) z1[o + i] = omega * Dinv[i] * v;
    }
    block_partial(acc, partial, (long long)rr * pstride + blockIdx.x);
}

int cg_rupdate(long long n, int R, const double* alpha, const double* rin, const double* q, double* rout,
               const double* Dinv, double omega, double* z1, double* partial, long long pstride, long long d0,
               long long d1, const int* active, const int* done, cudaStream_t s) {
    const int nb = vec_blocks(n);
    dim3 g(nb, R);
    launch_kp(false, rupdate_kernel, dim3(g), dim3(VEC_THREADS), 0, s, n, alpha, rin, q, rout, Dinv, omega, z1, partial, pstride, d0, d1,
                                              active, done);
    return nb;
}

__global__ void flush_x_kernel(long long n, CgCtl c, const double* __restrict__ p0, const double* __restrict__ p1,
                               double* __restrict__ x) {
    const int rr = blockIdx.y;
    const double al = c.xalpha[rr];
    if (al == 0.0) return;
    const double* p = c.xbuf[rr] ? p1 : p0;
    const long long o = (long long)rr * n;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        x[o + i] = fma(al, p[o + i], x[o + i]);
}

void cg_flush_x(long long n, int R, CgCtl c, const double* p0, const double* p1, double* x, cudaStream_t s) {
    dim3 g(vec_blocks(n), R);
    flush_x_kernel<<<g, VEC_THREADS, 0, s>>>(n, c, p0, p1, x);
}
