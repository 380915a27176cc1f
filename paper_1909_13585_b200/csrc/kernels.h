// Host-side launcher declarations shared by the translation units of libmgcg.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include "common.cuh"

// ---------------------------------------------------------------- fine level (matrix-free)
// FOP_RESTR3: 3D fused residual half of the fine V(1,1) level (h8t.cu), see there (5: retired)
// FOP_GPHI: y = G(u) phi (stress stiffness) on the compact user layout (h8t.cu)
enum FineOp { FOP_MATVEC = 0, FOP_RESID = 1, FOP_JACOBI = 2, FOP_CGP = 3, FOP_RESTR3 = 4, FOP_GPHI = 6 };

struct FineArgs {
    LevelGeom g;
    const double* E;        // nelem
    const uint8_t* mask;    // nnodes, bit k = comp k fixed
    const double* x;        // input vectors (R, ndof)      [MATVEC/RESID/JACOBI]
    const double* z;        // CGP: p_new = z + beta p_in
    const double* pin;
    double* pout;
    const double* b;        // RESID/JACOBI right-hand side
    const double* Dinv;     // JACOBI: ndof
    double* y;              // output vectors (R, ndof)
    double omega;
    const double* beta;     // CGP: per RHS
    double* xv;             // CGP: x += xalpha * p_in at owned nodes (deferred CG update) or NULL
    const double* xalpha;
    const int* active;      // per RHS or NULL
    const int* done;        // or NULL
    double* partial;        // dot partials, RHS r item i at partial[r * pstride + i], or NULL
    long long pstride;
    int R;
    int nu_paper;           // 1: nu == 0.3 -> compile-time K0
    int so0, so1;           // slab-owned local node planes (dots)
    // FOP_RESTR3: r = rin - alpha q (stored to rout), operator input omega D^-1 r, y = r - K(.)
    const double* rin;
    const double* q;
    double* rout;
    const double* alpha;
    double* z1out;          // FOP_RESTR3: omega D^-1 r stored here too (pre-smoothed z1) or NULL
    int ep2;                // 3D: E row pitch (elements along axis 2, even)
    int m2;                 // 3D: mask row pitch (bytes, multiple of 16)
    int goffA, goffB;       // FOP_GPHI: x (phi) / b (u) start this many doubles after a 16-byte boundary
    const double* sig;      // FOP_GPHI: element centroid stresses (nelem x 6, stress_sigma) or NULL (formed from u)
    int z1r;                // FOP_JACOBI: x holds the coarse correction P e only; the sweep's input is
                            // z2 = x + (omega D^-1) b, rounded as the prolongation formed it (MG_Z2_IN_POST)
};

void fine_set_constants(int dim, const double* K0, cudaStream_t s);
// Launch one fine-level layer-march kernel; returns number of dot partial items per RHS.
int fine_apply(int op, const FineArgs& a, cudaStream_t s);
int fine_items(const LevelGeom& g, int R);
void fine_diag(const LevelGeom& g, const double* E, const uint8_t* mask, double* Dinv, double* D, cudaStream_t s);
// 3D structured (sum/difference basis) fine operator, TMA plane-ring march (h8t.cu); fine_apply
// routes 3D here.  Level-0 3D vectors, masks, D^-1 (and E when N2 is odd) use the padded layout:
struct Pad3 {
    int p2;               // nodes per vector row (n2 rounded up to even: 16-byte TMA row strides)
    int m2;               // bytes per mask row (n2 rounded up to 16)
    int ep2;              // elements per E row (N2 rounded up to even)
    long long vstride;    // doubles per RHS vector: 3 n0 n1 p2
};
Pad3 pad3_layout(const LevelGeom& g);
LevelGeom pad3_geom(const LevelGeom& g, const Pad3& p);   // g with p2 / vstr of the padded vectors
void pad3_vectors_planes(const LevelGeom& g, const Pad3& p, int R, const uint8_t* mask, int p0, int np,
                         const double* src, long long src_ndof, double* dst, cudaStream_t s);
void unpad3_vectors_planes(const LevelGeom& g, const Pad3& p, int R, int p0, int np, const double* src, double* dst,
                           long long dst_ndof, cudaStream_t s);
void pad3_nodes(const LevelGeom& g, const Pad3& p, const uint8_t* mask, uint8_t* maskp, const double* dinv,
                double* dinvp, cudaStream_t s);
void pad3_elems(const LevelGeom& g, const Pad3& p, const double* E, double* Ep, cudaStream_t s);
void h8t_set_constants(const double* K0, double nu, cudaStream_t s);
int h8t_apply(int op, const FineArgs& a, cudaStream_t s);
int h8t_items(const LevelGeom& g, int R);
void h8t_chunks(int TR, int minb, int tiles, const LevelGeom& g, int R, int* nch_out, int* hch_out);

// ---------------------------------------------------------------- 2D fused march kernels (fine2d.cu)
enum March2Op { M2_MATVEC = 0, M2_RESID = 1, M2_JACOBI = 2, M2_CGP = 3, M2_RESTRICT = 4, M2_POST = 5 };

// Ghost-padded layout of the 2D fine level used by the march kernels: node (i, j) at
// org + i*pitch + j with one ghost ring (fixed mask, zero E / D^-1 / vectors) plus slack,
// so the kernels load without bounds checks.  Vectors: vstride doubles per RHS.
struct Pad2 {
    int pitch;            // nodes per padded row (n1 + 2)
    long long org;        // padded index of node (0, 0)
    long long nodes;      // padded node count incl. slack
    int pitchE;           // elements per padded row (N1 + 2)
    long long orgE;       // padded index of element (0, 0)
    long long elems;      // padded element count incl. slack
    long long vstride;    // doubles per RHS vector (2 * nodes, rounded to 4)
};

struct March2Args {
    LevelGeom g, gc;              // fine level and next-coarser level (RESTRICT / POST)
    Pad2 pd;                      // padded fine layout (x, x2, xv, y, y2 and E, mask, Dinv below)
    const double* E;              // padded E
    const uint8_t* mask;          // padded node masks (ghosts: 3)
    const double* Dinv;           // padded D^-1 (2 per node; ghosts 0)
    const uint8_t* maskc;         // compact coarse masks
    const double* x;              // MATVEC/RESID/JACOBI: x ; CGP: z ; RESTRICT: r_in ; POST: r
    const double* x2;             // RESID/JACOBI: b ; CGP: p_in ; RESTRICT: q
    double* xv;                   // CGP: x (deferred update x += xalpha p_in)
    double* y;                    // MATVEC/RESID/JACOBI: y ; CGP: q ; POST: z
    double* y2;                   // CGP: p_out ; RESTRICT: r_out
    double* coarse;               // RESTRICT: r_c = P^T t
    const double* ec;             // POST: coarse correction e_c
    double omega;
    const double* alpha;
    const double* beta;
    const double* xalpha;
    const int* active;
    const int* done;
    double* partial;              // dot partials, RHS r item i at partial[r * pstride + i]
    long long pstride;
    int R;
    int so0, so1;                 // slab-owned local node planes [so0, so1): dots and restriction sources
    int off0;                     // 1 if local plane 0 is at an odd global plane (slab ghost), else 0
};
void fine2d_set_constants(const double* K0, cudaStream_t s);
Pad2 pad2_layout(const LevelGeom& g);
// compact <-> padded conversions (2D fine level)
void pad2_nodes_u8(const LevelGeom& g, const Pad2& p, const uint8_t* src, uint8_t* dst, uint8_t fill, cudaStream_t s);
void pad2_nodes_f64(const LevelGeom& g, const Pad2& p, const double* src, double* dst, cudaStream_t s);   // 2 per node
void pad2_elems(const LevelGeom& g, const Pad2& p, const double* src, double* dst, cudaStream_t s);
void pad2_vectors(const LevelGeom& g, const Pad2& p, int R, const uint8_t* mask, const double* src, double* dst,
                  cudaStream_t s);   // compact (R, ndof) -> padded, masked (ghosts untouched)
void unpad2_vectors(const LevelGeom& g, const Pad2& p, int R, const double* src, double* dst, cudaStream_t s);
// slab variants: local planes [p0, p0 + nplanes) <-> compact planes [0, nplanes) of (R, ndof_c) vectors
void pad2_vectors_planes(const LevelGeom& g, const Pad2& p, int R, const uint8_t* mask, int p0, int nplanes,
                         const double* src, long long src_ndof, double* dst, cudaStream_t s);
void unpad2_vectors_planes(const LevelGeom& g, const Pad2& p, int R, int p0, int nplanes, const double* src,
                           double* dst, long long dst_ndof, cudaStream_t s);
int march2_apply(int op, const March2Args& a, bool nu_paper, cudaStream_t s);
int march2_items(int op, const LevelGeom& g, const LevelGeom* gc, int R);

// ---------------------------------------------------------------- coarse levels (assembled stencils)
enum CoarseOp { COP_MATVEC = 0, COP_RESID = 1, COP_JACOBI = 2 };

struct CoarseArgs {
    LevelGeom g;
    const double* st;       // stencil, SoA [3^d*d*d][nnodes]
    const double* x;
    const double* b;
    const double* Dinv;
    double* y;
    double omega;
    const int* active;
    const int* done;
    int R;
};
void coarse_apply(int op, const CoarseArgs& a, cudaStream_t s);

// Galerkin: coarse element matrices from children (level l-1) element matrices, or
// from E_e * K0 when from_E (level 0 children).
void galerkin_set_constants(int dim, const double* K0, cudaStream_t s);
void galerkin_elements(const LevelGeom& gc, const LevelGeom& gf, const double* E /*if from_E*/,
                       const double* elm_f, const uint8_t* mask_f, const uint8_t* mask_c,
                       double* elm_c, cudaStream_t s, int off0 = 0, const double* Mc = nullptr,
                       int* slow_ws = nullptr);
void galerkin_child_matrices(int dim, const double* K0, double* Mc_host);
void elements_from_E(const LevelGeom& g, const double* E, const uint8_t* mask, double* elm, cudaStream_t s);
// identity_fixed: identity rows at fixed DOFs (K); false for G (zero rows/cols)
void stencil_from_elements(const LevelGeom& g, const double* elm, uint8_t* mask, double* st, cudaStream_t s,
                           bool identity_fixed = true);
void galerkin_elements_G(const LevelGeom& gc, const LevelGeom& gf, const double* sig, const uint8_t* mask_f,
                         const uint8_t* mask_c, double* elm_c, cudaStream_t s);
void stencil_diag(const LevelGeom& g, const double* st, uint8_t* mask, double* st_rw, double* Dinv, double* D,
                  cudaStream_t s);

// 2D fused coarse-level V(1,1) halves (coarse2d.cu)
void coarse2d_down(const LevelGeom& g, const LevelGeom& gc, const double* st, const double* Dinv,
                   const uint8_t* mask, const uint8_t* maskc, const double* r, double* rc, int R, double omega,
                   int off0, int fo0, int fo1, const int* active, const int* done, cudaStream_t s);
void coarse2d_up(const LevelGeom& g, const LevelGeom& gc, const double* st, const double* Dinv, const uint8_t* mask,
                 const uint8_t* maskc, const double* r, const double* ec, double* z, int R, double omega, int off0,
                 const int* active, const int* done, cudaStream_t s);

// ---------------------------------------------------------------- transfers
// off0: 1 if the slab's local plane 0 is an (odd-global) ghost plane; [fo0, fo1): slab-owned fine
// planes that contribute to the restriction (fo1 < 0: all).
void restrict_apply(const LevelGeom& gf, const LevelGeom& gc, const uint8_t* mf, const uint8_t* mc,
                    const double* fine, double* coarse, int R, const int* active, const int* done, cudaStream_t s,
                    int off0 = 0, int fo0 = 0, int fo1 = -1);
// rb != NULL (padded 3D fine level, prolong_from_r_ok): fine = omega D^-1 rb + P coarse (the
// pre-smoothed z1 of the fused V-cycle formed from r instead of stored)
void prolong_add(const LevelGeom& gf, const LevelGeom& gc, const uint8_t* mf, const uint8_t* mc,
                 const double* coarse, double* fine, int R, const int* active, const int* done, bool accumulate,
                 cudaStream_t s, int off0 = 0, const double* rb = nullptr, const double* dinv = nullptr,
                 double omega = 0.0);
bool prolong_from_r_ok(const LevelGeom& gf, const LevelGeom& gc, const double* fine);

// ---------------------------------------------------------------- dense coarsest
void dense_from_stencil(const LevelGeom& g, const double* st, double* A, long long ld, cudaStream_t s);
void dense_pad_identity(double* A, long long n, long long npad, cudaStream_t s);
// In-place SPD inverse by blocked Gauss-Jordan (block 32). Work buffers sized npad*32*2 + 32*32.
// Returns via *d_status (device int) nonzero if a non-positive pivot is met.
void dense_spd_inverse(double* A, long long npad, double* work, int* d_status, cudaStream_t s);
int dense_spd_inverse_launches(long long npad);   // kernels dense_spd_inverse launches
void dense_apply(const double* Ainv, long long ld, long long n, const double* r, double* z, int R,
                 const int* active, const int* done, cudaStream_t s);

// ---------------------------------------------------------------- CG vector ops and reductions
int vec_blocks(long long n);
void cg_pointwise_jacobi(long long n, int R, const double* r, const double* Dinv, double omega, double* z,
                         const int* active, const int* done, cudaStream_t s);
void vec_dot(long long n, int R, const double* a, const double* b, double* partial, const int* active,
             const int* done, cudaStream_t s);
// dot over entries [d0, d1) of each RHS; partial[r * pstride + block]; returns the number of blocks
int vec_dot_range(long long n, long long d0, long long d1, int R, const double* a, const double* b, double* partial,
                  long long pstride, const int* active, const int* done, cudaStream_t s);
void vec_mask_copy(long long nnodes, int dim, int R, const uint8_t* mask, const double* src, double* dst,
                   cudaStream_t s);
void vec_axpy_masked_restart(long long n, int R, const double* t, double* r, const int* restart, cudaStream_t s);
// r_out = r_in - alpha q ; partial r_out.r_out over [d0, d1) ; z1 = omega Dinv r_out (z1 may be NULL).
// Returns the number of partial items per RHS.
int cg_rupdate(long long n, int R, const double* alpha, const double* rin, const double* q, double* rout,
               const double* Dinv, double omega, double* z1, double* partial, long long pstride, long long d0,
               long long d1, const int* active, const int* done, cudaStream_t s);
// x += xalpha * p_{xbuf} for every RHS with a pending deferred update
void cg_flush_x(long long n, int R, CgCtl c, const double* p0, const double* p1, double* x, cudaStream_t s);

enum ScalarMode { SM_INIT = 0, SM_ALPHA = 1, SM_CONV = 2, SM_BETA = 3, SM_RZ0 = 4, SM_TRUE = 5, SM_BB = 6 };
void cg_scalars(int mode, int R, const double* partial, int items, CgCtl c, double tol, cudaStream_t s,
                int aux = 0, long long pstride = -1);
void reduce_partials(int R, const double* partial, int items, long long pstride, double* sums, cudaStream_t s);

// ---------------------------------------------------------------- stress stiffness G(u) phi
void stress_set_constants(int dim, double nu, cudaStream_t s);
void stress_sigma(const LevelGeom& g, const double* Es, const double* u, double* sig, cudaStream_t s);
void stress_apply(const LevelGeom& g, const double* sig, const uint8_t* mask, const double* phi, double* y,
                  int nphi, cudaStream_t s);

// ---------------------------------------------------------------- NEXT-1: adjoint RHS, sensitivities (sens.cu)
void sens_set_constants(int dim, const double* K0, double nu, cudaStream_t s);
void adjoint_rhs_apply(const LevelGeom& g, const double* Es, const uint8_t* mask, const double* phi, int nphi,
                       double* w, double* b, cudaStream_t s);
void eigen_sensitivity_apply(const LevelGeom& g, const double* dEk, const double* dEs, const uint8_t* mask,
                             const double* u, const double* phi, const double* z, const double* lam, int nphi,
                             double* out, cudaStream_t s);

// ---------------------------------------------------------------- NEXT-3: block PCG (block.cu)
int gram_blocks(long long n, int R);
void gram(long long n, long long stride, int R, const double* A, const double* B, double* partial, double* G,
          cudaStream_t s);
void block_coef(int R, const double* Gam, const double* Rho, double* C, double thr, int* rank, cudaStream_t s);
void block_axpy(long long n, long long stride, int R, const double* X, const double* C, const double* base, double* Y,
                double sign, cudaStream_t s);
void block_conv(int R, const double* partial, int items, double tol, CgCtl c, cudaStream_t s);
void modes_finish(long long n, int q, double* Phi, const double* KPhi, const double* GPhi, const double* sc,
                  double lam1, double* y1, cudaStream_t s);
