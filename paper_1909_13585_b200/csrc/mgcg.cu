// C-ABI host side of libmgcg: handle, hierarchy setup, CUDA-graph solve loop.
// See include/mgcg.h for the contract and the paper passages each call follows.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/mgcg.h"
#include "element.cuh"
#include "kernels.h"

// ---------------------------------------------------------------- error plumbing
static thread_local std::string g_last_error;

static mg_status fail(mg_status s, const std::string& msg) {
    g_last_error = msg;
    return s;
}

#define CU(call)                                                                                  \
    do {                                                                                          \
        cudaError_t e_ = (call);                                                                  \
        if (e_ != cudaSuccess)                                                                    \
            return fail(e_ == cudaErrorMemoryAllocation ? MG_ERR_OOM : MG_ERR_CUDA,               \
                        std::string(#call) + ": " + cudaGetErrorString(e_));                      \
    } while (0)

#define CHECK_LAUNCH()                                                                            \
    do {                                                                                          \
        cudaError_t e_ = cudaGetLastError();                                                      \
        if (e_ != cudaSuccess) return fail(MG_ERR_CUDA, std::string("launch: ") + cudaGetErrorString(e_)); \
    } while (0)

#define TRY(expr)                        \
    do {                                 \
        mg_status s_ = (expr);           \
        if (s_ != MG_OK) return s_;      \
    } while (0)

// ---------------------------------------------------------------- element stiffness (host)
// K0[(a,i),(b,j)] = lam S_ij + mu S_ji + mu delta_ij sum_k S_kk with
// S_ij[a,b] = int dN_a/dx_i dN_b/dx_j over the unit element, a product of 1-D
// integrals (M, D, C on [0,1]); lam = E nu/(1-nu^2) in plane stress (2D),
// E nu/((1+nu)(1-2nu)) in 3D; mu = E/(2(1+nu)).  Equals exact 2x2(x2) Gauss of
// B^T D0 B (standard Q4/H8, PAPER.md:111 reading r1).  Local DOF = d*a + comp,
// local node a in C order (axis 0 most significant).
static void element_stiffness(int dim, double nu, std::vector<double>& K) {
    const int nl = dim * (1 << dim);
    K.assign(nl * nl, 0.0);
    for (int r = 0; r < nl; ++r)
        for (int c = 0; c < nl; ++c) K[r * nl + c] = dim == 2 ? k0_entry<2>(nu, r, c) : k0_entry<3>(nu, r, c);
}

// ---------------------------------------------------------------- small kernels
__global__ void fixed_to_mask_kernel(long long nnodes, int dim, const uint8_t* fixed, uint8_t* mask) {
    long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nnodes) return;
    int m = 0;
    for (int k = 0; k < dim; ++k) m |= (fixed[dim * i + k] ? 1 : 0) << k;
    mask[i] = (uint8_t)m;
}

__global__ void coarse_mask_kernel(LevelGeom gf, LevelGeom gc, const uint8_t* mf, uint8_t* mc) {
    long long I = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (I >= gc.nnodes) return;
    long long t = I, q = 0;
    int ci[3] = {0, 0, 0};
    for (int k = gc.dim - 1; k >= 0; --k) { ci[k] = (int)(t % gc.nn[k]); t /= gc.nn[k]; }
    for (int k = 0; k < gc.dim; ++k) q = q * gf.nn[k] + 2 * ci[k];
    mc[I] = mf[q];
}

__global__ void check_modulus_kernel(long long n, const double* E, int* bad) {
    long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double v = E[i];
    if (!(v > 0.0) || !isfinite(v)) atomicOr(bad, 1);
}

// ---------------------------------------------------------------- handle
struct Level {
    LevelGeom g;
    uint8_t* mask = nullptr;
    double* Dinv = nullptr;
    double* D = nullptr;
    double* st = nullptr;     // stencil (coarse levels; level 0 only when L == 1)
    double* r = nullptr;      // vectors (levels >= 1), R x ndof
    double* z = nullptr;
    double* w = nullptr;
};

struct mg_ctx {
    int dim = 0, L = 0;
    double nu = 0.3;
    bool nu_paper = true;     // nu == 0.3: compile-time K0 in the fine kernels
    bool fused2d = false;     // 2D, L >= 2, V(1,1): fused RESTRICT / POST fine kernels
    mg_opts opts{0.6, 1, 1, 1000};
    cudaStream_t user = nullptr, stream = nullptr;
    cudaEvent_t ev_in = nullptr, ev_out = nullptr;
    Level lv[MG_MAX_LEVELS];
    double* E = nullptr;
    std::vector<double> K0;
    // 2D fine level: ghost-padded copies used by the march kernels (fine2d.cu)
    Pad2 pd{};
    double* Epad = nullptr;
    uint8_t* maskpad = nullptr;
    double* Dinvpad = nullptr;
    long long vs = 0;         // doubles per RHS of a level-0 vector (padded in 2D, ndof in 3D)
    // coarsest dense inverse
    double* Ainv = nullptr;
    long long nL = 0, npad = 0;
    // fine vectors (R x ndof each)
    int Ralloc = 0;
    double *b = nullptr, *x = nullptr, *r0 = nullptr, *r1 = nullptr, *p0 = nullptr, *p1 = nullptr, *q = nullptr,
           *zf = nullptr, *z = nullptr, *t = nullptr;
    double* zpre = nullptr;   // generic path: buffer holding the pre-smoothed z after blk_restrict
    double *stage = nullptr, *stage2 = nullptr;   // compact (R x ndof) staging: host copies, 2D L == 1 solve
    double* partial = nullptr;
    long long partial_cap = 0;
    // CG control block
    CgCtl ctl{};
    void* ctl_mem = nullptr;
    int* h_pinned = nullptr;     // done, status, iters[64]
    double* h_dbl = nullptr;     // bb, rr, tt [64] each
    int* d_status = nullptr;
    // graphs
    cudaGraphExec_t g_init = nullptr, g_restart = nullptr, g_iter = nullptr, g_true = nullptr;
    long long n_init = 0, n_restart = 0, n_iter = 0, n_true = 0;
    int graph_R = -1;
    double graph_tol = -1.0;
    // stress
    double* sig = nullptr;
    // stats
    long long launches = 0;
};

static const LevelGeom& G0(mg_ctx* c) { return c->lv[0].g; }

static LevelGeom make_geom(int dim, const int* N) {
    LevelGeom g{};
    g.dim = dim;
    g.nnodes = 1;
    g.nelem = 1;
    for (int k = 0; k < 3; ++k) {
        g.N[k] = k < dim ? N[k] : 1;
        g.nn[k] = k < dim ? N[k] + 1 : 1;
        if (k < dim) { g.nnodes *= g.nn[k]; g.nelem *= g.N[k]; }
    }
    g.ndof = g.nnodes * dim;
    return g;
}

static bool is_device_ptr(const void* p) {
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

static void stream_enter(mg_ctx* c) {
    cudaEventRecord(c->ev_in, c->user);
    cudaStreamWaitEvent(c->stream, c->ev_in, 0);
}
static void stream_leave(mg_ctx* c) {
    cudaEventRecord(c->ev_out, c->stream);
    cudaStreamWaitEvent(c->user, c->ev_out, 0);
}

// ---------------------------------------------------------------- operators (per design)
static mg_status compute_operators(mg_ctx* c) {
    cudaStream_t s = c->stream;
    const int L = c->L, dim = c->dim;
    TRY(([&]() -> mg_status {
        CU(cudaMemsetAsync(c->d_status, 0, sizeof(int), s));
        long long m = G0(c).nelem;
        check_modulus_kernel<<<(unsigned)((m + 255) / 256), 256, 0, s>>>(m, c->E, c->d_status);
        CHECK_LAUNCH();
        int bad = 0;
        CU(cudaMemcpyAsync(&bad, c->d_status, sizeof(int), cudaMemcpyDeviceToHost, s));
        CU(cudaStreamSynchronize(s));
        if (bad) return fail(MG_ERR_MODULUS, "E_e must be positive and finite");
        return MG_OK;
    }()));
    fine_diag(G0(c), c->E, c->lv[0].mask, c->lv[0].Dinv, c->lv[0].D, s);
    c->launches += 2;
    if (dim == 2) {
        pad2_elems(G0(c), c->pd, c->E, c->Epad, s);
        pad2_nodes_u8(G0(c), c->pd, c->lv[0].mask, c->maskpad, 3, s);
        pad2_nodes_f64(G0(c), c->pd, c->lv[0].Dinv, c->Dinvpad, s);
        c->launches += 3;
    }
    CHECK_LAUNCH();
    const int NL = dim * (1 << dim);
    double* elm_prev = nullptr;
    if (L == 1) {
        CU(cudaMallocAsync(&elm_prev, sizeof(double) * G0(c).nelem * NL * NL, s));
        elements_from_E(G0(c), c->E, c->lv[0].mask, elm_prev, s);
        stencil_from_elements(G0(c), elm_prev, c->lv[0].mask, c->lv[0].st, s);
        c->launches += 2;
        CHECK_LAUNCH();
    }
    for (int l = 1; l < L; ++l) {
        Level& f = c->lv[l - 1];
        Level& g = c->lv[l];
        double* elm = nullptr;
        CU(cudaMallocAsync(&elm, sizeof(double) * g.g.nelem * NL * NL, s));
        galerkin_elements(g.g, f.g, l == 1 ? c->E : nullptr, elm_prev, f.mask, g.mask, elm, s);
        CHECK_LAUNCH();
        if (elm_prev) CU(cudaFreeAsync(elm_prev, s));
        elm_prev = elm;
        stencil_from_elements(g.g, elm, g.mask, g.st, s);
        stencil_diag(g.g, g.st, g.mask, g.st, g.Dinv, g.D, s);
        c->launches += 3;
        CHECK_LAUNCH();
    }
    if (elm_prev) CU(cudaFreeAsync(elm_prev, s));
    // coarsest dense inverse
    Level& cl = c->lv[L - 1];
    CU(cudaMemsetAsync(c->Ainv, 0, sizeof(double) * c->npad * c->npad, s));
    dense_from_stencil(cl.g, cl.st, c->Ainv, c->npad, s);
    dense_pad_identity(c->Ainv, c->nL, c->npad, s);
    double* work = nullptr;
    CU(cudaMallocAsync(&work, sizeof(double) * (32 * 32 + 2 * c->npad * 32), s));
    CU(cudaMemsetAsync(c->d_status, 0, sizeof(int), s));
    dense_spd_inverse(c->Ainv, c->npad, work, c->d_status, s);
    c->launches += 2 + 5 * (c->npad / 32);
    CHECK_LAUNCH();
    CU(cudaFreeAsync(work, s));
    int st = 0;
    CU(cudaMemcpyAsync(&st, c->d_status, sizeof(int), cudaMemcpyDeviceToHost, s));
    CU(cudaStreamSynchronize(s));
    if (st) return fail(MG_ERR_SINGULAR, "coarsest operator: non-positive pivot in the SPD inverse");
    return MG_OK;
}

static void free_vectors(mg_ctx* c) {
    double** fv[] = {&c->b, &c->x, &c->r0, &c->r1, &c->p0, &c->p1, &c->q, &c->zf, &c->z, &c->t, &c->partial,
                     &c->stage, &c->stage2};
    for (auto p : fv)
        if (*p) { cudaFree(*p); *p = nullptr; }
    for (int l = 1; l < c->L; ++l) {
        double** lvv[] = {&c->lv[l].r, &c->lv[l].z, &c->lv[l].w};
        for (auto p : lvv)
            if (*p) { cudaFree(*p); *p = nullptr; }
    }
    cudaGraphExec_t* gs[] = {&c->g_init, &c->g_restart, &c->g_iter, &c->g_true};
    for (auto g : gs)
        if (*g) { cudaGraphExecDestroy(*g); *g = nullptr; }
    c->graph_R = -1;
    c->Ralloc = 0;
}

static mg_status ensure_vectors(mg_ctx* c, int R) {
    if (R <= c->Ralloc) return MG_OK;
    CU(cudaStreamSynchronize(c->stream));
    free_vectors(c);
    const long long n = c->vs;
    double** fv[] = {&c->b, &c->x, &c->r0, &c->r1, &c->p0, &c->p1, &c->q, &c->zf, &c->z, &c->t};
    for (auto p : fv) {
        CU(cudaMalloc(p, sizeof(double) * n * R));
        CU(cudaMemset(*p, 0, sizeof(double) * n * R));   // ghost entries of the padded layout stay 0
    }
    CU(cudaMalloc(&c->stage, sizeof(double) * G0(c).ndof * R));
    CU(cudaMalloc(&c->stage2, sizeof(double) * G0(c).ndof * R));
    for (int l = 1; l < c->L; ++l) {
        long long nl = c->lv[l].g.ndof;
        CU(cudaMalloc(&c->lv[l].r, sizeof(double) * nl * R));
        CU(cudaMalloc(&c->lv[l].z, sizeof(double) * nl * R));
        CU(cudaMalloc(&c->lv[l].w, sizeof(double) * nl * R));
    }
    long long items = fine_items(G0(c));
    if (c->dim == 2) {
        for (int op : {M2_CGP, M2_RESTRICT, M2_POST, M2_RESID}) {
            long long it = march2_items(op, G0(c), c->L > 1 ? &c->lv[1].g : &c->lv[0].g);
            items = it > items ? it : items;
        }
    }
    long long vb = vec_blocks(n);
    c->partial_cap = (items > vb ? items : vb) * (long long)R;
    CU(cudaMalloc(&c->partial, sizeof(double) * c->partial_cap));
    c->Ralloc = R;
    return MG_OK;
}

// ---------------------------------------------------------------- recording helpers
struct Rec {
    mg_ctx* c;
    int R;
    const int* active;
    const int* done;
    long long launches = 0;
};

static FineArgs fine_args(mg_ctx* c, const Rec& rc) {
    FineArgs a{};
    a.g = G0(c); a.E = c->E; a.mask = c->lv[0].mask; a.omega = c->opts.omega;
    a.active = rc.active; a.done = rc.done; a.R = rc.R; a.nu_paper = c->nu_paper ? 1 : 0;
    return a;
}

// Level-0 operator application: 2D through the padded march kernels, 3D through fine_ops.
static int level0_apply(mg_ctx* c, int op, const FineArgs& f) {
    if (c->dim != 2) return fine_apply(op, f, c->stream);
    March2Args m{};
    m.g = G0(c);
    if (c->L > 1) { m.gc = c->lv[1].g; m.maskc = c->lv[1].mask; }
    m.pd = c->pd; m.E = c->Epad; m.mask = c->maskpad; m.Dinv = c->Dinvpad;
    m.omega = f.omega; m.active = f.active; m.done = f.done; m.partial = f.partial; m.R = f.R;
    int mop;
    switch (op) {
        case FOP_MATVEC: mop = M2_MATVEC; m.x = f.x; m.y = f.y; break;
        case FOP_RESID: mop = M2_RESID; m.x = f.x; m.x2 = f.b; m.y = f.y; break;
        case FOP_JACOBI: mop = M2_JACOBI; m.x = f.x; m.x2 = f.b; m.y = f.y; break;
        default:
            mop = M2_CGP; m.x = f.z; m.x2 = f.pin; m.y2 = f.pout; m.y = f.y; m.beta = f.beta;
            m.xv = f.xv; m.xalpha = f.xalpha;
            break;
    }
    return march2_apply(mop, m, c->nu_paper, c->stream);
}

static void level_smooth(Rec& rc, int l, const double* r, const double* z, double* w, double* partial) {
    mg_ctx* c = rc.c;
    if (l == 0 && c->L > 1) {
        FineArgs a = fine_args(c, rc);
        a.x = z; a.b = r; a.Dinv = c->lv[0].Dinv; a.y = w; a.partial = partial;
        level0_apply(c, FOP_JACOBI, a);
    } else {
        CoarseArgs a{};
        a.g = c->lv[l].g; a.st = c->lv[l].st; a.x = z; a.b = r; a.Dinv = c->lv[l].Dinv; a.y = w;
        a.omega = c->opts.omega; a.active = rc.active; a.done = rc.done; a.R = rc.R;
        coarse_apply(COP_JACOBI, a, c->stream);
    }
    rc.launches++;
}

static void level_resid(Rec& rc, int l, const double* r, const double* z, double* w) {
    mg_ctx* c = rc.c;
    if (l == 0) {
        FineArgs a = fine_args(c, rc);
        a.x = z; a.b = r; a.y = w;
        level0_apply(c, FOP_RESID, a);
    } else {
        CoarseArgs a{};
        a.g = c->lv[l].g; a.st = c->lv[l].st; a.x = z; a.b = r; a.y = w;
        a.active = rc.active; a.done = rc.done; a.R = rc.R;
        coarse_apply(COP_RESID, a, c->stream);
    }
    rc.launches++;
}

// Symmetric V(nu_pre, nu_post)-cycle on level l (generic kernels): z ~ A_l^-1 r.  Returns
// the buffer holding z (z or w).  Used for levels >= 1 in the solve and for mg_vcycle.
static double* vcycle(Rec& rc, int l, const double* r, double* z, double* w) {
    mg_ctx* c = rc.c;
    const Level& lv = c->lv[l];
    const int R = rc.R;
    if (l == c->L - 1) {
        dense_apply(c->Ainv, c->npad, c->nL, r, z, R, rc.active, rc.done, c->stream);
        rc.launches++;
        return z;
    }
    cg_pointwise_jacobi(lv.g.ndof, R, r, lv.Dinv, c->opts.omega, z, rc.active, rc.done, c->stream);
    rc.launches++;
    for (int s = 1; s < c->opts.nu_pre; ++s) {
        level_smooth(rc, l, r, z, w, nullptr);
        std::swap(z, w);
    }
    level_resid(rc, l, r, z, w);
    const Level& nx = c->lv[l + 1];
    restrict_apply(lv.g, nx.g, lv.mask, nx.mask, w, nx.r, R, rc.active, rc.done, c->stream);
    rc.launches++;
    double* zc = vcycle(rc, l + 1, nx.r, nx.z, nx.w);
    prolong_add(lv.g, nx.g, lv.mask, nx.mask, zc, z, R, rc.active, rc.done, true, c->stream);
    rc.launches++;
    for (int s = 0; s < c->opts.nu_post; ++s) {
        level_smooth(rc, l, r, z, w, nullptr);
        std::swap(z, w);
    }
    return z;
}

// ---- fine-level blocks of one CG iteration (fused kernels in 2D, composed kernels otherwise)
static March2Args march_args(mg_ctx* c, const Rec& rc) {
    March2Args a{};
    a.g = G0(c);
    if (c->L > 1) { a.gc = c->lv[1].g; a.maskc = c->lv[1].mask; }
    a.pd = c->pd; a.E = c->Epad; a.mask = c->maskpad; a.Dinv = c->Dinvpad; a.omega = c->opts.omega;
    a.alpha = c->ctl.alpha; a.beta = c->ctl.beta; a.xalpha = c->ctl.xalpha;
    a.active = rc.active; a.done = rc.done; a.R = rc.R;
    return a;
}

// p_out = zf + beta p_in ; q = K p_out ; partial p.q ; x += xalpha p_in.  Returns partial items.
static int blk_cgp(Rec& rc, const double* pin, double* pout) {
    mg_ctx* c = rc.c;
    rc.launches++;
    FineArgs a = fine_args(c, rc);
    a.z = c->zf; a.pin = pin; a.pout = pout; a.y = c->q; a.beta = c->ctl.beta;
    a.xv = c->x; a.xalpha = c->ctl.xalpha; a.partial = c->partial;
    return level0_apply(c, FOP_CGP, a);
}

// r_out = r_in - alpha q ; partial r.r ; pre-smooth z1 = omega D^-1 r_out ; r_1 = P^T (r_out - K z1)
static int blk_restrict(Rec& rc, const double* rin, double* rout) {
    mg_ctx* c = rc.c;
    const long long n = c->vs;
    if (c->fused2d) {
        March2Args a = march_args(c, rc);
        a.x = rin; a.x2 = c->q; a.y2 = rout; a.coarse = c->lv[1].r; a.partial = c->partial;
        rc.launches++;
        return march2_apply(M2_RESTRICT, a, c->nu_paper, c->stream);
    }
    cg_rupdate(n, rc.R, c->ctl.alpha, rin, c->q, rout, c->dim == 2 ? c->Dinvpad : c->lv[0].Dinv, c->opts.omega,
               c->L > 1 ? c->z : nullptr,
               c->partial, rc.active, rc.done, c->stream);
    rc.launches++;
    const int items = vec_blocks(n);
    if (c->L == 1) return items;
    double *z = c->z, *w = c->t;
    for (int s = 1; s < c->opts.nu_pre; ++s) {
        level_smooth(rc, 0, rout, z, w, nullptr);
        std::swap(z, w);
    }
    level_resid(rc, 0, rout, z, w);
    restrict_apply(G0(c), c->lv[1].g, c->lv[0].mask, c->lv[1].mask, w, c->lv[1].r, rc.R, rc.active, rc.done,
                   c->stream);
    rc.launches++;
    c->zpre = z;
    return items;
}

// levels 1..L-1 of the V-cycle on lv[1].r; returns the level-1 correction buffer
static double* coarse_cycle(Rec& rc) {
    mg_ctx* c = rc.c;
    if (c->L == 1) return nullptr;
    return vcycle(rc, 1, c->lv[1].r, c->lv[1].z, c->lv[1].w);
}

// zf = post-smoothed (z1 + P ec) ; partial r.zf.  Returns partial items.
static int blk_post(Rec& rc, const double* r, const double* ec) {
    mg_ctx* c = rc.c;
    const long long n = c->vs;
    if (c->L == 1) {
        if (c->dim == 2) {   // dense solve on the compact layout
            unpad2_vectors(G0(c), c->pd, rc.R, r, c->stage, c->stream);
            dense_apply(c->Ainv, c->npad, c->nL, c->stage, c->stage2, rc.R, rc.active, rc.done, c->stream);
            pad2_vectors(G0(c), c->pd, rc.R, nullptr, c->stage2, c->zf, c->stream);
            rc.launches += 2;
        } else {
            dense_apply(c->Ainv, c->npad, c->nL, r, c->zf, rc.R, rc.active, rc.done, c->stream);
        }
        vec_dot(n, rc.R, r, c->zf, c->partial, rc.active, rc.done, c->stream);
        rc.launches += 2;
        return vec_blocks(n);
    }
    if (c->fused2d) {
        March2Args a = march_args(c, rc);
        a.x = r; a.ec = ec; a.y = c->zf; a.partial = c->partial;
        rc.launches++;
        return march2_apply(M2_POST, a, c->nu_paper, c->stream);
    }
    prolong_add(G0(c), c->lv[1].g, c->lv[0].mask, c->lv[1].mask, ec, c->zpre, rc.R, rc.active, rc.done, true,
                c->stream);
    rc.launches++;
    double* src = c->zpre;
    int items = vec_blocks(n);
    if (c->opts.nu_post == 0) {
        cudaMemcpyAsync(c->zf, src, sizeof(double) * n * rc.R, cudaMemcpyDeviceToDevice, c->stream);
        vec_dot(n, rc.R, r, c->zf, c->partial, rc.active, rc.done, c->stream);
        rc.launches++;
        return items;
    }
    for (int s = 0; s < c->opts.nu_post; ++s) {
        const bool last = s == c->opts.nu_post - 1;
        double* dst = last ? c->zf : (src == c->z ? c->t : c->z);
        FineArgs a = fine_args(c, rc);
        a.x = src; a.b = r; a.Dinv = c->lv[0].Dinv; a.y = dst; a.partial = last ? c->partial : nullptr;
        items = level0_apply(c, FOP_JACOBI, a);
        rc.launches++;
        src = dst;
    }
    return items;
}

static mg_status capture_begin(mg_ctx* c) {
    CU(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
    return MG_OK;
}

static mg_status capture_end(mg_ctx* c, cudaGraphExec_t* exec, long long* nodes) {
    cudaGraph_t g = nullptr;
    CU(cudaStreamEndCapture(c->stream, &g));
    size_t nn = 0;
    CU(cudaGraphGetNodes(g, nullptr, &nn));
    *nodes = (long long)nn;
    CU(cudaGraphInstantiate(exec, g, 0));
    CU(cudaGraphDestroy(g));
    return MG_OK;
}

// Graphs (captured once per (R, tol)):
//   init    : b.b, x = 0, p0 = 0, q = 0, r1 = b
//   restart : z = B r (r1 -> r0, alpha = 0), r.z            (start and true-residual restarts)
//   iter    : two CG iterations (p and r ping-pong buffers)
//   true    : flush deferred x update, t = b - K x, t.t
static mg_status build_graphs(mg_ctx* c, int R, double tol) {
    for (cudaGraphExec_t* g : {&c->g_init, &c->g_restart, &c->g_iter, &c->g_true})
        if (*g) { cudaGraphExecDestroy(*g); *g = nullptr; }
    const long long n = c->vs;
    const int vb = vec_blocks(n);
    Rec rc{c, R, c->ctl.active, c->ctl.done};
    // ---- restart / initial preconditioning
    TRY(capture_begin(c));
    {
        blk_restrict(rc, c->r1, c->r0);
        double* ec = coarse_cycle(rc);
        const int k = blk_post(rc, c->r0, ec);
        cg_scalars(SM_RZ0, R, c->partial, k, c->ctl, 0.0, c->stream);
    }
    TRY(capture_end(c, &c->g_restart, &c->n_restart));
    // ---- init
    TRY(capture_begin(c));
    vec_dot(n, R, c->b, c->b, c->partial, nullptr, nullptr, c->stream);
    cg_scalars(SM_BB, R, c->partial, vb, c->ctl, 0.0, c->stream);
    CU(cudaMemsetAsync(c->x, 0, sizeof(double) * n * R, c->stream));
    CU(cudaMemsetAsync(c->p0, 0, sizeof(double) * n * R, c->stream));
    CU(cudaMemsetAsync(c->q, 0, sizeof(double) * n * R, c->stream));
    CU(cudaMemcpyAsync(c->r1, c->b, sizeof(double) * n * R, cudaMemcpyDeviceToDevice, c->stream));
    TRY(capture_end(c, &c->g_init, &c->n_init));
    // ---- two CG iterations
    TRY(capture_begin(c));
    for (int it = 0; it < 2; ++it) {
        double* pin = it == 0 ? c->p0 : c->p1;
        double* pout = it == 0 ? c->p1 : c->p0;
        double* rin = it == 0 ? c->r0 : c->r1;
        double* rout = it == 0 ? c->r1 : c->r0;
        int k = blk_cgp(rc, pin, pout);
        cg_scalars(SM_ALPHA, R, c->partial, k, c->ctl, 0.0, c->stream, pout == c->p1 ? 1 : 0);
        k = blk_restrict(rc, rin, rout);
        cg_scalars(SM_CONV, R, c->partial, k, c->ctl, tol, c->stream);
        double* ec = coarse_cycle(rc);
        k = blk_post(rc, rout, ec);
        cg_scalars(SM_BETA, R, c->partial, k, c->ctl, 0.0, c->stream);
    }
    TRY(capture_end(c, &c->g_iter, &c->n_iter));
    // ---- true residual
    TRY(capture_begin(c));
    {
        cg_flush_x(n, R, c->ctl, c->p0, c->p1, c->x, c->stream);
        Rec all{c, R, nullptr, nullptr};
        FineArgs a = fine_args(c, all);
        a.x = c->x; a.b = c->b; a.y = c->t;
        level0_apply(c, FOP_RESID, a);
        vec_dot(n, R, c->t, c->t, c->partial, nullptr, nullptr, c->stream);
        cg_scalars(SM_TRUE, R, c->partial, vb, c->ctl, 0.0, c->stream);
    }
    TRY(capture_end(c, &c->g_true, &c->n_true));
    c->graph_R = R;
    CHECK_LAUNCH();
    return MG_OK;
}

// ---------------------------------------------------------------- C ABI
extern "C" {

const char* mg_strerror(mg_status s) {
    switch (s) {
        case MG_OK: return "ok";
        case MG_ERR_ARG: return "invalid argument";
        case MG_ERR_NONDIVISIBLE: return "element counts not divisible by 2^(levels-1)";
        case MG_ERR_DIM: return "dimension mismatch";
        case MG_ERR_MODULUS: return "modulus not positive/finite";
        case MG_ERR_BREAKDOWN: return "CG breakdown (p.Kp <= 0)";
        case MG_ERR_MAXITER: return "maximum iterations reached";
        case MG_ERR_OOM: return "out of device memory";
        case MG_ERR_CUDA: return "CUDA error";
        case MG_ERR_NCCL: return "NCCL error";
        case MG_ERR_SINGULAR: return "coarsest operator not SPD";
    }
    return "unknown status";
}

const char* mg_last_error(void) { return g_last_error.c_str(); }

long long mg_kernel_launches(mg_handle h) { return h ? h->launches : -1; }

static mg_status setup_impl(mg_ctx* c, const mg_grid* grid, const double* E_e, const uint8_t* fixed, int levels,
                            const mg_opts* opts, void* stream) {
    c->dim = grid->dim;
    c->L = levels;
    c->nu = grid->nu;
    if (opts) c->opts = *opts;
    c->user = (cudaStream_t)stream;
    CU(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    CU(cudaEventCreateWithFlags(&c->ev_in, cudaEventDisableTiming));
    CU(cudaEventCreateWithFlags(&c->ev_out, cudaEventDisableTiming));
    stream_enter(c);
    cudaStream_t s = c->stream;
    int N[3] = {grid->nel[0], grid->nel[1], grid->dim == 3 ? grid->nel[2] : 1};
    for (int l = 0; l < levels; ++l) {
        int Nl[3];
        for (int k = 0; k < 3; ++k) Nl[k] = N[k] >> l;
        c->lv[l].g = make_geom(c->dim, Nl);
    }
    element_stiffness(c->dim, c->nu, c->K0);
    c->nu_paper = (c->nu == MG_NU_PAPER);
    c->fused2d = (c->dim == 2 && levels >= 2);
    fine_set_constants(c->dim, c->K0.data(), s);
    if (c->dim == 2) fine2d_set_constants(c->K0.data(), s);
    galerkin_set_constants(c->dim, c->K0.data(), s);
    stress_set_constants(c->dim, c->nu, s);
    const LevelGeom& g0 = G0(c);
    CU(cudaMalloc(&c->E, sizeof(double) * g0.nelem + 64));   // +64: aligned bulk-copy tails
    CU(cudaMemcpyAsync(c->E, E_e, sizeof(double) * g0.nelem,
                       is_device_ptr(E_e) ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, s));
    for (int l = 0; l < levels; ++l) {
        Level& v = c->lv[l];
        CU(cudaMalloc(&v.mask, v.g.nnodes + 64));
        CU(cudaMalloc(&v.Dinv, sizeof(double) * v.g.ndof));
        CU(cudaMalloc(&v.D, sizeof(double) * v.g.ndof));
        if (l >= 1 || levels == 1) {
            const int ns = c->dim == 2 ? 9 : 27;
            CU(cudaMalloc(&v.st, sizeof(double) * v.g.nnodes * ns * c->dim * c->dim));
        }
    }
    {
        uint8_t* dfix = nullptr;
        const uint8_t* fsrc = fixed;
        if (!is_device_ptr(fixed)) {
            CU(cudaMallocAsync(&dfix, g0.ndof, s));
            CU(cudaMemcpyAsync(dfix, fixed, g0.ndof, cudaMemcpyHostToDevice, s));
            fsrc = dfix;
        }
        fixed_to_mask_kernel<<<(unsigned)((g0.nnodes + 255) / 256), 256, 0, s>>>(g0.nnodes, c->dim, fsrc,
                                                                                 c->lv[0].mask);
        CHECK_LAUNCH();
        if (dfix) CU(cudaFreeAsync(dfix, s));
    }
    for (int l = 1; l < levels; ++l) {
        coarse_mask_kernel<<<(unsigned)((c->lv[l].g.nnodes + 255) / 256), 256, 0, s>>>(
            c->lv[l - 1].g, c->lv[l].g, c->lv[l - 1].mask, c->lv[l].mask);
        CHECK_LAUNCH();
    }
    c->launches += levels;
    if (c->dim == 2) {
        c->pd = pad2_layout(g0);
        CU(cudaMalloc(&c->Epad, sizeof(double) * c->pd.elems));
        CU(cudaMalloc(&c->maskpad, c->pd.nodes));
        CU(cudaMalloc(&c->Dinvpad, sizeof(double) * 2 * c->pd.nodes));
        c->vs = c->pd.vstride;
    } else {
        c->vs = g0.ndof;
    }
    c->nL = c->lv[levels - 1].g.ndof;
    c->npad = (c->nL + 31) / 32 * 32;
    CU(cudaMalloc(&c->Ainv, sizeof(double) * c->npad * c->npad));
    // control block
    const int MR = MG_MAX_RHS;
    size_t bytes = sizeof(double) * 8 * MR + sizeof(int) * (4 * MR + 4);
    CU(cudaMalloc(&c->ctl_mem, bytes));
    CU(cudaMemsetAsync(c->ctl_mem, 0, bytes, s));
    double* dp = (double*)c->ctl_mem;
    c->ctl.alpha = dp; c->ctl.beta = dp + MR; c->ctl.rz = dp + 2 * MR; c->ctl.rr = dp + 3 * MR;
    c->ctl.bb = dp + 4 * MR; c->ctl.pq = dp + 5 * MR; c->ctl.tt = dp + 6 * MR; c->ctl.xalpha = dp + 7 * MR;
    int* ip = (int*)(dp + 8 * MR);
    c->ctl.active = ip; c->ctl.iters = ip + MR; c->ctl.xbuf = ip + 2 * MR;
    c->ctl.done = ip + 3 * MR; c->ctl.status = ip + 3 * MR + 1;
    c->d_status = ip + 3 * MR + 2;
    CU(cudaMallocHost(&c->h_pinned, sizeof(int) * (2 * MR + 4)));
    CU(cudaMallocHost(&c->h_dbl, sizeof(double) * 4 * MR));
    TRY(compute_operators(c));
    stream_leave(c);
    return MG_OK;
}

mg_status mg_setup(const mg_grid* grid, const double* E_e, const uint8_t* fixed, int levels, const mg_opts* opts,
                   void* stream, mg_handle* out) {
    if (!grid || !E_e || !fixed || !out) return fail(MG_ERR_ARG, "NULL argument");
    if (grid->dim != 2 && grid->dim != 3) return fail(MG_ERR_ARG, "dim must be 2 or 3");
    if (levels < 1 || levels > MG_MAX_LEVELS) return fail(MG_ERR_ARG, "levels out of range");
    if (!(grid->nu > -1.0 && grid->nu < 0.5)) return fail(MG_ERR_ARG, "nu out of range");
    if (opts && (opts->nu_pre < 1 || opts->nu_post < 0 || opts->max_iter < 1 || !(opts->omega > 0)))
        return fail(MG_ERR_ARG, "invalid mg_opts");
    if (opts && grid->dim == 2 && (opts->nu_pre != 1 || opts->nu_post != 1))
        return fail(MG_ERR_ARG, "2D path implements the fused V(1,1) cycle only (nu_pre = nu_post = 1)");
    const int f = 1 << (levels - 1);
    long long nodes = 1;
    for (int k = 0; k < grid->dim; ++k) {
        if (grid->nel[k] < 1) return fail(MG_ERR_ARG, "nel must be >= 1");
        if (grid->nel[k] % f) return fail(MG_ERR_NONDIVISIBLE, "nel not divisible by 2^(levels-1) (SPEC.md:40)");
        nodes *= grid->nel[k] + 1;
    }
    if (nodes * grid->dim * MG_MAX_RHS >= (1LL << 40)) return fail(MG_ERR_DIM, "grid too large");
    long long ncoarse = grid->dim;
    for (int k = 0; k < grid->dim; ++k) ncoarse *= grid->nel[k] / f + 1;
    if (ncoarse > 20000) return fail(MG_ERR_DIM, "coarsest level too large for the dense direct solve; add levels");
    mg_ctx* c = new mg_ctx();
    mg_status st = setup_impl(c, grid, E_e, fixed, levels, opts, stream);
    if (st != MG_OK) {
        std::string keep = g_last_error;
        mg_destroy(c);
        g_last_error = keep;
        return st;
    }
    *out = c;
    return MG_OK;
}

mg_status mg_update_modulus(mg_handle c, const double* E_e) {
    if (!c || !E_e) return fail(MG_ERR_ARG, "NULL argument");
    stream_enter(c);
    CU(cudaMemcpyAsync(c->E, E_e, sizeof(double) * G0(c).nelem,
                       is_device_ptr(E_e) ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, c->stream));
    // E changes the stencils but not the masks; the masks of coarse levels may have been
    // augmented by zero-diagonal DOFs, which stay valid for the same BCs.
    TRY(compute_operators(c));
    stream_leave(c);
    return MG_OK;
}

mg_status mgcg_solve(mg_handle c, const double* rhs, int nrhs, double tol, double* x, mg_report* rep) {
    if (!c || !rhs || !x) return fail(MG_ERR_ARG, "NULL argument");
    if (nrhs < 1 || nrhs > MG_MAX_RHS) return fail(MG_ERR_ARG, "nrhs out of range");
    if (!(tol > 0.0) || !(tol < 1.0)) return fail(MG_ERR_ARG, "tol must be in (0,1)");
    const LevelGeom& g0 = G0(c);
    const long long n = g0.ndof;
    cudaStream_t s = c->stream;
    stream_enter(c);
    cudaEvent_t e0, e1;
    CU(cudaEventCreate(&e0));
    CU(cudaEventCreate(&e1));
    CU(cudaEventRecord(e0, s));
    TRY(ensure_vectors(c, nrhs));
    if (c->graph_R != nrhs || c->graph_tol != tol) {
        TRY(build_graphs(c, nrhs, tol));
        c->graph_tol = tol;
    }
    const bool rdev = is_device_ptr(rhs), xdev = is_device_ptr(x);
    const double* rsrc = rhs;
    if (!rdev) {
        CU(cudaMemcpyAsync(c->stage, rhs, sizeof(double) * n * nrhs, cudaMemcpyHostToDevice, s));
        rsrc = c->stage;
    }
    if (c->dim == 2) pad2_vectors(g0, c->pd, nrhs, c->lv[0].mask, rsrc, c->b, s);
    else vec_mask_copy(g0.nnodes, c->dim, nrhs, c->lv[0].mask, rsrc, c->b, s);
    c->launches += 1;
    CU(cudaMemsetAsync(c->ctl.status, 0, sizeof(int), s));
    CU(cudaGraphLaunch(c->g_init, s));
    CU(cudaGraphLaunch(c->g_restart, s));
    int glaunch = 2;
    long long klaunch = c->n_init + c->n_restart;
    int* hp = c->h_pinned;    // [0] done [1] status [2..2+R) iters
    double* hd = c->h_dbl;    // bb[64] rr[64] tt[64]
    const int maxit = c->opts.max_iter;
    int restarts = 0;
    mg_status result = MG_OK;
    for (;;) {
        // iterate until all RHS converged (recursive residual) or the cap
        for (;;) {
            CU(cudaMemcpyAsync(hp, c->ctl.done, sizeof(int) * 2, cudaMemcpyDeviceToHost, s));
            CU(cudaMemcpyAsync(hp + 2, c->ctl.iters, sizeof(int) * nrhs, cudaMemcpyDeviceToHost, s));
            CU(cudaStreamSynchronize(s));
            if (hp[0] || hp[1]) break;
            int mx = 0;
            for (int k = 0; k < nrhs; ++k) mx = hp[2 + k] > mx ? hp[2 + k] : mx;
            if (mx >= maxit) break;
            CU(cudaGraphLaunch(c->g_iter, s));
            ++glaunch;
            klaunch += c->n_iter;
        }
        if (hp[1]) { result = fail(MG_ERR_BREAKDOWN, "p.Kp <= 0 in CG"); break; }
        CU(cudaGraphLaunch(c->g_true, s));
        ++glaunch;
        klaunch += c->n_true;
        CU(cudaMemcpyAsync(hd, c->ctl.bb, sizeof(double) * MG_MAX_RHS, cudaMemcpyDeviceToHost, s));
        CU(cudaMemcpyAsync(hd + MG_MAX_RHS, c->ctl.rr, sizeof(double) * MG_MAX_RHS, cudaMemcpyDeviceToHost, s));
        CU(cudaMemcpyAsync(hd + 2 * MG_MAX_RHS, c->ctl.tt, sizeof(double) * MG_MAX_RHS, cudaMemcpyDeviceToHost, s));
        CU(cudaMemcpyAsync(hp + 2, c->ctl.iters, sizeof(int) * nrhs, cudaMemcpyDeviceToHost, s));
        CU(cudaStreamSynchronize(s));
        // restart the RHS whose true residual exceeds tol (reading r12)
        std::vector<int> restart(MG_MAX_RHS, 0);
        int nre = 0;
        for (int k = 0; k < nrhs; ++k) {
            const double bb = hd[k], tt = hd[2 * MG_MAX_RHS + k];
            if (bb > 0.0 && tt > tol * tol * bb && hp[2 + k] < maxit) { restart[k] = 1; ++nre; }
        }
        if (!nre || restarts >= 3) break;
        ++restarts;
        int* d_restart = c->ctl.active;   // active := restart flags, then r1 = t for them
        CU(cudaMemcpyAsync(d_restart, restart.data(), sizeof(int) * MG_MAX_RHS, cudaMemcpyHostToDevice, s));
        vec_axpy_masked_restart(c->vs, nrhs, c->t, c->r1, d_restart, s);
        CU(cudaMemsetAsync(c->ctl.alpha, 0, sizeof(double) * MG_MAX_RHS, s));
        int zero = 0;
        CU(cudaMemcpyAsync(c->ctl.done, &zero, sizeof(int), cudaMemcpyHostToDevice, s));
        CU(cudaGraphLaunch(c->g_restart, s));
        ++glaunch;
        klaunch += c->n_restart + 1;
    }
    // copy x out
    if (c->dim == 2) {
        if (xdev) {
            unpad2_vectors(g0, c->pd, nrhs, c->x, x, s);
        } else {
            unpad2_vectors(g0, c->pd, nrhs, c->x, c->stage, s);
            CU(cudaMemcpyAsync(x, c->stage, sizeof(double) * n * nrhs, cudaMemcpyDeviceToHost, s));
        }
    } else if (xdev) {
        CU(cudaMemcpyAsync(x, c->x, sizeof(double) * n * nrhs, cudaMemcpyDeviceToDevice, s));
    } else {
        CU(cudaMemcpyAsync(x, c->x, sizeof(double) * n * nrhs, cudaMemcpyDeviceToHost, s));
    }
    CU(cudaEventRecord(e1, s));
    CU(cudaStreamSynchronize(s));
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    c->launches += klaunch;
    bool all_conv = true;
    int mx = 0;
    for (int k = 0; k < nrhs; ++k) {
        const double bb = hd[k];
        const double tr = bb > 0 ? std::sqrt(hd[2 * MG_MAX_RHS + k] / bb) : 0.0;
        const bool conv = tr <= tol;
        all_conv = all_conv && conv;
        mx = hp[2 + k] > mx ? hp[2 + k] : mx;
        if (rep) {
            rep->iters[k] = hp[2 + k];
            rep->relres[k] = bb > 0 ? std::sqrt(hd[MG_MAX_RHS + k] / bb) : 0.0;
            rep->true_relres[k] = tr;
            rep->converged[k] = conv ? 1 : 0;
        }
    }
    if (rep) {
        rep->nrhs = nrhs;
        rep->max_iters = mx;
        rep->restarts = restarts;
        rep->graph_launches = glaunch;
        rep->kernel_launches = klaunch;
        rep->solve_ms = ms;
    }
    stream_leave(c);
    if (result != MG_OK) return result;
    if (!all_conv) return fail(MG_ERR_MAXITER, "not all right-hand sides reached tol");
    return MG_OK;
}

mg_status stress_stiffness_apply(mg_handle c, const double* Es_e, const double* u, const double* phi, int nphi,
                                 double* y) {
    if (!c || !Es_e || !u || !phi || !y) return fail(MG_ERR_ARG, "NULL argument");
    if (nphi < 1) return fail(MG_ERR_ARG, "nphi must be >= 1");
    const LevelGeom& g0 = G0(c);
    cudaStream_t s = c->stream;
    stream_enter(c);
    const int nv = c->dim == 2 ? 3 : 6;
    if (!c->sig) CU(cudaMalloc(&c->sig, sizeof(double) * g0.nelem * nv));
    const bool dev = is_device_ptr(phi) && is_device_ptr(y) && is_device_ptr(u) && is_device_ptr(Es_e);
    const long long n = g0.ndof;
    if (dev) {
        stress_sigma(g0, Es_e, u, c->sig, s);
        stress_apply(g0, c->sig, c->lv[0].mask, phi, y, nphi, s);
        c->launches += 2;
        CHECK_LAUNCH();
        stream_leave(c);
        return MG_OK;
    }
    // host buffers: stage through device temporaries (synchronous)
    double *dEs = nullptr, *du = nullptr, *dphi = nullptr, *dy = nullptr;
    CU(cudaMallocAsync(&dEs, sizeof(double) * g0.nelem, s));
    CU(cudaMallocAsync(&du, sizeof(double) * n, s));
    CU(cudaMallocAsync(&dphi, sizeof(double) * n * nphi, s));
    CU(cudaMallocAsync(&dy, sizeof(double) * n * nphi, s));
    CU(cudaMemcpyAsync(dEs, Es_e, sizeof(double) * g0.nelem, cudaMemcpyDefault, s));
    CU(cudaMemcpyAsync(du, u, sizeof(double) * n, cudaMemcpyDefault, s));
    CU(cudaMemcpyAsync(dphi, phi, sizeof(double) * n * nphi, cudaMemcpyDefault, s));
    stress_sigma(g0, dEs, du, c->sig, s);
    stress_apply(g0, c->sig, c->lv[0].mask, dphi, dy, nphi, s);
    c->launches += 2;
    CHECK_LAUNCH();
    CU(cudaMemcpyAsync(y, dy, sizeof(double) * n * nphi, cudaMemcpyDefault, s));
    for (double* p : {dEs, du, dphi, dy}) CU(cudaFreeAsync(p, s));
    CU(cudaStreamSynchronize(s));
    stream_leave(c);
    return MG_OK;
}

mg_status mg_matvec(mg_handle c, int level, const double* x, int nrhs, double* y) {
    if (!c || !x || !y) return fail(MG_ERR_ARG, "NULL argument");
    if (level < 0 || level >= c->L || nrhs < 1) return fail(MG_ERR_ARG, "bad level / nrhs");
    stream_enter(c);
    if (level == 0) {
        FineArgs a{};
        a.g = G0(c); a.E = c->E; a.mask = c->lv[0].mask; a.x = x; a.y = y; a.R = nrhs;
        a.nu_paper = c->nu_paper ? 1 : 0;
        if (c->dim == 2) {   // compact <-> padded around the march kernel
            TRY(ensure_vectors(c, nrhs));
            pad2_vectors(G0(c), c->pd, nrhs, nullptr, x, c->t, c->stream);
            a.x = c->t; a.y = c->q;
            level0_apply(c, FOP_MATVEC, a);
            unpad2_vectors(G0(c), c->pd, nrhs, c->q, y, c->stream);
        } else {
            fine_apply(FOP_MATVEC, a, c->stream);
        }
    } else {
        CoarseArgs a{};
        a.g = c->lv[level].g; a.st = c->lv[level].st; a.x = x; a.y = y; a.R = nrhs;
        coarse_apply(COP_MATVEC, a, c->stream);
    }
    c->launches++;
    CHECK_LAUNCH();
    stream_leave(c);
    return MG_OK;
}

mg_status mg_vcycle(mg_handle c, const double* r, int nrhs, double* z) {
    if (!c || !r || !z) return fail(MG_ERR_ARG, "NULL argument");
    if (nrhs < 1 || nrhs > MG_MAX_RHS) return fail(MG_ERR_ARG, "bad nrhs");
    TRY(ensure_vectors(c, nrhs));
    stream_enter(c);
    const long long n = G0(c).ndof;
    // the preconditioner exactly as the solve applies it (same fine blocks, alpha = 0)
    if (c->dim == 2) pad2_vectors(G0(c), c->pd, nrhs, c->lv[0].mask, r, c->r1, c->stream);
    else CU(cudaMemcpyAsync(c->r1, r, sizeof(double) * n * nrhs, cudaMemcpyDeviceToDevice, c->stream));
    CU(cudaMemsetAsync(c->ctl.alpha, 0, sizeof(double) * MG_MAX_RHS, c->stream));
    CU(cudaMemsetAsync(c->q, 0, sizeof(double) * c->vs * nrhs, c->stream));
    Rec rc{c, nrhs, nullptr, nullptr};
    blk_restrict(rc, c->r1, c->r0);
    double* ec = coarse_cycle(rc);
    blk_post(rc, c->r0, ec);
    if (c->dim == 2) unpad2_vectors(G0(c), c->pd, nrhs, c->zf, z, c->stream);
    else CU(cudaMemcpyAsync(z, c->zf, sizeof(double) * n * nrhs, cudaMemcpyDeviceToDevice, c->stream));
    c->launches += rc.launches;
    CHECK_LAUNCH();
    stream_leave(c);
    return MG_OK;
}

mg_status mg_restrict(mg_handle c, int level, const double* fine, int nrhs, double* coarse) {
    if (!c || !fine || !coarse) return fail(MG_ERR_ARG, "NULL argument");
    if (level < 0 || level >= c->L - 1 || nrhs < 1) return fail(MG_ERR_ARG, "bad level / nrhs");
    stream_enter(c);
    restrict_apply(c->lv[level].g, c->lv[level + 1].g, c->lv[level].mask, c->lv[level + 1].mask, fine, coarse, nrhs,
                   nullptr, nullptr, c->stream);
    c->launches++;
    CHECK_LAUNCH();
    stream_leave(c);
    return MG_OK;
}

mg_status mg_prolong(mg_handle c, int level, const double* coarse, int nrhs, double* fine) {
    if (!c || !fine || !coarse) return fail(MG_ERR_ARG, "NULL argument");
    if (level < 0 || level >= c->L - 1 || nrhs < 1) return fail(MG_ERR_ARG, "bad level / nrhs");
    stream_enter(c);
    prolong_add(c->lv[level].g, c->lv[level + 1].g, c->lv[level].mask, c->lv[level + 1].mask, coarse, fine, nrhs,
                nullptr, nullptr, false, c->stream);
    c->launches++;
    CHECK_LAUNCH();
    stream_leave(c);
    return MG_OK;
}

mg_status mg_level_info(mg_handle c, int level, int* nel3, long long* ndof, int* nlevels) {
    if (!c) return fail(MG_ERR_ARG, "NULL handle");
    if (nlevels) *nlevels = c->L;
    if (level < 0) return MG_OK;
    if (level >= c->L) return fail(MG_ERR_ARG, "bad level");
    if (nel3)
        for (int k = 0; k < 3; ++k) nel3[k] = k < c->dim ? c->lv[level].g.N[k] : 0;
    if (ndof) *ndof = c->lv[level].g.ndof;
    return MG_OK;
}

mg_status mg_get_diagonal(mg_handle c, int level, double* d) {
    if (!c || !d) return fail(MG_ERR_ARG, "NULL argument");
    if (level < 0 || level >= c->L) return fail(MG_ERR_ARG, "bad level");
    stream_enter(c);
    CU(cudaMemcpyAsync(d, c->lv[level].D, sizeof(double) * c->lv[level].g.ndof, cudaMemcpyDeviceToDevice, c->stream));
    stream_leave(c);
    return MG_OK;
}

mg_status mg_get_coarse_inverse(mg_handle c, double* Ainv) {
    if (!c || !Ainv) return fail(MG_ERR_ARG, "NULL argument");
    stream_enter(c);
    CU(cudaMemcpy2DAsync(Ainv, sizeof(double) * c->nL, c->Ainv, sizeof(double) * c->npad, sizeof(double) * c->nL,
                         c->nL, cudaMemcpyDeviceToDevice, c->stream));
    stream_leave(c);
    return MG_OK;
}

mg_status mg_profile_kernels(mg_handle c, int nrhs, int reps, double* ms) {
    if (!c || !ms) return fail(MG_ERR_ARG, "NULL argument");
    if (nrhs < 1 || nrhs > MG_MAX_RHS || reps < 1) return fail(MG_ERR_ARG, "bad nrhs / reps");
    TRY(ensure_vectors(c, nrhs));
    stream_enter(c);
    cudaStream_t s = c->stream;
    Rec rc{c, nrhs, nullptr, nullptr};
    cudaEvent_t e0, e1;
    CU(cudaEventCreate(&e0));
    CU(cudaEventCreate(&e1));
    for (int op = 0; op < 4; ++op) {
        auto launch = [&]() {
            switch (op) {
                case 0: blk_cgp(rc, c->p0, c->p1); break;
                case 1: blk_restrict(rc, c->r0, c->r1); break;
                case 2: blk_post(rc, c->r1, c->L > 1 ? c->lv[1].z : nullptr); break;
                default: {
                    FineArgs a = fine_args(c, rc);
                    a.x = c->p0; a.y = c->q;
                    level0_apply(c, FOP_MATVEC, a);
                }
            }
        };
        launch();
        CU(cudaEventRecord(e0, s));
        for (int k = 0; k < reps; ++k) launch();
        CU(cudaEventRecord(e1, s));
        CU(cudaEventSynchronize(e1));
        float t = 0.f;
        cudaEventElapsedTime(&t, e0, e1);
        ms[op] = t / reps;
    }
    CHECK_LAUNCH();
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    stream_leave(c);
    return MG_OK;
}

mg_status mg_destroy(mg_handle c) {
    if (!c) return MG_OK;
    if (c->stream) cudaStreamSynchronize(c->stream);
    free_vectors(c);
    for (int l = 0; l < MG_MAX_LEVELS; ++l) {
        Level& v = c->lv[l];
        if (v.mask) cudaFree(v.mask);
        if (v.Dinv) cudaFree(v.Dinv);
        if (v.D) cudaFree(v.D);
        if (v.st) cudaFree(v.st);
    }
    if (c->E) cudaFree(c->E);
    if (c->Epad) cudaFree(c->Epad);
    if (c->maskpad) cudaFree(c->maskpad);
    if (c->Dinvpad) cudaFree(c->Dinvpad);
    if (c->Ainv) cudaFree(c->Ainv);
    if (c->ctl_mem) cudaFree(c->ctl_mem);
    if (c->sig) cudaFree(c->sig);
    if (c->h_pinned) cudaFreeHost(c->h_pinned);
    if (c->h_dbl) cudaFreeHost(c->h_dbl);
    if (c->ev_in) cudaEventDestroy(c->ev_in);
    if (c->ev_out) cudaEventDestroy(c->ev_out);
    if (c->stream) cudaStreamDestroy(c->stream);
    delete c;
    return MG_OK;
}

}  // extern "C"
