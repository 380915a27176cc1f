// C-ABI host side of libmgcg: handle, slab decomposition, hierarchy setup, CUDA-graph solve
// loop.  See include/mgcg.h for the contract and the paper passages each call follows.
//
// Slabs: the global grid is cut along axis 0 into S = nranks x nslab slabs at
// coarsest-level element boundaries.  Every slab holds its owned element layers plus the
// ghost element layer below, and its owned node planes plus one ghost node plane on each
// side with a neighbour, at every level.  All kernels run unchanged on the slab's local grid
// (ghost rows of an operator output are wrong and never used); dots count owned planes
// only; restriction sums from owned fine planes only, leaving a partial sum in the upper
// coarse ghost plane that the owner adds in.  Validity of ghost planes is restored by the
// exchanges in comm.cu at the points listed in DESIGN.md §7.  With S = 1 every exchange is
// a no-op and the code path is the single-GPU one.
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/mgcg.h"
#include "comm.h"
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

#define COMM(expr)                                                                 \
    do {                                                                           \
        if (!(expr)) return fail(MG_ERR_NCCL, std::string("exchange: ") + comm_last_error()); \
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

// Incompatible-mode element ("Wilson quadrilaterals ... hexahedra"):
// per component the bubble modes M_k = 1 - (2 x_k - 1)^2, k < d, condensed on the unit element
// (material constant per element): K_e0 = K_cc - K_ci K_ii^-1 K_ic with
// K = int [B_c B_i]^T D0 [B_c B_i] by 2x2(x2) Gauss (exact for these polynomials).
static void element_stiffness_wilson(int dim, double nu, std::vector<double>& K0) {
    const int na = 1 << dim, n = dim * na, ni = dim * dim, nt = n + ni, nv = dim == 2 ? 3 : 6;
    double D[36] = {0};
    if (dim == 2) {
        const double c = 1.0 / (1.0 - nu * nu);
        const double m[9] = {c, c * nu, 0, c * nu, c, 0, 0, 0, c * (1 - nu) / 2};
        for (int i = 0; i < 9; ++i) D[i] = m[i];
    } else {
        const double lam = nu / ((1 + nu) * (1 - 2 * nu)), mu = 1.0 / (2 * (1 + nu));
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j) D[i * 6 + j] = lam + (i == j ? 2 * mu : 0.0);
        for (int i = 3; i < 6; ++i) D[i * 6 + i] = mu;
    }
    const int sh[3][2] = {{1, 2}, {0, 2}, {0, 1}};   // 3D engineering shear pairs (2D: (0, 1))
    auto shear = [&](int s, int& i, int& j) {
        if (dim == 2) { i = 0; j = 1; } else { i = sh[s][0]; j = sh[s][1]; }
    };
    const double g1[2] = {0.5 - 0.5 / std::sqrt(3.0), 0.5 + 0.5 / std::sqrt(3.0)};
    std::vector<double> K((size_t)nt * nt, 0.0), B((size_t)nv * nt);
    const int ng = 1 << dim;
    for (int q = 0; q < ng; ++q) {
        double x[3];
        for (int k = 0; k < dim; ++k) x[k] = g1[(q >> (dim - 1 - k)) & 1];
        const double w = 1.0 / ng;
        std::fill(B.begin(), B.end(), 0.0);
        for (int a = 0; a < na; ++a) {
            double gr[3];
            for (int j = 0; j < dim; ++j) {
                double v = 1.0;
                for (int k = 0; k < dim; ++k) {
                    const int bit = (a >> (dim - 1 - k)) & 1;
                    v *= (k == j) ? (bit ? 1.0 : -1.0) : (bit ? x[k] : 1.0 - x[k]);
                }
                gr[j] = v;
            }
            for (int i = 0; i < dim; ++i) B[i * nt + dim * a + i] = gr[i];
            for (int s = 0; s < nv - dim; ++s) {
                int i, j;
                shear(s, i, j);
                B[(dim + s) * nt + dim * a + i] += gr[j];
                B[(dim + s) * nt + dim * a + j] += gr[i];
            }
        }
        for (int k = 0; k < dim; ++k) {
            const double dm = -4.0 * (2.0 * x[k] - 1.0);   // dM_k/dx_k
            for (int c = 0; c < dim; ++c) {
                const int col = n + c * dim + k;
                if (c == k) B[c * nt + col] += dm;
                for (int s = 0; s < nv - dim; ++s) {
                    int i, j;
                    shear(s, i, j);
                    if (c == i && j == k) B[(dim + s) * nt + col] += dm;
                    if (c == j && i == k) B[(dim + s) * nt + col] += dm;
                }
            }
        }
        for (int r = 0; r < nt; ++r)
            for (int cc = 0; cc < nt; ++cc) {
                double v = 0.0;
                for (int p = 0; p < nv; ++p)
                    for (int p2 = 0; p2 < nv; ++p2) v += B[p * nt + r] * D[p * nv + p2] * B[p2 * nt + cc];
                K[(size_t)r * nt + cc] += w * v;
            }
    }
    // K_ii^-1 K_ic by Gauss-Jordan on the small SPD block
    std::vector<double> Kii((size_t)ni * ni), X((size_t)ni * n);
    for (int r = 0; r < ni; ++r) {
        for (int c = 0; c < ni; ++c) Kii[r * ni + c] = K[(size_t)(n + r) * nt + n + c];
        for (int c = 0; c < n; ++c) X[r * n + c] = K[(size_t)(n + r) * nt + c];
    }
    for (int p = 0; p < ni; ++p) {
        const double piv = Kii[p * ni + p];
        for (int c = 0; c < ni; ++c) Kii[p * ni + c] /= piv;
        for (int c = 0; c < n; ++c) X[p * n + c] /= piv;
        for (int r = 0; r < ni; ++r) {
            if (r == p) continue;
            const double f = Kii[r * ni + p];
            if (f == 0.0) continue;
            for (int c = 0; c < ni; ++c) Kii[r * ni + c] -= f * Kii[p * ni + c];
            for (int c = 0; c < n; ++c) X[r * n + c] -= f * X[p * n + c];
        }
    }
    K0.assign((size_t)n * n, 0.0);
    for (int r = 0; r < n; ++r)
        for (int c = 0; c < n; ++c) {
            double v = K[(size_t)r * nt + c];
            for (int p = 0; p < ni; ++p) v -= K[(size_t)r * nt + n + p] * X[p * n + c];
            K0[(size_t)r * n + c] = v;
        }
    // symmetrise the rounding
    for (int r = 0; r < n; ++r)
        for (int c = r + 1; c < n; ++c) {
            const double v = 0.5 * (K0[(size_t)r * n + c] + K0[(size_t)c * n + r]);
            K0[(size_t)r * n + c] = K0[(size_t)c * n + r] = v;
        }
}

// ---------------------------------------------------------------- small kernels
// mask[dst0 + i] = fixed bits of node (src0 + i) of the user's fixed array, i < count
__global__ void fixed_to_mask_kernel(long long count, int dim, const uint8_t* fixed, long long src0, uint8_t* mask,
                                     long long dst0) {
    long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= count) return;
    int m = 0;
    for (int k = 0; k < dim; ++k) m |= (fixed[dim * (src0 + i) + k] ? 1 : 0) << k;
    mask[dst0 + i] = (uint8_t)m;
}

// a coarse DOF is fixed iff its coincident fine DOF is (reading r11); fine local plane of
// coarse local plane I is 2I - off0 (slab ghost plane below has no local fine partner)
__global__ void coarse_mask_kernel(LevelGeom gf, LevelGeom gc, const uint8_t* mf, uint8_t* mc, int off0) {
    long long I = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (I >= gc.nnodes) return;
    long long t = I, q = 0;
    int ci[3] = {0, 0, 0};
    for (int k = gc.dim - 1; k >= 0; --k) { ci[k] = (int)(t % gc.nn[k]); t /= gc.nn[k]; }
    const int f0 = 2 * ci[0] - off0;
    if (f0 < 0) return;
    for (int k = 0; k < gc.dim; ++k) q = q * gf.nn[k] + (k == 0 ? f0 : 2 * ci[k]);
    mc[I] = mf[q];
}

__global__ void check_modulus_kernel(long long n, const double* E, int* bad) {
    long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double v = E[i];
    if (!(v > 0.0) || !isfinite(v)) atomicOr(bad, 4);
}

// ---------------------------------------------------------------- handle
struct Level {
    LevelGeom g;              // local geometry of the slab at this level (incl. ghosts)
    uint8_t* mask = nullptr;
    double* Dinv = nullptr;
    double* D = nullptr;
    double* st = nullptr;     // stencil (coarse levels; level 0 only when L == 1)
    double* r = nullptr;      // vectors (levels >= 1), R x ndof
    double* z = nullptr;
    double* w = nullptr;
    int o0 = 0, o1 = 0;       // owned local node planes [o0, o1)
    int gp0 = 0;              // global node plane of local plane 0
    long long pn = 0;         // nodes per plane
};

struct Slab {
    int id = 0;               // global slab index
    int e0 = 0, e1 = 0;       // owned global element layers at level 0
    int gl = 0, gh = 0;       // ghost plane below / above
    long long uoff = 0;       // node offset of the owned planes in the rank's user vectors
    Level lv[MG_MAX_LEVELS];
    double* E = nullptr;      // local elements (ghost layer first when gl)
    double *elmA = nullptr, *elmB = nullptr;
    // 2D fine level: ghost-padded copies used by the march kernels (fine2d.cu)
    Pad2 pd{};
    // 3D fine level: row-padded layout of the TMA march kernels (h8t.cu); g0p = level-0 geometry
    // with the padded vector pitch (maskpad / Dinvpad / Epad below hold the padded copies)
    Pad3 p3{};
    LevelGeom g0p{};
    double* Epad = nullptr;
    uint8_t* maskpad = nullptr;
    double* Dinvpad = nullptr;
    long long vs = 0;         // doubles per RHS of a level-0 vector (padded in 2D, ndof in 3D)
    double *b = nullptr, *x = nullptr, *r0 = nullptr, *r1 = nullptr, *p0 = nullptr, *p1 = nullptr, *q = nullptr,
           *zf = nullptr, *z = nullptr, *t = nullptr;
    double* zpre = nullptr;
    bool z1_from_r = false;   // fused 3D V-cycle: zpre is formed by the prolongation from r (not stored)
    double *u = nullptr, *phi = nullptr, *gy = nullptr, *sig = nullptr, *Es = nullptr;   // G(u) phi (slab mode)
    long long gphi_cap = 0;
    // NEXT-1 in slab mode: slab-local compact node vectors / element arrays (incl. ghosts)
    double* tn[4] = {nullptr, nullptr, nullptr, nullptr};
    long long tn_cap[4] = {0, 0, 0, 0};
    double* te[3] = {nullptr, nullptr, nullptr};
    long long te_cap[3] = {0, 0, 0};
};

struct mg_ctx {
    int dim = 0, L = 0;
    double nu = 0.3;
    int elem = 0;             // mg_grid.element
    bool nu_paper = true;     // nu == 0.3: compile-time K0 in the fine kernels
    bool fused2d = false;     // 2D, L >= 2, V(1,1): fused RESTRICT / POST fine kernels
    bool unfused_coarse = false;   // MG_UNFUSED_COARSE=1: generic coarse-level kernels (A/B checks)
    bool fused3d = false;     // 3D, L >= 2, V(1,1): fused h8 RESTR3 fine kernel
    mg_opts opts{0.6, 1, 1, 1000};
    cudaStream_t user = nullptr, stream = nullptr;
    cudaEvent_t ev_in = nullptr, ev_out = nullptr;
    LevelGeom G[MG_MAX_LEVELS];   // global geometry
    std::vector<Slab> sl;         // this handle's slabs (axis-0 order)
    int S = 1;                    // slabs in the job (nranks x nslab)
    Comm comm;
    std::vector<int> rank_p0, rank_p1;   // per rank: owned global fine node planes [p0, p1)
    long long n_rank = 0, m_rank = 0;    // this rank's owned DOFs / elements
    long long pn0 = 0;                   // fine nodes per plane
    std::vector<double> K0;
    // coarsest level (global, replicated on every rank)
    double* Ainv = nullptr;
    long long nL = 0, npad = 0;
    double *cr = nullptr, *cz = nullptr;         // (R, nL) gathered coarsest vectors
    double* stg = nullptr;                       // gathered coarsest stencil
    double *cpack = nullptr, *cgath = nullptr;   // cross-rank gather staging
    long long cpack_cap = 0;
    double* gj_work = nullptr;
    double* Mc = nullptr;                        // Galerkin child matrices Q_c^T K0 Q_c
    double* Estage = nullptr;                    // mg_update_modulus: host E staged here (allocated once)
    long long Estage_n = 0;
    // mg_update_modulus returns once the operators are enqueued; the coarsest inverse's pivot status
    // is copied to h_setup_st behind them and checked by the next call (setup_check)
    int* h_setup_st = nullptr;
    cudaEvent_t ev_setup = nullptr;
    bool setup_pending = false;
    // mgcg_solve with host right-hand sides: uploaded on cs_in into rstage while the handle stream
    // still runs an earlier (deferred-checked) setup
    double* rstage = nullptr;
    long long rstage_n = 0;
    cudaEvent_t ev_rhs = nullptr;
    double* gstage = nullptr;                    // G(u) phi host-path staging
    long long gstage_cap = 0;
    // G(u) phi with host buffers on one slab: phi chunks copied in / y chunks copied out on two
    // copy streams while the previous chunk computes (duplex H2D / D2H overlapped with the kernel)
    cudaStream_t cs_in = nullptr, cs_out = nullptr;
    static constexpr int NCHUNK_EV = 8;
    cudaEvent_t gev_in[NCHUNK_EV] = {}, gev_k[NCHUNK_EV] = {};
    cudaEvent_t gev_sig = nullptr, gev_done = nullptr;
    double* wbuf = nullptr;                      // adjoint RHS element terms (nphi x m x nv)
    long long wbuf_cap = 0;
    double* dlam = nullptr;                      // eigenvalues for mg_eigen_sensitivity (MG_MAX_RHS)
    // block PCG workspace
    double *bpart = nullptr, *bGam = nullptr, *bRho = nullptr, *bRhoN = nullptr, *bC = nullptr;
    int* brank = nullptr;
    int block_R = 0;
    cudaGraphExec_t g_block = nullptr;
    cudaGraphExec_t g_gj = nullptr;   // coarsest assembly + Gauss-Jordan inverse (fixed shapes per handle)
    double block_tol = -1.0;
    double* xtmp = nullptr;                      // NCCL reverse-add receive buffer
    long long xtmp_cap = 0;
    // shared solve state
    int Ralloc = 0;
    double *stage = nullptr, *stage2 = nullptr;  // (R, n_rank) staging: host copies, L == 1 dense solve
    double* partial = nullptr;
    long long pst = 0;                           // partial stride per RHS
    double* sums = nullptr;                      // multi-rank dot sums
    CgCtl ctl{};
    void* ctl_mem = nullptr;
    int* h_pinned = nullptr;     // done, status, iters[64]
    double* h_dbl = nullptr;     // bb, rr, tt [64] each
    int* d_status = nullptr;
    cudaGraphExec_t g_init = nullptr, g_restart = nullptr, g_iter = nullptr, g_true = nullptr;
    cudaGraphExec_t g_loop = nullptr;   // device-side CG loop (conditional WHILE node around g_iter's body)
    long long n_init = 0, n_restart = 0, n_iter = 0, n_true = 0;
    int graph_R = -1;
    double graph_tol = -1.0;
    long long launches = 0;
};

static int nslab(const mg_ctx* c) { return (int)c->sl.size(); }
static bool multi(const mg_ctx* c) { return c->S > 1; }

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
    g.p2 = g.nn[2];
    g.vstr = g.ndof;
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

// ---------------------------------------------------------------- API scope
// The element constants (K0, K^, Q, H, D0) live in __constant__ memory, shared by every handle of
// the process.  Each entry point that launches work therefore (1) holds the process-wide API lock,
// (2) makes the constants those of its own handle -- a handle with another (dim, element, nu) first
// waits for ALL device work (no kernel of another handle may still be reading them), then uploads
// and waits for the upload -- and (3) joins the handle stream to the caller's stream on entry and
// the caller's stream back to the handle stream on every exit path (RAII).
static std::recursive_mutex g_api_mu;
static bool g_const_valid = false;
static int g_const_dim = 0, g_const_elem = -1;
static double g_const_nu = 0.0;

static mg_status ensure_constants(mg_ctx* c) {
    if (g_const_valid && g_const_dim == c->dim && g_const_elem == c->elem && g_const_nu == c->nu) return MG_OK;
    if (g_const_valid) CU(cudaDeviceSynchronize());
    g_const_valid = false;
    cudaStream_t s = c->stream;
    fine_set_constants(c->dim, c->K0.data(), s);
    if (c->dim == 3) h8t_set_constants(c->K0.data(), c->nu, s);
    if (c->dim == 2) fine2d_set_constants(c->K0.data(), s);
    galerkin_set_constants(c->dim, c->K0.data(), s);
    stress_set_constants(c->dim, c->nu, s);
    sens_set_constants(c->dim, c->K0.data(), c->nu, s);
    CU(cudaGetLastError());
    CU(cudaStreamSynchronize(s));
    g_const_valid = true;
    g_const_dim = c->dim;
    g_const_elem = c->elem;
    g_const_nu = c->nu;
    return MG_OK;
}

// NVTX ranges: one per C-ABI call (named after the function) and one per phase of a solve, for
// nsys / `ncu --nvtx` timelines.  Header-only NVTX3: without an attached tool a push / pop is a
// check of a null function pointer.
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    void next(const char* name) {   // close the current phase, open the next
        nvtxRangePop();
        nvtxRangePushA(name);
    }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};

static mg_status setup_check(mg_ctx* c);

struct ApiScope {
    NvtxRange nv;   // first member: the range spans the lock, the stream join and the call
    mg_ctx* c;
    std::lock_guard<std::recursive_mutex> lk;
    mg_status status;
    // defer: the caller runs setup_check itself (mgcg_solve: after enqueueing its host upload)
    ApiScope(mg_ctx* c_, const char* fn, bool defer = false) : nv(fn), c(c_), lk(g_api_mu), status(MG_OK) {
        stream_enter(c);
        status = ensure_constants(c);
        if (status == MG_OK && !defer) status = setup_check(c);
    }
    ~ApiScope() { stream_leave(c); }
    ApiScope(const ApiScope&) = delete;
    ApiScope& operator=(const ApiScope&) = delete;
};
#define API_SCOPE(c)                    \
    ApiScope api_scope_(c, __func__);   \
    TRY(api_scope_.status)
#define API_SCOPE_DEFER_SETUP(c)              \
    ApiScope api_scope_(c, __func__, true);   \
    TRY(api_scope_.status)

// ---------------------------------------------------------------- partition (host)
// Slab k of S gets a contiguous run of coarsest-level element layers (sizes differ by at
// most one), so every slab boundary is a node plane of every level.
static bool partition(int N0, int levels, int S, int k, int* e0, int* e1) {
    const int f = 1 << (levels - 1);
    const int Nc = N0 / f;
    if (S < 1 || k < 0 || k >= S || Nc < S) return false;
    const int base = Nc / S, rem = Nc % S;
    const int c0 = k * base + std::min(k, rem);
    const int c1 = c0 + base + (k < rem ? 1 : 0);
    *e0 = c0 * f;
    *e1 = c1 * f;
    return true;
}

// ---------------------------------------------------------------- plane fields
static PlaneField node_field(const Slab& s, int l, void* base, int esize, long long per_node, long long vec_stride,
                             int nvec) {
    const Level& v = s.lv[l];
    PlaneField f{};
    f.base = base;
    f.esize = esize;
    f.plane_len = v.pn * per_node;
    f.vec_stride = vec_stride;
    f.nvec = nvec;
    f.first_own = v.o0;
    f.last_own = v.o1 - 1;
    f.lo_ghost = s.gl ? 0 : -1;
    f.hi_ghost = s.gh ? v.g.nn[0] - 1 : -1;
    f.dirs = 3;
    return f;
}
// level-l compact vectors (R, ndof_local)
static PlaneField vec_field(mg_ctx* c, const Slab& s, int l, double* v, int R) {
    return node_field(s, l, v, 8, c->dim, s.lv[l].g.ndof, R);
}
// level-0 vectors: padded in 2D (ghost ring) and in 3D (row pitch)
static PlaneField fine_field(mg_ctx* c, const Slab& s, double* v, int R) {
    if (c->dim != 2) {
        PlaneField f = node_field(s, 0, v, 8, 3, s.p3.vstride, R);
        f.plane_len = 3LL * s.lv[0].g.nn[1] * s.p3.p2;
        return f;
    }
    PlaneField f = node_field(s, 0, v + 2 * s.pd.org, 8, 2, s.pd.vstride, R);
    f.plane_len = 2LL * s.pd.pitch;
    return f;
}
// element arrays (per-element records of `per_elem` doubles): ghost layer below only
static PlaneField elem_field(const Slab& s, int l, double* e, long long per_elem) {
    const LevelGeom& g = s.lv[l].g;
    PlaneField f{};
    f.base = e;
    f.esize = 8;
    f.plane_len = g.nelem / g.N[0] * per_elem;
    f.vec_stride = 0;
    f.nvec = 1;
    f.first_own = s.gl;
    f.last_own = g.N[0] - 1;
    f.lo_ghost = s.gl ? 0 : -1;
    f.hi_ghost = -1;
    f.dirs = 1;
    return f;
}

static mg_status xchg(mg_ctx* c, const std::function<PlaneField(const Slab&)>& fn) {
    if (!multi(c)) return MG_OK;
    std::vector<PlaneField> f;
    for (const Slab& s : c->sl) f.push_back(fn(s));
    COMM(halo_forward(c->comm, f.data(), nslab(c), c->stream));
    return MG_OK;
}
static mg_status xchg_add(mg_ctx* c, const std::function<PlaneField(const Slab&)>& fn) {
    if (!multi(c)) return MG_OK;
    std::vector<PlaneField> f;
    for (const Slab& s : c->sl) f.push_back(fn(s));
    COMM(halo_reverse_add(c->comm, f.data(), nslab(c), c->xtmp, c->stream));
    return MG_OK;
}

// ---------------------------------------------------------------- coarsest level (global)
// Gather the owned planes of a per-slab level-(L-1) field of nvec vectors into the global
// array dst (nvec, nglob_per_vec) with planes of plen doubles.
static mg_status gather_coarsest(mg_ctx* c, const std::function<double*(Slab&)>& src,
                                 const std::function<long long(const Slab&)>& src_stride, long long plen, int nvec,
                                 double* dst, long long dst_stride) {
    cudaStream_t st = c->stream;
    const int l = c->L - 1;
    if (c->comm.nranks <= 1) {
        for (Slab& s : c->sl) {
            const Level& v = s.lv[l];
            CU(cudaMemcpy2DAsync(dst + (long long)(v.gp0 + v.o0) * plen, dst_stride * 8, src(s) + v.o0 * plen,
                                 src_stride(s) * 8, (v.o1 - v.o0) * plen * 8, nvec, cudaMemcpyDeviceToDevice, st));
        }
        return MG_OK;
    }
    // cross-rank: pack this rank's owned planes (padded to the largest rank), all-gather, unpack
    const int f = 1 << l;
    int maxp = 0;
    for (int q = 0; q < c->comm.nranks; ++q) {
        const int np = (c->rank_p1[q] - c->rank_p0[q]) / f + (q == c->comm.nranks - 1 ? 1 : 0);
        maxp = std::max(maxp, np);
    }
    const long long chunk = (long long)maxp * plen;   // per vector
    const long long need = chunk * nvec;
    if (need > c->cpack_cap) return fail(MG_ERR_DIM, "coarsest gather buffer too small");
    const int pr0 = c->rank_p0[c->comm.rank] / f;
    for (Slab& s : c->sl) {
        const Level& v = s.lv[l];
        CU(cudaMemcpy2DAsync(c->cpack + (long long)(v.gp0 + v.o0 - pr0) * plen, chunk * 8, src(s) + v.o0 * plen,
                             src_stride(s) * 8, (v.o1 - v.o0) * plen * 8, nvec, cudaMemcpyDeviceToDevice, st));
    }
    COMM(comm_allgather(c->comm, c->cpack, c->cgath, (size_t)need * 8, st));
    for (int q = 0; q < c->comm.nranks; ++q) {
        const int p0 = c->rank_p0[q] / f;
        const int np = (c->rank_p1[q] - c->rank_p0[q]) / f + (q == c->comm.nranks - 1 ? 1 : 0);
        CU(cudaMemcpy2DAsync(dst + (long long)p0 * plen, dst_stride * 8, c->cgath + q * need, chunk * 8, np * plen * 8,
                             nvec, cudaMemcpyDeviceToDevice, st));
    }
    return MG_OK;
}

// z_{L-1} = A_{L-1}^{-1} r_{L-1}: gather the owned planes of every slab, one dense product
// (replicated on every rank), scatter all local planes (owned and ghost) back.
static mg_status coarsest_solve(mg_ctx* c, int R, const int* active, const int* done,
                                const std::function<double*(Slab&)>& rsrc, const std::function<double*(Slab&)>& zdst) {
    const int l = c->L - 1;
    if (!multi(c)) {
        Slab& s = c->sl[0];
        dense_apply(c->Ainv, c->npad, c->nL, rsrc(s), zdst(s), R, active, done, c->stream);
        c->launches++;
        return MG_OK;
    }
    const long long plen = c->G[l].nnodes / c->G[l].nn[0] * c->dim;
    TRY(gather_coarsest(c, rsrc, [&](const Slab& s) { return s.lv[l].g.ndof; }, plen, R, c->cr, c->nL));
    dense_apply(c->Ainv, c->npad, c->nL, c->cr, c->cz, R, active, done, c->stream);
    c->launches++;
    for (Slab& s : c->sl) {
        const Level& v = s.lv[l];
        CU(cudaMemcpy2DAsync(zdst(s), v.g.ndof * 8, c->cz + (long long)v.gp0 * plen, c->nL * 8, v.g.nn[0] * plen * 8, R,
                             cudaMemcpyDeviceToDevice, c->stream));
    }
    return MG_OK;
}

// ---------------------------------------------------------------- operators (per design)
// MG_GAL_WARP (default on): 3D level-1 Galerkin by a warp per coarse element for the elements whose
// fine nodes are all free (sum_c E_c M_c), the general kernel on the listed rest
static bool gal_warp() {
    static const bool v = !getenv("MG_GAL_WARP") || atoi(getenv("MG_GAL_WARP")) != 0;
    return v;
}

static mg_status compute_operators(mg_ctx* c, bool defer_check = false) {
    cudaStream_t s = c->stream;
    const int L = c->L, dim = c->dim;
    const int NL = dim * (1 << dim);
    // E ghost layers, modulus check
    TRY(xchg(c, [&](const Slab& sl) { return elem_field(sl, 0, sl.E, 1); }));
    CU(cudaMemsetAsync(c->d_status, 0, sizeof(int), s));
    for (Slab& sl : c->sl) {
        const long long m = sl.lv[0].g.nelem;
        check_modulus_kernel<<<(unsigned)((m + 255) / 256), 256, 0, s>>>(m, sl.E, c->d_status);
        c->launches++;
    }
    CHECK_LAUNCH();
    for (Slab& sl : c->sl) fine_diag(sl.lv[0].g, sl.E, sl.lv[0].mask, sl.lv[0].Dinv, sl.lv[0].D, s);
    c->launches += nslab(c);
    TRY(xchg(c, [&](const Slab& sl) { return node_field(sl, 0, sl.lv[0].Dinv, 8, dim, 0, 1); }));
    TRY(xchg(c, [&](const Slab& sl) { return node_field(sl, 0, sl.lv[0].D, 8, dim, 0, 1); }));
    if (dim == 3) {
        for (Slab& sl : c->sl) {
            pad3_nodes(sl.lv[0].g, sl.p3, sl.lv[0].mask, sl.maskpad, sl.lv[0].Dinv, sl.Dinvpad, s);
            if (sl.Epad) pad3_elems(sl.lv[0].g, sl.p3, sl.E, sl.Epad, s);
            c->launches += sl.Epad ? 2 : 1;
        }
    }
    if (dim == 2) {
        for (Slab& sl : c->sl) {
            pad2_elems(sl.lv[0].g, sl.pd, sl.E, sl.Epad, s);
            pad2_nodes_u8(sl.lv[0].g, sl.pd, sl.lv[0].mask, sl.maskpad, 3, s);
            pad2_nodes_f64(sl.lv[0].g, sl.pd, sl.lv[0].Dinv, sl.Dinvpad, s);
            c->launches += 3;
        }
    }
    CHECK_LAUNCH();
    if (L == 1) {   // single level (one slab): the fine operator is the coarsest
        Slab& sl = c->sl[0];
        elements_from_E(sl.lv[0].g, sl.E, sl.lv[0].mask, sl.elmA, s);
        stencil_from_elements(sl.lv[0].g, sl.elmA, sl.lv[0].mask, sl.lv[0].st, s);
        c->launches += 2;
        CHECK_LAUNCH();
    }
    for (int l = 1; l < L; ++l) {
        for (Slab& sl : c->sl) {
            Level& f = sl.lv[l - 1];
            Level& g = sl.lv[l];
            double* elm = (l & 1) ? sl.elmA : sl.elmB;
            double* elm_prev = (l & 1) ? sl.elmB : sl.elmA;
            // level 1 (3D): the list of masked coarse elements lives in the idle level-2 buffer
            int* ws = (l == 1 && c->dim == 3 && gal_warp()) ? reinterpret_cast<int*>(sl.elmB) : nullptr;
            galerkin_elements(g.g, f.g, l == 1 ? sl.E : nullptr, elm_prev, f.mask, g.mask, elm, s, sl.gl, c->Mc, ws);
            c->launches++;
        }
        CHECK_LAUNCH();
        TRY(xchg(c, [&](const Slab& sl) { return elem_field(sl, l, (l & 1) ? sl.elmA : sl.elmB, NL * NL); }));
        for (Slab& sl : c->sl) {
            Level& g = sl.lv[l];
            double* elm = (l & 1) ? sl.elmA : sl.elmB;
            stencil_from_elements(g.g, elm, g.mask, g.st, s);
            stencil_diag(g.g, g.st, g.mask, g.st, g.Dinv, g.D, s);
            c->launches += 2;
        }
        CHECK_LAUNCH();
        TRY(xchg(c, [&](const Slab& sl) { return node_field(sl, l, sl.lv[l].mask, 1, 1, 0, 1); }));
        TRY(xchg(c, [&](const Slab& sl) { return node_field(sl, l, sl.lv[l].Dinv, 8, dim, 0, 1); }));
        TRY(xchg(c, [&](const Slab& sl) { return node_field(sl, l, sl.lv[l].D, 8, dim, 0, 1); }));
    }
    // coarsest dense inverse (global coarsest operator on every rank)
    const LevelGeom& gL = c->G[L - 1];
    const int ns = dim == 2 ? 9 : 27;
    const double* stc = c->sl[0].lv[L - 1].st;
    if (multi(c)) {
        TRY(gather_coarsest(c, [&](Slab& sl) { return sl.lv[L - 1].st; },
                            [&](const Slab& sl) { return sl.lv[L - 1].g.nnodes; }, gL.nnodes / gL.nn[0],
                            ns * dim * dim, c->stg, gL.nnodes));
        stc = c->stg;
    }
    // ~4 launches per 32-column block step: captured once into a graph (the shapes and buffers are
    // fixed for the handle) so a setup pays graph-node rather than stream-launch overhead
    if (!c->g_gj) {
        CU(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
        cudaMemsetAsync(c->Ainv, 0, sizeof(double) * c->npad * c->npad, s);
        dense_from_stencil(gL, stc, c->Ainv, c->npad, s);
        dense_pad_identity(c->Ainv, c->nL, c->npad, s);
        cudaMemsetAsync(c->gj_work, 0, sizeof(double) * (2 * 32 * 32 + 2 * c->npad * 32), s);
        dense_spd_inverse(c->Ainv, c->npad, c->gj_work, c->d_status, s);
        cudaGraph_t gg = nullptr;
        CU(cudaStreamEndCapture(s, &gg));
        CU(cudaGraphInstantiate(&c->g_gj, gg, 0));
        CU(cudaGraphDestroy(gg));
    }
    CU(cudaGraphLaunch(c->g_gj, s));
    c->launches += (c->npad > c->nL ? 2 : 1) + dense_spd_inverse_launches(c->npad);
    CHECK_LAUNCH();
    if (defer_check) {   // status read back behind the operators, checked by the next call
        if (!c->h_setup_st) CU(cudaMallocHost(&c->h_setup_st, sizeof(int)));
        if (!c->ev_setup) CU(cudaEventCreateWithFlags(&c->ev_setup, cudaEventDisableTiming));
        CU(cudaMemcpyAsync(c->h_setup_st, c->d_status, sizeof(int), cudaMemcpyDeviceToHost, s));
        CU(cudaEventRecord(c->ev_setup, s));
        c->setup_pending = true;
        return MG_OK;
    }
    int st[1] = {0};
    CU(cudaMemcpyAsync(st, c->d_status, sizeof(int), cudaMemcpyDeviceToHost, s));
    CU(cudaStreamSynchronize(s));
    if (st[0] & 4) return fail(MG_ERR_MODULUS, "E_e must be positive and finite");
    if (st[0]) return fail(MG_ERR_SINGULAR, "coarsest operator: non-positive pivot in the SPD inverse");
    return MG_OK;
}

// copy streams and their events (host-buffer pipelines of G(u) phi and of the solve's upload)
static mg_status ensure_copy_streams(mg_ctx* c) {
    if (c->cs_in) return MG_OK;
    CU(cudaStreamCreateWithFlags(&c->cs_in, cudaStreamNonBlocking));
    CU(cudaStreamCreateWithFlags(&c->cs_out, cudaStreamNonBlocking));
    for (int k = 0; k < mg_ctx::NCHUNK_EV; ++k) {
        CU(cudaEventCreateWithFlags(&c->gev_in[k], cudaEventDisableTiming));
        CU(cudaEventCreateWithFlags(&c->gev_k[k], cudaEventDisableTiming));
    }
    CU(cudaEventCreateWithFlags(&c->gev_sig, cudaEventDisableTiming));
    CU(cudaEventCreateWithFlags(&c->gev_done, cudaEventDisableTiming));
    CU(cudaEventCreateWithFlags(&c->ev_rhs, cudaEventDisableTiming));
    return MG_OK;
}

// pivot status of a deferred-checked setup (mg_update_modulus): waits for the operators
static mg_status setup_check(mg_ctx* c) {
    if (!c->setup_pending) return MG_OK;
    c->setup_pending = false;
    CU(cudaEventSynchronize(c->ev_setup));
    const int st = *c->h_setup_st;
    if (st & 4) return fail(MG_ERR_MODULUS, "E_e must be positive and finite");
    if (st) return fail(MG_ERR_SINGULAR, "coarsest operator: non-positive pivot in the SPD inverse (last mg_update_modulus)");
    return MG_OK;
}

static void free_vectors(mg_ctx* c) {
    for (Slab& s : c->sl) {
        double** fv[] = {&s.b, &s.x, &s.r0, &s.r1, &s.p0, &s.p1, &s.q, &s.zf, &s.z, &s.t};
        for (auto p : fv)
            if (*p) { cudaFree(*p); *p = nullptr; }
        for (int l = 1; l < c->L; ++l) {
            double** lvv[] = {&s.lv[l].r, &s.lv[l].z, &s.lv[l].w};
            for (auto p : lvv)
                if (*p) { cudaFree(*p); *p = nullptr; }
        }
    }
    double** cv[] = {&c->partial, &c->stage, &c->stage2, &c->cr, &c->cz, &c->xtmp};
    for (auto p : cv)
        if (*p) { cudaFree(*p); *p = nullptr; }
    cudaGraphExec_t* gs[] = {&c->g_init, &c->g_restart, &c->g_iter, &c->g_true, &c->g_loop, &c->g_block};
    for (auto g : gs)
        if (*g) { cudaGraphExecDestroy(*g); *g = nullptr; }
    c->graph_R = -1;
    c->block_tol = -1.0;   // the block-PCG graph referenced the freed vectors: recapture
    c->Ralloc = 0;
}

static mg_status ensure_vectors(mg_ctx* c, int R) {
    if (R <= c->Ralloc) return MG_OK;
    CU(cudaStreamSynchronize(c->stream));
    free_vectors(c);
    long long pst = 0, xplane = 0;
    for (Slab& s : c->sl) {
        const long long n = s.vs;
        double** fv[] = {&s.b, &s.x, &s.r0, &s.r1, &s.p0, &s.p1, &s.q, &s.zf, &s.z, &s.t};
        for (auto p : fv) {
            CU(cudaMalloc(p, sizeof(double) * n * R));
            CU(cudaMemset(*p, 0, sizeof(double) * n * R));   // ghost entries of the padded layout stay 0
        }
        for (int l = 1; l < c->L; ++l) {
            long long nl = s.lv[l].g.ndof;
            CU(cudaMalloc(&s.lv[l].r, sizeof(double) * nl * R));
            CU(cudaMalloc(&s.lv[l].z, sizeof(double) * nl * R));
            CU(cudaMalloc(&s.lv[l].w, sizeof(double) * nl * R));
            CU(cudaMemset(s.lv[l].r, 0, sizeof(double) * nl * R));
            CU(cudaMemset(s.lv[l].z, 0, sizeof(double) * nl * R));
            CU(cudaMemset(s.lv[l].w, 0, sizeof(double) * nl * R));
            xplane = std::max(xplane, s.lv[l].pn * c->dim);
        }
        long long items = fine_items(s.lv[0].g, R);
        if (c->dim == 2) {
            for (int op : {M2_CGP, M2_RESTRICT, M2_POST, M2_RESID, M2_JACOBI}) {
                long long it = march2_items(op, s.lv[0].g, c->L > 1 ? &s.lv[1].g : &s.lv[0].g, R);
                items = std::max(items, it);
            }
        }
        items = std::max<long long>(items, vec_blocks(n));
        pst += items;
    }
    c->pst = pst;
    CU(cudaMalloc(&c->partial, sizeof(double) * c->pst * R));
    CU(cudaMalloc(&c->stage, sizeof(double) * c->n_rank * R));
    CU(cudaMalloc(&c->stage2, sizeof(double) * c->n_rank * R));
    if (multi(c)) {
        CU(cudaMalloc(&c->cr, sizeof(double) * c->nL * R));
        CU(cudaMalloc(&c->cz, sizeof(double) * c->nL * R));
        c->xtmp_cap = xplane * R;
        CU(cudaMalloc(&c->xtmp, sizeof(double) * std::max<long long>(c->xtmp_cap, 1)));
        // packed halo messages: the largest vector plane (level 0 included) times R
        long long p0 = 0;
        for (const Slab& s : c->sl) {
            const LevelGeom& g0 = s.lv[0].g;
            p0 = std::max(p0, c->dim == 2 ? 2LL * s.pd.pitch : 3LL * g0.nn[1] * s.p3.p2);
        }
        if (!comm_reserve(c->comm, sizeof(double) * std::max(p0, xplane) * R))
            return fail(MG_ERR_OOM, comm_last_error());
    }
    c->Ralloc = R;
    return MG_OK;
}

// ---------------------------------------------------------------- user vectors <-> slabs
// user (R, n_rank) owned planes of this rank -> level-0 slab vectors (+ ghost exchange)
static mg_status scatter_fine(mg_ctx* c, const double* src, int R, bool masked, double* Slab::*dst) {
    for (Slab& s : c->sl) {
        const Level& v = s.lv[0];
        const int np = v.o1 - v.o0;
        if (c->dim == 2) {
            pad2_vectors_planes(v.g, s.pd, R, masked ? v.mask : nullptr, v.o0, np, src + 2 * s.uoff, c->n_rank,
                                s.*dst, c->stream);
        } else {
            pad3_vectors_planes(v.g, s.p3, R, masked ? v.mask : nullptr, v.o0, np, src + 3 * s.uoff, c->n_rank,
                                s.*dst, c->stream);
        }
        c->launches++;
    }
    return xchg(c, [&](const Slab& s) { return fine_field(c, s, s.*dst, R); });
}

// level-0 slab vectors (owned planes) -> user (R, n_rank)
static mg_status gather_fine(mg_ctx* c, double* Slab::*src, int R, double* dst) {
    for (Slab& s : c->sl) {
        const Level& v = s.lv[0];
        const int np = v.o1 - v.o0;
        if (c->dim == 2) {
            unpad2_vectors_planes(v.g, s.pd, R, v.o0, np, s.*src, dst + 2 * s.uoff, c->n_rank, c->stream);
            c->launches++;
        } else {
            unpad3_vectors_planes(v.g, s.p3, R, v.o0, np, s.*src, dst + 3 * s.uoff, c->n_rank, c->stream);
            c->launches++;
        }
    }
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

static FineArgs fine_args(mg_ctx* c, const Slab& s, const Rec& rc) {
    FineArgs a{};
    a.g = s.lv[0].g; a.E = s.E; a.mask = s.lv[0].mask; a.omega = c->opts.omega;
    if (c->dim == 3) {   // padded 3D fine layout (h8t.cu)
        a.g = s.g0p; a.E = s.Epad ? s.Epad : s.E; a.mask = s.maskpad; a.Dinv = s.Dinvpad;
        a.ep2 = s.p3.ep2; a.m2 = s.p3.m2;
    }
    a.active = rc.active; a.done = rc.done; a.R = rc.R; a.nu_paper = c->nu_paper ? 1 : 0;
    a.so0 = s.lv[0].o0; a.so1 = s.lv[0].o1; a.pstride = c->pst;
    return a;
}

static March2Args march_args(mg_ctx* c, const Slab& s, const Rec& rc) {
    March2Args a{};
    a.g = s.lv[0].g;
    if (c->L > 1) { a.gc = s.lv[1].g; a.maskc = s.lv[1].mask; }
    a.pd = s.pd; a.E = s.Epad; a.mask = s.maskpad; a.Dinv = s.Dinvpad; a.omega = c->opts.omega;
    a.alpha = c->ctl.alpha; a.beta = c->ctl.beta; a.xalpha = c->ctl.xalpha;
    a.active = rc.active; a.done = rc.done; a.R = rc.R;
    a.so0 = s.lv[0].o0; a.so1 = s.lv[0].o1; a.off0 = s.gl; a.pstride = c->pst;
    return a;
}

// Level-0 operator application: 2D through the padded march kernels, 3D through fine_ops.
static int level0_apply(mg_ctx* c, const Slab& s, int op, const FineArgs& f) {
    if (c->dim != 2) return fine_apply(op, f, c->stream);
    Rec rc{c, f.R, f.active, f.done};
    March2Args m = march_args(c, s, rc);
    m.omega = f.omega; m.partial = f.partial;
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

// owned entries [d0, d1) of a level-0 vector (for dots)
static void fine_own_range(mg_ctx* c, const Slab& s, long long* d0, long long* d1) {
    const Level& v = s.lv[0];
    if (c->dim == 2) {
        *d0 = 2 * (s.pd.org + (long long)v.o0 * s.pd.pitch);
        *d1 = 2 * (s.pd.org + (long long)v.o1 * s.pd.pitch);
    } else {
        *d0 = 3LL * v.o0 * v.g.nn[1] * s.p3.p2;
        *d1 = 3LL * v.o1 * v.g.nn[1] * s.p3.p2;
    }
}

// consume the dot partials (items per RHS, stride c->pst) with a scalar CG step; across ranks
// the per-RHS sums are all-reduced first
static mg_status finish_dots(mg_ctx* c, int mode, int R, long long items, int aux = 0, double tol = 0.0) {
    if (c->comm.nranks > 1) {
        reduce_partials(R, c->partial, (int)items, c->pst, c->sums, c->stream);
        COMM(comm_allreduce_sum(c->comm, c->sums, R, c->stream));
        cg_scalars(mode, R, c->sums, 1, c->ctl, tol, c->stream, aux, 1);
        c->launches += 2;
    } else {
        cg_scalars(mode, R, c->partial, (int)items, c->ctl, tol, c->stream, aux, c->pst);
        c->launches++;
    }
    return MG_OK;
}

static void level_smooth(Rec& rc, Slab& s, int l, const double* r, const double* z, double* w, double* partial) {
    mg_ctx* c = rc.c;
    if (l == 0 && c->L > 1) {
        FineArgs a = fine_args(c, s, rc);
        a.x = z; a.b = r; a.Dinv = s.Dinvpad; a.y = w; a.partial = partial;
        level0_apply(c, s, FOP_JACOBI, a);
    } else {
        CoarseArgs a{};
        a.g = s.lv[l].g; a.st = s.lv[l].st; a.x = z; a.b = r; a.Dinv = s.lv[l].Dinv; a.y = w;
        a.omega = c->opts.omega; a.active = rc.active; a.done = rc.done; a.R = rc.R;
        coarse_apply(COP_JACOBI, a, c->stream);
    }
    rc.launches++;
}

static void level_resid(Rec& rc, Slab& s, int l, const double* r, const double* z, double* w) {
    mg_ctx* c = rc.c;
    if (l == 0) {
        FineArgs a = fine_args(c, s, rc);
        a.x = z; a.b = r; a.y = w;
        level0_apply(c, s, FOP_RESID, a);
    } else {
        CoarseArgs a{};
        a.g = s.lv[l].g; a.st = s.lv[l].st; a.x = z; a.b = r; a.y = w;
        a.active = rc.active; a.done = rc.done; a.R = rc.R;
        coarse_apply(COP_RESID, a, c->stream);
    }
    rc.launches++;
}

// Symmetric V(nu_pre, nu_post)-cycle on level l >= 1 of every slab: z ~ A_l^-1 r, with r
// owned-valid on entry (ghosts exchanged here) and z valid on all local planes on exit.
// Per slab the result is in z or w (same choice on every slab); returns 0 for z, 1 for w.
static mg_status vcycle(Rec& rc, int l, int* which) {
    mg_ctx* c = rc.c;
    const int R = rc.R;
    if (l == c->L - 1) {
        TRY(coarsest_solve(c, R, rc.active, rc.done, [&](Slab& s) { return s.lv[l].r; },
                           [&](Slab& s) { return s.lv[l].z; }));
        rc.launches++;
        *which = 0;
        return MG_OK;
    }
    TRY(xchg(c, [&](const Slab& s) { return vec_field(c, s, l, s.lv[l].r, R); }));
    if (c->dim == 2 && c->opts.nu_pre == 1 && c->opts.nu_post == 1 && !c->unfused_coarse) {
        // fused V(1,1) halves (coarse2d.cu)
        for (Slab& s : c->sl) {
            Level& f = s.lv[l];
            Level& nx = s.lv[l + 1];
            coarse2d_down(f.g, nx.g, f.st, f.Dinv, f.mask, nx.mask, f.r, nx.r, R, c->opts.omega, s.gl, f.o0, f.o1,
                          rc.active, rc.done, c->stream);
            rc.launches++;
        }
        TRY(xchg_add(c, [&](const Slab& s) { return vec_field(c, s, l + 1, s.lv[l + 1].r, R); }));
        int cw = 0;
        TRY(vcycle(rc, l + 1, &cw));
        for (Slab& s : c->sl) {
            Level& f = s.lv[l];
            Level& nx = s.lv[l + 1];
            coarse2d_up(f.g, nx.g, f.st, f.Dinv, f.mask, nx.mask, f.r, cw ? nx.w : nx.z, f.z, R, c->opts.omega, s.gl,
                        rc.active, rc.done, c->stream);
            rc.launches++;
        }
        TRY(xchg(c, [&](const Slab& s) { return vec_field(c, s, l, s.lv[l].z, R); }));
        *which = 0;
        return MG_OK;
    }
    int zi = 0;   // 0: z holds the iterate, 1: w
    auto zb = [&](Slab& s) { return zi ? s.lv[l].w : s.lv[l].z; };
    auto wb = [&](Slab& s) { return zi ? s.lv[l].z : s.lv[l].w; };
    for (Slab& s : c->sl) {
        cg_pointwise_jacobi(s.lv[l].g.ndof, R, s.lv[l].r, s.lv[l].Dinv, c->opts.omega, s.lv[l].z, rc.active, rc.done,
                            c->stream);
        rc.launches++;
    }
    for (int it = 1; it < c->opts.nu_pre; ++it) {
        TRY(xchg(c, [&](const Slab& s) { return vec_field(c, s, l, zi ? s.lv[l].w : s.lv[l].z, R); }));
        for (Slab& s : c->sl) level_smooth(rc, s, l, s.lv[l].r, zb(s), wb(s), nullptr);
        zi ^= 1;
    }
    if (c->opts.nu_pre > 1)
        TRY(xchg(c, [&](const Slab& s) { return vec_field(c, s, l, zi ? s.lv[l].w : s.lv[l].z, R); }));
    for (Slab& s : c->sl) {
        level_resid(rc, s, l, s.lv[l].r, zb(s), wb(s));
        Level& f = s.lv[l];
        Level& nx = s.lv[l + 1];
        restrict_apply(f.g, nx.g, f.mask, nx.mask, wb(s), nx.r, R, rc.active, rc.done, c->stream, s.gl, f.o0, f.o1);
        rc.launches++;
    }
    TRY(xchg_add(c, [&](const Slab& s) { return vec_field(c, s, l + 1, s.lv[l + 1].r, R); }));
    int cw = 0;
    TRY(vcycle(rc, l + 1, &cw));
    for (Slab& s : c->sl) {
        Level& f = s.lv[l];
        Level& nx = s.lv[l + 1];
        prolong_add(f.g, nx.g, f.mask, nx.mask, cw ? nx.w : nx.z, zb(s), R, rc.active, rc.done, true, c->stream, s.gl);
        rc.launches++;
    }
    for (int it = 0; it < c->opts.nu_post; ++it) {
        if (it > 0) TRY(xchg(c, [&](const Slab& s) { return vec_field(c, s, l, zi ? s.lv[l].w : s.lv[l].z, R); }));
        for (Slab& s : c->sl) level_smooth(rc, s, l, s.lv[l].r, zb(s), wb(s), nullptr);
        zi ^= 1;
    }
    if (c->opts.nu_post > 0)
        TRY(xchg(c, [&](const Slab& s) { return vec_field(c, s, l, zi ? s.lv[l].w : s.lv[l].z, R); }));
    *which = zi;
    return MG_OK;
}

// ---- fine-level blocks of one CG iteration (fused kernels in 2D, composed kernels otherwise)
// p_out = zf + beta p_in ; q = K p_out ; partial p.q ; x += xalpha p_in.  Then q ghosts.
static mg_status blk_cgp(Rec& rc, double* Slab::*pin, double* Slab::*pout, long long* items) {
    mg_ctx* c = rc.c;
    long long off = 0;
    for (Slab& s : c->sl) {
        FineArgs a = fine_args(c, s, rc);
        a.z = s.zf; a.pin = s.*pin; a.pout = s.*pout; a.y = s.q; a.beta = c->ctl.beta;
        a.xv = s.x; a.xalpha = c->ctl.xalpha; a.partial = c->partial + off;
        off += level0_apply(c, s, FOP_CGP, a);
        rc.launches++;
    }
    *items = off;
    return MG_OK;
}

static bool z2_in_post() {
    static const bool v = !getenv("MG_Z2_IN_POST") || atoi(getenv("MG_Z2_IN_POST")) != 0;
    return v;
}

static bool z1_from_r() {
    static const bool v = !getenv("MG_Z1_FROM_R") || atoi(getenv("MG_Z1_FROM_R")) != 0;
    return v;
}

// r_out = r_in - alpha q ; partial r.r ; pre-smooth z1 = omega D^-1 r_out ; r_1 = P^T (r_out - K z1)
static mg_status blk_restrict(Rec& rc, double* Slab::*rin, double* Slab::*rout, long long* items) {
    mg_ctx* c = rc.c;
    const int R = rc.R;
    TRY(xchg(c, [&](const Slab& s) { return fine_field(c, s, s.q, R); }));
    long long off = 0;
    if (c->fused2d) {
        for (Slab& s : c->sl) {
            March2Args a = march_args(c, s, rc);
            a.x = s.*rin; a.x2 = s.q; a.y2 = s.*rout; a.coarse = s.lv[1].r; a.partial = c->partial + off;
            off += march2_apply(M2_RESTRICT, a, c->nu_paper, c->stream);
            rc.launches++;
        }
        *items = off;
        return xchg_add(c, [&](const Slab& s) { return vec_field(c, s, 1, s.lv[1].r, R); });
    }
    if (c->fused3d) {
        // 3D: r = rin - alpha q, r.r, t = r - K (omega D^-1 r) in one h8 kernel, then P^T t
        for (Slab& s : c->sl) {
            FineArgs a = fine_args(c, s, rc);
            a.rin = s.*rin; a.q = s.q; a.rout = s.*rout; a.alpha = c->ctl.alpha; a.Dinv = s.Dinvpad;
            a.y = s.t; a.partial = c->partial + off;
            // the post-smoother starts from z1 + P e; with the pair prolongation z1 = omega D^-1 r is
            // formed there from r (MG_Z1_FROM_R=0: stored here)
            s.z1_from_r = z1_from_r() && prolong_from_r_ok(s.g0p, s.lv[1].g, s.z);
            a.z1out = s.z1_from_r ? nullptr : s.z;
            s.zpre = s.z;
            off += fine_apply(FOP_RESTR3, a, c->stream);
            rc.launches++;
        }
        *items = off;
        for (Slab& s : c->sl) {
            restrict_apply(s.g0p, s.lv[1].g, s.lv[0].mask, s.lv[1].mask, s.t, s.lv[1].r, R, rc.active, rc.done,
                           c->stream, s.gl, s.lv[0].o0, s.lv[0].o1);
            rc.launches++;
        }
        return xchg_add(c, [&](const Slab& s) { return vec_field(c, s, 1, s.lv[1].r, R); });
    }
    for (Slab& s : c->sl) {
        long long d0, d1;
        fine_own_range(c, s, &d0, &d1);
        off += cg_rupdate(s.vs, R, c->ctl.alpha, s.*rin, s.q, s.*rout, s.Dinvpad,
                          c->opts.omega, c->L > 1 ? s.z : nullptr, c->partial + off, c->pst, d0, d1, rc.active,
                          rc.done, c->stream);
        rc.launches++;
    }
    *items = off;
    if (c->L == 1) return MG_OK;
    int zi = 0;
    for (int it = 1; it < c->opts.nu_pre; ++it) {
        TRY(xchg(c, [&](const Slab& s) { return fine_field(c, s, zi ? s.t : s.z, R); }));
        for (Slab& s : c->sl) level_smooth(rc, s, 0, s.*rout, zi ? s.t : s.z, zi ? s.z : s.t, nullptr);
        zi ^= 1;
    }
    if (c->opts.nu_pre > 1) TRY(xchg(c, [&](const Slab& s) { return fine_field(c, s, zi ? s.t : s.z, R); }));
    for (Slab& s : c->sl) {
        double* z = zi ? s.t : s.z;
        double* w = zi ? s.z : s.t;
        level_resid(rc, s, 0, s.*rout, z, w);
        restrict_apply(c->dim == 3 ? s.g0p : s.lv[0].g, s.lv[1].g, s.lv[0].mask, s.lv[1].mask, w, s.lv[1].r, R, rc.active, rc.done,
                       c->stream, s.gl, s.lv[0].o0, s.lv[0].o1);
        rc.launches++;
        s.zpre = z;
    }
    return xchg_add(c, [&](const Slab& s) { return vec_field(c, s, 1, s.lv[1].r, R); });
}

// levels 1..L-1 of the V-cycle on lv[1].r; *which: 0 -> lv[1].z, 1 -> lv[1].w
static mg_status coarse_cycle(Rec& rc, int* which) {
    *which = 0;
    if (rc.c->L == 1) return MG_OK;
    return vcycle(rc, 1, which);
}

// zf = post-smoothed (z1 + P ec) ; partial r.zf ; then zf ghosts.
static mg_status blk_post(Rec& rc, double* Slab::*r, int cw, long long* items) {
    mg_ctx* c = rc.c;
    const int R = rc.R;
    long long off = 0;
    if (c->L == 1) {   // single slab: dense solve on the compact layout
        Slab& s = c->sl[0];
        if (c->dim == 2) {
            unpad2_vectors(s.lv[0].g, s.pd, R, s.*r, c->stage, c->stream);
            dense_apply(c->Ainv, c->npad, c->nL, c->stage, c->stage2, R, rc.active, rc.done, c->stream);
            pad2_vectors(s.lv[0].g, s.pd, R, nullptr, c->stage2, s.zf, c->stream);
            rc.launches += 2;
        } else {
            const LevelGeom& g0 = s.lv[0].g;
            unpad3_vectors_planes(g0, s.p3, R, 0, g0.nn[0], s.*r, c->stage, g0.ndof, c->stream);
            dense_apply(c->Ainv, c->npad, c->nL, c->stage, c->stage2, R, rc.active, rc.done, c->stream);
            pad3_vectors_planes(g0, s.p3, R, nullptr, 0, g0.nn[0], c->stage2, g0.ndof, s.zf, c->stream);
            rc.launches += 2;
        }
        off = vec_dot_range(s.vs, 0, s.vs, R, s.*r, s.zf, c->partial, c->pst, rc.active, rc.done, c->stream);
        rc.launches += 2;
        *items = off;
        return MG_OK;
    }
    if (c->fused2d) {
        for (Slab& s : c->sl) {
            March2Args a = march_args(c, s, rc);
            a.x = s.*r; a.ec = cw ? s.lv[1].w : s.lv[1].z; a.y = s.zf; a.partial = c->partial + off;
            off += march2_apply(M2_POST, a, c->nu_paper, c->stream);
            rc.launches++;
        }
        *items = off;
        return xchg(c, [&](const Slab& s) { return fine_field(c, s, s.zf, R); });
    }
    // MG_Z2_IN_POST (default on): with z1 = omega D^-1 r not stored, the prolongation writes only the
    // correction P e and the first post-smoothing sweep forms z2 = P e + omega D^-1 r from the r and
    // D^-1 it reads anyway (the prolongation no longer reads them: one fine R-vector + D^-1 less)
    bool z2post = false;
    for (Slab& s : c->sl) {
        const bool zp = c->dim == 3 && s.z1_from_r && c->opts.nu_post > 0 && z2_in_post();
        z2post = zp;   // same decision on every slab (same level-0 layout rules)
        prolong_add(c->dim == 3 ? s.g0p : s.lv[0].g, s.lv[1].g, s.lv[0].mask, s.lv[1].mask, cw ? s.lv[1].w : s.lv[1].z, s.zpre, R,
                    rc.active, rc.done, !zp, c->stream, s.gl, (s.z1_from_r && !zp) ? s.*r : nullptr, s.Dinvpad,
                    c->opts.omega);
        s.z1_from_r = false;
        rc.launches++;
    }
    if (c->opts.nu_post == 0) {
        for (Slab& s : c->sl) {
            CU(cudaMemcpyAsync(s.zf, s.zpre, sizeof(double) * s.vs * R, cudaMemcpyDeviceToDevice, c->stream));
            long long d0, d1;
            fine_own_range(c, s, &d0, &d1);
            off += vec_dot_range(s.vs, d0, d1, R, s.*r, s.zf, c->partial + off, c->pst, rc.active, rc.done, c->stream);
            rc.launches++;
        }
        *items = off;
        return MG_OK;   // zf = zpre is ghost-valid (prolongation is local)
    }
    // post sweeps: src -> dst, the last one into zf with the r.zf dot
    std::vector<double*> src(nslab(c));
    for (int k = 0; k < nslab(c); ++k) src[k] = c->sl[k].zpre;
    for (int it = 0; it < c->opts.nu_post; ++it) {
        const bool last = it == c->opts.nu_post - 1;
        if (it > 0) {
            std::vector<PlaneField> f;
            for (int k = 0; k < nslab(c); ++k) f.push_back(fine_field(c, c->sl[k], src[k], R));
            if (multi(c)) COMM(halo_forward(c->comm, f.data(), nslab(c), c->stream));
        }
        off = 0;
        for (int k = 0; k < nslab(c); ++k) {
            Slab& s = c->sl[k];
            double* dst = last ? s.zf : (src[k] == s.z ? s.t : s.z);
            FineArgs a = fine_args(c, s, rc);
            a.x = src[k]; a.b = s.*r; a.Dinv = s.Dinvpad; a.y = dst; a.partial = last ? c->partial + off : nullptr;
            a.z1r = (it == 0 && z2post) ? 1 : 0;
            off += level0_apply(c, s, FOP_JACOBI, a);
            rc.launches++;
            src[k] = dst;
        }
    }
    *items = off;
    return xchg(c, [&](const Slab& s) { return fine_field(c, s, s.zf, R); });
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

// abort an open capture on error so the stream stays usable
static mg_status captured(mg_ctx* c, mg_status st) {
    if (st != MG_OK) {
        cudaGraph_t g = nullptr;
        cudaStreamEndCapture(c->stream, &g);
        if (g) cudaGraphDestroy(g);
        cudaGetLastError();
    }
    return st;
}

// b.b over owned entries (all slabs) -> SM_BB
static mg_status dot_finish(mg_ctx* c, int R, double* Slab::*a, double* Slab::*b, int mode) {
    long long off = 0;
    for (Slab& s : c->sl) {
        long long d0, d1;
        fine_own_range(c, s, &d0, &d1);
        off += vec_dot_range(s.vs, d0, d1, R, s.*a, s.*b, c->partial + off, c->pst, nullptr, nullptr, c->stream);
        c->launches++;
    }
    return finish_dots(c, mode, R, off);
}

// Graphs (captured once per (R, tol)):
//   init    : b.b, x = 0, p0 = 0, q = 0, r1 = b
//   restart : z = B r (r1 -> r0, alpha = 0), r.z            (start and true-residual restarts)
//   iter    : two CG iterations (p and r ping-pong buffers)
//   true    : flush deferred x update, t = b - K x, t.t
static mg_status record_restart(mg_ctx* c, int R) {
    Rec rc{c, R, c->ctl.active, c->ctl.done};
    long long k;
    TRY(blk_restrict(rc, &Slab::r1, &Slab::r0, &k));
    int cw;
    TRY(coarse_cycle(rc, &cw));
    TRY(blk_post(rc, &Slab::r0, cw, &k));
    return finish_dots(c, SM_RZ0, R, k);
}

static mg_status record_iter(mg_ctx* c, int R, double tol) {
    Rec rc{c, R, c->ctl.active, c->ctl.done};
    for (int it = 0; it < 2; ++it) {
        double* Slab::*pin = it == 0 ? &Slab::p0 : &Slab::p1;
        double* Slab::*pout = it == 0 ? &Slab::p1 : &Slab::p0;
        double* Slab::*rin = it == 0 ? &Slab::r0 : &Slab::r1;
        double* Slab::*rout = it == 0 ? &Slab::r1 : &Slab::r0;
        long long k;
        TRY(blk_cgp(rc, pin, pout, &k));
        TRY(finish_dots(c, SM_ALPHA, R, k, pout == &Slab::p1 ? 1 : 0));
        TRY(blk_restrict(rc, rin, rout, &k));
        const bool merged = c->comm.nranks > 1;
        if (merged) {   // r.r partials -> sums[0, R); all-reduced together with r.z below
            reduce_partials(R, c->partial, (int)k, c->pst, c->sums, c->stream);
            c->launches++;
        } else {
            TRY(finish_dots(c, SM_CONV, R, k, 0, tol));
        }
        int cw;
        TRY(coarse_cycle(rc, &cw));
        TRY(blk_post(rc, rout, cw, &k));
        if (merged) {
            // one allreduce of [r.r | r.z] per iteration (plus alpha's): the convergence test and
            // beta are taken together after the post-smoother; an RHS that converged in this
            // iteration ran one V-cycle it did not need (its result is never used)
            reduce_partials(R, c->partial, (int)k, c->pst, c->sums + R, c->stream);
            COMM(comm_allreduce_sum(c->comm, c->sums, 2 * R, c->stream));
            cg_scalars(SM_CONV, R, c->sums, 1, c->ctl, tol, c->stream, 0, 1);
            cg_scalars(SM_BETA, R, c->sums + R, 1, c->ctl, 0.0, c->stream, 0, 1);
            c->launches += 3;
        } else {
            TRY(finish_dots(c, SM_BETA, R, k));
        }
    }
    return MG_OK;
}

static mg_status record_true(mg_ctx* c, int R) {
    for (Slab& s : c->sl) {
        cg_flush_x(s.vs, R, c->ctl, s.p0, s.p1, s.x, c->stream);
        c->launches++;
    }
    TRY(xchg(c, [&](const Slab& s) { return fine_field(c, s, s.x, R); }));
    Rec all{c, R, nullptr, nullptr};
    for (Slab& s : c->sl) {
        FineArgs a = fine_args(c, s, all);
        a.x = s.x; a.b = s.b; a.y = s.t;
        level0_apply(c, s, FOP_RESID, a);
        c->launches++;
    }
    return dot_finish(c, R, &Slab::t, &Slab::t, SM_TRUE);
}

// WHILE condition of the device-side loop: continue while some RHS is active, no breakdown
// and no RHS has reached max_iter (the host loop's test, evaluated on the device).
__global__ void loop_cond_kernel(cudaGraphConditionalHandle h, const int* done, const int* status,
                                 const int* iters, int R, int maxit) {
    int go = !*done && !*status;
    for (int r = 0; go && r < R; ++r) go = iters[r] < maxit;
    cudaGraphSetConditional(h, go ? 1u : 0u);
}

// g_loop = [cond] -> WHILE(cond) { two CG iterations ; cond }: the whole iteration runs
// without host round trips (CUDA 12.4+ conditional graph nodes).  Single rank only (NCCL
// calls stay in host-driven graphs).
static mg_status build_loop_graph(mg_ctx* c, int R, double tol) {
    cudaGraph_t g = nullptr;
    CU(cudaGraphCreate(&g, 0));
    cudaGraphConditionalHandle h;
    CU(cudaGraphConditionalHandleCreate(&h, g, 0, cudaGraphCondAssignDefault));
    const int maxit = c->opts.max_iter;
    CU(cudaStreamBeginCaptureToGraph(c->stream, g, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
    loop_cond_kernel<<<1, 1, 0, c->stream>>>(h, c->ctl.done, c->ctl.status, c->ctl.iters, R, maxit);
    cudaGraph_t gc = nullptr;
    CU(cudaStreamEndCapture(c->stream, &gc));
    cudaGraphNode_t first = nullptr;
    size_t nn = 1;
    CU(cudaGraphGetNodes(g, &first, &nn));
    cudaGraphNodeParams np{};
    np.type = cudaGraphNodeTypeConditional;
    np.conditional.handle = h;
    np.conditional.type = cudaGraphCondTypeWhile;
    np.conditional.size = 1;
    cudaGraphNode_t wn = nullptr;
    CU(cudaGraphAddNode(&wn, g, &first, 1, &np));
    cudaGraph_t body = np.conditional.phGraph_out[0];
    CU(cudaStreamBeginCaptureToGraph(c->stream, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
    mg_status st = record_iter(c, R, tol);
    loop_cond_kernel<<<1, 1, 0, c->stream>>>(h, c->ctl.done, c->ctl.status, c->ctl.iters, R, maxit);
    cudaGraph_t bc = nullptr;
    CU(cudaStreamEndCapture(c->stream, &bc));
    TRY(st);
    CU(cudaGraphInstantiate(&c->g_loop, g, 0));
    CU(cudaGraphDestroy(g));
    return MG_OK;
}

static mg_status build_graphs(mg_ctx* c, int R, double tol) {
    for (cudaGraphExec_t* g : {&c->g_init, &c->g_restart, &c->g_iter, &c->g_true, &c->g_loop})
        if (*g) { cudaGraphExecDestroy(*g); *g = nullptr; }
    TRY(capture_begin(c));
    TRY(captured(c, record_restart(c, R)));
    TRY(capture_end(c, &c->g_restart, &c->n_restart));
    TRY(capture_begin(c));
    TRY(captured(c, [&]() -> mg_status {
        TRY(dot_finish(c, R, &Slab::b, &Slab::b, SM_BB));
        for (Slab& s : c->sl) {
            CU(cudaMemsetAsync(s.x, 0, sizeof(double) * s.vs * R, c->stream));
            CU(cudaMemsetAsync(s.p0, 0, sizeof(double) * s.vs * R, c->stream));
            CU(cudaMemsetAsync(s.q, 0, sizeof(double) * s.vs * R, c->stream));
            CU(cudaMemcpyAsync(s.r1, s.b, sizeof(double) * s.vs * R, cudaMemcpyDeviceToDevice, c->stream));
        }
        return MG_OK;
    }()));
    TRY(capture_end(c, &c->g_init, &c->n_init));
    TRY(capture_begin(c));
    TRY(captured(c, record_iter(c, R, tol)));
    TRY(capture_end(c, &c->g_iter, &c->n_iter));
    TRY(capture_begin(c));
    TRY(captured(c, record_true(c, R)));
    TRY(capture_end(c, &c->g_true, &c->n_true));
    if (c->comm.nranks == 1 && !getenv("MG_HOST_LOOP")) {
        if (build_loop_graph(c, R, tol) != MG_OK) {   // fall back to the host-driven loop
            cudaGraph_t g = nullptr;
            cudaStreamEndCapture(c->stream, &g);
            if (g) cudaGraphDestroy(g);
            cudaGetLastError();
            if (c->g_loop) { cudaGraphExecDestroy(c->g_loop); c->g_loop = nullptr; }
        }
    }
    c->graph_R = R;
    CHECK_LAUNCH();
    return MG_OK;
}

// ---------------------------------------------------------------- setup
static mg_status setup_impl(mg_ctx* c, const mg_grid* grid, const double* E_e, const uint8_t* fixed, int levels,
                            const mg_opts* opts, const mg_dist* dist, void* stream) {
    c->dim = grid->dim;
    c->L = levels;
    c->nu = grid->nu;
    c->elem = grid->element;
    if (opts) c->opts = *opts;
    c->user = (cudaStream_t)stream;
    const int rank = dist ? dist->rank : 0, nranks = dist ? dist->nranks : 1;
    const int nsl = dist ? dist->nslab : 1;
    c->S = nranks * nsl;
    CU(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    CU(cudaEventCreateWithFlags(&c->ev_in, cudaEventDisableTiming));
    CU(cudaEventCreateWithFlags(&c->ev_out, cudaEventDisableTiming));
    if (!comm_init(c->comm, rank, nranks, dist ? dist->nccl_id : nullptr))
        return fail(MG_ERR_NCCL, std::string("NCCL init: ") + comm_last_error());
    stream_enter(c);
    cudaStream_t s = c->stream;
    const int dim = c->dim;
    int N[3] = {grid->nel[0], grid->nel[1], dim == 3 ? grid->nel[2] : 1};
    for (int l = 0; l < levels; ++l) {
        int Nl[3];
        for (int k = 0; k < 3; ++k) Nl[k] = N[k] >> l;
        c->G[l] = make_geom(dim, Nl);
    }
    c->pn0 = c->G[0].nnodes / c->G[0].nn[0];
    // partition: rank q holds slabs [q*nsl, (q+1)*nsl)
    c->rank_p0.assign(nranks, 0);
    c->rank_p1.assign(nranks, 0);
    for (int q = 0; q < nranks; ++q) {
        int a, b, d;
        partition(N[0], levels, c->S, q * nsl, &a, &d);
        partition(N[0], levels, c->S, q * nsl + nsl - 1, &d, &b);
        c->rank_p0[q] = a;
        c->rank_p1[q] = b;
    }
    const int rp0 = c->rank_p0[rank], rp1 = c->rank_p1[rank];
    const long long le0 = c->G[0].nelem / N[0];   // elements per fine layer
    c->m_rank = (long long)(rp1 - rp0) * le0;
    c->n_rank = (long long)(rp1 - rp0 + (rank == nranks - 1 ? 1 : 0)) * c->pn0 * dim;
    c->sl.resize(nsl);
    for (int k = 0; k < nsl; ++k) {
        Slab& sl = c->sl[k];
        sl.id = rank * nsl + k;
        partition(N[0], levels, c->S, sl.id, &sl.e0, &sl.e1);
        sl.gl = sl.id > 0 ? 1 : 0;
        sl.gh = sl.id < c->S - 1 ? 1 : 0;
        sl.uoff = (long long)(sl.e0 - rp0) * c->pn0;
        for (int l = 0; l < levels; ++l) {
            Level& v = sl.lv[l];
            int Nl[3];
            for (int q = 0; q < 3; ++q) Nl[q] = N[q] >> l;
            const int own = (sl.e1 - sl.e0) >> l;
            Nl[0] = own + sl.gl;
            v.g = make_geom(dim, Nl);
            v.pn = v.g.nnodes / v.g.nn[0];
            v.o0 = sl.gl;
            v.o1 = sl.gl + own + (sl.gh ? 0 : 1);
            v.gp0 = (sl.e0 >> l) - sl.gl;
        }
    }
    if (grid->element == MG_ELEM_WILSON) element_stiffness_wilson(dim, c->nu, c->K0);
    else element_stiffness(dim, c->nu, c->K0);
    // compile-time K0 / K^ immediates only for the standard element at the paper's nu
    c->nu_paper = (c->nu == MG_NU_PAPER) && grid->element == MG_ELEM_STD;
    c->fused2d = (dim == 2 && levels >= 2);
    c->unfused_coarse = getenv("MG_UNFUSED_COARSE") && atoi(getenv("MG_UNFUSED_COARSE")) == 1;
    // 3D: r update + pre-smoother + residual in one h8t kernel (RESTR3, default) instead of
    // cg_rupdate + RESID (MG_FUSED3D=0); both parity-tested
    {
        const char* e = getenv("MG_FUSED3D");
        const int f3 = e ? atoi(e) : 1;
        const bool ok3 = dim == 3 && levels >= 2 && c->opts.nu_pre == 1 && c->opts.nu_post == 1 && !c->unfused_coarse;
        c->fused3d = ok3 && (f3 & 1);
    }
    TRY(ensure_constants(c));
    {
        const int na = 1 << dim, nl = dim * na;
        std::vector<double> Mh((size_t)na * nl * nl);
        galerkin_child_matrices(dim, c->K0.data(), Mh.data());
        CU(cudaMalloc(&c->Mc, sizeof(double) * Mh.size()));
        CU(cudaMemcpy(c->Mc, Mh.data(), sizeof(double) * Mh.size(), cudaMemcpyHostToDevice));
    }
    const int NL = dim * (1 << dim);
    const bool edev = is_device_ptr(E_e), fdev = is_device_ptr(fixed);
    uint8_t* dfix = nullptr;
    const uint8_t* fsrc = fixed;
    if (!fdev) {
        CU(cudaMalloc(&dfix, c->n_rank));
        CU(cudaMemcpyAsync(dfix, fixed, c->n_rank, cudaMemcpyHostToDevice, s));
        fsrc = dfix;
    }
    for (Slab& sl : c->sl) {
        const LevelGeom& g0 = sl.lv[0].g;
        CU(cudaMalloc(&sl.E, sizeof(double) * g0.nelem + 64));   // +64: aligned tails
        CU(cudaMemsetAsync(sl.E, 0, sizeof(double) * g0.nelem, s));
        for (int l = 0; l < levels; ++l) {
            Level& v = sl.lv[l];
            CU(cudaMalloc(&v.mask, v.g.nnodes + 64));
            CU(cudaMemsetAsync(v.mask, 0, v.g.nnodes, s));
            CU(cudaMalloc(&v.Dinv, sizeof(double) * v.g.ndof));
            CU(cudaMalloc(&v.D, sizeof(double) * v.g.ndof));
            if (l >= 1 || levels == 1) {
                const int ns = dim == 2 ? 9 : 27;
                CU(cudaMalloc(&v.st, sizeof(double) * v.g.nnodes * ns * dim * dim));
            }
        }
        // element-matrix ping-pong buffers (level 1 in A, level 2 in B, ...)
        const long long nA = levels >= 2 ? sl.lv[1].g.nelem : (levels == 1 ? g0.nelem : 1);
        // (elmB also holds the level-1 Galerkin's list of masked elements: nA + 1 ints)
        const long long nB = std::max<long long>(levels >= 3 ? sl.lv[2].g.nelem : 1, (nA + 1 + 2 * NL * NL - 1) / (2 * NL * NL));
        CU(cudaMalloc(&sl.elmA, sizeof(double) * nA * NL * NL));
        CU(cudaMalloc(&sl.elmB, sizeof(double) * nB * NL * NL));
        // owned fixed planes -> fine mask
        const Level& v0 = sl.lv[0];
        const long long cnt = (long long)(v0.o1 - v0.o0) * v0.pn;
        fixed_to_mask_kernel<<<(unsigned)((cnt + 255) / 256), 256, 0, s>>>(cnt, dim, fsrc, sl.uoff, v0.mask,
                                                                            v0.o0 * v0.pn);
        c->launches++;
        CHECK_LAUNCH();
    }
    TRY(xchg(c, [&](const Slab& sl) { return node_field(sl, 0, sl.lv[0].mask, 1, 1, 0, 1); }));
    for (int l = 1; l < levels; ++l) {
        for (Slab& sl : c->sl) {
            coarse_mask_kernel<<<(unsigned)((sl.lv[l].g.nnodes + 255) / 256), 256, 0, s>>>(
                sl.lv[l - 1].g, sl.lv[l].g, sl.lv[l - 1].mask, sl.lv[l].mask, sl.gl);
            c->launches++;
        }
        CHECK_LAUNCH();
        TRY(xchg(c, [&](const Slab& sl) { return node_field(sl, l, sl.lv[l].mask, 1, 1, 0, 1); }));
    }
    if (dfix) CU(cudaFreeAsync(dfix, s));
    for (Slab& sl : c->sl) {
        const LevelGeom& g0 = sl.lv[0].g;
        const long long le = g0.nelem / g0.N[0];
        CU(cudaMemcpyAsync(sl.E + sl.gl * le, E_e + (long long)(sl.e0 - rp0) * le,
                           sizeof(double) * (sl.e1 - sl.e0) * le,
                           edev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, s));
        if (dim == 2) {
            sl.pd = pad2_layout(g0);
            CU(cudaMalloc(&sl.Epad, sizeof(double) * sl.pd.elems));
            CU(cudaMalloc(&sl.maskpad, sl.pd.nodes));
            CU(cudaMalloc(&sl.Dinvpad, sizeof(double) * 2 * sl.pd.nodes));
            sl.vs = sl.pd.vstride;
        } else {
            sl.p3 = pad3_layout(g0);
            sl.g0p = pad3_geom(g0, sl.p3);
            sl.vs = sl.p3.vstride;
            CU(cudaMalloc(&sl.maskpad, (size_t)g0.nn[0] * g0.nn[1] * sl.p3.m2 + 64));
            CU(cudaMemsetAsync(sl.maskpad, 0, (size_t)g0.nn[0] * g0.nn[1] * sl.p3.m2, s));
            CU(cudaMalloc(&sl.Dinvpad, sizeof(double) * sl.p3.vstride));
            CU(cudaMemsetAsync(sl.Dinvpad, 0, sizeof(double) * sl.p3.vstride, s));
            if (sl.p3.ep2 != g0.N[2]) {
                const size_t ne = (size_t)g0.N[0] * g0.N[1] * sl.p3.ep2;
                CU(cudaMalloc(&sl.Epad, sizeof(double) * ne));
                CU(cudaMemsetAsync(sl.Epad, 0, sizeof(double) * ne, s));
            }
        }
    }
    const LevelGeom& gL = c->G[levels - 1];
    c->nL = gL.ndof;
    c->npad = (c->nL + 31) / 32 * 32;
    CU(cudaMalloc(&c->Ainv, sizeof(double) * c->npad * c->npad));
    CU(cudaMalloc(&c->gj_work, sizeof(double) * (2 * 32 * 32 + 2 * c->npad * 32)));
    if (multi(c)) {
        const int ns = dim == 2 ? 9 : 27;
        CU(cudaMalloc(&c->stg, sizeof(double) * gL.nnodes * ns * dim * dim));
        if (nranks > 1) {
            // per rank: at most (largest rank's coarsest planes) x plane x max(ns d^2, MG_MAX_RHS d)
            int maxp = 0;
            const int f = 1 << (levels - 1);
            for (int q = 0; q < nranks; ++q) maxp = std::max(maxp, (c->rank_p1[q] - c->rank_p0[q]) / f + 1);
            const long long pnL = gL.nnodes / gL.nn[0];
            c->cpack_cap = (long long)maxp * pnL * std::max(ns * dim * dim, MG_MAX_RHS * dim);
            CU(cudaMalloc(&c->cpack, sizeof(double) * c->cpack_cap));
            CU(cudaMalloc(&c->cgath, sizeof(double) * c->cpack_cap * nranks));
            CU(cudaMalloc(&c->sums, sizeof(double) * 2 * MG_MAX_RHS));
        }
    }
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

mg_status mg_partition(const mg_grid* grid, int levels, int nparts, int part, int* e_begin, int* e_end) {
    if (!grid || !e_begin || !e_end) return fail(MG_ERR_ARG, "NULL argument");
    if (levels < 1 || levels > MG_MAX_LEVELS) return fail(MG_ERR_ARG, "levels out of range");
    if (grid->nel[0] % (1 << (levels - 1))) return fail(MG_ERR_NONDIVISIBLE, "nel[0] not divisible by 2^(levels-1)");
    if (!partition(grid->nel[0], levels, nparts, part, e_begin, e_end))
        return fail(MG_ERR_DIM, "need 0 <= part < nparts <= coarsest-level element layers");
    return MG_OK;
}

mg_status mg_nccl_unique_id(void* out128) {
    if (!out128) return fail(MG_ERR_ARG, "NULL argument");
    if (!comm_nccl_unique_id(out128)) return fail(MG_ERR_NCCL, comm_last_error());
    return MG_OK;
}

mg_status mg_setup_dist(const mg_grid* grid, const double* E_e, const uint8_t* fixed, int levels, const mg_opts* opts,
                        const mg_dist* dist, void* stream, mg_handle* out) {
    NvtxRange nv(__func__);
    if (!grid || !E_e || !fixed || !out) return fail(MG_ERR_ARG, "NULL argument");
    if (grid->dim != 2 && grid->dim != 3) return fail(MG_ERR_ARG, "dim must be 2 or 3");
    if (grid->element != MG_ELEM_STD && grid->element != MG_ELEM_WILSON) return fail(MG_ERR_ARG, "unknown element");
    if (levels < 1 || levels > MG_MAX_LEVELS) return fail(MG_ERR_ARG, "levels out of range");
    if (!(grid->nu > -1.0 && grid->nu < 0.5)) return fail(MG_ERR_ARG, "nu out of range");
    if (opts && (opts->nu_pre < 1 || opts->nu_post < 0 || opts->max_iter < 1 || !(opts->omega > 0)))
        return fail(MG_ERR_ARG, "invalid mg_opts");
    if (opts && grid->dim == 2 && (opts->nu_pre != 1 || opts->nu_post != 1))
        return fail(MG_ERR_ARG, "2D path implements the fused V(1,1) cycle only (nu_pre = nu_post = 1)");
    if (dist) {
        if (dist->nranks < 1 || dist->rank < 0 || dist->rank >= dist->nranks || dist->nslab < 1)
            return fail(MG_ERR_ARG, "invalid mg_dist");
        if (dist->nranks > 1 && !dist->nccl_id) return fail(MG_ERR_ARG, "mg_dist.nccl_id required for nranks > 1");
        if (dist->nranks * dist->nslab > 1 && levels < 2) return fail(MG_ERR_ARG, "slab decomposition needs levels >= 2");
    }
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
    if (dist && grid->nel[0] / f < dist->nranks * dist->nslab)
        return fail(MG_ERR_DIM, "more slabs than coarsest-level element layers along axis 0");
    std::lock_guard<std::recursive_mutex> lk(g_api_mu);
    mg_ctx* c = new mg_ctx();
    mg_status st = setup_impl(c, grid, E_e, fixed, levels, opts, dist, stream);
    if (st != MG_OK) {
        std::string keep = g_last_error;
        mg_destroy(c);
        g_last_error = keep;
        return st;
    }
    *out = c;
    return MG_OK;
}

mg_status mg_setup(const mg_grid* grid, const double* E_e, const uint8_t* fixed, int levels, const mg_opts* opts,
                   void* stream, mg_handle* out) {
    return mg_setup_dist(grid, E_e, fixed, levels, opts, nullptr, stream, out);
}

mg_status mg_local_info(mg_handle c, long long* ndof_local, long long* nelem_local, int* e_begin, int* e_end) {
    if (!c) return fail(MG_ERR_ARG, "NULL handle");
    if (ndof_local) *ndof_local = c->n_rank;
    if (nelem_local) *nelem_local = c->m_rank;
    if (e_begin) *e_begin = c->rank_p0[c->comm.rank];
    if (e_end) *e_end = c->rank_p1[c->comm.rank];
    return MG_OK;
}

mg_status mg_update_modulus(mg_handle c, const double* E_e) {
    if (!c || !E_e) return fail(MG_ERR_ARG, "NULL argument");
    API_SCOPE(c);
    cudaStream_t s = c->stream;
    const long long m = c->m_rank;
    // validate the new moduli BEFORE touching the handle (argument errors have no side effects):
    // host input is staged on the device first and the slabs are then filled from the staging copy
    const bool edev = is_device_ptr(E_e);
    double* stage = nullptr;
    const double* src = E_e;
    if (!edev) {   // a staging buffer kept by the handle: no pool allocation (and trim) per call
        if (c->Estage_n < std::max<long long>(m, 1)) {
            CU(cudaStreamSynchronize(s));
            if (c->Estage) cudaFree(c->Estage);
            c->Estage = nullptr;
            CU(cudaMalloc((void**)&c->Estage, sizeof(double) * std::max<long long>(m, 1)));
            c->Estage_n = std::max<long long>(m, 1);
        }
        stage = c->Estage;
        CU(cudaMemcpyAsync(stage, E_e, sizeof(double) * m, cudaMemcpyHostToDevice, s));
        src = stage;
    }
    int bad = 0;
    if (cudaMemsetAsync(c->d_status, 0, sizeof(int), s) != cudaSuccess) return fail(MG_ERR_CUDA, "memset");
    if (m > 0) check_modulus_kernel<<<(unsigned)((m + 255) / 256), 256, 0, s>>>(m, src, c->d_status);
    c->launches++;
    if (cudaMemcpyAsync(c->h_pinned, c->d_status, sizeof(int), cudaMemcpyDeviceToHost, s) != cudaSuccess ||
        cudaStreamSynchronize(s) != cudaSuccess) {
        return fail(MG_ERR_CUDA, "mg_update_modulus: modulus check");
    }
    bad = c->h_pinned[0];
    if (c->comm.nranks > 1) {   // every rank takes the same decision
        double f = bad ? 1.0 : 0.0;
        if (cudaMemcpyAsync(c->sums, &f, sizeof(double), cudaMemcpyHostToDevice, s) != cudaSuccess ||
            !comm_allreduce_sum(c->comm, c->sums, 1, s) ||
            cudaMemcpyAsync(&f, c->sums, sizeof(double), cudaMemcpyDeviceToHost, s) != cudaSuccess ||
            cudaStreamSynchronize(s) != cudaSuccess) {
            return fail(MG_ERR_NCCL, "mg_update_modulus: modulus check allreduce");
        }
        bad = f != 0.0;
    }
    if (bad) {
        return fail(MG_ERR_MODULUS, "E_e must be positive and finite (handle unchanged)");
    }
    const int rp0 = c->rank_p0[c->comm.rank];
    for (Slab& sl : c->sl) {
        const LevelGeom& g0 = sl.lv[0].g;
        const long long le = g0.nelem / g0.N[0];
        if (cudaMemcpyAsync(sl.E + sl.gl * le, src + (long long)(sl.e0 - rp0) * le, sizeof(double) * (sl.e1 - sl.e0) * le,
                            cudaMemcpyDeviceToDevice, s) != cudaSuccess) {
            return fail(MG_ERR_CUDA, "mg_update_modulus: copy");
        }
    }
    // E changes the stencils but not the masks; the masks of coarse levels may have been
    // augmented by zero-diagonal DOFs, which stay valid for the same BCs.  Returns once the
    // operators are enqueued: the coarsest pivot status is checked by the next call.
    return compute_operators(c, true);
}

mg_status mgcg_solve(mg_handle c, const double* rhs, int nrhs, double tol, double* x, mg_report* rep) {
    if (!c || !rhs || !x) return fail(MG_ERR_ARG, "NULL argument");
    if (nrhs < 1 || nrhs > MG_MAX_RHS) return fail(MG_ERR_ARG, "nrhs out of range");
    if (!(tol > 0.0) || !(tol < 1.0)) return fail(MG_ERR_ARG, "tol must be in (0,1)");
    const long long n = c->n_rank;
    cudaStream_t s = c->stream;
    API_SCOPE_DEFER_SETUP(c);
    const bool rdev = is_device_ptr(rhs), xdev = is_device_ptr(x);
    NvtxRange phase("mgcg_solve: rhs in");
    if (!rdev) {
        // host right-hand sides: uploaded on the copy stream into a buffer only this upload and the
        // scatter below use (the previous solve's scatter finished: every solve ends synchronised),
        // overlapping a setup that mg_update_modulus may still be running on the handle stream
        if (c->rstage_n < n * nrhs) {
            CU(cudaStreamSynchronize(s));
            if (c->cs_in) CU(cudaStreamSynchronize(c->cs_in));
            if (c->rstage) cudaFree(c->rstage);
            c->rstage = nullptr;
            c->rstage_n = 0;
            CU(cudaMalloc(&c->rstage, sizeof(double) * n * nrhs));
            c->rstage_n = n * nrhs;
        }
        TRY(ensure_copy_streams(c));
        CU(cudaMemcpyAsync(c->rstage, rhs, sizeof(double) * n * nrhs, cudaMemcpyHostToDevice, c->cs_in));
        CU(cudaEventRecord(c->ev_rhs, c->cs_in));
    }
    TRY(setup_check(c));
    cudaEvent_t e0, e1;
    CU(cudaEventCreate(&e0));
    CU(cudaEventCreate(&e1));
    CU(cudaEventRecord(e0, s));
    TRY(ensure_vectors(c, nrhs));
    if (c->graph_R != nrhs || c->graph_tol != tol) {
        TRY(build_graphs(c, nrhs, tol));
        c->graph_tol = tol;
    }
    const double* rsrc = rhs;
    if (!rdev) {
        CU(cudaStreamWaitEvent(s, c->ev_rhs, 0));
        rsrc = c->rstage;
    }
    TRY(scatter_fine(c, rsrc, nrhs, true, &Slab::b));
    phase.next("mgcg_solve: iterate");
    CU(cudaMemsetAsync(c->ctl.status, 0, sizeof(int), s));
    CU(cudaGraphLaunch(c->g_init, s));
    CU(cudaGraphLaunch(c->g_restart, s));
    int glaunch = 2;
    long long klaunch = c->n_init + c->n_restart;
    int* hp = c->h_pinned;    // [0] done [1] status [2..2+R) iters
    double* hd = c->h_dbl;    // bb[64] rr[64] tt[64]
    const int maxit = c->opts.max_iter;
    int restarts = 0;
    int host_mx = 0;   // largest per-RHS iteration count seen by the host (launch accounting)
    mg_status result = MG_OK;
    for (;;) {
        // iterate until all RHS converged (recursive residual) or the cap
        if (c->g_loop) {
            const int mx0 = host_mx;
            CU(cudaGraphLaunch(c->g_loop, s));
            ++glaunch;
            CU(cudaMemcpyAsync(hp, c->ctl.done, sizeof(int) * 2, cudaMemcpyDeviceToHost, s));
            CU(cudaMemcpyAsync(hp + 2, c->ctl.iters, sizeof(int) * nrhs, cudaMemcpyDeviceToHost, s));
            CU(cudaStreamSynchronize(s));
            int mx1 = 0;
            for (int k = 0; k < nrhs; ++k) mx1 = hp[2 + k] > mx1 ? hp[2 + k] : mx1;
            klaunch += 1 + (long long)((mx1 - mx0 + 1) / 2) * (c->n_iter + 1);
            host_mx = mx1;
        } else
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
        // on breakdown the true residual is still evaluated (it also flushes the deferred x
        // update), so x and the report describe the last iterate
        const bool breakdown = hp[1] != 0;
        if (breakdown) result = fail(MG_ERR_BREAKDOWN, "p.Kp <= 0 in CG");
        CU(cudaGraphLaunch(c->g_true, s));
        ++glaunch;
        klaunch += c->n_true;
        CU(cudaMemcpyAsync(hd, c->ctl.bb, sizeof(double) * MG_MAX_RHS, cudaMemcpyDeviceToHost, s));
        CU(cudaMemcpyAsync(hd + MG_MAX_RHS, c->ctl.rr, sizeof(double) * MG_MAX_RHS, cudaMemcpyDeviceToHost, s));
        CU(cudaMemcpyAsync(hd + 2 * MG_MAX_RHS, c->ctl.tt, sizeof(double) * MG_MAX_RHS, cudaMemcpyDeviceToHost, s));
        CU(cudaMemcpyAsync(hp + 2, c->ctl.iters, sizeof(int) * nrhs, cudaMemcpyDeviceToHost, s));
        CU(cudaStreamSynchronize(s));
        if (breakdown) break;
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
        for (Slab& sl : c->sl) vec_axpy_masked_restart(sl.vs, nrhs, sl.t, sl.r1, d_restart, s);
        TRY(xchg(c, [&](const Slab& sl) { return fine_field(c, sl, sl.r1, nrhs); }));
        CU(cudaMemsetAsync(c->ctl.alpha, 0, sizeof(double) * MG_MAX_RHS, s));
        int zero = 0;
        CU(cudaMemcpyAsync(c->ctl.done, &zero, sizeof(int), cudaMemcpyHostToDevice, s));
        CU(cudaGraphLaunch(c->g_restart, s));
        ++glaunch;
        klaunch += c->n_restart + nslab(c);
    }
    // copy x out
    phase.next("mgcg_solve: x out");
    double* xdst = xdev ? x : c->stage;
    TRY(gather_fine(c, &Slab::x, nrhs, xdst));
    if (!xdev) CU(cudaMemcpyAsync(x, c->stage, sizeof(double) * n * nrhs, cudaMemcpyDeviceToHost, s));
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
    if (result != MG_OK) return result;
    if (!all_conv) return fail(MG_ERR_MAXITER, "not all right-hand sides reached tol");
    return MG_OK;
}

// ---------------------------------------------------------------- block PCG (NEXT-3)
// O'Leary's block CG with the same V(1,1) preconditioner (Alg. 2 l.15):
//   Q = A P; Gamma = P^T Q; alpha = Gamma^+ Rho; X += P alpha; R -= Q alpha; Z = M R;
//   Rho' = Z^T R; beta = Rho^+ Rho'; P = Z + P beta; Rho = Rho'
// with pivoted-Cholesky pseudo-inverses (dependent / converged directions deflated).
static mg_status record_block_iter(mg_ctx* c, int R, double tol) {
    Slab& s = c->sl[0];
    const long long n = s.vs;
    Rec all{c, R, nullptr, nullptr};
    {
        FineArgs a = fine_args(c, s, all);
        a.x = s.p0; a.y = s.q;
        level0_apply(c, s, FOP_MATVEC, a);
    }
    gram(n, n, R, s.p0, s.q, c->bpart, c->bGam, c->stream);
    block_coef(R, c->bGam, c->bRho, c->bC, 1e-13, c->brank, c->stream);
    block_axpy(n, n, R, s.p0, c->bC, nullptr, s.x, 1.0, c->stream);
    block_axpy(n, n, R, s.q, c->bC, nullptr, s.r1, -1.0, c->stream);
    const int items = vec_dot_range(n, 0, n, R, s.r1, s.r1, c->partial, c->pst, nullptr, nullptr, c->stream);
    block_conv(R, c->partial, items, tol, c->ctl, c->stream);
    long long k;
    TRY(blk_restrict(all, &Slab::r1, &Slab::r0, &k));
    int cw;
    TRY(coarse_cycle(all, &cw));
    TRY(blk_post(all, &Slab::r0, cw, &k));
    gram(n, n, R, s.zf, s.r1, c->bpart, c->bRhoN, c->stream);
    block_coef(R, c->bRho, c->bRhoN, c->bC, 1e-13, c->brank, c->stream);
    block_axpy(n, n, R, s.p0, c->bC, s.zf, s.p0, 1.0, c->stream);
    CU(cudaMemcpyAsync(c->bRho, c->bRhoN, sizeof(double) * R * R, cudaMemcpyDeviceToDevice, c->stream));
    c->launches += 14;
    return MG_OK;
}

// y = G(u) phi on one slab's compact device arrays (local geometry g).  3D with an even element
// count along axis 2 and 8-byte aligned arrays: the TMA march kernel (h8t.cu, FOP_GPHI; the
// stress matrix in the sum/difference basis), reading the centroid stresses `sig` (stress_sigma,
// once per call when several phi share them) or forming them in the kernel from u (sig = NULL);
// otherwise centroid stresses + stress_apply.
static void gphi_slab(mg_ctx* c, Slab& sl, const LevelGeom& g, const uint8_t* mask, const double* Es, const double* u,
                      const double* phi, double* y, int nphi, const double* sig) {
    cudaStream_t s = c->stream;
    const int nv = c->dim == 2 ? 3 : 6;
    auto a8 = [](const void* p) { return ((uintptr_t)p & 7) == 0; };
    if (c->dim == 3 && g.N[2] % 2 == 0 && a8(Es) && a8(u) && a8(phi) && ((uintptr_t)Es & 15) == 0 &&
        !getenv("MG_GPHI_LEGACY")) {
        FineArgs a{};
        a.g = g;   // compact vectors (p2 = n2, vstr = ndof)
        a.E = Es; a.mask = sl.maskpad; a.m2 = sl.p3.m2; a.ep2 = g.N[2];
        a.x = phi; a.b = u; a.y = y; a.R = nphi; a.nu_paper = c->nu_paper ? 1 : 0;
        a.goffA = (int)(((uintptr_t)phi & 15) >> 3);
        a.goffB = (int)(((uintptr_t)u & 15) >> 3);
        a.sig = sig;
        if (fine_apply(FOP_GPHI, a, s) >= 0) {
            c->launches++;
            return;
        }
    }
    if (!sig) {
        if (!sl.sig) cudaMalloc(&sl.sig, sizeof(double) * g.nelem * nv);
        stress_sigma(g, Es, u, sl.sig, s);
        c->launches++;
        sig = sl.sig;
    }
    stress_apply(g, sig, mask, phi, y, nphi, s);
    c->launches++;
}

// centroid stresses of one slab (3 or 6 per element) when several phi share them, else NULL
// (MG_GPHI_SIGMA=0/1 forces either)
static const double* gphi_sigma(mg_ctx* c, Slab& sl, const LevelGeom& g, const double* Es, const double* u, int nphi) {
    const char* e = getenv("MG_GPHI_SIGMA");
    const bool pre = e ? atoi(e) != 0 : (nphi > 1 || c->dim == 2);
    if (!pre) return nullptr;
    const int nv = c->dim == 2 ? 3 : 6;
    if (!sl.sig) cudaMalloc(&sl.sig, sizeof(double) * g.nelem * nv);
    stress_sigma(g, Es, u, sl.sig, c->stream);
    c->launches++;
    return sl.sig;
}

mg_status stress_stiffness_apply(mg_handle c, const double* Es_e, const double* u, const double* phi, int nphi,
                                 double* y) {
    if (!c || !Es_e || !u || !phi || !y) return fail(MG_ERR_ARG, "NULL argument");
    if (nphi < 1) return fail(MG_ERR_ARG, "nphi must be >= 1");
    cudaStream_t s = c->stream;
    const int dim = c->dim;
    const int nv = dim == 2 ? 3 : 6;
    API_SCOPE(c);
    const bool dev = is_device_ptr(phi) && is_device_ptr(y) && is_device_ptr(u) && is_device_ptr(Es_e);
    if (!multi(c) && dev) {   // one slab, device buffers: direct
        Slab& sl = c->sl[0];
        const double* sig = gphi_sigma(c, sl, sl.lv[0].g, Es_e, u, nphi);
        gphi_slab(c, sl, sl.lv[0].g, sl.lv[0].mask, Es_e, u, phi, y, nphi, sig);
        CHECK_LAUNCH();
        return MG_OK;
    }
    if (!multi(c) && !dev && nslab(c) == 1) {
        // one slab, host buffers: Es and u in, sigma, then phi in chunks -- H2D of chunk k + 1 and
        // D2H of chunk k - 1 overlap the kernel of chunk k (stream-ordered through events)
        Slab& sl = c->sl[0];
        const LevelGeom& g0 = sl.lv[0].g;
        const long long n = g0.ndof, m = g0.nelem;
        const long long need = m + n + 2 * n * nphi;
        if (need > c->gstage_cap) {
            CU(cudaStreamSynchronize(s));
            if (c->gstage) cudaFree(c->gstage);
            c->gstage = nullptr;
            CU(cudaMalloc(&c->gstage, sizeof(double) * need));
            c->gstage_cap = need;
        }
        TRY(ensure_copy_streams(c));
        double* dEs = c->gstage;
        double* du = dEs + m;
        double* dphi = du + n;
        double* dy = dphi + n * nphi;
        if (!sl.sig) CU(cudaMalloc(&sl.sig, sizeof(double) * m * nv));
        // the copy streams must not overtake earlier work on the handle stream (staging reuse)
        CU(cudaEventRecord(c->gev_sig, s));
        CU(cudaStreamWaitEvent(c->cs_in, c->gev_sig, 0));
        CU(cudaStreamWaitEvent(c->cs_out, c->gev_sig, 0));
        CU(cudaMemcpyAsync(dEs, Es_e, sizeof(double) * m, cudaMemcpyDefault, s));
        CU(cudaMemcpyAsync(du, u, sizeof(double) * n, cudaMemcpyDefault, s));
        const double* sig = gphi_sigma(c, sl, g0, dEs, du, nphi);   // once for all chunks
        const int nch = std::min(mg_ctx::NCHUNK_EV, nphi);
        const int per = (nphi + nch - 1) / nch;
        for (int k = 0, k0 = 0; k0 < nphi; ++k, k0 += per) {
            const int kc = std::min(per, nphi - k0);
            const size_t bytes = sizeof(double) * n * kc;
            CU(cudaMemcpyAsync(dphi + n * k0, phi + n * k0, bytes, cudaMemcpyDefault, c->cs_in));
            CU(cudaEventRecord(c->gev_in[k], c->cs_in));
            CU(cudaStreamWaitEvent(s, c->gev_in[k], 0));
            gphi_slab(c, sl, g0, sl.lv[0].mask, dEs, du, dphi + n * k0, dy + n * k0, kc, sig);
            CU(cudaEventRecord(c->gev_k[k], s));
            CU(cudaStreamWaitEvent(c->cs_out, c->gev_k[k], 0));
            CU(cudaMemcpyAsync(y + n * k0, dy + n * k0, bytes, cudaMemcpyDefault, c->cs_out));
        }
        CHECK_LAUNCH();
        CU(cudaEventRecord(c->gev_done, c->cs_out));
        CU(cudaStreamWaitEvent(s, c->gev_done, 0));
        CU(cudaStreamSynchronize(s));
        return MG_OK;
    }
    // general path: this rank's owned planes -> slab-local compact arrays (+ ghosts) -> kernels
    // -> owned planes back.  Host buffers are staged (synchronous).
    const long long n = c->n_rank, m = c->m_rank;
    double *dEs = nullptr, *du = nullptr, *dphi = nullptr, *dy = nullptr;
    const double *Es_src = Es_e, *u_src = u, *phi_src = phi;
    if (!dev) {
        // persistent staging (grown on demand): Es | u | phi | y
        const long long need = m + n + 2 * n * nphi;
        if (need > c->gstage_cap) {
            if (c->gstage) cudaFree(c->gstage);
            c->gstage = nullptr;
            CU(cudaMalloc(&c->gstage, sizeof(double) * need));
            c->gstage_cap = need;
        }
        dEs = c->gstage;
        du = dEs + m;
        dphi = du + n;
        dy = dphi + n * nphi;
        CU(cudaMemcpyAsync(dEs, Es_e, sizeof(double) * m, cudaMemcpyDefault, s));
        CU(cudaMemcpyAsync(du, u, sizeof(double) * n, cudaMemcpyDefault, s));
        CU(cudaMemcpyAsync(dphi, phi, sizeof(double) * n * nphi, cudaMemcpyDefault, s));
        Es_src = dEs; u_src = du; phi_src = dphi;
    }
    double* y_dst = dev ? y : dy;
    const int rp0 = c->rank_p0[c->comm.rank];
    for (Slab& sl : c->sl) {
        const Level& v = sl.lv[0];
        const long long nd = v.g.ndof;
        if (!sl.sig) CU(cudaMalloc(&sl.sig, sizeof(double) * v.g.nelem * nv));
        if (!sl.u) CU(cudaMalloc(&sl.u, sizeof(double) * nd));
        if (sl.gphi_cap < nphi) {
            if (sl.phi) cudaFree(sl.phi);
            if (sl.gy) cudaFree(sl.gy);
            CU(cudaMalloc(&sl.phi, sizeof(double) * nd * nphi));
            CU(cudaMalloc(&sl.gy, sizeof(double) * nd * nphi));
            sl.gphi_cap = nphi;
        }
        CU(cudaMemsetAsync(sl.u, 0, sizeof(double) * nd, s));
        CU(cudaMemsetAsync(sl.phi, 0, sizeof(double) * nd * nphi, s));
        const long long pl = v.pn * dim, np = v.o1 - v.o0;
        CU(cudaMemcpyAsync(sl.u + v.o0 * pl, u_src + dim * sl.uoff, sizeof(double) * np * pl,
                           cudaMemcpyDeviceToDevice, s));
        CU(cudaMemcpy2DAsync(sl.phi + v.o0 * pl, nd * 8, phi_src + dim * sl.uoff, n * 8, np * pl * 8, nphi,
                             cudaMemcpyDeviceToDevice, s));
        // stress moduli of the owned element layers (ghost layer below by exchange)
        const long long le = v.g.nelem / v.g.N[0];
        if (!sl.Es) CU(cudaMalloc(&sl.Es, sizeof(double) * v.g.nelem));
        CU(cudaMemsetAsync(sl.Es, 0, sizeof(double) * v.g.nelem, s));
        CU(cudaMemcpyAsync(sl.Es + sl.gl * le, Es_src + (long long)(sl.e0 - rp0) * le,
                           sizeof(double) * (sl.e1 - sl.e0) * le, cudaMemcpyDeviceToDevice, s));
    }
    TRY(xchg(c, [&](const Slab& sl) { return vec_field(c, sl, 0, sl.u, 1); }));
    TRY(xchg(c, [&](const Slab& sl) { return vec_field(c, sl, 0, sl.phi, nphi); }));
    TRY(xchg(c, [&](const Slab& sl) { return elem_field(sl, 0, sl.Es, 1); }));
    for (Slab& sl : c->sl) {
        const Level& v = sl.lv[0];
        const double* sig = gphi_sigma(c, sl, v.g, sl.Es, sl.u, nphi);
        gphi_slab(c, sl, v.g, v.mask, sl.Es, sl.u, sl.phi, sl.gy, nphi, sig);
        const long long pl = v.pn * dim, np = v.o1 - v.o0;
        CU(cudaMemcpy2DAsync(y_dst + dim * sl.uoff, n * 8, sl.gy + v.o0 * pl, v.g.ndof * 8, np * pl * 8, nphi,
                             cudaMemcpyDeviceToDevice, s));
    }
    CHECK_LAUNCH();
    if (!dev) {
        CU(cudaMemcpyAsync(y, dy, sizeof(double) * n * nphi, cudaMemcpyDefault, s));
        CU(cudaStreamSynchronize(s));
    }
    return MG_OK;
}

// ---- slab mode of the NEXT-1 calls: this rank's owned arrays <-> slab-local compact copies
// (owned planes / element layers copied, ghosts by exchange), the kernels then run unchanged on
// each slab's local grid (the ghost element layer below and the ghost node planes make every
// owned node / element exact, as for the operator).
static mg_status stage_nodes(mg_ctx* c, const double* src, int nv, int k) {
    cudaStream_t s = c->stream;
    for (Slab& sl : c->sl) {
        const Level& v = sl.lv[0];
        const long long nd = v.g.ndof, need = nd * nv;
        if (sl.tn_cap[k] < need) {
            if (sl.tn[k]) cudaFree(sl.tn[k]);
            sl.tn[k] = nullptr;
            CU(cudaMalloc(&sl.tn[k], sizeof(double) * need));
            sl.tn_cap[k] = need;
        }
        CU(cudaMemsetAsync(sl.tn[k], 0, sizeof(double) * need, s));
        const long long pl = v.pn * c->dim, np = v.o1 - v.o0;
        CU(cudaMemcpy2DAsync(sl.tn[k] + v.o0 * pl, nd * 8, src + c->dim * sl.uoff, c->n_rank * 8, np * pl * 8, nv,
                             cudaMemcpyDeviceToDevice, s));
    }
    return xchg(c, [&](const Slab& sl) { return vec_field(c, sl, 0, sl.tn[k], nv); });
}
static mg_status unstage_nodes(mg_ctx* c, int k, int nv, double* dst) {
    for (Slab& sl : c->sl) {
        const Level& v = sl.lv[0];
        const long long pl = v.pn * c->dim, np = v.o1 - v.o0;
        CU(cudaMemcpy2DAsync(dst + c->dim * sl.uoff, c->n_rank * 8, sl.tn[k] + v.o0 * pl, v.g.ndof * 8, np * pl * 8, nv,
                             cudaMemcpyDeviceToDevice, c->stream));
    }
    return MG_OK;
}
static mg_status stage_elems(mg_ctx* c, const double* src, int k) {
    cudaStream_t s = c->stream;
    const int rp0 = c->rank_p0[c->comm.rank];
    for (Slab& sl : c->sl) {
        const LevelGeom& g = sl.lv[0].g;
        if (sl.te_cap[k] < g.nelem) {
            if (sl.te[k]) cudaFree(sl.te[k]);
            sl.te[k] = nullptr;
            CU(cudaMalloc(&sl.te[k], sizeof(double) * g.nelem));
            sl.te_cap[k] = g.nelem;
        }
        const long long le = g.nelem / g.N[0];
        CU(cudaMemsetAsync(sl.te[k], 0, sizeof(double) * g.nelem, s));
        CU(cudaMemcpyAsync(sl.te[k] + sl.gl * le, src + (long long)(sl.e0 - rp0) * le,
                           sizeof(double) * (sl.e1 - sl.e0) * le, cudaMemcpyDeviceToDevice, s));
    }
    return xchg(c, [&](const Slab& sl) { return elem_field(sl, 0, sl.te[k], 1); });
}

mg_status mg_adjoint_rhs(mg_handle c, const double* Es_e, const double* phi, int nphi, double* b) {
    if (!c || !Es_e || !phi || !b) return fail(MG_ERR_ARG, "NULL argument");
    if (nphi < 1) return fail(MG_ERR_ARG, "nphi must be >= 1");
    if (!is_device_ptr(Es_e) || !is_device_ptr(phi) || !is_device_ptr(b))
        return fail(MG_ERR_ARG, "mg_adjoint_rhs: device pointers required");
    API_SCOPE(c);
    if (multi(c)) {   // slab-local copies, kernels per slab, owned planes back
        TRY(stage_elems(c, Es_e, 0));
        TRY(stage_nodes(c, phi, nphi, 0));
        long long need = 0;
        for (Slab& sl : c->sl) need = std::max(need, (long long)nphi * sl.lv[0].g.nelem * (c->dim == 2 ? 3 : 6));
        if (need > c->wbuf_cap) {
            CU(cudaStreamSynchronize(c->stream));
            if (c->wbuf) cudaFree(c->wbuf);
            c->wbuf = nullptr;
            CU(cudaMalloc(&c->wbuf, sizeof(double) * need));
            c->wbuf_cap = need;
        }
        for (Slab& sl : c->sl) {
            const long long nd = sl.lv[0].g.ndof * nphi;
            if (sl.tn_cap[1] < nd) {
                if (sl.tn[1]) cudaFree(sl.tn[1]);
                sl.tn[1] = nullptr;
                CU(cudaMalloc(&sl.tn[1], sizeof(double) * nd));
                sl.tn_cap[1] = nd;
            }
            adjoint_rhs_apply(sl.lv[0].g, sl.te[0], sl.lv[0].mask, sl.tn[0], nphi, c->wbuf, sl.tn[1], c->stream);
            c->launches += 2;
        }
        CHECK_LAUNCH();
        return unstage_nodes(c, 1, nphi, b);
    }
    const LevelGeom& g = c->G[0];
    const long long need = (long long)nphi * g.nelem * (c->dim == 2 ? 3 : 6);
    if (need > c->wbuf_cap) {
        CU(cudaStreamSynchronize(c->stream));
        if (c->wbuf) cudaFree(c->wbuf);
        c->wbuf = nullptr;
        CU(cudaMalloc(&c->wbuf, sizeof(double) * need));
        c->wbuf_cap = need;
    }
    adjoint_rhs_apply(g, Es_e, c->sl[0].lv[0].mask, phi, nphi, c->wbuf, b, c->stream);
    c->launches += 2;
    CHECK_LAUNCH();
    return MG_OK;
}

mg_status mg_eigen_sensitivity(mg_handle c, const double* dEk, const double* dEs, const double* u, const double* phi,
                               const double* z, const double* lambda, int nphi, double* out) {
    if (!c || !dEk || !dEs || !u || !phi || !z || !lambda || !out) return fail(MG_ERR_ARG, "NULL argument");
    if (nphi < 1 || nphi > MG_MAX_RHS) return fail(MG_ERR_ARG, "nphi out of range");
    for (const void* p : {(const void*)dEk, (const void*)dEs, (const void*)u, (const void*)phi, (const void*)z,
                          (const void*)out})
        if (!is_device_ptr(p)) return fail(MG_ERR_ARG, "mg_eigen_sensitivity: device pointers required");
    API_SCOPE(c);
    if (!c->dlam) CU(cudaMalloc(&c->dlam, sizeof(double) * MG_MAX_RHS));
    CU(cudaMemcpyAsync(c->dlam, lambda, sizeof(double) * nphi,
                       is_device_ptr(lambda) ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, c->stream));
    if (multi(c)) {   // slab-local copies; per slab the owned element layers of out are copied back
        TRY(stage_elems(c, dEk, 0));
        TRY(stage_elems(c, dEs, 1));
        TRY(stage_nodes(c, u, 1, 0));
        TRY(stage_nodes(c, phi, nphi, 1));
        TRY(stage_nodes(c, z, nphi, 2));
        const int rp0 = c->rank_p0[c->comm.rank];
        for (Slab& sl : c->sl) {
            const LevelGeom& g = sl.lv[0].g;
            const long long no = g.nelem * nphi;
            if (sl.tn_cap[3] < no) {
                if (sl.tn[3]) cudaFree(sl.tn[3]);
                sl.tn[3] = nullptr;
                CU(cudaMalloc(&sl.tn[3], sizeof(double) * no));
                sl.tn_cap[3] = no;
            }
            eigen_sensitivity_apply(g, sl.te[0], sl.te[1], sl.lv[0].mask, sl.tn[0], sl.tn[1], sl.tn[2], c->dlam, nphi,
                                    sl.tn[3], c->stream);
            c->launches++;
            const long long le = g.nelem / g.N[0];
            CU(cudaMemcpy2DAsync(out + (long long)(sl.e0 - rp0) * le, c->m_rank * 8, sl.tn[3] + sl.gl * le, g.nelem * 8,
                                 (sl.e1 - sl.e0) * le * 8, nphi, cudaMemcpyDeviceToDevice, c->stream));
        }
        CHECK_LAUNCH();
        CU(cudaStreamSynchronize(c->stream));
        return MG_OK;
    }
    eigen_sensitivity_apply(c->G[0], dEk, dEs, c->sl[0].lv[0].mask, u, phi, z, c->dlam, nphi, out, c->stream);
    c->launches++;
    CHECK_LAUNCH();
    CU(cudaStreamSynchronize(c->stream));   // lambda may be a host temporary
    return MG_OK;
}

mg_status mgcg_block_solve(mg_handle c, const double* rhs, int nrhs, double tol, double* x, mg_report* rep) {
    if (!c || !rhs || !x) return fail(MG_ERR_ARG, "NULL argument");
    if (nrhs < 1 || nrhs > MG_MAX_RHS) return fail(MG_ERR_ARG, "nrhs out of range");
    if (!(tol > 0.0) || !(tol < 1.0)) return fail(MG_ERR_ARG, "tol must be in (0,1)");
    if (multi(c)) return fail(MG_ERR_ARG, "mgcg_block_solve: single slab only (this round)");
    const int R = nrhs;
    const long long nr = c->n_rank;
    cudaStream_t s = c->stream;
    API_SCOPE(c);
    cudaEvent_t e0, e1;
    CU(cudaEventCreate(&e0));
    CU(cudaEventCreate(&e1));
    CU(cudaEventRecord(e0, s));
    TRY(ensure_vectors(c, R));
    Slab& sl = c->sl[0];
    const long long n = sl.vs;
    if (c->block_R != R) {   // workspace and the captured iteration are both sized for R
        for (double** p : {&c->bpart, &c->bGam, &c->bRho, &c->bRhoN, &c->bC})
            if (*p) { cudaFree(*p); *p = nullptr; }
        CU(cudaMalloc(&c->bpart, sizeof(double) * (long long)R * R * gram_blocks(n, R)));
        for (double** p : {&c->bGam, &c->bRho, &c->bRhoN, &c->bC}) CU(cudaMalloc(p, sizeof(double) * R * R));
        if (!c->brank) CU(cudaMalloc(&c->brank, sizeof(int)));
        c->block_R = R;
        if (c->g_block) { cudaGraphExecDestroy(c->g_block); c->g_block = nullptr; }
    }
    const bool rdev = is_device_ptr(rhs), xdev = is_device_ptr(x);
    const double* rsrc = rhs;
    if (!rdev) {
        CU(cudaMemcpyAsync(c->stage, rhs, sizeof(double) * nr * R, cudaMemcpyHostToDevice, s));
        rsrc = c->stage;
    }
    TRY(scatter_fine(c, rsrc, R, true, &Slab::b));
    // init: bb, active, iters; x = 0; r = b; Z = M r; P = Z; Rho = Z^T r
    TRY(dot_finish(c, R, &Slab::b, &Slab::b, SM_BB));
    CU(cudaMemsetAsync(c->ctl.alpha, 0, sizeof(double) * MG_MAX_RHS, s));
    CU(cudaMemsetAsync(c->ctl.status, 0, sizeof(int), s));
    CU(cudaMemsetAsync(sl.x, 0, sizeof(double) * n * R, s));
    CU(cudaMemsetAsync(sl.q, 0, sizeof(double) * n * R, s));
    CU(cudaMemcpyAsync(sl.r1, sl.b, sizeof(double) * n * R, cudaMemcpyDeviceToDevice, s));
    if (!c->g_block || c->block_tol != tol) {
        if (c->g_block) { cudaGraphExecDestroy(c->g_block); c->g_block = nullptr; }
        TRY(capture_begin(c));
        TRY(captured(c, record_block_iter(c, R, tol)));
        long long nn;
        TRY(capture_end(c, &c->g_block, &nn));
        c->block_tol = tol;
    }
    int* hp = c->h_pinned;
    double* hd = c->h_dbl;
    int it = 0, restarts = 0;
    const int maxit = c->opts.max_iter;
    for (;;) {
        // (re)start the block Krylov space from r: Z = M r, P = Z, Rho = Z^T r
        {
            Rec all{c, R, nullptr, nullptr};
            long long k;
            TRY(blk_restrict(all, &Slab::r1, &Slab::r0, &k));
            int cw;
            TRY(coarse_cycle(all, &cw));
            TRY(blk_post(all, &Slab::r0, cw, &k));
        }
        CU(cudaMemcpyAsync(sl.p0, sl.zf, sizeof(double) * n * R, cudaMemcpyDeviceToDevice, s));
        gram(n, n, R, sl.zf, sl.r1, c->bpart, c->bRho, s);
        int zero = 0;
        CU(cudaMemcpyAsync(c->ctl.done, &zero, sizeof(int), cudaMemcpyHostToDevice, s));
        for (; it < maxit;) {
            CU(cudaGraphLaunch(c->g_block, s));
            ++it;
            CU(cudaMemcpyAsync(hp, c->ctl.done, sizeof(int), cudaMemcpyDeviceToHost, s));
            CU(cudaStreamSynchronize(s));
            if (hp[0]) break;
        }
        TRY(record_true(c, R));   // x has no deferred update; flush is a no-op (xalpha = 0)
        CU(cudaMemcpyAsync(hd, c->ctl.bb, sizeof(double) * MG_MAX_RHS, cudaMemcpyDeviceToHost, s));
        CU(cudaMemcpyAsync(hd + MG_MAX_RHS, c->ctl.rr, sizeof(double) * MG_MAX_RHS, cudaMemcpyDeviceToHost, s));
        CU(cudaMemcpyAsync(hd + 2 * MG_MAX_RHS, c->ctl.tt, sizeof(double) * MG_MAX_RHS, cudaMemcpyDeviceToHost, s));
        CU(cudaMemcpyAsync(hp + 2, c->ctl.iters, sizeof(int) * R, cudaMemcpyDeviceToHost, s));
        CU(cudaStreamSynchronize(s));
        bool need = false;
        for (int k = 0; k < R; ++k)
            if (hd[k] > 0.0 && hd[2 * MG_MAX_RHS + k] > tol * tol * hd[k]) need = true;
        // residual gap of block CG (recursive vs true residual): restart from r = b - K x
        if (!need || restarts >= 3 || it >= maxit) break;
        ++restarts;
        CU(cudaMemcpyAsync(sl.r1, sl.t, sizeof(double) * n * R, cudaMemcpyDeviceToDevice, s));
    }
    double* xdst = xdev ? x : c->stage;
    TRY(gather_fine(c, &Slab::x, R, xdst));
    if (!xdev) CU(cudaMemcpyAsync(x, c->stage, sizeof(double) * nr * R, cudaMemcpyDeviceToHost, s));
    CU(cudaEventRecord(e1, s));
    CU(cudaStreamSynchronize(s));
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    bool all_conv = true;
    for (int k = 0; k < R; ++k) {
        const double bb = hd[k];
        const double tr = bb > 0 ? std::sqrt(hd[2 * MG_MAX_RHS + k] / bb) : 0.0;
        all_conv = all_conv && tr <= tol;
        if (rep) {
            rep->iters[k] = hp[2 + k];
            rep->relres[k] = bb > 0 ? std::sqrt(hd[MG_MAX_RHS + k] / bb) : 0.0;
            rep->true_relres[k] = tr;
            rep->converged[k] = tr <= tol ? 1 : 0;
        }
    }
    if (rep) {
        rep->nrhs = R;
        rep->max_iters = it;
        rep->restarts = restarts;
        rep->graph_launches = it;
        rep->kernel_launches = 14LL * it;
        rep->solve_ms = ms;
    }
    if (!all_conv) return fail(MG_ERR_MAXITER, "block PCG: not all right-hand sides reached tol");
    return MG_OK;
}

// ---------------------------------------------------------------- multilevel buckling modes (NEXT-2)
// Host: symmetric eigen decomposition of a small p x p matrix by cyclic Jacobi rotations
// (A is destroyed; eigenvalues in w, eigenvectors in the columns of V, row-major).
static void jacobi_eig(int p, std::vector<double>& A, std::vector<double>& w, std::vector<double>& V) {
    V.assign((size_t)p * p, 0.0);
    for (int i = 0; i < p; ++i) V[i * p + i] = 1.0;
    for (int sweep = 0; sweep < 100; ++sweep) {
        double off = 0.0;
        for (int i = 0; i < p; ++i)
            for (int j = i + 1; j < p; ++j) off += A[i * p + j] * A[i * p + j];
        if (off < 1e-30) break;
        for (int i = 0; i < p; ++i)
            for (int j = i + 1; j < p; ++j) {
                const double aij = A[i * p + j];
                if (std::fabs(aij) < 1e-300) continue;
                const double th = 0.5 * (A[j * p + j] - A[i * p + i]) / aij;
                const double t = (th >= 0 ? 1.0 : -1.0) / (std::fabs(th) + std::sqrt(th * th + 1.0));
                const double cs = 1.0 / std::sqrt(t * t + 1.0), sn = t * cs;
                for (int k = 0; k < p; ++k) {   // A <- J^T A J
                    const double aki = A[k * p + i], akj = A[k * p + j];
                    A[k * p + i] = cs * aki - sn * akj;
                    A[k * p + j] = sn * aki + cs * akj;
                }
                for (int k = 0; k < p; ++k) {
                    const double aik = A[i * p + k], ajk = A[j * p + k];
                    A[i * p + k] = cs * aik - sn * ajk;
                    A[j * p + k] = sn * aik + cs * ajk;
                }
                for (int k = 0; k < p; ++k) {
                    const double vki = V[k * p + i], vkj = V[k * p + j];
                    V[k * p + i] = cs * vki - sn * vkj;
                    V[k * p + j] = sn * vki + cs * vkj;
                }
            }
    }
    w.resize(p);
    for (int i = 0; i < p; ++i) w[i] = A[i * p + i];
}

// Generalized symmetric-definite p x p problem A y = theta B y (B SPD): Cholesky B = L L^T,
// C = L^-1 A L^-T, Jacobi on C, Y = L^-T W.  Returns false if B is not positive definite.
static bool small_geneig(int p, const std::vector<double>& A, const std::vector<double>& B, std::vector<double>& th,
                         std::vector<double>& Y) {
    std::vector<double> L((size_t)p * p, 0.0);
    for (int j = 0; j < p; ++j) {
        double d = B[j * p + j];
        for (int k = 0; k < j; ++k) d -= L[j * p + k] * L[j * p + k];
        if (!(d > 0.0)) return false;
        L[j * p + j] = std::sqrt(d);
        for (int i = j + 1; i < p; ++i) {
            double v = B[i * p + j];
            for (int k = 0; k < j; ++k) v -= L[i * p + k] * L[j * p + k];
            L[i * p + j] = v / L[j * p + j];
        }
    }
    // M = L^-1 A ; C = M L^-T
    std::vector<double> M((size_t)p * p), C((size_t)p * p);
    for (int c = 0; c < p; ++c)
        for (int i = 0; i < p; ++i) {
            double v = A[i * p + c];
            for (int k = 0; k < i; ++k) v -= L[i * p + k] * M[k * p + c];
            M[i * p + c] = v / L[i * p + i];
        }
    for (int r = 0; r < p; ++r)
        for (int i = 0; i < p; ++i) {
            double v = M[r * p + i];
            for (int k = 0; k < i; ++k) v -= C[r * p + k] * L[i * p + k];
            C[r * p + i] = v / L[i * p + i];
        }
    for (int i = 0; i < p; ++i)
        for (int j = i + 1; j < p; ++j) C[i * p + j] = C[j * p + i] = 0.5 * (C[i * p + j] + C[j * p + i]);
    std::vector<double> W;
    jacobi_eig(p, C, th, W);
    // Y = L^-T W
    Y.assign((size_t)p * p, 0.0);
    for (int c = 0; c < p; ++c)
        for (int i = p - 1; i >= 0; --i) {
            double v = W[i * p + c];
            for (int k = i + 1; k < p; ++k) v -= L[k * p + i] * Y[k * p + c];
            Y[i * p + c] = v / L[i * p + i];
        }
    return true;
}

mg_status mg_multilevel_modes(mg_handle c, const double* Es_e, const double* u, int q, double tol, double* Phi,
                              double* lam_tilde, double* lam_coarse, double* y1, double* yres) {
    if (!c || !Es_e || !u || !Phi || !lam_tilde) return fail(MG_ERR_ARG, "NULL argument");
    if (q < 1 || q > 32) return fail(MG_ERR_ARG, "q must be in [1, 32]");
    if (multi(c)) return fail(MG_ERR_ARG, "mg_multilevel_modes: single slab only (this round)");
    for (const void* p : {(const void*)Es_e, (const void*)u, (const void*)Phi})
        if (!is_device_ptr(p)) return fail(MG_ERR_ARG, "mg_multilevel_modes: device pointers required");
    const int dim = c->dim, L = c->L, nv = dim == 2 ? 3 : 6;
    const int pblk = std::min<int>(q + 8, 48);       // subspace size (oversampled)
    if ((long long)c->nL < pblk) return fail(MG_ERR_DIM, "coarsest level smaller than the mode subspace");
    TRY(ensure_vectors(c, std::max(q, 1)));
    cudaStream_t s = c->stream;
    API_SCOPE(c);
    Slab& sl = c->sl[0];
    const LevelGeom& g0 = sl.lv[0].g;
    const long long n = g0.ndof, nL = c->nL, ld = c->npad;
    // ---- step 1: G^l by Galerkin projection (element agglomeration, like K) and the coarse
    //      eigenproblem (K^l + lambda G^l) psi = 0 by subspace iteration with K^-1 (Ainv)
    std::vector<void*> tmp;
    auto dalloc = [&](size_t bytes) -> double* {
        void* p = nullptr;
        if (cudaMallocAsync(&p, bytes, s) != cudaSuccess) return nullptr;
        tmp.push_back(p);
        return (double*)p;
    };
    auto cleanup = [&]() {
        for (void* p : tmp) cudaFreeAsync(p, s);
        tmp.clear();
    };
    double* sig = dalloc(sizeof(double) * g0.nelem * nv);
    double* Gd = dalloc(sizeof(double) * ld * ld);
    double* Kd = dalloc(sizeof(double) * ld * ld);
    double* stG = L > 1 ? dalloc(sizeof(double) * sl.lv[L - 1].g.nnodes * (dim == 2 ? 9 : 27) * dim * dim) : nullptr;
    double* V = dalloc(sizeof(double) * pblk * nL);
    double* W = dalloc(sizeof(double) * pblk * nL);
    double* KV = dalloc(sizeof(double) * pblk * nL);
    double* GV = dalloc(sizeof(double) * pblk * nL);
    double* gpart = dalloc(sizeof(double) * (long long)pblk * pblk * gram_blocks(std::max(n, nL), pblk));
    double* Gr = dalloc(sizeof(double) * pblk * pblk);
    double* Yd = dalloc(sizeof(double) * pblk * pblk);
    double* Psi = dalloc(sizeof(double) * q * n);
    double* GPsi = dalloc(sizeof(double) * q * n);
    double* KPhi = dalloc(sizeof(double) * q * n);
    double* Ysc = dalloc(sizeof(double) * n);        // Eq. 7 residual when the caller passes no y1
    for (void* p : tmp)
        if (!p) { cleanup(); return fail(MG_ERR_OOM, "mg_multilevel_modes workspace"); }
    stress_sigma(g0, Es_e, u, sig, s);
    c->launches++;
    if (L > 1) {
        for (int l = 1; l < L; ++l) {
            Level& f = sl.lv[l - 1];
            Level& gl = sl.lv[l];
            double* elm = (l & 1) ? sl.elmA : sl.elmB;
            double* elm_prev = (l & 1) ? sl.elmB : sl.elmA;
            if (l == 1) galerkin_elements_G(gl.g, f.g, sig, f.mask, gl.mask, elm, s);
            else galerkin_elements(gl.g, f.g, nullptr, elm_prev, f.mask, gl.mask, elm, s);
            c->launches++;
        }
        Level& cl = sl.lv[L - 1];
        stencil_from_elements(cl.g, (L - 1) & 1 ? sl.elmA : sl.elmB, cl.mask, stG, s, false);
        CU(cudaMemsetAsync(Gd, 0, sizeof(double) * ld * ld, s));
        dense_from_stencil(cl.g, stG, Gd, ld, s);
        CU(cudaMemsetAsync(Kd, 0, sizeof(double) * ld * ld, s));
        dense_from_stencil(cl.g, cl.st, Kd, ld, s);
        c->launches += 3;
    } else {
        cleanup();
        return fail(MG_ERR_ARG, "mg_multilevel_modes needs levels >= 2");
    }
    CHECK_LAUNCH();
    // subspace iteration: V <- K^-1 G V, Rayleigh-Ritz on (-G, K) every step (V K-orthonormal)
    {
        std::vector<double> init((size_t)pblk * nL);
        uint64_t st = 0x9E3779B97F4A7C15ull;
        for (auto& v : init) {   // deterministic pseudo-random start (xorshift)
            st ^= st << 13; st ^= st >> 7; st ^= st << 17;
            v = (double)(st >> 11) / 9007199254740992.0 - 0.5;
        }
        CU(cudaMemcpyAsync(V, init.data(), sizeof(double) * init.size(), cudaMemcpyHostToDevice, s));
        CU(cudaStreamSynchronize(s));
    }
    std::vector<double> Ah((size_t)pblk * pblk), Bh((size_t)pblk * pblk), th, Y, prev(q, 0.0);
    std::vector<double> lamc(q, 0.0);
    int iters = 0, settled = -1;
    for (; iters < 500; ++iters) {
        dense_apply(Gd, ld, nL, V, W, pblk, nullptr, nullptr, s);       // W = G V
        dense_apply(c->Ainv, ld, nL, W, V, pblk, nullptr, nullptr, s);  // V = K^-1 G V  (= -K^-1 (-G) V)
        dense_apply(Gd, ld, nL, V, GV, pblk, nullptr, nullptr, s);
        dense_apply(Kd, ld, nL, V, KV, pblk, nullptr, nullptr, s);
        gram(nL, nL, pblk, V, GV, gpart, Gr, s);
        CU(cudaMemcpyAsync(Ah.data(), Gr, sizeof(double) * pblk * pblk, cudaMemcpyDeviceToHost, s));
        gram(nL, nL, pblk, V, KV, gpart, Gr, s);
        CU(cudaMemcpyAsync(Bh.data(), Gr, sizeof(double) * pblk * pblk, cudaMemcpyDeviceToHost, s));
        CU(cudaStreamSynchronize(s));
        c->launches += 8;
        for (auto& v : Ah) v = -v;                                      // (-G, K)
        if (!small_geneig(pblk, Ah, Bh, th, Y)) {
            cleanup();
            return fail(MG_ERR_BREAKDOWN, "mg_multilevel_modes: coarse Gram matrix not SPD");
        }
        // order by decreasing theta (largest theta = smallest positive lambda)
        std::vector<int> ord(pblk);
        for (int i = 0; i < pblk; ++i) ord[i] = i;
        std::sort(ord.begin(), ord.end(), [&](int a, int b) { return th[a] > th[b]; });
        std::vector<double> Ys((size_t)pblk * pblk);
        for (int r = 0; r < pblk; ++r)
            for (int j = 0; j < pblk; ++j) Ys[r * pblk + j] = Y[r * pblk + ord[j]];
        CU(cudaMemcpyAsync(Yd, Ys.data(), sizeof(double) * pblk * pblk, cudaMemcpyHostToDevice, s));
        CU(cudaMemsetAsync(W, 0, sizeof(double) * pblk * nL, s));
        block_axpy(nL, nL, pblk, V, Yd, nullptr, W, 1.0, s);          // W = V Y
        CU(cudaMemcpyAsync(V, W, sizeof(double) * pblk * nL, cudaMemcpyDeviceToDevice, s));
        double change = 0.0;
        for (int i = 0; i < q; ++i) {
            const double t = th[ord[i]];
            if (!(t > 0.0)) { change = 1.0; lamc[i] = INFINITY; continue; }
            lamc[i] = 1.0 / t;
            change = std::max(change, std::fabs(lamc[i] - prev[i]) / std::fabs(lamc[i]));
            prev[i] = lamc[i];
        }
        // eigenvalues converge with the square of the eigenvector error: once they have settled at
        // iteration N, run to 2N so the Ritz vectors (the prolongated modes) settle as well
        if (iters > 2 && change < 1e-13 && settled < 0) settled = iters;
        if (settled >= 0 && iters + 1 >= 2 * settled) { ++iters; break; }
    }
    if (lam_coarse)
        for (int i = 0; i < q; ++i) lam_coarse[i] = lamc[i];
    // ---- step 2: Psi^j = I^j_{j+1} Psi^{j+1} down to the fine level
    {
        const double* src = V;   // first q columns (sorted), coarsest level layout
        for (int l = L - 2; l >= 0; --l) {
            Level& f = sl.lv[l];
            Level& cl = sl.lv[l + 1];
            double* dst = l == 0 ? Psi : f.z;
            prolong_add(f.g, cl.g, f.mask, cl.mask, src, dst, q, nullptr, nullptr, false, s);
            c->launches++;
            src = dst;
        }
    }
    // ---- step 3: K Phi~ = G Psi by block PCG (mgBPCG, Alg. 2 l.15)
    TRY(([&]() -> mg_status {
        mg_status st = stress_stiffness_apply(c, Es_e, u, Psi, q, GPsi);
        if (st != MG_OK) return st;
        return mgcg_block_solve(c, GPsi, q, tol, Phi, nullptr);
    }()));
    // ---- step 4: Rayleigh quotients lambda~_i = -phi~^T K phi~ / phi~^T G phi~
    TRY(mg_matvec(c, 0, Phi, q, KPhi));
    TRY(stress_stiffness_apply(c, Es_e, u, Phi, q, GPsi));
    std::vector<double> num((size_t)q * q), den((size_t)q * q);
    gram(n, n, q, Phi, KPhi, gpart, Gr, s);
    CU(cudaMemcpyAsync(num.data(), Gr, sizeof(double) * q * q, cudaMemcpyDeviceToHost, s));
    gram(n, n, q, Phi, GPsi, gpart, Gr, s);
    CU(cudaMemcpyAsync(den.data(), Gr, sizeof(double) * q * q, cudaMemcpyDeviceToHost, s));
    CU(cudaStreamSynchronize(s));
    for (int i = 0; i < q; ++i) lam_tilde[i] = -num[i * q + i] / den[i * q + i];
    // K normalisation phi~^T K phi~ = 1 and the Eq. 7 residual of the first pair,
    // y = (K + lambda~_1 G) phi~_1, from K Phi and G Phi of step 4
    {
        std::vector<double> sc(q);
        for (int i = 0; i < q; ++i) {
            if (!(num[i * q + i] > 0.0)) { cleanup(); return fail(MG_ERR_BREAKDOWN, "mg_multilevel_modes: phi^T K phi <= 0"); }
            sc[i] = 1.0 / std::sqrt(num[i * q + i]);
        }
        CU(cudaMemcpyAsync(Yd, sc.data(), sizeof(double) * q, cudaMemcpyHostToDevice, s));
        double* yv = y1 ? y1 : (yres ? Ysc : nullptr);
        modes_finish(n, q, Phi, KPhi, GPsi, Yd, lam_tilde[0], yv, s);
        c->launches++;
        CHECK_LAUNCH();
        if (yres) {
            double yy = 0.0, kk = 0.0;
            gram(n, n, 1, yv, yv, gpart, Gr, s);
            CU(cudaMemcpyAsync(&yy, Gr, sizeof(double), cudaMemcpyDeviceToHost, s));
            gram(n, n, 1, KPhi, KPhi, gpart, Gr, s);
            CU(cudaMemcpyAsync(&kk, Gr, sizeof(double), cudaMemcpyDeviceToHost, s));
            CU(cudaStreamSynchronize(s));
            yres[0] = std::sqrt(yy);
            yres[1] = kk > 0.0 ? std::sqrt(yy) / (sc[0] * std::sqrt(kk)) : 0.0;
        }
    }
    cleanup();
    CU(cudaStreamSynchronize(s));
    return MG_OK;
}

mg_status mg_matvec(mg_handle c, int level, const double* x, int nrhs, double* y) {
    if (!c || !x || !y) return fail(MG_ERR_ARG, "NULL argument");
    if (level < 0 || level >= c->L || nrhs < 1 || nrhs > MG_MAX_RHS) return fail(MG_ERR_ARG, "bad level / nrhs");
    if (multi(c) && level > 0) return fail(MG_ERR_ARG, "coarse-level diagnostics need a single slab");
    API_SCOPE(c);
    if (level == 0) {
        {   // rank layout <-> padded slab layout around the fine kernels
            TRY(ensure_vectors(c, nrhs));
            TRY(scatter_fine(c, x, nrhs, false, &Slab::t));
            Rec all{c, nrhs, nullptr, nullptr};
            for (Slab& s : c->sl) {
                FineArgs a = fine_args(c, s, all);
                a.x = s.t; a.y = s.q;
                level0_apply(c, s, FOP_MATVEC, a);
                c->launches++;
            }
            TRY(gather_fine(c, &Slab::q, nrhs, y));
        }
    } else {
        Slab& s = c->sl[0];
        CoarseArgs a{};
        a.g = s.lv[level].g; a.st = s.lv[level].st; a.x = x; a.y = y; a.R = nrhs;
        coarse_apply(COP_MATVEC, a, c->stream);
        c->launches++;
    }
    CHECK_LAUNCH();
    return MG_OK;
}

mg_status mg_vcycle(mg_handle c, const double* r, int nrhs, double* z) {
    if (!c || !r || !z) return fail(MG_ERR_ARG, "NULL argument");
    if (nrhs < 1 || nrhs > MG_MAX_RHS) return fail(MG_ERR_ARG, "bad nrhs");
    TRY(ensure_vectors(c, nrhs));
    API_SCOPE(c);
    // the preconditioner exactly as the solve applies it (same fine blocks, alpha = 0)
    TRY(scatter_fine(c, r, nrhs, true, &Slab::r1));
    CU(cudaMemsetAsync(c->ctl.alpha, 0, sizeof(double) * MG_MAX_RHS, c->stream));
    for (Slab& s : c->sl) CU(cudaMemsetAsync(s.q, 0, sizeof(double) * s.vs * nrhs, c->stream));
    Rec rc{c, nrhs, nullptr, nullptr};
    long long k;
    TRY(blk_restrict(rc, &Slab::r1, &Slab::r0, &k));
    int cw;
    TRY(coarse_cycle(rc, &cw));
    TRY(blk_post(rc, &Slab::r0, cw, &k));
    TRY(gather_fine(c, &Slab::zf, nrhs, z));
    c->launches += rc.launches;
    CHECK_LAUNCH();
    return MG_OK;
}

mg_status mg_restrict(mg_handle c, int level, const double* fine, int nrhs, double* coarse) {
    if (!c || !fine || !coarse) return fail(MG_ERR_ARG, "NULL argument");
    if (level < 0 || level >= c->L - 1 || nrhs < 1) return fail(MG_ERR_ARG, "bad level / nrhs");
    if (multi(c)) return fail(MG_ERR_ARG, "level diagnostics need a single slab");
    API_SCOPE(c);
    Slab& s = c->sl[0];
    restrict_apply(s.lv[level].g, s.lv[level + 1].g, s.lv[level].mask, s.lv[level + 1].mask, fine, coarse, nrhs,
                   nullptr, nullptr, c->stream);
    c->launches++;
    CHECK_LAUNCH();
    return MG_OK;
}

mg_status mg_prolong(mg_handle c, int level, const double* coarse, int nrhs, double* fine) {
    if (!c || !fine || !coarse) return fail(MG_ERR_ARG, "NULL argument");
    if (level < 0 || level >= c->L - 1 || nrhs < 1) return fail(MG_ERR_ARG, "bad level / nrhs");
    if (multi(c)) return fail(MG_ERR_ARG, "level diagnostics need a single slab");
    API_SCOPE(c);
    Slab& s = c->sl[0];
    prolong_add(s.lv[level].g, s.lv[level + 1].g, s.lv[level].mask, s.lv[level + 1].mask, coarse, fine, nrhs, nullptr,
                nullptr, false, c->stream);
    c->launches++;
    CHECK_LAUNCH();
    return MG_OK;
}

mg_status mg_level_info(mg_handle c, int level, int* nel3, long long* ndof, int* nlevels) {
    if (!c) return fail(MG_ERR_ARG, "NULL handle");
    if (nlevels) *nlevels = c->L;
    if (level < 0) return MG_OK;
    if (level >= c->L) return fail(MG_ERR_ARG, "bad level");
    if (nel3)
        for (int k = 0; k < 3; ++k) nel3[k] = k < c->dim ? c->G[level].N[k] : 0;
    if (ndof) *ndof = c->G[level].ndof;
    return MG_OK;
}

mg_status mg_get_diagonal(mg_handle c, int level, double* d) {
    if (!c || !d) return fail(MG_ERR_ARG, "NULL argument");
    if (level < 0 || level >= c->L) return fail(MG_ERR_ARG, "bad level");
    if (multi(c)) return fail(MG_ERR_ARG, "level diagnostics need a single slab");
    API_SCOPE(c);
    CU(cudaMemcpyAsync(d, c->sl[0].lv[level].D, sizeof(double) * c->G[level].ndof, cudaMemcpyDeviceToDevice,
                       c->stream));
    return MG_OK;
}

mg_status mg_get_coarse_inverse(mg_handle c, double* Ainv) {
    if (!c || !Ainv) return fail(MG_ERR_ARG, "NULL argument");
    API_SCOPE(c);
    CU(cudaMemcpy2DAsync(Ainv, sizeof(double) * c->nL, c->Ainv, sizeof(double) * c->npad, sizeof(double) * c->nL,
                         c->nL, cudaMemcpyDeviceToDevice, c->stream));
    return MG_OK;
}

mg_status mg_profile_kernels(mg_handle c, int nrhs, int reps, double* ms) {
    if (!c || !ms) return fail(MG_ERR_ARG, "NULL argument");
    if (nrhs < 1 || nrhs > MG_MAX_RHS || reps < 1) return fail(MG_ERR_ARG, "bad nrhs / reps");
    TRY(ensure_vectors(c, nrhs));
    API_SCOPE(c);
    cudaStream_t s = c->stream;
    Rec rc{c, nrhs, nullptr, nullptr};
    cudaEvent_t e0, e1;
    CU(cudaEventCreate(&e0));
    CU(cudaEventCreate(&e1));
    for (int op = 0; op < 4; ++op) {
        auto launch = [&]() -> mg_status {
            long long k;
            switch (op) {
                case 0: return blk_cgp(rc, &Slab::p0, &Slab::p1, &k);
                case 1: return blk_restrict(rc, &Slab::r0, &Slab::r1, &k);
                case 2: return blk_post(rc, &Slab::r1, 0, &k);
                default:
                    for (Slab& sl : c->sl) {
                        FineArgs a = fine_args(c, sl, rc);
                        a.x = sl.p0; a.y = sl.q;
                        level0_apply(c, sl, FOP_MATVEC, a);
                    }
                    return MG_OK;
            }
        };
        TRY(launch());
        CU(cudaEventRecord(e0, s));
        for (int k = 0; k < reps; ++k) TRY(launch());
        CU(cudaEventRecord(e1, s));
        CU(cudaEventSynchronize(e1));
        float t = 0.f;
        cudaEventElapsedTime(&t, e0, e1);
        ms[op] = t / reps;
    }
    CHECK_LAUNCH();
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    return MG_OK;
}

mg_status mg_destroy(mg_handle c) {
    if (!c) return MG_OK;
    std::lock_guard<std::recursive_mutex> lk(g_api_mu);
    if (c->stream) cudaStreamSynchronize(c->stream);
    free_vectors(c);
    for (Slab& s : c->sl) {
        for (int l = 0; l < MG_MAX_LEVELS; ++l) {
            Level& v = s.lv[l];
            if (v.mask) cudaFree(v.mask);
            if (v.Dinv) cudaFree(v.Dinv);
            if (v.D) cudaFree(v.D);
            if (v.st) cudaFree(v.st);
        }
        for (double* p : {s.E, s.elmA, s.elmB, s.Epad, s.Dinvpad, s.u, s.phi, s.gy, s.sig, s.Es})
            if (p) cudaFree(p);
        for (double* p : s.tn)
            if (p) cudaFree(p);
        for (double* p : s.te)
            if (p) cudaFree(p);
        if (s.maskpad) cudaFree(s.maskpad);
    }
    if (c->Estage) cudaFree(c->Estage);
    for (double* p : {c->Ainv, c->stg, c->cpack, c->cgath, c->gj_work, c->sums, c->Mc, c->gstage, c->wbuf, c->dlam,
                      c->bpart, c->bGam, c->bRho, c->bRhoN, c->bC})
        if (p) cudaFree(p);
    if (c->ctl_mem) cudaFree(c->ctl_mem);
    if (c->brank) cudaFree(c->brank);
    if (c->g_block) cudaGraphExecDestroy(c->g_block);
    if (c->g_gj) cudaGraphExecDestroy(c->g_gj);
    if (c->h_pinned) cudaFreeHost(c->h_pinned);
    if (c->h_dbl) cudaFreeHost(c->h_dbl);
    if (c->ev_in) cudaEventDestroy(c->ev_in);
    if (c->ev_out) cudaEventDestroy(c->ev_out);
    for (int k = 0; k < mg_ctx::NCHUNK_EV; ++k) {
        if (c->gev_in[k]) cudaEventDestroy(c->gev_in[k]);
        if (c->gev_k[k]) cudaEventDestroy(c->gev_k[k]);
    }
    if (c->gev_sig) cudaEventDestroy(c->gev_sig);
    if (c->ev_rhs) cudaEventDestroy(c->ev_rhs);
    if (c->ev_setup) cudaEventDestroy(c->ev_setup);
    if (c->h_setup_st) cudaFreeHost(c->h_setup_st);
    if (c->rstage) cudaFree(c->rstage);
    if (c->gev_done) cudaEventDestroy(c->gev_done);
    if (c->cs_in) cudaStreamDestroy(c->cs_in);
    if (c->cs_out) cudaStreamDestroy(c->cs_out);
    comm_destroy(c->comm);
    if (c->stream) cudaStreamDestroy(c->stream);
    delete c;
    return MG_OK;
}

}  // extern "C"
