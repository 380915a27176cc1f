// Slab decomposition along axis 0 (BASELINE.json:5 "partitioned into slabs ...
// NCCL halo exchange over NVLink and allreduce for CG dot products").
//
// A handle holds `nslab` consecutive slabs of the global grid; the job holds
// nranks x nslab slabs (one process per GPU, ranks in slab order).  Every slab stores one
// ghost node plane on each side that has a neighbour (and the ghost element layer below),
// so a fine or coarse operator application is exact on the slab's owned planes.  Three
// exchange patterns keep the ghosts valid:
//   forward      owned boundary plane -> neighbour's ghost plane (both directions)
//   reverse-add  restriction partial sum held in the upper ghost plane -> added into the
//                upper neighbour's first owned plane
//   allreduce    per-RHS dot products (CG alpha / beta / convergence)
// Neighbours inside the handle exchange by device copies on the handle's stream; neighbours
// on other ranks through NCCL point-to-point and collectives (loaded with dlopen so the
// library has no link-time NCCL dependency; all calls are stream-ordered and CUDA-graph
// capturable).
#include <dlfcn.h>

#include <cstdio>
#include <cstdlib>
#include <string>

#include "comm.h"

// ---------------------------------------------------------------- NCCL entry points
namespace {
struct NcclApi {
    bool loaded = false;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
};
NcclApi g_nccl;
std::string g_nccl_err;

bool load_nccl() {
    if (g_nccl.loaded) return true;
    void* h = nullptr;
    if (const char* p = std::getenv("MG_NCCL_LIB")) h = dlopen(p, RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
        g_nccl_err = std::string("dlopen libnccl.so.2 failed (set MG_NCCL_LIB): ") + dlerror();
        return false;
    }
#define SYM(field, name)                                                             \
    g_nccl.field = reinterpret_cast<decltype(g_nccl.field)>(dlsym(h, name));          \
    if (!g_nccl.field) {                                                             \
        g_nccl_err = std::string("NCCL symbol missing: ") + name;                    \
        return false;                                                                \
    }
    SYM(GetUniqueId, "ncclGetUniqueId");
    SYM(CommInitRank, "ncclCommInitRank");
    SYM(CommDestroy, "ncclCommDestroy");
    SYM(Send, "ncclSend");
    SYM(Recv, "ncclRecv");
    SYM(GroupStart, "ncclGroupStart");
    SYM(GroupEnd, "ncclGroupEnd");
    SYM(AllReduce, "ncclAllReduce");
    SYM(AllGather, "ncclAllGather");
    SYM(GetErrorString, "ncclGetErrorString");
#undef SYM
    g_nccl.loaded = true;
    return true;
}

bool nccl_ok(ncclResult_t r, const char* what) {
    if (r == ncclSuccess) return true;
    g_nccl_err = std::string(what) + ": " + (g_nccl.GetErrorString ? g_nccl.GetErrorString(r) : "error");
    return false;
}

// dst[v][i] += src[v][i] for one plane of nvec vectors
__global__ void plane_add_kernel(double* dst, long long dst_stride, const double* src, long long src_stride,
                                 long long len) {
    const int v = blockIdx.y;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < len; i += (long long)gridDim.x * blockDim.x)
        dst[v * dst_stride + i] += src[v * src_stride + i];
}

void plane_add(double* dst, long long dst_stride, const double* src, long long src_stride, long long len, int nvec,
               cudaStream_t s) {
    unsigned bx = (unsigned)((len + 255) / 256);
    if (bx > 148) bx = 148;
    plane_add_kernel<<<dim3(bx, nvec), 256, 0, s>>>(dst, dst_stride, src, src_stride, len);
}

char* plane_ptr(const PlaneField& f, int plane) {
    return static_cast<char*>(f.base) + (long long)plane * f.plane_len * f.esize;
}
}  // namespace

const char* comm_last_error() { return g_nccl_err.c_str(); }

bool comm_nccl_unique_id(void* out128) {
    if (!load_nccl()) return false;
    ncclUniqueId id;
    if (!nccl_ok(g_nccl.GetUniqueId(&id), "ncclGetUniqueId")) return false;
    memcpy(out128, &id, sizeof(id));
    return true;
}

bool comm_init(Comm& c, int rank, int nranks, const void* id128) {
    c.rank = rank;
    c.nranks = nranks;
    c.nccl = nullptr;
    c.stage_local = std::getenv("MG_COMM_STAGE") && std::atoi(std::getenv("MG_COMM_STAGE")) == 1;
    if (nranks <= 1) return true;
    if (!load_nccl()) return false;
    ncclUniqueId id;
    memcpy(&id, id128, sizeof(id));
    ncclComm_t comm = nullptr;
    if (!nccl_ok(g_nccl.CommInitRank(&comm, nranks, id, rank), "ncclCommInitRank")) return false;
    c.nccl = comm;
    return true;
}

void comm_destroy(Comm& c) {
    if (c.nccl && g_nccl.loaded) g_nccl.CommDestroy(static_cast<ncclComm_t>(c.nccl));
    c.nccl = nullptr;
    if (c.stage) cudaFree(c.stage);
    c.stage = nullptr;
    c.stage_cap = 0;
}

bool comm_reserve(Comm& c, size_t bytes) {
    if (c.nranks <= 1 && !c.stage_local) return true;
    bytes = (bytes + 255) / 256 * 256;
    if (bytes <= c.stage_cap) return true;
    if (c.stage) cudaFree(c.stage);
    c.stage = nullptr;
    c.stage_cap = 0;
    if (cudaMalloc(&c.stage, 4 * bytes) != cudaSuccess) {
        g_nccl_err = "comm_reserve: cudaMalloc of the halo staging failed";
        return false;
    }
    c.stage_cap = bytes;
    return true;
}

namespace {
// all nvec vectors of one plane <-> a contiguous message (nvec x plane bytes)
bool pack_plane(char* buf, const PlaneField& f, int plane, cudaStream_t s) {
    const size_t w = (size_t)f.plane_len * f.esize;
    return cudaMemcpy2DAsync(buf, w, plane_ptr(f, plane), (size_t)f.vec_stride * f.esize, w, f.nvec,
                             cudaMemcpyDeviceToDevice, s) == cudaSuccess;
}
bool unpack_plane(const PlaneField& f, int plane, const char* buf, cudaStream_t s) {
    const size_t w = (size_t)f.plane_len * f.esize;
    return cudaMemcpy2DAsync(plane_ptr(f, plane), (size_t)f.vec_stride * f.esize, buf, w, w, f.nvec,
                             cudaMemcpyDeviceToDevice, s) == cudaSuccess;
}
size_t msg_bytes(const PlaneField& f) { return (size_t)f.plane_len * f.esize * f.nvec; }
}  // namespace

// ---------------------------------------------------------------- exchanges
// f[k]: the field on local slab k (slabs in axis-0 order).
bool halo_forward(const Comm& c, const PlaneField* f, int nslab, cudaStream_t s) {
    auto copy_plane = [&](const PlaneField& dst, int pd, const PlaneField& src, int ps) {
        const size_t w = (size_t)src.plane_len * src.esize;
        return cudaMemcpy2DAsync(plane_ptr(dst, pd), (size_t)dst.vec_stride * dst.esize, plane_ptr(src, ps),
                                 (size_t)src.vec_stride * src.esize, w, src.nvec, cudaMemcpyDeviceToDevice,
                                 s) == cudaSuccess;
    };
    for (int k = 0; k + 1 < nslab; ++k) {
        const PlaneField& lo = f[k];
        const PlaneField& up = f[k + 1];
        if (c.stage_local && lo.nvec > 1 && msg_bytes(lo) <= c.stage_cap) {
            // the packed-message path of the cross-rank exchange, with a device copy as transport
            // (MG_COMM_STAGE=1: exercises the packing on one GPU)
            char* sbuf = c.stage;
            char* rbuf = c.stage + 2 * c.stage_cap;
            const size_t mb = msg_bytes(lo);
            if (lo.dirs & 1) {
                if (!pack_plane(sbuf, lo, lo.last_own, s)) return false;
                if (cudaMemcpyAsync(rbuf, sbuf, mb, cudaMemcpyDeviceToDevice, s) != cudaSuccess) return false;
                if (!unpack_plane(up, up.lo_ghost, rbuf, s)) return false;
            }
            if (lo.dirs & 2) {
                if (!pack_plane(sbuf, up, up.first_own, s)) return false;
                if (cudaMemcpyAsync(rbuf, sbuf, mb, cudaMemcpyDeviceToDevice, s) != cudaSuccess) return false;
                if (!unpack_plane(lo, lo.hi_ghost, rbuf, s)) return false;
            }
            continue;
        }
        if ((lo.dirs & 1) && !copy_plane(up, up.lo_ghost, lo, lo.last_own)) return false;
        if ((lo.dirs & 2) && !copy_plane(lo, lo.hi_ghost, up, up.first_own)) return false;
    }
    if (c.nranks <= 1) return true;
    // across ranks: first local slab <-> rank - 1, last local slab <-> rank + 1
    const PlaneField& first = f[0];
    const PlaneField& last = f[nslab - 1];
    ncclComm_t comm = static_cast<ncclComm_t>(c.nccl);
    const ncclDataType_t ty = first.esize == 8 ? ncclFloat64 : ncclUint8;
    const size_t cnt = (size_t)first.plane_len;
    const int dirs = first.dirs;
    const bool lower = c.rank > 0, upper = c.rank + 1 < c.nranks;
    if (first.nvec > 1 && msg_bytes(first) <= c.stage_cap) {
        // one message per neighbour and direction: the boundary plane of all nvec vectors packed
        char* s_dn = c.stage;
        char* s_up = c.stage + c.stage_cap;
        char* r_dn = c.stage + 2 * c.stage_cap;
        char* r_up = c.stage + 3 * c.stage_cap;
        const size_t n_all = cnt * first.nvec;
        if (lower && (dirs & 2) && !pack_plane(s_dn, first, first.first_own, s)) return false;
        if (upper && (dirs & 1) && !pack_plane(s_up, last, last.last_own, s)) return false;
        if (!nccl_ok(g_nccl.GroupStart(), "ncclGroupStart")) return false;
        if (lower) {
            if (dirs & 2) g_nccl.Send(s_dn, n_all, ty, c.rank - 1, comm, s);
            if (dirs & 1) g_nccl.Recv(r_dn, n_all, ty, c.rank - 1, comm, s);
        }
        if (upper) {
            if (dirs & 1) g_nccl.Send(s_up, n_all, ty, c.rank + 1, comm, s);
            if (dirs & 2) g_nccl.Recv(r_up, n_all, ty, c.rank + 1, comm, s);
        }
        if (!nccl_ok(g_nccl.GroupEnd(), "ncclGroupEnd")) return false;
        if (lower && (dirs & 1) && !unpack_plane(first, first.lo_ghost, r_dn, s)) return false;
        if (upper && (dirs & 2) && !unpack_plane(last, last.hi_ghost, r_up, s)) return false;
        return true;
    }
    if (!nccl_ok(g_nccl.GroupStart(), "ncclGroupStart")) return false;
    for (int v = 0; v < first.nvec; ++v) {
        const long long ofl = (long long)v * first.vec_stride * first.esize;
        const long long oll = (long long)v * last.vec_stride * last.esize;
        if (lower) {
            if (dirs & 2) g_nccl.Send(plane_ptr(first, first.first_own) + ofl, cnt, ty, c.rank - 1, comm, s);
            if (dirs & 1) g_nccl.Recv(plane_ptr(first, first.lo_ghost) + ofl, cnt, ty, c.rank - 1, comm, s);
        }
        if (upper) {
            if (dirs & 1) g_nccl.Send(plane_ptr(last, last.last_own) + oll, cnt, ty, c.rank + 1, comm, s);
            if (dirs & 2) g_nccl.Recv(plane_ptr(last, last.hi_ghost) + oll, cnt, ty, c.rank + 1, comm, s);
        }
    }
    return nccl_ok(g_nccl.GroupEnd(), "ncclGroupEnd");
}

// upper ghost plane (partial restriction sums) of each slab -> added into the first owned
// plane of the slab above.  fp64 fields only; tmp: nvec * plane_len doubles (NCCL receive).
bool halo_reverse_add(const Comm& c, const PlaneField* f, int nslab, double* tmp, cudaStream_t s) {
    for (int k = 0; k + 1 < nslab; ++k) {
        const PlaneField& lo = f[k];
        const PlaneField& up = f[k + 1];
        plane_add(reinterpret_cast<double*>(plane_ptr(up, up.first_own)), up.vec_stride,
                  reinterpret_cast<const double*>(plane_ptr(lo, lo.hi_ghost)), lo.vec_stride, lo.plane_len,
                  lo.nvec, s);
    }
    if (c.nranks <= 1) return true;
    const PlaneField& first = f[0];
    const PlaneField& last = f[nslab - 1];
    ncclComm_t comm = static_cast<ncclComm_t>(c.nccl);
    const bool packed = first.nvec > 1 && msg_bytes(last) <= c.stage_cap;
    if (packed && c.rank + 1 < c.nranks && !pack_plane(c.stage + c.stage_cap, last, last.hi_ghost, s)) return false;
    if (!nccl_ok(g_nccl.GroupStart(), "ncclGroupStart")) return false;
    if (packed) {   // one message: the upper ghost plane of all vectors; received contiguous into tmp
        if (c.rank + 1 < c.nranks)
            g_nccl.Send(c.stage + c.stage_cap, (size_t)last.plane_len * last.nvec, ncclFloat64, c.rank + 1, comm, s);
        if (c.rank > 0) g_nccl.Recv(tmp, (size_t)first.plane_len * first.nvec, ncclFloat64, c.rank - 1, comm, s);
    } else {
        for (int v = 0; v < first.nvec; ++v) {
            if (c.rank + 1 < c.nranks)
                g_nccl.Send(plane_ptr(last, last.hi_ghost) + (long long)v * last.vec_stride * 8, last.plane_len,
                            ncclFloat64, c.rank + 1, comm, s);
            if (c.rank > 0)
                g_nccl.Recv(tmp + (long long)v * first.plane_len, first.plane_len, ncclFloat64, c.rank - 1, comm, s);
        }
    }
    if (!nccl_ok(g_nccl.GroupEnd(), "ncclGroupEnd")) return false;
    if (c.rank > 0)
        plane_add(reinterpret_cast<double*>(plane_ptr(first, first.first_own)), first.vec_stride, tmp,
                  first.plane_len, first.plane_len, first.nvec, s);
    return true;
}

bool comm_allreduce_sum(const Comm& c, double* d, long long n, cudaStream_t s) {
    if (c.nranks <= 1) return true;
    return nccl_ok(g_nccl.AllReduce(d, d, (size_t)n, ncclFloat64, ncclSum, static_cast<ncclComm_t>(c.nccl), s),
                   "ncclAllReduce");
}

bool comm_allgather(const Comm& c, const void* send, void* recv, size_t bytes_per_rank, cudaStream_t s) {
    if (c.nranks <= 1) {
        if (send != recv) return cudaMemcpyAsync(recv, send, bytes_per_rank, cudaMemcpyDeviceToDevice, s) == cudaSuccess;
        return true;
    }
    return nccl_ok(g_nccl.AllGather(send, recv, bytes_per_rank, ncclUint8, static_cast<ncclComm_t>(c.nccl), s),
                   "ncclAllGather");
}
