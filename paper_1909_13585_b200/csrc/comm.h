// Halo exchange / collectives between axis-0 slabs (see comm.cu).
#pragma once
#include <cuda_runtime.h>
#include <nccl.h>
#include <string.h>

struct Comm {
    int rank = 0, nranks = 1;
    void* nccl = nullptr;   // ncclComm_t when nranks > 1
    // staging for packed halo messages (all vectors of a boundary plane in one message):
    // send-down, send-up, recv-down, recv-up, `stage_cap` bytes each (comm_reserve, outside capture)
    char* stage = nullptr;
    size_t stage_cap = 0;
    bool stage_local = false;   // MG_COMM_STAGE=1: in-process neighbours through the staging path too
};

// One field (vector family, mask, diagonal, element matrices ...) on one slab: plane p of
// vector v starts at base + (v * vec_stride + p * plane_len) * esize.  Planes are node planes
// (or element layers) along axis 0 in local numbering.
struct PlaneField {
    void* base;
    int esize;              // 8 (fp64) or 1 (uint8 masks)
    long long plane_len;    // elements per plane
    long long vec_stride;   // elements between consecutive vectors
    int nvec;
    int first_own, last_own;  // owned planes [first_own, last_own]
    int lo_ghost, hi_ghost;   // ghost plane indices or -1
    int dirs;                 // 1: lower's last owned -> upper's lo ghost; 2: upper's first owned -> lower's hi ghost
};

bool comm_init(Comm& c, int rank, int nranks, const void* id128);
bool comm_reserve(Comm& c, size_t bytes_per_message);
void comm_destroy(Comm& c);
bool comm_nccl_unique_id(void* out128);
const char* comm_last_error();

bool halo_forward(const Comm& c, const PlaneField* f, int nslab, cudaStream_t s);
bool halo_reverse_add(const Comm& c, const PlaneField* f, int nslab, double* tmp, cudaStream_t s);
bool comm_allreduce_sum(const Comm& c, double* d, long long n, cudaStream_t s);
bool comm_allgather(const Comm& c, const void* send, void* recv, size_t bytes_per_rank, cudaStream_t s);
