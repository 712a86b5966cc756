// amtc_internal.cuh -- types shared by the CUDA translation units of libamtc
// (not part of the public C-ABI, see include/amtc.h).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

namespace amtc {

enum : int { KIND_PUT = 0, KIND_CALL = 1, KIND_BULL = 2 };
enum : int {
    STATUS_OK = 0,
    STATUS_EINVAL = 1,
    STATUS_EARBITRAGE = 2,
    STATUS_ECAPACITY = 3,
    STATUS_EUNBOUNDED = 4,
    STATUS_ECUDA = 5,
    STATUS_ENCCL = 6
};

// mirrors amtc_batch_soa (device pointers)
struct BatchPtrs {
    const double* S0;
    const double* K;
    const double* K2;
    const double* T;
    const double* sigma;
    const double* R;
    const double* k;
    const int32_t* kind;
};

// mirrors amtc_quote (24 bytes)
struct Quote {
    double ask, bid;
    int status, max_bp;
};
static_assert(sizeof(Quote) == 24, "amtc_quote layout");

constexpr int TC_THREADS = 128;

void note_launch();

// amtc_tc.cu
struct TcLaunch {
    BatchPtrs in;
    int N;
    Quote* out;
    const int* items;  // item codes 2*option + party
    const int* n_items;  // device: number of queued items
    int* work_counter;
    int* ovf_items;    // items that overflowed this pass
    int* ovf_count;
    unsigned long long* vertex_sum;  // sum of output vertex counts (work metric)
    char* ws;          // per-CTA workspaces
    size_t ws_stride;  // bytes per CTA
    int arena_cap;     // vertices per arena
    int bmul, badd;    // per-node scratch bound b = bmul (nU + nD) + badd
};
size_t tc_workspace_bytes(int N, int arena_cap);
constexpr int TC_CLASSES = 16;
void tc_launch_prepare(const BatchPtrs& in, int64_t n, int N, Quote* out, unsigned char* cls, int* hist,
                       int* items, cudaStream_t s);
void launch_status_reduce(const Quote* out, int64_t n, int* worst, cudaStream_t s);
void tc_launch_solve(const TcLaunch& L, int grid, cudaStream_t s);
void tc_launch_mark_capacity(const int* items, int n_items, Quote* out, cudaStream_t s);
int tc_solve_occupancy();

// amtc_tc2.cu (shared-memory solver)
struct Tc2Launch {
    BatchPtrs in;
    int N;
    Quote* out;
    const int* items;
    const int* n_items;
    int* work_counter;
    int* ovf_items;
    int* ovf_count;
    unsigned long long* vertex_sum;
    char* ws;
    size_t ws_stride;
    int big_cap;    // vertices per big arena (two per CTA)
    int heavy_scr;  // vertices of warp-cooperative scratch per warp
};
size_t tc2_workspace_bytes(int N, int big_cap, int heavy_scr);
int tc2_launch(const Tc2Launch& L, int grid, cudaStream_t s);
int tc2_max_n();
int tc2_pick_ks(int N);

// amtc_crr.cu
int crr_launch(const BatchPtrs& in, int64_t n, int N, double* out, cudaStream_t s);
int crr_max_n();

}  // namespace amtc
