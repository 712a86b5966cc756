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
    const uint32_t* flags;  // may be null (all 0)
};
enum : unsigned { FLAG_EUROPEAN = 1u, FLAG_CASH = 2u, FLAG_COST_T0 = 4u, FLAG_ALL = 7u };

// mirrors amtc_quote (24 bytes)
struct Quote {
    double ask, bid;
    int status, max_bp;
};
static_assert(sizeof(Quote) == 24, "amtc_quote layout");

void note_launch();

constexpr int TC_CLASSES = 64;  // cost classes 1 + floor(4 k/h) up to k/h = 15.5 (config 4 reaches 12.5)

// amtc_prepare.cu
void tc_launch_prepare(const BatchPtrs& in, int64_t n, int N, Quote* out, unsigned char* cls, int* hist,
                       int* items, cudaStream_t s);
void launch_status_reduce(Quote* out, int64_t n, int* worst, cudaStream_t s);
void tc_launch_mark_capacity(const int* items, int n_items, Quote* out, cudaStream_t s);
// every option still STATUS_OK -> ECAPACITY with NaN prices (no workspace fits)
void tc_launch_mark_all_capacity(Quote* out, int64_t n, cudaStream_t s);

// amtc_strip.cu (the transaction-cost solver)
struct StripLaunchArgs {
    BatchPtrs in;
    int N;
    Quote* out;
    const int* items;    // item codes 2*option + party
    const int* n_items;  // device: number of queued items
    int* work_counter;
    int* ovf_items;      // items that overflowed this pass
    int* ovf_count;
    unsigned long long* vertex_sum;  // sum of produced vertex counts (work metric)
    char* ws;            // per-warp workspaces
    size_t ws_stride;    // bytes per warp
    int level;           // capacity level (0 = first pass; +1 = 4x arenas)
    int ctas;
    // split mode (strips of one tree on different warps); split_S = 0: off
    int split_S = 0;
    int* progress = nullptr;
    char* carry = nullptr;
    size_t carry_stride = 0;
    void* carena_split = nullptr;
    int* carena_cnt = nullptr;
    int carena_split_cap = 0;
    // light kernel (no tier 3) and the first item of the launch (device pointer)
    bool light = false;
    const int* item_lo = nullptr;
    // sharded single tree (split mode over GPUs)
    int peer_strip = -1;
    int sys_fence = 0;
    char* peer_carry = nullptr;
    void* peer_carena = nullptr;
    int* peer_progress = nullptr;
    double* hedge = nullptr;  // optional root hedges (2 n doubles, device)
};
// the transaction-cost tree sharded over the ranks of an NCCL communicator
// (amtc_capi.cu); comm is an ncclComm_t
int tc_tree_sharded(const void* params, int N, const void* payoff, double k, void* comm, int rank, int nranks,
                    void* out, cudaStream_t s);
size_t strip_ws_bytes_per_warp_light(int N);
size_t strip_ws_bytes_per_warp_split(int N);
int strip_split_warps_per_cta();
int strip_light_warps_per_cta();
int strip_light_ctas_per_sm();
size_t strip_carry_bytes(int N);
int strip_split_arena_cap(int N);
size_t strip_vtx_bytes();
void tc_launch_split_expand(const int* items, const int* n_items, int S, int64_t max_items, int* out, int* n_out,
                            cudaStream_t s, int s_lo = 0, int s_hi = -1);
size_t strip_ws_bytes_per_warp(int N, int level);
int strip_warps_per_cta();
int strip_ctas_per_sm();
int strip_launch(const StripLaunchArgs& a, cudaStream_t s);
void strip_set_heavy_threshold(int tl);
void strip_set_arena_shift(int sh);
// the capacities (vertices) of capacity level `level` (arena shift and heavy
// threshold testing hooks applied), shared by the full solver
void strip_tc_caps(int N, int level, int& rarena, int& carena, int& hscr, int& zbuf, int& tl);

// amtc_full.cu (the full solver of the batched path: strip matrix + arenas + tier 3)
size_t full_ws_bytes_per_warp(int N, int level);
int full_warps_per_cta();
int full_ctas_per_sm();
int full_launch(const StripLaunchArgs& a, cudaStream_t s);
int full_profile(unsigned long long out[8], int reset);

// amtc_light.cu (the light solver: small node functions, no tiers)
size_t light2_ws_bytes_per_warp(int N);
int light2_warps_per_cta();
int light2_ctas_per_sm();
int light2_launch(const StripLaunchArgs& a, cudaStream_t s);
size_t light2_split_carry_bytes(int N);
int light_profile(unsigned long long out[8], int reset);  // -DAMTC_L2_PROF=1 developer counters  // one (tree, strip) carry column of the light kernel's split mode

// amtc_crr.cu
int crr_launch(const BatchPtrs& in, int64_t n, int N, double* out, cudaStream_t s);
int crr_max_n();
// N > crr_max_n(): strip kernel with a per-warp carry workspace (crr_strip_ws_bytes)
int64_t crr_strip_warps(int64_t n);
size_t crr_strip_ws_bytes(int N, int64_t warps);
int crr_strip_launch(const BatchPtrs& in, int64_t n, int N, double* out, double* ws, int64_t warps, cudaStream_t s);

}  // namespace amtc
