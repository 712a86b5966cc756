// amtc_capi.cu -- the C-ABI of include/amtc.h (host side).
//
// Owns per-device scratch (grow-only, mutex-guarded), validates arguments,
// schedules the transaction-cost passes (first pass with small per-node
// scratch bounds for every item, then re-runs of overflowed items with larger
// bounds and fewer resident CTAs), and marshals host buffers for the *_host
// variants.  No exception crosses the boundary.
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "amtc.h"
#include "amtc_internal.cuh"

namespace amtc {

static std::atomic<int64_t> g_launches{0};
void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

static thread_local std::string g_last_error;

static int cuda_fail(cudaError_t e, const char* what) {
    g_last_error = std::string(what) + ": " + cudaGetErrorString(e);
    return STATUS_ECUDA;
}

#define AMTC_CUDA(call)                                  \
    do {                                                 \
        cudaError_t e_ = (call);                         \
        if (e_ != cudaSuccess) return cuda_fail(e_, #call); \
    } while (0)

// grow-only device buffer
struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
    cudaError_t ensure(size_t want) {
        if (want <= bytes) return cudaSuccess;
        if (p) cudaFree(p);
        p = nullptr;
        bytes = 0;
        cudaError_t e = cudaMalloc(&p, want);
        if (e == cudaSuccess) bytes = want;
        return e;
    }
};

struct DevState {
    std::mutex mu;
    DevBuf items[2], cls, small, ws, stage_in, stage_out;
    DevBuf sp_items, sp_progress, sp_carry, sp_arena, sp_cnt;  // split mode
    DevBuf ws_light;                                          // light-kernel workspaces
    DevBuf crr_ws;                                            // CRR strip kernel carry buffers (N > 1152)
    DevBuf ipc;                                               // IPC handle exchange
    cudaStream_t s2 = nullptr;                                // light-kernel stream
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    size_t budget = 0;  // cached workspace budget (bytes)
    void* h_stage = nullptr;  // pinned host staging of small host batches
    size_t h_stage_bytes = 0;
    size_t held() const {
        return ws.bytes + sp_items.bytes + sp_progress.bytes + sp_carry.bytes + sp_arena.bytes + sp_cnt.bytes +
               ws_light.bytes;
    }
    int sm_count = 0;
    int occupancy = 0;
    int light_occupancy = 0;
    int light2_occupancy = 0;
    int full_occupancy = 0;
    // stats of the last TC batch
    unsigned long long vertex_sum = 0;
    int passes = 0;
    int64_t retried = 0;
    double solve_ms = 0.0;   // device time of the solver launches (CUDA events)
    double full_ms = 0.0, light_ms = 0.0;  // first pass: each kernel on its own stream
    cudaEvent_t ev[2 * 8] = {};
    cudaEvent_t kev[4] = {};  // full kernel start / end (stream s), light kernel start / end (stream s2)
};

static DevState* state_for_device(int dev) {
    static std::mutex mu;
    static std::vector<DevState*> states;
    std::lock_guard<std::mutex> g(mu);
    if ((int)states.size() <= dev) states.resize(dev + 1, nullptr);
    if (!states[dev]) states[dev] = new DevState();
    return states[dev];
}

static BatchPtrs to_ptrs(const amtc_batch_soa* b) {
    BatchPtrs p;
    p.S0 = b->S0; p.K = b->K; p.K2 = b->K2; p.T = b->T;
    p.sigma = b->sigma; p.R = b->R; p.k = b->k; p.kind = b->kind; p.flags = b->flags;
    return p;
}

static bool soa_ok(const amtc_batch_soa* b) {
    return b && b->S0 && b->K && b->T && b->sigma && b->R && b->kind;
}

// small device scratch layout (ints)
enum { SM_HIST = 0, SM_WORK = TC_CLASSES + 1, SM_OVF0, SM_OVF1, SM_WORST, SM_SPLITN, SM_WORK2,
       SM_VSUM = TC_CLASSES + 8 /* 8-byte aligned */, SM_INTS = TC_CLASSES + 16 };
static_assert(SM_WORK2 < SM_VSUM && SM_VSUM % 2 == 0 && SM_VSUM + 2 <= SM_INTS, "small scratch layout");

// split mode policy (testing hook amtc_debug_set_split_mode): -1 auto, 0 off, 1 on when it fits
static int g_split_mode = -1;
// light kernel for class-0 items (testing hook amtc_debug_set_light_kernel):
// 1 = amtc_light.cu (default), 2 = the strip kernel's light variant, 0 = none
static int g_light_kernel = 1;
// the whole-tree solver for the other items (testing hook amtc_debug_set_full_kernel):
// 1 = amtc_full.cu, 0 = the strip kernel (amtc_strip.cu; default: faster on the whole config-4 batch)
static int g_full_kernel = 0;
// split mode of the light kernel for batches of light trees (testing hook amtc_debug_set_light_split)
static int g_light_split = 1;

// solver passes: every item first runs at capacity level 0; items that
// overflowed a capacity (arena, scratch) are re-run at the next level (4x the
// arenas, fewer concurrent warps), up to kMaxLevel; then ECAPACITY.
constexpr int kMaxLevel = 4;

static int tc_batch_device(const amtc_batch_soa* d_in, int64_t n, int32_t N, amtc_quote* d_out,
                           cudaStream_t s, double* d_hedge = nullptr) {
    if (!soa_ok(d_in) || !d_out || n < 0 || N < 1) return STATUS_EINVAL;
    if (n == 0) return STATUS_OK;
    if (2 * n > (int64_t)INT32_MAX / 2) return STATUS_EINVAL;
    int dev = 0;
    AMTC_CUDA(cudaGetDevice(&dev));
    DevState* st = state_for_device(dev);
    std::lock_guard<std::mutex> guard(st->mu);
    if (!st->sm_count) {
        AMTC_CUDA(cudaDeviceGetAttribute(&st->sm_count, cudaDevAttrMultiProcessorCount, dev));
        st->occupancy = strip_ctas_per_sm();
        st->light_occupancy = strip_light_ctas_per_sm();
        st->light2_occupancy = light2_ctas_per_sm();
        st->full_occupancy = full_ctas_per_sm();
        if (st->occupancy < 1 || st->full_occupancy < 1) {
            g_last_error = "strip solver cannot be resident on this device";
            return STATUS_ECUDA;
        }
    }
    const int64_t n2 = 2 * n;
    AMTC_CUDA(st->items[0].ensure(sizeof(int) * n2));
    AMTC_CUDA(st->items[1].ensure(sizeof(int) * n2));
    AMTC_CUDA(st->cls.ensure(n2));
    AMTC_CUDA(st->small.ensure(sizeof(int) * SM_INTS));
    int* small = static_cast<int*>(st->small.p);
    Quote* out = reinterpret_cast<Quote*>(d_out);
    BatchPtrs in = to_ptrs(d_in);

    tc_launch_prepare(in, n, N, out, static_cast<unsigned char*>(st->cls.p), small + SM_HIST,
                      static_cast<int*>(st->items[0].p), s);
    AMTC_CUDA(cudaGetLastError());
    AMTC_CUDA(cudaMemsetAsync(small + SM_VSUM, 0, sizeof(unsigned long long), s));

    // workspace budget: 60% of (free + what this library already holds), at most
    // 48 GB; cudaMemGetInfo is queried once per device and refreshed only when
    // a call would need more than the cached budget allows
    auto refresh_budget = [&]() -> int {
        size_t free_b = 0, total_b = 0;
        AMTC_CUDA(cudaMemGetInfo(&free_b, &total_b));
        st->budget = std::min<size_t>((size_t)(0.6 * (double)(free_b + st->held())), (size_t)48 << 30);
        return STATUS_OK;
    };
    if (!st->budget) {
        if (int rc = refresh_budget()) return rc;
    }
    size_t budget = st->budget;

    const int* q_items = static_cast<int*>(st->items[0].p);
    const int* q_count = small + SM_HIST + TC_CLASSES;  // total valid items
    int64_t queued = n2;                                // upper bound for grid sizing
    int ovf_host = 0;
    int passes = 0;
    const int wpc = strip_warps_per_cta();
    const bool full2 = g_full_kernel == 1;
    const int fwpc = full2 ? full_warps_per_cta() : wpc;
    const int focc = full2 ? st->full_occupancy : st->occupancy;
    if (!st->ev[0]) {
        for (auto& e : st->ev) AMTC_CUDA(cudaEventCreate(&e));
        for (auto& e : st->kev) AMTC_CUDA(cudaEventCreate(&e));
    }
    st->retried = 0;
    bool light_ran = false, full_ran = false;

    // Split mode: with few trees (fewer items than a quarter of the resident
    // warps) the strips of each tree run on different warps, pipelined through
    // per-strip progress counters (intra-tree parallelism: configs 1, 3, 5b).
    {
        const int S = N / 32 + 1;
        const int64_t warps_total = (int64_t)st->sm_count * st->occupancy * wpc;
        const int64_t nsp = n2 * S;
        bool want = (g_split_mode == 1 || (g_split_mode < 0 && n2 <= warps_total / 4)) && N >= 64 &&
                    nsp < ((int64_t)1 << 30);
        // every queued item light (sellers of puts / calls, put buyers: class 0)?
        // then the light kernel's split mode (prefetched hand-off, one level ahead)
        if (want && g_light_kernel == 1 && g_light_split && st->light2_occupancy > 0) {
            int h1 = -1;
            AMTC_CUDA(cudaMemcpyAsync(&h1, small + SM_HIST + 1, sizeof(int), cudaMemcpyDeviceToHost, s));
            AMTC_CUDA(cudaStreamSynchronize(s));
            const size_t lcarry = light2_split_carry_bytes(N);
            const size_t lneed = (size_t)nsp * (lcarry + sizeof(int));
            if (h1 == 0 && lneed <= budget / 2) {
                const size_t wsl = light2_ws_bytes_per_warp(N);
                const int lw = light2_warps_per_cta();
                // every CTA slot of the device, not just enough for the items: strips are
                // claimed first-come, so they spread over all SMs (a strip pipeline is
                // latency bound; packing 8 strips per SM triples the per-level time)
                int64_t ctas = (int64_t)st->sm_count * st->light2_occupancy;
                ctas = std::min<int64_t>(ctas, (int64_t)((budget - lneed) / (wsl * lw)));
                if (ctas >= 1) {
                    AMTC_CUDA(st->ws_light.ensure(wsl * lw * (size_t)ctas));
                    AMTC_CUDA(st->items[1].ensure(sizeof(int) * (size_t)std::max<int64_t>(n2, nsp)));
                    AMTC_CUDA(st->sp_items.ensure(sizeof(int) * (size_t)nsp));
                    AMTC_CUDA(st->sp_progress.ensure(sizeof(int) * (size_t)nsp));
                    AMTC_CUDA(st->sp_carry.ensure(lcarry * (size_t)nsp));
                    AMTC_CUDA(cudaMemsetAsync(st->sp_progress.p, 0x7f, sizeof(int) * (size_t)nsp, s));
                    tc_launch_split_expand(q_items, q_count, S, nsp, static_cast<int*>(st->sp_items.p),
                                           small + SM_SPLITN, s);
                    AMTC_CUDA(cudaMemsetAsync(small + SM_WORK, 0, sizeof(int), s));
                    AMTC_CUDA(cudaMemsetAsync(small + SM_OVF0, 0, sizeof(int), s));
                    AMTC_CUDA(cudaEventRecord(st->ev[0], s));
                    AMTC_CUDA(cudaEventRecord(st->kev[2], s));
                    StripLaunchArgs A;
                    A.in = in;
                    A.N = N;
                    A.out = out;
                    A.items = static_cast<int*>(st->sp_items.p);
                    A.n_items = small + SM_SPLITN;
                    A.work_counter = small + SM_WORK;
                    A.ovf_items = static_cast<int*>(st->items[1].p);
                    A.ovf_count = small + SM_OVF0;
                    A.vertex_sum = reinterpret_cast<unsigned long long*>(small + SM_VSUM);
                    A.ws = static_cast<char*>(st->ws_light.p);
                    A.ws_stride = wsl;
                    A.level = 0;
                    A.ctas = (int)ctas;
                    A.split_S = S;
                    A.progress = static_cast<int*>(st->sp_progress.p);
                    A.carry = static_cast<char*>(st->sp_carry.p);
                    A.carry_stride = lcarry;
                    A.hedge = d_hedge;
                    if (light2_launch(A, s) != STATUS_OK) return cuda_fail(cudaGetLastError(), "light_kernel launch");
                    AMTC_CUDA(cudaEventRecord(st->kev[3], s));
                    AMTC_CUDA(cudaEventRecord(st->ev[1], s));
                    passes = 1;
                    light_ran = true;
                    AMTC_CUDA(cudaMemcpyAsync(&ovf_host, small + SM_OVF0, sizeof(int), cudaMemcpyDeviceToHost, s));
                    AMTC_CUDA(cudaStreamSynchronize(s));
                    if (ovf_host == 0) goto finish;
                    // a strip outgrew the light kernel: redo every tree on the general split / whole-tree path
                    st->retried = ovf_host;
                    tc_launch_prepare(in, n, N, out, static_cast<unsigned char*>(st->cls.p), small + SM_HIST,
                                      static_cast<int*>(st->items[0].p), s);
                    AMTC_CUDA(cudaMemsetAsync(small + SM_VSUM, 0, sizeof(unsigned long long), s));
                    ovf_host = 0;
                    passes = 0;
                    light_ran = false;
                }
            }
        }
        const size_t carry_b = strip_carry_bytes(N);
        const int acap = strip_split_arena_cap(N);
        const size_t need_b = (size_t)nsp * (carry_b + 2 * sizeof(int)) + (size_t)n2 * acap * strip_vtx_bytes();
        if (want && need_b > budget / 2) want = false;
        if (want) {
            const size_t wsb = strip_ws_bytes_per_warp_split(N);
            const int swpc = strip_split_warps_per_cta();
            // every SM (one split-kernel CTA each): strips are claimed first-come,
            // so they spread over all SMs (a strip pipeline is latency bound)
            int64_t ctas = std::min<int64_t>((int64_t)st->sm_count, nsp);
            ctas = std::min<int64_t>(ctas, (int64_t)((budget - need_b) / (wsb * swpc)));
            if (ctas < 1) want = false;
            if (want) {
                AMTC_CUDA(st->ws.ensure(wsb * swpc * (size_t)ctas));
                // every failing strip item (up to S per tree) appends its code
                AMTC_CUDA(st->items[1].ensure(sizeof(int) * (size_t)std::max<int64_t>(n2, nsp)));
                AMTC_CUDA(st->sp_items.ensure(sizeof(int) * (size_t)nsp));
                AMTC_CUDA(st->sp_progress.ensure(sizeof(int) * (size_t)nsp));
                AMTC_CUDA(st->sp_carry.ensure(carry_b * (size_t)nsp));
                AMTC_CUDA(st->sp_arena.ensure((size_t)n2 * acap * strip_vtx_bytes()));
                AMTC_CUDA(st->sp_cnt.ensure(sizeof(int) * (size_t)n2));
                AMTC_CUDA(cudaMemsetAsync(st->sp_progress.p, 0x7f, sizeof(int) * (size_t)nsp, s));
                AMTC_CUDA(cudaMemsetAsync(st->sp_cnt.p, 0, sizeof(int) * (size_t)n2, s));
                tc_launch_split_expand(q_items, q_count, S, nsp, static_cast<int*>(st->sp_items.p), small + SM_SPLITN,
                                       s);
                AMTC_CUDA(cudaMemsetAsync(small + SM_WORK, 0, sizeof(int), s));
                AMTC_CUDA(cudaMemsetAsync(small + SM_OVF0, 0, sizeof(int), s));
                AMTC_CUDA(cudaEventRecord(st->ev[0], s));
                StripLaunchArgs A;
                A.in = in;
                A.N = N;
                A.out = out;
                A.items = static_cast<int*>(st->sp_items.p);
                A.n_items = small + SM_SPLITN;
                A.work_counter = small + SM_WORK;
                A.ovf_items = static_cast<int*>(st->items[1].p);
                A.ovf_count = small + SM_OVF0;
                A.vertex_sum = reinterpret_cast<unsigned long long*>(small + SM_VSUM);
                A.ws = static_cast<char*>(st->ws.p);
                A.ws_stride = wsb;
                A.level = 0;
                A.ctas = (int)ctas;
                A.split_S = S;
                A.progress = static_cast<int*>(st->sp_progress.p);
                A.carry = static_cast<char*>(st->sp_carry.p);
                A.carry_stride = carry_b;
                A.carena_split = st->sp_arena.p;
                A.carena_cnt = static_cast<int*>(st->sp_cnt.p);
                A.carena_split_cap = acap;
                A.hedge = d_hedge;
                if (strip_launch(A, s) != STATUS_OK) return cuda_fail(cudaGetLastError(), "strip_kernel launch");
                AMTC_CUDA(cudaEventRecord(st->ev[1], s));
                passes = 1;
                AMTC_CUDA(cudaMemcpyAsync(&ovf_host, small + SM_OVF0, sizeof(int), cudaMemcpyDeviceToHost, s));
                AMTC_CUDA(cudaStreamSynchronize(s));
                if (ovf_host > 0) {
                    // a strip outgrew the split-mode capacities: redo every tree in whole-tree mode
                    st->retried = ovf_host;
                    tc_launch_prepare(in, n, N, out, static_cast<unsigned char*>(st->cls.p), small + SM_HIST,
                                      static_cast<int*>(st->items[0].p), s);
                    AMTC_CUDA(cudaMemsetAsync(small + SM_VSUM, 0, sizeof(unsigned long long), s));
                    ovf_host = 0;
                } else {
                    goto finish;
                }
            }
        }
    }
    for (int level = 0; level <= kMaxLevel; ++level) {
        const int wpc = fwpc;
        const size_t wsb = full2 ? full_ws_bytes_per_warp(N, level) : strip_ws_bytes_per_warp(N, level);
        int64_t ctas = (int64_t)st->sm_count * focc;
        ctas = std::min<int64_t>(ctas, (queued + wpc - 1) / wpc);
        ctas = std::min<int64_t>(ctas, (int64_t)(budget / (wsb * wpc)));
        if (ctas < 1) {
            // the cached budget may predate memory freed since: query again once
            if (int rc = refresh_budget()) return rc;
            budget = st->budget;
            ctas = std::min<int64_t>((int64_t)st->sm_count * focc, (queued + wpc - 1) / wpc);
            ctas = std::min<int64_t>(ctas, (int64_t)(budget / (wsb * wpc)));
        }
        if (ctas < 1) {
            // not even one CTA's workspace fits: every still-queued item fails
            // with ECAPACITY (prices stay NaN), never a silent STATUS_OK
            if (level == 0) tc_launch_mark_all_capacity(out, n, s);
            else ovf_host = (int)queued;
            break;
        }
        AMTC_CUDA(st->ws.ensure(wsb * wpc * (size_t)ctas));
        int* ovf_count = small + (passes % 2 == 0 ? SM_OVF0 : SM_OVF1);
        int* ovf_items = static_cast<int*>(st->items[(passes + 1) % 2].p);
        if (q_items == ovf_items) ovf_items = static_cast<int*>(st->items[passes % 2].p);
        AMTC_CUDA(cudaMemsetAsync(small + SM_WORK, 0, sizeof(int), s));
        AMTC_CUDA(cudaMemsetAsync(ovf_count, 0, sizeof(int), s));
        AMTC_CUDA(cudaEventRecord(st->ev[2 * passes], s));
        const bool light2 = g_light_kernel == 1;
        bool light_pass = level == 0 && g_light_kernel &&
                          (light2 ? st->light2_occupancy : st->light_occupancy) > 0;
        StripLaunchArgs AL;
        if (light_pass) {
            // class-0 items (sellers, put buyers: items [hist[1], total) of the
            // heavy-first queue) run on the light kernel, on a second stream, so
            // its CTAs take over the SMs the full kernel's CTAs release
            const size_t wsl = light2 ? light2_ws_bytes_per_warp(N) : strip_ws_bytes_per_warp_light(N);
            const int lw = light2 ? light2_warps_per_cta() : strip_light_warps_per_cta();
            int64_t lctas = (int64_t)st->sm_count * (light2 ? st->light2_occupancy : st->light_occupancy);
            lctas = std::min<int64_t>(lctas, (queued + lw - 1) / lw);
            const size_t full_b = wsb * wpc * (size_t)ctas;
            lctas = std::min<int64_t>(lctas, (int64_t)((budget > full_b ? budget - full_b : 0) / (wsl * lw)));
            if (lctas < 1) {
                light_pass = false;
            } else {
                AMTC_CUDA(st->ws_light.ensure(wsl * lw * (size_t)lctas));
                if (!st->s2) AMTC_CUDA(cudaStreamCreateWithFlags(&st->s2, cudaStreamNonBlocking));
                if (!st->ev_fork) {
                    AMTC_CUDA(cudaEventCreateWithFlags(&st->ev_fork, cudaEventDisableTiming));
                    AMTC_CUDA(cudaEventCreateWithFlags(&st->ev_join, cudaEventDisableTiming));
                }
                AMTC_CUDA(cudaMemsetAsync(small + SM_WORK2, 0, sizeof(int), s));
                AL.in = in;
                AL.N = N;
                AL.out = out;
                AL.items = q_items;
                AL.item_lo = small + SM_HIST + 1;
                AL.n_items = q_count;
                AL.work_counter = small + SM_WORK2;
                AL.ovf_items = ovf_items;
                AL.ovf_count = ovf_count;
                AL.vertex_sum = reinterpret_cast<unsigned long long*>(small + SM_VSUM);
                AL.ws = static_cast<char*>(st->ws_light.p);
                AL.ws_stride = wsl;
                AL.level = 0;
                AL.ctas = (int)lctas;
                AL.light = true;
                AL.hedge = d_hedge;
            }
        }
        StripLaunchArgs A;
        A.in = in;
        A.N = N;
        A.out = out;
        A.items = q_items;
        A.n_items = light_pass ? small + SM_HIST + 1 : q_count;  // the light pass took class 0
        A.work_counter = small + SM_WORK;
        A.ovf_items = ovf_items;
        A.ovf_count = ovf_count;
        A.vertex_sum = reinterpret_cast<unsigned long long*>(small + SM_VSUM);
        A.ws = static_cast<char*>(st->ws.p);
        A.ws_stride = wsb;
        A.level = level;
        A.ctas = (int)ctas;
        A.hedge = d_hedge;
        if (light_pass) AMTC_CUDA(cudaEventRecord(st->ev_fork, s));
        if (level == 0) AMTC_CUDA(cudaEventRecord(st->kev[0], s));
        if ((full2 ? full_launch(A, s) : strip_launch(A, s)) != STATUS_OK)
            return cuda_fail(cudaGetLastError(), "full solver launch");
        if (level == 0) {
            AMTC_CUDA(cudaEventRecord(st->kev[1], s));
            full_ran = true;
            light_ran = light_pass;
        }
        if (light_pass) {
            AMTC_CUDA(cudaStreamWaitEvent(st->s2, st->ev_fork, 0));
            AMTC_CUDA(cudaEventRecord(st->kev[2], st->s2));
            if ((light2 ? light2_launch(AL, st->s2) : strip_launch(AL, st->s2)) != STATUS_OK)
                return cuda_fail(cudaGetLastError(), "light kernel launch");
            AMTC_CUDA(cudaEventRecord(st->kev[3], st->s2));
            AMTC_CUDA(cudaEventRecord(st->ev_join, st->s2));
            AMTC_CUDA(cudaStreamWaitEvent(s, st->ev_join, 0));
        }
        AMTC_CUDA(cudaEventRecord(st->ev[2 * passes + 1], s));
        passes++;
        AMTC_CUDA(cudaMemcpyAsync(&ovf_host, ovf_count, sizeof(int), cudaMemcpyDeviceToHost, s));
        AMTC_CUDA(cudaStreamSynchronize(s));
        if (level == 0) st->retried += ovf_host;
        if (ovf_host == 0) break;
        q_items = ovf_items;
        q_count = ovf_count;
        queued = ovf_host;
        if (passes >= 8) break;  // event slots
    }
    if (ovf_host > 0) tc_launch_mark_capacity(q_items, ovf_host, out, s);
finish:
    launch_status_reduce(out, n, small + SM_WORST, s);
    int worst = 0;
    unsigned long long vs = 0;
    AMTC_CUDA(cudaMemcpyAsync(&worst, small + SM_WORST, sizeof(int), cudaMemcpyDeviceToHost, s));
    AMTC_CUDA(cudaMemcpyAsync(&vs, small + SM_VSUM, sizeof(vs), cudaMemcpyDeviceToHost, s));
    AMTC_CUDA(cudaStreamSynchronize(s));
    AMTC_CUDA(cudaGetLastError());
    st->vertex_sum = vs;
    st->passes = passes;
    st->solve_ms = 0.0;
    st->full_ms = st->light_ms = 0.0;
    if (full_ran) {
        float ms = 0.f;
        AMTC_CUDA(cudaEventElapsedTime(&ms, st->kev[0], st->kev[1]));
        st->full_ms = ms;
    }
    if (light_ran) {
        float ms = 0.f;
        AMTC_CUDA(cudaEventElapsedTime(&ms, st->kev[2], st->kev[3]));
        st->light_ms = ms;
    }
    for (int p = 0; p < passes; ++p) {
        float ms = 0.f;
        AMTC_CUDA(cudaEventElapsedTime(&ms, st->ev[2 * p], st->ev[2 * p + 1]));
        st->solve_ms += ms;
    }
    return worst;
}

// ---------------------------------------------------------------------------
// One transaction-cost tree sharded over the GPUs of an NCCL communicator
// (SURVEY 8(e), config 5b).  The tree's strips (split mode) are partitioned
// into contiguous ranges of equal work (strip s has N - 32 s + 1 levels); rank
// g owns [lo_g, hi_g), rank 0 the root strip.  The only cross-GPU dependency is
// the carry column of strip hi_g (the first strip of rank g+1), read by rank
// g's strip hi_g - 1 at every level: rank g maps rank g+1's carry, carry-arena
// and progress buffers through CUDA IPC (handles all-gathered over NCCL) and
// its kernel reads them over NVLink, waiting on the peer's progress counter,
// which the producer publishes with system-scope fences.  NCCL collectives
// before and after the launch order the buffer resets and the reuse.
// ---------------------------------------------------------------------------
static int nccl_fail(ncclResult_t r, const char* what) {
    g_last_error = std::string(what) + ": " + ncclGetErrorString(r);
    return STATUS_ENCCL;
}
#define AMTC_NCCL(call)                                   \
    do {                                                  \
        ncclResult_t r_ = (call);                         \
        if (r_ != ncclSuccess) return nccl_fail(r_, #call); \
    } while (0)

// strip ranges of equal work: strip s carries N - 32 s + 1 levels
static void shard_strips(int N, int nranks, std::vector<int>& lo) {
    const int S = N / 32 + 1;
    std::vector<double> cum(S + 1, 0.0);
    for (int s = 0; s < S; ++s) cum[s + 1] = cum[s] + (double)(N - 32 * s + 1);
    lo.assign(nranks + 1, S);
    lo[0] = 0;
    int s = 0;
    for (int g = 1; g < nranks; ++g) {
        const double target = cum[S] * g / nranks;
        while (s < S && cum[s] < target) ++s;
        lo[g] = std::max(s, lo[g - 1]);
    }
    lo[nranks] = S;
}

static size_t soa_bytes(int64_t n);
static int stage_in(DevState* st, const amtc_batch_soa* h, int64_t n, amtc_batch_soa* d, cudaStream_t s);

int tc_tree_sharded(const void* params_v, int N, const void* payoff_v, double k, void* comm_v, int rank, int nranks,
                    void* out_v, cudaStream_t s) {
    const amtc_params* p = static_cast<const amtc_params*>(params_v);
    const amtc_payoff* y = static_cast<const amtc_payoff*>(payoff_v);
    amtc_quote* out = static_cast<amtc_quote*>(out_v);
    ncclComm_t comm = static_cast<ncclComm_t>(comm_v);
    if (N < 64) return STATUS_EINVAL;  // fewer than three strips: nothing to shard
    int dev = 0;
    AMTC_CUDA(cudaGetDevice(&dev));
    DevState* st = state_for_device(dev);
    // one option, host -> device
    double S0 = p->S0, K = y->K, K2 = y->K2, T = p->T, sg = p->sigma, R = p->R, kk = k;
    int32_t kind = y->kind;
    uint32_t fl = y->flags;
    amtc_batch_soa h;
    h.S0 = &S0; h.K = &K; h.K2 = &K2; h.T = &T; h.sigma = &sg; h.R = &R; h.k = &kk; h.kind = &kind;
    h.flags = &fl;
    std::lock_guard<std::mutex> guard(st->mu);
    if (!st->sm_count) {
        AMTC_CUDA(cudaDeviceGetAttribute(&st->sm_count, cudaDevAttrMultiProcessorCount, dev));
        st->occupancy = strip_ctas_per_sm();
        st->light_occupancy = strip_light_ctas_per_sm();
    }
    amtc_batch_soa d;
    int rc = stage_in(st, &h, 1, &d, s);
    if (rc) return rc;
    BatchPtrs in = to_ptrs(&d);
    AMTC_CUDA(st->stage_out.ensure(sizeof(amtc_quote)));
    Quote* dq = static_cast<Quote*>(st->stage_out.p);
    AMTC_CUDA(st->items[0].ensure(sizeof(int) * 2));
    AMTC_CUDA(st->cls.ensure(2));
    AMTC_CUDA(st->small.ensure(sizeof(int) * SM_INTS));
    int* small = static_cast<int*>(st->small.p);
    tc_launch_prepare(in, 1, N, dq, static_cast<unsigned char*>(st->cls.p), small + SM_HIST,
                      static_cast<int*>(st->items[0].p), s);
    AMTC_CUDA(cudaMemsetAsync(small + SM_VSUM, 0, sizeof(unsigned long long), s));
    AMTC_CUDA(cudaMemsetAsync(small + SM_OVF0, 0, sizeof(int), s));  // also on a rank without strips
    // split-mode buffers for both trees (seller, buyer) over ALL strips (IPC-mapped by rank-1)
    const int S = N / 32 + 1;
    const int64_t nsp = 2 * (int64_t)S;
    const size_t carry_b = strip_carry_bytes(N);
    const int acap = strip_split_arena_cap(N);
    AMTC_CUDA(st->sp_items.ensure(sizeof(int) * (size_t)nsp));
    AMTC_CUDA(st->sp_progress.ensure(sizeof(int) * (size_t)nsp));
    AMTC_CUDA(st->sp_carry.ensure(carry_b * (size_t)nsp));
    AMTC_CUDA(st->sp_arena.ensure((size_t)2 * acap * strip_vtx_bytes()));
    AMTC_CUDA(st->sp_cnt.ensure(sizeof(int) * 2));
    AMTC_CUDA(cudaMemsetAsync(st->sp_progress.p, 0x7f, sizeof(int) * (size_t)nsp, s));
    AMTC_CUDA(cudaMemsetAsync(st->sp_cnt.p, 0, sizeof(int) * 2, s));
    std::vector<int> lo;
    shard_strips(N, nranks, lo);
    const int s_lo = lo[rank], s_hi = lo[rank + 1];
    // exchange IPC handles of (carry, arena, progress); map rank+1's
    char* peer_carry = nullptr;
    void* peer_arena = nullptr;
    int* peer_prog = nullptr;
    if (nranks > 1) {
        cudaIpcMemHandle_t mine[3];
        AMTC_CUDA(cudaIpcGetMemHandle(&mine[0], st->sp_carry.p));
        AMTC_CUDA(cudaIpcGetMemHandle(&mine[1], st->sp_arena.p));
        AMTC_CUDA(cudaIpcGetMemHandle(&mine[2], st->sp_progress.p));
        const size_t hb = sizeof(mine);
        AMTC_CUDA(st->ipc.ensure(hb * (size_t)(nranks + 1)));
        char* dh = static_cast<char*>(st->ipc.p);
        AMTC_CUDA(cudaMemcpyAsync(dh + hb * nranks, mine, hb, cudaMemcpyHostToDevice, s));
        AMTC_NCCL(ncclAllGather(dh + hb * nranks, dh, hb, ncclUint8, comm, s));
        std::vector<char> all(hb * nranks);
        AMTC_CUDA(cudaMemcpyAsync(all.data(), dh, hb * nranks, cudaMemcpyDeviceToHost, s));
        AMTC_CUDA(cudaStreamSynchronize(s));
        if (rank + 1 < nranks) {
            cudaIpcMemHandle_t peer[3];
            std::memcpy(peer, all.data() + hb * (rank + 1), hb);
            void* pc = nullptr;
            void* pa = nullptr;
            void* pp = nullptr;
            AMTC_CUDA(cudaIpcOpenMemHandle(&pc, peer[0], cudaIpcMemLazyEnablePeerAccess));
            AMTC_CUDA(cudaIpcOpenMemHandle(&pa, peer[1], cudaIpcMemLazyEnablePeerAccess));
            AMTC_CUDA(cudaIpcOpenMemHandle(&pp, peer[2], cudaIpcMemLazyEnablePeerAccess));
            peer_carry = static_cast<char*>(pc);
            peer_arena = pa;
            peer_prog = static_cast<int*>(pp);
        }
        // every rank's progress reset is done before any kernel reads a peer's
        AMTC_NCCL(ncclAllReduce(small + SM_WORK2, small + SM_WORK2, 1, ncclInt32, ncclSum, comm, s));
    }
    // this rank's strip items, right to left
    tc_launch_split_expand(static_cast<int*>(st->items[0].p), small + SM_HIST + TC_CLASSES, S, nsp,
                           static_cast<int*>(st->sp_items.p), small + SM_SPLITN, s, s_lo, s_hi);
    const size_t wsb = strip_ws_bytes_per_warp_split(N);
    const int wpc = strip_split_warps_per_cta();
    const int64_t ctas = std::min<int64_t>((int64_t)st->sm_count, 2 * (int64_t)(s_hi - s_lo));
    int ovf = 0;
    if (ctas >= 1 && s_hi > s_lo) {
        AMTC_CUDA(st->ws.ensure(wsb * wpc * (size_t)ctas));
        AMTC_CUDA(cudaMemsetAsync(small + SM_WORK, 0, sizeof(int), s));
        AMTC_CUDA(cudaMemsetAsync(small + SM_OVF0, 0, sizeof(int), s));
        StripLaunchArgs A;
        A.in = in;
        A.N = N;
        A.out = dq;
        A.items = static_cast<int*>(st->sp_items.p);
        A.n_items = small + SM_SPLITN;
        A.work_counter = small + SM_WORK;
        A.ovf_items = static_cast<int*>(st->items[1].p);
        AMTC_CUDA(st->items[1].ensure(sizeof(int) * (size_t)nsp));
        A.ovf_items = static_cast<int*>(st->items[1].p);
        A.ovf_count = small + SM_OVF0;
        A.vertex_sum = reinterpret_cast<unsigned long long*>(small + SM_VSUM);
        A.ws = static_cast<char*>(st->ws.p);
        A.ws_stride = wsb;
        A.level = 0;
        A.ctas = (int)ctas;
        A.split_S = S;
        A.progress = static_cast<int*>(st->sp_progress.p);
        A.carry = static_cast<char*>(st->sp_carry.p);
        A.carry_stride = carry_b;
        A.carena_split = st->sp_arena.p;
        A.carena_cnt = static_cast<int*>(st->sp_cnt.p);
        A.carena_split_cap = acap;
        A.peer_strip = (rank + 1 < nranks) ? s_hi : -1;
        A.sys_fence = nranks > 1 ? 1 : 0;
        A.peer_carry = peer_carry;
        A.peer_carena = peer_arena;
        A.peer_progress = peer_prog;
        if (strip_launch(A, s) != STATUS_OK) return cuda_fail(cudaGetLastError(), "strip_kernel launch");
        AMTC_CUDA(cudaMemcpyAsync(&ovf, small + SM_OVF0, sizeof(int), cudaMemcpyDeviceToHost, s));
    }
    // rank 0 holds the quote (root strip); share it -- also the barrier before any
    // rank reuses buffers a peer may still read
    if (nranks > 1) {
        // barrier: no rank returns (and may reset or reallocate the buffers its
        // left neighbour reads through IPC) before every rank's kernel is done --
        // an all-reduce needs every rank's contribution, a broadcast does not
        AMTC_NCCL(ncclAllReduce(small + SM_WORK2, small + SM_WORK2, 1, ncclInt32, ncclSum, comm, s));
        AMTC_NCCL(ncclBroadcast(dq, dq, sizeof(Quote), ncclUint8, 0, comm, s));
        AMTC_NCCL(ncclAllReduce(small + SM_OVF0, small + SM_OVF1, 1, ncclInt32, ncclMax, comm, s));
        AMTC_CUDA(cudaMemcpyAsync(&ovf, small + SM_OVF1, sizeof(int), cudaMemcpyDeviceToHost, s));
    }
    launch_status_reduce(dq, 1, small + SM_WORST, s);
    AMTC_CUDA(cudaMemcpyAsync(out, dq, sizeof(amtc_quote), cudaMemcpyDeviceToHost, s));
    AMTC_CUDA(cudaStreamSynchronize(s));
    if (ovf > 0 && (out->status == 0 || out->status == STATUS_ECAPACITY)) {
        // a strip of this tree (on any rank) outgrew its capacities: no price
        out->status = STATUS_ECAPACITY;
        out->ask = out->bid = NAN;
    }
    if (peer_carry) {
        cudaIpcCloseMemHandle(peer_carry);
        cudaIpcCloseMemHandle(peer_arena);
        cudaIpcCloseMemHandle(peer_prog);
    }
    AMTC_CUDA(cudaGetLastError());
    return out->status;
}

// host-pointer variants: stage through device buffers
static size_t soa_bytes(int64_t n) { return (size_t)n * (7 * sizeof(double) + 2 * sizeof(int32_t)); }

static int stage_in(DevState* st, const amtc_batch_soa* h, int64_t n, amtc_batch_soa* d, cudaStream_t s) {
    cudaError_t e = st->stage_in.ensure(soa_bytes(n) + 64);
    if (e != cudaSuccess) return cuda_fail(e, "stage_in");
    char* base = static_cast<char*>(st->stage_in.p);
    double* f = reinterpret_cast<double*>(base);
    const double* src[7] = {h->S0, h->K, h->K2, h->T, h->sigma, h->R, h->k};
    const double** dst[7] = {&d->S0, &d->K, &d->K2, &d->T, &d->sigma, &d->R, &d->k};
    if (soa_bytes(n) <= ((size_t)1 << 20)) {
        // small batch (e.g. the north-star single option): pack into pinned
        // memory and copy once
        const size_t need = soa_bytes(n);
        if (st->h_stage_bytes < need) {
            if (st->h_stage) cudaFreeHost(st->h_stage);
            st->h_stage = nullptr;
            st->h_stage_bytes = 0;
            AMTC_CUDA(cudaMallocHost(&st->h_stage, (size_t)1 << 20));
            st->h_stage_bytes = (size_t)1 << 20;
        }
        double* hf = static_cast<double*>(st->h_stage);
        for (int a = 0; a < 7; ++a) {
            if (src[a]) std::memcpy(hf + a * n, src[a], sizeof(double) * n);
            *dst[a] = src[a] ? f + a * n : nullptr;
        }
        std::memcpy(reinterpret_cast<int32_t*>(hf + 7 * n), h->kind, sizeof(int32_t) * n);
        if (h->flags) std::memcpy(reinterpret_cast<uint32_t*>(hf + 7 * n) + n, h->flags, sizeof(uint32_t) * n);
        AMTC_CUDA(cudaMemcpyAsync(f, hf, need, cudaMemcpyHostToDevice, s));
        AMTC_CUDA(cudaStreamSynchronize(s));  // the pinned buffer is reused by the next call
        d->kind = reinterpret_cast<int32_t*>(f + 7 * n);
        d->flags = h->flags ? reinterpret_cast<uint32_t*>(f + 7 * n) + n : nullptr;
        return STATUS_OK;
    }
    for (int a = 0; a < 7; ++a) {
        if (src[a]) {
            AMTC_CUDA(cudaMemcpyAsync(f + a * n, src[a], sizeof(double) * n, cudaMemcpyHostToDevice, s));
            *dst[a] = f + a * n;
        } else {
            *dst[a] = nullptr;
        }
    }
    int32_t* kd = reinterpret_cast<int32_t*>(f + 7 * n);
    AMTC_CUDA(cudaMemcpyAsync(kd, h->kind, sizeof(int32_t) * n, cudaMemcpyHostToDevice, s));
    d->kind = kd;
    d->flags = nullptr;
    if (h->flags) {
        uint32_t* fd = reinterpret_cast<uint32_t*>(kd + n);
        AMTC_CUDA(cudaMemcpyAsync(fd, h->flags, sizeof(uint32_t) * n, cudaMemcpyHostToDevice, s));
        d->flags = fd;
    }
    return STATUS_OK;
}

}  // namespace amtc

using namespace amtc;

extern "C" {

int amtc_price_american_tc_batch(const amtc_batch_soa* d_in, int64_t n, int32_t N, amtc_quote* d_out,
                                 void* cuda_stream) {
    try {
        return tc_batch_device(d_in, n, N, d_out, static_cast<cudaStream_t>(cuda_stream));
    } catch (...) {
        g_last_error = "unexpected host exception";
        return STATUS_ECUDA;
    }
}

int amtc_price_american_tc_batch_host(const amtc_batch_soa* h_in, int64_t n, int32_t N, amtc_quote* h_out,
                                      void* cuda_stream) {
    try {
        if (!soa_ok(h_in) || !h_out || n < 0 || N < 1) return STATUS_EINVAL;
        if (n == 0) return STATUS_OK;
        cudaStream_t s = static_cast<cudaStream_t>(cuda_stream);
        int dev = 0;
        AMTC_CUDA(cudaGetDevice(&dev));
        DevState* st = state_for_device(dev);
        amtc_batch_soa d;
        {
            std::lock_guard<std::mutex> g(st->mu);
            int rc = stage_in(st, h_in, n, &d, s);
            if (rc) return rc;
            AMTC_CUDA(st->stage_out.ensure(sizeof(amtc_quote) * (size_t)n));
        }
        amtc_quote* d_out = static_cast<amtc_quote*>(st->stage_out.p);
        int rc = tc_batch_device(&d, n, N, d_out, s);
        if (rc == STATUS_ECUDA) return rc;
        AMTC_CUDA(cudaMemcpyAsync(h_out, d_out, sizeof(amtc_quote) * (size_t)n, cudaMemcpyDeviceToHost, s));
        AMTC_CUDA(cudaStreamSynchronize(s));
        return rc;
    } catch (...) {
        g_last_error = "unexpected host exception";
        return STATUS_ECUDA;
    }
}

amtc_quote amtc_price_american_tc(const amtc_params* params, int32_t N, const amtc_payoff* payoff, double k) {
    amtc_quote q;
    q.ask = NAN;
    q.bid = NAN;
    q.max_bp = 0;
    if (!params || !payoff) {
        q.status = STATUS_EINVAL;
        return q;
    }
    double S0 = params->S0, K = payoff->K, K2 = payoff->K2, T = params->T, sg = params->sigma, R = params->R;
    int32_t kind = payoff->kind;
    uint32_t fl = payoff->flags;
    amtc_batch_soa h;
    h.S0 = &S0; h.K = &K; h.K2 = &K2; h.T = &T; h.sigma = &sg; h.R = &R; h.k = &k; h.kind = &kind;
    h.flags = &fl;
    int rc = amtc_price_american_tc_batch_host(&h, 1, N, &q, nullptr);
    if (rc == STATUS_ECUDA || (rc == STATUS_EINVAL && N < 1)) q.status = rc;
    return q;
}

int amtc_price_american_tc_hedge(const amtc_params* params, int32_t N, const amtc_payoff* payoff, double k,
                                 amtc_quote* out, double* y_ask, double* y_bid) {
    try {
        if (!out || !y_ask || !y_bid) return STATUS_EINVAL;
        out->ask = out->bid = NAN;
        out->max_bp = 0;
        out->status = STATUS_EINVAL;
        *y_ask = *y_bid = NAN;
        if (!params || !payoff) return STATUS_EINVAL;
        double S0 = params->S0, K = payoff->K, K2 = payoff->K2, T = params->T, sg = params->sigma, R = params->R;
        double kk = k;
        int32_t kind = payoff->kind;
        uint32_t fl = payoff->flags;
        amtc_batch_soa h;
        h.S0 = &S0; h.K = &K; h.K2 = &K2; h.T = &T; h.sigma = &sg; h.R = &R; h.k = &kk; h.kind = &kind;
        h.flags = &fl;
        cudaStream_t s = nullptr;
        int dev = 0;
        AMTC_CUDA(cudaGetDevice(&dev));
        DevState* st = state_for_device(dev);
        amtc_batch_soa d;
        {
            std::lock_guard<std::mutex> g(st->mu);
            int rc = stage_in(st, &h, 1, &d, s);
            if (rc) return rc;
            AMTC_CUDA(st->stage_out.ensure(sizeof(amtc_quote) + 4 * sizeof(double)));
        }
        amtc_quote* d_out = static_cast<amtc_quote*>(st->stage_out.p);
        double* d_hedge = reinterpret_cast<double*>(static_cast<char*>(st->stage_out.p) + 32);
        AMTC_CUDA(cudaMemsetAsync(d_hedge, 0xff, 2 * sizeof(double), s));  // NaN unless written
        int rc = tc_batch_device(&d, 1, N, d_out, s, d_hedge);
        if (rc == STATUS_ECUDA) return rc;
        double hy[2];
        AMTC_CUDA(cudaMemcpyAsync(out, d_out, sizeof(amtc_quote), cudaMemcpyDeviceToHost, s));
        AMTC_CUDA(cudaMemcpyAsync(hy, d_hedge, sizeof(hy), cudaMemcpyDeviceToHost, s));
        AMTC_CUDA(cudaStreamSynchronize(s));
        *y_ask = out->status ? NAN : hy[0];
        *y_bid = out->status ? NAN : hy[1];
        return out->status;
    } catch (...) {
        g_last_error = "unexpected host exception";
        return STATUS_ECUDA;
    }
}

// caller holds st->mu (the strip path's carry workspace lives in st->crr_ws)
static int crr_batch_locked(DevState* st, const amtc_batch_soa* d_in, int64_t n, int32_t N, double* d_price,
                            cudaStream_t s) {
    if (N <= crr_max_n()) return crr_launch(to_ptrs(d_in), n, N, d_price, s);
    const int64_t warps = crr_strip_warps(n);
    const cudaError_t e = st->crr_ws.ensure(crr_strip_ws_bytes(N, warps));
    if (e != cudaSuccess) return cuda_fail(e, "CRR strip workspace");
    return crr_strip_launch(to_ptrs(d_in), n, N, d_price, static_cast<double*>(st->crr_ws.p), warps, s);
}

int amtc_price_crr_batch(const amtc_batch_soa* d_in, int64_t n, int32_t N, double* d_price, void* cuda_stream) {
    try {
        if (!soa_ok(d_in) || !d_price || n < 0 || N < 1) return STATUS_EINVAL;
        if (n == 0) return STATUS_OK;
        int dev = 0;
        AMTC_CUDA(cudaGetDevice(&dev));
        DevState* st = state_for_device(dev);
        std::lock_guard<std::mutex> g(st->mu);
        int rc = crr_batch_locked(st, d_in, n, N, d_price, static_cast<cudaStream_t>(cuda_stream));
        AMTC_CUDA(cudaGetLastError());
        return rc;
    } catch (...) {
        g_last_error = "unexpected host exception";
        return STATUS_ECUDA;
    }
}

int amtc_price_crr_batch_host(const amtc_batch_soa* h_in, int64_t n, int32_t N, double* h_price,
                              void* cuda_stream) {
    try {
        if (!soa_ok(h_in) || !h_price || n < 0 || N < 1) return STATUS_EINVAL;
        if (n == 0) return STATUS_OK;
        cudaStream_t s = static_cast<cudaStream_t>(cuda_stream);
        int dev = 0;
        AMTC_CUDA(cudaGetDevice(&dev));
        DevState* st = state_for_device(dev);
        std::lock_guard<std::mutex> g(st->mu);
        amtc_batch_soa d;
        int rc = stage_in(st, h_in, n, &d, s);
        if (rc) return rc;
        AMTC_CUDA(st->stage_out.ensure(sizeof(double) * (size_t)n));
        double* d_price = static_cast<double*>(st->stage_out.p);
        rc = crr_batch_locked(st, &d, n, N, d_price, s);
        if (!rc && cudaGetLastError() != cudaSuccess) rc = STATUS_ECUDA;
        if (rc) return rc;
        AMTC_CUDA(cudaMemcpyAsync(h_price, d_price, sizeof(double) * (size_t)n, cudaMemcpyDeviceToHost, s));
        AMTC_CUDA(cudaStreamSynchronize(s));
        return STATUS_OK;
    } catch (...) {
        g_last_error = "unexpected host exception";
        return STATUS_ECUDA;
    }
}

const char* amtc_strerror(int status) {
    switch (status) {
        case STATUS_OK: return "AMTC_OK";
        case STATUS_EINVAL: return "AMTC_EINVAL: invalid argument";
        case STATUS_EARBITRAGE: return "AMTC_EARBITRAGE: calibration violates d < r < u";
        case STATUS_ECAPACITY: return "AMTC_ECAPACITY: node function exceeded every scratch capacity";
        case STATUS_EUNBOUNDED: return "AMTC_EUNBOUNDED: slope restriction unbounded below";
        case STATUS_ECUDA: return "AMTC_ECUDA: CUDA runtime error";
        case STATUS_ENCCL: return "AMTC_ENCCL: NCCL error";
        default: return "AMTC: unknown status";
    }
}

const char* amtc_last_error(void) { return g_last_error.c_str(); }

int amtc_tree_shard_plan(int32_t N, int nranks, int32_t* lo) {
    if (N < 1 || nranks < 1 || !lo) return STATUS_EINVAL;
    std::vector<int> v;
    shard_strips(N, nranks, v);
    for (int g = 0; g <= nranks; ++g) lo[g] = v[g];
    return STATUS_OK;
}

int amtc_batch_shard_plan(const amtc_batch_soa* h_in, int64_t n, int32_t N, int nranks, int32_t* rank_of,
                          double* rank_cost) {
    try {
        if (!h_in || !h_in->T || !h_in->sigma || !h_in->kind || !rank_of || n < 0 || N < 1 || nranks < 1)
            return STATUS_EINVAL;
        const double nodes = 0.5 * ((double)N + 1.0) * ((double)N + 2.0);
        std::vector<double> cost((size_t)n);
        for (int64_t i = 0; i < n; ++i) {
            const double h = h_in->sigma[i] * std::sqrt(h_in->T[i] / (double)N);
            const double k = h_in->k ? h_in->k[i] : 0.0;
            const double kh = (h > 0.0 && std::isfinite(h) && k > 0.0) ? k / h : 0.0;
            cost[(size_t)i] = nodes * (2.0 + (h_in->kind[i] != AMTC_PUT ? AMTC_HEAVY_WEIGHT * kh : 0.0));
        }
        std::vector<int64_t> order((size_t)n);
        for (int64_t i = 0; i < n; ++i) order[(size_t)i] = i;
        std::stable_sort(order.begin(), order.end(),
                         [&](int64_t a, int64_t b) { return cost[(size_t)a] > cost[(size_t)b]; });
        if (rank_cost)
            for (int g = 0; g < nranks; ++g) rank_cost[g] = 0.0;
        for (int64_t q = 0; q < n; ++q) {
            const int64_t round = q / nranks, pos = q % nranks;
            const int g = (int)((round & 1) ? nranks - 1 - pos : pos);  // snake order
            rank_of[order[(size_t)q]] = g;
            if (rank_cost) rank_cost[g] += cost[(size_t)order[(size_t)q]];
        }
        return STATUS_OK;
    } catch (...) {
        g_last_error = "unexpected host exception";
        return STATUS_ECUDA;
    }
}

void amtc_debug_set_heavy_threshold(int tl) { strip_set_heavy_threshold(tl); }

void amtc_debug_set_split_mode(int mode) { g_split_mode = mode < 0 ? -1 : (mode ? 1 : 0); }

int amtc_debug_full_profile(uint64_t out[8], int reset) {
    // the full solver's counters (-DAMTC_F_PROF=1), else the light kernel's split-mode ones (-DAMTC_L2_PROF=1)
    const int rc = full_profile(reinterpret_cast<unsigned long long*>(out), reset);
    if (rc == STATUS_OK) return rc;
    return light_profile(reinterpret_cast<unsigned long long*>(out), reset);
}
void amtc_debug_set_full_kernel(int which) { g_full_kernel = (which == 0) ? 0 : 1; }

void amtc_debug_set_light_split(int on) { g_light_split = on ? 1 : 0; }
void amtc_debug_set_light_kernel(int on) { g_light_kernel = (on >= 0 && on <= 2) ? on : 1; }

void amtc_debug_set_arena_shift(int shift) { strip_set_arena_shift(shift); }

int64_t amtc_launch_count(void) { return g_launches.load(); }

int amtc_tc_last_stats(amtc_tc_stats* out) {
    if (!out) return STATUS_EINVAL;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return STATUS_ECUDA;
    DevState* st = state_for_device(dev);
    std::lock_guard<std::mutex> g(st->mu);
    out->vertex_sum = (int64_t)st->vertex_sum;
    out->passes = st->passes;
    out->retried_items = st->retried;
    out->solve_ms = st->solve_ms;
    out->full_ms = st->full_ms;
    out->light_ms = st->light_ms;
    return STATUS_OK;
}

}  // extern "C"
