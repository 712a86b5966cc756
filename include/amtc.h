/*
 * amtc.h -- C-ABI of the B200-native American-option ask/bid pricer under
 * proportional transaction costs (Zhang, Roux & Zastawniak 2011).
 *
 * Citations: P:n = PAPER.md line n.
 *
 * All arithmetic is IEEE fp64 on the GPU (sm_100a).  Every pointer is owned by
 * the caller; the library keeps only lazily created per-device scratch
 * workspaces (guarded by a mutex) that it reuses across calls.  No C++
 * exception crosses this boundary.  Functions return an amtc_status (0 = OK);
 * per-option failures leave NaN prices and a non-zero per-option status.
 *
 * Model (Sec. 4.1): N steps, u = exp(sigma sqrt(T/N)), d = 1/u,
 * r = exp(R T / N); stock price S0 u^(t-j) d^j at node (t, j) (j = number of
 * down-moves); stock ask/bid (1+k)S, (1-k)S for t >= 1 and S0 at t = 0
 * (P:92); an extra time instant t = N+1 with payoff (0,0).
 */
#ifndef AMTC_H
#define AMTC_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* payoff kinds (the payoff process (xi, zeta) of P:94) */
typedef enum {
    AMTC_PUT = 0,        /* physical delivery: (xi, zeta) = (K, -1)  */
    AMTC_CALL = 1,       /* physical delivery: (-K, +1)            (reading R6)       */
    AMTC_BULL_SPREAD = 2 /* cash: ((S-K)^+ - (S-K2)^+, 0), K < K2 */
} amtc_kind;

/* payoff flags (amtc_payoff.flags, amtc_batch_soa.flags) */
enum {
    AMTC_EUROPEAN = 1u << 0,   /* no exercise before N: z_t = v_t for t < N (reading A21)  */
    AMTC_CASH = 1u << 1,       /* put / call settled in cash: ((K-S)^+, 0) / ((S-K)^+, 0)  */
    AMTC_COST_AT_T0 = 1u << 2  /* costs also at t = 0: quotes (1 +- k) S0 instead of S0
                                  (P:159's convention is the default); no root hedge     */
};

/* status codes (per option and per call; a call returns the worst status) */
typedef enum {
    AMTC_OK = 0,
    AMTC_EINVAL = 1,      /* S0, K, T, sigma <= 0; N < 1; k not in [0,1); bull with K >= K2;
                             unknown kind or flag bit; AMTC_CASH on a bull spread; null pointer */
    AMTC_EARBITRAGE = 2,  /* not d < r < u (risk-neutral p outside (0,1))                   */
    AMTC_ECAPACITY = 3,   /* a node function outgrew every scratch capacity tried           */
    AMTC_EUNBOUNDED = 4,  /* slope restriction infimum is -inf (impossible when d<r<u)      */
    AMTC_ECUDA = 5,       /* a CUDA runtime error (message: amtc_last_error())              */
    AMTC_ENCCL = 6
} amtc_status;

/* market and tenor of one option */
typedef struct {
    double S0;    /* spot price at t = 0, > 0                       */
    double T;     /* expiry in years, > 0                           */
    double sigma; /* volatility, > 0                                */
    double R;     /* continuously compounded annual interest rate   */
} amtc_params;

/* payoff of one option */
typedef struct {
    int32_t kind;   /* amtc_kind                                   */
    uint32_t flags; /* AMTC_EUROPEAN | AMTC_CASH | AMTC_COST_AT_T0 (0: American, physical) */
    double K;       /* strike (bull spread: the long strike K1)    */
    double K2;      /* bull spread: the short strike, > K; else 0  */
} amtc_payoff;

/* result for one option (24 bytes) */
typedef struct {
    double ask;      /* pi^a_0 = z_0(0) of the seller recursion  */
    double bid;      /* pi^b_0 = -z'_0(0) of the buyer recursion */
    int32_t status;  /* amtc_status of this option                               */
    int32_t max_bp;  /* largest vertex count of any node function (capacity audit) */
} amtc_quote;

/* Structure-of-arrays batch of n options.  For the *_batch calls every
   pointer is a DEVICE pointer (fp64 / int32 arrays of length n); for the
   *_batch_host calls every pointer is a HOST pointer. */
typedef struct {
    const double* S0;
    const double* K;
    const double* K2;     /* may be NULL when no option is a bull spread */
    const double* T;
    const double* sigma;
    const double* R;
    const double* k;      /* proportional transaction cost rate, in [0,1); may be NULL for CRR */
    const int32_t* kind;  /* amtc_kind */
    const uint32_t* flags; /* AMTC_EUROPEAN | AMTC_CASH | AMTC_COST_AT_T0 per option; may be NULL */
} amtc_batch_soa;

/*
 * North-star call: ask and bid of ONE American option under proportional
 * costs k on an N-step tree (Sec. 3 seller/buyer recursions).
 * Synchronous; runs on the current CUDA device.  On error the quote carries
 * NaN prices and the status.
 */
amtc_quote amtc_price_american_tc(const amtc_params* params, int32_t N, const amtc_payoff* payoff,
                                  double k);

/*
 * As amtc_price_american_tc, plus the root hedge: the
 * share position the seller (*y_ask) and the buyer (*y_bid) take at t = 0,
 * argmin_y [ w_0(y)/r + S0 y ] over the vertices of w_0 = max(z_{1,0}, z_{1,1})
 * (no costs at t = 0; derived A.4; smallest minimiser on ties).  At k = 0
 * it is the CRR delta (pi^u - pi^d)/(S0 (u - d)) and its negative (derived A.1).
 * out, y_ask, y_bid: HOST pointers; NaN on error.  Synchronous.  Returns the status.
 */
int amtc_price_american_tc_hedge(const amtc_params* params, int32_t N, const amtc_payoff* payoff, double k,
                                 amtc_quote* out, double* y_ask, double* y_bid);

/*
 * Batched ask/bid for n independent options on N-step trees (DEVICE pointers).
 * d_out: device array of n amtc_quote.  Work is enqueued on cuda_stream
 * (a cudaStream_t, NULL = legacy default stream); the call synchronises that
 * stream once at the end (to re-run any option whose node functions outgrew
 * the first scratch capacity), so d_out is complete on return.
 * Returns the worst per-option status, or AMTC_ECUDA.
 */
int amtc_price_american_tc_batch(const amtc_batch_soa* d_in, int64_t n, int32_t N, amtc_quote* d_out,
                                 void* cuda_stream);

/* As above with HOST pointers: copies inputs host->device and quotes
   device->host inside the call (h_out: host array of n amtc_quote). */
int amtc_price_american_tc_batch_host(const amtc_batch_soa* h_in, int64_t n, int32_t N,
                                      amtc_quote* h_out, void* cuda_stream);

/*
 * k = 0 (frictionless) batched CRR American prices (Appendix: no
 * extra level, scalar max(exercise, continuation)).  d_in->k and ->K2 are
 * ignored except for bull spreads (K2).  d_price: device array of n doubles.
 * Any N >= 1: N <= 1152 keeps one tree's level in a warp's registers; larger N
 * (Table III's N = 5,000-40,000 trees) sweeps each tree in
 * 512-column strips with a carry buffer of 2 (N + 2) doubles per resident
 * warp, owned by the library (grow-only, per device).  Asynchronous on
 * cuda_stream.  Per-option validation failures write NaN.
 */
int amtc_price_crr_batch(const amtc_batch_soa* d_in, int64_t n, int32_t N, double* d_price,
                         void* cuda_stream);

/* As above with HOST pointers (synchronous). */
int amtc_price_crr_batch_host(const amtc_batch_soa* h_in, int64_t n, int32_t N, double* h_price,
                              void* cuda_stream);

/*
 * k = 0 CRR price of ONE large tree on the current device (config 5a, N up to
 * 10^5 and beyond).  The level is swept in bands of 256
 * levels over warp tiles with ghost columns (region-B dependency).
 * Synchronous on cuda_stream.  *price (HOST pointer) receives V_0(0); NaN and a
 * non-zero status on invalid input (as amtc_price_crr_batch's validation).
 */
int amtc_price_crr_tree(const amtc_params* params, int32_t N, const amtc_payoff* payoff, double* price,
                        void* cuda_stream);

/*
 * NCCL communicator for amtc_price_tree_sharded.  Rank 0 calls
 * amtc_comm_unique_id and shares the 128 bytes with every rank (e.g. over the
 * torch.distributed store); each rank then calls amtc_comm_init on its own
 * device.  The communicator is owned by the caller (amtc_comm_destroy).
 */
int amtc_comm_unique_id(unsigned char id[128]);
int amtc_comm_init(const unsigned char id[128], int nranks, int rank, void** comm);
int amtc_comm_destroy(void* comm);

/*
 * One tree sharded over the nranks GPUs of an amtc_comm_init communicator
 * (SURVEY 8(e), config 5): every rank calls it with the same arguments.  k = 0:
 * rank g owns columns [ceil(g w/na), ceil((g+1) w/na)) of the current level
 * (w = t+1) on the first na = clamp(w/4096, 1, nranks) ranks,
 * re-split every band of 256 levels (the paper's per-round rebalancing,
 * P:178); before each band the ranks exchange their window halos with
 * ncclSend/ncclRecv (region-B dependency).  k > 0: the tree's
 * 32-column strips (strip-split mode of the transaction-cost solver) are
 * partitioned into contiguous ranges of equal work; the only cross-GPU
 * dependency is the carry column of each range's first strip, which the left
 * neighbour's kernel reads from the owner's memory through CUDA IPC (handles
 * all-gathered over the communicator) while polling the owner's per-level
 * progress counter (published with system-scope fences).  Every rank receives
 * the quote in *out (HOST pointer).  nccl_comm may be NULL when nranks = 1
 * (then k > 0 is amtc_price_american_tc); trees with N < 64 are not sharded.
 * Synchronous on cuda_stream.  Returns the status (also in out->status).
 */
int amtc_price_tree_sharded(const amtc_params* params, int32_t N, const amtc_payoff* payoff, double k,
                            void* nccl_comm, int rank, int nranks, amtc_quote* out, void* cuda_stream);

/* Host-only helper (no GPU needed): the exchange plan of band `band` (0 = the
   top band, levels N-1 .. N-D computed from level N) of the k = 0 sharded tree
   as rank `rank` of nranks executes it -- the very function
   amtc_price_tree_sharded runs before each band.  D = levels per band and
   min_cols = the processor-reduction threshold (columns per active rank,
   P:286-288); 0 selects the library's values (256, 4096).  Rank g owns columns
   [ceil(g w/na), ceil((g+1) w/na)) of a level of width w on the first
   na = clamp(w/min_cols, 1, nranks) ranks, re-split every band; its
   window at t_top is its new range plus Dp halo columns from the right (the
   region-B dependency cone).  out (HOST): the band's levels, the
   own / new / window column ranges [lo, hi) and `cap`, the columns of each of
   the library's level buffers.  send / recv (HOST, 2 nranks int64 each): the
   columns [lo, hi) of level t_top sent to / received from each peer (lo == hi:
   none).  *n_bands (may be NULL) receives the band count; band = -1 with
   n_bands != NULL only queries it.  Returns AMTC_EINVAL on bad arguments. */
typedef struct {
    int32_t t_top, Dp;
    int64_t own_lo, own_hi, new_lo, new_hi, win_lo, win_hi, cap;
} amtc_band;
int amtc_tree_band_plan(int32_t N, int nranks, int rank, int32_t band, int32_t D, int64_t min_cols,
                        amtc_band* out, int64_t* send, int64_t* recv, int32_t* n_bands);

/* Host-only helper (no GPU needed): the strip partition amtc_price_tree_sharded
   uses for k > 0 -- rank g owns the 32-column strips [lo[g], lo[g+1]) of the
   N-step tree (N/32 + 1 strips, strip s carrying N - 32 s + 1 levels), ranges of
   equal work, rank 0 holding strip 0 (the root).  lo: nranks + 1 ints. */
int amtc_tree_shard_plan(int32_t N, int nranks, int32_t* lo);

/* Host-only deal of ONE batch of n options over nranks GPUs for the batched
   transaction-cost path ("Sort options by estimated cost ...
   deal to ranks LPT / snake order so per-GPU work is equal; equal option
   counts ('split evenly')"; the paper's load-balance concern).
   Estimated cost of an option (both parties) at N steps:
     (N+1)(N+2)/2 * (2 + AMTC_HEAVY_WEIGHT * [kind != put] * k/h),  h = sigma sqrt(T/N):
   the buyer of a call / bull spread carries ~c k/h heavy columns per level
   (the weight is fitted to the oracle's vertex counts).
   Options are sorted by cost (descending, ties by index) and dealt in snake
   order 0,1,..,n-1,n-1,..,0,0,1,..: per-rank counts differ by at most one.
   h_in: HOST SoA (only T, sigma, k, kind are read; k may be NULL = 0).
   rank_of: n ints (out), the rank that prices option i.  rank_cost: nranks
   doubles (out, may be NULL), the summed estimate per rank.
   Returns AMTC_EINVAL on n < 0, N < 1, nranks < 1 or a NULL pointer; invalid
   options are dealt like any other (the rank that prices them reports their
   status).  No device memory, no CUDA call. */
#define AMTC_HEAVY_WEIGHT 4.0
int amtc_batch_shard_plan(const amtc_batch_soa* h_in, int64_t n, int32_t N, int nranks, int32_t* rank_of,
                          double* rank_cost);

/* Human-readable name of a status code (static storage). */
const char* amtc_strerror(int status);

/* Message of the last CUDA error seen by this thread (static storage per thread). */
const char* amtc_last_error(void);

/* Number of kernels this library has launched in this process (monotonic). */
int64_t amtc_launch_count(void);

/* Work statistics of the last amtc_price_american_tc_batch* call on the
   current device (for throughput / roofline accounting). */
typedef struct {
    int64_t vertex_sum;    /* sum over all node-updates t = N..1, both parties, of the
                              vertex count of the produced node function z_t(j)     */
    int32_t passes;        /* solver passes run (1 + capacity retries)               */
    int32_t pad;
    int64_t retried_items; /* (option, party) items re-run with larger scratch       */
    double solve_ms;       /* device time of the solver kernel launches (CUDA events
                              recorded around them on the call's stream)            */
    double full_ms;        /* first pass: the full solver kernel alone (events on the call's
                              stream around its launch; 0 if it did not run)          */
    double light_ms;       /* first pass: the light solver kernel alone (events on the
                              library's second stream; it overlaps full_ms)           */
} amtc_tc_stats;
int amtc_tc_last_stats(amtc_tc_stats* out);

/* TESTING HOOK (not for production use): node updates whose two children hold
   more than `tl` vertices in total take the warp-cooperative path (default 64);
   a small tl forces that path onto ordinary nodes so tests can check it
   against the oracle.  tl <= 0 restores the default.  Affects later calls. */
void amtc_debug_set_heavy_threshold(int tl);

/* TESTING HOOK: strip-split mode of the transaction-cost solver (the strips
   of one tree on different warps, pipelined through progress counters):
   -1 automatic (default: when the batch has fewer items than a quarter of
   the resident warps), 0 never, 1 whenever it fits in memory. */
void amtc_debug_set_split_mode(int mode);

/* TESTING HOOK: which kernel runs the items that never grow heavy node
   functions (sellers of puts / calls at k/h < 4, put buyers), concurrently
   with the full kernel: 1 (default) the light solver of amtc_light.cu (shared-
   memory strip matrix, prefetched carry, no arenas); 2 the strip kernel's
   light variant (amtc_strip.cu); 0 none (everything on the full kernel).
   Any other value restores the default. */
void amtc_debug_set_light_kernel(int on);

/* TESTING HOOK: which kernel runs the whole-tree items that may grow heavy
   node functions (buyers of calls / bull spreads, bull-spread sellers, and
   every item when the light kernel is off): 0 (default; measured faster on
   the whole config-4 batch) the strip kernel of amtc_strip.cu, also the
   split-mode and sharded-tree kernel; any other value the full solver of
   amtc_full.cu (strip matrix in shared memory, row / carry arenas, tier-3
   CTA work sharing). */
void amtc_debug_set_full_kernel(int which);

/* TESTING HOOK: split mode (few trees, strips pipelined over warps) runs
   batches whose items are all light (sellers of puts / calls, put buyers) on
   the light kernel's split variant (carry hand-off staged one level ahead);
   on = 0 sends them to the strip kernel's split mode instead.  Default 1. */
void amtc_debug_set_light_split(int on);

/* DEVELOPER HOOK: the full solver's clock64 phase accumulators (summed over
   warps since the last reset; out: 8 uint64, HOST): [0] cycles inside heavy
   node updates served, [1] cycles an owner waited for its posted heavy nodes
   (serving excluded), [2] end-of-work idle cycles, [3] total warp cycles, [4]
   heavy nodes served, [5] levels with posted nodes, [6] tier-2 cycles.  Only a
   build with -DAMTC_F_PROF=1 records them (else returns AMTC_EINVAL). */
int amtc_debug_full_profile(uint64_t out[8], int reset);

/* TESTING HOOK: divide the whole-tree solver's row and carry arena capacities
   by 2^shift (0 restores them), so tests can drive items through the capacity
   retry passes (4x arenas per retry) and, past the last retry, AMTC_ECAPACITY. */
void amtc_debug_set_arena_shift(int shift);

/* TESTING HOOK: how amtc_price_crr_tree (and amtc_price_tree_sharded with
   k = 0 on one rank without a communicator) sweeps one k = 0 tree.  0 (default)
   automatic: one cooperative wavefront launch (every warp owns a fixed slot of
   columns and waits on its neighbours' band counters instead of a launch
   boundary per band), falling back to one launch per band of D levels when the
   warps cannot be co-resident; 1 always one launch per band; 2..5 the
   wavefront with (columns per lane M, levels per band D) = (16, 256), (8, 128),
   (12, 128), (8, 64).  Affects later calls. */
void amtc_debug_set_tree_shape(int shape);

#ifdef __cplusplus
}
#endif

#endif /* AMTC_H */
