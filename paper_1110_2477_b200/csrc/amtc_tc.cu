// amtc_tc.cu -- batched ask/bid pricing under proportional transaction costs
// (Sec. 3 seller/buyer recursions P:94-144 on the Sec. 4.1 tree P:159).
//
// Work item = (option, party): party 0 = seller (ask), party 1 =
// buyer (bid).  The two recursions are independent (the paper keeps
// two separate buffers), so they run as separate items.
//
// One CTA owns one item at a time (persistent grid, items pulled from a
// cost-sorted queue).  Levels t = N .. 1 are swept level-synchronously; each
// thread owns a contiguous range of the level's nodes.  Node functions live in
// two ping-pong arenas in global memory (L2-resident for typical items) with a
// compact variable-length layout: per level a block-wide prefix sum of per-node
// scratch bounds assigns every node a private slot
//     [ region0 : b_j vertices | region1 : b_j vertices ]
// used as W (envelope) -> A (restriction pass A, reversed) -> V (pass B) -> Z
// (envelope with the exercise function u); Z stays in region1 as the node's
// function for the next level.  A node whose bound is exceeded raises
// DEV_OVERFLOW and the host re-runs that item with larger bounds.
#include <cuda_runtime.h>

#include "amtc_internal.cuh"
#include "pwl_device.cuh"

namespace amtc {

// ---------------------------------------------------------------------------
// per-option constants (row a1 of SURVEY 8(a))
// ---------------------------------------------------------------------------
struct OptionConsts {
    double S0, K, K2, k, h, rho;
    int kind;
};

__device__ __forceinline__ int validate_option(const BatchPtrs& in, int64_t i, int N, bool need_k,
                                               OptionConsts& oc) {
    oc.S0 = in.S0[i];
    oc.K = in.K[i];
    oc.K2 = in.K2 ? in.K2[i] : 0.0;
    double T = in.T[i], sigma = in.sigma[i], R = in.R[i];
    oc.k = (need_k && in.k) ? in.k[i] : 0.0;
    oc.kind = in.kind[i];
    if (!(oc.S0 > 0.0) || !(T > 0.0) || !(sigma > 0.0) || N < 1) return STATUS_EINVAL;
    if (!(oc.k >= 0.0 && oc.k < 1.0)) return STATUS_EINVAL;
    if (oc.kind != KIND_PUT && oc.kind != KIND_CALL && oc.kind != KIND_BULL) return STATUS_EINVAL;
    if (oc.kind != KIND_BULL && !(oc.K > 0.0)) return STATUS_EINVAL;
    if (oc.kind == KIND_BULL && !(oc.K < oc.K2)) return STATUS_EINVAL;
    if (!isfinite(R)) return STATUS_EINVAL;
    oc.h = sigma * sqrt(T / (double)N);
    oc.rho = R * T / (double)N;
    // d < r < u  <=>  -h < rho < h   (P:79 risk-neutral p in (0,1))
    if (!(oc.rho < oc.h && -oc.h < oc.rho)) return STATUS_EARBITRAGE;
    return STATUS_OK;
}

// ---------------------------------------------------------------------------
// prepare: validate, initialise quotes, order items heavy-first
// ---------------------------------------------------------------------------
constexpr int N_CLASSES = 16;

// cost class of an item: the buyer of a call / bull spread grows "teeth" when
// k/h is large (breakpoint counts measured with the oracle), so
// those items are scheduled first (longest-processing-time order)
__device__ __forceinline__ int item_class(const OptionConsts& oc, int party) {
    if (party == 0 || oc.kind == KIND_PUT) return 0;
    double kh = oc.k / oc.h;
    return min(N_CLASSES - 1, 1 + (int)(4.0 * kh));
}

__global__ void tc_prepare_kernel(BatchPtrs in, int64_t n, int N, Quote* out, unsigned char* cls,
                                  int* hist) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    OptionConsts oc;
    int st = validate_option(in, i, N, true, oc);
    out[i].ask = NAN;
    out[i].bid = NAN;
    out[i].status = st;
    out[i].max_bp = 0;
    for (int p = 0; p < 2; ++p) {
        int c = (st == STATUS_OK) ? item_class(oc, p) : 255;
        cls[2 * i + p] = (unsigned char)c;
        if (c != 255) atomicAdd(&hist[c], 1);
    }
}

// hist[c] -> start offset of class c in heavy-first order; hist[N_CLASSES] = total
__global__ void tc_order_kernel(int* hist) {
    if (threadIdx.x != 0) return;
    int acc = 0;
    for (int c = N_CLASSES - 1; c >= 0; --c) {
        int v = hist[c];
        hist[c] = acc;
        acc += v;
    }
    hist[N_CLASSES] = acc;
}

__global__ void tc_scatter_kernel(int64_t n2, const unsigned char* cls, int* hist, int* items) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n2) return;
    int c = cls[i];
    if (c == 255) return;
    int pos = atomicAdd(&hist[c], 1);
    items[pos] = (int)i;
}

// ---------------------------------------------------------------------------
// block-wide exclusive scan of one int per thread
// ---------------------------------------------------------------------------
__device__ __forceinline__ int block_exclusive_scan(int v, int* s_warp, int& total) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) s_warp[wid] = x;
    __syncthreads();
    if (wid == 0) {
        int w = (lane < nw) ? s_warp[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int y = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w += y;
        }
        if (lane < nw) s_warp[lane] = w;  // inclusive warp prefix
    }
    __syncthreads();
    int base = (wid > 0) ? s_warp[wid - 1] : 0;
    total = s_warp[nw - 1];
    __syncthreads();
    return base + x - v;
}

// ---------------------------------------------------------------------------
// the solver
// ---------------------------------------------------------------------------


__device__ __forceinline__ void payoff(const OptionConsts& oc, double S, double& xi, double& zeta) {
    if (oc.kind == KIND_PUT) { xi = oc.K; zeta = -1.0; }            // (K, -1)
    else if (oc.kind == KIND_CALL) { xi = -oc.K; zeta = 1.0; }      // (-K, +1)   reading R6
    else { xi = fmax(S - oc.K, 0.0) - fmax(S - oc.K2, 0.0); zeta = 0.0; }
}

__global__ void __launch_bounds__(TC_THREADS) tc_solve_kernel(TcLaunch L) {
    __shared__ int s_warp[32];
    __shared__ int s_item, s_err, s_maxn;
    const int N = L.N;
    const int tid = threadIdx.x, nth = blockDim.x;

    // workspace carve-up
    char* base = L.ws + (size_t)blockIdx.x * L.ws_stride;
    double* Epow = reinterpret_cast<double*>(base);              // e^{h i}, i in [-(N+1), N+1]
    double* Dpow = Epow + (2 * N + 3);                           // e^{-rho t}, t in [0, N+1]
    double* slb[2] = {Dpow + (N + 2), Dpow + 2 * (N + 2)};       // left-tail slopes
    int* cnt[2] = {reinterpret_cast<int*>(slb[1] + (N + 2)), nullptr};
    cnt[1] = cnt[0] + (N + 2);
    int* off[2] = {cnt[1] + (N + 2), cnt[1] + 2 * (N + 2)};
    size_t head = (size_t)((char*)(off[1] + (N + 2)) - base);
    head = (head + 255) & ~(size_t)255;
    Vtx* arena[2] = {reinterpret_cast<Vtx*>(base + head), reinterpret_cast<Vtx*>(base + head) + L.arena_cap};

    for (;;) {
        if (tid == 0) {
            s_item = atomicAdd(L.work_counter, 1);
            s_err = 0;
            s_maxn = 1;
        }
        __syncthreads();
        const int it = s_item;
        if (it >= *L.n_items) break;
        const int code = L.items[it];
        const int64_t opt = code >> 1;
        const int party = code & 1;
        OptionConsts oc;
        int st = validate_option(L.in, opt, N, true, oc);
        if (st != STATUS_OK) {  // prepare already recorded the status
            __syncthreads();
            continue;
        }
        // a1: tables
        for (int i = tid; i < 2 * N + 3; i += nth) Epow[i] = exp(oc.h * (double)(i - (N + 1)));
        for (int t = tid; t < N + 2; t += nth) Dpow[t] = exp(-oc.rho * (double)t);
        __syncthreads();
        const double kp = 1.0 + oc.k, km = 1.0 - oc.k;

        // a2: leaves, t = N+1, payoff (0,0): z = u = y^- S^a - y^+ S^b  (Alg.1 l.5)
        int cur = 0;
        for (int j = tid; j <= N + 1; j += nth) {
            double Sd = oc.S0 * Epow[(N + 1) - 2 * j + (N + 1)] * Dpow[N + 1];
            Vtx* v = arena[0] + j;
            v->x = 0.0;
            v->f = 0.0;
            v->s = -km * Sd;
            slb[0][j] = -kp * Sd;
            cnt[0][j] = 1;
            off[0][j] = j;
        }
        __syncthreads();

        // a3/a4/a5: levels t = N .. 1
        unsigned long long my_vertices = 0;
        for (int t = N; t >= 1; --t) {
            const int width = t + 1;
            const int chunk = (width + nth - 1) / nth;
            const int j0 = min(tid * chunk, width), j1 = min(j0 + chunk, width);
            const int* cc = cnt[cur];
            int mine = 0;
            for (int j = j0; j < j1; ++j) mine += 2 * (L.bmul * (cc[j] + cc[j + 1]) + L.badd);
            int total;
            int slot = block_exclusive_scan(mine, s_warp, total);
            if (total > L.arena_cap) {
                if (tid == 0) s_err |= DEV_OVERFLOW;
            }
            __syncthreads();
            if (s_err) break;
            const int nxt = cur ^ 1;
            const Vtx* A0 = arena[cur];
            Vtx* A1 = arena[nxt];
            const double disc = Dpow[t];
            int err = DEV_OK;
            for (int j = j0; j < j1 && !err; ++j) {
                const int b = L.bmul * (cc[j] + cc[j + 1]) + L.badd;
                Vtx* r0 = A1 + slot;
                Vtx* r1 = r0 + b;
                slot += 2 * b;
                const double S = oc.S0 * Epow[t - 2 * j + (N + 1)];
                const double lo = -kp * S * disc, hi = -km * S * disc;  // [-S^a, -S^b] r^-t
                Fn U{A0 + off[cur][j], cc[j], slb[cur][j]};
                Fn D{A0 + off[cur][j + 1], cc[j + 1], slb[cur][j + 1]};
                // u_t: seller Eq.(1), buyer Eq.(6) P:133 (discounted)
                double xi, zeta;
                payoff(oc, S, xi, zeta);
                const double ux = party == 0 ? zeta : -zeta;
                const double uf = (party == 0 ? xi : -xi) * disc;
                int nZ;
                double slZ;
                err |= node_update(U, D, lo, hi, ux, uf, party == 0, r0, r1, b, nZ, slZ);
                if (err) break;
                cnt[nxt][j] = nZ;
                off[nxt][j] = (int)(r1 - A1);
                slb[nxt][j] = slZ;
                my_vertices += (unsigned long long)nZ;
                if (nZ > 1) atomicMax(&s_maxn, nZ);
            }
            if (err) atomicOr(&s_err, err);
            __syncthreads();
            if (s_err) break;
            cur = nxt;
        }
        // a6: root, t = 0, no costs: v_0 is the line of slope -S0
        // through min_b [w_0(b) + S0 b]; ask = max(u_0(0), v_0(0)),
        // bid = -min(u'_0(0), v'_0(0)).
        if (!s_err && tid == 0) {
            const Vtx* A0 = arena[cur];
            Fn U{A0 + off[cur][0], cnt[cur][0], slb[cur][0]};
            Fn D{A0 + off[cur][1], cnt[cur][1], slb[cur][1]};
            Emit E;
            E.out = arena[cur ^ 1];
            E.cap = L.arena_cap;
            envelope(U, D, true, E);
            int err = E.err;
            double S0 = oc.S0;
            if (!(E.sl + S0 < 0.0) || !(E.out[E.m - 1].s + S0 > 0.0)) err |= DEV_UNBOUNDED;
            double mv = INFINITY;
            for (int i = 0; i < E.m; ++i) mv = fmin(mv, fma(S0, E.out[i].x, E.out[i].f));
            double xi, zeta;
            payoff(oc, S0, xi, zeta);
            double intrinsic = xi + zeta * S0;
            if (err) {
                s_err |= err;
            } else if (party == 0) {
                L.out[opt].ask = fmax(intrinsic, mv);
            } else {
                L.out[opt].bid = fmax(intrinsic, -mv);
            }
            if (E.m > s_maxn) s_maxn = E.m;
        }
        if (my_vertices) atomicAdd(L.vertex_sum, my_vertices);
        __syncthreads();
        if (tid == 0) {
            if (s_err & DEV_OVERFLOW) {
                int k = atomicAdd(L.ovf_count, 1);
                L.ovf_items[k] = code;
            } else if (s_err & DEV_UNBOUNDED) {
                atomicMax(&L.out[opt].status, STATUS_EUNBOUNDED);
            }
            atomicMax(&L.out[opt].max_bp, s_maxn);
        }
        __syncthreads();
    }
}

__global__ void status_reduce_kernel(const Quote* out, int64_t n, int* worst) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n && out[i].status) atomicMax(worst, out[i].status);
}

void launch_status_reduce(const Quote* out, int64_t n, int* worst, cudaStream_t s) {
    cudaMemsetAsync(worst, 0, sizeof(int), s);
    status_reduce_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(out, n, worst);
    note_launch();
}

// mark items that exhausted every capacity
__global__ void tc_mark_capacity_kernel(const int* items, int n_items, Quote* out) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_items) return;
    atomicMax(&out[items[i] >> 1].status, STATUS_ECAPACITY);
}

size_t tc_workspace_bytes(int N, int arena_cap) {
    size_t head = sizeof(double) * (size_t)(2 * N + 3 + (N + 2) + 2 * (N + 2)) + sizeof(int) * 4 * (size_t)(N + 2);
    head = (head + 255) & ~(size_t)255;
    return head + 2 * sizeof(Vtx) * (size_t)arena_cap;
}

void tc_launch_prepare(const BatchPtrs& in, int64_t n, int N, Quote* out, unsigned char* cls, int* hist,
                       int* items, cudaStream_t s) {
    const int threads = 256;
    cudaMemsetAsync(hist, 0, sizeof(int) * (N_CLASSES + 1), s);
    tc_prepare_kernel<<<(unsigned)((n + threads - 1) / threads), threads, 0, s>>>(in, n, N, out, cls, hist);
    note_launch();
    tc_order_kernel<<<1, 32, 0, s>>>(hist);
    note_launch();
    tc_scatter_kernel<<<(unsigned)((2 * n + threads - 1) / threads), threads, 0, s>>>(2 * n, cls, hist, items);
    note_launch();
}

void tc_launch_solve(const TcLaunch& L, int grid, cudaStream_t s) {
    tc_solve_kernel<<<grid, TC_THREADS, 0, s>>>(L);
    note_launch();
}

void tc_launch_mark_capacity(const int* items, int n_items, Quote* out, cudaStream_t s) {
    if (n_items <= 0) return;
    tc_mark_capacity_kernel<<<(n_items + 255) / 256, 256, 0, s>>>(items, n_items, out);
    note_launch();
}

int tc_solve_occupancy() {
    int nb = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, tc_solve_kernel, TC_THREADS, 0);
    return nb < 1 ? 1 : nb;
}

}  // namespace amtc
