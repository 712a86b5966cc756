// amtc_prepare.cu -- batch preparation for the transaction-cost solver:
// per-option validation (SURVEY 8(b) error conventions), output
// initialisation (NaN prices), and the heavy-first work queue of items
// (option, party) for the persistent solver (longest-processing-time order:
// the buyer of a call / bull spread at large k/h grows the long "sawtooth"
// node functions).
#include <cuda_runtime.h>

#include "amtc_internal.cuh"
#include "amtc_option.cuh"

namespace amtc {

// ---------------------------------------------------------------------------
// prepare: validate, initialise quotes, order items heavy-first
// ---------------------------------------------------------------------------
constexpr int N_CLASSES = TC_CLASSES;

// cost class of an item: the buyer of a call / bull spread grows "teeth" when
// k/h is large (breakpoint counts measured with the oracle), so
// those items are scheduled first (longest-processing-time order)
// Class 0 (the light kernel): put buyers and sellers of puts / calls; the bull
// spread's seller grows heavy functions too (measured: 230 config-4 bull sellers
// overflowed the light kernel), so both bull items take the full kernel.
// The seller of a call at large k/h reaches 7-9 vertices (oracle, config 4):
// above KH_LIGHT_CALL_SELLER it starts on the full kernel instead of
// overflowing the light kernel's 6-vertex slots into a serial re-run pass.
constexpr double KH_LIGHT_CALL_SELLER = 4.0;
__device__ __forceinline__ int item_class(const OptionConsts& oc, int party) {
    const double kh = oc.k / oc.h;
    if (oc.kind == KIND_PUT || (party == 0 && oc.kind == KIND_CALL && kh < KH_LIGHT_CALL_SELLER)) return 0;
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

// worst status of the batch; a failed option keeps NaN prices (amtc.h) even if
// one of its two items (seller / buyer) completed
__global__ void status_reduce_kernel(Quote* out, int64_t n, int* worst) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n && out[i].status) {
        atomicMax(worst, out[i].status);
        out[i].ask = NAN;
        out[i].bid = NAN;
    }
}

void launch_status_reduce(Quote* out, int64_t n, int* worst, cudaStream_t s) {
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

// split mode: item c -> S strip items c S + s, strips right to left (s = S-1 .. 0),
// so a strip is always claimed after the strip whose carry column it reads
// (a sharded tree keeps only strips [s_lo, s_hi) on this GPU)
__global__ void tc_split_expand_kernel(const int* items, const int* n_items, int S, int s_lo, int s_hi, int* out,
                                       int* n_out) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int n = *n_items, w = s_hi - s_lo;
    if (i == 0) *n_out = n * w;
    if (i >= (int64_t)n * w) return;
    const int k = (int)(i / w), q = (int)(i % w);
    out[i] = items[k] * S + (s_hi - 1 - q);
}

void tc_launch_split_expand(const int* items, const int* n_items, int S, int64_t max_items, int* out, int* n_out,
                            cudaStream_t s, int s_lo, int s_hi) {
    if (s_hi < 0) s_hi = S;
    tc_split_expand_kernel<<<(unsigned)((max_items + 255) / 256), 256, 0, s>>>(items, n_items, S, s_lo, s_hi, out,
                                                                                n_out);
    note_launch();
}

__global__ void tc_mark_all_capacity_kernel(int64_t n, Quote* out) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    if (out[i].status == STATUS_OK) {  // invalid options keep their own status
        out[i].status = STATUS_ECAPACITY;
        out[i].ask = out[i].bid = NAN;
    }
}

void tc_launch_mark_all_capacity(Quote* out, int64_t n, cudaStream_t s) {
    if (n <= 0) return;
    tc_mark_all_capacity_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(n, out);
    note_launch();
}

void tc_launch_mark_capacity(const int* items, int n_items, Quote* out, cudaStream_t s) {
    if (n_items <= 0) return;
    tc_mark_capacity_kernel<<<(n_items + 255) / 256, 256, 0, s>>>(items, n_items, out);
    note_launch();
}

}  // namespace amtc
