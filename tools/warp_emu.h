// tools/warp_emu.h -- HOST emulation of the warp collectives used by the
// device headers (32 std::threads, one per lane, synchronised by a barrier at
// every collective), so warp-cooperative device code can be unit-tested on the
// CPU.  Test infrastructure only.
#pragma once
#include <atomic>
#include <algorithm>
#include <cmath>
#include <cstring>
#include <thread>
#include <vector>

#define __device__
#define __host__
#define __forceinline__ inline
#define __noinline__
#define __global__

namespace warp_emu {
// sense-reversing spin barrier (yielding): much cheaper than a futex barrier
struct SpinBarrier {
    std::atomic<int> count{0};
    std::atomic<int> gen{0};
    int n;
    explicit SpinBarrier(int n_) : n(n_) {}
    void arrive_and_wait() {
        const int g = gen.load(std::memory_order_acquire);
        if (count.fetch_add(1, std::memory_order_acq_rel) == n - 1) {
            count.store(0, std::memory_order_relaxed);
            gen.fetch_add(1, std::memory_order_acq_rel);
        } else {
            while (gen.load(std::memory_order_acquire) == g) std::this_thread::yield();
        }
    }
};
inline SpinBarrier*& bar() { static SpinBarrier* b = nullptr; return b; }
inline unsigned long long* slots() { static unsigned long long s[32]; return s; }
inline int& lane_id() { thread_local int l = 0; return l; }
template <class T>
inline T xchg(T v, int src) {
    static_assert(sizeof(T) <= 8, "64-bit max");
    unsigned long long u = 0;
    std::memcpy(&u, &v, sizeof(T));
    slots()[lane_id()] = u;
    bar()->arrive_and_wait();
    const unsigned long long r = slots()[src];
    bar()->arrive_and_wait();
    T out;
    std::memcpy(&out, &r, sizeof(T));
    return out;
}
// run f(lane) on 32 emulated lanes
template <class F>
inline void run_warp(F f) {
    SpinBarrier b(32);
    bar() = &b;
    std::vector<std::thread> th;
    for (int l = 0; l < 32; ++l) th.emplace_back([&, l] { lane_id() = l; f(l); });
    for (auto& t : th) t.join();
    bar() = nullptr;
}
}  // namespace warp_emu

using std::isfinite;
using std::max;
using std::min;

template <class T> inline T __shfl_sync(unsigned, T v, int src) { return warp_emu::xchg(v, src & 31); }
template <class T> inline T __shfl_up_sync(unsigned, T v, unsigned d) {
    const int l = warp_emu::lane_id();
    return warp_emu::xchg(v, l >= (int)d ? l - (int)d : l);
}
template <class T> inline T __shfl_down_sync(unsigned, T v, unsigned d) {
    const int l = warp_emu::lane_id();
    return warp_emu::xchg(v, l + (int)d < 32 ? l + (int)d : l);
}
template <class T> inline T __shfl_xor_sync(unsigned, T v, int m) { return warp_emu::xchg(v, warp_emu::lane_id() ^ m); }
inline int __reduce_or_sync(unsigned, int v) {
    int r = 0;
    for (int l = 0; l < 32; ++l) r |= warp_emu::xchg(v, l);
    return r;
}
inline bool __any_sync(unsigned, int v) {
    int r = 0;
    for (int l = 0; l < 32; ++l) r |= warp_emu::xchg(v != 0 ? 1 : 0, l);
    return r != 0;
}
inline void __syncwarp(unsigned = 0xffffffffu) { warp_emu::bar()->arrive_and_wait(); }
inline unsigned __ballot_sync(unsigned, int v) {
    unsigned r = 0;
    for (int l = 0; l < 32; ++l) r |= (warp_emu::xchg(v != 0 ? 1 : 0, l) ? 1u : 0u) << l;
    return r;
}
inline int __popc(unsigned v) { return __builtin_popcount(v); }
