// Sweep over the occupied slots of a table.
//
// A table is a few percent occupied, so one thread per slot leaves most lanes idle
// and every occupied slot's dependent loads form one latency chain.  Instead a CTA
// streams kChunk tags with 16-byte loads, compacts the occupied slots into a shared
// queue (warp-aggregated appends), then hands the queue to all of its threads.
#pragma once

#include "pf_device.cuh"

namespace pf {

template <int THREADS>
struct SweepSmem {
    static constexpr int kPairsPerThread = 4;
    static constexpr int kChunk = THREADS * 2 * kPairsPerThread;
    int64_t slot[kChunk];
    uint64_t tag[kChunk];
    int n;
};

// f(slot, tag) runs once per occupied slot, spread over the CTA's threads.  The CTA is
// block `blk` of `nblk` sweeping this table (a kernel may split its grid over jobs).
template <int THREADS, typename F>
__device__ __forceinline__ void for_each_occupied(const uint64_t *tags, int64_t capacity,
                                                  SweepSmem<THREADS> &q, int64_t blk,
                                                  int64_t nblk, F &&f) {
    constexpr int kP = SweepSmem<THREADS>::kPairsPerThread;
    constexpr int kChunk = SweepSmem<THREADS>::kChunk;
    const int lane = threadIdx.x & 31;
    const ulonglong2 *tags2 = reinterpret_cast<const ulonglong2 *>(tags);
    for (int64_t base = blk * kChunk; base < capacity; base += nblk * kChunk) {
        if (threadIdx.x == 0) q.n = 0;
        __syncthreads();
        ulonglong2 tg[kP];
#pragma unroll
        for (int j = 0; j < kP; ++j) {
            const int64_t p = base / 2 + j * THREADS + threadIdx.x;
            tg[j] = 2 * p < capacity ? tags2[p] : make_ulonglong2(kEmptyTag, kEmptyTag);
        }
#pragma unroll
        for (int j = 0; j < kP; ++j) {
            const int64_t p = base / 2 + j * THREADS + threadIdx.x;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const uint64_t tag = h ? tg[j].y : tg[j].x;
                const bool occ = tag != kEmptyTag;
                const unsigned m = __ballot_sync(0xFFFFFFFFu, occ);
                if (m) {
                    int q0 = 0;
                    if (lane == __ffs(m) - 1) q0 = atomicAdd(&q.n, __popc(m));
                    q0 = __shfl_sync(0xFFFFFFFFu, q0, __ffs(m) - 1);
                    if (occ) {
                        const int k = q0 + __popc(m & ((1u << lane) - 1u));
                        q.slot[k] = 2 * p + h;
                        q.tag[k] = tag;
                    }
                }
            }
        }
        __syncthreads();
        const int n_q = q.n;
        for (int k = threadIdx.x; k < n_q; k += THREADS) f(q.slot[k], q.tag[k]);
        __syncthreads();
    }
}

template <int THREADS, typename F>
__device__ __forceinline__ void for_each_occupied(const uint64_t *tags, int64_t capacity,
                                                  SweepSmem<THREADS> &q, F &&f) {
    for_each_occupied<THREADS>(tags, capacity, q, blockIdx.x, gridDim.x, f);
}

// CTAs for a sweep over `capacity` slots (each CTA step covers kChunk slots).
template <int THREADS>
inline unsigned sweep_blocks(int64_t capacity, int sms) {
    const int64_t chunks = (capacity + SweepSmem<THREADS>::kChunk - 1) / SweepSmem<THREADS>::kChunk;
    const int64_t cap = static_cast<int64_t>(sms) * 8;
    return static_cast<unsigned>(chunks < cap ? chunks : cap);
}

}  // namespace pf
