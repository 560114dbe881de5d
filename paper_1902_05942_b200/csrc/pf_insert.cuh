// Warp-merged insert: the table write path shared by the batch-accumulate kernel
// and the fused frame-insert kernel.
#pragma once

#include "pf_device.cuh"

namespace pf {

constexpr unsigned kFull = 0xFFFFFFFFu;


// 16.16 fixed point, half up (src/_native.pyx:251-253): floor(v*65536 + 0.5).
__device__ __forceinline__ int64_t quantize_fixed(double v) {
    return np_floor_i64(dadd(dmul(v, kFixedScale), 0.5));
}

struct LaneInsert {
    int64_t slot;
    int32_t status;
    int32_t probe_len;
    uint64_t victim_tag;
    int64_t victim_touch;
    bool leader;      // this lane performed the probe for its key group
    unsigned peers;   // lanes holding the same (index, fingerprint)
};

// All 32 lanes must call this together.  Lanes holding the same (index, fp) are
// merged with __match_any_sync; the lowest lane (= earliest vertex) probes and
// claims once and adds the group's summed radiance with one atomic per channel,
// plus the group's weight to the count (popc(peers) for one vertex per lane, the
// summed per-lane weights when WEIGHTED -- pre-aggregated shard records).  Lane
// sums arrive already quantised (FIXED) or as float64.  Followers report what a
// sequential caller would see after the leader: same slot and probe length,
// status 1 -> 0.
template <bool FIXED, bool WEIGHTED>
__device__ __forceinline__ LaneInsert warp_insert_sums(const pf_table &t, bool valid, uint64_t idx,
                                                       uint32_t fp, int64_t qsum[3],
                                                       double fsum[3], uint64_t weight,
                                                       int64_t frame, uint64_t home_tag,
                                                       bool merge = true, bool touch = true) {
    const unsigned lane = threadIdx.x & 31u;
    const uint64_t k2 = static_cast<uint64_t>(fp) | (static_cast<uint64_t>(valid) << 32);
    // merge == false: every lane is its own group; lanes with the same key then probe
    // side by side (the claim CAS / eviction protocol of probe_insert resolves them to
    // one cell exactly as the merged path does) and each adds its own vertex
    const unsigned peers = merge ? (__match_any_sync(kFull, valid ? idx : 0ull) &
                                    __match_any_sync(kFull, k2))
                                 : (1u << lane);
    const int leader = __ffs(peers) - 1;
    const bool is_leader = valid && static_cast<int>(lane) == leader;
    if (WEIGHTED && !valid) weight = 0;

    // Group sums by pointer jumping over each group's member list: every lane links to
    // the next higher lane of its group and adds its successor's partial sum, doubling
    // the stride each round, so the leader holds the group total after
    // ceil(log2(group size)) rounds (0 rounds when all 32 keys differ).  The
    // summation tree depends only on lane positions, so float totals are repeatable.
    const unsigned above = valid && lane < 31 ? (peers & (0xFFFFFFFFu << (lane + 1))) : 0u;
    int nxt = above ? __ffs(above) - 1 : -1;
    while (__any_sync(kFull, nxt >= 0)) {
        const int src = nxt >= 0 ? nxt : static_cast<int>(lane);
        const int nn = __shfl_sync(kFull, nxt, src);
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            if (FIXED) {
                const long long x = __shfl_sync(kFull, static_cast<long long>(qsum[c]), src);
                if (nxt >= 0) qsum[c] += x;
            } else {
                const double x = __shfl_sync(kFull, fsum[c], src);
                if (nxt >= 0) fsum[c] = dadd(fsum[c], x);
            }
        }
        if (WEIGHTED) {
            const unsigned long long x = __shfl_sync(kFull, static_cast<unsigned long long>(weight), src);
            if (nxt >= 0) weight += x;
        }
        if (nxt >= 0) nxt = nn;
    }

    InsertResult r;
    r.slot = -1;
    r.status = 2;
    r.probe_len = 0;
    r.victim_tag = 0;
    r.victim_touch = 0;
    r.counted = false;
    const uint64_t group_weight = WEIGHTED ? weight : static_cast<uint64_t>(__popc(peers));
    if (is_leader) {
        r = probe_insert(t, idx, fp, home_tag, group_weight);
        if (r.status != 2) {
            const int64_t s = r.slot;
            const uint64_t keep = l2_policy(PF_TABLE_RED_POLICY);
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                if (FIXED)
                    red_add_u64(reinterpret_cast<int64_t *>(sum_at(t, s, c)),
                                static_cast<uint64_t>(qsum[c]), keep);
                else
                    red_add_f64(reinterpret_cast<double *>(sum_at(t, s, c)), fsum[c], keep);
            }
            if (!r.counted) red_add_u64(cnt_at(t, s), group_weight, keep);
            if (touch) st_relaxed_u64(touch_at(t, s), static_cast<uint64_t>(frame));
        }
    }
    LaneInsert out;
    out.slot = __shfl_sync(kFull, static_cast<long long>(r.slot), leader);
    out.status = __shfl_sync(kFull, r.status, leader);
    out.probe_len = __shfl_sync(kFull, r.probe_len, leader);
    out.victim_tag = is_leader ? r.victim_tag : 0ull;
    out.victim_touch = is_leader ? r.victim_touch : 0;
    if (!is_leader && out.status == 1) {
        // a later vertex of the same key finds the freshly evicted cell
        out.status = 0;
        out.probe_len = static_cast<int32_t>(
            ((static_cast<uint64_t>(out.slot) - (idx & static_cast<uint64_t>(t.capacity - 1))) &
             static_cast<uint64_t>(t.capacity - 1)) + 1);
    }
    out.leader = is_leader;
    out.peers = peers;
    return out;
}

// One vertex per lane, no warp collectives: every valid lane probes / claims for its own
// key and adds its own quantised radiance and a count of 1 (lanes holding the same key
// resolve to the same cell through probe_insert's claim CAS and eviction protocol).
// q: the lane's radiance already quantised (FIXED), val: as float64 (float mode).
template <bool FIXED>
__device__ __forceinline__ LaneInsert lane_insert(const pf_table &t, bool valid, uint64_t idx,
                                                  uint32_t fp, const int64_t q[3],
                                                  const double val[3], int64_t frame,
                                                  uint64_t home_tag, bool touch = true) {
    LaneInsert out;
    out.slot = -1;
    out.status = 2;
    out.probe_len = 0;
    out.victim_tag = 0;
    out.victim_touch = 0;
    out.leader = valid;
    out.peers = 1u << (threadIdx.x & 31u);
    if (!valid) return out;
    const InsertResult r = probe_insert(t, idx, fp, home_tag, 1ull);
    if (r.status != 2) {
        const int64_t s = r.slot;
        const uint64_t keep = l2_policy(PF_TABLE_RED_POLICY);
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            if (FIXED)
                red_add_u64(reinterpret_cast<int64_t *>(sum_at(t, s, c)),
                            static_cast<uint64_t>(q[c]), keep);
            else
                red_add_f64(reinterpret_cast<double *>(sum_at(t, s, c)), val[c], keep);
        }
        if (!r.counted) red_add_u64(cnt_at(t, s), 1ull, keep);
        if (touch) st_relaxed_u64(touch_at(t, s), static_cast<uint64_t>(frame));
    }
    out.slot = r.slot;
    out.status = r.status;
    out.probe_len = r.probe_len;
    out.victim_tag = r.victim_tag;
    out.victim_touch = r.victim_touch;
    return out;
}

// One vertex per lane: quantise the lane's radiance and insert it (weight 1).
template <bool FIXED>
__device__ __forceinline__ LaneInsert warp_insert(const pf_table &t, bool valid, uint64_t idx,
                                                  uint32_t fp, const double val[3], int64_t frame,
                                                  uint64_t home_tag, bool merge = true,
                                                  bool touch = true) {
    int64_t qsum[3];
    double fsum[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        if (FIXED) qsum[c] = valid ? quantize_fixed(val[c]) : 0;
        else fsum[c] = valid ? val[c] : 0.0;
    }
    return warp_insert_sums<FIXED, false>(t, valid, idx, fp, qsum, fsum, 1, frame, home_tag, merge,
                                           touch);
}

}  // namespace pf
