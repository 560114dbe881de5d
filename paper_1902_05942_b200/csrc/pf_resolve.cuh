// Resolve-phase building blocks shared by the single-GPU frame kernels (pf_frame.cu)
// and the key-sharded multi-GPU kernels (pf_shard.cu): packed effective records,
// per-row means, the lookup/coarse keys of a vertex, the ordered 3x3x3 pool and the
// fallback ladder of src/pipeline.py:207-283.
#pragma once

#include "pf_insert.cuh"

namespace pf {

// Per-CTA counters in 32-bit shared words (native ATOMS; a CTA never sees 2^32
// events), flushed once as 64-bit global adds.
struct BlockStats {
    unsigned v[PF_STAT_HIST_BASE];
    unsigned hist[256];
};

// with_hist false: the kernel never counts probe lengths (and flushes without them)
__device__ __forceinline__ void stats_init(BlockStats &b, bool with_hist = true) {
    for (int k = threadIdx.x; k < PF_STAT_HIST_BASE; k += blockDim.x) b.v[k] = 0;
    if (with_hist)
        for (int k = threadIdx.x; k < 256; k += blockDim.x) b.hist[k] = 0;
}

// warp-aggregated add of a per-lane predicate into a block counter
__device__ __forceinline__ void warp_count(BlockStats &b, int slot, bool pred) {
    const unsigned m = __ballot_sync(kFull, pred);
    if ((threadIdx.x & 31) == 0 && m) atomicAdd(&b.v[slot], static_cast<unsigned>(__popc(m)));
}

__device__ __forceinline__ void stats_flush(const BlockStats &b, int64_t *stats, bool with_hist) {
    for (int k = threadIdx.x; k < PF_STAT_HIST_BASE; k += blockDim.x)
        if (b.v[k])
            atomicAdd(reinterpret_cast<unsigned long long *>(stats + k),
                      static_cast<unsigned long long>(b.v[k]));
    if (with_hist)
        for (int k = threadIdx.x; k < 256; k += blockDim.x)
            if (b.hist[k])
                atomicAdd(reinterpret_cast<unsigned long long *>(stats + PF_STAT_HIST_BASE + k),
                          static_cast<unsigned long long>(b.hist[k]));
}


// Per-slot effective record: three sum words (int64 or float64 bits, as
// VoxelTable.effective's dtype) and the count as a float64 -- one 32-byte sector.
// A count word of all ones marks "no such cell" (the lookup found nothing).
constexpr unsigned long long kAbsentCount = ~0ull;

__device__ __forceinline__ ulonglong4 pack_effective(const Effective &e, bool as_int) {
    ulonglong4 r;
    r.x = as_int ? static_cast<unsigned long long>(e.isum[0]) : __double_as_longlong(e.fsum[0]);
    r.y = as_int ? static_cast<unsigned long long>(e.isum[1]) : __double_as_longlong(e.fsum[1]);
    r.z = as_int ? static_cast<unsigned long long>(e.isum[2]) : __double_as_longlong(e.fsum[2]);
    r.w = __double_as_longlong(e.fcnt);
    return r;
}

__device__ __forceinline__ ulonglong4 absent_record() {
    return make_ulonglong4(0ull, 0ull, 0ull, kAbsentCount);
}

__device__ __forceinline__ Effective unpack_effective(const ulonglong4 &r, bool as_int) {
    Effective e;
    const unsigned long long w[3] = {r.x, r.y, r.z};
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        e.isum[c] = as_int ? static_cast<int64_t>(w[c]) : 0;
        e.fsum[c] = as_int ? 0.0 : __longlong_as_double(w[c]);
    }
    e.fcnt = __longlong_as_double(r.w);
    e.icnt = static_cast<int64_t>(e.fcnt);  // exact: counts < 2^53
    return e;
}

__device__ __forceinline__ ulonglong4 load_record(const ulonglong4 *rec, int64_t k) {
    const ulonglong2 *p = reinterpret_cast<const ulonglong2 *>(rec + k);
    const ulonglong2 lo = __ldg(p), hi = __ldg(p + 1);
    return make_ulonglong4(lo.x, lo.y, hi.x, hi.y);
}

// _mean_rows (src/pipeline.py:196-200) for one row.
__device__ __forceinline__ double row_mean(double sum, double cnt, bool fixed) {
    double d = np_max(cnt, 1e-300);
    if (fixed) d = dmul(d, kFixedScale);
    return ddiv(sum, d);
}

// The three channels of one row: one correctly rounded reciprocal of the shared
// divisor and Markstein's correction per channel (div3_rcp), each quotient equal to
// IEEE sum / d; a divisor outside the theorem's range (cnt 0 -> 1e-300) takes IEEE
// division inside div3_rcp.
#ifndef PF_ROW_MEAN_RCP
#define PF_ROW_MEAN_RCP 1
#endif
__device__ __forceinline__ void row_mean3(const double sum[3], double cnt, bool fixed, double m[3]) {
#if PF_ROW_MEAN_RCP
    double d = np_max(cnt, 1e-300);
    if (fixed) d = dmul(d, kFixedScale);
    div3_rcp(sum, d, __drcp_rn(d), m);
#else
#pragma unroll
    for (int c = 0; c < 3; ++c) m[c] = row_mean(sum[c], cnt, fixed);
#endif
}

struct KeyAndHash {
    CellKey first;
    CellHash second;
};

// The key of one vertex on jitter stream base h0 with the given level delta
// (src/pipeline.py:126-135): the resolve phase's fine lookup key (stream 3, delta 0)
// and coarse key (stream 3 or 2, coarse_delta).
__device__ __forceinline__ KeyAndHash vertex_key(const pf_config &cfg, const pf_vertices &v,
                                                 uint64_t h0, int64_t row, int32_t delta) {
    const VertexIn x = load_vertex(v, row, cfg);
    double du = 0.0, dv = 0.0;
    if (cfg.jitter) {
        double u1, u2;
        jitter_draws(h0, x.pixel, x.sample, u1, u2);
        disc_offset(u1, u2, du, dv);
    }
    const KeyShared ks = key_shared(cfg, x);
    double jt[3];
    KeyAndHash r;
    r.first = make_key(cfg, x, ks, cfg.jitter, du, dv, delta, jt);
    r.second = key_hash(r.first, ks);
    return r;
}

// The 3x3x3 neighbourhood pool of one work row (src/pipeline.py:185-192, 241-254):
// lane j < 27 holds cell (dx, dy, dz) = (j/9-1, j/3%3-1, j%3-1) with `found` and its
// effective value; every lane returns the sums accumulated in j order, numpy's order
// for the float64 pools.  The pool's keys carry no normal_fp_bins.
struct Pool {
    int64_t isum[3];
    int64_t icnt;
    double fsum[3];
    double fcnt;
};

__device__ __forceinline__ Pool pool_neighbours(bool found, const Effective &e, bool as_int,
                                                int mode) {
    Pool p{{0, 0, 0}, 0, {0.0, 0.0, 0.0}, 0.0};
    const unsigned fm = __ballot_sync(kFull, found);
    for (int j = 0; j < 27; ++j) {
        if (!((fm >> j) & 1u)) continue;  // warp-uniform
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            if (as_int) p.isum[c] += __shfl_sync(kFull, static_cast<long long>(e.isum[c]), j);
            else p.fsum[c] = dadd(p.fsum[c], __shfl_sync(kFull, e.fsum[c], j));
        }
        if (mode == PF_INTEGRATE) p.icnt += __shfl_sync(kFull, static_cast<long long>(e.icnt), j);
        else p.fcnt = dadd(p.fcnt, __shfl_sync(kFull, e.fcnt, j));
    }
    return p;
}

__device__ __forceinline__ int neighbour_dx(int j) { return j / 9 - 1; }
__device__ __forceinline__ int neighbour_dy(int j) { return (j / 3) % 3 - 1; }
__device__ __forceinline__ int neighbour_dz(int j) { return j % 3 - 1; }

// Rungs 2-5 of the ladder (src/pipeline.py:256-283) for one row, given the pooled
// neighbourhood and the coarse cell's effective value (coarse_found false when the
// coarse rung did not find the cell or was not consulted).  Returns the source code
// (1 neighbourhood, 2 coarse, 3 unfiltered) and writes the chosen mean.
__device__ __forceinline__ int ladder_choose(const Pool &p, bool as_int, int mode, bool fixed,
                                             double thr, bool coarse_found, const Effective &ce,
                                             bool c_int, const double contrib[3],
                                             double chosen[3]) {
    const double cnt_n = (mode == PF_INTEGRATE) ? static_cast<double>(p.icnt) : p.fcnt;
    const bool ok_n = cnt_n >= thr;
    double mean_n[3] = {0.0, 0.0, 0.0};
    if (cnt_n > 0.0) {
        const double sums[3] = {as_int ? static_cast<double>(p.isum[0]) : p.fsum[0],
                                as_int ? static_cast<double>(p.isum[1]) : p.fsum[1],
                                as_int ? static_cast<double>(p.isum[2]) : p.fsum[2]};
        row_mean3(sums, cnt_n, fixed, mean_n);
    }
    double cnt_c = 0.0;
    double mean_c[3] = {0.0, 0.0, 0.0};
    if (!ok_n && coarse_found) {
        cnt_c = ce.fcnt;
        if (cnt_c > 0.0) {
            const double sums[3] = {eff_sum_f64(ce, c_int, 0), eff_sum_f64(ce, c_int, 1),
                                    eff_sum_f64(ce, c_int, 2)};
            row_mean3(sums, cnt_c, fixed, mean_c);
        }
    }
    const bool ok_c = !ok_n && cnt_c >= thr;
    const bool any_n = !ok_n && !ok_c && cnt_n >= 1.0;
    const bool any_c = !ok_n && !ok_c && !any_n && cnt_c >= 1.0;
    // written as selects: an if/else-if chain here was mis-compiled (nvcc 12.9, sm_100a),
    // taking the unfiltered branch with ok_c set (tests/test_gpu_parity.py::test_frame_golden)
    const int src = (ok_n || any_n) ? 1 : ((ok_c || any_c) ? 2 : 3);
#pragma unroll
    for (int c = 0; c < 3; ++c) chosen[c] = src == 1 ? mean_n[c] : (src == 2 ? mean_c[c] : contrib[c]);
    return src;
}

}  // namespace pf
