// Table kernels behind the reference kernel-module ABI and the VoxelTable API:
// batch accumulate (parallel warp-merged, or sequential-order), lookup, key build,
// hashing, effective sums, the temporal update (begin_frame) and occupancy.
#include "pf_insert.cuh"
#include "pf_sweep.cuh"
#include "pf_internal.cuh"

namespace pf {

constexpr int kThreads = 256;

// ------------------------------------------------------------------ accumulate

struct BatchOut {
    uint8_t *status;
    int64_t *slots;
    uint8_t *probe_len;
    uint64_t *victim_tags;
    int64_t *victim_touch;
};

// Parallel batch insert (src/_native.pyx:186-258 semantics, warp-merged atomics).
template <bool FIXED>
__global__ void __launch_bounds__(kThreads)
accumulate_kernel(const PF_GRID_CONST pf_table t, const uint64_t *__restrict__ idx, const uint32_t *__restrict__ fp,
                  const double *__restrict__ vals, int64_t n, int64_t frame, BatchOut o) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const bool valid = i < n;
    double v[3] = {0.0, 0.0, 0.0};
    uint64_t k = 0;
    uint32_t f = 0;
    if (valid) {
        k = __ldg(reinterpret_cast<const unsigned long long *>(idx) + i);
        f = __ldg(fp + i);
#pragma unroll
        for (int c = 0; c < 3; ++c) v[c] = __ldg(vals + 3 * i + c);
    }
    const uint64_t home_tag =
        valid ? ld_relaxed(t.tags + (k & static_cast<uint64_t>(t.capacity - 1))) : 0ull;
    const LaneInsert r = warp_insert<FIXED>(t, valid, k, f, v, frame, home_tag);
    if (!valid) return;
    if (o.status) o.status[i] = static_cast<uint8_t>(r.status);
    if (o.slots) o.slots[i] = r.status == 2 ? -1 : r.slot;
    if (o.probe_len) o.probe_len[i] = static_cast<uint8_t>(r.probe_len);
    if (o.victim_tags) o.victim_tags[i] = r.victim_tag;
    if (o.victim_touch) o.victim_touch[i] = r.victim_touch;
}

// Sequential-order batch insert: one warp walks the batch in vertex order, reading
// each probe window 32 slots at a time.  Reproduces the reference's threads=1 table
// layout bit for bit (claims, evictions, probe lengths, statuses).
template <bool FIXED>
__global__ void __launch_bounds__(32)
accumulate_ordered_kernel(pf_table t, const uint64_t *__restrict__ idx,
                          const uint32_t *__restrict__ fp, const double *__restrict__ vals,
                          int64_t n, int64_t frame, BatchOut o) {
    const int lane = threadIdx.x;
    const uint64_t mask = static_cast<uint64_t>(t.capacity) - 1;
    const int P = t.probe_limit;
    for (int64_t i = 0; i < n; ++i) {
        const uint64_t home = idx[i] & mask;
        const uint64_t want = static_cast<uint64_t>(fp[i]);
        int stop_j = -1;
        bool stop_empty = false;
        int64_t victim = -1;
        uint64_t victim_tag = 0;
        for (int base = 0; base < P; base += 32) {
            const int j = base + lane;
            const bool in = j < P;
            const uint64_t s = (home + static_cast<uint64_t>(j)) & mask;
            const uint64_t tag = in ? ld_relaxed(t.tags + s) : 0ull;
            const bool is_empty = in && tag == kEmptyTag;
            const bool stop = in && (is_empty || (tag & kFpMask) == want);
            const unsigned m = __ballot_sync(kFull, stop);
            if (m) {
                const int first = __ffs(m) - 1;
                stop_j = base + first;
                stop_empty = __shfl_sync(kFull, is_empty, first);
                break;
            }
            // eviction candidates in this chunk: largest tag, earliest slot on ties
            bool elig = false;
            if (in) {
                const uint64_t age = (tag >> 32) & kAgeMask;
                elig = age >= static_cast<uint64_t>(t.evict_min_age) &&
                       ld_relaxed_i64(cnt_at(t, s)) == 0;
            }
            uint64_t best_tag = tag;
            int best_j = elig ? j : INT32_MAX;
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) {
                const uint64_t ot = __shfl_xor_sync(kFull, best_tag, off);
                const int oj = __shfl_xor_sync(kFull, best_j, off);
                const bool take = oj != INT32_MAX &&
                                  (best_j == INT32_MAX || ot > best_tag ||
                                   (ot == best_tag && oj < best_j));
                if (take) {
                    best_tag = ot;
                    best_j = oj;
                }
            }
            if (best_j != INT32_MAX && (victim < 0 || best_tag > victim_tag)) {
                victim = static_cast<int64_t>((home + static_cast<uint64_t>(best_j)) & mask);
                victim_tag = best_tag;
            }
        }
        if (lane == 0) {
            int status = 0;
            int64_t slot = -1;
            int plen = P;
            uint64_t vt = 0;
            int64_t vtt = 0;
            if (stop_j >= 0) {
                slot = static_cast<int64_t>((home + static_cast<uint64_t>(stop_j)) & mask);
                plen = stop_j + 1;
                if (stop_empty) st_relaxed_u64(t.tags + slot, (kFresh << 32) | want);
            } else if (victim >= 0) {
                status = 1;
                slot = victim;
                vt = victim_tag;
                vtt = ld_relaxed_i64(touch_at(t, victim));
                zero_cell(t, victim);
                st_relaxed_u64(t.tags + victim, (kFresh << 32) | want);
            } else {
                status = 2;
            }
            if (status != 2) {
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    const double x = vals[3 * i + c];
                    if (FIXED) {
                        int64_t *p = reinterpret_cast<int64_t *>(sum_at(t, slot, c));
                        st_relaxed_u64(p, static_cast<uint64_t>(ld_relaxed_i64(p) + quantize_fixed(x)));
                    } else {
                        double *p = reinterpret_cast<double *>(sum_at(t, slot, c));
                        const uint64_t bits = ld_relaxed(reinterpret_cast<const uint64_t *>(p));
                        st_relaxed_u64(p, __double_as_longlong(dadd(__longlong_as_double(bits), x)));
                    }
                }
                st_relaxed_u64(cnt_at(t, slot), static_cast<uint64_t>(ld_relaxed_i64(cnt_at(t, slot)) + 1));
                st_relaxed_u64(touch_at(t, slot), static_cast<uint64_t>(frame));
            }
            if (o.status) o.status[i] = static_cast<uint8_t>(status);
            if (o.slots) o.slots[i] = slot;
            if (o.probe_len) o.probe_len[i] = static_cast<uint8_t>(plen);
            if (o.victim_tags) o.victim_tags[i] = vt;
            if (o.victim_touch) o.victim_touch[i] = vtt;
            __threadfence_block();
        }
        __syncwarp();
    }
}

// ------------------------------------------------------------------ lookup

__global__ void __launch_bounds__(kThreads)
lookup_kernel(const uint64_t *__restrict__ tags, uint64_t mask, int probe_limit,
              const uint64_t *__restrict__ idx, const uint32_t *__restrict__ fp, int64_t n,
              int64_t *__restrict__ out) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    out[i] = probe_lookup(tags, mask, probe_limit,
                          __ldg(reinterpret_cast<const unsigned long long *>(idx) + i), __ldg(fp + i));
}

// ------------------------------------------------------------------ keys

__device__ __forceinline__ void store_key(const pf_key_out &o, int64_t i, const CellKey &k,
                                          const CellHash &h, const double jt[3]) {
    if (o.qx) o.qx[i] = k.q[0];
    if (o.qy) o.qy[i] = k.q[1];
    if (o.qz) o.qz[i] = k.q[2];
    if (o.level) o.level[i] = k.level;
    if (o.aux) o.aux[i] = k.aux;
    if (o.index) o.index[i] = h.index;
    if (o.fingerprint) o.fingerprint[i] = h.fp;
    if (o.jittered) {
#pragma unroll
        for (int c = 0; c < 3; ++c) o.jittered[3 * i + c] = jt[c];
    }
}

// mode 0: explicit draws (u1/u2 may be NULL -> no jitter); mode 1: counter RNG.
__global__ void __launch_bounds__(kThreads)
keys_kernel(pf_config cfg, pf_vertices v, const double *__restrict__ u1,
            const double *__restrict__ u2, int use_rng, uint64_t h0, int32_t level_delta,
            pf_key_out o) {
    __shared__ double lod_dist[32];
    stage_lod_dist(lod_dist, cfg);
    __syncthreads();
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= v.n) return;
    const VertexIn x = load_vertex(v, i, cfg);
    const KeyShared ks = key_shared(cfg, x, lod_dist);
    int jit = 0;
    double du = 0.0, dv = 0.0;
    if (cfg.jitter) {
        double a, b;
        if (use_rng) {
            jitter_draws(h0, x.pixel, x.sample, a, b);
            jit = 1;
        } else if (u1 != nullptr && u2 != nullptr) {
            a = __ldg(u1 + i);
            b = __ldg(u2 + i);
            jit = 1;
        }
        if (jit) disc_offset(a, b, du, dv);
    }
    double jt[3];
    const CellKey k = make_key(cfg, x, ks, jit, du, dv, level_delta, jt);
    store_key(o, i, k, key_hash(k, ks), jt);
}

__global__ void __launch_bounds__(kThreads)
hash_kernel(const int64_t *__restrict__ qx, const int64_t *__restrict__ qy,
            const int64_t *__restrict__ qz, const int64_t *__restrict__ level,
            const uint64_t *__restrict__ aux, const uint32_t *__restrict__ fp_bins, int64_t n,
            uint64_t *__restrict__ index, uint32_t *__restrict__ fp) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const CellHash h = cell_hash(qx[i], qy[i], qz[i], level[i], aux[i], fp_bins != nullptr,
                                 fp_bins ? fp_bins[i] : 0u);
    index[i] = h.index;
    fp[i] = h.fp;
}

// ------------------------------------------------------------------ effective / begin_frame

__global__ void __launch_bounds__(kThreads)
effective_kernel(pf_table t, int mode, double ema, double delta_max, void *eff_sum,
                 void *eff_count) {
    const int64_t s = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (s >= t.capacity) return;
    const Effective e = effective_at(t, s, mode, ema, delta_max);
    const bool as_int = eff_is_int(t, mode);
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        if (as_int) static_cast<int64_t *>(eff_sum)[3 * s + c] = e.isum[c];
        else static_cast<double *>(eff_sum)[3 * s + c] = e.fsum[c];
    }
    if (mode == PF_INTEGRATE) static_cast<int64_t *>(eff_count)[s] = e.icnt;
    else static_cast<double *>(eff_count)[s] = e.fcnt;
}

template <bool FIXED>
__device__ __forceinline__ int fold_slot(const pf_table &t, int64_t s, uint64_t tag, int64_t frame,
                                         int mode, double ema, double delta_max,
                                         int32_t sample_cap);

// begin_frame (src/table.py:242-298) as one sweep over the tag array.  Empty slots
// hold all-zero state (invariant of every reference code path), so only occupied
// slots are folded.
template <bool FIXED>
__global__ void __launch_bounds__(kThreads)
begin_frame_kernel(pf_table t, int64_t frame, int mode, double ema, double delta_max,
                   int32_t sample_cap, int64_t *horizon_clears) {
    __shared__ SweepSmem<kThreads> q;
    __shared__ int block_clears;
    if (threadIdx.x == 0) block_clears = 0;
    int cleared = 0;
    for_each_occupied<kThreads>(t.tags, t.capacity, q, [&](int64_t s, uint64_t tag) {
        cleared += fold_slot<FIXED>(t, s, tag, frame, mode, ema, delta_max, sample_cap);
    });
    if (cleared) atomicAdd(&block_clears, cleared);
    __syncthreads();
    if (threadIdx.x == 0 && block_clears && horizon_clears)
        atomicAdd(reinterpret_cast<unsigned long long *>(horizon_clears),
                  static_cast<unsigned long long>(block_clears));
}

// begin_frame for one occupied slot (src/table.py:242-298); returns 1 when the slot
// is cleared by the horizon.
template <bool FIXED>
__device__ __forceinline__ int fold_slot(const pf_table &t, int64_t s, uint64_t tag, int64_t frame,
                                         int mode, double ema, double delta_max,
                                         int32_t sample_cap) {
    // every field loaded at once, folded in registers, stored once
    const CellState cs = load_cell(t, s, false);
    uint64_t hist[3];
    int64_t hc = cs.hist_counts;
#pragma unroll
    for (int c = 0; c < 3; ++c) hist[c] = cs.hist[c];
    const int64_t age = frame - cs.last_touch;
    const bool cleared = age > t.evict_horizon;
    uint64_t new_tag = kEmptyTag;
    if (!cleared) {
        if (mode == PF_INTEGRATE) {
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                if (FIXED) hist[c] = cs.hist[c] + cs.sums[c];
                else hist[c] = __double_as_longlong(dadd(__longlong_as_double(cs.hist[c]),
                                                          __longlong_as_double(cs.sums[c])));
            }
            hc = cs.hist_counts + cs.counts;
        } else {
            const Effective e = effective_of(cs, FIXED, mode, ema, delta_max);
            int64_t cnt = np_i64(rint(e.fcnt));
            if (mode == PF_FILTER && cnt > 1) cnt = 1;
            if (cnt > 0) {
                const double denom = np_max(e.fcnt, 1e-300);
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    const double nh = dmul(ddiv(e.fsum[c], denom), static_cast<double>(cnt));
                    hist[c] = FIXED ? static_cast<uint64_t>(np_floor_i64(dadd(nh, 0.5)))
                                    : static_cast<uint64_t>(__double_as_longlong(nh));
                }
                hc = cnt;
            } else {
#pragma unroll
                for (int c = 0; c < 3; ++c) hist[c] = 0;  // int64 0 / +0.0
                hc = 0;
            }
        }
        if (sample_cap && (mode == PF_INTEGRATE || mode == PF_HYBRID) && hc > sample_cap) {
            const double scale = ddiv(static_cast<double>(sample_cap), static_cast<double>(hc));
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                if (FIXED)
                    hist[c] = static_cast<uint64_t>(np_floor_i64(dadd(
                        dmul(static_cast<double>(static_cast<int64_t>(hist[c])), scale), 0.5)));
                else
                    hist[c] = __double_as_longlong(dmul(__longlong_as_double(hist[c]), scale));
            }
            hc = sample_cap;
        }
        // re-prioritise (src/table.py:53-57, 289-290)
        const uint64_t c8 = static_cast<uint64_t>(hc < 255 ? hc : 255);
        const uint64_t a24 = static_cast<uint64_t>(
            age < static_cast<int64_t>(kPrioAgeMask) ? age : static_cast<int64_t>(kPrioAgeMask));
        const uint64_t prio = ((255ull - c8) << 24) | a24;
        new_tag = (prio << 32) | (tag & kFpMask);
    } else {
        hist[0] = hist[1] = hist[2] = 0;
        hc = 0;
        *touch_at(t, s) = 0;
    }
    uint64_t *hsum = hsum_at(t, s);
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        *sum_at(t, s, c) = 0;  // live generation reset (bits of 0.0)
        hsum[c] = hist[c];
    }
    *cnt_at(t, s) = 0;
    *hcnt_at(t, s) = hc;
    *delta_at(t, s) = 0.0;
    t.tags[s] = new_tag;
    return cleared ? 1 : 0;
}

__global__ void __launch_bounds__(kThreads)
count_occupied_kernel(const uint64_t *__restrict__ tags, int64_t capacity, int64_t *out) {
    __shared__ int block_count;
    if (threadIdx.x == 0) block_count = 0;
    __syncthreads();
    int local = 0;
    for (int64_t s = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; s < capacity;
         s += static_cast<int64_t>(gridDim.x) * blockDim.x)
        local += __ldg(reinterpret_cast<const unsigned long long *>(tags) + s) != kEmptyTag;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) local += __shfl_xor_sync(kFull, local, off);
    if ((threadIdx.x & 31) == 0 && local) atomicAdd(&block_count, local);
    __syncthreads();
    if (threadIdx.x == 0 && block_count)
        atomicAdd(reinterpret_cast<unsigned long long *>(out),
                  static_cast<unsigned long long>(block_count));
}

__global__ void __launch_bounds__(kThreads)
check_contributions_kernel(const double *__restrict__ vals, int64_t count, int32_t *bad) {
    bool any = false;
    for (int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; k < count;
         k += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const double x = __ldg(vals + k);
        any |= !(x >= 0.0 && x <= 1.7976931348623157e308);  // NaN, +-inf or negative
    }
    if (__any_sync(kFull, any) && (threadIdx.x & 31) == 0) atomicExch(bad, 1);
}

// Self-test of div_rcp / div3_rcp against IEEE division: random numerators and divisors over a
// wide exponent range, plus the quantiser's divisors base_voxel * 2^level with the
// reciprocal scaled by 2^-level (mismatches[0] and [1]).
__global__ void __launch_bounds__(kThreads)
selftest_division_kernel(uint64_t seed, int64_t n, double base_voxel, unsigned long long *bad) {
    unsigned long long b0 = 0, b1 = 0;
    const double rbv = __drcp_rn(base_voxel);
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const uint64_t h1 = mix64(seed ^ (2 * static_cast<uint64_t>(i) + 1));
        const uint64_t h2 = mix64(h1 ^ 0x9E3779B97F4A7C15ull);
        const int ex = static_cast<int>((h1 >> 52) % 241) - 120;
        const int ey = static_cast<int>((h2 >> 52) % 241) - 120;
        const double mx = 1.0 + static_cast<double>(h1 & 0xFFFFFFFFFFFFFull) * 0x1p-52;
        const double my = 1.0 + static_cast<double>(h2 & 0xFFFFFFFFFFFFFull) * 0x1p-52;
        const double x = ((h1 >> 51) & 1 ? -mx : mx) * pow2i(ex);
        const double y = ((h2 >> 51) & 1 ? -my : my) * pow2i(ey);
        if (__double_as_longlong(div_rcp(x, y, __drcp_rn(y))) != __double_as_longlong(__ddiv_rn(x, y)))
            ++b0;
        // div3_rcp: a regular numerator, a signed zero and one scaled far out of the
        // Markstein range (IEEE fallback), by one divisor
        const int ez = static_cast<int>((h1 >> 8) % 2001) - 1000;
        const double x3[3] = {x, (h2 & 1) ? -0.0 : 0.0, x * pow2i(ez)};
        double q3[3];
        div3_rcp(x3, y, __drcp_rn(y), q3);
        for (int c = 0; c < 3; ++c)
            if (__double_as_longlong(q3[c]) != __double_as_longlong(__ddiv_rn(x3[c], y))) ++b0;
        const int64_t lv = static_cast<int64_t>(h2 % 32);
        const double step = voxel_step(base_voxel, lv);
        const double xs = (static_cast<double>(static_cast<int64_t>(h1 >> 20)) - 8.0e12) * 0x1p-30;
        const double xq[3] = {xs, -xs * 0.5, xs * 3.0};
        double q[3];
        div3_rcp(xq, step, dmul(rbv, pow2i(-lv)), q);
        for (int c = 0; c < 3; ++c)
            if (__double_as_longlong(q[c]) != __double_as_longlong(__ddiv_rn(xq[c], step))) ++b1;
    }
    if (b0) atomicAdd(bad, b0);
    if (b1) atomicAdd(bad + 1, b1);
}

// The frame prologue of pf_filter_frame in one launch: begin_frame on the fine and the
// coarse table and the input check, interleaved over the grid (job = block % jobs) so
// the three sweeps run side by side; block 0 also clears the frame's counters.
template <bool FIXED>
__global__ void __launch_bounds__(kThreads)
frame_prologue_kernel(const PF_GRID_CONST pf_table fine, const PF_GRID_CONST pf_table coarse,
                      int jobs, int64_t frame, int mode,
                      double ema, double delta_max, int32_t sample_cap, int64_t *clears_fine,
                      int64_t *clears_coarse, const double *vals, int64_t count, int32_t *bad,
                      int64_t *zero0, int64_t n0, int64_t *zero1, int64_t n1, int64_t *zero2,
                      const int32_t *occ_fine, const int32_t *occ_coarse, const int64_t *occ_n,
                      int64_t *zero3) {
    __shared__ SweepSmem<kThreads> q;
    __shared__ int block_clears;
    pdl_wait();
    if (blockIdx.x == 0) {
        for (int64_t k = threadIdx.x; k < n0; k += blockDim.x) zero0[k] = 0;
        for (int64_t k = threadIdx.x; k < n1; k += blockDim.x) zero1[k] = 0;
        if (zero2 && threadIdx.x == 0) *zero2 = 0;
        if (zero3 && threadIdx.x < 2) zero3[threadIdx.x] = 0;
    }
    const int job = static_cast<int>(blockIdx.x % jobs);
    const int64_t blk = blockIdx.x / jobs, nblk = gridDim.x / jobs;
    const bool check = vals != nullptr && job == jobs - 1;
    if (check) {  // NaN, +-inf or negative contributions; 16-byte loads, 4 per thread in flight
        const double2 *v2 = reinterpret_cast<const double2 *>(vals);
        const int64_t n2 = count / 2;
        bool any = false;
        const int64_t stride = nblk * blockDim.x;
        for (int64_t k = blk * blockDim.x + threadIdx.x; k < n2; k += 4 * stride) {
            double2 x[4];
#pragma unroll
            for (int u = 0; u < 4; ++u)
                x[u] = k + u * stride < n2 ? __ldg(v2 + k + u * stride) : make_double2(0.0, 0.0);
#pragma unroll
            for (int u = 0; u < 4; ++u)
                any |= !(x[u].x >= 0.0 && x[u].x <= 1.7976931348623157e308) ||
                       !(x[u].y >= 0.0 && x[u].y <= 1.7976931348623157e308);
        }
        if (blk == 0 && threadIdx.x == 0 && (count & 1)) {
            const double x = __ldg(vals + count - 1);
            any |= !(x >= 0.0 && x <= 1.7976931348623157e308);
        }
        if (__any_sync(kFull, any) && (threadIdx.x & 31) == 0) atomicExch(bad, 1);
        return;
    }
    const pf_table &t = job == 0 ? fine : coarse;
    if (threadIdx.x == 0) block_clears = 0;
    int cleared = 0;
    const int32_t *occ = job == 0 ? occ_fine : occ_coarse;
    if (occ != nullptr) {
        // the slots occupied when the previous frame ended (its effective-record sweep's
        // list; the host passes it only when nothing touched the tables since): exactly
        // the slots the tag sweep would find, without reading the tag arrays
        const int64_t m = occ_n[job == 0 ? 0 : 1];
        for (int64_t d = blk * blockDim.x + threadIdx.x; d < m; d += nblk * blockDim.x) {
            const int64_t s = occ[d];
            const uint64_t tag = ld_relaxed(t.tags + s);
            if (tag != kEmptyTag)
                cleared += fold_slot<FIXED>(t, s, tag, frame, mode, ema, delta_max, sample_cap);
        }
    } else {
        for_each_occupied<kThreads>(t.tags, t.capacity, q, blk, nblk, [&](int64_t s, uint64_t tag) {
            cleared += fold_slot<FIXED>(t, s, tag, frame, mode, ema, delta_max, sample_cap);
        });
    }
    if (cleared) atomicAdd(&block_clears, cleared);
    __syncthreads();
    int64_t *clears = job == 0 ? clears_fine : clears_coarse;
    if (threadIdx.x == 0 && block_clears && clears)
        atomicAdd(reinterpret_cast<unsigned long long *>(clears),
                  static_cast<unsigned long long>(block_clears));
}

// temporal.reevaluation_deltas per voxel (src/temporal.py:80-92): voxel v's rows are
// order[offsets[v] .. offsets[v+1]) in stream order, so the float sums follow np.add.at.
__global__ void __launch_bounds__(kThreads)
segment_deltas_kernel(const int64_t *order, const int64_t *offsets, int64_t n_vox,
                      const double *c_old, const double *c_new, double eps, double *delta) {
    const int64_t v = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (v >= n_vox) return;
    double so[3] = {0.0, 0.0, 0.0}, sn[3] = {0.0, 0.0, 0.0}, cnt = 0.0;
    for (int64_t j = offsets[v]; j < offsets[v + 1]; ++j) {
        const int64_t r = order[j];
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            so[c] = dadd(so[c], c_old[3 * r + c]);
            sn[c] = dadd(sn[c], c_new[3 * r + c]);
        }
        cnt = dadd(cnt, 1.0);
    }
    double num = 0.0, den = 0.0;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        const double mo = ddiv(so[c], cnt), mn = ddiv(sn[c], cnt);
        num = c == 0 ? fabs(dsub(mn, mo)) : dadd(num, fabs(dsub(mn, mo)));
        den = c == 0 ? fabs(mo) : dadd(den, fabs(mo));
    }
    delta[v] = ddiv(num, dadd(den, eps));
}

// glibc_sincos over an array (diagnostic entry point for the bit-exactness test).
__global__ void __launch_bounds__(kThreads)
sincos_kernel(const double *x, int64_t n, double *s, double *c) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) glibc_sincos(x[i], s[i], c[i]);
}

// ------------------------------------------------------------------ host wrappers

static int accumulate_table(const char *fn, const pf_table &t, const uint64_t *idx,
                            const uint32_t *fp, const double *vals, int64_t n, int64_t frame,
                            int32_t ordered, BatchOut o, void *stream) {
    if (int rc = validate_table(fn, &t)) return rc;
    const bool fixed = t.sum_mode == PF_SUM_FIXED;
    if (n < 0) return fail_arg(fn, "negative batch size");
    if (n == 0) return PF_OK;
    if (!idx || !fp || !vals) return fail_arg(fn, "idx/fp/vals is NULL");
    cudaStream_t st = as_stream(stream);
    if (ordered) {
        if (fixed) accumulate_ordered_kernel<true><<<1, 32, 0, st>>>(t, idx, fp, vals, n, frame, o);
        else accumulate_ordered_kernel<false><<<1, 32, 0, st>>>(t, idx, fp, vals, n, frame, o);
    } else {
        const unsigned g = blocks_for(n, kThreads);
        if (fixed) accumulate_kernel<true><<<g, kThreads, 0, st>>>(t, idx, fp, vals, n, frame, o);
        else accumulate_kernel<false><<<g, kThreads, 0, st>>>(t, idx, fp, vals, n, frame, o);
    }
    return check_launch(fn);
}

// The kernel-module ABI's caller-owned arrays: the reference's SoA layout.
static int accumulate_impl(const char *fn, bool fixed, uint64_t *tags, void *sums, int64_t *counts,
                           void *hist_sums, int64_t *hist_counts, int64_t *last_touch,
                           double *deltas, int64_t capacity, const uint64_t *idx,
                           const uint32_t *fp, const double *vals, int64_t n, int64_t frame,
                           int32_t probe_limit, int32_t evict_min_age, int32_t ordered,
                           BatchOut o, void *stream) {
    const pf_table t{tags, sums, counts, hist_sums, hist_counts, last_touch, deltas, capacity,
                     fixed ? PF_SUM_FIXED : PF_SUM_FLOAT, probe_limit, evict_min_age, 0,
                     1, 3, 1, 3, 1};
    return accumulate_table(fn, t, idx, fp, vals, n, frame, ordered, o, stream);
}

}  // namespace pf

using namespace pf;

extern "C" {

int pf_accumulate_table(const pf_table *t, const uint64_t *idx, const uint32_t *fp,
                        const double *vals, int64_t n, int64_t frame, int32_t ordered,
                        uint8_t *status, int64_t *slots, uint8_t *probe_len,
                        uint64_t *victim_tags, int64_t *victim_touch, void *stream) {
    if (t == nullptr) return fail_arg("pf_accumulate_table", "table is NULL");
    return accumulate_table("pf_accumulate_table", *t, idx, fp, vals, n, frame, ordered,
                            BatchOut{status, slots, probe_len, victim_tags, victim_touch}, stream);
}

int pf_accumulate_fixed(uint64_t *tags, int64_t *sums, int64_t *counts, int64_t *hist_sums,
                        int64_t *hist_counts, int64_t *last_touch, double *deltas,
                        int64_t capacity, const uint64_t *idx, const uint32_t *fp,
                        const double *vals, int64_t n, int64_t frame, int32_t probe_limit,
                        int32_t evict_min_age, int32_t ordered, uint8_t *status,
                        int64_t *slots, uint8_t *probe_len, uint64_t *victim_tags,
                        int64_t *victim_touch, void *stream) {
    return accumulate_impl("pf_accumulate_fixed", true, tags, sums, counts, hist_sums, hist_counts,
                           last_touch, deltas, capacity, idx, fp, vals, n, frame, probe_limit,
                           evict_min_age, ordered,
                           BatchOut{status, slots, probe_len, victim_tags, victim_touch}, stream);
}

int pf_accumulate_float(uint64_t *tags, double *sums, int64_t *counts, double *hist_sums,
                        int64_t *hist_counts, int64_t *last_touch, double *deltas,
                        int64_t capacity, const uint64_t *idx, const uint32_t *fp,
                        const double *vals, int64_t n, int64_t frame, int32_t probe_limit,
                        int32_t evict_min_age, int32_t ordered, uint8_t *status,
                        int64_t *slots, uint8_t *probe_len, uint64_t *victim_tags,
                        int64_t *victim_touch, void *stream) {
    return accumulate_impl("pf_accumulate_float", false, tags, sums, counts, hist_sums,
                           hist_counts, last_touch, deltas, capacity, idx, fp, vals, n, frame,
                           probe_limit, evict_min_age, ordered,
                           BatchOut{status, slots, probe_len, victim_tags, victim_touch}, stream);
}

int pf_lookup_slots(const uint64_t *tags, int64_t capacity, const uint64_t *idx,
                    const uint32_t *fp, int64_t n, int32_t probe_limit, int64_t *out,
                    void *stream) {
    const char *fn = "pf_lookup_slots";
    if (!is_pow2(capacity)) return fail_arg(fn, "capacity must be a power of two >= 2");
    if (probe_limit < 1) return fail_arg(fn, "probe_limit must be >= 1");
    if (n < 0) return fail_arg(fn, "negative batch size");
    if (n == 0) return PF_OK;
    if (!tags || !idx || !fp || !out) return fail_arg(fn, "NULL pointer");
    lookup_kernel<<<blocks_for(n, kThreads), kThreads, 0, as_stream(stream)>>>(
        tags, static_cast<uint64_t>(capacity) - 1, probe_limit, idx, fp, n, out);
    return check_launch(fn);
}

int pf_make_key_arrays(const pf_config *cfg, const pf_vertices *v, const double *u1,
                       const double *u2, int32_t level_delta, pf_key_out *out, void *stream) {
    const char *fn = "pf_make_key_arrays";
    if (int rc = validate_vertices(fn, v, cfg)) return rc;
    if (out == nullptr) return fail_arg(fn, "out is NULL");
    pf_config kc;
    if (int rc = prepare_config(fn, cfg, &kc)) return rc;
    if (v->n == 0) return PF_OK;
    keys_kernel<<<blocks_for(v->n, kThreads), kThreads, 0, as_stream(stream)>>>(
        kc, *v, u1, u2, 0, 0ull, level_delta, *out);
    return check_launch(fn);
}

int pf_vertex_keys(const pf_config *cfg, const pf_vertices *v, uint64_t stream_base,
                   int32_t level_delta, pf_key_out *out, void *stream) {
    const char *fn = "pf_vertex_keys";
    if (int rc = validate_vertices(fn, v, cfg)) return rc;
    if (out == nullptr) return fail_arg(fn, "out is NULL");
    pf_config kc;
    if (int rc = prepare_config(fn, cfg, &kc)) return rc;
    if (v->n == 0) return PF_OK;
    keys_kernel<<<blocks_for(v->n, kThreads), kThreads, 0, as_stream(stream)>>>(
        kc, *v, nullptr, nullptr, 1, stream_base, level_delta, *out);
    return check_launch(fn);
}

int pf_hash_arrays(const int64_t *qx, const int64_t *qy, const int64_t *qz, const int64_t *level,
                   const uint64_t *aux, const uint32_t *normal_fp_bins, int64_t n,
                   uint64_t *index, uint32_t *fingerprint, void *stream) {
    const char *fn = "pf_hash_arrays";
    if (n < 0) return fail_arg(fn, "negative size");
    if (n == 0) return PF_OK;
    if (!qx || !qy || !qz || !level || !aux || !index || !fingerprint)
        return fail_arg(fn, "NULL pointer");
    hash_kernel<<<blocks_for(n, kThreads), kThreads, 0, as_stream(stream)>>>(
        qx, qy, qz, level, aux, normal_fp_bins, n, index, fingerprint);
    return check_launch(fn);
}

int pf_effective(const pf_table *t, int32_t mode, double ema_alpha, double delta_max,
                 void *eff_sum, void *eff_count, void *stream) {
    const char *fn = "pf_effective";
    if (int rc = validate_table(fn, t)) return rc;
    if (mode < PF_INTEGRATE || mode > PF_HYBRID) return fail_arg(fn, "unknown temporal mode");
    if (!eff_sum || !eff_count) return fail_arg(fn, "NULL output");
    effective_kernel<<<blocks_for(t->capacity, kThreads), kThreads, 0, as_stream(stream)>>>(
        *t, mode, ema_alpha, delta_max, eff_sum, eff_count);
    return check_launch(fn);
}

int pf_begin_frame(const pf_table *t, int64_t frame, int32_t mode, double ema_alpha,
                   double delta_max, int32_t sample_cap, int64_t *horizon_clears, void *stream) {
    const char *fn = "pf_begin_frame";
    if (int rc = validate_table(fn, t)) return rc;
    if (mode < PF_INTEGRATE || mode > PF_HYBRID) return fail_arg(fn, "unknown temporal mode");
    const unsigned g = sweep_blocks<kThreads>(t->capacity, sm_count());
    if (t->sum_mode == PF_SUM_FIXED)
        begin_frame_kernel<true><<<g, kThreads, 0, as_stream(stream)>>>(
            *t, frame, mode, ema_alpha, delta_max, sample_cap, horizon_clears);
    else
        begin_frame_kernel<false><<<g, kThreads, 0, as_stream(stream)>>>(
            *t, frame, mode, ema_alpha, delta_max, sample_cap, horizon_clears);
    return check_launch(fn);
}

}  // extern "C"

namespace pf {

int frame_prologue(const pf_table *fine, const pf_table *coarse, int64_t frame, int32_t mode,
                   double ema, double delta_max, int32_t sample_cap, int64_t *clears_fine,
                   int64_t *clears_coarse, const double *vals, int64_t count, int32_t *bad,
                   int64_t *zero0, int64_t n0, int64_t *zero1, int64_t n1, int64_t *zero2,
                   cudaStream_t st, const int32_t *occ_fine, const int32_t *occ_coarse,
                   const int64_t *occ_n, int64_t *zero3) {
    const char *fn = "pf_filter_frame";
    if (int rc = validate_table(fn, fine)) return rc;
    if (coarse) {
        if (int rc = validate_table(fn, coarse)) return rc;
        if (coarse->sum_mode != fine->sum_mode) return fail_arg(fn, "fine/coarse sum_mode differ");
    }
    if (mode < PF_INTEGRATE || mode > PF_HYBRID) return fail_arg(fn, "unknown temporal mode");
    const bool checking = vals != nullptr && bad != nullptr && count > 0;
    const int jobs = (coarse ? 2 : 1) + (checking ? 1 : 0);
    const unsigned per_job = sweep_blocks<kThreads>(fine->capacity, sm_count());
    const pf_table c = coarse ? *coarse : *fine;
    const unsigned g = per_job * static_cast<unsigned>(jobs);
    launch_pdl(fine->sum_mode == PF_SUM_FIXED ? frame_prologue_kernel<true>
                                              : frame_prologue_kernel<false>,
               dim3(g), dim3(kThreads), st, *fine, c, jobs, frame, mode, ema, delta_max,
               sample_cap, clears_fine, clears_coarse, checking ? vals : nullptr, count, bad,
               zero0, n0, zero1, n1, zero2, occ_n ? occ_fine : nullptr,
               occ_n && coarse ? occ_coarse : nullptr, occ_n, zero3);
    return check_launch(fn);
}

}  // namespace pf

extern "C" {

int pf_begin_frame_checked(const pf_table *fine, const pf_table *coarse, int64_t frame,
                           int32_t mode, double ema_alpha, double delta_max, int32_t sample_cap,
                           int64_t *clears_fine, int64_t *clears_coarse, const double *vals,
                           int64_t count, int32_t *bad, void *stream) {
    cudaStream_t st = as_stream(stream);
    if (bad && cudaMemsetAsync(bad, 0, sizeof(int32_t), st) != cudaSuccess)
        return check_launch("pf_begin_frame_checked");
    return frame_prologue(fine, coarse, frame, mode, ema_alpha, delta_max, sample_cap,
                          clears_fine, clears_coarse, vals, count, bad, nullptr, 0, nullptr, 0,
                          nullptr, st);
}

int pf_selftest_division(uint64_t seed, int64_t n, double base_voxel, int64_t *mismatches,
                         void *stream) {
    const char *fn = "pf_selftest_division";
    if (n < 0 || !mismatches) return fail_arg(fn, "bad arguments");
    selftest_division_kernel<<<static_cast<unsigned>(sm_count()) * 8, kThreads, 0,
                               as_stream(stream)>>>(
        seed, n, base_voxel, reinterpret_cast<unsigned long long *>(mismatches));
    return check_launch(fn);
}

int pf_check_contributions(const double *vals, int64_t count, int32_t *bad, void *stream) {
    const char *fn = "pf_check_contributions";
    if (count < 0 || !bad) return fail_arg(fn, "bad arguments");
    if (count == 0) return PF_OK;
    if (!vals) return fail_arg(fn, "vals is NULL");
    int64_t blocks = (count + kThreads - 1) / kThreads;
    const int64_t cap = static_cast<int64_t>(sm_count()) * 8;
    if (blocks > cap) blocks = cap;
    check_contributions_kernel<<<static_cast<unsigned>(blocks), kThreads, 0, as_stream(stream)>>>(
        vals, count, bad);
    return check_launch(fn);
}

int pf_segment_deltas(const int64_t *order, const int64_t *offsets, int64_t n_vox,
                      const double *c_old, const double *c_new, double delta_eps, double *delta,
                      void *stream) {
    if (n_vox < 0 || (n_vox > 0 && (!order || !offsets || !c_old || !c_new || !delta)))
        return fail_arg("pf_segment_deltas", "bad arguments");
    if (n_vox == 0) return PF_OK;
    segment_deltas_kernel<<<blocks_for(n_vox, kThreads), kThreads, 0, as_stream(stream)>>>(
        order, offsets, n_vox, c_old, c_new, delta_eps, delta);
    return check_launch("pf_segment_deltas");
}

int pf_sincos(const double *x, int64_t n, double *s, double *c, void *stream) {
    if (n < 0 || (n > 0 && (!x || !s || !c))) return fail_arg("pf_sincos", "bad arguments");
    if (n == 0) return PF_OK;
    sincos_kernel<<<blocks_for(n, kThreads), kThreads, 0, as_stream(stream)>>>(x, n, s, c);
    return check_launch("pf_sincos");
}

int pf_count_occupied(const uint64_t *tags, int64_t capacity, int64_t *out, void *stream) {
    const char *fn = "pf_count_occupied";
    if (!is_pow2(capacity)) return fail_arg(fn, "capacity must be a power of two >= 2");
    if (!tags || !out) return fail_arg(fn, "NULL pointer");
    int64_t blocks = (capacity + kThreads - 1) / kThreads;
    const int64_t cap_blocks = static_cast<int64_t>(sm_count()) * 8;
    if (blocks > cap_blocks) blocks = cap_blocks;
    count_occupied_kernel<<<static_cast<unsigned>(blocks), kThreads, 0, as_stream(stream)>>>(
        tags, capacity, out);
    return check_launch(fn);
}

}  // extern "C"
