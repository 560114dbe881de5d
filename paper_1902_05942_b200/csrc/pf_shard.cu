// Key-sharded multi-GPU frame: each rank owns a contiguous slice of
// the global tables' home slots; vertices are pre-aggregated per distinct key on the
// rank that traced them, shipped to the owner as records, and lookups go to the owner
// as deduplicated requests answered with the cell's effective (sum, count).
//
// The per-rank kernels here do everything but the exchanges, which the host runs as
// all-to-alls between them (NCCL over NVLink/NVSwitch; pipeline_sharded.py).  The
// results equal the single-GPU frame: every key's records reach the one rank that
// owns its home slot, fixed-point sums are exactly associative, and the resolve
// ladder consumes the same effective values in the same order (src/pipeline.py:152-283).
#include "pf_resolve.cuh"
#include "pf_sweep.cuh"
#include "pf_internal.cuh"

namespace pf {

namespace {

constexpr int kT = 256;
constexpr int kTW = kT / 32;
constexpr int kMaxWorld = 64;
constexpr int kWorkKeys = 28;  // 27 neighbourhood cells + the coarse cell
constexpr int kHomeBits = 29;
constexpr uint64_t kAggEmpty = ~0ull;

enum : int {
    kKindFineRecord = 0,
    kKindCoarseRecord = 1,
    kKindFineLookup = 2,
    kKindNeighbour = 3,
    kKindCoarseLookup = 4,
};

// Per-launch constants derived from pf_shard on the host.
struct ShardK {
    pf_shard s;
    int owner_shift;      // log2 C - log2 G
    uint64_t home_mask;   // C - 1
    uint64_t slice_base;  // rank * S
};

__device__ __forceinline__ uint64_t agg_key(int kind, uint64_t home, uint32_t fp) {
    return (static_cast<uint64_t>(kind) << 61) | (home << 32) | static_cast<uint64_t>(fp);
}
__device__ __forceinline__ int key_kind(uint64_t k) { return static_cast<int>(k >> 61); }
__device__ __forceinline__ uint64_t key_home(uint64_t k) {
    return (k >> 32) & ((1ull << kHomeBits) - 1);
}
__device__ __forceinline__ uint32_t key_fp(uint64_t k) { return static_cast<uint32_t>(k); }
__device__ __forceinline__ int key_group(int kind) { return kind <= kKindCoarseRecord ? 0 : 1; }

// Per-CTA claim counters per (group, owner), flushed once per CTA.
struct OwnerCounts {
    unsigned c[2][kMaxWorld];
};

__device__ __forceinline__ void owner_init(OwnerCounts &oc, int world) {
    for (int k = threadIdx.x; k < 2 * world; k += blockDim.x) oc.c[k / world][k % world] = 0;
}

__device__ __forceinline__ void owner_flush(const OwnerCounts &oc, const ShardK &k) {
    const int world = k.s.world;
    for (int j = threadIdx.x; j < 2 * world; j += blockDim.x) {
        const unsigned v = oc.c[j / world][j % world];
        if (v)
            atomicAdd(reinterpret_cast<unsigned long long *>(k.s.owner_counts + j),
                      static_cast<unsigned long long>(v));
    }
}

// Warp-merged insert into the aggregation table.  Lanes with equal keys merge; the
// leader finds or claims the key's slot (linear probing from mix64(key); a claim
// first reserves a distinct-list entry so the table never passes half full) and, for
// records, adds the group's summed values and weight.  Returns the slot to every lane
// of the group, -1 when the round overflowed.
template <bool VALUES, bool FIXED>
__device__ __forceinline__ int64_t warp_agg_insert(const ShardK &k, OwnerCounts &oc, bool valid,
                                                   uint64_t key, int64_t qsum[3], double fsum[3],
                                                   uint64_t weight) {
    const unsigned lane = threadIdx.x & 31u;
    const unsigned peers = __match_any_sync(kFull, valid ? key : kAggEmpty);
    const int leader = __ffs(peers) - 1;
    const bool is_leader = valid && static_cast<int>(lane) == leader;
    if (VALUES) {
        if (!valid) weight = 0;
        // group totals by pointer jumping (as warp_insert_sums)
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
            const unsigned long long w = __shfl_sync(kFull, static_cast<unsigned long long>(weight), src);
            if (nxt >= 0) weight += w;
            if (nxt >= 0) nxt = nn;
        }
    }
    long long slot = -1;
    if (is_leader) {
        const pf_shard &s = k.s;
        const uint64_t mask = static_cast<uint64_t>(s.agg_capacity) - 1;
        const unsigned long long limit = static_cast<unsigned long long>(s.agg_capacity / 2);
        uint64_t p = mix64(key) & mask;
        for (;;) {
            const uint64_t cur = ld_relaxed(s.agg_keys + p);
            if (cur == key) {
                slot = static_cast<long long>(p);
                break;
            }
            if (cur == kAggEmpty) {
                const unsigned long long d =
                    atomicAdd(reinterpret_cast<unsigned long long *>(s.n_distinct), 1ull);
                if (d >= limit) {
                    atomicExch(s.overflow, 1);
                    break;
                }
                const unsigned long long prev = atomicCAS(
                    reinterpret_cast<unsigned long long *>(s.agg_keys + p), kAggEmpty, key);
                if (prev == kAggEmpty) {
                    slot = static_cast<long long>(p);
                    s.distinct[d] = static_cast<int32_t>(p);
                    const int owner = static_cast<int>(key_home(key) >> k.owner_shift);
                    atomicAdd(&oc.c[key_group(key_kind(key))][owner], 1u);
                    break;
                }
                s.distinct[d] = -1;  // lost the race for this slot: leave a hole
                if (prev == key) {
                    slot = static_cast<long long>(p);
                    break;
                }
            }
            p = (p + 1) & mask;
        }
        if (VALUES && slot >= 0) {
            const uint64_t keep = l2_evict_last();
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                if (FIXED)
                    red_add_u64(s.agg_sums + 3 * slot + c, static_cast<uint64_t>(qsum[c]), keep);
                else
                    red_add_f64(reinterpret_cast<double *>(s.agg_sums) + 3 * slot + c, fsum[c], keep);
            }
            red_add_u64(s.agg_counts + slot, weight, keep);
        }
    }
    return __shfl_sync(kFull, slot, leader);
}

// ------------------------------------------------------------------ round 1 keys

template <bool FIXED>
__global__ void __launch_bounds__(kT, 2)
shard_keys_kernel(pf_config cfg, pf_vertices v, ShardK k, int has_coarse, uint64_t h0,
                  uint64_t h0_lookup, const int32_t *abort_flag) {
    __shared__ OwnerCounts oc;
    __shared__ double2 sincos_tab[220];
    if (abort_flag != nullptr && *abort_flag != 0) return;
    owner_init(oc, k.s.world);
    stage_sincos_table(sincos_tab);
    __syncthreads();
    const int64_t tiles = (v.n + kT - 1) / kT;
    for (int64_t tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
        const int64_t i0 = tile * kT + threadIdx.x;
        const bool valid = i0 < v.n;
        const int64_t i = valid ? i0 : v.n - 1;
        const uint64_t stream = l2_evict_first();
        const VertexIn x = load_vertex(v, i, cfg, stream);
        int64_t q[3];
        double f[3];
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            const double val = ld_stream(v.contribution + 3 * i + c, stream);
            if (FIXED) q[c] = quantize_fixed(val);
            else f[c] = val;
        }
        const KeyShared ks = key_shared(cfg, x);
        double du = 0.0, dv = 0.0;
#pragma unroll 1
        for (int set = 0; set < 3; ++set) {
            if (set == 1 && !has_coarse) continue;
            if (set != 1 && cfg.jitter) {  // the coarse set reuses the fine set's offsets
                double u1, u2;
                jitter_draws(set == 0 ? h0 : h0_lookup, x.pixel, x.sample, u1, u2);
                disc_offset(u1, u2, du, dv, sincos_tab);
            }
            double jt[3];
            const CellHash h = key_hash(
                make_key(cfg, x, ks, cfg.jitter, du, dv, set == 1 ? cfg.coarse_delta : 0, jt), ks);
            const uint64_t key = agg_key(set, h.index & k.home_mask, h.fp);
            if (set < 2) {
                int64_t qs[3] = {q[0], q[1], q[2]};
                double fs[3] = {f[0], f[1], f[2]};
                warp_agg_insert<true, FIXED>(k, oc, valid, key, qs, fs, 1);
            } else {
                const int64_t slot = warp_agg_insert<false, FIXED>(k, oc, valid, key, nullptr,
                                                                   nullptr, 0);
                if (valid) k.s.vertex_slot[i] = static_cast<int32_t>(slot);
            }
        }
    }
    __syncthreads();
    owner_flush(oc, k);
}

// ------------------------------------------------------------------ emit

__global__ void __launch_bounds__(kT)
shard_emit_kernel(ShardK k, int64_t *send_rec, uint64_t *send_req) {
    __shared__ int64_t base[2][kMaxWorld];
    const pf_shard &s = k.s;
    if (*s.overflow != 0) return;
    const int world = s.world;
    if (threadIdx.x < 2 * world) {
        const int g = threadIdx.x / world, o = threadIdx.x % world;
        int64_t b = 0;
        for (int j = 0; j < o; ++j) b += s.owner_counts[g * world + j];
        base[g][o] = b;
    }
    __syncthreads();
    const int64_t limit = s.agg_capacity / 2;
    const int64_t nd = *s.n_distinct < limit ? *s.n_distinct : limit;
    const int lane = threadIdx.x & 31;
    const int64_t span = (nd + 31) / 32 * 32;  // whole warps take part in the shuffles
    for (int64_t d = static_cast<int64_t>(blockIdx.x) * kT + threadIdx.x; d < span;
         d += static_cast<int64_t>(gridDim.x) * kT) {
        const int32_t slot = d < nd ? s.distinct[d] : -1;
        const bool valid = slot >= 0;
        const uint64_t key = valid ? s.agg_keys[slot] : kAggEmpty;
        const int kind = key_kind(key);
        const int group = key_group(kind);
        const int owner = static_cast<int>(key_home(key) >> k.owner_shift);
        const int gid = valid ? group * world + owner : -1;
        const unsigned peers = __match_any_sync(kFull, gid);
        const int leader = __ffs(peers) - 1;
        unsigned long long b = 0;
        if (valid && lane == leader)
            b = atomicAdd(reinterpret_cast<unsigned long long *>(s.owner_cursor + gid),
                          static_cast<unsigned long long>(__popc(peers)));
        b = __shfl_sync(kFull, b, leader);
        if (!valid) continue;
        const int64_t pos = base[group][owner] + static_cast<int64_t>(b) +
                            __popc(peers & ((1u << lane) - 1u));
        if (group == 0) {
            int64_t *r = send_rec + 5 * pos;
            r[0] = static_cast<int64_t>(key);
            r[1] = s.agg_sums[3 * slot + 0];
            r[2] = s.agg_sums[3 * slot + 1];
            r[3] = s.agg_sums[3 * slot + 2];
            r[4] = s.agg_counts[slot];
        } else {
            send_req[pos] = key;
            s.agg_counts[slot] = pos;
        }
    }
}

// ------------------------------------------------------------------ owner side

__device__ __forceinline__ uint64_t local_index(const ShardK &k, uint64_t home) {
    return home - k.slice_base;
}

template <bool FIXED>
__global__ void __launch_bounds__(kT)
shard_apply_kernel(ShardK k, pf_table fine, pf_table coarse, int has_coarse, const int64_t *rec,
                   int64_t n, int64_t frame, int64_t *stats) {
    __shared__ BlockStats bs;
    stats_init(bs);
    __syncthreads();
    const int64_t tiles = (n + kT - 1) / kT;
    for (int64_t tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
        const int64_t j = tile * kT + threadIdx.x;
        const bool valid = j < n;
        const int64_t *r = rec + 5 * (valid ? j : 0);
        const uint64_t key = valid ? static_cast<uint64_t>(r[0]) : 0ull;
        const uint64_t idx = local_index(k, key_home(key));
        const uint32_t fp = key_fp(key);
        const int kind = key_kind(key);
        const uint64_t weight = valid ? static_cast<uint64_t>(r[4]) : 0ull;
#pragma unroll
        for (int tb = 0; tb < 2; ++tb) {
            if (tb == 1 && !has_coarse) break;
            const pf_table &t = tb == 0 ? fine : coarse;
            const bool mine = valid && kind == tb;
            int64_t qs[3];
            double fs[3];
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                const int64_t w = mine ? r[1 + c] : 0;
                qs[c] = w;
                fs[c] = __longlong_as_double(w);
            }
            const uint64_t home_tag =
                mine ? ld_relaxed(t.tags + (idx & static_cast<uint64_t>(t.capacity - 1))) : 0ull;
            const LaneInsert res = warp_insert_sums<FIXED, true>(t, mine, idx, fp, qs, fs, weight,
                                                                 frame, home_tag);
            const unsigned wt = static_cast<unsigned>(weight);
            if (mine && res.status == 2)
                atomicAdd(&bs.v[tb == 0 ? PF_STAT_PROBE_FAILURES : PF_STAT_COARSE_PROBE_FAILURES], wt);
            warp_count(bs, tb == 0 ? PF_STAT_EVICTIONS : PF_STAT_COARSE_EVICTIONS,
                       mine && res.leader && res.status == 1);
            if (tb == 0 && mine) {
                atomicAdd(&bs.hist[res.probe_len & 255], wt);
                atomicAdd(&bs.v[PF_STAT_PROBE_LEN_SUM], wt * static_cast<unsigned>(res.probe_len));
            }
        }
        warp_count(bs, PF_STAT_SHARD_RECORDS, valid);
    }
    __syncthreads();
    stats_flush(bs, stats, true);
}

__global__ void __launch_bounds__(kT)
shard_answer_kernel(ShardK k, pf_config cfg, pf_table fine, pf_table coarse, int has_coarse,
                    const uint64_t *req, int64_t n, ulonglong4 *ans, int64_t *stats) {
    const int64_t j = static_cast<int64_t>(blockIdx.x) * kT + threadIdx.x;
    if (j == 0) atomicAdd(reinterpret_cast<unsigned long long *>(stats + PF_STAT_SHARD_REQUESTS),
                          static_cast<unsigned long long>(n));
    if (j >= n) return;
    const uint64_t key = __ldg(reinterpret_cast<const unsigned long long *>(req) + j);
    const bool to_coarse = key_kind(key) == kKindCoarseLookup;
    ulonglong4 out = absent_record();
    if (!to_coarse || has_coarse) {
        const pf_table &t = to_coarse ? coarse : fine;
        const int64_t s = probe_lookup(t.tags, static_cast<uint64_t>(t.capacity) - 1, t.probe_limit,
                                       local_index(k, key_home(key)), key_fp(key));
        if (s >= 0)
            out = pack_effective(effective_at(t, s, cfg.temporal_mode, cfg.ema_alpha, cfg.delta_max),
                                 eff_is_int(t, cfg.temporal_mode));
    }
    ulonglong2 *o = reinterpret_cast<ulonglong2 *>(ans + j);
    o[0] = make_ulonglong2(out.x, out.y);
    o[1] = make_ulonglong2(out.z, out.w);
}

// ------------------------------------------------------------------ requester side

__device__ __forceinline__ bool as_int_mode(int sum_mode, int mode) {
    return mode == PF_INTEGRATE && sum_mode == PF_SUM_FIXED;
}

// The answer to the request held in aggregation slot `slot` (its send position was
// stored there by the emit kernel).
__device__ __forceinline__ ulonglong4 answer_of(const ShardK &k, const ulonglong4 *ans,
                                                int32_t slot) {
    if (slot < 0) return absent_record();
    const int64_t pos = __ldg(k.s.agg_counts + slot);
    return load_record(ans, pos);
}

__device__ __forceinline__ void composite_local(double *flat, int64_t n_pixels, int64_t pixel,
                                                const double *throughput, const double chosen[3],
                                                BlockStats &bs, bool count_bad) {
    const uint64_t stream = l2_evict_first(), keep = l2_evict_last();
    if (pixel >= 0 && pixel < n_pixels) {
#pragma unroll
        for (int c = 0; c < 3; ++c)
            red_add_f64(flat + 3 * pixel + c, dmul(ld_stream(throughput + c, stream), chosen[c]), keep);
    } else if (count_bad) {
        atomicAdd(&bs.v[PF_STAT_BAD_PIXELS], 1u);
    }
}

__global__ void __launch_bounds__(kT)
shard_resolve_kernel(ShardK k, pf_config cfg, pf_vertices v, const ulonglong4 *ans, double *flat,
                     int64_t n_pixels, double thr, int64_t *work, int64_t *work_count,
                     uint8_t *source, double *chosen, int64_t *stats) {
    __shared__ BlockStats bs;
    stats_init(bs);
    __syncthreads();
    const int mode = cfg.temporal_mode;
    const bool as_int = as_int_mode(k.s.sum_mode, mode);
    const bool fixed = k.s.sum_mode == PF_SUM_FIXED;
    const int lane = threadIdx.x & 31;
    const uint64_t stream = l2_evict_first();
    const int64_t tiles = (v.n + kT - 1) / kT;
    for (int64_t tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
        const int64_t i0 = tile * kT + threadIdx.x;
        const bool valid = i0 < v.n;
        const int64_t i = valid ? i0 : v.n - 1;
        const ulonglong4 rec = answer_of(k, ans, k.s.vertex_slot[i]);
        const bool found = rec.w != kAbsentCount;
        const Effective e = unpack_effective(rec, as_int);
        const bool fine_ok = valid && found && e.fcnt >= thr;
        if (fine_ok) {
            double m[3];
#pragma unroll
            for (int c = 0; c < 3; ++c) m[c] = row_mean(eff_sum_f64(e, as_int, c), e.fcnt, fixed);
            const int64_t pixel = ld_stream(v.pixel + i, stream) - k.s.pixel_base;
            composite_local(flat, n_pixels, pixel, v.throughput + 3 * i, m, bs, true);
            if (source) source[i] = 0;
            if (chosen) {
#pragma unroll
                for (int c = 0; c < 3; ++c) chosen[3 * i + c] = m[c];
            }
        }
        const bool need = valid && !fine_ok;
        const unsigned mk = __ballot_sync(kFull, need);
        if (mk) {
            unsigned long long wb = 0;
            if (lane == __ffs(mk) - 1)
                wb = atomicAdd(reinterpret_cast<unsigned long long *>(work_count),
                               static_cast<unsigned long long>(__popc(mk)));
            wb = __shfl_sync(kFull, wb, __ffs(mk) - 1);
            if (need) work[static_cast<int64_t>(wb) + __popc(mk & ((1u << lane) - 1u))] = i;
        }
        warp_count(bs, PF_STAT_SOURCE_FINE, fine_ok);
        warp_count(bs, PF_STAT_FALLBACK_ROWS, need);
    }
    __syncthreads();
    stats_flush(bs, stats, false);
}

// Each work row's lookup key (stream 3) and coarse hash, one row per thread (the FP64
// key recipe SIMT-wide); record: q0, q1, q2, level, aux, coarse index, coarse fp, 0.
__global__ void __launch_bounds__(kT)
shard_row_keys_kernel(pf_config cfg, pf_vertices v, ShardK k, int has_coarse, uint64_t h0_lookup,
                      uint64_t h0_coarse, const int64_t *work, const int64_t *work_count) {
    __shared__ double2 sincos_tab[220];
    stage_sincos_table(sincos_tab);
    __syncthreads();
    const int64_t n_work = *work_count;
    for (int64_t w = static_cast<int64_t>(blockIdx.x) * kT + threadIdx.x; w < n_work;
         w += static_cast<int64_t>(gridDim.x) * kT) {
        const int64_t row = work[w];
        const VertexIn x = load_vertex(v, row, cfg);
        const KeyShared ks = key_shared(cfg, x);
        double du = 0.0, dv = 0.0, cdu = 0.0, cdv = 0.0;
        if (cfg.jitter) {  // the coarse key shares the lookup draws when jitter is on
            double u1, u2;
            jitter_draws(h0_lookup, x.pixel, x.sample, u1, u2);
            disc_offset(u1, u2, du, dv, sincos_tab);
            cdu = du;
            cdv = dv;
            if (h0_coarse != h0_lookup) {
                jitter_draws(h0_coarse, x.pixel, x.sample, u1, u2);
                disc_offset(u1, u2, cdu, cdv, sincos_tab);
            }
        }
        double jt[3];
        const CellKey lk = make_key(cfg, x, ks, cfg.jitter, du, dv, 0, jt);
        CellHash hc{0ull, 0u};
        if (has_coarse)
            hc = key_hash(make_key(cfg, x, ks, cfg.jitter, cdu, cdv, cfg.coarse_delta, jt), ks);
        longlong4 *o = reinterpret_cast<longlong4 *>(k.s.row_keys + 8 * w);
        o[0] = make_longlong4(lk.q[0], lk.q[1], lk.q[2], lk.level);
        o[1] = make_longlong4(static_cast<long long>(lk.aux), static_cast<long long>(hc.index),
                              static_cast<long long>(hc.fp), 0);
    }
}

// One work row per warp: lanes 0..26 hash the neighbourhood cells of the row's lookup key
// (shard_row_keys_kernel) and lane 27 carries the coarse cell; all 28 go into the
// aggregation table as deduplicated requests.
__global__ void __launch_bounds__(kT)
shard_fallback_keys_kernel(pf_config cfg, pf_vertices v, ShardK k, int has_coarse,
                           uint64_t h0_lookup, uint64_t h0_coarse, const int64_t *work,
                           const int64_t *work_count) {
    __shared__ OwnerCounts oc;
    owner_init(oc, k.s.world);
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int64_t n_work = *work_count;
    const int64_t nwarps = static_cast<int64_t>(gridDim.x) * kTW;
    for (int64_t w = static_cast<int64_t>(blockIdx.x) * kTW + (threadIdx.x >> 5); w < n_work;
         w += nwarps) {
        const long long rec = lane < 8 ? k.s.row_keys[8 * w + lane] : 0;
        const long long q0 = __shfl_sync(kFull, rec, 0);
        const long long q1 = __shfl_sync(kFull, rec, 1);
        const long long q2 = __shfl_sync(kFull, rec, 2);
        const long long lev = __shfl_sync(kFull, rec, 3);
        const unsigned long long aux = static_cast<unsigned long long>(__shfl_sync(kFull, rec, 4));
        const unsigned long long cidx = static_cast<unsigned long long>(__shfl_sync(kFull, rec, 5));
        const unsigned cfp = static_cast<unsigned>(__shfl_sync(kFull, rec, 6));
        uint64_t key = kAggEmpty;
        bool valid = false;
        if (lane < 27) {
            const CellHash h = cell_hash(q0 + neighbour_dx(lane), q1 + neighbour_dy(lane),
                                         q2 + neighbour_dz(lane), lev, aux, 0, 0u);
            key = agg_key(kKindNeighbour, h.index & k.home_mask, h.fp);
            valid = true;
        } else if (lane == 27 && has_coarse) {
            key = agg_key(kKindCoarseLookup, cidx & k.home_mask, cfp);
            valid = true;
        }
        const int64_t slot = warp_agg_insert<false, true>(k, oc, valid, key, nullptr, nullptr, 0);
        if (lane < kWorkKeys) k.s.work_slot[w * kWorkKeys + lane] = valid ? static_cast<int32_t>(slot) : -1;
    }
    __syncthreads();
    owner_flush(oc, k);
}

__global__ void __launch_bounds__(kT)
shard_ladder_kernel(ShardK k, pf_config cfg, pf_vertices v, int has_coarse, const ulonglong4 *ans,
                    const int64_t *work, const int64_t *work_count, double *flat, int64_t n_pixels,
                    double thr, uint8_t *source, double *chosen, int64_t *stats) {
    __shared__ BlockStats bs;
    stats_init(bs);
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int mode = cfg.temporal_mode;
    const bool as_int = as_int_mode(k.s.sum_mode, mode);
    const bool fixed = k.s.sum_mode == PF_SUM_FIXED;
    const int64_t n_work = *work_count;
    const int64_t nwarps = static_cast<int64_t>(gridDim.x) * kTW;
    for (int64_t w = static_cast<int64_t>(blockIdx.x) * kTW + (threadIdx.x >> 5); w < n_work;
         w += nwarps) {
        const int64_t row = work[w];
        bool found = false;
        Effective e{};
        if (lane < 27) {
            const ulonglong4 rec = answer_of(k, ans, k.s.work_slot[w * kWorkKeys + lane]);
            found = rec.w != kAbsentCount;
            if (found) e = unpack_effective(rec, as_int);
        }
        const Pool pool = pool_neighbours(found, e, as_int, mode);
        if (lane == 0) {
            bool coarse_found = false;
            Effective ce{};
            if (has_coarse) {
                const ulonglong4 rec = answer_of(k, ans, k.s.work_slot[w * kWorkKeys + 27]);
                coarse_found = rec.w != kAbsentCount;
                if (coarse_found) ce = unpack_effective(rec, as_int);
            }
            double contrib[3], ch[3];
#pragma unroll
            for (int c = 0; c < 3; ++c) contrib[c] = __ldg(v.contribution + 3 * row + c);
            const int src = ladder_choose(pool, as_int, mode, fixed, thr, coarse_found, ce, as_int,
                                          contrib, ch);
            const int64_t pixel = __ldg(v.pixel + row) - k.s.pixel_base;
            composite_local(flat, n_pixels, pixel, v.throughput + 3 * row, ch, bs, true);
            if (source) source[row] = static_cast<uint8_t>(src);
            if (chosen) {
#pragma unroll
                for (int c = 0; c < 3; ++c) chosen[3 * row + c] = ch[c];
            }
            atomicAdd(&bs.v[PF_STAT_SOURCE_FINE + src], 1u);
        }
        __syncwarp();
    }
    __syncthreads();
    stats_flush(bs, stats, false);
}

__global__ void __launch_bounds__(kT) shard_reset_kernel(ShardK k) {
    const pf_shard &s = k.s;
    const int64_t limit = s.agg_capacity / 2;
    const int64_t nd = *s.n_distinct < limit ? *s.n_distinct : limit;
    for (int64_t d = static_cast<int64_t>(blockIdx.x) * kT + threadIdx.x; d < nd;
         d += static_cast<int64_t>(gridDim.x) * kT) {
        const int32_t slot = s.distinct[d];
        if (slot < 0) continue;
        s.agg_keys[slot] = kAggEmpty;
        s.agg_sums[3 * slot + 0] = 0;
        s.agg_sums[3 * slot + 1] = 0;
        s.agg_sums[3 * slot + 2] = 0;
        s.agg_counts[slot] = 0;
    }
}

// ------------------------------------------------------------------ host helpers

int prepare_shard(const char *fn, const pf_shard *sh, ShardK *out) {
    if (sh == nullptr) return fail_arg(fn, "shard is NULL");
    const int g = sh->world;
    if (g < 1 || g > kMaxWorld || (g & (g - 1)) != 0)
        return fail_arg(fn, "world must be a power of two <= 64");
    if (sh->rank < 0 || sh->rank >= g) return fail_arg(fn, "rank out of range");
    int lg = 0;
    while ((1 << lg) < g) ++lg;
    if (sh->log2_capacity < lg || sh->log2_capacity < 1 || sh->log2_capacity > kHomeBits)
        return fail_arg(fn, "log2_capacity must satisfy world <= C <= 2^29");
    if (!is_pow2(sh->agg_capacity) || sh->agg_capacity < 64 || sh->agg_capacity > (1ll << 31))
        return fail_arg(fn, "agg_capacity must be a power of two in [64, 2^31]");
    if (!sh->agg_keys || !sh->agg_sums || !sh->agg_counts || !sh->distinct || !sh->n_distinct ||
        !sh->overflow || !sh->owner_counts || !sh->owner_cursor)
        return fail_arg(fn, "shard buffer is NULL");
    if (sh->sum_mode != PF_SUM_FIXED && sh->sum_mode != PF_SUM_FLOAT)
        return fail_arg(fn, "unknown sum_mode");
    out->s = *sh;
    out->owner_shift = sh->log2_capacity - lg;
    out->home_mask = (1ull << sh->log2_capacity) - 1;
    out->slice_base = static_cast<uint64_t>(sh->rank) << out->owner_shift;
    return PF_OK;
}

// The local slice table: capacity C for one rank, 2S otherwise (see the header).
int check_slice(const char *fn, const ShardK &k, const pf_table *t) {
    if (int rc = validate_table(fn, t)) return rc;
    const int64_t c = 1ll << k.s.log2_capacity;
    const int64_t want = k.s.world == 1 ? c : 2 * (c / k.s.world);
    if (t->capacity != want) return fail_arg(fn, "local table capacity must be C (world 1) or 2C/world");
    if (t->sum_mode != k.s.sum_mode) return fail_arg(fn, "table sum_mode differs from the shard's");
    if (k.s.world > 1 && t->probe_limit > c / k.s.world)
        return fail_arg(fn, "probe_limit exceeds the slice size");
    return PF_OK;
}

template <typename K>
int grid_for(K kernel, int64_t n, int per_sm_cap) {
    int b = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kernel, kT, 0) != cudaSuccess || b < 1) b = 1;
    if (b > per_sm_cap) b = per_sm_cap;
    const int64_t tiles = (n + kT - 1) / kT;
    const int64_t cap = static_cast<int64_t>(sm_count()) * b;
    return static_cast<int>(tiles < cap ? (tiles > 0 ? tiles : 1) : cap);
}

}  // namespace

}  // namespace pf

using namespace pf;

extern "C" {

int pf_shard_keys(const pf_config *cfg, const pf_vertices *v, const pf_shard *sh,
                  int32_t has_coarse, uint64_t stream_base_accum, uint64_t stream_base_lookup,
                  const int32_t *abort_flag, void *stream) {
    const char *fn = "pf_shard_keys";
    ShardK k;
    if (int rc = prepare_shard(fn, sh, &k)) return rc;
    if (int rc = validate_vertices(fn, v, cfg)) return rc;
    pf_config kc;
    if (int rc = prepare_config(fn, cfg, &kc)) return rc;
    if (v->n == 0) return PF_OK;
    if (!v->contribution || !sh->vertex_slot) return fail_arg(fn, "contribution/vertex_slot is NULL");
    cudaStream_t st = as_stream(stream);
    if (sh->sum_mode == PF_SUM_FIXED)
        shard_keys_kernel<true><<<grid_for(shard_keys_kernel<true>, v->n, 8), kT, 0, st>>>(
            kc, *v, k, has_coarse != 0, stream_base_accum, stream_base_lookup, abort_flag);
    else
        shard_keys_kernel<false><<<grid_for(shard_keys_kernel<false>, v->n, 8), kT, 0, st>>>(
            kc, *v, k, has_coarse != 0, stream_base_accum, stream_base_lookup, abort_flag);
    return check_launch(fn);
}

int pf_shard_emit(const pf_shard *sh, int64_t *send_records, uint64_t *send_requests,
                  void *stream) {
    const char *fn = "pf_shard_emit";
    ShardK k;
    if (int rc = prepare_shard(fn, sh, &k)) return rc;
    if (!send_records || !send_requests) return fail_arg(fn, "send buffers are NULL");
    cudaStream_t st = as_stream(stream);
    if (cudaMemsetAsync(sh->owner_cursor, 0, sizeof(int64_t) * 2 * sh->world, st) != cudaSuccess)
        return check_launch(fn);
    const int blocks = sweep_blocks<kT>(sh->agg_capacity / 2, sm_count());
    shard_emit_kernel<<<blocks, kT, 0, st>>>(k, send_records, send_requests);
    return check_launch(fn);
}

int pf_shard_apply(const pf_shard *sh, const pf_table *fine, const pf_table *coarse,
                   const int64_t *records, int64_t n_records, int64_t frame, int64_t *stats,
                   void *stream) {
    const char *fn = "pf_shard_apply";
    ShardK k;
    if (int rc = prepare_shard(fn, sh, &k)) return rc;
    if (int rc = check_slice(fn, k, fine)) return rc;
    if (coarse)
        if (int rc = check_slice(fn, k, coarse)) return rc;
    if (!stats) return fail_arg(fn, "stats is NULL");
    if (n_records < 0) return fail_arg(fn, "negative record count");
    if (n_records == 0) return PF_OK;
    if (!records) return fail_arg(fn, "records is NULL");
    const pf_table c = coarse ? *coarse : *fine;
    cudaStream_t st = as_stream(stream);
    if (sh->sum_mode == PF_SUM_FIXED)
        shard_apply_kernel<true><<<grid_for(shard_apply_kernel<true>, n_records, 8), kT, 0, st>>>(
            k, *fine, c, coarse != nullptr, records, n_records, frame, stats);
    else
        shard_apply_kernel<false><<<grid_for(shard_apply_kernel<false>, n_records, 8), kT, 0, st>>>(
            k, *fine, c, coarse != nullptr, records, n_records, frame, stats);
    return check_launch(fn);
}

int pf_shard_answer(const pf_shard *sh, const pf_config *cfg, const pf_table *fine,
                    const pf_table *coarse, const uint64_t *requests, int64_t n_requests,
                    uint64_t *answers, int64_t *stats, void *stream) {
    const char *fn = "pf_shard_answer";
    ShardK k;
    if (int rc = prepare_shard(fn, sh, &k)) return rc;
    if (cfg == nullptr) return fail_arg(fn, "config is NULL");
    if (int rc = check_slice(fn, k, fine)) return rc;
    if (coarse)
        if (int rc = check_slice(fn, k, coarse)) return rc;
    if (!stats) return fail_arg(fn, "stats is NULL");
    if (n_requests < 0) return fail_arg(fn, "negative request count");
    if (n_requests == 0) return PF_OK;
    if (!requests || !answers) return fail_arg(fn, "requests/answers is NULL");
    shard_answer_kernel<<<blocks_for(n_requests, kT), kT, 0, as_stream(stream)>>>(
        k, *cfg, *fine, coarse ? *coarse : *fine, coarse != nullptr, requests, n_requests,
        reinterpret_cast<ulonglong4 *>(answers), stats);
    return check_launch(fn);
}

int pf_shard_resolve(const pf_shard *sh, const pf_config *cfg, const pf_vertices *v,
                     const uint64_t *answers, double *flat, int64_t n_pixels, int64_t *work,
                     int64_t *work_count, uint8_t *source, double *chosen, int64_t *stats,
                     void *stream) {
    const char *fn = "pf_shard_resolve";
    ShardK k;
    if (int rc = prepare_shard(fn, sh, &k)) return rc;
    if (int rc = validate_vertices(fn, v, cfg)) return rc;
    if (!flat || !work || !work_count || !stats || n_pixels < 0)
        return fail_arg(fn, "flat/work/work_count/stats is NULL");
    if (v->n == 0) return PF_OK;
    if (!v->throughput || !sh->vertex_slot) return fail_arg(fn, "throughput/vertex_slot is NULL");
    if (!answers) return fail_arg(fn, "answers is NULL");
    const double thr = static_cast<double>(cfg->low_count_threshold > 1 ? cfg->low_count_threshold : 1);
    shard_resolve_kernel<<<grid_for(shard_resolve_kernel, v->n, 8), kT, 0, as_stream(stream)>>>(
        k, *cfg, *v, reinterpret_cast<const ulonglong4 *>(answers), flat, n_pixels, thr, work,
        work_count, source, chosen, stats);
    return check_launch(fn);
}

int pf_shard_fallback_keys(const pf_config *cfg, const pf_vertices *v, const pf_shard *sh,
                           int32_t has_coarse, uint64_t stream_base_lookup,
                           uint64_t stream_base_coarse, const int64_t *work,
                           const int64_t *work_count, void *stream) {
    const char *fn = "pf_shard_fallback_keys";
    ShardK k;
    if (int rc = prepare_shard(fn, sh, &k)) return rc;
    if (int rc = validate_vertices(fn, v, cfg)) return rc;
    pf_config kc;
    if (int rc = prepare_config(fn, cfg, &kc)) return rc;
    if (v->n == 0) return PF_OK;
    if (!work || !work_count || !sh->work_slot || !sh->row_keys)
        return fail_arg(fn, "work/work_slot/row_keys is NULL");
    int64_t kb = (v->n + kT - 1) / kT;
    const int64_t kcap = static_cast<int64_t>(sm_count()) * 4;
    if (kb > kcap) kb = kcap;
    shard_row_keys_kernel<<<static_cast<unsigned>(kb), kT, 0, as_stream(stream)>>>(
        kc, *v, k, has_coarse != 0, stream_base_lookup, stream_base_coarse, work, work_count);
    if (int rc = check_launch(fn)) return rc;
    int64_t blocks = (v->n + kTW - 1) / kTW;
    const int64_t cap = static_cast<int64_t>(sm_count()) * 8;
    if (blocks > cap) blocks = cap;
    shard_fallback_keys_kernel<<<static_cast<unsigned>(blocks), kT, 0, as_stream(stream)>>>(
        kc, *v, k, has_coarse != 0, stream_base_lookup, stream_base_coarse, work, work_count);
    return check_launch(fn);
}

int pf_shard_ladder(const pf_shard *sh, const pf_config *cfg, const pf_vertices *v,
                    int32_t has_coarse, const uint64_t *answers, const int64_t *work,
                    const int64_t *work_count, double *flat, int64_t n_pixels, uint8_t *source,
                    double *chosen, int64_t *stats, void *stream) {
    const char *fn = "pf_shard_ladder";
    ShardK k;
    if (int rc = prepare_shard(fn, sh, &k)) return rc;
    if (int rc = validate_vertices(fn, v, cfg)) return rc;
    if (!flat || !work || !work_count || !stats || n_pixels < 0)
        return fail_arg(fn, "flat/work/work_count/stats is NULL");
    if (v->n == 0) return PF_OK;
    if (!v->throughput || !v->contribution || !sh->work_slot || !answers)
        return fail_arg(fn, "throughput/contribution/work_slot/answers is NULL");
    const double thr = static_cast<double>(cfg->low_count_threshold > 1 ? cfg->low_count_threshold : 1);
    int64_t blocks = (v->n + kTW - 1) / kTW;
    const int64_t cap = static_cast<int64_t>(sm_count()) * 8;
    if (blocks > cap) blocks = cap;
    shard_ladder_kernel<<<static_cast<unsigned>(blocks), kT, 0, as_stream(stream)>>>(
        k, *cfg, *v, has_coarse != 0, reinterpret_cast<const ulonglong4 *>(answers), work,
        work_count, flat, n_pixels, thr, source, chosen, stats);
    return check_launch(fn);
}

int pf_shard_reset(const pf_shard *sh, void *stream) {
    const char *fn = "pf_shard_reset";
    ShardK k;
    if (int rc = prepare_shard(fn, sh, &k)) return rc;
    cudaStream_t st = as_stream(stream);
    shard_reset_kernel<<<sweep_blocks<kT>(sh->agg_capacity / 2, sm_count()), kT, 0, st>>>(k);
    if (int rc = check_launch(fn)) return rc;
    if (cudaMemsetAsync(sh->n_distinct, 0, sizeof(int64_t), st) != cudaSuccess ||
        cudaMemsetAsync(sh->overflow, 0, sizeof(int32_t), st) != cudaSuccess ||
        cudaMemsetAsync(sh->owner_counts, 0, sizeof(int64_t) * 2 * sh->world, st) != cudaSuccess)
        return check_launch(fn);
    return PF_OK;
}

}  // extern "C"
