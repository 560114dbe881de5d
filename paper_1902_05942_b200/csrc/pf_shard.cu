// Key-sharded multi-GPU frame: each rank owns a contiguous slice of
// the global tables' home slots.  Inserts: vertices are pre-aggregated per distinct key
// on the rank that traced them and shipped to the owner as records (one all-to-all).
// Queries: after the inserts every owner publishes its occupied cells' effective
// (sum, count) records, the ranks all-gather them into a read-only replica of the whole
// global table (a few MB: ~4 % of the slots are occupied), and each rank resolves its
// own vertices against the replica with the single-GPU resolve kernels
// (pf_resolve_replica) -- no per-lookup round trips.
//
// The host runs the collectives between the kernels (sharded.py).  Results equal the
// single-GPU frame: each key's records reach exactly one owner, 16.16 fixed-point sums
// are exactly associative, and the replica holds the owners' cells verbatim
// (src/pipeline.py:152-283).
#include "pf_resolve.cuh"
#include "pf_sweep.cuh"
#include "pf_internal.cuh"

namespace pf {

namespace {

constexpr int kT = 256;
constexpr int kMaxWorld = 64;
constexpr int kHomeBits = 29;
constexpr uint64_t kAggEmpty = ~0ull;

enum : int {
    kKindFineRecord = 0,
    kKindCoarseRecord = 1,
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
                                                   uint64_t weight, bool merge = true) {
    const unsigned lane = threadIdx.x & 31u;
    // merge == false: every lane adds its own key (equal keys racing for one empty slot
    // resolve through the claim CAS; the loser leaves a hole in the distinct list)
    const unsigned peers = merge ? __match_any_sync(kFull, valid ? key : kAggEmpty) : (1u << lane);
    const int leader = __ffs(peers) - 1;
    const bool is_leader = valid && static_cast<int>(lane) == leader;
    if (VALUES && merge) {
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
    return merge ? __shfl_sync(kFull, slot, leader) : slot;
}

// ------------------------------------------------------------------ round 1 keys

#ifndef PF_SHARD_MERGE
#define PF_SHARD_MERGE 1  // warp-merge equal keys before the aggregation table: without it racing
                          // duplicates leave holes that overflow the distinct list (regrows)
#endif

// 3 CTAs per SM (80 registers): per-rank frame 1.58-1.68 -> 1.45 ms at G = 2 and
// 1.50 -> 1.37 ms at G = 4 (tools/shard_sim.py); 4 CTAs or parking the frame and position
// in shared memory (PF_SHARD_PARK) measured the same.
#ifndef PF_SHARD_KEYS_MIN_BLOCKS
#define PF_SHARD_KEYS_MIN_BLOCKS 3
#endif
#ifndef PF_SHARD_PARK
#define PF_SHARD_PARK 0  // tangent frame and position wait in shared memory (as the fused insert)
#endif

template <bool FIXED>
__global__ void __launch_bounds__(kT, PF_SHARD_KEYS_MIN_BLOCKS)
shard_keys_kernel(const PF_GRID_CONST pf_config cfg, const PF_GRID_CONST pf_vertices v,
                  const PF_GRID_CONST ShardK k, int has_coarse, uint64_t h0,
                  uint64_t h0_lookup, const int32_t *abort_flag, uint64_t *lk_keys) {
    __shared__ OwnerCounts oc;
    __shared__ double2 sincos_tab[220];
    __shared__ double lod_dist[32];
    __shared__ double2 lvsteps[32];
#if PF_SHARD_PARK
    __shared__ double park[9][kT];  // t1, t2, position per thread
#endif
    if (abort_flag != nullptr && *abort_flag != 0) return;
    owner_init(oc, k.s.world);
    stage_sincos_table(sincos_tab);
    stage_lod_dist(lod_dist, cfg);
    stage_level_steps(lvsteps, cfg);
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
        const KeyShared ks = key_shared(cfg, x, lod_dist);
#if PF_SHARD_PARK
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            park[c][threadIdx.x] = ks.frame.t1[c];
            park[3 + c][threadIdx.x] = ks.frame.t2[c];
            park[6 + c][threadIdx.x] = x.pos[c];
        }
#endif
        const uint64_t pid = path_id(x.pixel, x.sample);
        double w[3] = {0.0, 0.0, 0.0};  // jitter direction u*t1 + v*t2
#pragma unroll 1
        for (int set = 0; set < 3; ++set) {
            if (set == 1 && !has_coarse) continue;
            if (set != 1 && cfg.jitter) {  // the coarse set reuses the fine set's offsets
                double u1, u2, du, dv;
                jitter_draws_pid(set == 0 ? h0 : h0_lookup, pid, u1, u2);
                disc_offset(u1, u2, du, dv, sincos_tab);
#if PF_SHARD_PARK
                double t1[3], t2[3];
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    t1[c] = park[c][threadIdx.x];
                    t2[c] = park[3 + c][threadIdx.x];
                }
                jitter_dir(du, dv, t1, t2, w);
#else
                jitter_dir(du, dv, ks.frame.t1, ks.frame.t2, w);
#endif
            }
            double jt[3];
#if PF_SHARD_PARK
            VertexIn xk = x;
#pragma unroll
            for (int c = 0; c < 3; ++c) xk.pos[c] = park[6 + c][threadIdx.x];
#else
            const VertexIn &xk = x;
#endif
            const CellHash h = key_hash(
                make_key_w(cfg, xk, ks, cfg.jitter, w, set == 1 ? cfg.coarse_delta : 0, jt,
                           lvsteps), ks);
            if (set < 2) {
                const uint64_t key = agg_key(set, h.index & k.home_mask, h.fp);
                int64_t qs[3] = {q[0], q[1], q[2]};
                double fs[3] = {f[0], f[1], f[2]};
                warp_agg_insert<true, FIXED>(k, oc, valid, key, qs, fs, 1, PF_SHARD_MERGE);
            } else if (valid) {  // the resolve phase's lookup key (stream 3)
                lk_keys[i] = pack_lookup_key(h);
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
    return home - k.slice_base;  // < S: the local table's home slot
}

template <bool FIXED>
__global__ void __launch_bounds__(kT)
shard_apply_kernel(ShardK k, const PF_GRID_CONST pf_table fine, const PF_GRID_CONST pf_table coarse,
                   int has_coarse, const int64_t *rec,
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

// ------------------------------------------------------------------ replica

// Owner side: every occupied slot of the local slice -> one 48-byte entry
// {global slot | table bit 62, tag, effective record (4 words)}.
__global__ void __launch_bounds__(kT)
shard_publish_kernel(ShardK k, pf_table t, int table_bit, int mode, double ema, double delta_max,
                     uint64_t *out, int64_t *count) {
    __shared__ SweepSmem<kT> q;
    const bool fixed = t.sum_mode == PF_SUM_FIXED;
    const bool as_int = eff_is_int(t, mode);
    for_each_occupied<kT>(t.tags, t.capacity, q, [&](int64_t s, uint64_t tag) {
        const ulonglong4 r = pack_effective(effective_of(load_cell(t, s, true), fixed, mode, ema,
                                                         delta_max), as_int);
        const unsigned long long j = atomicAdd(reinterpret_cast<unsigned long long *>(count), 1ull);
        uint64_t *e = out + 6 * j;
        e[0] = (k.slice_base + static_cast<uint64_t>(s)) | (static_cast<uint64_t>(table_bit) << 62);
        e[1] = tag;
        e[2] = r.x;
        e[3] = r.y;
        e[4] = r.z;
        e[5] = r.w;
    });
}

// All-gathered entries: rank r's rows are [r * stride, r * stride + counts[r]).  clear=1
// empties the entries' slots (last frame's replica), clear=0 writes tags and records.
__global__ void __launch_bounds__(kT)
replica_update_kernel(pf_replica rp, const uint64_t *entries, const int64_t *counts, int world,
                      int64_t stride, int clear) {
    const int64_t n = stride * world;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * kT + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * kT) {
        const int r = static_cast<int>(i / stride);
        if (i - r * stride >= counts[r]) continue;
        const uint64_t *e = entries + 6 * i;
        const bool coarse = (e[0] >> 62) & 1u;
        const uint64_t slot = e[0] & ((1ull << 62) - 1);
        uint64_t *tags = coarse ? rp.coarse_tags : rp.fine_tags;
        uint64_t *rec = coarse ? rp.coarse_records : rp.fine_records;
        if (tags == nullptr) continue;
        if (clear) {
            tags[slot] = kEmptyTag;
        } else {
            tags[slot] = e[1];
            reinterpret_cast<ulonglong2 *>(rec + 4 * slot)[0] = make_ulonglong2(e[2], e[3]);
            reinterpret_cast<ulonglong2 *>(rec + 4 * slot)[1] = make_ulonglong2(e[4], e[5]);
        }
    }
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

// The local slice table: capacity S = C / world, probe windows wrap within it.
int check_slice(const char *fn, const ShardK &k, const pf_table *t) {
    if (int rc = validate_table(fn, t)) return rc;
    const int64_t want = (1ll << k.s.log2_capacity) / k.s.world;
    if (t->capacity != want) return fail_arg(fn, "local table capacity must be C / world");
    if (t->sum_mode != k.s.sum_mode) return fail_arg(fn, "table sum_mode differs from the shard's");
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
                  const int32_t *abort_flag, uint64_t *lookup_keys, void *stream) {
    const char *fn = "pf_shard_keys";
    ShardK k;
    if (int rc = prepare_shard(fn, sh, &k)) return rc;
    if (int rc = validate_vertices(fn, v, cfg)) return rc;
    pf_config kc;
    if (int rc = prepare_config(fn, cfg, &kc)) return rc;
    if (v->n == 0) return PF_OK;
    if (!v->contribution || !lookup_keys)
        return fail_arg(fn, "contribution/lookup_keys is NULL");
    cudaStream_t st = as_stream(stream);
    if (sh->sum_mode == PF_SUM_FIXED)
        shard_keys_kernel<true><<<grid_for(shard_keys_kernel<true>, v->n, 8), kT, 0, st>>>(
            kc, *v, k, has_coarse != 0, stream_base_accum, stream_base_lookup, abort_flag,
            lookup_keys);
    else
        shard_keys_kernel<false><<<grid_for(shard_keys_kernel<false>, v->n, 8), kT, 0, st>>>(
            kc, *v, k, has_coarse != 0, stream_base_accum, stream_base_lookup, abort_flag,
            lookup_keys);
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

int pf_shard_publish(const pf_shard *sh, const pf_config *cfg, const pf_table *fine,
                     const pf_table *coarse, uint64_t *entries, int64_t *count, void *stream) {
    const char *fn = "pf_shard_publish";
    ShardK k;
    if (int rc = prepare_shard(fn, sh, &k)) return rc;
    if (cfg == nullptr || !entries || !count) return fail_arg(fn, "config/entries/count is NULL");
    if (int rc = check_slice(fn, k, fine)) return rc;
    if (coarse)
        if (int rc = check_slice(fn, k, coarse)) return rc;
    cudaStream_t st = as_stream(stream);
    if (cudaMemsetAsync(count, 0, sizeof(int64_t), st) != cudaSuccess) return check_launch(fn);
    const pf_table *tabs[2] = {fine, coarse};
    for (int tb = 0; tb < 2; ++tb) {
        if (!tabs[tb]) continue;
        shard_publish_kernel<<<sweep_blocks<kT>(tabs[tb]->capacity, sm_count()), kT, 0, st>>>(
            k, *tabs[tb], tb, cfg->temporal_mode, cfg->ema_alpha, cfg->delta_max, entries, count);
        if (int rc = check_launch(fn)) return rc;
    }
    return PF_OK;
}

int pf_replica_update(const pf_replica *rp, const uint64_t *entries, const int64_t *counts,
                      int32_t world, int64_t stride, int32_t clear, void *stream) {
    const char *fn = "pf_replica_update";
    if (!rp || !rp->fine_tags || !rp->fine_records || world < 1 || stride < 0)
        return fail_arg(fn, "bad replica / sizes");
    if (stride == 0) return PF_OK;
    if (!entries || !counts) return fail_arg(fn, "entries/counts is NULL");
    int64_t blocks = (stride * world + kT - 1) / kT;
    const int64_t cap = static_cast<int64_t>(sm_count()) * 8;
    if (blocks > cap) blocks = cap;
    replica_update_kernel<<<static_cast<unsigned>(blocks), kT, 0, as_stream(stream)>>>(
        *rp, entries, counts, world, stride, clear);
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
