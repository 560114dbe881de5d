// Fused per-frame kernels: accumulate_phase (keys + warp-merged insert into the fine
// and coarse tables in one pass over the vertex buffer) and resolve_phase (lookup
// keys, fine rung, 3x3x3 neighbourhood + coarse rungs on a compacted work list,
// composite).  src/pipeline.py:152-283.
#include "pf_resolve.cuh"
#include "pf_sweep.cuh"
#include "pf_internal.cuh"

namespace pf {

constexpr int kThreads = 256;
#ifndef PF_RESOLVE_KV
#define PF_RESOLVE_KV 1  // at 4 CTAs per SM (64 registers): 0.325 ms vs 0.336 for 2 rows per thread
#endif
constexpr int kResolveKV = PF_RESOLVE_KV;
#ifndef PF_RESOLVE_HOIST
#define PF_RESOLVE_HOIST 1
#endif  // vertices per thread in resolve_main
constexpr int kWarps = kThreads / 32;

// Rows per work list: resolve_main block b (kThreads * kResolveKV rows) appends to list
// b % PF_WORK_LISTS, so a list holds at most ceil(blocks / PF_WORK_LISTS) blocks' rows.
inline int64_t work_list_capacity(int64_t n) {
    const int64_t rows = static_cast<int64_t>(kThreads) * kResolveKV;
    const int64_t blocks = (n + rows - 1) / rows;
    return (blocks + PF_WORK_LISTS - 1) / PF_WORK_LISTS * rows;
}

__device__ __forceinline__ void log_eviction(pf_evict_event *events, int64_t *count, int64_t cap,
                                             int64_t vertex, const LaneInsert &r) {
    if (events == nullptr || count == nullptr) return;
    const unsigned long long k = atomicAdd(reinterpret_cast<unsigned long long *>(count), 1ull);
    if (static_cast<int64_t>(k) < cap) {
        pf_evict_event e;
        e.vertex = vertex;
        e.slot = r.slot;
        e.victim_tag = r.victim_tag;
        e.victim_touch = r.victim_touch;
        events[k] = e;
    }
}

// ------------------------------------------------------------------ insert

// The fused insert does not warp-merge equal keys (bit 0: merge fine keys, bit 1:
// coarse): after the merge only 1.21 (fine) / 1.29 (coarse) vertices share an update
// on the 1080p 4-bounce stream (tools/merge_stats.py), and the two MATCH.ANY plus the
// pointer-jumping rounds cost more issue slots than the extra REDs (insert 0.93 ->
// 0.82 ms; merging one table only: 0.83-0.86 ms).  Lanes with equal keys probe side by
// side and resolve to the same cell through probe_insert's claim / evict protocol.
#ifndef PF_FRAME_MERGE
#define PF_FRAME_MERGE 0
#endif
// The vertex's tangent frame (t1, t2: 12 registers) is parked in shared memory between
// the fine and the lookup disc draws: at the 80-register cap this trims spills
// (stack 280 -> 232 bytes) and the insert goes 0.796 -> 0.779 ms.
#ifndef PF_FRAME_SMEM
#define PF_FRAME_SMEM 1
#endif
#ifndef PF_POS_SMEM
#define PF_POS_SMEM 1  // the position too (0.784 -> 0.775 ms)
#endif

// The home-slot tags reach the insert by cp.async (L2, 16 bytes: the home tag's aligned
// pair) into shared memory as each hash exists, and one wait_all after the key loop.  A
// register load there is waited for at the rolled key loop's back-edge (the compiler
// does not keep a load in flight across it; at 4K, where the tables miss L2, that wait
// was the kernel's largest stall): hd4 insert 0.774 -> 0.757 ms.  L2 prefetches instead
// evict table lines (uhd4 4.60 -> 5.13 ms), as did an L2 prefetch of each CTA's next
// vertex tile (+5 us).  DESIGN.md 4.
#ifndef PF_INSERT_MIN_BLOCKS
#define PF_INSERT_MIN_BLOCKS 3  // 3 x 256 threads per SM: <= 85 registers
#endif

template <bool FIXED>
__global__ void __launch_bounds__(kThreads, PF_INSERT_MIN_BLOCKS)
insert_frame_kernel(const PF_GRID_CONST pf_config cfg, const PF_GRID_CONST pf_vertices v,
                    const PF_GRID_CONST pf_table fine, const PF_GRID_CONST pf_table coarse,
                    int has_coarse,
                    uint64_t h0, int64_t frame, int64_t *stats, pf_evict_event *events,
                    int64_t *event_count, int64_t event_cap, const int32_t *abort_flag,
                    uint64_t h0_lookup, uint64_t *lk_keys) {
    __shared__ BlockStats bs;
    __shared__ double2 sincos_tab[220];
    __shared__ double lod_dist[32];
#if PF_FRAME_SMEM
    __shared__ double onb[6][kThreads];  // per-thread tangent frame (t1, t2)
#endif
#if PF_POS_SMEM
    __shared__ double posm[3][kThreads];  // per-thread vertex position
#endif
    __shared__ __align__(16) uint64_t home_pair[2][kThreads][2];  // fine / coarse home tag pairs
    __shared__ double2 lvsteps[32];

    stats_init(bs);
    stage_sincos_table(sincos_tab);
    stage_lod_dist(lod_dist, cfg);
    stage_level_steps(lvsteps, cfg);
    pdl_wait();
    pdl_trigger();
    if (abort_flag != nullptr && *abort_flag != 0) return;  // invalid input: no mutation
    __syncthreads();
    // persistent: each block walks 256-vertex tiles; block counters flush once at exit
    const int64_t tiles = (v.n + kThreads - 1) / kThreads;
    for (int64_t tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
    const int64_t i0 = tile * kThreads + threadIdx.x;
    const bool valid = i0 < v.n;
    // tail lanes recompute the last vertex (no divergent key code); warp_insert ignores them
    const int64_t i = valid ? i0 : v.n - 1;
    double val[3];
    CellHash hf{0ull, 0u}, hc{0ull, 0u};
    uint64_t ht_f = 0, ht_c = 0;
    {
        const uint64_t stream = l2_evict_first();
        const VertexIn x = load_vertex(v, i, cfg, stream);
#pragma unroll
        for (int c = 0; c < 3; ++c) val[c] = ld_stream(v.contribution + 3 * i + c, stream);
        const KeyShared ks = key_shared(cfg, x, lod_dist);
#if PF_FRAME_SMEM
        // the tangent frame waits in shared memory between the two disc draws
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            onb[c][threadIdx.x] = ks.frame.t1[c];
            onb[3 + c][threadIdx.x] = ks.frame.t2[c];
        }
#endif
#if PF_POS_SMEM
#pragma unroll
        for (int c = 0; c < 3; ++c) posm[c][threadIdx.x] = x.pos[c];
#endif
        const uint64_t pid = path_id(x.pixel, x.sample);
        // Key sets in one rolled loop (one copy of the key code keeps the kernel's
        // instruction footprint inside the SM's instruction caches):
        //   0 fine (jitter stream 2), 1 coarse (stream 2, level + coarse_delta),
        //   2 the resolve phase's fine lookup key (stream 3)
        const int nsets = lk_keys != nullptr ? 3 : (has_coarse ? 2 : 1);
        double w[3] = {0.0, 0.0, 0.0};  // jitter direction u*t1 + v*t2
#pragma unroll 1
        for (int set = 0; set < nsets; ++set) {
            if (set == 1 && !has_coarse) continue;
            if (set != 1 && cfg.jitter) {  // set 1 reuses set 0's disc offsets
                double u1, u2, du, dv;
                jitter_draws_pid(set == 0 ? h0 : h0_lookup, pid, u1, u2);
                disc_offset(u1, u2, du, dv, sincos_tab);
#if PF_FRAME_SMEM
                double t1[3], t2[3];
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    t1[c] = onb[c][threadIdx.x];
                    t2[c] = onb[3 + c][threadIdx.x];
                }
                jitter_dir(du, dv, t1, t2, w);
#else
                jitter_dir(du, dv, ks.frame.t1, ks.frame.t2, w);
#endif
            }
            double jt[3];
#if PF_POS_SMEM
            VertexIn xk = x;
#pragma unroll
            for (int c = 0; c < 3; ++c) xk.pos[c] = posm[c][threadIdx.x];
#else
            const VertexIn &xk = x;
#endif
            const CellHash h = key_hash(
                make_key_w(cfg, xk, ks, cfg.jitter, w, set == 1 ? cfg.coarse_delta : 0, jt,
                           lvsteps), ks);
            // home-slot tag copies go out as soon as a hash exists; the next key set's
            // arithmetic hides their L2 latency before warp_insert consumes them
            if (set < 2) {
                const pf_table &t = set == 0 ? fine : coarse;
                const int64_t home = static_cast<int64_t>(h.index & static_cast<uint64_t>(t.capacity - 1));
                if (set == 0) hf = h;
                else hc = h;
                cp_async_16(&home_pair[set][threadIdx.x][0], t.tags + (home & ~int64_t(1)));
            } else if (valid) {
                lk_keys[i] = pack_lookup_key(h);
            }
        }
    }
    cp_async_wait_all();
    ht_f = home_pair[0][threadIdx.x][hf.index & 1];
    if (has_coarse) ht_c = home_pair[1][threadIdx.x][hc.index & 1];
    int64_t qval[3];  // quantised once for both tables
#pragma unroll
    for (int c = 0; c < 3; ++c) qval[c] = FIXED ? quantize_fixed(val[c]) : 0;
    // unrolled: each copy of warp_insert addresses its table's parameters directly
#pragma unroll
    for (int tb = 0; tb < 2; ++tb) {
        if (tb == 1 && !has_coarse) break;
        const pf_table &t = tb == 0 ? fine : coarse;
        const CellHash h = tb == 0 ? hf : hc;
        const uint64_t home_tag = tb == 0 ? ht_f : ht_c;
        const LaneInsert r = ((PF_FRAME_MERGE >> tb) & 1)
            ? warp_insert<FIXED>(t, valid, h.index, h.fp, val, frame, home_tag, true, false)
            : lane_insert<FIXED>(t, valid, h.index, h.fp, qval, val, frame, home_tag, false);
        warp_count(bs, tb == 0 ? PF_STAT_PROBE_FAILURES : PF_STAT_COARSE_PROBE_FAILURES,
                   valid && r.status == 2);
        warp_count(bs, tb == 0 ? PF_STAT_EVICTIONS : PF_STAT_COARSE_EVICTIONS,
                   valid && r.leader && r.status == 1);
        if (tb == 0) {
            // probe-length histogram and sum, merged per distinct length in the warp
            const int pl = valid ? r.probe_len : -1;
            const unsigned same = __match_any_sync(kFull, pl);
            if (valid && (threadIdx.x & 31) == static_cast<unsigned>(__ffs(same) - 1)) {
                const unsigned cnt = __popc(same);
                atomicAdd(&bs.hist[pl & 255], cnt);
                atomicAdd(&bs.v[PF_STAT_PROBE_LEN_SUM], cnt * static_cast<unsigned>(pl));
            }
            if (valid && r.leader && r.status == 1)
                log_eviction(events, event_count, event_cap, i, r);
        }
    }
    }
    __syncthreads();
    stats_flush(bs, stats, true);
}

// Resident blocks per SM for a kernel (cached per function), for persistent grids.
template <typename K>
static int resident_blocks(K kernel, int threads) {
    int b = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kernel, threads, 0) != cudaSuccess || b < 1)
        b = 1;
    return b;
}

// ------------------------------------------------------------------ resolve

struct ResolveArgs {
    pf_config cfg;
    pf_vertices v;
    pf_table fine;
    pf_table coarse;
    int has_coarse;
    uint64_t h0_lookup;
    uint64_t h0_coarse;
    double *flat;
    int64_t *work;             // PF_WORK_LISTS lists of wcap rows each
    int64_t *work_count;       // [PF_WORK_LISTS]
    int64_t wcap;
    uint8_t *source;
    double *chosen;
    int64_t *stats;
    double thr;
    const uint64_t *lk_keys;   // precomputed packed lookup keys (or NULL)
    const ulonglong4 *rec;     // per-slot effective records of the fine table (or NULL)
    int64_t n_pixels;          // flat holds pixels [pixel_base, pixel_base + n_pixels)
    int64_t *fb_keys;          // [work row][8] lookup key, coarse slot, row, pixel (or NULL)
    int64_t pixel_base;        // first pixel of flat (0 unless a rank composites a band)
    uint64_t seg_mask;         // probe-window segment (~0: plain table; replica: slice - 1)
    const ulonglong4 *crec;    // per-slot effective records of the coarse table (or NULL)
};

// The coarse table's effective value of slot s.
__device__ __forceinline__ Effective coarse_effective(const ResolveArgs &a, int64_t s) {
    const int mode = a.cfg.temporal_mode;
    if (a.crec != nullptr) return unpack_effective(load_record(a.crec, s), eff_is_int(a.coarse, mode));
    return effective_at(a.coarse, s, mode, a.cfg.ema_alpha, a.cfg.delta_max);
}

// The fine table's effective value of slot s: its record when the effective pass ran.
__device__ __forceinline__ Effective fine_effective(const ResolveArgs &a, int64_t s) {
    const int mode = a.cfg.temporal_mode;
    if (a.rec != nullptr) return unpack_effective(load_record(a.rec, s), eff_is_int(a.fine, mode));
    return effective_at(a.fine, s, mode, a.cfg.ema_alpha, a.cfg.delta_max);
}

constexpr int64_t kNoTouch = INT64_MIN;  // touch_frame of a sweep without deferred touches

// VoxelTable.effective of every occupied fine slot, once per resolve: lookups then
// read one sector instead of the five SoA sectors of a slot's state.  The same sweep
// finishes the frame insert's deferred last_touch stores (touch_frame != kNoTouch): every cell
// an accumulate reached this frame has a live count > 0 (begin_frame zeroed them), so
// last_touch = frame there leaves the table byte-identical to the reference's
// per-vertex store (src/_native.pyx:257) at a fraction of its L2 traffic.  Blocks
// [0, nb_fine) sweep the fine table, the rest the coarse table (touch only).
// Append slot s to an occupied-slot list (opportunistic warp aggregation over the lanes
// that reach this call together).
__device__ __forceinline__ void occ_append(int32_t *list, int64_t *count, int64_t s) {
    const unsigned m = __activemask();
    const int lane = threadIdx.x & 31;
    const int leader = __ffs(m) - 1;
    unsigned long long base = 0;
    if (lane == leader)
        base = atomicAdd(reinterpret_cast<unsigned long long *>(count),
                         static_cast<unsigned long long>(__popc(m)));
    base = __shfl_sync(m, base, leader);
    list[base + __popc(m & ((1u << lane) - 1u))] = static_cast<int32_t>(s);
}

__global__ void __launch_bounds__(kThreads)
effective_records_kernel(const PF_GRID_CONST pf_table t, int mode, double ema, double delta_max,
                         ulonglong4 *rec, const PF_GRID_CONST pf_table coarse, int has_coarse,
                         int64_t touch_frame, unsigned nb_fine, double *flat, int64_t flat_words,
                         int64_t *counter, const double *flat_init, int32_t *occ_fine,
                         int32_t *occ_coarse, int64_t *occ_n) {
    __shared__ SweepSmem<kThreads> q;
    pdl_wait();  // multi-wave kernels do not trigger early: waiting dependents would take
                 // the slots of their later waves
    // the resolve's composite buffer and work counter start at zero (in this launch rather
    // than a memset, which would break the frame's PDL chain); with flat_init the buffer
    // starts at flat_init + 0.0 instead (the image itself at spp = 1, see resolve_frame)
    if (flat != nullptr) {
        double2 *f2 = reinterpret_cast<double2 *>(flat);
        const double2 *i2 = reinterpret_cast<const double2 *>(flat_init);
        const int64_t pairs = flat_words / 2;
        for (int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; k < pairs;
             k += static_cast<int64_t>(gridDim.x) * blockDim.x) {
            double2 v = make_double2(0.0, 0.0);
            if (i2 != nullptr) {
                const double2 b = __ldg(i2 + k);
                v = make_double2(dadd(b.x, 0.0), dadd(b.y, 0.0));
            }
            f2[k] = v;
        }
        if (blockIdx.x == 0 && threadIdx.x == 0 && (flat_words & 1))
            flat[flat_words - 1] = flat_init ? dadd(flat_init[flat_words - 1], 0.0) : 0.0;
    }
    if (counter != nullptr && blockIdx.x == 0 && threadIdx.x < PF_WORK_LISTS) counter[threadIdx.x] = 0;
    if (blockIdx.x >= nb_fine) {
        const int64_t blk = blockIdx.x - nb_fine, nblk = gridDim.x - nb_fine;
        for_each_occupied<kThreads>(coarse.tags, coarse.capacity, q, blk, nblk,
                                    [&](int64_t s, uint64_t) {
            if (ld_relaxed_i64(cnt_at(coarse, s)) > 0) *touch_at(coarse, s) = touch_frame;
            if (occ_coarse != nullptr) occ_append(occ_coarse, occ_n + 1, s);
        });
        return;
    }
    const bool fixed = t.sum_mode == PF_SUM_FIXED;
    const bool as_int = eff_is_int(t, mode);
    for_each_occupied<kThreads>(t.tags, t.capacity, q, blockIdx.x, nb_fine,
                                [&](int64_t s, uint64_t) {
        const CellState cs = load_cell(t, s, true);
        if (rec != nullptr) rec[s] = pack_effective(effective_of(cs, fixed, mode, ema, delta_max), as_int);
        if (touch_frame != kNoTouch && cs.counts > 0) *touch_at(t, s) = touch_frame;
        if (occ_fine != nullptr) occ_append(occ_fine, occ_n, s);
    });
}

// Launch the sweep above (records and / or deferred touches, and the zeroing of the
// composite buffer / work counter when given); no-op when there is nothing to do.
static int launch_post_insert(const char *fn, const pf_table &fine, const pf_table *coarse,
                              const pf_config &kc, uint64_t *eff_records, int64_t touch_frame,
                              cudaStream_t st, double *flat = nullptr, int64_t flat_words = 0,
                              int64_t *counter = nullptr, const double *flat_init = nullptr,
                              int32_t *occ_fine = nullptr, int32_t *occ_coarse = nullptr,
                              int64_t *occ_n = nullptr) {
    if (eff_records == nullptr && touch_frame == kNoTouch && flat == nullptr && counter == nullptr)
        return PF_OK;
    const unsigned nf = sweep_blocks<kThreads>(fine.capacity, sm_count());
    const bool tc = coarse != nullptr && touch_frame != kNoTouch;
    const unsigned nc = tc ? sweep_blocks<kThreads>(coarse->capacity, sm_count()) : 0u;
    launch_pdl(effective_records_kernel, dim3(nf + nc), dim3(kThreads), st, fine,
               kc.temporal_mode, kc.ema_alpha, kc.delta_max,
               reinterpret_cast<ulonglong4 *>(eff_records), tc ? *coarse : fine,
               static_cast<int>(tc), touch_frame, nf, flat, flat_words, counter, flat_init,
               occ_n ? occ_fine : nullptr, occ_n && tc ? occ_coarse : nullptr, occ_n);
    return check_launch(fn);
}

// The fine lookup key of one vertex: jitter stream 3 when jitter is on
// (src/pipeline.py:222-225), level_delta 0.
__device__ __forceinline__ KeyAndHash lookup_key(const ResolveArgs &a, int64_t row) {
    return vertex_key(a.cfg, a.v, a.h0_lookup, row, 0);
}

__device__ __forceinline__ void composite(const ResolveArgs &a, int64_t i, int64_t pixel,
                                          const double chosen[3], int source) {
    pixel -= a.pixel_base;
    const uint64_t stream = l2_evict_first(), keep = l2_policy(PF_FLAT_POLICY);
    if (pixel >= 0 && pixel < a.n_pixels) {
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            const double tp = ld_stream(a.v.throughput + 3 * i + c, stream);
            red_add_f64(a.flat + 3 * pixel + c, dmul(tp, chosen[c]), keep);
        }
    }
    if (a.source) a.source[i] = static_cast<uint8_t>(source);
    if (a.chosen) {
#pragma unroll
        for (int c = 0; c < 3; ++c) a.chosen[3 * i + c] = chosen[c];
    }
}

// Rung 1 for every vertex; rows below the threshold go to the work list (row ids).
// KV vertices per thread, each step issued for all KV rows before the next (key ->
// home tag -> cell state -> composite), so a thread keeps KV independent L2/HBM
// round trips in flight: the kernel is bound by memory latency, not arithmetic.
#ifndef PF_RESOLVE_MIN_BLOCKS
#define PF_RESOLVE_MIN_BLOCKS 4  // 4 x 256 threads per SM: <= 64 registers
#endif
#ifndef PF_RESOLVE_SPEC
#define PF_RESOLVE_SPEC 1  // the home slot's record loaded beside its tag
#endif
#ifndef PF_RESOLVE_STAGE
#define PF_RESOLVE_STAGE 1  // composite stream words staged in shared memory by cp.async
#endif
#ifndef PF_RESOLVE_KEYS_MIN_BLOCKS
#define PF_RESOLVE_KEYS_MIN_BLOCKS 5  // with the insert's keys and staging: <= 48 registers
#endif
template <int KV, bool HAVE_KEYS>
__global__ void __launch_bounds__(kThreads, HAVE_KEYS ? PF_RESOLVE_KEYS_MIN_BLOCKS
                                                      : PF_RESOLVE_MIN_BLOCKS)
resolve_main_kernel(ResolveArgs a) {
    // no CTA counters and no barriers: the fine / fallback row counts follow from the
    // work list (main_row_counts in the next kernel), rows outside the image are rare
    pdl_wait();
    const pf_config &cfg = a.cfg;
    const uint64_t stream = l2_evict_first(), keep = l2_policy(PF_FLAT_POLICY);
    const uint64_t fmask = static_cast<uint64_t>(a.fine.capacity) - 1;
    const int64_t base = static_cast<int64_t>(blockIdx.x) * blockDim.x * KV + threadIdx.x;
    int64_t row[KV];
    bool valid[KV];
    CellHash h[KV];
    uint64_t tag[KV];
    int64_t pixel[KV];
    double tp[KV][3];
#pragma unroll
    for (int k = 0; k < KV; ++k) {
        const int64_t i0 = base + static_cast<int64_t>(k) * blockDim.x;
        valid[k] = i0 < a.v.n;
        row[k] = valid[k] ? i0 : a.v.n - 1;  // tail lanes shadow the last vertex
        if (HAVE_KEYS) {  // keys emitted by the insert pass
            h[k] = unpack_lookup_key(ld_stream(a.lk_keys + row[k], stream));
        } else {
            h[k] = lookup_key(a, row[k]).second;
        }
    }
#if PF_RESOLVE_STAGE
    // the composite's stream words go to shared memory by cp.async beside the key load:
    // in flight through the key -> tag -> record chain without holding registers
    static_assert(KV == 1, "staged resolve is one row per thread");
    __shared__ int64_t stg_pix[kThreads];
    __shared__ double stg_tp[3][kThreads];
    cp_async_8_hint(&stg_pix[threadIdx.x], a.v.pixel + row[0], stream);
#pragma unroll
    for (int c = 0; c < 3; ++c)
        cp_async_8_hint(&stg_tp[c][threadIdx.x], a.v.throughput + 3 * row[0] + c, stream);
#elif PF_RESOLVE_HOIST
    // the composite's stream loads depend on nothing: in flight beside the key loads
#pragma unroll
    for (int k = 0; k < KV; ++k) {
        pixel[k] = ld_stream(a.v.pixel + row[k], stream) - a.pixel_base;
#pragma unroll
        for (int c = 0; c < 3; ++c) tp[k][c] = ld_stream(a.v.throughput + 3 * row[k] + c, stream);
    }
#endif
#pragma unroll
    for (int k = 0; k < KV; ++k) tag[k] = __ldg(reinterpret_cast<const unsigned long long *>(
                                      a.fine.tags) + (h[k].index & fmask));
#if PF_RESOLVE_SPEC
    // the home slot's record in flight beside its tag (most keys sit at home)
    ulonglong4 srec[KV];
    if (a.rec != nullptr) {
#pragma unroll
        for (int k = 0; k < KV; ++k) srec[k] = load_record(a.rec, static_cast<int64_t>(h[k].index & fmask));
    }
#endif
    int64_t slot[KV];
#pragma unroll
    for (int k = 0; k < KV; ++k) {
        // first probe from the prefetched home tag; longer chains are rare
        if (tag[k] == kEmptyTag) slot[k] = -1;
        else if ((tag[k] & kFpMask) == h[k].fp) slot[k] = static_cast<int64_t>(h[k].index & fmask);
        else slot[k] = probe_lookup(a.fine.tags, fmask, a.fine.probe_limit, h[k].index, h[k].fp,
                                    a.seg_mask);
    }
    Effective ef[KV];
#pragma unroll
    for (int k = 0; k < KV; ++k) {
#if PF_RESOLVE_SPEC
        if (slot[k] >= 0 && a.rec != nullptr && slot[k] == static_cast<int64_t>(h[k].index & fmask))
            ef[k] = unpack_effective(srec[k], eff_is_int(a.fine, cfg.temporal_mode));
        else
#endif
        if (slot[k] >= 0) ef[k] = fine_effective(a, slot[k]);
#if !PF_RESOLVE_HOIST && !PF_RESOLVE_STAGE
        pixel[k] = ld_stream(a.v.pixel + row[k], stream) - a.pixel_base;
#pragma unroll
        for (int c = 0; c < 3; ++c) tp[k][c] = ld_stream(a.v.throughput + 3 * row[k] + c, stream);
#endif
    }
#if PF_RESOLVE_STAGE
    cp_async_wait_all();
    pixel[0] = stg_pix[threadIdx.x] - a.pixel_base;
#pragma unroll
    for (int c = 0; c < 3; ++c) tp[0][c] = stg_tp[c][threadIdx.x];
#endif
    const bool as_int = eff_is_int(a.fine, cfg.temporal_mode);
    const bool fixed = a.fine.sum_mode == PF_SUM_FIXED;
#pragma unroll
    for (int k = 0; k < KV; ++k) {
        bool fine_ok = false;
        if (slot[k] >= 0) {
            const Effective &e = ef[k];
            const double cnt = e.fcnt;
            if (valid[k] && cnt >= a.thr) {
                fine_ok = true;
                double m[3];
                const bool in_image = pixel[k] >= 0 && pixel[k] < a.n_pixels;
                const double sums[3] = {eff_sum_f64(e, as_int, 0), eff_sum_f64(e, as_int, 1),
                                        eff_sum_f64(e, as_int, 2)};
                row_mean3(sums, cnt, fixed, m);
#pragma unroll
                for (int c = 0; c < 3; ++c)
                    if (in_image) red_add_f64(a.flat + 3 * pixel[k] + c, dmul(tp[k][c], m[c]), keep);
                if (a.source) a.source[row[k]] = 0;
                if (a.chosen) {
#pragma unroll
                    for (int c = 0; c < 3; ++c) a.chosen[3 * row[k] + c] = m[c];
                }
            }
        }
        // rows below the threshold: append the row id to the work list (warp-aggregated)
        const bool need = valid[k] && !fine_ok;
        const unsigned m = __ballot_sync(kFull, need);
        if (m) {
            unsigned long long wb = 0;
            const int lane = threadIdx.x & 31;
            // one of PF_WORK_LISTS lists per block (by block index): a single counter
            // hit by every warp with a low-count row was a hot L2 atomic
            const int list = static_cast<int>(blockIdx.x) & (PF_WORK_LISTS - 1);
            if (lane == __ffs(m) - 1)
                wb = atomicAdd(reinterpret_cast<unsigned long long *>(a.work_count + list),
                               static_cast<unsigned long long>(__popc(m)));
            wb = __shfl_sync(kFull, wb, __ffs(m) - 1);
            if (need)
                a.work[list * a.wcap + static_cast<int64_t>(wb) + __popc(m & ((1u << lane) - 1u))] =
                    row[k];
        }
        const bool bad = valid[k] && fine_ok && !(pixel[k] >= 0 && pixel[k] < a.n_pixels);
        if (__any_sync(kFull, bad)) {
            const unsigned b = __ballot_sync(kFull, bad);
            if ((threadIdx.x & 31) == 0)
                atomicAdd(reinterpret_cast<unsigned long long *>(a.stats + PF_STAT_BAD_PIXELS),
                          static_cast<unsigned long long>(__popc(b)));
        }
    }
}

// The resolve's work lists as one sequence: a CTA loads the PF_WORK_LISTS counts into
// shared memory once; entry w of the sequence is row work_row(w).
struct WorkLists {
    int64_t start[PF_WORK_LISTS + 1];  // prefix sums of the list counts
};
__device__ __forceinline__ int64_t load_work_lists(const ResolveArgs &a, WorkLists &wl) {
    if (threadIdx.x == 0) {
        int64_t acc = 0;
        for (int j = 0; j < PF_WORK_LISTS; ++j) {
            wl.start[j] = acc;
            acc += a.work_count[j];
        }
        wl.start[PF_WORK_LISTS] = acc;
    }
    __syncthreads();
    return wl.start[PF_WORK_LISTS];
}
__device__ __forceinline__ int64_t work_row(const ResolveArgs &a, const WorkLists &wl, int64_t w) {
    int lo = 0, hi = PF_WORK_LISTS;  // the list j with start[j] <= w < start[j + 1]
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (wl.start[mid] <= w) lo = mid;
        else hi = mid;
    }
    return a.work[lo * a.wcap + (w - wl.start[lo])];
}

// resolve_main's row counters, once per resolve: every row it saw either took the fine
// rung or went to the work list (called by one thread of the kernel that follows it).
__device__ __forceinline__ void main_row_counts(const ResolveArgs &a, int64_t n_work) {
    atomicAdd(reinterpret_cast<unsigned long long *>(a.stats + PF_STAT_FALLBACK_ROWS),
              static_cast<unsigned long long>(n_work));
    atomicAdd(reinterpret_cast<unsigned long long *>(a.stats + PF_STAT_SOURCE_FINE),
              static_cast<unsigned long long>(a.v.n - n_work));
}

// The work rows' lookup keys (q, level, aux; stream 3) and coarse slots, one row per
// thread -- the FP64 key recipe and the coarse probe run SIMT-wide instead of on the
// pool's critical path.  Record per work row: q0, q1, q2, level, aux, coarse slot (-1:
// absent), row, pixel.
__global__ void __launch_bounds__(kThreads) fallback_keys_kernel(ResolveArgs a) {
    __shared__ double2 sincos_tab[220];
    __shared__ double lod_dist[32];
    __shared__ double2 lvsteps[32];
    stage_sincos_table(sincos_tab);
    stage_lod_dist(lod_dist, a.cfg);
    stage_level_steps(lvsteps, a.cfg);
    __shared__ WorkLists wl;
    pdl_wait();
    pdl_trigger();
    __syncthreads();
    const pf_config &cfg = a.cfg;
    const int64_t n_work = load_work_lists(a, wl);
    for (int64_t w = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; w < n_work;
         w += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t row = work_row(a, wl, w);
        const VertexIn x = load_vertex(a.v, row, cfg);
        const KeyShared ks = key_shared(cfg, x, lod_dist);
        double du = 0.0, dv = 0.0, cdu = 0.0, cdv = 0.0;
        if (cfg.jitter) {  // the coarse key uses stream 3 too when jitter is on (:255)
            double u1, u2;
            jitter_draws(a.h0_lookup, x.pixel, x.sample, u1, u2);
            disc_offset(u1, u2, du, dv, sincos_tab);
            cdu = du;
            cdv = dv;
            if (a.h0_coarse != a.h0_lookup) {
                jitter_draws(a.h0_coarse, x.pixel, x.sample, u1, u2);
                disc_offset(u1, u2, cdu, cdv, sincos_tab);
            }
        }
        double jt[3];
        const CellKey k = make_key(cfg, x, ks, cfg.jitter, du, dv, 0, jt, lvsteps);
        int64_t cslot = -1;  // the coarse rung's slot: probed here, where rows run SIMT-wide
        if (a.has_coarse) {
            const CellHash hc =
                key_hash(make_key(cfg, x, ks, cfg.jitter, cdu, cdv, cfg.coarse_delta, jt, lvsteps), ks);
            cslot = probe_lookup(a.coarse.tags, static_cast<uint64_t>(a.coarse.capacity) - 1,
                                 a.coarse.probe_limit, hc.index, hc.fp, a.seg_mask);
        }
        longlong4 *o = reinterpret_cast<longlong4 *>(a.fb_keys + 8 * w);
        o[0] = make_longlong4(k.q[0], k.q[1], k.q[2], k.level);
        o[1] = make_longlong4(static_cast<long long>(k.aux), cslot, row, x.pixel);
    }
}

// Rungs 2-5 for one work row per warp: lanes 0..26 probe the 3x3x3 neighbourhood in
// (dx, dy, dz) nested order; lane 0 sums them in that order (numpy's order for the
// float64 pools), then runs the coarse rung, the ladder and the composite.
__global__ void __launch_bounds__(kThreads) resolve_fallback_kernel(ResolveArgs a) {
    __shared__ BlockStats bs;
    __shared__ WorkLists wl;
    stats_init(bs, false);
    pdl_wait();
    pdl_trigger();
    __syncthreads();
    const pf_config &cfg = a.cfg;
    const int lane = threadIdx.x & 31;
    const int64_t n_work = load_work_lists(a, wl);
    if (blockIdx.x == 0 && threadIdx.x == 0) main_row_counts(a, n_work);
    const int64_t warp0 = static_cast<int64_t>(blockIdx.x) * kWarps + (threadIdx.x >> 5);
    const int64_t nwarps = static_cast<int64_t>(gridDim.x) * kWarps;
    const int mode = cfg.temporal_mode;
    const bool as_int = eff_is_int(a.fine, mode);
    const bool fixed = a.fine.sum_mode == PF_SUM_FIXED;
    const uint64_t fmask = static_cast<uint64_t>(a.fine.capacity) - 1;
    for (int64_t w = warp0; w < n_work; w += nwarps) {
        const int64_t row = work_row(a, wl, w);
        // the row's lookup key, built by lane 0 and broadcast to the 27 probing lanes
        int64_t kq[3] = {0, 0, 0}, klev = 0, kaux = 0;
        if (lane == 0) {
            const CellKey k = lookup_key(a, row).first;
            kq[0] = k.q[0];
            kq[1] = k.q[1];
            kq[2] = k.q[2];
            klev = k.level;
            kaux = static_cast<int64_t>(k.aux);
        }
#pragma unroll
        for (int c = 0; c < 3; ++c) kq[c] = __shfl_sync(kFull, static_cast<long long>(kq[c]), 0);
        klev = __shfl_sync(kFull, static_cast<long long>(klev), 0);
        kaux = __shfl_sync(kFull, static_cast<long long>(kaux), 0);
        bool found = false;
        Effective e{};
        if (lane < 27) {
            const CellHash h = cell_hash(kq[0] + neighbour_dx(lane), kq[1] + neighbour_dy(lane),
                                         kq[2] + neighbour_dz(lane), klev,
                                         static_cast<uint64_t>(kaux), 0, 0u);
            const int64_t s = probe_lookup(a.fine.tags, fmask, a.fine.probe_limit, h.index, h.fp,
                                           a.seg_mask);
            if (s >= 0) {
                found = true;
                e = fine_effective(a, s);
            }
        }
        const Pool pool = pool_neighbours(found, e, as_int, mode);
        // every lane now holds the same pooled sums; lane 0 finishes the row
        const bool ok_n = ((mode == PF_INTEGRATE) ? static_cast<double>(pool.icnt) : pool.fcnt) >= a.thr;
        if (lane == 0) {
        const int64_t pixel = __ldg(a.v.pixel + row);
        bool coarse_found = false;
        Effective ce{};
        if (!ok_n && a.has_coarse) {
            const CellHash h = vertex_key(cfg, a.v, a.h0_coarse, row, cfg.coarse_delta).second;
            const int64_t s = probe_lookup(a.coarse.tags, static_cast<uint64_t>(a.coarse.capacity) - 1,
                                           a.coarse.probe_limit, h.index, h.fp, a.seg_mask);
            if (s >= 0) {
                coarse_found = true;
                ce = coarse_effective(a, s);
            }
        }
        double contrib[3], ch[3];
#pragma unroll
        for (int c = 0; c < 3; ++c) contrib[c] = __ldg(a.v.contribution + 3 * row + c);
        const int src = ladder_choose(pool, as_int, mode, fixed, a.thr, coarse_found, ce,
                                      eff_is_int(a.coarse, mode), contrib, ch);
        composite(a, row, pixel, ch, src);
        if (!(pixel - a.pixel_base >= 0 && pixel - a.pixel_base < a.n_pixels))
            atomicAdd(&bs.v[PF_STAT_BAD_PIXELS], 1u);
        atomicAdd(&bs.v[PF_STAT_SOURCE_FINE + src], 1u);
        }
        __syncwarp();
    }
    __syncthreads();
    stats_flush(bs, a.stats, false);
}

// Rungs 2-5 with the neighbourhood probes spread over the whole CTA: a pass takes
// kPoolRows work rows (keys, coarse slots, rows and pixels from fallback_keys_kernel),
// their 27 x kPoolRows cell probes run 3-4 per thread with all home tags, then all
// records, in flight together (records by cp.async into shared memory), the last warp
// fetches the rows' coarse records and composite inputs meanwhile, and the rows are
// then pooled (kLanesPerRow threads per row for integer pools; one, in (dx, dy, dz)
// order, for float64 pools), laddered and composited.
#ifndef PF_POOL_ROWS
#define PF_POOL_ROWS 32
#endif
constexpr int kPoolRows = PF_POOL_ROWS;
constexpr int kPoolCells = 27 * kPoolRows;
constexpr int kLanesPerRow = kThreads / kPoolRows;  // the per-row phase's threads per row
static_assert(kLanesPerRow >= 1 && kLanesPerRow <= 32 && (kLanesPerRow & (kLanesPerRow - 1)) == 0,
              "rows of the pool's per-row phase must tile warps");

struct PoolSmem {
    int64_t key[kPoolRows][8];
    alignas(16) uint64_t word[kPoolCells][4];  // sum x3 (int64 or float64 bits), count (float64)
    uint8_t found[kPoolCells];
    // per row, fetched in the probe phase by the CTA's last warp (so the serial per-row
    // phase does no global round trips): the coarse cell's effective value, the row's
    // contribution (the unfiltered rung), pixel and throughput (the composite)
    Effective coarse[kPoolRows];
    uint8_t coarse_found[kPoolRows];
    double contrib[kPoolRows][3];
    double tp[kPoolRows][3];
    int64_t pixel[kPoolRows];
    int64_t row[kPoolRows];
};

#ifndef PF_POOL_MIN_BLOCKS
#define PF_POOL_MIN_BLOCKS 3
#endif
__global__ void __launch_bounds__(kThreads, PF_POOL_MIN_BLOCKS) resolve_pool_kernel(ResolveArgs a) {
    __shared__ BlockStats bs;
    __shared__ PoolSmem ps;
    stats_init(bs, false);
    pdl_wait();
    pdl_trigger();
    __syncthreads();
    const pf_config &cfg = a.cfg;
    const int mode = cfg.temporal_mode;
    const bool as_int = eff_is_int(a.fine, mode);
    const bool int_cnt = mode == PF_INTEGRATE;
    const bool fixed = a.fine.sum_mode == PF_SUM_FIXED;
    const uint64_t fmask = static_cast<uint64_t>(a.fine.capacity) - 1;
    __shared__ WorkLists wl;
    const int64_t n_work = load_work_lists(a, wl);
    if (blockIdx.x == 0 && threadIdx.x == 0) main_row_counts(a, n_work);
    for (int64_t base = static_cast<int64_t>(blockIdx.x) * kPoolRows; base < n_work;
         base += static_cast<int64_t>(gridDim.x) * kPoolRows) {
        const int rows = static_cast<int>(n_work - base < kPoolRows ? n_work - base : kPoolRows);
        {  // stage the pass's key records (8 words per row)
            for (int q = threadIdx.x; q < 8 * rows; q += kThreads)
                ps.key[q >> 3][q & 7] = a.fb_keys[8 * base + q];
        }
        __syncthreads();
        {  // the CTA's last warp: each lane one row's coarse rung and composite inputs, one
           // round trip beside the probes (slot, row and pixel come with the key record)
            const int r = kThreads - 1 - static_cast<int>(threadIdx.x);
            if (r < rows) {
                const int64_t cs = ps.key[r][5], row = ps.key[r][6];
                ps.row[r] = row;
                ps.pixel[r] = ps.key[r][7];
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    ps.contrib[r][c] = __ldg(a.v.contribution + 3 * row + c);
                    ps.tp[r][c] = __ldg(a.v.throughput + 3 * row + c);
                }
                if (cs >= 0) ps.coarse[r] = coarse_effective(a, cs);
                ps.coarse_found[r] = cs >= 0;
            }
        }
        {  // this thread's probes p = threadIdx.x + u * kThreads: every home tag, then
           // every found cell's record, each batch issued back to back
            constexpr int kPP = (kPoolCells + kThreads - 1) / kThreads;
            const int np = 27 * rows;
            uint64_t home[kPP], tg[kPP];
            uint32_t fp[kPP];
#pragma unroll
            for (int u = 0; u < kPP; ++u) {
                const int p = static_cast<int>(threadIdx.x) + u * kThreads;
                tg[u] = kEmptyTag;
                if (p < np) {
                    const int r = p / 27, j = p - 27 * (p / 27);
                    const CellHash h = cell_hash(ps.key[r][0] + neighbour_dx(j),
                                                 ps.key[r][1] + neighbour_dy(j),
                                                 ps.key[r][2] + neighbour_dz(j), ps.key[r][3],
                                                 static_cast<uint64_t>(ps.key[r][4]), 0, 0u);
                    home[u] = h.index;
                    fp[u] = h.fp;
                    tg[u] = __ldg(reinterpret_cast<const unsigned long long *>(a.fine.tags) +
                                  (h.index & fmask));
                }
            }
            int64_t slot[kPP];
#pragma unroll
            for (int u = 0; u < kPP; ++u) {
                const int p = static_cast<int>(threadIdx.x) + u * kThreads;
                slot[u] = -1;
                if (p < np && tg[u] != kEmptyTag) {
                    slot[u] = (tg[u] & kFpMask) == static_cast<uint64_t>(fp[u])
                                  ? static_cast<int64_t>(home[u] & fmask)
                                  : probe_lookup(a.fine.tags, fmask, a.fine.probe_limit, home[u],
                                                 fp[u], a.seg_mask, 1);
                }
            }
            if (a.rec != nullptr) {  // records straight into shared memory (cp.async)
#pragma unroll
                for (int u = 0; u < kPP; ++u) {
                    const int p = static_cast<int>(threadIdx.x) + u * kThreads;
                    if (p < np) ps.found[p] = slot[u] >= 0;
                    if (slot[u] >= 0) {
                        const uint64_t *rp = reinterpret_cast<const uint64_t *>(a.rec + slot[u]);
                        cp_async_16(&ps.word[p][0], rp);
                        cp_async_16(&ps.word[p][2], rp + 2);
                    }
                }
                cp_async_wait_all();
            } else {
#pragma unroll
                for (int u = 0; u < kPP; ++u) {
                    const int p = static_cast<int>(threadIdx.x) + u * kThreads;
                    if (p < np) ps.found[p] = slot[u] >= 0;
                    if (slot[u] >= 0) {
                        const Effective e = fine_effective(a, slot[u]);
#pragma unroll
                        for (int c = 0; c < 3; ++c)
                            ps.word[p][c] = as_int ? static_cast<uint64_t>(e.isum[c])
                                                   : static_cast<uint64_t>(__double_as_longlong(e.fsum[c]));
                        ps.word[p][3] = static_cast<uint64_t>(__double_as_longlong(e.fcnt));
                    }
                }
            }
        }
        __syncthreads();
        // kLanesPerRow threads per row: integer pools (order-free) are summed over the
        // 27 cells in parallel and reduced by shuffles; float64 pools keep numpy's
        // (dx, dy, dz) order on the row's first lane, which then runs the ladder
        const int r = static_cast<int>(threadIdx.x) / kLanesPerRow;
        const int sub = static_cast<int>(threadIdx.x) % kLanesPerRow;
        Pool pool{{0, 0, 0}, 0, {0.0, 0.0, 0.0}, 0.0};
        if (as_int && int_cnt) {
            if (r < rows) {
                for (int j = sub; j < 27; j += kLanesPerRow) {
                    const int p = 27 * r + j;
                    if (!ps.found[p]) continue;
#pragma unroll
                    for (int c = 0; c < 3; ++c) pool.isum[c] += static_cast<int64_t>(ps.word[p][c]);
                    pool.icnt += static_cast<int64_t>(__longlong_as_double(ps.word[p][3]));
                }
            }
#pragma unroll
            for (int off = kLanesPerRow / 2; off > 0; off >>= 1) {
#pragma unroll
                for (int c = 0; c < 3; ++c)
                    pool.isum[c] += __shfl_xor_sync(kFull, static_cast<long long>(pool.isum[c]), off);
                pool.icnt += __shfl_xor_sync(kFull, static_cast<long long>(pool.icnt), off);
            }
        } else if (r < rows && sub == 0) {
            for (int j = 0; j < 27; ++j) {  // numpy's order for the float64 pools
                const int p = 27 * r + j;
                if (!ps.found[p]) continue;
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    if (as_int) pool.isum[c] += static_cast<int64_t>(ps.word[p][c]);
                    else pool.fsum[c] = dadd(pool.fsum[c], __longlong_as_double(ps.word[p][c]));
                }
                // count: float64 bits (the record's word; integral in integrate mode)
                if (int_cnt) pool.icnt += static_cast<int64_t>(__longlong_as_double(ps.word[p][3]));
                else pool.fcnt = dadd(pool.fcnt, __longlong_as_double(ps.word[p][3]));
            }
        }
        if (r < rows && sub == 0) {
            const int64_t row = ps.row[r];
            double contrib[3], ch[3];
#pragma unroll
            for (int c = 0; c < 3; ++c) contrib[c] = ps.contrib[r][c];
            const bool cf = ps.coarse_found[r];
            const Effective ce = cf ? ps.coarse[r] : Effective{};
            const int src = ladder_choose(pool, as_int, mode, fixed, a.thr, cf, ce,
                                          eff_is_int(a.coarse, mode), contrib, ch);
            const int64_t pixel = ps.pixel[r] - a.pixel_base;
            const uint64_t keep = l2_policy(PF_FLAT_POLICY);
            const bool in_image = pixel >= 0 && pixel < a.n_pixels;
            if (in_image) {
#pragma unroll
                for (int c = 0; c < 3; ++c)
                    red_add_f64(a.flat + 3 * pixel + c, dmul(ps.tp[r][c], ch[c]), keep);
            }
            if (a.source) a.source[row] = static_cast<uint8_t>(src);
            if (a.chosen) {
#pragma unroll
                for (int c = 0; c < 3; ++c) a.chosen[3 * row + c] = ch[c];
            }
            if (!in_image) atomicAdd(&bs.v[PF_STAT_BAD_PIXELS], 1u);
            atomicAdd(&bs.v[PF_STAT_SOURCE_FINE + src], 1u);
        }
        __syncthreads();
    }
    __syncthreads();
    stats_flush(bs, a.stats, false);
}

// flat[0, m) = 0 (two words per thread) and *counter = 0: a chain kernel instead of
// cudaMemsetAsync, which would break the frame's PDL chain.
__global__ void __launch_bounds__(kThreads) zero_kernel(double *flat, int64_t m, int64_t *counter) {
    pdl_wait();
    const int64_t k = 2 * (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x);
    if (k + 1 < m) {
        reinterpret_cast<double2 *>(flat)[k / 2] = make_double2(0.0, 0.0);
    } else if (k < m) {
        flat[k] = 0.0;
    }
    if (counter != nullptr && k == 0) *counter = 0;
}

__global__ void __launch_bounds__(kThreads)
finalize_image_kernel(const double *__restrict__ base, const double *__restrict__ flat,
                      double *__restrict__ image, int64_t n, double spp) {
    pdl_wait();
    const int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (k < n) image[k] = dadd(base[k], ddiv(flat[k], spp));
}

// The resolve rungs after the effective records exist: the fine rung (keys from the
// insert pass, or rebuilt), the work rows' keys, the neighbourhood pool + coarse rung +
// ladder + composite.
static int launch_rungs(const char *fn, const ResolveArgs &a, int64_t n, bool have_keys,
                        bool have_fb_keys, cudaStream_t st) {
    if (have_keys)
        launch_pdl(resolve_main_kernel<kResolveKV, true>, dim3(blocks_for(n, kThreads * kResolveKV)),
                   dim3(kThreads), st, a);
    else
        launch_pdl(resolve_main_kernel<1, false>, dim3(blocks_for(n, kThreads)), dim3(kThreads),
                   st, a);
    if (int rc = check_launch(fn)) return rc;
    if (have_fb_keys) {
        static const int per_sm = resident_blocks(fallback_keys_kernel, kThreads);
        int64_t kb = (n + kThreads - 1) / kThreads;
        const int64_t kcap = static_cast<int64_t>(sm_count()) * per_sm;
        if (kb > kcap) kb = kcap;
        launch_pdl(fallback_keys_kernel, dim3(static_cast<unsigned>(kb)), dim3(kThreads), st, a);
        if (int rc = check_launch(fn)) return rc;
        static const int per_sm_pool = resident_blocks(resolve_pool_kernel, kThreads);
        int64_t pb = (n + kPoolRows - 1) / kPoolRows;
        const int64_t pcap = static_cast<int64_t>(sm_count()) * per_sm_pool;
        if (pb > pcap) pb = pcap;
        launch_pdl(resolve_pool_kernel, dim3(static_cast<unsigned>(pb)), dim3(kThreads), st, a);
    } else {
        int64_t fb_blocks = (n + kWarps - 1) / kWarps;
        const int64_t cap = static_cast<int64_t>(sm_count()) * 8;
        if (fb_blocks > cap) fb_blocks = cap;
        launch_pdl(resolve_fallback_kernel, dim3(static_cast<unsigned>(fb_blocks)), dim3(kThreads),
                   st, a);
    }
    return check_launch(fn);
}

}  // namespace pf

using namespace pf;

// The fused insert.  Its last_touch stores are deferred to a sweep over the occupied
// slots: run here unless the caller (pf_filter_frame) folds it into the resolve's
// effective-record sweep (defer_touch).
static int insert_frame(const char *fn, const pf_config *cfg, const pf_vertices *v,
                        const pf_table *fine, const pf_table *coarse, uint64_t stream_base_accum,
                        int64_t frame, int64_t *stats, pf_evict_event *events,
                        int64_t *event_count, int64_t event_capacity, const int32_t *abort_flag,
                        uint64_t stream_base_lookup, uint64_t *lookup_keys, bool defer_touch,
                        void *stream) {
    if (lookup_keys && fine && fine->capacity > (1ll << 32))
        return fail_arg(fn, "packed lookup keys need a fine capacity <= 2^32");
    if (int rc = validate_vertices(fn, v, cfg)) return rc;
    pf_config kc;
    if (int rc = prepare_config(fn, cfg, &kc)) return rc;
    if (int rc = validate_table(fn, fine)) return rc;
    if (coarse) {
        if (int rc = validate_table(fn, coarse)) return rc;
        if (coarse->sum_mode != fine->sum_mode) return fail_arg(fn, "fine/coarse sum_mode differ");
    }
    if (!stats) return fail_arg(fn, "stats is NULL");
    if (v->n > 0 && !v->contribution) return fail_arg(fn, "contribution is NULL");
    if (v->n == 0) return PF_OK;
    const pf_table c = coarse ? *coarse : *fine;
    static const int per_sm_fixed = resident_blocks(insert_frame_kernel<true>, kThreads);
    static const int per_sm_float = resident_blocks(insert_frame_kernel<false>, kThreads);
    const int64_t tiles = (v->n + kThreads - 1) / kThreads;
    int64_t cap = static_cast<int64_t>(sm_count()) *
                  (fine->sum_mode == PF_SUM_FIXED ? per_sm_fixed : per_sm_float);
    const unsigned g = static_cast<unsigned>(tiles < cap ? tiles : cap);
    launch_pdl(fine->sum_mode == PF_SUM_FIXED ? insert_frame_kernel<true> : insert_frame_kernel<false>,
               dim3(g), dim3(kThreads), as_stream(stream), kc, *v, *fine, c, coarse != nullptr,
               stream_base_accum, frame, stats, events, event_count, event_capacity, abort_flag,
               stream_base_lookup, lookup_keys);
    if (int rc = check_launch(fn)) return rc;
    return defer_touch ? PF_OK
                       : launch_post_insert(fn, *fine, coarse, kc, nullptr, frame, as_stream(stream));
}

// The resolve phase; touch_frame != kNoTouch also finishes a deferred insert's last_touch.
static int resolve_frame(const char *fn, const pf_config *cfg, const pf_vertices *v,
                         const pf_table *fine, const pf_table *coarse, uint64_t stream_base_lookup,
                         uint64_t stream_base_coarse, int64_t spp, const double *base_image,
                         int64_t n_pixels, double *image, double *flat, int64_t *work,
                         int64_t *work_count, uint8_t *source, double *chosen, int64_t *stats,
                         const uint64_t *lookup_keys, uint64_t *eff_records,
                         int64_t *fallback_keys, int64_t touch_frame, void *stream,
                         bool fold_base = false, int32_t *const *occ_out = nullptr,
                         int64_t *occ_count_out = nullptr) {
    if (int rc = validate_vertices(fn, v, cfg)) return rc;
    pf_config kc;
    if (int rc = prepare_config(fn, cfg, &kc)) return rc;
    if (int rc = validate_table(fn, fine)) return rc;
    if (coarse)
        if (int rc = validate_table(fn, coarse)) return rc;
    if (spp < 1) return fail_arg(fn, "spp must be >= 1");
    if (n_pixels < 0 || !base_image || !image || !flat || !stats)
        return fail_arg(fn, "image buffers / stats are NULL");
    if (v->n > 0 && (!v->throughput || !v->contribution || !work || !work_count))
        return fail_arg(fn, "throughput/contribution/work is NULL");
    cudaStream_t st = as_stream(stream);
    if (v->n == 0) {  // only the image: base + 0 / spp
        launch_pdl(zero_kernel, dim3(blocks_for(3 * n_pixels / 2 + 1, kThreads)), dim3(kThreads),
                   st, flat, 3 * n_pixels, static_cast<int64_t *>(nullptr));
    } else {
        ResolveArgs a;
        a.cfg = kc;
        a.v = *v;
        a.fine = *fine;
        a.coarse = coarse ? *coarse : *fine;
        a.has_coarse = coarse != nullptr;
        a.h0_lookup = stream_base_lookup;
        a.h0_coarse = stream_base_coarse;
        a.flat = flat;
        a.work = work;
        a.work_count = work_count;
        a.wcap = work_list_capacity(v->n);
        a.source = source;
        a.chosen = chosen;
        a.stats = stats;
        a.thr = static_cast<double>(cfg->low_count_threshold > 1 ? cfg->low_count_threshold : 1);
        a.lk_keys = lookup_keys;
        a.rec = reinterpret_cast<const ulonglong4 *>(eff_records);
        a.n_pixels = n_pixels;
        a.fb_keys = fallback_keys;
        a.pixel_base = 0;
        a.seg_mask = ~0ull;
        a.crec = nullptr;
        // At spp = 1 (fold_base) the composite goes straight into the image, which
        // starts at base + 0.0: image = base + flat / 1 without the finalize pass.  A pixel
        // with one vertex gets RN(base + c) as the reference does (and base + 0.0 with
        // none); with several, the float sums' order changes as it already does with
        // the order of the composite REDs.
        const bool fold = fold_base && spp == 1 &&
                          ((reinterpret_cast<uintptr_t>(image) |
                            reinterpret_cast<uintptr_t>(base_image)) & 15) == 0;
        if (fold) a.flat = image;
        // flat = 0 (or base) and the work counter = 0 ride on the effective-record sweep
        if (int rc = launch_post_insert(fn, *fine, coarse, kc, eff_records, touch_frame, st,
                                        a.flat, 3 * n_pixels, work_count,
                                        fold ? base_image : nullptr,
                                        occ_count_out ? occ_out[0] : nullptr,
                                        occ_count_out ? occ_out[1] : nullptr, occ_count_out))
            return rc;
        if (int rc = launch_rungs(fn, a, v->n, lookup_keys != nullptr, fallback_keys != nullptr, st))
            return rc;
        if (fold) return check_launch(fn);
    }
    const int64_t m = 3 * n_pixels;
    if (m > 0)
        launch_pdl(finalize_image_kernel, dim3(blocks_for(m, kThreads)), dim3(kThreads), st,
                   static_cast<const double *>(base_image), static_cast<const double *>(flat),
                   image, m, static_cast<double>(spp));
    return check_launch(fn);
}

extern "C" {

int pf_insert_frame(const pf_config *cfg, const pf_vertices *v, const pf_table *fine,
                    const pf_table *coarse, uint64_t stream_base_accum, int64_t frame,
                    int64_t *stats, pf_evict_event *events, int64_t *event_count,
                    int64_t event_capacity, const int32_t *abort_flag,
                    uint64_t stream_base_lookup, uint64_t *lookup_keys, void *stream) {
    return insert_frame("pf_insert_frame", cfg, v, fine, coarse, stream_base_accum, frame, stats,
                        events, event_count, event_capacity, abort_flag, stream_base_lookup,
                        lookup_keys, false, stream);
}

int pf_resolve_frame(const pf_config *cfg, const pf_vertices *v, const pf_table *fine,
                     const pf_table *coarse, uint64_t stream_base_lookup,
                     uint64_t stream_base_coarse, int64_t spp, const double *base_image,
                     int64_t n_pixels, double *image, double *flat, int64_t *work,
                     int64_t *work_count, uint8_t *source, double *chosen, int64_t *stats,
                     const uint64_t *lookup_keys, uint64_t *eff_records,
                     int64_t *fallback_keys, void *stream) {
    return resolve_frame("pf_resolve_frame", cfg, v, fine, coarse, stream_base_lookup,
                         stream_base_coarse, spp, base_image, n_pixels, image, flat, work,
                         work_count, source, chosen, stats, lookup_keys, eff_records,
                         fallback_keys, kNoTouch, stream);
}

int pf_resolve_replica(const pf_config *cfg, const pf_vertices *v, const pf_replica *rp,
                       uint64_t stream_base_lookup, uint64_t stream_base_coarse,
                       const uint64_t *lookup_keys, double *flat,
                       int64_t n_pixels, int64_t pixel_base, int64_t *work,
                       int64_t *work_count, int64_t *fallback_keys, uint8_t *source,
                       double *chosen, int64_t *stats, void *stream) {
    const char *fn = "pf_resolve_replica";
    if (int rc = validate_vertices(fn, v, cfg)) return rc;
    pf_config kc;
    if (int rc = prepare_config(fn, cfg, &kc)) return rc;
    if (rp == nullptr || !rp->fine_tags || !rp->fine_records || !is_pow2(rp->capacity) ||
        rp->probe_limit < 1 || rp->slice_log2 < 1 || (1ll << rp->slice_log2) > rp->capacity ||
        (rp->coarse_tags == nullptr) != (rp->coarse_records == nullptr))
        return fail_arg(fn, "bad replica");
    if (n_pixels < 0 || !flat || !stats) return fail_arg(fn, "flat / stats are NULL");
    if (v->n > 0 && (!v->throughput || !v->contribution || !work || !work_count ||
                     !fallback_keys || !lookup_keys))
        return fail_arg(fn, "throughput/contribution/work/keys is NULL");
    cudaStream_t st = as_stream(stream);
    if (cudaMemsetAsync(flat, 0, sizeof(double) * 3 * n_pixels, st) != cudaSuccess)
        return check_launch(fn);
    if (v->n == 0) return PF_OK;
    if (cudaMemsetAsync(work_count, 0, sizeof(int64_t) * PF_WORK_LISTS, st) != cudaSuccess)
        return check_launch(fn);
    pf_table view{};
    view.cnt_stride = view.cold_stride = 1;
    view.sum_stride = view.hsum_stride = 3;
    view.sum_cstride = 1;
    view.tags = rp->fine_tags;
    view.capacity = rp->capacity;
    view.sum_mode = rp->sum_mode;
    view.probe_limit = rp->probe_limit;
    pf_table cview = view;
    cview.tags = rp->coarse_tags ? rp->coarse_tags : rp->fine_tags;
    ResolveArgs a;
    a.cfg = kc;
    a.v = *v;
    a.fine = view;
    a.coarse = cview;
    a.has_coarse = rp->coarse_tags != nullptr;
    a.h0_lookup = stream_base_lookup;
    a.h0_coarse = stream_base_coarse;
    a.flat = flat;
    a.work = work;
    a.work_count = work_count;
    a.wcap = work_list_capacity(v->n);
    a.source = source;
    a.chosen = chosen;
    a.stats = stats;
    a.thr = static_cast<double>(cfg->low_count_threshold > 1 ? cfg->low_count_threshold : 1);
    a.lk_keys = lookup_keys;
    a.rec = reinterpret_cast<const ulonglong4 *>(rp->fine_records);
    a.n_pixels = n_pixels;
    a.fb_keys = fallback_keys;
    a.pixel_base = pixel_base;
    a.seg_mask = (1ull << rp->slice_log2) - 1;
    a.crec = reinterpret_cast<const ulonglong4 *>(rp->coarse_records);
    return launch_rungs(fn, a, v->n, true, true, st);
}

int pf_finalize_image(const double *base_image, const double *flat, double *image,
                      int64_t n_pixels, int64_t spp, void *stream) {
    const char *fn = "pf_finalize_image";
    if (n_pixels < 0 || spp < 1) return fail_arg(fn, "n_pixels must be >= 0 and spp >= 1");
    const int64_t m = 3 * n_pixels;
    if (m == 0) return PF_OK;
    if (!base_image || !flat || !image) return fail_arg(fn, "image buffers are NULL");
    finalize_image_kernel<<<blocks_for(m, kThreads), kThreads, 0, as_stream(stream)>>>(
        base_image, flat, image, m, static_cast<double>(spp));
    return check_launch(fn);
}

int pf_filter_frame(const pf_config *cfg, const pf_vertices *v, const pf_table *fine,
                    const pf_table *coarse, int64_t frame, uint64_t stream_base_accum,
                    uint64_t stream_base_lookup, uint64_t stream_base_coarse, int64_t spp,
                    const double *base_image, int64_t n_pixels, double *image, uint8_t *source,
                    double *chosen, const pf_frame_buffers *b, void *stream) {
    const char *fn = "pf_filter_frame";
    if (b == nullptr || cfg == nullptr) return fail_arg(fn, "config/buffers are NULL");
    if (!b->acc_stats || !b->res_stats) return fail_arg(fn, "stats buffers are NULL");
    cudaStream_t st = as_stream(stream);
    auto mark = [&](int k) {
        if (b->phase_events[k]) cudaEventRecord(static_cast<cudaEvent_t>(b->phase_events[k]), st);
    };
    mark(0);
    if (b->occ_count_in != nullptr && (!b->occ_in[0] || (coarse && !b->occ_in[1])))
        return fail_arg(fn, "occ_count_in without the occupied-slot lists");
    if (b->occ_count_in != nullptr && b->occ_count_in == b->occ_count_out)
        return fail_arg(fn, "occ_count_in and occ_count_out must be different buffers");
    // the lists this frame leaves behind (written by the effective-record sweep, which
    // runs only with a non-empty stream)
    const bool occ_out = b->occ_count_out != nullptr && b->occ_out[0] != nullptr &&
                         (!coarse || b->occ_out[1] != nullptr) && v->n > 0;
    // prologue in one launch: generation fold on both tables (src/pipeline.py:331-333),
    // the input check and the counter resets, side by side over the grid
    if (b->bad_flag && cudaMemsetAsync(b->bad_flag, 0, sizeof(int32_t), st) != cudaSuccess)
        return check_launch(fn);
    if (int rc = frame_prologue(fine, coarse, frame, cfg->temporal_mode, cfg->ema_alpha,
                                cfg->delta_max, cfg->sample_cap, b->horizon_clears_fine,
                                b->horizon_clears_coarse, v->n > 0 ? v->contribution : nullptr,
                                3 * v->n, b->bad_flag, b->acc_stats, PF_STAT_COUNT, b->res_stats,
                                PF_STAT_COUNT, b->event_count, st, b->occ_in[0], b->occ_in[1],
                                b->occ_count_in, occ_out ? b->occ_count_out : nullptr))
        return rc;
    // accumulate_phase (fused, flag-guarded) + the resolve phase's lookup keys
    mark(1);
    // (last_touch stores deferred to the resolve's effective-record sweep)
    if (int rc = insert_frame(fn, cfg, v, fine, coarse, stream_base_accum, frame, b->acc_stats,
                              b->events, b->event_count, b->event_capacity, b->bad_flag,
                              stream_base_lookup, b->lookup_keys, true, stream))
        return rc;
    mark(2);
    const int rc = resolve_frame(fn, cfg, v, fine, coarse, stream_base_lookup, stream_base_coarse,
                                 spp, base_image, n_pixels, image, b->flat, b->work,
                                 b->work_count, source, chosen, b->res_stats, b->lookup_keys,
                                 b->eff_records, b->fallback_keys, frame, stream, true,
                                 occ_out ? b->occ_out : nullptr,
                                 occ_out ? b->occ_count_out : nullptr);
    mark(3);
    return rc;
}

}  // extern "C"
