/*
 * pathfilter_b200 -- C ABI of the B200-native hashed path-space filter.
 *
 * Drop-in boundary for the reference package `pathfilter`
 * (/root/reference/pkg/src/pathfilter, cited as src/<file>:<line>).
 * Every entry point is stream-ordered, takes DEVICE pointers (B200 HBM) and
 * plain sizes, returns 0 on success or a nonzero pf_status, and never throws.
 * pf_last_error() describes the most recent failure on the calling thread.
 *
 * Two groups of entry points:
 *   1. the reference kernel-module ABI (src/_backend.py:14-42, src/_native.pyx:261-295):
 *      pf_accumulate_fixed / pf_accumulate_float / pf_lookup_slots -- same arrays,
 *      same in-place mutation, same per-vertex outputs;
 *   2. the filter API (src/keys.py, src/table.py, src/pipeline.py): key build, fused
 *      frame insert, fused frame resolve, effective sums and the temporal update.
 */
#ifndef PATHFILTER_B200_H
#define PATHFILTER_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PF_ABI_VERSION 7

enum pf_status {
    PF_OK = 0,
    PF_ERR_ARGUMENT = 1,   /* bad size / null pointer / capacity not a power of two */
    PF_ERR_CUDA = 2,       /* a CUDA launch or API call failed (see pf_last_error) */
};

enum pf_temporal_mode { PF_INTEGRATE = 0, PF_FILTER = 1, PF_HYBRID = 2 };
enum pf_sum_mode { PF_SUM_FIXED = 0, PF_SUM_FLOAT = 1 };

/* FilterConfig (src/keys.py:30-79) reduced to what the device reads. */
typedef struct pf_config {
    double c_lod;            /* footprint_scale * s_pixels / base_voxel, evaluated on the host
                                exactly as src/keys.py:246 does */
    double base_voxel;
    double ema_alpha;
    double delta_max;
    double lod_threshold[32];/* [k] = smallest double r with floor(np.log2(r)) >= k, k=1..31
                                (exact floor(log2) of src/keys.py:247; [0] unused) */
    int32_t normal_bins;
    int32_t incident_angle_bins;
    int32_t include_normal;
    int32_t include_incident_angle;
    int32_t include_layer;
    int32_t normal_in_fingerprint;
    int32_t jitter;
    int32_t multi_level;
    int32_t coarse_delta;
    int32_t low_count_threshold;
    int32_t temporal_mode;   /* pf_temporal_mode */
    int32_t sample_cap;
    uint64_t lod_ulps[2];    /* filled by the library from lod_threshold (callers leave 0):
                                4-bit count of doubles between T[k] and 2^k, k = 0..31 */
    double inv_base_voxel;   /* filled by the library: RN(1 / base_voxel) */
    double lod_dist[32];     /* filled by the library: [k] = smallest distance d >= 0 with
                                RN(d * c_lod) >= lod_threshold[k] for k = 1..31, and
                                RN(d * c_lod) = +inf for k = 0; +inf when no finite d
                                reaches it, NaN unless 0 < c_lod < inf */
} pf_config;

/* VertexStream (src/tracer.py:66-104): row-major [n][3] float64 triples. */
typedef struct pf_vertices {
    const double *position;
    const double *normal;
    const double *omega_r;          /* may be NULL unless include_incident_angle */
    const double *contribution;
    const double *throughput;       /* may be NULL for insert-only calls */
    const int64_t *pixel;
    const int64_t *sample;
    const int64_t *layer_id;        /* may be NULL unless include_incident_angle/include_layer */
    const double *camera_distance;
    int64_t n;
} pf_vertices;

/* VoxelTable state (src/table.py:96-103).  Fields are addressed through strides, in
 * 8-byte words: slot s's count at counts + s * cnt_stride, its live sums at
 * sums + s * sum_stride + c * sum_cstride, hist_counts / last_touch / deltas at
 * ptr + s * cold_stride and hist_sums at hist_sums + s * hsum_stride + c; `tags` is
 * always dense.  The reference's SoA layout (the kernel-module ABI's caller-owned
 * arrays) is cnt 1, sum 3 / 1, cold 1, hsum 3.  The device-private VoxelTable keeps
 * tags and counts dense, the live sums channel-major (sum_stride 1, sum_cstride C: the
 * insert's three REDs per vertex land in three different lines, which the L2 atomic
 * units serve in parallel) and the fields only the per-frame sweeps touch in one
 * 64-byte cold record per slot (cold_stride = hsum_stride = 8: last_touch, hist_count,
 * delta, pad, hist_sum[3], pad). */
typedef struct pf_table {
    uint64_t *tags;                 /* [C]   EMPTY = 0xFFFFFFFF00000000 */
    void *sums;                     /* [C][3] int64 (fixed) or float64 (float) */
    int64_t *counts;                /* [C] */
    void *hist_sums;                /* [C][3] */
    int64_t *hist_counts;           /* [C] */
    int64_t *last_touch;            /* [C] */
    double *deltas;                 /* [C] */
    int64_t capacity;               /* power of two >= 2 */
    int32_t sum_mode;               /* pf_sum_mode */
    int32_t probe_limit;
    int32_t evict_min_age;
    int32_t evict_horizon;
    int32_t cnt_stride;             /* counts: slot stride                     (SoA: 1) */
    int32_t sum_stride;             /* sums: slot stride                       (SoA: 3) */
    int32_t cold_stride;            /* hist_counts, last_touch, deltas         (SoA: 1) */
    int32_t hsum_stride;            /* hist_sums: slot stride (channels adjacent; SoA: 3) */
    int64_t sum_cstride;            /* sums: channel stride                    (SoA: 1) */
} pf_table;

/* KeyArrays (src/keys.py:302-320); every pointer may be NULL (not written). */
typedef struct pf_key_out {
    int64_t *qx, *qy, *qz, *level;
    uint64_t *aux;
    uint64_t *index;
    uint32_t *fingerprint;
    double *jittered;               /* [n][3] */
} pf_key_out;

/* Per-frame counters written by the fused kernels (int64 device array). */
enum pf_stat_slot {
    PF_STAT_PROBE_FAILURES = 0,       /* fine table, status == 2 (src/pipeline.py:166) */
    PF_STAT_COARSE_PROBE_FAILURES = 1,/* src/pipeline.py:174 */
    PF_STAT_PROBE_LEN_SUM = 2,        /* sum of fine probe_len (collisions = this - n) */
    PF_STAT_EVICTIONS = 3,            /* fine-table status == 1 */
    PF_STAT_COARSE_EVICTIONS = 4,
    PF_STAT_SOURCE_FINE = 5,          /* src/pipeline.py:45-48 */
    PF_STAT_SOURCE_NEIGHBORHOOD = 6,
    PF_STAT_SOURCE_COARSE = 7,
    PF_STAT_SOURCE_UNFILTERED = 8,
    PF_STAT_FALLBACK_ROWS = 9,        /* rows that left the fine rung (resolve work list) */
    PF_STAT_BAD_PIXELS = 10,          /* rows whose pixel lies outside the image (skipped) */
    PF_STAT_SHARD_RECORDS = 11,       /* sharded insert: records applied by this owner */
    PF_STAT_SHARD_REQUESTS = 12,      /* sharded resolve: lookups answered by this owner */
    PF_STAT_HIST_BASE = 16,           /* [16 + k] = #vertices with fine probe_len == k, k < 256 */
    PF_STAT_COUNT = 16 + 256
};

/* The resolve's work list (rows that leave the fine rung) is PF_WORK_LISTS lists, one
 * per group of resolve blocks (256 rows each), so its append counters are not one hot
 * L2 atomic: work needs PF_WORK_ROWS(n) entries and work_count PF_WORK_LISTS. */
#define PF_WORK_LISTS 64
#define PF_WORK_ROWS(n) \
    ((((((n) + 255) / 256) + PF_WORK_LISTS - 1) / PF_WORK_LISTS) * PF_WORK_LISTS * 256)

/* Eviction event record (src/table.py:72-77, 137-141). */
typedef struct pf_evict_event {
    int64_t vertex;                 /* row in the batch */
    int64_t slot;
    uint64_t victim_tag;
    int64_t victim_touch;
} pf_evict_event;

int pf_abi_version(void);
/* Source id of the build: SHA-256 prefix of the CUDA sources, headers and nvcc flags
 * (paper_1902_05942_b200/_lib.py: source_id).  Ties a binary to the tree it came from. */
const char *pf_build_id(void);
const char *pf_last_error(void);
int pf_device_sm_count(void);
/* Host only: the config every entry point actually runs with -- `in` plus the
 * library-derived fields (lod_ulps, inv_base_voxel, lod_dist).  Validates thresholds. */
int pf_prepare_config(const pf_config *in, pf_config *out);
/* Host only: page-lock (cudaHostRegister) / release a caller-owned host buffer in place,
 * so the kernel-module drop-in stages numpy tables at DMA rate.  A failed registration
 * (already registered, not supported) returns PF_ERR_CUDA and leaves no CUDA error
 * pending; the buffer stays usable as pageable memory. */
int pf_host_register(void *ptr, int64_t bytes);
/* Host only: set aside `bytes` of L2 for lines accessed with an evict_last policy (the
 * tables' and the composite's REDs); -1 = the device maximum.  Without a set-aside the
 * evict_last hint does not keep lines resident.  *applied (may be NULL) = the size set. */
int pf_set_l2_persisting(int64_t bytes, int64_t *applied);
int pf_host_unregister(void *ptr);

/* ---- 1. reference kernel-module ABI ------------------------------------------------ */

/* src/_native.pyx:261-266 accumulate_fixed (sums/hist_sums int64) and :268-272
 * accumulate_float (float64).  Per-vertex outputs status u8, slots i64, probe_len u8,
 * victim_tags u64, victim_touch i64 (any may be NULL).  ordered != 0 reproduces the
 * reference's sequential (threads=1) slot layout exactly; ordered == 0 is the
 * massively parallel insert whose per-key sums, counts and statuses are identical
 * but whose slot order among keys that first appear in the same batch and share a
 * probe window may differ (as the reference's own threads>1 mode may). */
int pf_accumulate_fixed(uint64_t *tags, int64_t *sums, int64_t *counts, int64_t *hist_sums,
                        int64_t *hist_counts, int64_t *last_touch, double *deltas,
                        int64_t capacity, const uint64_t *idx, const uint32_t *fp,
                        const double *vals, int64_t n, int64_t frame, int32_t probe_limit,
                        int32_t evict_min_age, int32_t ordered, uint8_t *status,
                        int64_t *slots, uint8_t *probe_len, uint64_t *victim_tags,
                        int64_t *victim_touch, void *stream);
int pf_accumulate_float(uint64_t *tags, double *sums, int64_t *counts, double *hist_sums,
                        int64_t *hist_counts, int64_t *last_touch, double *deltas,
                        int64_t capacity, const uint64_t *idx, const uint32_t *fp,
                        const double *vals, int64_t n, int64_t frame, int32_t probe_limit,
                        int32_t evict_min_age, int32_t ordered, uint8_t *status,
                        int64_t *slots, uint8_t *probe_len, uint64_t *victim_tags,
                        int64_t *victim_touch, void *stream);
/* accumulate_batch on a table described by pf_table (any layout: the device-private
 * interleaved VoxelTable or SoA); sum_mode picks fixed / float, probe_limit and
 * evict_min_age come from the table.  Outputs as pf_accumulate_fixed. */
int pf_accumulate_table(const pf_table *t, const uint64_t *idx, const uint32_t *fp,
                        const double *vals, int64_t n, int64_t frame, int32_t ordered,
                        uint8_t *status, int64_t *slots, uint8_t *probe_len,
                        uint64_t *victim_tags, int64_t *victim_touch, void *stream);
/* src/_native.pyx:275-295 lookup_slots: first matching slot, -1 when absent. */
int pf_lookup_slots(const uint64_t *tags, int64_t capacity, const uint64_t *idx,
                    const uint32_t *fp, int64_t n, int32_t probe_limit, int64_t *out,
                    void *stream);

/* ---- 2. filter API ---------------------------------------------------------------- */

/* keys.make_key_arrays (src/keys.py:342-359) with explicit jitter draws u1/u2
 * (NULL = no jitter). */
int pf_make_key_arrays(const pf_config *cfg, const pf_vertices *v, const double *u1,
                       const double *u2, int32_t level_delta, pf_key_out *out, void *stream);
/* pipeline.vertex_keys (src/pipeline.py:126-135): draws from the counter RNG of
 * src/rng.py:62-78 keyed by path id; stream_base = mix64(seed ^ stream_tag*G). */
int pf_vertex_keys(const pf_config *cfg, const pf_vertices *v, uint64_t stream_base,
                   int32_t level_delta, pf_key_out *out, void *stream);
/* keys.hash_arrays (src/keys.py:327-339); normal_fp_bins may be NULL. */
int pf_hash_arrays(const int64_t *qx, const int64_t *qy, const int64_t *qz,
                   const int64_t *level, const uint64_t *aux, const uint32_t *normal_fp_bins,
                   int64_t n, uint64_t *index, uint32_t *fingerprint, void *stream);

/* Fused accumulate_phase (src/pipeline.py:152-175): keys (stream 2) for the fine
 * and, if coarse != NULL, the coarse table (level + coarse_delta), each inserted
 * with warp-merged atomics.  stats: int64[PF_STAT_COUNT] accumulated (not cleared);
 * events: optional eviction log of capacity `event_capacity` with its int64 counter.
 * abort_flag (device int32, may be NULL): when nonzero at launch the kernel leaves
 * the tables untouched (set by pf_check_contributions for invalid input).
 * lookup_keys (may be NULL): also emit the resolve phase's fine lookup key
 * (stream_base_lookup, level_delta 0) for every vertex as one packed word,
 * fingerprint << 32 | (slot index & 0xFFFFFFFF) (fine capacity <= 2^32), so
 * pf_resolve_frame does not rebuild it from the vertex buffer. */
int pf_insert_frame(const pf_config *cfg, const pf_vertices *v, const pf_table *fine,
                    const pf_table *coarse, uint64_t stream_base_accum, int64_t frame,
                    int64_t *stats, pf_evict_event *events, int64_t *event_count,
                    int64_t event_capacity, const int32_t *abort_flag,
                    uint64_t stream_base_lookup, uint64_t *lookup_keys, void *stream);

/* Fused resolve_phase (src/pipeline.py:207-283): lookup keys, fine rung, 3x3x3
 * neighbourhood, coarse rung, ladder, composite.  flat: float64[n_pixels][3]
 * scratch; work: int64 scratch of PF_WORK_ROWS(n) entries plus work_count
 * (int64[PF_WORK_LISTS]);
 * image = base_image + flat/spp.  source (u8[n]) and chosen (f64[n][3]) may be NULL.
 * lookup_keys: the packed keys pf_insert_frame emitted for the same vertices and
 * stream_base_lookup, or NULL to build them here.
 * eff_records (may be NULL): scratch of 4 * fine->capacity uint64; when given, the
 * fine table's effective (sum, count) is computed once per occupied slot into one
 * 32-byte record that every lookup then reads.
 * fallback_keys (may be NULL): scratch of 8 * n int64; when given, the lookup key and
 * coarse slot of every row that leaves the fine rung are built (and probed) one row per
 * thread before the 3x3x3 pool instead of by one lane per row. */
int pf_resolve_frame(const pf_config *cfg, const pf_vertices *v, const pf_table *fine,
                     const pf_table *coarse, uint64_t stream_base_lookup,
                     uint64_t stream_base_coarse, int64_t spp, const double *base_image,
                     int64_t n_pixels, double *image, double *flat, int64_t *work,
                     int64_t *work_count, uint8_t *source, double *chosen, int64_t *stats,
                     const uint64_t *lookup_keys, uint64_t *eff_records,
                     int64_t *fallback_keys, void *stream);

/* Device scratch and outputs of pf_filter_frame (all device pointers). */
typedef struct pf_frame_buffers {
    int64_t *acc_stats;             /* int64[PF_STAT_COUNT]: accumulate counters (zeroed) */
    int64_t *res_stats;             /* int64[PF_STAT_COUNT]: resolve counters (zeroed) */
    pf_evict_event *events;         /* eviction log (may be NULL) ... */
    int64_t *event_count;           /* ... and its counter (zeroed) */
    int64_t event_capacity;
    int32_t *bad_flag;              /* input check flag, or NULL to skip validation */
    int64_t *horizon_clears_fine;   /* int64[1] counters incremented by begin_frame */
    int64_t *horizon_clears_coarse;
    uint64_t *lookup_keys;          /* n: packed lookup keys handed from insert to resolve */
    uint64_t *eff_records;          /* 4 * fine->capacity */
    double *flat;                   /* [n_pixels][3] */
    int64_t *work;                  /* PF_WORK_ROWS(n) */
    int64_t *work_count;            /* PF_WORK_LISTS */
    int64_t *fallback_keys;         /* 8 * n, or NULL (see pf_resolve_frame) */
    void *phase_events[4];          /* optional cudaEvent_t recorded at frame start, just
                                       before the insert kernel, after it, at frame end */
    /* Occupied-slot lists (optional).  occ_out[0] / occ_out[1] (int32[fine / coarse
     * capacity]) receive the slots occupied when this frame ends and occ_count_out
     * (int64[2], zeroed here) their counts.  A later frame may pass them back as occ_in /
     * occ_count_in ONLY if nothing changed either table in between: its begin_frame then
     * folds exactly those slots instead of sweeping the tag arrays.  NULL: sweep. */
    int32_t *occ_in[2];
    const int64_t *occ_count_in;
    int32_t *occ_out[2];
    int64_t *occ_count_out;
} pf_frame_buffers;

/* One whole frame of the filter -- src/pipeline.py:321-363 (render_frame) minus the
 * tracer -- in one call and one stream: begin_frame on both tables, the input check,
 * the flag-guarded fused insert, and the resolve.  The host reads bad_flag afterwards
 * (nonzero: the tables were left untouched and the inputs must be rejected). */
int pf_filter_frame(const pf_config *cfg, const pf_vertices *v, const pf_table *fine,
                    const pf_table *coarse, int64_t frame, uint64_t stream_base_accum,
                    uint64_t stream_base_lookup, uint64_t stream_base_coarse, int64_t spp,
                    const double *base_image, int64_t n_pixels, double *image, uint8_t *source,
                    double *chosen, const pf_frame_buffers *buffers, void *stream);

/* image = base + flat / spp over n_pixels RGB pixels (the last line of
 * src/pipeline.py:282-283). */
int pf_finalize_image(const double *base_image, const double *flat, double *image,
                      int64_t n_pixels, int64_t spp, void *stream);

/* ---- 3. key-sharded multi-GPU frame --------------------------------
 * G ranks (one per GPU, G a power of two <= 64) hold the global fine and coarse
 * tables of capacity C = 2^log2_capacity as G contiguous slices of S = C/G home
 * slots: owner(home) = home >> (log2 C - log2 G).  The owner keeps its slice in a local
 * pf_table of capacity S indexed by home - rank*S; probe windows wrap within the slice
 * (with G == 1 this is exactly the single-GPU table).
 *
 * One frame, per rank (the exchanges are the caller's collectives, e.g. NCCL):
 *   pf_begin_frame (both local slices) ; pf_shard_keys ; pf_shard_emit
 *   -> all-to-all of the records (int64[5]) ; pf_shard_apply ; pf_shard_reset
 *   pf_shard_publish -> all-gather of the entries (uint64[6]) into a replica of the
 *   whole table ; pf_replica_update (clear last frame's entries, write this frame's)
 *   pf_resolve_replica (the single-GPU resolve against the replica) ; pf_finalize_image
 * Every rank pre-aggregates its vertices per distinct key before sending (fixed-point
 * sums are exactly associative), so the record exchange carries one record per
 * distinct key per rank; the published entries are the occupied cells only.
 *
 * Aggregation table key: kind << 61 | home << 32 | fingerprint (home < 2^29), EMPTY
 * = ~0; kinds 0 fine record, 1 coarse record.  Record = int64[5] {key, sum[3], weight}
 * with sums in the tables' sum_mode.  Entry = uint64[6] {global slot | coarse << 62,
 * tag, effective sum[3] (int64 or float64 bits, as VoxelTable.effective), effective
 * count as float64 bits}. */
typedef struct pf_shard {
    int32_t rank;
    int32_t world;                  /* power of two, <= 64 */
    int32_t log2_capacity;          /* global C of both tables, C >= world, <= 2^29 */
    int32_t sum_mode;               /* pf_sum_mode of both tables */
    uint64_t *agg_keys;             /* [agg_capacity], EMPTY = ~0 */
    int64_t *agg_sums;              /* [agg_capacity][3] */
    int64_t *agg_counts;            /* [agg_capacity] record weights */
    int64_t agg_capacity;           /* power of two >= 64; at most agg_capacity/2 keys a round */
    int32_t *distinct;              /* [agg_capacity/2] claimed slots in claim order (-1 hole) */
    int64_t *n_distinct;            /* [1] slot reservations of the current round */
    int32_t *overflow;              /* [1] set when a round needed more than agg_capacity/2 keys */
    int64_t *owner_counts;          /* [2][world] records per owner (row 1 unused) */
    int64_t *owner_cursor;          /* [2][world] emit cursors */
} pf_shard;

/* Read-only replica of the global tables for the resolve (device arrays of C slots). */
typedef struct pf_replica {
    uint64_t *fine_tags;            /* [C] EMPTY where no owner published a cell */
    uint64_t *fine_records;         /* [C][4] effective records */
    uint64_t *coarse_tags;          /* [C] or NULL (no coarse table) */
    uint64_t *coarse_records;
    int64_t capacity;               /* C */
    int32_t slice_log2;             /* log2(C / world): probe windows wrap within slices */
    int32_t probe_limit;
    int32_t sum_mode;
    int32_t pad0;
} pf_replica;

/* Keys of every local vertex: the fine and coarse keys (jitter stream 2) go into the
 * aggregation table as records, the packed fine lookup key (stream 3; as
 * pf_insert_frame's lookup_keys) to lookup_keys (n) for pf_resolve_replica.
 * abort_flag as in pf_insert_frame. */
int pf_shard_keys(const pf_config *cfg, const pf_vertices *v, const pf_shard *sh,
                  int32_t has_coarse, uint64_t stream_base_accum, uint64_t stream_base_lookup,
                  const int32_t *abort_flag, uint64_t *lookup_keys, void *stream);
/* Write the round's records grouped by owner: owner o's records start at row
 * sum(owner_counts[0][:o]) of send_records.  No-op when overflow is set. */
int pf_shard_emit(const pf_shard *sh, int64_t *send_records, uint64_t *send_requests,
                  void *stream);
/* Owner side: insert received records into the local slices (warp-merged, weighted),
 * stats as pf_insert_frame (probe failures / histogram weighted by vertex count). */
int pf_shard_apply(const pf_shard *sh, const pf_table *fine, const pf_table *coarse,
                   const int64_t *records, int64_t n_records, int64_t frame, int64_t *stats,
                   void *stream);
/* Owner side: one entry per occupied local slot of both slices into `entries`
 * (capacity: occupied slots), their number into *count. */
int pf_shard_publish(const pf_shard *sh, const pf_config *cfg, const pf_table *fine,
                     const pf_table *coarse, uint64_t *entries, int64_t *count, void *stream);
/* Apply all-gathered entries to a replica: rank r's entries are rows
 * [r * stride, r * stride + counts[r]) of `entries` (counts: device int64[world]);
 * clear != 0 empties their slots instead (last frame's entries). */
int pf_replica_update(const pf_replica *replica, const uint64_t *entries, const int64_t *counts,
                      int32_t world, int64_t stride, int32_t clear, void *stream);
/* Empty the aggregation table (only the slots this round claimed) and its counters. */
int pf_shard_reset(const pf_shard *sh, void *stream);
/* resolve_phase (src/pipeline.py:207-283) of this rank's vertices against a replica:
 * the fine rung from lookup_keys (pf_shard_keys), the neighbourhood and
 * coarse rungs, the ladder, the composite into flat (pixels [pixel_base, pixel_base +
 * n_pixels), zeroed here).  work: PF_WORK_ROWS(n) int64 (+ work_count[PF_WORK_LISTS]),
 * fallback_keys: 8 * n int64 scratch. */
int pf_resolve_replica(const pf_config *cfg, const pf_vertices *v, const pf_replica *replica,
                       uint64_t stream_base_lookup, uint64_t stream_base_coarse,
                       const uint64_t *lookup_keys, double *flat,
                       int64_t n_pixels, int64_t pixel_base, int64_t *work,
                       int64_t *work_count, int64_t *fallback_keys, uint8_t *source,
                       double *chosen, int64_t *stats, void *stream);

/* ---- 4. phase one: the path tracer that produces the vertex stream ----
 * src/tracer.py:211-383 (_walk) with src/_native.pyx:83-167 (intersect_closest/any):
 * one path per (pixel, sample); the scene is a triangle soup in device memory. */
typedef struct pf_scene {
    const double *v0, *e1, *e2;     /* [m][3] triangle corner and edges (src/scene.py:170-195) */
    const double *normal;           /* [m][3] unit geometric normals */
    const double *emission;         /* [m][3] */
    const double *area;             /* [m] */
    const int32_t *material_id;     /* [m] */
    int64_t n_triangles;
    const double *albedo;           /* [k][3] */
    const double *glossy_weight;    /* [k] */
    const double *glossy_exponent;  /* [k] */
    int64_t n_materials;
    const int64_t *light_tri;       /* [L] triangles with emission > 0, ascending */
    int64_t n_lights;
    double background[3];
    double cam_pos[3], cam_right[3], cam_up[3], cam_fwd[3];  /* Camera.basis() */
    double ndc_scale_x;             /* 2.0 * tan(fov / 2) * (width / height), as Python */
    double ndc_scale_y;             /* 2.0 * tan(fov / 2) */
    int32_t width, height;
} pf_scene;

/* TraceOptions (src/tracer.py:35-43). */
typedef struct pf_trace_options {
    int32_t max_depth;
    int32_t rr_start;
    int32_t nee;
    int32_t select_k;
    int32_t pixel_jitter;
    int32_t pad0;
    double rr_lo, rr_hi;            /* rr_clamp */
    double diffuse_threshold;
} pf_trace_options;

/* Per-path results, row i for path i (device arrays; any vertex field may be NULL). */
typedef struct pf_path_out {
    double *base;                   /* [n][3] radiance not routed through the vertex */
    double *radiance;               /* [n][3] base + throughput * contribution */
    uint8_t *has_vertex;            /* [n] */
    double *position, *normal, *omega_r, *contribution, *throughput;  /* [n][3] */
    int64_t *layer_id;              /* [n] */
    double *camera_distance;        /* [n] */
} pf_path_out;

/* Trace n paths (pixels[i], samples[i]) with draws from (seed, STREAM_TRACE). */
int pf_trace_paths(const pf_scene *scene, const pf_trace_options *opt, uint64_t seed,
                   const int64_t *pixels, const int64_t *samples, int64_t n,
                   const pf_path_out *out, void *stream);

/* VoxelTable.effective (src/table.py:205-238) over all slots.  eff_sum is int64 for
 * (integrate, fixed) else float64; eff_count is int64 for integrate else float64. */
int pf_effective(const pf_table *t, int32_t mode, double ema_alpha, double delta_max,
                 void *eff_sum, void *eff_count, void *stream);

/* VoxelTable.begin_frame (src/table.py:242-298).  horizon_clears (int64[1]) is
 * incremented by the number of slots cleared. */
int pf_begin_frame(const pf_table *t, int64_t frame, int32_t mode, double ema_alpha,
                   double delta_max, int32_t sample_cap, int64_t *horizon_clears,
                   void *stream);

/* begin_frame on a fine and (optionally) a coarse table plus the input check of
 * `count` contributions (vals/bad may be NULL: no check; *bad is cleared first), in one
 * launch -- the prologue of a frame (pf_filter_frame, the sharded frame). */
int pf_begin_frame_checked(const pf_table *fine, const pf_table *coarse, int64_t frame,
                           int32_t mode, double ema_alpha, double delta_max, int32_t sample_cap,
                           int64_t *clears_fine, int64_t *clears_coarse, const double *vals,
                           int64_t count, int32_t *bad, void *stream);
/* Input validation of accumulate_batch (src/table.py:127-129): *bad (int32, device) is
 * set to 1 when any of the `count` float64 values is NaN, infinite or negative. */
int pf_check_contributions(const double *vals, int64_t count, int32_t *bad, void *stream);

/* Diagnostic: counts (into mismatches[0..1], int64 device) the inputs for which the
 * kernels' reciprocal-based division differs from IEEE division -- [0] random
 * operands, [1] quantiser divisors base_voxel*2^level.  Both must stay 0. */
int pf_selftest_division(uint64_t seed, int64_t n, double base_voxel, int64_t *mismatches,
                         void *stream);

/* temporal.reevaluation_deltas (src/temporal.py:60-92) after the host grouped the
 * replayed rows by voxel: voxel v owns rows order[offsets[v] .. offsets[v+1]) (stream
 * order); delta[v] = |mean_new - mean_old|_1 / (|mean_old|_1 + delta_eps) with the sums
 * in np.add.at's order.  c_old / c_new: [rows][3] contributions. */
int pf_segment_deltas(const int64_t *order, const int64_t *offsets, int64_t n_vox,
                      const double *c_old, const double *c_new, double delta_eps, double *delta,
                      void *stream);
/* Diagnostic: sin(x[i]) and cos(x[i]) as the library computes them for the jitter and
 * the tracer -- glibc's dbl-64 algorithm, equal to numpy's float64 sin/cos here. */
int pf_sincos(const double *x, int64_t n, double *s, double *c, void *stream);
/* Number of non-EMPTY tags (VoxelTable.occupancy numerator, src/table.py:302-303). */
int pf_count_occupied(const uint64_t *tags, int64_t capacity, int64_t *out, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* PATHFILTER_B200_H */
