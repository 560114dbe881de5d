/*
 * ORACLE -- TEST INFRASTRUCTURE ONLY.
 *
 * Sequential C restatement of the reference voxel-table kernels, used as the
 * CPU checker by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline
 * leg.  Nothing in paper_1902_05942_b200/ links or calls this file.
 *
 * Semantics follow the reference Cython kernels one step at a time:
 *   orc_accumulate  <- pkg/src/pathfilter/_native.pyx:186-258 (_accumulate_impl)
 *                      and its numpy twin _pykernels.py:91-155
 *   orc_lookup      <- pkg/src/pathfilter/_native.pyx:275-295 (lookup_slots)
 * Single-threaded, so every CAS of the reference is a plain compare+store.
 */
#include <math.h>
#include <stdint.h>
#include <string.h>

#define ORC_EMPTY 0xFFFFFFFF00000000ULL   /* table.py:39 */
#define ORC_FRESH 0xFF000000ULL           /* _native.pyx:18 */
#define ORC_AGE_MASK 0xFFFFFFULL          /* _native.pyx:75 */
#define ORC_FP_MASK 0xFFFFFFFFULL

static void orc_zero_cell(int fixed, void *sums, void *hist_sums, int64_t *counts,
                          int64_t *hist_counts, double *deltas, int64_t s)
{
    /* _native.pyx:170-183: the victim's live and history state is wiped */
    if (fixed) {
        memset((int64_t *)sums + 3 * s, 0, 3 * sizeof(int64_t));
        memset((int64_t *)hist_sums + 3 * s, 0, 3 * sizeof(int64_t));
    } else {
        double *a = (double *)sums + 3 * s, *b = (double *)hist_sums + 3 * s;
        for (int c = 0; c < 3; ++c) { a[c] = 0.0; b[c] = 0.0; }
    }
    counts[s] = 0;
    hist_counts[s] = 0;
    deltas[s] = 0.0;
}

int orc_accumulate(uint64_t *tags, void *sums, int fixed, int64_t *counts,
                   void *hist_sums, int64_t *hist_counts, int64_t *last_touch,
                   double *deltas, int64_t capacity,
                   const uint64_t *idx, const uint32_t *fp, const double *vals,
                   int64_t n, int64_t frame, int probe_limit, int evict_min_age,
                   uint8_t *status, int64_t *slots, uint8_t *probe_len,
                   uint64_t *victim_tags, int64_t *victim_touch)
{
    const uint64_t mask = (uint64_t)capacity - 1;
    for (int64_t i = 0; i < n; ++i) {
        const uint64_t home = idx[i] & mask;
        const uint64_t key_fp = (uint64_t)fp[i];
        const uint64_t incoming = (ORC_FRESH << 32) | key_fp;
        int64_t victim = -1, slot = -1;
        uint64_t victim_tag = 0;
        status[i] = 0;
        slots[i] = -1;
        probe_len[i] = 0;
        victim_tags[i] = 0;
        victim_touch[i] = 0;
        for (int j = 0; j < probe_limit; ++j) {
            const uint64_t s = (home + (uint64_t)j) & mask;
            const uint64_t tag = tags[s];
            probe_len[i] = (uint8_t)(j + 1);
            if (tag == ORC_EMPTY) {          /* first hole in the window: claim */
                tags[s] = incoming;
                slot = (int64_t)s;
                break;
            }
            if ((tag & ORC_FP_MASK) == key_fp) {   /* resident key */
                slot = (int64_t)s;
                break;
            }
            /* eviction candidate: old enough (tag age) and no live samples */
            const uint64_t age = (tag >> 32) & ORC_AGE_MASK;
            if (age >= (uint64_t)evict_min_age && counts[s] == 0) {
                if (victim < 0 || tag > victim_tag) {
                    victim = (int64_t)s;
                    victim_tag = tag;
                }
            }
        }
        if (slot < 0 && victim >= 0) {
            tags[victim] = incoming;
            status[i] = 1;
            slot = victim;
            victim_tags[i] = victim_tag;
            victim_touch[i] = last_touch[victim];
            orc_zero_cell(fixed, sums, hist_sums, counts, hist_counts, deltas, victim);
        }
        if (slot < 0) {
            status[i] = 2;
            continue;
        }
        slots[i] = slot;
        if (fixed) {
            int64_t *row = (int64_t *)sums + 3 * slot;
            for (int c = 0; c < 3; ++c)   /* 16.16 fixed point, _native.pyx:251-253 */
                row[c] += (int64_t)floor(vals[3 * i + c] * 65536.0 + 0.5);
        } else {
            double *row = (double *)sums + 3 * slot;
            for (int c = 0; c < 3; ++c)
                row[c] += vals[3 * i + c];
        }
        counts[slot] += 1;
        last_touch[slot] = frame;
    }
    return 0;
}

int orc_lookup(const uint64_t *tags, int64_t capacity, const uint64_t *idx,
               const uint32_t *fp, int64_t n, int probe_limit, int64_t *out)
{
    const uint64_t mask = (uint64_t)capacity - 1;
    for (int64_t i = 0; i < n; ++i) {
        const uint64_t home = idx[i] & mask;
        out[i] = -1;
        for (int j = 0; j < probe_limit; ++j) {
            const uint64_t s = (home + (uint64_t)j) & mask;
            const uint64_t tag = tags[s];
            if (tag == ORC_EMPTY)
                break;                  /* a hole ends the chain */
            if ((tag & ORC_FP_MASK) == (uint64_t)fp[i]) {
                out[i] = (int64_t)s;
                break;
            }
        }
    }
    return 0;
}
