// Host-side helpers shared by the C-ABI translation units.
#pragma once

#include <utility>

#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <limits>
#include <string>

#include "../../include/pathfilter_b200.h"

namespace pf {

// A non-blocking helper stream (plus fork/join events) for work that can overlap the
// caller's stream inside one C-ABI call; one per device, created on first use.
struct SideStream {
    cudaStream_t stream = nullptr;
    cudaEvent_t fork = nullptr, join = nullptr;
    bool ok = false;
};
SideStream &side_stream();

void set_error(const std::string &msg);
int fail_arg(const char *fn, const char *what);
int check_launch(const char *fn);
int sm_count();

inline bool is_pow2(int64_t c) { return c >= 2 && (c & (c - 1)) == 0; }

inline int validate_table(const char *fn, const pf_table *t) {
    if (t == nullptr) return fail_arg(fn, "table is NULL");
    if (!is_pow2(t->capacity)) return fail_arg(fn, "capacity must be a power of two >= 2");
    if (t->probe_limit < 1) return fail_arg(fn, "probe_limit must be >= 1");
    if (!t->tags || !t->sums || !t->counts || !t->hist_sums || !t->hist_counts ||
        !t->last_touch || !t->deltas)
        return fail_arg(fn, "table array pointer is NULL");
    if (t->sum_mode != PF_SUM_FIXED && t->sum_mode != PF_SUM_FLOAT)
        return fail_arg(fn, "unknown sum_mode");
    if (t->cnt_stride < 1 || t->cold_stride < 1 || t->sum_stride < 1 || t->hsum_stride < 3 ||
        t->sum_cstride < 1 || (t->sum_cstride < 3 && t->sum_stride < 3 * t->sum_cstride))
        return fail_arg(fn, "bad table strides");
    return PF_OK;
}

inline int validate_vertices(const char *fn, const pf_vertices *v, const pf_config *cfg) {
    if (v == nullptr || cfg == nullptr) return fail_arg(fn, "vertices/config is NULL");
    if (v->n < 0) return fail_arg(fn, "negative vertex count");
    if (v->n == 0) return PF_OK;
    if (!v->position || !v->normal || !v->camera_distance || !v->pixel || !v->sample)
        return fail_arg(fn, "vertex array pointer is NULL");
    if (cfg->include_incident_angle && (!v->omega_r || !v->layer_id))
        return fail_arg(fn, "include_incident_angle needs omega_r and layer_id");
    if (cfg->include_layer && !v->layer_id)
        return fail_arg(fn, "include_layer needs layer_id");
    return PF_OK;
}

inline cudaStream_t as_stream(void *s) { return static_cast<cudaStream_t>(s); }

#ifndef PF_PDL
#define PF_PDL 1
#endif
// Launch with programmatic dependent launch (PDL) when PF_PDL: the kernel's CTAs may be
// scheduled while the previous kernel in the stream drains (each chain kernel triggers
// its dependents at its start, pdl_trigger) and they wait in pdl_wait until it has
// completed and its writes are visible -- kernel boundaries lose their launch gap.
template <typename... KArgs, typename... Args>
inline void launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, cudaStream_t st,
                       Args &&...args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = 0;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = PF_PDL ? 1 : 0;
    cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

// Copy of the caller's config with the derived fields the kernels read: lod_ulps[]
// packs m_k = (bits(2^k) - bits(T[k])) for k = 1..31 in 4-bit fields.  Thresholds
// must lie in [2^k - 15 ulp, 2^k] (numpy's log2 rounds up at most a few ulps).
inline int prepare_config(const char *fn, const pf_config *in, pf_config *out) {
    *out = *in;
    out->lod_ulps[0] = out->lod_ulps[1] = 0;
    for (int k = 1; k < 32; ++k) {
        const double p = static_cast<double>(1ull << k);
        int64_t bp, bt;
        std::memcpy(&bp, &p, 8);
        std::memcpy(&bt, &in->lod_threshold[k], 8);
        const int64_t m = bp - bt;
        if (m < 0 || m > 15) return fail_arg(fn, "lod_threshold[k] must be within 15 ulps below 2^k");
        out->lod_ulps[k >> 4] |= static_cast<uint64_t>(m) << ((k & 15) * 4);
    }
    out->inv_base_voxel = 1.0 / in->base_voxel;  // IEEE division: RN(1/base_voxel)
    // lod_dist[k]: smallest non-negative double d with RN(d * c_lod) >= T[k], by bisection
    // over the (monotone) bit patterns of non-negative doubles.  make_key skips the exact
    // LOD of the jittered distance when the jitter cannot reach the next threshold.
    const double c = in->c_lod;
    // the bisection (32 x ~63 steps) runs once per distinct (c_lod, thresholds): a frame
    // loop passes the same config every call
    thread_local double memo_c = std::numeric_limits<double>::quiet_NaN();
    thread_local double memo_t[32], memo_d[32];
    if (c == memo_c && std::memcmp(memo_t, in->lod_threshold, sizeof(memo_t)) == 0) {
        std::memcpy(out->lod_dist, memo_d, sizeof(memo_d));
        return PF_OK;
    }
    for (int k = 0; k < 32; ++k) {
        double dk = std::numeric_limits<double>::quiet_NaN();
        if (c > 0.0 && c < std::numeric_limits<double>::infinity()) {
            // [0]: the first distance whose ratio overflows (LOD(inf) is INT64_MIN)
            const double t = k == 0 ? std::numeric_limits<double>::infinity()
                                    : in->lod_threshold[k];
            uint64_t lo = 0, hi = 0x7FF0000000000000ull;  // P(hi) holds: inf * c >= t
            while (lo < hi) {                               // smallest bits with P
                const uint64_t mid = lo + (hi - lo) / 2;
                double d;
                std::memcpy(&d, &mid, 8);
                if (d * c >= t) hi = mid;
                else lo = mid + 1;
            }
            std::memcpy(&dk, &lo, 8);
        }
        out->lod_dist[k] = dk;
    }
    memo_c = c;
    std::memcpy(memo_t, in->lod_threshold, sizeof(memo_t));
    std::memcpy(memo_d, out->lod_dist, sizeof(memo_d));
    return PF_OK;
}

// pf_filter_frame's prologue in one launch (pf_table.cu): begin_frame on both tables
// (over the occupied-slot lists occ_* when given, else a tag sweep), the input check
// (vals/bad may be NULL) and the zeroing of the counter arrays (zero3: int64[2]).
int frame_prologue(const pf_table *fine, const pf_table *coarse, int64_t frame, int32_t mode,
                   double ema, double delta_max, int32_t sample_cap, int64_t *clears_fine,
                   int64_t *clears_coarse, const double *vals, int64_t count, int32_t *bad,
                   int64_t *zero0, int64_t n0, int64_t *zero1, int64_t n1, int64_t *zero2,
                   cudaStream_t st, const int32_t *occ_fine = nullptr,
                   const int32_t *occ_coarse = nullptr, const int64_t *occ_n = nullptr,
                   int64_t *zero3 = nullptr);

inline unsigned blocks_for(int64_t n, int threads) {
    return static_cast<unsigned>((n + threads - 1) / threads);
}

}  // namespace pf
