// Device building blocks of the hashed path-space filter (sm_100a).
//
// Everything that must be bit-exact with the reference lives here: the counter
// RNG (src/rng.py), the key recipe (src/keys.py:245-359) and the
// per-slot temporal math (src/table.py:205-298).  The whole library is compiled
// with -fmad=false, and the FP64 key arithmetic additionally spells every
// multiply/add with __dmul_rn/__dadd_rn so numpy's op order (no FMA contraction)
// survives any flag change.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/pathfilter_b200.h"
#include "pf_sincos_tab.h"

namespace pf {

constexpr uint64_t kEmptyTag = 0xFFFFFFFF00000000ull;   // src/table.py:39
constexpr uint64_t kFresh = 0xFF000000ull;              // src/_native.pyx:18
constexpr uint64_t kAgeMask = 0xFFFFFFull;              // src/_native.pyx:75 (probe side)
constexpr uint64_t kPrioAgeMask = 0xFFFFFEull;          // src/table.py:40 (packing side)
constexpr uint64_t kFpMask = 0xFFFFFFFFull;
// Transient tag held while an eviction wipes the victim cell.  Fingerprint bits are
// the sentinel 0 (never a real key, src/keys.py:18, 214-215) so nothing matches it, and it
// is never EMPTY; probers that meet it wait for the evictor to publish the new tag.
constexpr uint64_t kBusyTag = 0ull;
constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ull;     // src/rng.py:16
constexpr uint64_t kInitIndex = 0x9E3779B97F4A7C15ull;  // src/keys.py:22
constexpr uint64_t kInitFp = 0xC2B2AE3D27D4EB4Full;     // src/keys.py:23
constexpr double kTwoPi = 6.283185307179586;            // 2.0 * math.pi (src/keys.py:265)
constexpr double kFixedScale = 65536.0;                 // src/table.py:38
constexpr int kMaxLevel = 31;                           // src/keys.py:19

// ------------------------------------------------------------------ PDL
#ifndef PF_PDL
#define PF_PDL 1
#endif
// The chain kernels of a frame (launch_pdl): wait for the previous kernel's completion
// before reading what it wrote.  Single-wave (persistent) kernels also let the next
// kernel's CTAs launch into the slots their finished CTAs free; a multi-wave kernel
// must not (the waiting CTAs would take its later waves' slots), so its dependents
// launch when its last CTA exits, which still saves the launch gap.
__device__ __forceinline__ void pdl_wait() {
#if PF_PDL
    asm volatile("griddepcontrol.wait;" ::: "memory");
#endif
}
__device__ __forceinline__ void pdl_trigger() {
#if PF_PDL
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
}

// Kernel parameters the key / insert loops (and the shard apply) address dynamically (the fine or the coarse
// table by key set) stay in parameter space: without __grid_constant__ the compiler
// copies every such struct to local memory at entry and the loops read it back with LDL.
#ifndef PF_GRID_CONSTANT
#define PF_GRID_CONSTANT 1
#endif
#if PF_GRID_CONSTANT
#define PF_GRID_CONST __grid_constant__
#else
#define PF_GRID_CONST
#endif

// ------------------------------------------------------------------ slot fields
// Addresses of slot s's fields (pf_table: SoA or the interleaved 128-byte record).
__device__ __forceinline__ int64_t *cnt_at(const pf_table &t, int64_t s) {
    return t.counts + s * t.cnt_stride;
}
__device__ __forceinline__ int64_t *hcnt_at(const pf_table &t, int64_t s) {
    return t.hist_counts + s * t.cold_stride;
}
__device__ __forceinline__ int64_t *touch_at(const pf_table &t, int64_t s) {
    return t.last_touch + s * t.cold_stride;
}
__device__ __forceinline__ double *delta_at(const pf_table &t, int64_t s) {
    return t.deltas + s * t.cold_stride;
}
// channel c of slot s's live sums / the three adjacent channels of its history sums
// (raw 64-bit words)
__device__ __forceinline__ uint64_t *sum_at(const pf_table &t, int64_t s, int c) {
    return static_cast<uint64_t *>(t.sums) + s * t.sum_stride + c * t.sum_cstride;
}
__device__ __forceinline__ uint64_t *hsum_at(const pf_table &t, int64_t s) {
    return static_cast<uint64_t *>(t.hist_sums) + s * t.hsum_stride;
}

// ------------------------------------------------------------------ integer helpers

__device__ __forceinline__ uint64_t mix64(uint64_t x) {  // src/rng.py:51-59
    x ^= x >> 33;
    x *= 0xFF51AFD7ED558CCDull;
    x ^= x >> 33;
    x *= 0xC4CEB9FE1A85EC53ull;
    x ^= x >> 33;
    return x;
}

// numpy float64 -> int64 cast on x86 (cvttsd2si): NaN and out-of-range give INT64_MIN
// (-2^63 itself converts to INT64_MIN too, so one |x| < 2^63 test covers every case).
__device__ __forceinline__ int64_t np_i64(double x) {
    if (!(fabs(x) < 0x1p63))
        return INT64_MIN;
    return static_cast<int64_t>(x);
}

// np_i64(floor(x)) as ONE F2I.FLOOR and a compare on x itself: floor(x) < 2^63 iff
// x < 2^63; below -2^63 (and at it) the conversion saturates to INT64_MIN, which is
// numpy's value there; NaN fails the compare.
__device__ __forceinline__ int64_t np_floor_i64(double x) {
    long long r;
    asm("cvt.rmi.s64.f64 %0, %1;" : "=l"(r) : "d"(x));
    return x < 0x1p63 ? static_cast<int64_t>(r) : INT64_MIN;
}

__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double ddiv(double a, double b) { return __ddiv_rn(a, b); }

// Correctly rounded x / y from r = RN(1/y) (Markstein's theorem): q0 = RN(x*r) is a
// faithful quotient, rem = x - q0*y is exact under FMA, and RN(q0 + rem*r) = RN(x/y).
// Three FP64 ops instead of a full division when the reciprocal is shared; zero,
// huge and tiny numerators (outside the theorem's no-underflow range) take __ddiv_rn.
// Verified bitwise against __ddiv_rn by pf_selftest_division (tests/test_gpu_parity.py).
// Out of line: the full IEEE division is a cold path, kept out of the hot loops'
// instruction footprint.
static __device__ __noinline__ double ddiv_cold(double x, double y) { return __ddiv_rn(x, y); }

__device__ __forceinline__ double div_rcp(double x, double y, double r) {
    const double ax = fabs(x);
    if (!(fabs(y) > 0x1p-900 && fabs(y) < 0x1p+900))
        return ddiv_cold(x, y);
    if (ax == 0.0)
        return __dmul_rn(x, r);  // signed zero: sign(x) * sign(y), like IEEE division
    if (!(ax > 0x1p-900 && ax < 0x1p+900))
        return ddiv_cold(x, y);
    const double q0 = __dmul_rn(x, r);
    const double rem = __fma_rn(-q0, y, x);
    return __fma_rn(rem, r, q0);
}

// Three quotients by one divisor, branch-free on the common path: the Markstein
// results are formed for all three (signed zeros selected), and one warp-wide test
// sends any numerator outside the theorem's range to IEEE division.
__device__ __forceinline__ void div3_rcp(const double x[3], double y, double r, double q[3]) {
    // a divisor outside the theorem's range (0, inf, NaN, subnormal: a level of INT64_MIN
    // from an infinite distance gives step 0) sends all three to IEEE division
    const bool y_bad = !(fabs(y) > 0x1p-900 && fabs(y) < 0x1p+900);
    bool slow = y_bad;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        const double ax = fabs(x[c]);
        const double q0 = __dmul_rn(x[c], r);
        const double rem = __fma_rn(-q0, y, x[c]);
        q[c] = ax == 0.0 ? q0 : __fma_rn(rem, r, q0);
        slow |= ax != 0.0 && !(ax > 0x1p-900 && ax < 0x1p+900);
    }
    if (slow) {
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            const double ax = fabs(x[c]);
            if (y_bad || (ax != 0.0 && !(ax > 0x1p-900 && ax < 0x1p+900)))
                q[c] = ddiv_cold(x[c], y);
        }
    }
}

// np.maximum / np.minimum propagate NaN from either side.
__device__ __forceinline__ double np_max(double a, double b) {
    return (a != a) ? a : ((b != b) ? b : (a >= b ? a : b));
}
__device__ __forceinline__ double np_min(double a, double b) {
    return (a != a) ? a : ((b != b) ? b : (a <= b ? a : b));
}

// ------------------------------------------------------------------ RNG (src/rng.py)

// draw_unit_array(seed, stream, path_id, 0, dim) for dims 0 and 1
// (src/rng.py:62-78, src/pipeline.py:119-123); h0 = mix64(seed ^ stream*G) is a
// host constant.
__device__ __forceinline__ uint64_t path_id(int64_t pixel, int64_t sample) {  // src/tracer.py:82-84
    return (static_cast<uint64_t>(sample) << 32) | static_cast<uint64_t>(pixel);
}

__device__ __forceinline__ void jitter_draws_pid(uint64_t h0, uint64_t pid, double &u1, double &u2) {
    uint64_t h = mix64(h0 ^ (pid + kGolden));
    h = mix64(h ^ (0ull + kGolden));
    const uint64_t a = mix64(h ^ (0ull + kGolden));
    const uint64_t b = mix64(h ^ (1ull + kGolden));
    const double inv = 1.0 / 9007199254740992.0;  // 2^-53, exact
    u1 = static_cast<double>(a >> 11) * inv;
    u2 = static_cast<double>(b >> 11) * inv;
}

__device__ __forceinline__ void jitter_draws(uint64_t h0, int64_t pixel, int64_t sample,
                                             double &u1, double &u2) {
    jitter_draws_pid(h0, path_id(pixel, sample), u1, u2);
}

// ------------------------------------------------------------------ glibc sin / cos
//
// numpy's float64 sin/cos here are glibc 2.39's (bit for bit; glibc picks its FMA
// build on this host), and glibc's are not correctly rounded, so CUDA's sin/cos give
// jittered positions a few ulps off.  This is a restatement of glibc's dbl-64 algorithm
// (sysdeps/ieee754/dbl-64/s_sin.c: do_sin, do_cos, reduce_sincos, TAYLOR_SIN) with its
// table (pf_sincos_tab.h) and the FMA contractions of the FMA build, valid for
// |x| < 105414350 (beyond that glibc switches to a multi-word reduction; we fall back
// to CUDA's).  tests/test_gpu_parity.py::test_glibc_sincos checks it bit for bit
// against numpy on 2^22 arguments.
namespace glibc {
constexpr double s1 = -0x1.5555555555555p-3, s2 = 0x1.1111111110ecep-7,
                 s3 = -0x1.a01a019db08b8p-13, s4 = 0x1.71de27b9a7ed9p-19,
                 s5 = -0x1.addffc2fcdf59p-26;
constexpr double sn3 = -0x1.5555555555515p-3, sn5 = 0x1.11110e829872fp-7, cs2 = 0.5,
                 cs4 = -0x1.5555555555535p-5, cs6 = 0x1.6c16bedd9e239p-10;
constexpr double big = 0x1.8p45, toint = 0x1.8p52, hpinv = 0x1.45f306dc9c883p-1,
                 mp1 = 0x1.921fb58p0, mp2 = -0x1.dde973cp-27, pp3 = -0x1.cb3b398p-55,
                 pp4 = -0x1.d747f23e32ed7p-83, hp0 = 0x1.921fb54442d18p0,
                 hp1 = 0x1.1a62633145c07p-54;

__device__ __forceinline__ uint32_t hi_word(double x) {
    return static_cast<uint32_t>(static_cast<uint64_t>(__double_as_longlong(x)) >> 32);
}
__device__ __forceinline__ uint32_t lo_word(double x) {
    return static_cast<uint32_t>(static_cast<uint64_t>(__double_as_longlong(x)));
}

// Entry i = (sn, ssn, cs, ccs) of sin/cos(i/128) as two 16-byte loads (entries are
// 32-byte aligned); i <= 109 on every path that uses the value.  `tab` is the table in
// global memory or a kernel's shared-memory copy (stage_sincos_table): lanes gather
// random entries, which shared memory serves without L1 tag lookups.
__device__ __forceinline__ double4 table_entry(const double2 *tab, uint32_t i) {
    const double2 *p = tab + 2 * (i < 110u ? i : 0u);
    const double2 a = p[0], b = p[1];
    return make_double4(a.x, a.y, b.x, b.y);
}

__device__ __forceinline__ double do_cos(double x, double dx, const double2 *tab) {
    if (x < 0) dx = -dx;
    const double ax = fabs(x);
    const double u = __dadd_rn(big, ax);
    x = __dadd_rn(__dsub_rn(ax, __dsub_rn(u, big)), dx);
    const double xx = __dmul_rn(x, x);
    const double s = __fma_rn(__dmul_rn(x, xx), __fma_rn(xx, sn5, sn3), x);
    const double c = __dmul_rn(xx, __fma_rn(xx, __fma_rn(xx, cs6, cs4), cs2));
    const double4 e = table_entry(tab, lo_word(u));
    const double sn = e.x, ssn = e.y, cs = e.z, ccs = e.w;
    const double cor = __fma_rn(-sn, s, __fma_rn(-cs, c, __fma_rn(-s, ssn, ccs)));
    return __dadd_rn(cs, cor);
}

__device__ __forceinline__ double do_sin(double x, double dx, const double2 *tab) {
    const double xold = x;
    const double ax = fabs(x);
    // TAYLOR_SIN for |x| < 0.126 (computed alongside; selected below)
    const double x2 = __dmul_rn(x, x);
    const double poly =
        __fma_rn(__fma_rn(__fma_rn(__fma_rn(s5, x2, s4), x2, s3), x2, s2), x2, s1);
    const double taylor =
        __dadd_rn(x, __fma_rn(__fma_rn(poly, x, -__dmul_rn(0.5, dx)), x2, dx));
    if (x <= 0) dx = -dx;
    const double u = __dadd_rn(big, ax);
    const double y = __dsub_rn(ax, __dsub_rn(u, big));
    const double yy = __dmul_rn(y, y);
    const double s = __dadd_rn(y, __fma_rn(__dmul_rn(y, yy), __fma_rn(yy, sn5, sn3), dx));
    const double c = __fma_rn(y, dx, __dmul_rn(yy, __fma_rn(yy, __fma_rn(yy, cs6, cs4), cs2)));
    const double4 e = table_entry(tab, lo_word(u));
    const double sn = e.x, ssn = e.y, cs = e.z, ccs = e.w;
    const double cor = __fma_rn(cs, s, __fma_rn(-sn, c, __fma_rn(s, ccs, ssn)));
    const double table = copysign(__dadd_rn(sn, cor), xold);
    return ax < 0.126 ? taylor : table;
}
}  // namespace glibc

// sin(x) and cos(x) exactly as glibc computes them (see above): each lane evaluates one
// do_sin and one do_cos with region-dependent arguments, without divergent branches.
// |x| >= 105414350, inf, nan: CUDA's sincos out of line (never reached by the jitter,
// whose argument is 2*pi*u in [0, 2*pi), nor by the tracer's directions).
static __device__ __noinline__ void sincos_cold(double x, double *s, double *c) { sincos(x, s, c); }

__device__ __forceinline__ const double2 *global_sincos_table() {
    return reinterpret_cast<const double2 *>(kSinCosTab);
}

// Copy the table into shared memory (220 x 16 B); the caller syncs before use.
__device__ __forceinline__ void stage_sincos_table(double2 *smem) {
    for (int i = threadIdx.x; i < 220; i += blockDim.x) smem[i] = global_sincos_table()[i];
}

__device__ __forceinline__ void glibc_sincos(double x, double &sn, double &cs,
                                             const double2 *tab = global_sincos_table()) {
    using namespace glibc;
    const uint32_t k = hi_word(x) & 0x7fffffffu;
    if (k >= 0x419921FBu) {  // |x| >= 105414350 (or inf / nan): not on our paths
        sincos_cold(x, &sn, &cs);
        return;
    }
    double as, das, ac, dac;       // do_sin / do_cos arguments
    bool sin_from_cos = false, sin_neg = false, cos_from_sin = false, cos_neg = false;
    if (k < 0x3feb6000u) {         // |x| < 0.855469: no reduction
        as = x; das = 0.0; ac = x; dac = 0.0;
    } else if (k < 0x400368fdu) {  // |x| < 2.426265: around pi/2
        const double t = __dsub_rn(hp0, fabs(x));
        const double a = __dadd_rn(t, hp1);
        ac = t; dac = hp1;                                   // sin = copysign(do_cos(t, hp1), x)
        as = a; das = __dadd_rn(__dsub_rn(t, a), hp1);       // cos = do_sin(a, da)
        sin_from_cos = true;
        cos_from_sin = true;
    } else {                       // reduce_sincos: x = n * pi/2 + (a + da)
        const double t = __fma_rn(x, hpinv, toint);
        const double xn = __dsub_rn(t, toint);
        const double y = __fma_rn(-xn, mp2, __fma_rn(-xn, mp1, x));
        const int n = static_cast<int>(lo_word(t) & 3u);
        const double t2 = __fma_rn(-xn, pp3, y);
        double db = __fma_rn(-xn, pp3, __dsub_rn(y, t2));
        const double b = __fma_rn(-xn, pp4, t2);
        db = __dadd_rn(db, __fma_rn(-xn, pp4, __dsub_rn(t2, b)));
        as = ac = b;
        das = dac = db;
        sin_from_cos = (n & 1) != 0;                   // do_sincos(a, da, n)
        sin_neg = (n & 2) != 0;
        cos_from_sin = ((n + 1) & 1) == 0;             // do_sincos(a, da, n + 1)
        cos_neg = ((n + 1) & 2) != 0;
    }
    const double vs = do_sin(as, das, tab);
    const double vc = do_cos(ac, dac, tab);
    if (k < 0x3feb6000u || k >= 0x400368fdu) {
        sn = sin_from_cos ? vc : vs;
        cs = cos_from_sin ? vs : vc;
    } else {
        sn = copysign(vc, x);
        cs = vs;
    }
    if (sin_neg) sn = -sn;
    if (cos_neg) cs = -cs;
    if (k < 0x3e500000u) sn = x;    // |x| < 2^-26
    if (k < 0x3e400000u) cs = 1.0;  // |x| < 2^-27
}

// Disc offsets: r = 0.5*sqrt(u1), phi = 2pi*u2, (r cos phi, r sin phi)
// (src/keys.py:264-267).  sqrt is IEEE-exact and sin/cos are glibc's (glibc_sincos),
// so jittered positions equal numpy's bit for bit.
#ifndef PF_GLIBC_SINCOS
#define PF_GLIBC_SINCOS 1
#endif
__device__ __forceinline__ void disc_offset(double u1, double u2, double &u, double &v,
                                            const double2 *tab = global_sincos_table()) {
    const double r = dmul(0.5, __dsqrt_rn(u1));
    const double phi = dmul(kTwoPi, u2);
    double s, c;
#if PF_GLIBC_SINCOS
    glibc_sincos(phi, s, c, tab);
#else
    sincos(phi, &s, &c);
#endif
    u = dmul(r, c);
    v = dmul(r, s);
}

// ------------------------------------------------------------------ keys (src/keys.py)

// floor(log2(max(d * c_lod, 1))) clamped to 31 (src/keys.py:245-248).  numpy's log2
// rounds up to k just below 2^k, so the exact floor is exponent + (r >= T[e+1]).
// T[k] = 2^k - m_k ulps with m_k < 16 packed as 4-bit fields in cfg.lod_ulps, so
// ratio >= T[e+1] <=> mantissa >= 2^52 - m_{e+1}: pure integer work on the bits
// (no dynamic indexing into the kernel-parameter array, which would spill it).
__device__ __forceinline__ int64_t lod_level(double dist, const pf_config &cfg) {
    const double ratio = np_max(dmul(dist, cfg.c_lod), 1.0);
    if (!(ratio <= 1.7976931348623157e308))  // NaN or inf: floor(log2) casts to INT64_MIN
        return INT64_MIN;
    if (ratio >= 2147483648.0)
        return kMaxLevel;
    const uint64_t bits = static_cast<uint64_t>(__double_as_longlong(ratio));
    const int e = static_cast<int>(bits >> 52) - 1023;  // ratio in [1, 2^31): exact floor(log2)
    const int k = e + 1;
    const uint64_t word = k >= 16 ? cfg.lod_ulps[1] : cfg.lod_ulps[0];
    const uint64_t m = (word >> ((k & 15) * 4)) & 15u;
    const uint64_t mant = bits & 0xFFFFFFFFFFFFFull;
    return mant >= (0x10000000000000ull - m) ? k : e;
}

__device__ __forceinline__ int64_t clamp_level(int64_t lv, int32_t delta) {
    const int64_t l = lv + delta;
    return l < kMaxLevel ? l : kMaxLevel;
}

// exp2(e) for integer e, as numpy computes it: normal powers from the exponent field,
// subnormals below 2^-1022, 0 below 2^-1074 and +inf above 2^1023.
static __device__ __noinline__ double pow2i_cold(int64_t e) {
    if (e > 1023) return __longlong_as_double(0x7FF0000000000000ll);
    const int64_t sh = e + 1074;  // subnormal bit index
    return __longlong_as_double((sh >= 0 && sh < 52) ? (1ll << sh) : 0ll);
}

__device__ __forceinline__ double pow2i(int64_t e) {
    if (e >= -1022 && e <= 1023)  // every level the key recipe produces
        return __longlong_as_double(static_cast<long long>(e + 1023) << 52);
    return pow2i_cold(e);
}

// base_voxel * exp2(level): exact power-of-two scaling.
__device__ __forceinline__ double voxel_step(double base_voxel, int64_t level) {
    return dmul(base_voxel, pow2i(level));
}

struct Frame3 {
    double t1[3], t2[3];
};

// Branchless ONB (src/keys.py:251-258) in numpy's left-to-right order.
__device__ __forceinline__ Frame3 tangent_frame(double x, double y, double z) {
    const double s = (z >= 0.0) ? 1.0 : -1.0;
    const double a = -__drcp_rn(dadd(s, z));  // -1.0 / (s + z): negation is exact
    const double b = dmul(dmul(x, y), a);
    Frame3 f;
    f.t1[0] = dadd(1.0, dmul(dmul(dmul(s, x), x), a));
    f.t1[1] = dmul(s, b);
    f.t1[2] = dmul(-s, x);
    f.t2[0] = b;
    f.t2[1] = dadd(s, dmul(dmul(y, y), a));
    f.t2[2] = -y;
    return f;
}

// Octahedral normal bin (src/keys.py:273-283).
__device__ __forceinline__ int64_t octa_bin(double x, double y, double z, int bins) {
    const double s = np_max(dadd(dadd(fabs(x), fabs(y)), fabs(z)), 1e-300);
    const double rs = __drcp_rn(s);
    const double n3[3] = {x, y, z};
    double p3[3];
    div3_rcp(n3, s, rs, p3);
    const double px = p3[0], py = p3[1], pz = p3[2];
    double fx = px, fy = py;
    if (pz < 0.0) {
        fx = dmul(dsub(1.0, fabs(py)), px >= 0.0 ? 1.0 : -1.0);
        fy = dmul(dsub(1.0, fabs(px)), py >= 0.0 ? 1.0 : -1.0);
    }
    const double fb = static_cast<double>(bins);
    int64_t bx = np_i64(dmul(dadd(dmul(fx, 0.5), 0.5), fb));
    int64_t by = np_i64(dmul(dadd(dmul(fy, 0.5), 0.5), fb));
    if (bx > bins - 1) bx = bins - 1;
    if (by > bins - 1) by = bins - 1;
    return by * bins + bx;
}

// aux word (src/keys.py:286-299).  The incident-angle dot product follows numpy's
// einsum("ij,ij->i") reduction order for length 3: (n0*o0 + n2*o2) + n1*o1
// (measured in this image; see tests/test_oracle_golden.py).
__device__ __forceinline__ uint64_t aux_word(const pf_config &cfg, double nx, double ny,
                                             double nz, const double *omega, int64_t layer) {
    uint64_t aux = 0;
    if (cfg.include_normal && !cfg.normal_in_fingerprint)
        aux |= static_cast<uint64_t>(octa_bin(nx, ny, nz, cfg.normal_bins));
    if (cfg.include_incident_angle) {
        const double c0 = dadd(dadd(dmul(nx, omega[0]), dmul(nz, omega[2])), dmul(ny, omega[1]));
        const double c = np_min(np_max(c0, 0.0), 1.0);
        int64_t ab = np_i64(dmul(c, static_cast<double>(cfg.incident_angle_bins)));
        if (ab > cfg.incident_angle_bins - 1) ab = cfg.incident_angle_bins - 1;
        if (layer != 1) ab = 0;
        aux |= static_cast<uint64_t>(ab) << 16;
    }
    if (cfg.include_layer)
        aux |= static_cast<uint64_t>(layer) << 24;
    return aux;
}

struct CellKey {
    int64_t q[3];
    int64_t level;
    uint64_t aux;
};

struct CellHash {
    uint64_t index;
    uint32_t fp;
};

// A lookup key handed from the insert pass to the resolve pass in one word: the low 32
// bits of the slot index (all a probe of a table with capacity <= 2^32 reads) and the
// fingerprint.
__device__ __forceinline__ uint64_t pack_lookup_key(const CellHash &h) {
    return (static_cast<uint64_t>(h.fp) << 32) | (h.index & 0xFFFFFFFFull);
}
__device__ __forceinline__ CellHash unpack_lookup_key(uint64_t w) {
    CellHash h;
    h.index = w & 0xFFFFFFFFull;
    h.fp = static_cast<uint32_t>(w >> 32);
    return h;
}

// hash_arrays (src/keys.py:327-339).
__device__ __forceinline__ CellHash cell_hash(int64_t qx, int64_t qy, int64_t qz, int64_t level,
                                              uint64_t aux, int has_fp_bin, uint32_t fp_bin) {
    const uint64_t f[5] = {static_cast<uint64_t>(qx), static_cast<uint64_t>(qy),
                           static_cast<uint64_t>(qz), static_cast<uint64_t>(level), aux};
    uint64_t h = kInitIndex, g = kInitFp;
#pragma unroll
    for (int i = 0; i < 5; ++i) h = mix64(h ^ f[i]);
#pragma unroll
    for (int i = 0; i < 5; ++i) g = mix64(g ^ f[i]);
    uint32_t fp = static_cast<uint32_t>((g ^ (g >> 32)) & kFpMask);
    if (has_fp_bin)
        fp = (fp << 6) | fp_bin;
    if (fp == 0u)
        fp = 1u;
    CellHash r;
    r.index = h;
    r.fp = fp;
    return r;
}

// Per-vertex inputs shared by every key set of one vertex.
struct VertexIn {
    double pos[3];
    double nrm[3];
    double dist;
    int64_t pixel, sample, layer;
    double omega[3];
};

// ------------------------------------------------------------------ L2 residency
//
// The vertex stream is read exactly once per pass; the voxel tables and the
// composite buffer are re-touched all frame.  Stream loads therefore carry an L2
// evict_first policy and table/composite updates an evict_last one, so a 1 GB
// vertex buffer does not flush the ~40 MB of live table lines out of the 126 MB L2.
__device__ __forceinline__ uint64_t l2_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t l2_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t l2_evict_normal() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
    return p;
}
// Policy for the insert's table REDs / the resolve's composite REDs (0 normal,
// 1 evict_last, 2 evict_first).
#ifndef PF_TABLE_RED_POLICY
#define PF_TABLE_RED_POLICY 1
#endif
#ifndef PF_FLAT_POLICY
#define PF_FLAT_POLICY 1
#endif
__device__ __forceinline__ uint64_t l2_policy(int k) {
    return k == 1 ? l2_evict_last() : k == 2 ? l2_evict_first() : l2_evict_normal();
}
__device__ __forceinline__ double ld_stream(const double *p, uint64_t pol) {
    double d;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;"
                 : "=d"(d) : "l"(p), "l"(pol));
    return d;
}
__device__ __forceinline__ int64_t ld_stream(const int64_t *p, uint64_t pol) {
    int64_t d;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.s64 %0, [%1], %2;"
                 : "=l"(d) : "l"(p), "l"(pol));
    return d;
}
__device__ __forceinline__ uint64_t ld_stream(const uint64_t *p, uint64_t pol) {
    uint64_t d;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.u64 %0, [%1], %2;"
                 : "=l"(d) : "l"(p), "l"(pol));
    return d;
}
__device__ __forceinline__ uint32_t ld_stream(const uint32_t *p, uint64_t pol) {
    uint32_t d;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.u32 %0, [%1], %2;"
                 : "=r"(d) : "l"(p), "l"(pol));
    return d;
}

__device__ __forceinline__ void prefetch_l2(const void *p) {
    asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}

// 16 bytes global -> shared through L2 only (coherent at gpu scope like a relaxed load),
// tracked by cp.async groups instead of a register scoreboard.
__device__ __forceinline__ void cp_async_16(void *smem, const void *gmem) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n\tcp.async.commit_group;"
                 ::"r"(s), "l"(gmem) : "memory");
}
// 8-byte global -> shared copy (L1-allocating .ca: .cg takes only 16 bytes) with an L2
// policy, committed as its own group
__device__ __forceinline__ void cp_async_8_hint(void *smem, const void *gmem, uint64_t pol) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.ca.shared.global.L2::cache_hint [%0], [%1], 8, %2;\n\tcp.async.commit_group;"
                 ::"r"(s), "l"(gmem), "l"(pol) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
    asm volatile("cp.async.wait_all;" ::: "memory");
}

__device__ __forceinline__ VertexIn load_vertex(const pf_vertices &v, int64_t i,
                                                const pf_config &cfg, uint64_t pol) {
    VertexIn x;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        x.pos[c] = ld_stream(v.position + 3 * i + c, pol);
        x.nrm[c] = ld_stream(v.normal + 3 * i + c, pol);
        x.omega[c] = 0.0;
    }
    x.dist = ld_stream(v.camera_distance + i, pol);
    x.pixel = ld_stream(v.pixel + i, pol);
    x.sample = ld_stream(v.sample + i, pol);
    // the layer only enters the aux word (aux_word); the default key reads no layer ids
    x.layer = (v.layer_id != nullptr && (cfg.include_incident_angle || cfg.include_layer))
                  ? ld_stream(v.layer_id + i, pol) : 0;
    if (cfg.include_incident_angle && v.omega_r != nullptr) {
#pragma unroll
        for (int c = 0; c < 3; ++c) x.omega[c] = ld_stream(v.omega_r + 3 * i + c, pol);
    }
    return x;
}

__device__ __forceinline__ VertexIn load_vertex(const pf_vertices &v, int64_t i,
                                                const pf_config &cfg) {
    return load_vertex(v, i, cfg, l2_evict_first());
}

// Level-independent part of a key set: ONB, aux, structured fp bin.
struct KeyShared {
    Frame3 frame;
    uint64_t aux;
    uint32_t fp_bin;
    int has_fp_bin;
    double rbv;  // RN(1 / base_voxel): RN(1/step) = rbv * 2^-level exactly
    int64_t lv0; // LOD of the unjittered vertex (before any level_delta)
    double gmove;  // d2 < gmove => LOD(dist + |x' - x|) == lv0 (see moved_bound)
};

// Copy cfg.lod_dist into shared memory (static indices: no local copy of the params).
__device__ __forceinline__ void stage_lod_dist(double *smem, const pf_config &cfg) {
    if (threadIdx.x == 0) {
#pragma unroll
        for (int j = 0; j < 32; ++j) smem[j] = cfg.lod_dist[j];
    }
}

// Bound on the squared jitter length below which the jittered distance keeps the level:
// moved = RN(d + RN(sqrt(d2))) >= d and LOD is monotone while the ratio is finite, so
// LOD(moved) == lv0 whenever moved < D = lod_dist[lv0 + 1] (lod_dist[0] for level 31:
// the distance whose ratio overflows to inf).  With e = D * 2^-50 covering the roundings
// of D - d, of the sqrt and of the final sum, d2 < ((D - d) - e)^2 (1 - 2^-50) implies it.
// -1 (never) for negative/NaN distances, huge D or a missing table.
__device__ __forceinline__ double moved_bound(const double *lod_dist, double dist, int64_t lv0) {
    if (lod_dist == nullptr || !(dist >= 0.0) || lv0 < 0) return -1.0;
    const double inf = __longlong_as_double(0x7FF0000000000000ll);
    const double dk = lod_dist[(lv0 + 1) & 31];
    if (dk == inf) return dist <= 1e300 ? inf : -1.0;  // moved stays finite
    if (!(dk >= 0x1p-900)) return -1.0;
    const double g = dsub(dsub(dk, dist), dmul(dk, 0x1p-50));
    if (!(g > 0.0)) return -1.0;
    return dmul(dmul(g, g), 1.0 - 0x1p-50);
}

__device__ __forceinline__ KeyShared key_shared(const pf_config &cfg, const VertexIn &x,
                                                const double *lod_dist = nullptr) {
    KeyShared k;
    k.rbv = cfg.inv_base_voxel;  // prepare_config: RN(1 / base_voxel)
    k.lv0 = lod_level(x.dist, cfg);
    k.gmove = moved_bound(lod_dist, x.dist, k.lv0);
    k.frame = tangent_frame(x.nrm[0], x.nrm[1], x.nrm[2]);
    k.aux = aux_word(cfg, x.nrm[0], x.nrm[1], x.nrm[2], x.omega, x.layer);
    k.has_fp_bin = cfg.include_normal && cfg.normal_in_fingerprint;
    k.fp_bin = k.has_fp_bin
        ? static_cast<uint32_t>(octa_bin(x.nrm[0], x.nrm[1], x.nrm[2], 8) & 0x3F) : 0u;
    return k;
}

// The level-independent jitter direction u*t1 + v*t2 (src/keys.py:268, before the
// scaling by the voxel size), numpy's operation order.
__device__ __forceinline__ void jitter_dir(double u, double v, const double t1[3],
                                           const double t2[3], double w[3]) {
#pragma unroll
    for (int c = 0; c < 3; ++c) w[c] = dadd(dmul(u, t1[c]), dmul(v, t2[c]));
}

#ifndef PF_STEP_TABLE
#define PF_STEP_TABLE 1
#endif
// Per-level {step, RN(1/step)} = {base_voxel * 2^l, rbv * 2^-l} for l = 0..31 (every level
// of a finite distance), staged in shared memory by the key kernels: one LDS.128 instead
// of two exponent builds and products per use.
__device__ __forceinline__ void stage_level_steps(double2 *smem, const pf_config &cfg) {
    if (threadIdx.x < 32) {
        const int64_t l = threadIdx.x;
        smem[l] = make_double2(voxel_step(cfg.base_voxel, l), dmul(cfg.inv_base_voxel, pow2i(-l)));
    }
}

// make_key_arrays for one vertex and one level_delta (src/keys.py:342-359), given the
// jitter direction w (jitter_dir; ignored when jit = 0).  steps: stage_level_steps'
// table (or NULL).
__device__ __forceinline__ CellKey make_key_w(const pf_config &cfg, const VertexIn &x,
                                              const KeyShared &ks, int jit, const double w[3],
                                              int32_t level_delta, double jittered[3],
                                              const double2 *steps = nullptr) {
    int64_t lv = clamp_level(ks.lv0, level_delta);
    const bool tab = PF_STEP_TABLE && steps != nullptr;
    if (jit) {
        const double step = tab && static_cast<uint64_t>(lv) < 32u ? steps[lv].x
                                                                  : voxel_step(cfg.base_voxel, lv);
        double d2 = 0.0;
#pragma unroll
        for (int c = 0; c < 3; ++c) jittered[c] = dadd(x.pos[c], dmul(w[c], step));
        // np.linalg.norm(x' - x, axis=1): sqrt of the sequential sum of squares
        const double e0 = dsub(jittered[0], x.pos[0]);
        const double e1 = dsub(jittered[1], x.pos[1]);
        const double e2 = dsub(jittered[2], x.pos[2]);
        d2 = dadd(dadd(dmul(e0, e0), dmul(e1, e1)), dmul(e2, e2));
        if (!(d2 < ks.gmove)) {  // the jitter may cross a LOD threshold: exact recipe
            const double moved = dadd(x.dist, __dsqrt_rn(d2));
            lv = clamp_level(lod_level(moved, cfg), level_delta);
        }
    } else {
#pragma unroll
        for (int c = 0; c < 3; ++c) jittered[c] = x.pos[c];
    }
    double step, rstep;
    if (tab && static_cast<uint64_t>(lv) < 32u) {
        const double2 sr = steps[lv];
        step = sr.x;
        rstep = sr.y;
    } else {
        step = voxel_step(cfg.base_voxel, lv);
        rstep = dmul(ks.rbv, pow2i(-lv));
    }
    CellKey k;
    // IEEE x / step (not a reciprocal multiply: base_voxel is inexact), via Markstein
    double qd[3];
    div3_rcp(jittered, step, rstep, qd);
#pragma unroll
    for (int c = 0; c < 3; ++c) k.q[c] = np_floor_i64(qd[c]);
    k.level = lv;
    k.aux = ks.aux;
    return k;
}

// make_key_arrays for one vertex and one level_delta (src/keys.py:342-359).
// jit = 0 disables jitter; (u, v) are the disc offsets.
__device__ __forceinline__ CellKey make_key(const pf_config &cfg, const VertexIn &x,
                                            const KeyShared &ks, int jit, double u, double v,
                                            int32_t level_delta, double jittered[3],
                                            const double2 *steps = nullptr) {
    double w[3] = {0.0, 0.0, 0.0};
    if (jit) jitter_dir(u, v, ks.frame.t1, ks.frame.t2, w);
    return make_key_w(cfg, x, ks, jit, w, level_delta, jittered, steps);
}

__device__ __forceinline__ CellHash key_hash(const CellKey &k, const KeyShared &ks) {
    return cell_hash(k.q[0], k.q[1], k.q[2], k.level, k.aux, ks.has_fp_bin, ks.fp_bin);
}

// ------------------------------------------------------------------ table access

// L2-coherent loads/stores for state other threads mutate inside the same launch.
__device__ __forceinline__ uint64_t ld_relaxed(const uint64_t *p) {
    uint64_t v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ uint64_t ld_acquire(const uint64_t *p) {
    uint64_t v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(uint64_t *p, uint64_t v) {
    asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ int64_t ld_acquire_i64(const int64_t *p) {
    return static_cast<int64_t>(ld_acquire(reinterpret_cast<const uint64_t *>(p)));
}
__device__ __forceinline__ int64_t ld_relaxed_i64(const int64_t *p) {
    return static_cast<int64_t>(ld_relaxed(reinterpret_cast<const uint64_t *>(p)));
}
__device__ __forceinline__ void st_relaxed_u64(void *p, uint64_t v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Fire-and-forget L2 reductions (RED, no return value): nvcc otherwise emits ATOMG
// with a result round trip for 64-bit atomicAdd even when the result is unused.
// `pol` is an L2 cache policy (l2_evict_last() keeps table / composite lines resident).
__device__ __forceinline__ void red_add_u64(void *p, uint64_t v, uint64_t pol) {
    asm volatile("red.relaxed.gpu.global.add.L2::cache_hint.u64 [%0], %1, %2;" ::"l"(p), "l"(v),
                 "l"(pol)
                 : "memory");
}
__device__ __forceinline__ void red_add_f64(double *p, double v, uint64_t pol) {
    asm volatile("red.relaxed.gpu.global.add.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(p), "d"(v),
                 "l"(pol)
                 : "memory");
}

__device__ __forceinline__ uint64_t wait_not_busy(const uint64_t *p, uint64_t tag) {
    while (tag == kBusyTag) {
        __nanosleep(32);
        tag = ld_acquire(p);
    }
    return tag;
}

struct InsertResult {
    int64_t slot;
    int32_t status;  // 0 accumulated, 1 evicted then accumulated, 2 probe limit
    int32_t probe_len;
    uint64_t victim_tag;
    int64_t victim_touch;
    bool counted;    // the key's weight is already in counts[slot] (pinned / evicted / claimed)
};

// Live count of a cell an evictor owns: counts[s] is CAS'd 0 -> kEvictMark before the
// wipe and moved back to the incoming key's weight after the new tag is published, so a
// prober whose count add returns a negative value knows the cell is going away.
constexpr int64_t kEvictMark = INT64_MIN / 2;

// Wipe an evicted cell (src/_native.pyx:170-183): live + history sums, counts, delta.
__device__ __forceinline__ void zero_cell(const pf_table &t, int64_t s) {
    uint64_t *hsums = hsum_at(t, s);
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        st_relaxed_u64(sum_at(t, s, c), 0ull);  // int64 0 and float64 +0.0 share bits
        st_relaxed_u64(hsums + c, 0ull);
    }
    st_relaxed_u64(cnt_at(t, s), 0ull);
    st_relaxed_u64(hcnt_at(t, s), 0ull);
    st_relaxed_u64(delta_at(t, s), 0ull);
}

// Eviction (cold path, out of line).  The evictor CASes the victim's exact tag to BUSY
// (probers that meet BUSY wait), then takes the victim's live count 0 -> kEvictMark.
// A prober that pinned the cell first (pin_cell) made the count nonzero: the CAS fails
// and the evictor restores the tag.  Otherwise no prober can pin it any more (a count
// add returns a negative value and backs off), the cell is wiped, the new tag is
// published (release), and the count moves from the mark to the incoming key's weight
// in one add (stray pin attempts undo their own adds, so they net to zero).  Returns
// the victim's last_touch, or INT64_MIN when the victim changed or was pinned first
// (the caller re-probes).
static __device__ __noinline__ int64_t evict_cell(const pf_table &t, int64_t victim,
                                                  uint64_t victim_tag, uint64_t incoming,
                                                  uint64_t weight) {
    uint64_t *vp = t.tags + victim;
    if (atomicCAS(reinterpret_cast<unsigned long long *>(vp), victim_tag, kBusyTag) != victim_tag)
        return INT64_MIN;
    __threadfence();
    unsigned long long *cp = reinterpret_cast<unsigned long long *>(cnt_at(t, victim));
    if (atomicCAS(cp, 0ull, static_cast<unsigned long long>(kEvictMark)) != 0ull) {
        st_release(vp, victim_tag);  // pinned by an accumulate since we read it
        return INT64_MIN;
    }
    const int64_t touch = ld_relaxed_i64(touch_at(t, victim));
    uint64_t *hsums = hsum_at(t, victim);
#pragma unroll
    for (int c = 0; c < 3; ++c) {  // zero_cell minus the live count, which the mark holds
        st_relaxed_u64(sum_at(t, victim, c), 0ull);
        st_relaxed_u64(hsums + c, 0ull);
    }
    st_relaxed_u64(hcnt_at(t, victim), 0ull);
    st_relaxed_u64(delta_at(t, victim), 0ull);
    __threadfence();
    st_release(vp, incoming);
    __threadfence();
    atomicAdd(cp, static_cast<unsigned long long>(-kEvictMark) + weight);
    return touch;
}

// Pin a matched cell that an eviction could take (age >= evict_min_age): add the
// key's weight to its live count, then confirm the tag (once no eviction holds it
// BUSY) is still the one matched.  A negative old count (an evictor holds the mark) or
// a changed tag (an eviction finished between the probe's load and the add) undoes
// the add; the caller re-probes.
static __device__ __noinline__ bool pin_cell(const pf_table &t, int64_t s, uint64_t tag,
                                             uint64_t weight) {
    unsigned long long *cp = reinterpret_cast<unsigned long long *>(cnt_at(t, s));
    const long long old = static_cast<long long>(atomicAdd(cp, weight));
    if (old >= 0) {
        __threadfence();
        if (wait_not_busy(t.tags + s, ld_relaxed(t.tags + s)) == tag) return true;
    }
    atomicAdd(cp, static_cast<unsigned long long>(-static_cast<long long>(weight)));
    return false;
}

// Claim an EMPTY slot when evict_min_age == 0 (fresh cells are eviction candidates):
// EMPTY -> BUSY, count the weight, then publish, so no evictor ever sees the new key
// with a zero live count -- which a sequential caller never could.  Returns the tag
// that held the slot (EMPTY when this key claimed it).
static __device__ __noinline__ uint64_t claim_counted(const pf_table &t, int64_t s,
                                                      uint64_t incoming, uint64_t weight) {
    uint64_t *tp = t.tags + s;
    const uint64_t old = atomicCAS(reinterpret_cast<unsigned long long *>(tp), kEmptyTag, kBusyTag);
    if (old != kEmptyTag) return old;
    atomicAdd(reinterpret_cast<unsigned long long *>(cnt_at(t, s)), weight);
    __threadfence();
    st_release(tp, incoming);
    return kEmptyTag;
}

// Probe / claim / evict for one key (src/_native.pyx:209-247) on the live table.
// Concurrency (every outcome is one a sequential caller could see):
// - a claim is one 64-bit CAS of the whole tag (EMPTY -> FRESH|fp);
// - an eviction CASes the victim's exact tag to BUSY, takes its live count (evict_cell),
//   wipes the cell and publishes FRESH|fp, so no accumulate lands in a half-wiped cell;
// - a match on a cell an eviction could take (age >= evict_min_age) pins it first
//   (pin_cell), so the cell cannot be wiped between the match and the adds.  Matches on
//   younger cells -- every cell touched in the last evict_min_age frames, the common
//   case -- need no pin: their tags cannot change inside a frame.
// A lost victim or pin re-probes the window instead of the reference's racy give-up.
// `home_tag` is the caller's early (prefetched) load of tags[home]; it only seeds the
// first probe of the first attempt and is re-read after any contention.  `weight` is
// what the caller adds to the live count; r.counted says the protocol already added it.
__device__ __forceinline__ InsertResult probe_insert(const pf_table &t, uint64_t idx, uint32_t fp,
                                                     uint64_t home_tag, uint64_t weight) {
    const uint64_t mask = static_cast<uint64_t>(t.capacity) - 1;
    const uint64_t home = idx & mask;
    const uint64_t want = static_cast<uint64_t>(fp);
    const uint64_t incoming = (kFresh << 32) | want;
    const uint64_t min_age = static_cast<uint64_t>(t.evict_min_age);
    InsertResult r;
    r.slot = -1;
    r.status = 2;
    r.probe_len = t.probe_limit;
    r.victim_tag = 0;
    r.victim_touch = 0;
    r.counted = false;
    for (int attempt = 0; attempt < 64; ++attempt) {
        int64_t victim = -1;
        uint64_t victim_tag = 0;
        bool retry = false, reread = false;
        for (int j = 0; j < t.probe_limit; ++j) {
            const uint64_t s = (home + static_cast<uint64_t>(j)) & mask;
            uint64_t tag = (attempt == 0 && j == 0 && !reread) ? home_tag : ld_relaxed(t.tags + s);
            reread = false;
            tag = wait_not_busy(t.tags + s, tag);
            if (tag == kEmptyTag) {
                uint64_t old;
                if (min_age == 0) {
                    old = claim_counted(t, static_cast<int64_t>(s), incoming, weight);
                    if (old == kEmptyTag) r.counted = true;
                    else old = wait_not_busy(t.tags + s, old);
                } else {
                    old = atomicCAS(reinterpret_cast<unsigned long long *>(t.tags + s), kEmptyTag,
                                    incoming);
                }
                if (old == kEmptyTag) {
                    r.slot = static_cast<int64_t>(s);
                    r.status = 0;
                    r.probe_len = j + 1;
                    return r;
                }
                if ((old & kFpMask) != want)
                    continue;  // lost the claim to a different key (src/_native.pyx:221-222)
                tag = old;     // lost it to the same key: a match
            }
            if ((tag & kFpMask) == want) {
                if (((tag >> 32) & kAgeMask) >= min_age) {
                    if (!pin_cell(t, static_cast<int64_t>(s), tag, weight)) {
                        retry = true;
                        break;
                    }
                    r.counted = true;
                }
                r.slot = static_cast<int64_t>(s);
                r.status = 0;
                r.probe_len = j + 1;
                return r;
            }
            const uint64_t age = (tag >> 32) & kAgeMask;
            if (age >= min_age) {
                // A candidate needs a consistent (tag, live count) snapshot: a negative
                // count is an eviction in flight (its new key may be ours), a changed
                // tag a torn read.  Either way wait for the slot to settle and look at
                // it again, so every prober of a key sees the same candidates and the
                // same victim -- two lanes of one key can never evict two cells.
                const int64_t c = ld_acquire_i64(cnt_at(t, s));
                if (c < 0 || ld_relaxed(t.tags + s) != tag) {
                    while (ld_acquire_i64(cnt_at(t, s)) < 0) __nanosleep(32);
                    reread = true;
                    --j;
                    continue;
                }
                if (c == 0 && (victim < 0 || tag > victim_tag)) {
                    victim = static_cast<int64_t>(s);
                    victim_tag = tag;
                }
            }
        }
        if (retry) continue;
        if (victim < 0)
            return r;  // status 2, no mutation
        const int64_t touch = evict_cell(t, victim, victim_tag, incoming, weight);
        if (touch != INT64_MIN) {
            r.victim_touch = touch;
            r.slot = victim;
            r.status = 1;
            r.probe_len = t.probe_limit;
            r.victim_tag = victim_tag;
            r.counted = true;
            return r;
        }
        // window changed under us: re-probe
    }
    return r;
}

// lookup_slots for one key (src/_native.pyx:285-294).  seg_mask (default: the whole
// table) confines the probe window to the aligned segment of size seg_mask + 1 that holds
// the home slot -- the layout of a replica of owner-sliced tables (pf_resolve_replica).
// `first` > 0 resumes a probe whose earlier window slots the caller already checked.
__device__ __forceinline__ int64_t probe_lookup(const uint64_t *tags, uint64_t mask,
                                                int probe_limit, uint64_t idx, uint32_t fp,
                                                uint64_t seg_mask = ~0ull, int first = 0) {
    const uint64_t home = idx & mask;
    const uint64_t sm = seg_mask & mask;
    const uint64_t seg = home & ~sm;
    for (int j = first; j < probe_limit; ++j) {
        const uint64_t s = seg | ((home + static_cast<uint64_t>(j)) & sm);
        const uint64_t tag = __ldg(reinterpret_cast<const unsigned long long *>(tags + s));
        if (tag == kEmptyTag)
            return -1;
        if ((tag & kFpMask) == static_cast<uint64_t>(fp))
            return static_cast<int64_t>(s);
    }
    return -1;
}

// ------------------------------------------------------------------ temporal math

// VoxelTable.effective for one slot (src/table.py:205-238).  In integrate mode the
// storage dtype is kept: isum (fixed) or fsum (float) and icnt; filter/hybrid produce
// float sums and float counts.  Every value equals numpy's elementwise result.
struct Effective {
    int64_t isum[3];
    double fsum[3];
    int64_t icnt;
    double fcnt;
};

// One slot's stored state, raw 64-bit words (int64 or float64 sums by sum_mode).
struct CellState {
    uint64_t sums[3], hist[3];
    int64_t counts, hist_counts, last_touch;
    double delta;
};

// All loads of a slot issued together (one memory latency).  `ro` selects the
// read-only path for kernels that never write the table.
__device__ __forceinline__ CellState load_cell(const pf_table &t, int64_t s, bool ro) {
    CellState c;
    const unsigned long long *hist = reinterpret_cast<const unsigned long long *>(hsum_at(t, s));
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const unsigned long long *sp = reinterpret_cast<const unsigned long long *>(sum_at(t, s, k));
        c.sums[k] = ro ? __ldg(sp) : *sp;
        c.hist[k] = ro ? __ldg(hist + k) : hist[k];
    }
    const int64_t *cp = cnt_at(t, s), *hp = hcnt_at(t, s), *lp = touch_at(t, s);
    const double *dp = delta_at(t, s);
    c.counts = ro ? __ldg(cp) : *cp;
    c.hist_counts = ro ? __ldg(hp) : *hp;
    c.last_touch = ro ? __ldg(lp) : *lp;
    c.delta = ro ? __ldg(dp) : *dp;
    return c;
}

__device__ __forceinline__ Effective effective_of(const CellState &cs, bool fixed, int mode,
                                                  double ema, double delta_max) {
    Effective e;
    const int64_t lc_i = cs.counts;
    const int64_t hc_i = cs.hist_counts;
    if (mode == PF_INTEGRATE) {
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            if (fixed) {
                e.isum[c] = static_cast<int64_t>(cs.sums[c]) + static_cast<int64_t>(cs.hist[c]);
                e.fsum[c] = 0.0;
            } else {
                e.fsum[c] = dadd(__longlong_as_double(cs.sums[c]), __longlong_as_double(cs.hist[c]));
                e.isum[c] = 0;
            }
        }
        e.icnt = lc_i + hc_i;
        e.fcnt = static_cast<double>(e.icnt);
        return e;
    }
    const double lc = static_cast<double>(lc_i), hc = static_cast<double>(hc_i);
    double alpha, cnt;
    if (mode == PF_FILTER) {
        alpha = hc > 0.0 ? (lc > 0.0 ? ema : 1.0) : 0.0;
        cnt = dadd(lc, hc);
    } else {
        const double k = np_min(np_max(ddiv(cs.delta, delta_max), 0.0), 1.0);
        const double both = np_max(dadd(lc, hc), 1.0);
        alpha = hc > 0.0 ? (lc > 0.0 ? ddiv(dmul(dsub(1.0, k), hc), both) : 1.0) : 0.0;
        cnt = dadd(rint(dmul(dsub(1.0, k), hc)), lc);
    }
    const double one_minus = dsub(1.0, alpha);
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        double live, hist;
        if (fixed) {
            live = static_cast<double>(static_cast<int64_t>(cs.sums[c])) / kFixedScale;
            hist = static_cast<double>(static_cast<int64_t>(cs.hist[c])) / kFixedScale;
        } else {
            live = __longlong_as_double(cs.sums[c]);
            hist = __longlong_as_double(cs.hist[c]);
        }
        const double lmean = lc > 0.0 ? ddiv(live, np_max(lc, 1.0)) : 0.0;
        const double hmean = hc > 0.0 ? ddiv(hist, np_max(hc, 1.0)) : 0.0;
        const double mean = dadd(dmul(alpha, hmean), dmul(one_minus, lmean));
        double es = dmul(mean, cnt);
        if (fixed) es = dmul(es, kFixedScale);
        e.fsum[c] = es;
        e.isum[c] = 0;
    }
    e.icnt = 0;
    e.fcnt = cnt;
    return e;
}

// VoxelTable.effective of one slot of a table the kernel does not write.
__device__ __forceinline__ Effective effective_at(const pf_table &t, int64_t s, int mode,
                                                  double ema, double delta_max) {
    return effective_of(load_cell(t, s, true), t.sum_mode == PF_SUM_FIXED, mode, ema, delta_max);
}

// True when eff sums are int64 (fixed-point integrate), i.e. numpy kept int64 dtype.
__device__ __forceinline__ bool eff_is_int(const pf_table &t, int mode) {
    return mode == PF_INTEGRATE && t.sum_mode == PF_SUM_FIXED;
}

__device__ __forceinline__ double eff_sum_f64(const Effective &e, bool as_int, int c) {
    return as_int ? static_cast<double>(e.isum[c]) : e.fsum[c];
}

}  // namespace pf
