// Phase one on the device: the deterministic forward path tracer that produces the
// vertex stream the filter consumes (src/tracer.py:211-383 _walk, with the brute-force
// ray/triangle tests of src/_native.pyx:83-167).  One thread walks one path (pixel,
// sample) through up to max_depth bounces: closest hit, emission, selection of the
// select_k-th sufficiently diffuse vertex, next-event estimation toward a sampled
// light point with a shadow ray, one-sample continuation over the layered BRDF,
// Russian roulette.  All randomness is the counter RNG keyed by (seed, path id,
// bounce, dimension) (src/rng.py:62-78), so any path replays exactly.
//
// FP64 throughout with numpy's operation order and no FMA contraction (the library is
// built with -fmad=false); sqrt and division are IEEE and sin/cos are glibc's
// (glibc_sincos), so diffuse paths replay the reference bit for bit.  The glossy
// lobe's pow is CUDA's (numpy's float64 pow here is its own SIMD routine, not libm),
// so glossy paths agree to a few ulps (tests/test_gpu_tracer.py states the bars).
#include "pf_device.cuh"
#include "pf_internal.cuh"

namespace pf {

namespace {

constexpr double kTMin = 1e-7;                 // src/tracer.py:30
constexpr double kShadowShrink = 1.0 - 1e-6;   // src/tracer.py:31
constexpr double kDetEps = 1e-14;              // src/_native.pyx:72
constexpr double kPi = 3.141592653589793;      // math.pi
constexpr double kTwoPiT = 6.283185307179586;  // 2.0 * math.pi
enum Dim { kLightSel = 0, kLightU = 1, kLightV = 2, kLobe = 3, kDirU = 4, kDirV = 5, kRR = 6 };

struct V3 {
    double x, y, z;
};

__device__ __forceinline__ V3 ld3(const double *p, int64_t i) {
    return V3{__ldg(p + 3 * i), __ldg(p + 3 * i + 1), __ldg(p + 3 * i + 2)};
}
__device__ __forceinline__ V3 add(V3 a, V3 b) { return V3{a.x + b.x, a.y + b.y, a.z + b.z}; }
__device__ __forceinline__ V3 sub(V3 a, V3 b) { return V3{a.x - b.x, a.y - b.y, a.z - b.z}; }
__device__ __forceinline__ V3 mul(V3 a, V3 b) { return V3{a.x * b.x, a.y * b.y, a.z * b.z}; }
__device__ __forceinline__ V3 scale(double s, V3 a) { return V3{s * a.x, s * a.y, s * a.z}; }
__device__ __forceinline__ V3 neg(V3 a) { return V3{-a.x, -a.y, -a.z}; }
// np.einsum("ij,ij->i") for rows of 3: (a0*b0 + a2*b2) + a1*b1 (see aux_word)
__device__ __forceinline__ double dot(V3 a, V3 b) { return (a.x * b.x + a.z * b.z) + a.y * b.y; }
// np.linalg.norm(axis=1): sqrt of the sequential sum of squares
__device__ __forceinline__ double norm(V3 a) { return sqrt((a.x * a.x + a.y * a.y) + a.z * a.z); }
__device__ __forceinline__ double vmax(V3 a) { return fmax(fmax(a.x, a.y), a.z); }

// draw_unit_array(seed, STREAM_TRACE, path_id, bounce, dim) = mix64 over the fields in
// turn; hp = the hash after the path id (per path), hb = after the bounce (shared by
// that bounce's seven dimensions).
__device__ __forceinline__ uint64_t bounce_hash(uint64_t hp, int64_t bounce) {
    return mix64(hp ^ (static_cast<uint64_t>(bounce) + kGolden));
}
__device__ __forceinline__ double draw(uint64_t hb, int dim) {
    const uint64_t u = mix64(hb ^ (static_cast<uint64_t>(dim) + kGolden));
    return static_cast<double>(u >> 11) * (1.0 / 9007199254740992.0);
}

// Moeller-Trumbore exactly as src/_native.pyx:95-124: closest t in (t_min, t_max).
__device__ __forceinline__ int64_t hit_closest(const pf_scene &sc, V3 o, V3 d, double &t_best) {
    double best = INFINITY;
    int64_t best_i = -1;
    for (int64_t k = 0; k < sc.n_triangles; ++k) {
        const V3 e1 = ld3(sc.e1, k), e2 = ld3(sc.e2, k);
        const double px = d.y * e2.z - d.z * e2.y;
        const double py = d.z * e2.x - d.x * e2.z;
        const double pz = d.x * e2.y - d.y * e2.x;
        const double det = e1.x * px + e1.y * py + e1.z * pz;
        if (det <= kDetEps && det >= -kDetEps) continue;
        const double inv = 1.0 / det;
        const V3 v0 = ld3(sc.v0, k);
        const double tx = o.x - v0.x, ty = o.y - v0.y, tz = o.z - v0.z;
        const double u = (tx * px + ty * py + tz * pz) * inv;
        if (u < 0.0) continue;
        const double qx = ty * e1.z - tz * e1.y;
        const double qy = tz * e1.x - tx * e1.z;
        const double qz = tx * e1.y - ty * e1.x;
        const double v = (d.x * qx + d.y * qy + d.z * qz) * inv;
        if (v < 0.0 || u + v > 1.0) continue;
        const double t = (e2.x * qx + e2.y * qy + e2.z * qz) * inv;
        if (t > kTMin && t < best) {
            best = t;
            best_i = k;
        }
    }
    t_best = best;
    return best_i;
}

// src/_native.pyx:128-167: any hit in (t_min, t_max).
__device__ __forceinline__ bool hit_any(const pf_scene &sc, V3 o, V3 d, double t_max) {
    for (int64_t k = 0; k < sc.n_triangles; ++k) {
        const V3 e1 = ld3(sc.e1, k), e2 = ld3(sc.e2, k);
        const double px = d.y * e2.z - d.z * e2.y;
        const double py = d.z * e2.x - d.x * e2.z;
        const double pz = d.x * e2.y - d.y * e2.x;
        const double det = e1.x * px + e1.y * py + e1.z * pz;
        if (det <= kDetEps && det >= -kDetEps) continue;
        const double inv = 1.0 / det;
        const V3 v0 = ld3(sc.v0, k);
        const double tx = o.x - v0.x, ty = o.y - v0.y, tz = o.z - v0.z;
        const double u = (tx * px + ty * py + tz * pz) * inv;
        if (u < 0.0) continue;
        const double qx = ty * e1.z - tz * e1.y;
        const double qy = tz * e1.x - tx * e1.z;
        const double qz = tx * e1.y - ty * e1.x;
        const double v = (d.x * qx + d.y * qy + d.z * qz) * inv;
        if (v < 0.0 || u + v > 1.0) continue;
        const double t = (e2.x * qx + e2.y * qy + e2.z * qz) * inv;
        if (t > kTMin && t < t_max) return true;
    }
    return false;
}

// _tangent_frame (src/tracer.py:124-131)
__device__ __forceinline__ void frame_of(V3 n, V3 &t1, V3 &t2) {
    const double s = n.z >= 0.0 ? 1.0 : -1.0;
    const double a = -1.0 / (s + n.z);
    const double b = n.x * n.y * a;
    t1 = V3{1.0 + s * n.x * n.x * a, s * b, -s * n.x};
    t2 = V3{b, s + n.y * n.y * a, -n.y};
}

// (c1 * t1 + c2 * t2) + c3 * axis, numpy's left-to-right sum of the three rows
__device__ __forceinline__ V3 lobe_dir(double c1, double c2, double c3, V3 axis) {
    V3 t1, t2;
    frame_of(axis, t1, t2);
    return add(add(scale(c1, t1), scale(c2, t2)), scale(c3, axis));
}

struct Mat {
    V3 albedo;
    double gw, ge, dw;
};

__device__ __forceinline__ Mat material(const pf_scene &sc, int m) {
    Mat r;
    r.albedo = ld3(sc.albedo, m);
    r.gw = __ldg(sc.glossy_weight + m);
    r.ge = __ldg(sc.glossy_exponent + m);
    r.dw = 1.0 - r.gw;
    return r;
}

// glossy lobe value gw*(e+c)/(2pi) * max(dot(reflect(wo), wi), 0)^e
__device__ __forceinline__ double glossy_term(const Mat &m, V3 n, V3 wo, V3 wi, double c) {
    const V3 r = sub(scale(2.0 * dot(n, wo), n), wo);
    const double align = fmax(dot(r, wi), 0.0);
    return m.gw * (m.ge + c) / kTwoPiT * pow(align, m.ge);
}

// _bsdf_eval (src/tracer.py:171-183)
__device__ __forceinline__ V3 bsdf_eval(const Mat &m, V3 wo, V3 wi, V3 n) {
    const double cosi = dot(n, wi);
    const double kd = m.dw / kPi;
    V3 f = V3{m.albedo.x * kd, m.albedo.y * kd, m.albedo.z * kd};
    if (m.gw > 0.0) {
        const double spec = glossy_term(m, n, wo, wi, 2.0);
        f = V3{f.x + spec, f.y + spec, f.z + spec};
    }
    return cosi > 0.0 ? f : V3{0.0, 0.0, 0.0};
}

// _bsdf_pdf (src/tracer.py:186-195)
__device__ __forceinline__ double bsdf_pdf(const Mat &m, V3 wo, V3 wi, V3 n) {
    const double cosi = fmax(dot(n, wi), 0.0);
    double pdf = m.dw * cosi / kPi;
    if (m.gw > 0.0) pdf = pdf + glossy_term(m, n, wo, wi, 1.0);
    return pdf;
}

__global__ void __launch_bounds__(128)
trace_kernel(pf_scene sc, pf_trace_options opt, uint64_t h0, const int64_t *pixels,
             const int64_t *samples, int64_t n, pf_path_out out) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int64_t pixel = pixels[i];
    const int64_t sample = samples[i];
    const uint64_t pid = (static_cast<uint64_t>(sample) << 32) | static_cast<uint64_t>(pixel);

    // primary ray (src/tracer.py:220-230)
    const uint64_t hp = mix64(h0 ^ (pid + kGolden));
    const uint64_t hb0 = bounce_hash(hp, 0);
    const double jx = opt.pixel_jitter ? draw(hb0, 0) : 0.5;
    const double jy = opt.pixel_jitter ? draw(hb0, 1) : 0.5;
    const double col = static_cast<double>(pixel % sc.width);
    const double row = static_cast<double>(pixel / sc.width);
    const double ndc_x = ((col + jx) / static_cast<double>(sc.width) - 0.5) * sc.ndc_scale_x;
    const double ndc_y = (0.5 - (row + jy) / static_cast<double>(sc.height)) * sc.ndc_scale_y;
    const V3 right{sc.cam_right[0], sc.cam_right[1], sc.cam_right[2]};
    const V3 up{sc.cam_up[0], sc.cam_up[1], sc.cam_up[2]};
    const V3 fwd{sc.cam_fwd[0], sc.cam_fwd[1], sc.cam_fwd[2]};
    V3 d = add(add(fwd, scale(ndc_x, right)), scale(ndc_y, up));
    {
        const double len = norm(d);
        d = V3{d.x / len, d.y / len, d.z / len};
    }
    V3 o{sc.cam_pos[0], sc.cam_pos[1], sc.cam_pos[2]};

    const V3 zero{0.0, 0.0, 0.0};
    const V3 bg{sc.background[0], sc.background[1], sc.background[2]};
    const bool has_bg = vmax(bg) > 0.0;
    bool alive = true, post = false, has_v = false;
    V3 T{1.0, 1.0, 1.0}, Tsfx = zero, base = zero, contrib = zero;
    int64_t qual = 0, v_layer = 0;
    double pathlen = 0.0, v_dist = 0.0;
    V3 v_pos = zero, v_n = zero, v_wr = zero, v_T = zero;
    // add radiance L weighted by the stage's attenuation to base or to contrib
    auto gather = [&](V3 L) {
        if (post) contrib = add(contrib, mul(Tsfx, L));
        else base = add(base, mul(T, L));
    };

    for (int k = 1; k <= opt.max_depth && alive; ++k) {
        double t;
        const int64_t tri = hit_closest(sc, o, d, t);
        if (tri < 0) {  // escaped
            if (has_bg) gather(bg);
            alive = false;
            break;
        }
        const V3 x = add(o, scale(t, d));
        pathlen += t;
        const int mid = __ldg(sc.material_id + tri);
        const Mat m = material(sc, mid);
        const V3 n_g = ld3(sc.normal, tri);
        const double facing = -dot(n_g, d);
        const V3 nrm = facing > 0.0 ? n_g : neg(n_g);
        const V3 wo = neg(d);

        if (k == 1 || !opt.nee) {  // emission (later hits are covered by NEE)
            const V3 em0 = ld3(sc.emission, tri);
            const double vis = facing > 0.0 ? 1.0 : 0.0;
            const V3 em{em0.x * vis, em0.y * vis, em0.z * vis};
            if (vmax(em) > 0.0) gather(em);
        }

        // selection of the select_k-th sufficiently diffuse vertex (src/tracer.py:287-301)
        bool selected_now = false;
        if (!post && m.dw >= opt.diffuse_threshold) {
            ++qual;
            if (qual == opt.select_k) {
                post = true;
                has_v = true;
                selected_now = true;
                v_pos = x;
                v_n = nrm;
                v_wr = wo;
                v_T = T;
                v_dist = pathlen;
                Tsfx = V3{1.0, 1.0, 1.0};
            }
        }
        const uint64_t hb = bounce_hash(hp, k);

        if (opt.nee) {  // next event estimation (src/tracer.py:303-334)
            const int64_t nl = sc.n_lights;
            const double xi = draw(hb, kLightSel);
            int64_t li = np_i64(xi * static_cast<double>(nl));
            if (li > nl - 1) li = nl - 1;
            const double r1 = draw(hb, kLightU), r2 = draw(hb, kLightV);
            const double sq = sqrt(r1);
            const int64_t lt = __ldg(sc.light_tri + li);
            const V3 y = add(add(ld3(sc.v0, lt), scale(sq * (1.0 - r2), ld3(sc.e1, lt))),
                             scale(sq * r2, ld3(sc.e2, lt)));
            V3 wl = sub(y, x);
            const double dl = norm(wl);
            const bool ok = dl > 1e-6;
            const double dn = fmax(dl, 1e-6);
            wl = ok ? V3{wl.x / dn, wl.y / dn, wl.z / dn} : zero;
            const double cosx = dot(nrm, wl);
            const double cosl = -dot(ld3(sc.normal, lt), wl);
            if (ok && cosx > 0.0 && cosl > 0.0 && !hit_any(sc, x, wl, dl * kShadowShrink)) {
                const V3 f = bsdf_eval(m, wo, wl, nrm);
                const double geo = cosx * cosl / (dl * dl);
                const double inv_pdf = static_cast<double>(nl) * __ldg(sc.area + lt);
                const double w = geo * inv_pdf;
                const V3 le = ld3(sc.emission, lt);
                const V3 lf = mul(le, f);
                gather(V3{lf.x * w, lf.y * w, lf.z * w});
            }
        }

        // continuation over the layered BRDF (src/tracer.py:336-357)
        const bool pick_gloss = draw(hb, kLobe) < m.gw;
        const double u1 = draw(hb, kDirU), u2 = draw(hb, kDirV);
        const double phi = kTwoPiT * u2;
        double sphi, cphi;
        glibc_sincos(phi, sphi, cphi);
        V3 wi;
        if (pick_gloss) {
            const V3 mirror = sub(scale(2.0 * dot(nrm, wo), nrm), wo);
            const double c = pow(u1, 1.0 / (m.ge + 1.0));
            const double s = sqrt(fmax(1.0 - c * c, 0.0));
            wi = lobe_dir(s * cphi, s * sphi, c, mirror);
        } else {
            const double r = sqrt(u1);
            wi = lobe_dir(r * cphi, r * sphi, sqrt(fmax(1.0 - u1, 0.0)), nrm);
        }
        if (selected_now) v_layer = pick_gloss ? 1 : 0;
        const double cosi = dot(nrm, wi);
        const double pdf = bsdf_pdf(m, wo, wi, nrm);
        const bool up_ok = cosi > 0.0 && pdf > 0.0;
        V3 w = zero;
        if (up_ok) {
            const V3 f = bsdf_eval(m, wo, wi, nrm);
            const double g = cosi / fmax(pdf, 1e-300);
            w = V3{f.x * g, f.y * g, f.z * g};
        }
        if (post) Tsfx = mul(Tsfx, w);
        else T = mul(T, w);
        alive = up_ok;

        if (alive && k >= opt.rr_start) {  // Russian roulette (src/tracer.py:359-369)
            const V3 eff = post ? mul(v_T, Tsfx) : T;
            const double q = fmin(fmax(vmax(eff), opt.rr_lo), opt.rr_hi);
            if (draw(hb, kRR) >= q) {
                alive = false;
            } else if (post) {
                Tsfx = V3{Tsfx.x / q, Tsfx.y / q, Tsfx.z / q};
            } else {
                T = V3{T.x / q, T.y / q, T.z / q};
            }
        }
        if (alive && vmax(post ? Tsfx : T) <= 0.0) alive = false;
        o = x;
        d = wi;
    }

    const V3 rad = has_v ? add(base, mul(v_T, contrib)) : base;
    auto st3 = [&](double *p, V3 v) {
        if (p) {
            p[3 * i] = v.x;
            p[3 * i + 1] = v.y;
            p[3 * i + 2] = v.z;
        }
    };
    st3(out.base, base);
    st3(out.radiance, rad);
    out.has_vertex[i] = has_v ? 1 : 0;
    st3(out.position, v_pos);
    st3(out.normal, v_n);
    st3(out.omega_r, v_wr);
    st3(out.contribution, has_v ? contrib : zero);
    st3(out.throughput, v_T);
    if (out.layer_id) out.layer_id[i] = v_layer;
    if (out.camera_distance) out.camera_distance[i] = v_dist;
}

}  // namespace

}  // namespace pf

using namespace pf;

extern "C" int pf_trace_paths(const pf_scene *scene, const pf_trace_options *opt, uint64_t seed,
                              const int64_t *pixels, const int64_t *samples, int64_t n,
                              const pf_path_out *out, void *stream) {
    const char *fn = "pf_trace_paths";
    if (!scene || !opt || !out) return fail_arg(fn, "scene/options/out is NULL");
    if (n < 0) return fail_arg(fn, "negative path count");
    if (n == 0) return PF_OK;
    if (!pixels || !samples || !out->has_vertex) return fail_arg(fn, "pixels/samples/has_vertex is NULL");
    if (scene->n_triangles < 1 || scene->n_lights < 1 || scene->width < 1 || scene->height < 1)
        return fail_arg(fn, "scene needs triangles, a light and a positive image size");
    if (!scene->v0 || !scene->e1 || !scene->e2 || !scene->normal || !scene->emission ||
        !scene->area || !scene->material_id || !scene->albedo || !scene->glossy_weight ||
        !scene->glossy_exponent || !scene->light_tri)
        return fail_arg(fn, "scene array is NULL");
    if (opt->max_depth < 0 || opt->select_k < 1) return fail_arg(fn, "max_depth >= 0, select_k >= 1");
    uint64_t h0 = seed ^ kGolden;  // mix64(seed ^ STREAM_TRACE * G), STREAM_TRACE = 1
    h0 ^= h0 >> 33;
    h0 *= 0xFF51AFD7ED558CCDull;
    h0 ^= h0 >> 33;
    h0 *= 0xC4CEB9FE1A85EC53ull;
    h0 ^= h0 >> 33;
    const unsigned blocks = static_cast<unsigned>((n + 127) / 128);
    trace_kernel<<<blocks, 128, 0, as_stream(stream)>>>(*scene, *opt, h0, pixels, samples, n, *out);
    return check_launch(fn);
}
