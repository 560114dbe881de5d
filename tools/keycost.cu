// Micro-benchmark: cost of each stage of the per-vertex key recipe on B200.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -std=c++17 tools/keycost.cu -o tools/keycost
#include <cstdio>
#include <vector>

#include "../paper_1902_05942_b200/csrc/pf_device.cuh"

using namespace pf;

template <int STAGE>
__global__ void __launch_bounds__(256) stage_kernel(pf_config cfg, pf_vertices v, uint64_t h0,
                                                    unsigned long long *sink) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= v.n) return;
    const VertexIn x = load_vertex(v, i, cfg);
    uint64_t acc = static_cast<uint64_t>(x.pixel) ^ static_cast<uint64_t>(x.sample) ^
                   __double_as_longlong(x.pos[0] + x.nrm[2] + x.dist);
    double u1 = 0, u2 = 0, du = 0, dv = 0;
    if (STAGE >= 1) {
        jitter_draws(h0, x.pixel, x.sample, u1, u2);
        acc ^= __double_as_longlong(u1) ^ __double_as_longlong(u2);
    }
    if (STAGE >= 2) {
        disc_offset(u1, u2, du, dv);
        acc ^= __double_as_longlong(du) ^ __double_as_longlong(dv);
    }
    KeyShared ks{};
    if (STAGE >= 3) {
        ks = key_shared(cfg, x);
        acc ^= ks.aux ^ __double_as_longlong(ks.frame.t1[0] + ks.frame.t2[1]);
    }
    if (STAGE >= 4) {
        double jt[3];
        const CellKey k = make_key(cfg, x, ks, 1, du, dv, 0, jt);
        acc ^= k.q[0] ^ k.q[1] ^ k.q[2] ^ k.level;
        if (STAGE >= 5) {
            const CellHash h = key_hash(k, ks);
            acc ^= h.index ^ h.fp;
        }
    }
    if (acc == 0x123456789ull) atomicAdd(sink, 1ull);  // keep the work alive
}

int main() {
    const int64_t n = 8294400;
    std::vector<double> pos(3 * n), nrm(3 * n), dist(n);
    std::vector<int64_t> pix(n), smp(n);
    for (int64_t i = 0; i < n; ++i) {
        pos[3 * i] = (i % 1920) * 0.003;
        pos[3 * i + 1] = 0.0;
        pos[3 * i + 2] = (i / 1920 % 1080) * 0.005;
        nrm[3 * i] = 0.0;
        nrm[3 * i + 1] = 1.0;
        nrm[3 * i + 2] = 0.0;
        dist[i] = 3.5 + (i % 7) * 0.3;
        pix[i] = i % 2073600;
        smp[i] = i / 2073600;
    }
    double *dp, *dn, *dd;
    int64_t *dpx, *dsm;
    unsigned long long *sink;
    cudaMalloc(&dp, 24 * n);
    cudaMalloc(&dn, 24 * n);
    cudaMalloc(&dd, 8 * n);
    cudaMalloc(&dpx, 8 * n);
    cudaMalloc(&dsm, 8 * n);
    cudaMalloc(&sink, 8);
    cudaMemcpy(dp, pos.data(), 24 * n, cudaMemcpyHostToDevice);
    cudaMemcpy(dn, nrm.data(), 24 * n, cudaMemcpyHostToDevice);
    cudaMemcpy(dd, dist.data(), 8 * n, cudaMemcpyHostToDevice);
    cudaMemcpy(dpx, pix.data(), 8 * n, cudaMemcpyHostToDevice);
    cudaMemcpy(dsm, smp.data(), 8 * n, cudaMemcpyHostToDevice);
    pf_config cfg{};
    cfg.c_lod = 0.0011111 * 8 / 0.01;
    cfg.base_voxel = 0.01;
    for (int k = 1; k < 32; ++k) cfg.lod_threshold[k] = static_cast<double>(1ll << k);
    cfg.normal_bins = 8;
    cfg.include_normal = 1;
    cfg.jitter = 1;
    pf_vertices v{dp, dn, nullptr, nullptr, nullptr, dpx, dsm, nullptr, dd, n};
    const unsigned g = static_cast<unsigned>((n + 255) / 256);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const char *names[] = {"loads", "+draws", "+sincos", "+frame/aux", "+make_key", "+hash"};
    auto run = [&](auto kern, int s) {
        for (int w = 0; w < 3; ++w) kern<<<g, 256>>>(cfg, v, 12345ull, sink);
        cudaEventRecord(a);
        for (int r = 0; r < 10; ++r) kern<<<g, 256>>>(cfg, v, 12345ull, sink);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        printf("%-12s %8.3f ms\n", names[s], ms / 10);
    };
    run(stage_kernel<0>, 0);
    run(stage_kernel<1>, 1);
    run(stage_kernel<2>, 2);
    run(stage_kernel<3>, 3);
    run(stage_kernel<4>, 4);
    run(stage_kernel<5>, 5);
    printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
