// Micro-benchmark: the resolve composite pattern -- 8.3M vertices in 4 pixel-order
// sweeps, each RED-adding 3 doubles into a 2,073,600 x 3 float64 buffer, plus a
// 44 B/vertex streamed read -- under different L2 policies.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/redbench.cu -o tools/redbench
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint64_t pol(int kind) {
    uint64_t p;
    if (kind == 1) asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    else if (kind == 2) asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    else asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
    return p;
}

template <int STREAM_POL, int RED_POL, bool DO_RED>
__global__ void comp(const double *tp, const int64_t *pix, double *flat, int64_t n, double *sink) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint64_t ps = pol(STREAM_POL), pr = pol(RED_POL);
    int64_t p;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.s64 %0, [%1], %2;" : "=l"(p) : "l"(pix + i), "l"(ps));
    double acc = 0;
    for (int c = 0; c < 3; ++c) {
        double t;
        asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(t) : "l"(tp + 3 * i + c), "l"(ps));
        if (DO_RED)
            asm volatile("red.relaxed.gpu.global.add.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(flat + 3 * p + c), "d"(t), "l"(pr) : "memory");
        acc += t;
    }
    if (acc == -1.0) *sink = acc;
}

int main() {
    const int64_t npix = 2073600, n = 4 * npix;
    double *tp, *flat, *sink;
    int64_t *pix;
    cudaMalloc(&tp, 24 * n);
    cudaMalloc(&flat, 24 * npix);
    cudaMalloc(&pix, 8 * n);
    cudaMalloc(&sink, 8);
    int64_t *h = new int64_t[n];
    for (int64_t i = 0; i < n; ++i) h[i] = i % npix;
    cudaMemcpy(pix, h, 8 * n, cudaMemcpyHostToDevice);
    cudaMemset(tp, 0, 24 * n);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const unsigned g = static_cast<unsigned>((n + 255) / 256);
    auto run = [&](auto k, const char *name) {
        for (int w = 0; w < 3; ++w) k<<<g, 256>>>(tp, pix, flat, n, sink);
        cudaEventRecord(a);
        for (int r = 0; r < 10; ++r) k<<<g, 256>>>(tp, pix, flat, n, sink);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        printf("%-36s %8.3f ms\n", name, ms / 10);
    };
    run(comp<0, 0, false>, "stream only (normal)");
    run(comp<1, 0, false>, "stream only (evict_first)");
    run(comp<0, 0, true>, "red normal, stream normal");
    run(comp<1, 2, true>, "red evict_last, stream evict_first");
    run(comp<1, 0, true>, "red normal, stream evict_first");
    printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
