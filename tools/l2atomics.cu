// Sustained L2 atomic throughput on this GPU (SURVEY.md 8d asks for the distinct- and
// same-address red/atom rates the insert kernel is compared against).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/l2atomics.cu -o tools/l2atomics
//   ./tools/l2atomics            -> one line per pattern: G atomic ops / s
//
// Patterns (each thread issues kPer operations, 148 x 8 CTAs x 256 threads):
//   red_u64_random     RED.ADD.U64 to hashed addresses in a 32 MB (L2-resident) buffer
//   red_f64_random     RED.ADD.F64, same addresses
//   red_u64_coalesced  RED.ADD.U64, a warp's lanes on 32 consecutive words
//   red_u64_same_warp  RED.ADD.U64, all lanes of a warp on one word (one word per warp)
//   red_u64_same_all   RED.ADD.U64, every thread on one word
//   atom_cas_random    ATOM.CAS.64 to hashed addresses (returns a value)
#include <cstdint>
#include <cstdio>

constexpr int kPer = 64;

__device__ __forceinline__ uint64_t mix(uint64_t x) {
    x ^= x >> 33;
    x *= 0xFF51AFD7ED558CCDull;
    x ^= x >> 33;
    return x;
}

template <int PATTERN>
__global__ void __launch_bounds__(256) k(unsigned long long *buf, uint64_t words, uint64_t salt) {
    const uint64_t tid = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const uint64_t warp = tid >> 5, lane = tid & 31;
    unsigned long long acc = 0;
#pragma unroll 4
    for (int j = 0; j < kPer; ++j) {
        uint64_t a;
        if (PATTERN == 0 || PATTERN == 1 || PATTERN == 5) a = mix(tid * kPer + j + salt) % words;
        else if (PATTERN == 2) a = ((warp * kPer + j) * 32 + lane) % words;
        else if (PATTERN == 3) a = (warp * 97 + j) % words;
        else a = 0;
        if (PATTERN == 1) {
            asm volatile("red.relaxed.gpu.global.add.f64 [%0], %1;" ::"l"(buf + a), "d"(1.0) : "memory");
        } else if (PATTERN == 5) {
            acc += atomicCAS(buf + a, 0ull, 1ull);
        } else {
            asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" ::"l"(buf + a), "l"(1ull) : "memory");
        }
    }
    if (acc == 0xdeadbeefull) buf[0] = acc;
}

int main() {
    const uint64_t words = (32ull << 20) / 8;
    unsigned long long *buf;
    cudaMalloc(&buf, words * 8);
    cudaMemset(buf, 0, words * 8);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const unsigned blocks = static_cast<unsigned>(sms) * 8;
    const double ops = static_cast<double>(blocks) * 256 * kPer;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    auto run = [&](auto kern, const char *name) {
        for (int w = 0; w < 3; ++w) kern<<<blocks, 256>>>(buf, words, w);
        cudaEventRecord(a);
        const int reps = 20;
        for (int r = 0; r < reps; ++r) kern<<<blocks, 256>>>(buf, words, 100 + r);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        printf("{\"pattern\": \"%s\", \"gops_per_s\": %.2f}\n", name, ops * reps / (ms * 1e-3) / 1e9);
    };
    run(k<0>, "red_u64_random");
    run(k<1>, "red_f64_random");
    run(k<2>, "red_u64_coalesced");
    run(k<3>, "red_u64_same_warp");
    run(k<4>, "red_u64_same_all");
    run(k<5>, "atom_cas_random");
    return 0;
}
