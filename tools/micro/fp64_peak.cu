// Microbenchmark: non-FMA fp64 throughput on this GPU (the ALU roofline of
// the decision kernels, which evaluate the reference's 4 DMUL + 3 DADD
// bilinear with no contraction).  Each thread runs 8 independent chains;
// the grid covers every SM many times.  Prints one JSON line:
//   dmul_per_s, dadd_per_s, mix_per_s (4 DMUL : 3 DADD, the bilinear's mix),
//   bilinear_evals_per_s = mix_per_s / 7, plus the SM clock it ran at.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a --fmad=false
#include <cuda_runtime.h>

#include <cstdio>

constexpr int kChains = 8;
constexpr int kIters = 4096;

template <int MODE>
__global__ void k(double seed, double* out) {
    double a[kChains], b[kChains];
#pragma unroll
    for (int c = 0; c < kChains; ++c) {
        a[c] = seed + threadIdx.x * 1e-9 + c;
        b[c] = 1.0 + c * 1e-12;
    }
    for (int i = 0; i < kIters; ++i) {
#pragma unroll
        for (int c = 0; c < kChains; ++c) {
            if (MODE == 0) {  // 7 DMUL
#pragma unroll
                for (int j = 0; j < 7; ++j) a[c] = __dmul_rn(a[c], b[c]);
            } else if (MODE == 1) {  // 7 DADD
#pragma unroll
                for (int j = 0; j < 7; ++j) a[c] = __dadd_rn(a[c], b[c]);
            } else {  // 4 DMUL + 3 DADD, the bilinear's operation mix
                double t = __dmul_rn(__dmul_rn(a[c], b[c]), b[c]);
                t = __dadd_rn(t, __dmul_rn(b[c], a[c]));
                t = __dadd_rn(t, __dmul_rn(b[c], b[c]));
                a[c] = __dadd_rn(t, b[c]);
            }
        }
    }
    double s = 0;
#pragma unroll
    for (int c = 0; c < kChains; ++c) s += a[c];
    if (s == 12345.678) out[0] = s;  // keep the work alive
}

int main() {
    int dev = 0, sms = 0, clk = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
    double* out;
    cudaMalloc(&out, 8);
    const int threads = 256, blocks = sms * 16;
    const double ops = double(blocks) * threads * kIters * kChains * 7;
    double rate[3];
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int mode = 0; mode < 3; ++mode) {
        auto launch = [&] {
            if (mode == 0) k<0><<<blocks, threads>>>(1.0, out);
            else if (mode == 1) k<1><<<blocks, threads>>>(1.0, out);
            else k<2><<<blocks, threads>>>(1.0, out);
        };
        launch();
        cudaDeviceSynchronize();
        float best = 1e30f;
        for (int r = 0; r < 5; ++r) {
            cudaEventRecord(e0);
            launch();
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms = 0;
            cudaEventElapsedTime(&ms, e0, e1);
            if (ms < best) best = ms;
        }
        rate[mode] = ops / (best * 1e-3);
    }
    std::printf("{\"dmul_per_s\": %.4e, \"dadd_per_s\": %.4e, \"mix_per_s\": %.4e, \"bilinear_evals_per_s\": %.4e, "
                "\"sms\": %d, \"max_sm_clock_mhz\": %d, \"per_sm_per_clk_mix\": %.2f}\n",
                rate[0], rate[1], rate[2], rate[2] / 7.0, sms, clk / 1000, rate[2] / sms / (clk * 1e3));
    return 0;
}
