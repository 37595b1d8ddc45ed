// Microbenchmark: the DRAM ceiling of the gather's traffic pattern.  For n
// queries, read three int32 streams (M, N, K: 12 B / query) and write three
// result streams (macro, micro int32 + latency f64: 16 B / query) with the
// gather's 16-byte streaming loads / stores (ld.global.cs / st.global.cs),
// persistent grid of 3 x 256 threads per SM, one grid-stride prefetch -- no
// lookup work.  Also a 1:1 int4 copy for comparison with MEASURED_PEAKS.json.
// Prints one JSON line: GB/s of each (read + write bytes, best of 20 after 3
// warm-ups, CUDA events).
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a
#include <cuda_runtime.h>

#include <cstdio>

__global__ void __launch_bounds__(256) k_mix(const int4* M, const int4* N, const int4* K, int4* mac, int4* mic,
                                             double2* lat, long nv) {
    const long stride = long(gridDim.x) * blockDim.x;
    long v = long(blockIdx.x) * blockDim.x + threadIdx.x;
    int4 pm = make_int4(0, 0, 0, 0), pn = pm, pk = pm;
    if (v < nv) {
        pm = __ldcs(M + v);
        pn = __ldcs(N + v);
        pk = __ldcs(K + v);
    }
    for (; v < nv; v += stride) {
        const int4 m = pm, n = pn, k = pk;
        if (v + stride < nv) {
            pm = __ldcs(M + v + stride);
            pn = __ldcs(N + v + stride);
            pk = __ldcs(K + v + stride);
        }
        __stcs(mac + v, make_int4(m.x ^ n.x, m.y ^ n.y, m.z ^ n.z, m.w ^ n.w));
        __stcs(mic + v, make_int4(k.x, k.y, k.z, k.w));
        __stcs(lat + 2 * v, make_double2(double(m.x), double(m.y)));
        __stcs(lat + 2 * v + 1, make_double2(double(m.z), double(m.w)));
    }
}

__global__ void __launch_bounds__(256) k_copy(const int4* a, int4* b, long nv) {
    const long stride = long(gridDim.x) * blockDim.x;
    for (long v = long(blockIdx.x) * blockDim.x + threadIdx.x; v < nv; v += stride) __stcs(b + v, __ldcs(a + v));
}

int main() {
    const long n = 100000000;  // queries (the bench stream)
    const long nv = n / 4;
    int4 *M, *N, *K, *mac, *mic, *A, *B;
    double2* lat;
    cudaMalloc(&M, n * 4);
    cudaMalloc(&N, n * 4);
    cudaMalloc(&K, n * 4);
    cudaMalloc(&mac, n * 4);
    cudaMalloc(&mic, n * 4);
    cudaMalloc(&lat, n * 8);
    const long cb = 1l << 30;  // 1 GiB each way
    cudaMalloc(&A, cb);
    cudaMalloc(&B, cb);
    cudaMemset(M, 1, n * 4);
    cudaMemset(N, 2, n * 4);
    cudaMemset(K, 3, n * 4);
    cudaMemset(A, 4, cb);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto best = [&](auto launch) {
        float b = 1e30f;
        for (int i = 0; i < 23; ++i) {
            cudaEventRecord(e0);
            launch();
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (i >= 3 && ms < b) b = ms;
        }
        return b;
    };
    const float t_mix = best([&] { k_mix<<<sms * 3, 256>>>(M, N, K, mac, mic, lat, nv); });
    const float t_mix8 = best([&] { k_mix<<<sms * 8, 256>>>(M, N, K, mac, mic, lat, nv); });
    const float t_copy = best([&] { k_copy<<<sms * 8, 256>>>(A, B, cb / 16); });
    const double mix_bytes = double(n) * 28.0, copy_bytes = 2.0 * cb;
    printf("{\"gather_pattern_3x256_gbs\": %.1f, \"gather_pattern_8x256_gbs\": %.1f, \"copy_1to1_gbs\": %.1f, "
           "\"gather_pattern_ms\": %.4f, \"queries\": %ld, \"bytes_per_query\": 28, \"error\": \"%s\"}\n",
           mix_bytes / (t_mix * 1e-3) / 1e9, mix_bytes / (t_mix8 * 1e-3) / 1e9, copy_bytes / (t_copy * 1e-3) / 1e9,
           t_mix, n, cudaGetErrorString(cudaGetLastError()));
    return 0;
}
