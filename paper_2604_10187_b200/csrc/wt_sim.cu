// wt_sim.cu -- the synthetic-profile generator on the GPU (SURVEY.md 8(f)
// row 1): the reference's discrete-event wave simulator
// (wave_sim.cpp:80-117) and its SimulatorBackend profile sweep
// (profiler.cpp:192-218, run_profile order profiler.cpp:286-329).
//
// One warp per simulation: the S slot free-times live in registers, K per
// lane (S <= 32*K).  Each dispatched block takes the lexicographically
// smallest (free time, insertion counter) slot -- exactly the element the
// reference's std::priority_queue<pair<double,i64>, ..., greater> pops -- via
// a 5-step xor-shuffle argmin; block durations for 32 consecutive blocks are
// drawn in parallel (one splitmix64 stream per block, Box-Muller) and
// broadcast in order.  All arithmetic is binary64 _rn; with sigma = 0 the
// makespans are bit-identical to the reference, with sigma > 0 they differ
// only through libm log/cos ulps.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <string>
#include <vector>

#include "wavetune_c.h"
#include "wt_decide.h"
#include "wt_internal.h"

namespace wtb {
namespace sim {

constexpr unsigned FULL = 0xffffffffu;

__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {  // rng.hpp:9-14
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}
__device__ __forceinline__ uint64_t mix2(uint64_t a, uint64_t b) { return splitmix64(a ^ splitmix64(b)); }

// SplitMix64(seed).next_gaussian() (rng.hpp:31-57): two draws, Box-Muller.
__device__ __forceinline__ double gaussian(uint64_t seed) {
    uint64_t st = seed;
    auto next = [&]() {
        st += 0x9e3779b97f4a7c15ULL;
        uint64_t z = st;
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
        return z ^ (z >> 31);
    };
    const double u1 = __dmul_rn(__dadd_rn(double(next() >> 11), 1.0), 0x1.0p-53);
    const double u2 = __dmul_rn(__dadd_rn(double(next() >> 11), 1.0), 0x1.0p-53);
    return __dmul_rn(__dsqrt_rn(__dmul_rn(-2.0, log(u1))), cos(__dmul_rn(6.283185307179586, u2)));
}

struct Job {
    int64_t g;
    double mean, sigma, eps, gap;
    uint64_t seed;
};

__device__ __forceinline__ bool lex_lt(double ta, int ia, double tb, int ib) {
    return ta < tb || (ta == tb && ia < ib);
}

// Makespan of one simulation, computed by the calling warp (all lanes return it).
template <int K>
__device__ double simulate_warp(const Job& jb, int slots, int lane) {
    double t[K];
    int id[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
        const int e = lane + 32 * k;
        t[k] = e < slots ? 0.0 : __longlong_as_double(0x7ff0000000000000LL);
        id[k] = e < slots ? e : INT32_MAX;
    }
    // local minimum of this lane
    double lt = t[0];
    int li = id[0], lk = 0;
#pragma unroll
    for (int k = 1; k < K; ++k)
        if (lex_lt(t[k], id[k], lt, li)) {
            lt = t[k];
            li = id[k];
            lk = k;
        }
    int counter = slots;
    double next_dispatch = 0.0, makespan = 0.0;
    for (int64_t b0 = 0; b0 < jb.g; b0 += 32) {
        const int64_t blk = b0 + lane;
        double dur = jb.mean;
        if (jb.sigma > 0.0 && blk < jb.g)
            dur = __dadd_rn(jb.mean, __dmul_rn(jb.sigma, gaussian(mix2(jb.seed, uint64_t(blk)))));
        dur = (jb.eps < dur) ? dur : jb.eps;  // std::max(eps, dur)
        const int nb = int(jb.g - b0 < 32 ? jb.g - b0 : 32);
        for (int j = 0; j < nb; ++j) {
            // warp argmin of (free time, counter)
            double mt = lt;
            int mi = li;
#pragma unroll
            for (int off = 16; off >= 1; off >>= 1) {
                const double ot = __shfl_xor_sync(FULL, mt, off);
                const int oi = __shfl_xor_sync(FULL, mi, off);
                if (lex_lt(ot, oi, mt, mi)) {
                    mt = ot;
                    mi = oi;
                }
            }
            const double start = (mt < next_dispatch) ? next_dispatch : mt;  // std::max(t_slot, next)
            if (jb.gap > 0.0) next_dispatch = __dadd_rn(start, jb.gap);
            const double d = __shfl_sync(FULL, dur, j);
            const double finish = __dadd_rn(start, d);
            makespan = (makespan < finish) ? finish : makespan;
            if (li == mi) {  // owner lane: replace the popped slot, refresh local min
#pragma unroll
                for (int k = 0; k < K; ++k)
                    if (k == lk) {
                        t[k] = finish;
                        id[k] = counter;
                    }
                lt = t[0];
                li = id[0];
                lk = 0;
#pragma unroll
                for (int k = 1; k < K; ++k)
                    if (lex_lt(t[k], id[k], lt, li)) {
                        lt = t[k];
                        li = id[k];
                        lk = k;
                    }
            }
            ++counter;
        }
    }
    return makespan;
}

// Generic batch: one job per warp.
template <int K>
__global__ void k_simulate(const Job* jobs, int64_t n, int slots, double* out) {
    const int lane = threadIdx.x & 31;
    const int64_t w0 = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
    for (int64_t q = w0; q < n; q += nw) {
        const Job jb = jobs[q];
        const double m = simulate_warp<K>(jb, slots, lane);
        if (lane == 0) out[q] = m;
    }
}

// SimulatorBackend profile: record r = ((point * A) + anchor) * F + pair.
struct ProfileArgs {
    const int64_t* point_g;  // [P]
    const int64_t* anchor_l; // [A]
    const int32_t* pair_macro;  // [F] feasible (macro, micro) in run_profile order
    const int32_t* pair_micro;
    const double* pair_base;
    const double* pair_per_iter;
    const double* pair_gap;
    int64_t P, A, F;
    double sigma, floor_frac;
    uint64_t seed;
    int32_t warmup, measured, slots;
    double* lat;     // [P*A*F]
    int32_t* status; // [P*A*F]
};

template <int K>
__global__ void k_profile(ProfileArgs a) {
    const int lane = threadIdx.x & 31;
    const int64_t w0 = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
    const int64_t total = a.P * a.A * a.F;
    for (int64_t r = w0; r < total; r += nw) {
        const int64_t f = r % a.F, pa = r / a.F;
        const int64_t an = pa % a.A, p = pa / a.A;
        const int64_t g = a.point_g[p], l = a.anchor_l[an];
        const int32_t ma = a.pair_macro[f], mi = a.pair_micro[f];
        // mean_fn = ground.mean (wave_sim.cpp:37-40): base + per_iter * l
        const double mean = __dadd_rn(a.pair_base[f], __dmul_rn(a.pair_per_iter[f], double(l)));
        int32_t st = 0;
        if (g < 1 || l < 1) st = WT_INVALID_ARGUMENT;
        else if (!(mean > 0.0)) st = WT_INVALID_ARGUMENT;  // wave_sim.cpp:87
        double total_lat = 0.0;
        if (!st) {
            Job jb;
            jb.g = g;
            jb.mean = mean;
            jb.sigma = a.sigma;
            jb.eps = __dmul_rn(a.floor_frac, mean);
            jb.gap = a.pair_gap[f];
            const uint64_t inner = mix2(mix2(uint64_t(l), uint64_t(int64_t(ma))), uint64_t(int64_t(mi)));
            const uint64_t base = mix2(mix2(a.seed, uint64_t(g)), inner);
            for (int it = 0; it < a.warmup + a.measured; ++it) {
                jb.seed = mix2(base, uint64_t(it));  // profiler.cpp:209-212
                const double m = simulate_warp<K>(jb, a.slots, lane);
                if (it >= a.warmup) total_lat = __dadd_rn(total_lat, m);
            }
        }
        if (lane == 0) {
            a.lat[r] = st ? 0.0 : __ddiv_rn(total_lat, double(a.measured));
            a.status[r] = st;
        }
    }
}

template <typename F>
cudaError_t by_k(int slots, F&& f) {
    if (slots <= 32) return f(std::integral_constant<int, 1>{});
    if (slots <= 64) return f(std::integral_constant<int, 2>{});
    if (slots <= 128) return f(std::integral_constant<int, 4>{});
    if (slots <= 160) return f(std::integral_constant<int, 5>{});
    if (slots <= 256) return f(std::integral_constant<int, 8>{});
    if (slots <= 512) return f(std::integral_constant<int, 16>{});
    return f(std::integral_constant<int, 32>{});
}

}  // namespace sim
}  // namespace wtb

using namespace wtb::sim;

extern "C" {

wt_status wt_simulate_batch(const int64_t* g, const double* mean, const double* sigma, const double* eps,
                            const double* gap, const uint64_t* seed, int64_t n, int32_t slots, double* makespan,
                            int device) {
    if (n <= 0) return WT_OK;
    if (slots < 1) {
        wtb::set_last_error("hardware spec must have positive capacities");
        return WT_INVALID_ARGUMENT;
    }
    if (slots > 1024) {
        wtb::set_last_error("simulated slots above 1024 are outside the device path's range");
        return WT_UNSUPPORTED;
    }
    std::vector<Job> jobs(n);
    for (int64_t i = 0; i < n; ++i) {
        if (g[i] < 1) {
            wtb::set_last_error("grid size and loop count must be >= 1");
            return WT_INVALID_ARGUMENT;
        }
        if (!(mean[i] > 0)) {
            wtb::set_last_error("mean block duration must be positive");
            return WT_INVALID_ARGUMENT;
        }
        jobs[i] = Job{g[i], mean[i], sigma[i], eps[i], gap[i], seed[i]};
    }
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(device);
    Job* dj = nullptr;
    double* dout = nullptr;
    cudaError_t ce = cudaMalloc(&dj, sizeof(Job) * n);
    if (ce == cudaSuccess) ce = cudaMalloc(&dout, sizeof(double) * n);
    if (ce == cudaSuccess) ce = cudaMemcpy(dj, jobs.data(), sizeof(Job) * n, cudaMemcpyHostToDevice);
    if (ce == cudaSuccess) {
        const int grid = int(std::min<int64_t>((n + 7) / 8, 148 * 64));
        ce = by_k(slots, [&](auto kc) {
            k_simulate<decltype(kc)::value><<<grid, 256>>>(dj, n, slots, dout);
            return cudaGetLastError();
        });
    }
    if (ce == cudaSuccess) ce = cudaMemcpy(makespan, dout, sizeof(double) * n, cudaMemcpyDeviceToHost);
    cudaFree(dj);
    cudaFree(dout);
    cudaSetDevice(prev);
    if (ce != cudaSuccess) {
        wtb::set_last_error(std::string("wt_simulate_batch: ") + cudaGetErrorString(ce));
        return WT_CUDA_ERROR;
    }
    return WT_OK;
}

wt_status wt_profile_sim(const wt_sim_profile_desc* d, double* latency_us, int32_t* status, int device,
                         double* device_ms) {
    if (!d || !latency_us || !status) {
        wtb::set_last_error("null argument");
        return WT_INVALID_ARGUMENT;
    }
    if (d->measured < 1) {
        wtb::set_last_error("measured iterations must be >= 1");
        return WT_INVALID_ARGUMENT;
    }
    if (d->slots < 1 || d->slots > 1024) {
        wtb::set_last_error(d->slots < 1 ? "hardware spec must have positive capacities"
                                         : "simulated slots above 1024 are outside the device path's range");
        return d->slots < 1 ? WT_INVALID_ARGUMENT : WT_UNSUPPORTED;
    }
    const int64_t P = d->n_points, A = d->n_anchors, F = d->n_pairs, total = P * A * F;
    if (total <= 0) return WT_OK;
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(device);
    std::vector<void*> owned;
    auto put = [&](const void* src, size_t bytes) -> void* {
        void* p = nullptr;
        if (cudaMalloc(&p, std::max<size_t>(bytes, 8)) != cudaSuccess) return nullptr;
        owned.push_back(p);
        if (src) cudaMemcpy(p, src, bytes, cudaMemcpyHostToDevice);
        return p;
    };
    ProfileArgs a{};
    a.point_g = static_cast<const int64_t*>(put(d->point_g, P * 8));
    a.anchor_l = static_cast<const int64_t*>(put(d->anchor_l, A * 8));
    a.pair_macro = static_cast<const int32_t*>(put(d->pair_macro, F * 4));
    a.pair_micro = static_cast<const int32_t*>(put(d->pair_micro, F * 4));
    a.pair_base = static_cast<const double*>(put(d->pair_base, F * 8));
    a.pair_per_iter = static_cast<const double*>(put(d->pair_per_iter, F * 8));
    a.pair_gap = static_cast<const double*>(put(d->pair_gap, F * 8));
    a.P = P;
    a.A = A;
    a.F = F;
    a.sigma = d->sigma;
    a.floor_frac = d->floor_frac;
    a.seed = d->seed;
    a.warmup = d->warmup;
    a.measured = d->measured;
    a.slots = d->slots;
    a.lat = static_cast<double*>(put(nullptr, total * 8));
    a.status = static_cast<int32_t*>(put(nullptr, total * 4));
    cudaError_t ce = a.status ? cudaSuccess : cudaErrorMemoryAllocation;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    if (ce == cudaSuccess) {
        cudaEventRecord(e0);
        const int grid = int(std::min<int64_t>((total + 7) / 8, 148 * 64));
        ce = by_k(d->slots, [&](auto kc) {
            k_profile<decltype(kc)::value><<<grid, 256>>>(a);
            return cudaGetLastError();
        });
        cudaEventRecord(e1);
    }
    if (ce == cudaSuccess) ce = cudaMemcpy(latency_us, a.lat, total * 8, cudaMemcpyDeviceToHost);
    if (ce == cudaSuccess) ce = cudaMemcpy(status, a.status, total * 4, cudaMemcpyDeviceToHost);
    float ms = 0.f;
    if (ce == cudaSuccess) cudaEventElapsedTime(&ms, e0, e1);
    if (device_ms) *device_ms = ms;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    for (void* p : owned) cudaFree(p);
    cudaSetDevice(prev);
    if (ce != cudaSuccess) {
        wtb::set_last_error(std::string("wt_profile_sim: ") + cudaGetErrorString(ce));
        return WT_CUDA_ERROR;
    }
    return WT_OK;
}

}  // extern "C"
