// Microbenchmark: shared-memory wavefronts per LDS.128 / LDS.64 warp load
// for the lane->address patterns the list-mode evaluator produces.
// Run under: ncu --metrics l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum,smsp__inst_executed_op_shared_ld.sum
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ITERS = 1024;

__device__ __forceinline__ int slot_of(int pat, int lane) {
    switch (pat) {
        case 0: return 0;                                   // uniform
        case 1: return lane < 16 ? 0 : 17;                  // 2 rows, halves
        case 2: return (lane & 1) ? 17 : 0;                 // 2 rows, interleaved
        case 3: return (lane >> 3) * 17;                    // 4 rows, quarters
        case 4: return lane;                                // 32 distinct consecutive
        case 5: return lane < 10 ? 0 : (lane < 21 ? 17 : 34);  // 3 rows contiguous
        case 6: return lane < 24 ? 0 : 17;                  // 2 rows, 24/8
        case 7: return (lane >> 2) * 17;                    // 8 rows, groups of 4
        default: return 0;
    }
}

template <int W>
__global__ void k(int pat, double* out) {
    __shared__ double4 s[1024];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) s[i] = make_double4(i, i + 1, i + 2, i + 3);
    __syncthreads();
    const int lane = threadIdx.x & 31;
    int sl = slot_of(pat, lane);
    double acc = 0;
    const double2* s2 = reinterpret_cast<const double2*>(s);
    const double* s1 = reinterpret_cast<const double*>(s);
#pragma unroll 4
    for (int it = 0; it < ITERS; ++it) {
        if (W == 16) {
            double2 v = s2[sl + (it & 7) * 2];
            acc += v.x + v.y;
        } else {
            double v = s1[sl * 2 + (it & 7) * 4];
            acc += v;
        }
        sl ^= (acc > 1e300);  // keep the load in the loop
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

int main() {
    double* o;
    cudaMalloc(&o, 1 << 20);
    for (int p = 0; p < 8; ++p) {
        k<16><<<1, 32>>>(p, o);
        k<8><<<1, 32>>>(p, o);
    }
    cudaDeviceSynchronize();
    printf("done\n");
}
