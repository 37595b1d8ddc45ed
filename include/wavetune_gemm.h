/* wavetune_gemm.h -- C-ABI of the validation GEMM family (lib/libwtgemm.so).
 *
 * The reference validates WaveTune on real kernels behind its
 * MeasurementBackend interface (the interface is
 * proj/src/profiler.h:MeasurementBackend::measure and the kernel family is
 * described by proj/src/kernel_map.h:KernelRegistry).  This library is that
 * family on B200: bf16 GEMMs on tcgen05 tensor cores (CUTLASS sm100
 * collectives), one instantiation per (BM, BN, BK, stages), raster swizzle
 * chosen per launch.  WaveTune's macro = the tile (BM, BN, BK); micro =
 * (stages, swizzle).
 *
 * Layouts: A bf16 [M, K] row-major, B bf16 [N, K] row-major (the nn.Linear
 * weight layout), C bf16 [M, N] row-major, fp32 accumulate, C = A * B^T.
 * Status codes are the WT_* codes of wavetune_c.h.
 */
#ifndef WAVETUNE_GEMM_H
#define WAVETUNE_GEMM_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* number of compiled kernel instantiations */
int wt_gemm_family_size(void);

/* tile and pipeline depth of instantiation `cfg` */
int wt_gemm_config(int cfg, int* bm, int* bn, int* bk, int* stages);

/* C = A * B^T with instantiation `cfg` and raster swizzle `swizzle`
 * (1, 2, 4 or 8) on `stream` (a cudaStream_t; NULL = legacy default). */
int wt_gemm_run(int cfg, int swizzle, int M, int N, int K, const void* A, const void* B, void* C, void* stream);

/* Device time of one launch, averaged over `reps` back-to-back launches
 * after `warmup` untimed ones, on the caller's buffers (blocks). */
int wt_gemm_time(int cfg, int swizzle, int M, int N, int K, const void* A, const void* B, void* C, int warmup,
                 int reps, double* mean_us);

/* Batched measurement: for i < n, time (cfg[i], swizzle[i]) on an
 * M[i] x N[i] x K[i] problem; library-owned operands (uniform [-1, 1) bf16,
 * seeded) sized for the largest problem.  latency_us[i] = mean device time of
 * one launch (us).  This is the MeasurementBackend::measure of the family.
 * Entries whose shape the kernel cannot run get latency -1 (status stays OK). */
int wt_gemm_measure_batch(int n, const int32_t* cfg, const int32_t* swizzle, const int32_t* M, const int32_t* N,
                          const int32_t* K, int warmup, int reps, uint64_t seed, double* latency_us);

/* Fill n bf16 elements at p with uniform [-1, 1) values from `seed`. */
int wt_gemm_fill_uniform(void* p, size_t n, uint64_t seed, void* stream);

#ifdef __cplusplus
}
#endif
#endif
