// wt_tc.cuh -- the validation GEMM family, hand-written for sm_100a
// (the kernels WaveTune's macro/micro configs
// parameterise: macro = tile (BM, BN, BK), micro = pipeline depth x raster
// swizzle).  C[M, N] = A[M, K] * B[N, K]^T, bf16 in, fp32 accumulate in TMEM,
// bf16 out.
//
// One persistent, warp-specialised kernel template:
//   warp 0      TMA producer: one elected lane streams K-major 128-byte
//               swizzled boxes of A and B into a ST-deep shared-memory ring
//               (full / empty mbarrier pairs, expect-tx byte counts);
//   warp 1      MMA issuer: one lane issues tcgen05.mma.kind::f16 (UMMA_K =
//               16) from shared-memory descriptors into a double-buffered
//               TMEM accumulator, tcgen05.commit frees ring slots and
//               signals the epilogue;
//   warp 2      TMEM allocator (tcgen05.alloc / dealloc);
//   warps 2..5  epilogue: tcgen05.ld 32x32b.x32 (warp w owns TMEM lanes
//               32*(w%4)..), fp32 -> bf16, 16-byte global stores; releases
//               the accumulator buffer so tile i's drain overlaps tile i+1's
//               main loop.
// Split-K (runtime): when the tile grid underfills the GPU (decode-sized M
// with few N blocks), each tile's K range is cut into `splits` slices run by
// different CTAs; partial accumulators go to an fp32 workspace and the last
// slice to arrive reduces them in slice order (bitwise deterministic).
// Variants (template parameters):
//   BM = 256       CTA pair (cluster of 2, tcgen05.mma.cta_group::2, UMMA
//                  M = 256): each CTA stages its 128 rows of A and half of
//                  B's BN rows; TMA completions land on the leader's barrier;
//                  commits multicast to both CTAs.
//   SWAP           small-M (decode) tiles, BM in {32, 64}: the weight tile
//                  (BN = 128 rows of B) takes the UMMA M slot and the BM
//                  token rows take UMMA N, so the tensor core runs at M = 128
//                  even when the GEMM's M is tiny; the epilogue writes the
//                  transposed accumulator (lanes = n, columns = m).
//   BK = 128       two 64-element swizzle atoms per stage.
// TMA multicast (runtime, single-CTA tiles): clusters of 2 / 4 CTAs on
// neighbouring n-blocks of one m-block load the shared operand once (each CTA
// 1/mc of its rows, .multicast::cluster to all); commits release ring slots
// in every CTA of the cluster, a producer tail drains them before exit.
// Tile order: persistent CTAs (clusters) stride the tile list; tile index ->
// (m block, n block) goes through a raster swizzle of `swizzle` m-blocks per
// group (L2 reuse of B across neighbouring CTAs), a runtime knob.
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace wtb::tc {

struct Params {
    int M, N, K;
    __nv_bfloat16* C;
    int m_blocks, n_blocks, k_blocks, tiles, swizzle;
    // split-K (splits > 1): work unit = (tile, K slice); fp32 partial tiles in
    // `ws` [unit][CTA of the pair][128 lanes][UN]; the last slice of a tile to
    // finish (arrival counter cnt[tile][CTA], self-resetting) sums the slices
    // in slice order -- deterministic -- and writes C
    int splits;
    float* ws;
    int* cnt;
    long long* trace;  // debug (WT_GEMM_TRACE): CTA 0's per-k-block clocks, else null
    // TMA multicast (single-CTA tiles): clusters of `mc` CTAs take `mc`
    // consecutive n-blocks of one m-block; the operand they share (A, or the
    // activations of a swap-AB tile) is loaded once per cluster, each CTA
    // fetching 1/mc of its rows and multicasting them to all; tiles counts
    // cluster tiles (m_blocks x n_groups)
    int mc, n_groups;
    int nomma;  // debug (WT_GEMM_NOMMA): stream operands without issuing MMAs (timing experiments)
};

// ------------------------------------------------------------------ PTX
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
// the suspend-time hint parks the waiting thread in hardware until the
// phase completes (no spin loop competing for issue slots)
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(bar),
        "r"(parity), "r"(0x989680u)
        : "memory");
}
// arrive on the barrier at the same offset in CTA `rank` of the cluster
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t bar, uint32_t rank) {
    uint32_t remote;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(bar), "r"(rank));
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}

__device__ __forceinline__ void tma_prefetch(const CUtensorMap* m) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(m)) : "memory");
}
// 2-D TMA box load; completion (bytes) on `bar`.  PAIR: the CTA-pair form
// whose completion lands on the leader CTA's barrier (peer bit cleared).
template <bool PAIR>
__device__ __forceinline__ void tma_load(const CUtensorMap* m, uint32_t dst, uint32_t bar, int x, int y) {
    if constexpr (PAIR) {
        asm volatile(
            "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%3, %4}], [%2];" ::"r"(dst),
            "l"(reinterpret_cast<uint64_t>(m)), "r"(bar & 0xFEFFFFFFu), "r"(x), "r"(y)
            : "memory");
    } else {
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%3, %4}], [%2];" ::"r"(dst),
            "l"(reinterpret_cast<uint64_t>(m)), "r"(bar), "r"(x), "r"(y)
            : "memory");
    }
}

// multicast form: the box lands at the same offset in every CTA of `mask`,
// completing bytes on the barrier at `bar`'s offset in each of them
__device__ __forceinline__ void tma_load_mc(const CUtensorMap* m, uint32_t dst, uint32_t bar, int x, int y,
                                            uint16_t mask) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
        " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(m)), "r"(bar), "r"(x), "r"(y), "h"(mask)
        : "memory");
}

__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

template <int CG>
__device__ __forceinline__ void tmem_alloc(uint32_t dst_smem, uint32_t cols) {
    if constexpr (CG == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(dst_smem), "r"(cols)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    } else {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(dst_smem), "r"(cols)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    }
}
template <int CG>
__device__ __forceinline__ void tmem_free(uint32_t addr, uint32_t cols) {
    if constexpr (CG == 1)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(addr), "r"(cols) : "memory");
    else
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(addr), "r"(cols) : "memory");
}

// D[tmem] (+)= A[smem] * B[smem]^T, both K-major
template <int CG>
__device__ __forceinline__ void umma(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    if constexpr (CG == 1)
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
            "l"(a), "l"(b), "r"(idesc), "r"(acc)
            : "memory");
    else
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
            "l"(a), "l"(b), "r"(idesc), "r"(acc)
            : "memory");
}
// completion of every prior MMA of this thread -> one arrive on `bar`
// (CTA pair: on the barrier at that offset in both CTAs; mask != 0: in every
// CTA of the multicast cluster)
template <int CG>
__device__ __forceinline__ void umma_commit(uint32_t bar, uint16_t mask = 0) {
    if constexpr (CG == 1) {
        if (mask)
            asm volatile(
                "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::
                    "r"(bar),
                "h"(mask)
                : "memory");
        else
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
                         : "memory");
    }
    else
        asm volatile(
            "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                bar),
            "h"(uint16_t(3))
            : "memory");
}

// 32 consecutive fp32 columns of this thread's TMEM lane
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
        "%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
          "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
          "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// Shared-memory matrix descriptor of a K-major, 128-byte-swizzled operand:
// rows of 128 bytes, 8-row core groups 1024 bytes apart (SBO), start address
// advanced by 32 bytes per UMMA_K step inside the swizzle atom; version 1
// (sm_100), layout type 2 = SWIZZLE_128B.
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr) {
    return uint64_t((saddr & 0x3FFFFu) >> 4) | (uint64_t(1) << 16) | (uint64_t(1024 >> 4) << 32) |
           (uint64_t(1) << 46) | (uint64_t(2) << 61);
}

// Instruction descriptor, kind::f16: D fp32, A/B bf16, both K-major.
__host__ __device__ constexpr uint32_t idesc_bf16(int um, int un) {
    return (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(un >> 3) << 17) | (uint32_t(um >> 4) << 24);
}

__device__ __forceinline__ uint32_t pack_bf16(uint32_t lo, uint32_t hi) {
    const __nv_bfloat162 h = __floats2bfloat162_rn(__uint_as_float(lo), __uint_as_float(hi));
    return *reinterpret_cast<const uint32_t*>(&h);
}

// cluster tile index -> (m block, n block of multicast rank `crank`):
// groups of `sw` m-blocks walk the n groups
__device__ __forceinline__ void raster(int t, const Params& p, int crank, int* mb, int* nb) {
    const int sw = p.swizzle;
    const int per = sw * p.n_groups;
    const int g = t / per, r = t - g * per;
    const int m0 = g * sw;
    const int gw = min(sw, p.m_blocks - m0);
    *mb = m0 + r % gw;
    *nb = (r / gw) * p.mc + crank;
}

template <int BM, int BN, int BK, int ST, bool SWAP>
struct Shape {
    static constexpr int CG = (BM == 256) ? 2 : 1;   // CTAs per MMA (cluster size)
    static constexpr int UM = SWAP ? BN : BM;        // UMMA M (per pair when CG = 2)
    static constexpr int UN = SWAP ? BM : BN;        // UMMA N
    static constexpr int A_ROWS = UM / CG;           // rows of the M-slot operand staged per CTA
    static constexpr int B_ROWS = UN / CG;           // rows of the N-slot operand staged per CTA
    static constexpr int ATOMS = BK / 64;            // 128-byte swizzle atoms per stage
    static constexpr int A_BYTES = A_ROWS * BK * 2;
    static constexpr int B_BYTES = B_ROWS * BK * 2;
    static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
    static constexpr int TMEM_COLS = (2 * UN <= 32) ? 32 : (2 * UN <= 64) ? 64 : (2 * UN <= 128) ? 128
                                     : (2 * UN <= 256) ? 256 : 512;
    static constexpr int BAR_BYTES = 1024;
    static constexpr int SMEM = 1024 /* alignment slack */ + ST * STAGE_BYTES + BAR_BYTES;
    static constexpr int THREADS = 192;
    static_assert(UM == 128 || (UM == 256 && CG == 2), "UMMA M");
    static_assert(UN % 16 == 0 && UN >= 16 && UN <= 256, "UMMA N");
    static_assert(BK % 64 == 0, "BK = whole 128-byte swizzle atoms");
    static_assert(!(SWAP && CG == 2), "swap-AB tiles are single-CTA");
    static_assert(B_ROWS % 8 == 0 && (B_BYTES / ATOMS) % 1024 == 0, "swizzle atoms stay 1024-byte aligned");
};

template <int BM, int BN, int BK, int ST, bool SWAP>
__global__ void __launch_bounds__(192, 1)
    k_tc_gemm(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, const Params p) {
    using S = Shape<BM, BN, BK, ST, SWAP>;
    constexpr int CG = S::CG;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* ring = smem;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + ST * S::STAGE_BYTES);
    // bars: full[ST] | empty[ST] | tfull[2] | tempty[2] | tmem address
    const uint32_t full0 = smem_u32(bars), empty0 = full0 + 8 * ST, tfull0 = empty0 + 8 * ST, tempty0 = tfull0 + 16;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * ST + 4);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int mc = CG == 1 ? p.mc : 1;
    const bool clustered = CG == 2 || mc > 1;
    const uint32_t rank = CG == 2 ? cluster_rank() : 0u;           // CTA of the pair
    const int crank = (CG == 1 && mc > 1) ? int(cluster_rank()) : 0;  // CTA of the multicast cluster
    const bool leader = rank == 0;
    const uint16_t mc_mask = mc > 1 ? uint16_t((1u << mc) - 1u) : uint16_t(0);

    if (warp == 0 && lane == 0) {
        tma_prefetch(&tmA);
        tma_prefetch(&tmB);
    }
    if (warp == 1 && lane == 0) {
        for (int s = 0; s < ST; ++s) {
            mbar_init(full0 + 8 * s, 1);
            mbar_init(empty0 + 8 * s, uint32_t(mc));  // every consumer of the cluster frees the slot
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(tfull0 + 8 * s, 1);
            mbar_init(tempty0 + 8 * s, 4 * CG);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 2) tmem_alloc<CG>(smem_u32(tmem_slot), S::TMEM_COLS);
    tc_fence_before();
    if (clustered)
        cluster_sync();
    else
        __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    const int nclusters = gridDim.x / (CG * mc);
    const int cid = blockIdx.x / (CG * mc);

    if (warp == 0) {
        // ===== TMA producer
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            for (int u = cid; u < p.tiles * p.splits; u += nclusters) {
                const int t = u / p.splits, sl = u - t * p.splits;
                int mb, nb;
                raster(t, p, crank, &mb, &nb);
                const int kb0 = int((long long)sl * p.k_blocks / p.splits);
                const int kb1 = int((long long)(sl + 1) * p.k_blocks / p.splits);
                // M-slot operand rows / N-slot operand rows of this CTA
                const int ra = SWAP ? nb * BN : mb * BM + int(rank) * S::A_ROWS;
                const int rb = SWAP ? mb * BM : nb * BN + int(rank) * S::B_ROWS;
                const CUtensorMap* ta = SWAP ? &tmB : &tmA;
                const CUtensorMap* tb = SWAP ? &tmA : &tmB;
                for (int kb = kb0; kb < kb1; ++kb) {
                    mbar_wait(empty0 + 8 * stage, phase ^ 1u);
                    if (p.trace && blockIdx.x == 0 && u == cid && kb - kb0 < 512) p.trace[kb - kb0] = clock64();
                    const uint32_t fb = full0 + 8 * stage;
                    if (leader) mbar_expect_tx(fb, uint32_t(S::STAGE_BYTES * CG));
                    const uint32_t sa = smem_u32(ring + stage * S::STAGE_BYTES);
                    const uint32_t sb = sa + S::A_BYTES;
#pragma unroll
                    for (int j = 0; j < S::ATOMS; ++j) {
                        const int k0 = kb * BK + 64 * j;
                        if (mc > 1) {
                            // the m-block's operand: this CTA's 1/mc of its rows, to every CTA
                            if constexpr (!SWAP) {
                                const int sr = S::A_ROWS / mc;
                                tma_load_mc(ta, sa + j * (S::A_ROWS * 128) + crank * sr * 128, fb, k0,
                                            ra + crank * sr, mc_mask);
                                tma_load<false>(tb, sb + j * (S::B_ROWS * 128), fb, k0, rb);
                            } else {
                                const int sr = S::B_ROWS / mc;
                                tma_load<false>(ta, sa + j * (S::A_ROWS * 128), fb, k0, ra);
                                tma_load_mc(tb, sb + j * (S::B_ROWS * 128) + crank * sr * 128, fb, k0,
                                            rb + crank * sr, mc_mask);
                            }
                        } else {
                            tma_load<CG == 2>(ta, sa + j * (S::A_ROWS * 128), fb, k0, ra);
                            tma_load<CG == 2>(tb, sb + j * (S::B_ROWS * 128), fb, k0, rb);
                        }
                    }
                    if (++stage == ST) {
                        stage = 0;
                        phase ^= 1u;
                    }
                }
            }
            // producer tail: every slot released by every consumer of the
            // cluster before this CTA may exit (peers' commits target our barriers)
            for (int i = 0; i < ST; ++i) {
                mbar_wait(empty0 + 8 * stage, phase ^ 1u);
                if (++stage == ST) {
                    stage = 0;
                    phase ^= 1u;
                }
            }
        }
    } else if (warp == 1) {
        // ===== MMA issuer (leader CTA of the pair)
        if (leader && lane == 0) {
            constexpr uint32_t idesc = idesc_bf16(S::UM, S::UN);
            int stage = 0;
            uint32_t phase = 0;
            int it = 0;
            for (int u = cid; u < p.tiles * p.splits; u += nclusters, ++it) {
                const int sl = u % p.splits;
                const int kb0 = int((long long)sl * p.k_blocks / p.splits);
                const int kb1 = int((long long)(sl + 1) * p.k_blocks / p.splits);
                const int acc = it & 1;
                const uint32_t aph = uint32_t(it >> 1) & 1u;
                mbar_wait(tempty0 + 8 * acc, aph ^ 1u);
                tc_fence_after();
                const uint32_t d = tmem + uint32_t(acc * S::UN);
                for (int kb = kb0; kb < kb1; ++kb) {
                    mbar_wait(full0 + 8 * stage, phase);
                    if (p.trace && blockIdx.x == 0 && u == cid && kb - kb0 < 512) p.trace[512 + kb - kb0] = clock64();
                    tc_fence_after();
                    const uint32_t sa = smem_u32(ring + stage * S::STAGE_BYTES);
                    const uint32_t sb = sa + S::A_BYTES;
#pragma unroll
                    for (int k = 0; k < BK / 16; ++k) {
                        const int j = k >> 2, kk = k & 3;
                        const uint64_t ad = sdesc(sa + j * (S::A_ROWS * 128) + kk * 32);
                        const uint64_t bd = sdesc(sb + j * (S::B_ROWS * 128) + kk * 32);
                        if (!p.nomma) umma<CG>(d, ad, bd, idesc, ((kb - kb0) | k) != 0);
                    }
                    umma_commit<CG>(empty0 + 8 * stage, mc_mask);
                    if (++stage == ST) {
                        stage = 0;
                        phase ^= 1u;
                    }
                }
                umma_commit<CG>(tfull0 + 8 * acc);
            }
        }
    } else {
        // ===== epilogue (warps 2..5): warp w drains TMEM lanes 32*(w%4)..
        const int q = warp & 3;
        const int row = 32 * q + lane;  // TMEM lane
        __shared__ int last_flag;
        // 32 accumulator columns [c, c+32) of this lane -> C
        auto store = [&](const float (&f)[32], int mb, int nb, int c) {
            if constexpr (!SWAP) {
                const int m = mb * BM + int(rank) * 128 + row;
                const int n0 = nb * BN + c;
                if (m < p.M && n0 < p.N) {
                    __nv_bfloat16* dst = p.C + size_t(m) * p.N + n0;
#pragma unroll
                    for (int g = 0; g < 4; ++g) {
                        if (n0 + 8 * g < p.N) {
                            uint4 w;
                            w.x = pack_bf16(__float_as_uint(f[8 * g + 0]), __float_as_uint(f[8 * g + 1]));
                            w.y = pack_bf16(__float_as_uint(f[8 * g + 2]), __float_as_uint(f[8 * g + 3]));
                            w.z = pack_bf16(__float_as_uint(f[8 * g + 4]), __float_as_uint(f[8 * g + 5]));
                            w.w = pack_bf16(__float_as_uint(f[8 * g + 6]), __float_as_uint(f[8 * g + 7]));
                            *reinterpret_cast<uint4*>(dst + 8 * g) = w;
                        }
                    }
                }
            } else {
                // accumulator = C^T tile: lane = n, column = m
                const int n = nb * BN + row;
                const int m0 = mb * BM + c;
                if (n < p.N) {
#pragma unroll
                    for (int j = 0; j < 32; ++j)
                        if (m0 + j < p.M) p.C[size_t(m0 + j) * p.N + n] = __float2bfloat16_rn(f[j]);
                }
            }
        };
        int it = 0;
        for (int u = cid; u < p.tiles * p.splits; u += nclusters, ++it) {
            const int t = u / p.splits;
            int mb, nb;
            raster(t, p, crank, &mb, &nb);
            const int acc = it & 1;
            mbar_wait(tfull0 + 8 * acc, uint32_t(it >> 1) & 1u);
            tc_fence_after();
            const uint32_t tbase = tmem + (uint32_t(32 * q) << 16) + uint32_t(acc * S::UN);
            if (p.splits == 1) {
#pragma unroll 1
                for (int c = 0; c < S::UN; c += 32) {
                    uint32_t v[32];
                    tmem_ld32(tbase + uint32_t(c), v);
                    float f[32];
#pragma unroll
                    for (int j = 0; j < 32; ++j) f[j] = __uint_as_float(v[j]);
                    store(f, mb, nb, c);
                }
            } else {
                float* mine = p.ws + (((size_t(u) * mc + crank) * CG + rank) * 128 + row) * S::UN;
#pragma unroll 1
                for (int c = 0; c < S::UN; c += 32) {
                    uint32_t v[32];
                    tmem_ld32(tbase + uint32_t(c), v);
#pragma unroll
                    for (int g = 0; g < 8; ++g)
                        __stcg(reinterpret_cast<uint4*>(mine + c) + g,
                               make_uint4(v[4 * g], v[4 * g + 1], v[4 * g + 2], v[4 * g + 3]));
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) {
                if constexpr (CG == 2)
                    mbar_arrive_cluster(tempty0 + 8 * acc, 0);
                else
                    mbar_arrive(tempty0 + 8 * acc);
            }
            if (p.splits > 1) {
                __threadfence();
                asm volatile("bar.sync 1, 128;" ::: "memory");
                int* ctr = p.cnt + (size_t(t) * mc + crank) * CG + rank;
                if (threadIdx.x == 64) last_flag = atomicAdd(ctr, 1) == p.splits - 1;
                asm volatile("bar.sync 1, 128;" ::: "memory");
                if (last_flag) {
                    __threadfence();
                    const size_t u0 = size_t(t) * p.splits;
#pragma unroll 1
                    for (int c = 0; c < S::UN; c += 32) {
                        float f[32];
#pragma unroll 1
                        for (int sl = 0; sl < p.splits; ++sl) {
                            const float4* src = reinterpret_cast<const float4*>(
                                p.ws + ((((u0 + sl) * mc + crank) * CG + rank) * 128 + row) * S::UN + c);
#pragma unroll
                            for (int g = 0; g < 8; ++g) {
                                const float4 x = __ldcg(src + g);
                                if (sl == 0) {
                                    f[4 * g] = x.x, f[4 * g + 1] = x.y, f[4 * g + 2] = x.z, f[4 * g + 3] = x.w;
                                } else {
                                    f[4 * g] += x.x, f[4 * g + 1] += x.y, f[4 * g + 2] += x.z, f[4 * g + 3] += x.w;
                                }
                            }
                        }
                        store(f, mb, nb, c);
                    }
                    if (threadIdx.x == 64) *ctr = 0;  // ready for the next launch
                }
                asm volatile("bar.sync 1, 128;" ::: "memory");
            }
        }
    }

    tc_fence_before();
    if (clustered)
        cluster_sync();
    else
        __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        tmem_free<CG>(tmem, S::TMEM_COLS);
    }
}

}  // namespace wtb::tc
