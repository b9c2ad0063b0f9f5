// gemm_tc.cu -- K5: the decode contraction on the 5th-generation tensor cores.
//
//   acc[m][n] = sum_j A[m][j] B[n][j]     (A: [M][K], B: [N][K], 16-bit, K-major)
//
// With the tables of tables.cu, row m = (class c, band row i), column n = grid
// column, acc = D q_c (Eq. 11 after Eq. 10 normalisation).
// The VSA epilogue applies the Born rule p = q^2, clamped to
// [0, 1] against rounding, and the per-cell binary entropy H_b(p) that Alg. 2
// averages; it writes H_b for every decoded row (band +
// halo) and q for the band's own rows.
//
// Two tcgen05 kernels, both persistent with warp-specialised roles:
//
// k_decode_gemm2 (default): CTA pairs (cluster 2x1, cta_group::2), UMMA
//   M = 256 (128 rows per CTA) x N = BN (BN/2 rows of B per CTA) x K = 16.
//   Each CTA's TMA producer loads its own A rows and its half of B into a
//   6-stage ring and counts the bytes on CTA 0's barrier; CTA 0's single MMA
//   thread issues for the pair and commits (multicast) to both CTAs' "slot
//   free" and "accumulator ready" barriers; each CTA's 4 epilogue warps drain
//   its own TMEM half (double-buffered accumulator) and signal CTA 0.  Half the
//   B bytes per SM relative to the 1-CTA tile (L2 -> SM traffic is the limit).
//   BN is chosen per problem from {256, 224, 192, 160, 128} to minimise
//   waves x BN on the 74 SM pairs.
// k_decode_gemm (1-CTA, M=128 x N=256): the first version, kept as a
//   measured comparison point (VSAOGM_GEMM=1cta) and for the test hook.
#include <cudaTypedefs.h>

#include <stdlib.h>
#include <string.h>

#include "common.cuh"

namespace {

constexpr int GEMM_THREADS = 192;
constexpr uint32_t A_TILE_BYTES = VSA_BM * VSA_BK * 2;   // 16 KB
constexpr uint32_t B_TILE_BYTES = VSA_BN * VSA_BK * 2;   // 32 KB
constexpr uint32_t STAGE_BYTES = A_TILE_BYTES + B_TILE_BYTES;
constexpr uint32_t TMEM_COLS = 512;                       // double-buffered fp32 accumulator
constexpr size_t GEMM_SMEM = 1024 + (size_t)VSA_STAGES * STAGE_BYTES + 256;
constexpr int STAGES2 = 6;                                // 2-CTA ring depth (32 KB / stage at BN=256)

struct Epi {
    float *C;          // raw mode output [M][N]
    float inv_scale;   // VSA mode: q = acc * inv_scale
    float *hb;         // VSA mode: [M][ldh], ldh = N rounded up to 8
    float *q;          // VSA mode: [2][band_rows][N] or null
    int r_ext, band_off, band_rows, ldh;
    float *ws;         // split-K workspace [splits][M][N] fp32
    int splits, kb_per;
};

__device__ __forceinline__ float hb_of_p(float p)
{
    // binary entropy in bits, 0 log 0 = 0; log1p keeps (1-p) log(1-p) accurate for small p
    float h = 0.f;
    if (p > 0.f) h = -p * log2f(p);
    if (p < 1.f) h -= (1.f - p) * log1pf(-p) * 1.44269504088896341f;
    return h;
}

// One thread's 32 consecutive accumulator columns of row m, starting at column n0.
template <int MODE>
__device__ __forceinline__ void epilogue_chunk(const uint32_t (&v)[32], int m, int n0, int M, int N, const Epi &epi)
{
    if (m >= M || n0 >= N) return;
    const bool full_chunk = (n0 + 32 <= N) && ((N & 3) == 0);
    if (MODE == 0) {
        float *dst = epi.C + (size_t)m * N + n0;
        if (full_chunk) {
#pragma unroll
            for (int j = 0; j < 32; j += 4)
                *reinterpret_cast<float4 *>(dst + j) = make_float4(__uint_as_float(v[j]), __uint_as_float(v[j + 1]),
                                                                   __uint_as_float(v[j + 2]), __uint_as_float(v[j + 3]));
        } else {
#pragma unroll
            for (int j = 0; j < 32; ++j)
                if (n0 + j < N) dst[j] = __uint_as_float(v[j]);
        }
        return;
    }
    const int cls = m / epi.r_ext;
    const int i = m - cls * epi.r_ext;
    const bool q_row = epi.q && i >= epi.band_off && i < epi.band_off + epi.band_rows;
    float qv[32], hv[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) {
        qv[j] = __uint_as_float(v[j]) * epi.inv_scale;
        hv[j] = hb_of_p(fminf(qv[j] * qv[j], 1.f));
    }
    float *hdst = epi.hb + (size_t)m * epi.ldh + n0;
    if (n0 + 32 <= N) {
#pragma unroll
        for (int j = 0; j < 32; j += 4)
            *reinterpret_cast<float4 *>(hdst + j) = make_float4(hv[j], hv[j + 1], hv[j + 2], hv[j + 3]);
    } else {
#pragma unroll
        for (int j = 0; j < 32; ++j)
            if (n0 + j < N) hdst[j] = hv[j];
    }
    if (q_row) {
        float *qdst = epi.q + ((size_t)cls * epi.band_rows + (i - epi.band_off)) * N + n0;
        if (full_chunk) {
#pragma unroll
            for (int j = 0; j < 32; j += 4)
                *reinterpret_cast<float4 *>(qdst + j) = make_float4(qv[j], qv[j + 1], qv[j + 2], qv[j + 3]);
        } else {
#pragma unroll
            for (int j = 0; j < 32; ++j)
                if (n0 + j < N) qdst[j] = qv[j];
        }
    }
}

// ------------------------------------------------------------------ 1-CTA kernel
template <int MODE>   // 0 = raw fp32 store (test hook), 1 = VSA epilogue
__global__ void __launch_bounds__(GEMM_THREADS, 1)
    k_decode_gemm(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, int M, int N,
                  int K, uint32_t idesc, Epi epi)
{
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw_addr = smem_u32(smem_raw);
    uint8_t *smem = smem_raw + ((1024 - (raw_addr & 1023)) & 1023);
    uint8_t *sA = smem;
    uint8_t *sB = smem + VSA_STAGES * A_TILE_BYTES;
    uint64_t *bars = reinterpret_cast<uint64_t *>(sB + VSA_STAGES * B_TILE_BYTES);
    uint64_t *full = bars;
    uint64_t *empty = bars + VSA_STAGES;
    uint64_t *tfull = bars + 2 * VSA_STAGES;
    uint64_t *tempty = tfull + 2;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tempty + 2);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int num_m = (M + VSA_BM - 1) / VSA_BM;
    const int num_n = (N + VSA_BN - 1) / VSA_BN;
    const int num_tiles = num_m * num_n;
    const int num_kb = K / VSA_BK;

    if (threadIdx.x == 0) {
        for (int s = 0; s < VSA_STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(&tfull[s], 1);
            mbar_init(&tempty[s], 128);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(TMEM_COLS)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {
            asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
            asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
            uint32_t stage = 0, phase = 0;
            for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
                const int mb = tile % num_m, nb = tile / num_m;
                for (int kb = 0; kb < num_kb; ++kb) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    mbar_expect_tx(&full[stage], STAGE_BYTES);
                    tma_load_2d(sA + stage * A_TILE_BYTES, &tmA, &full[stage], kb * VSA_BK, mb * VSA_BM);
                    tma_load_2d(sB + stage * B_TILE_BYTES, &tmB, &full[stage], kb * VSA_BK, nb * VSA_BN);
                    if (++stage == VSA_STAGES) { stage = 0; phase ^= 1; }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            uint32_t stage = 0, phase = 0, as = 0, aphase = 0;
            for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
                mbar_wait(&tempty[as], aphase ^ 1);
                tc_fence_after();
                const uint32_t d = tmem_base + as * VSA_BN;
                for (int kb = 0; kb < num_kb; ++kb) {
                    mbar_wait(&full[stage], phase);
                    tc_fence_after();
                    const uint32_t a0 = smem_u32(sA + stage * A_TILE_BYTES);
                    const uint32_t b0 = smem_u32(sB + stage * B_TILE_BYTES);
#pragma unroll
                    for (int k = 0; k < VSA_BK / 16; ++k)
                        tc_mma_f16(d, sw128_kmajor_desc(a0 + 32 * k), sw128_kmajor_desc(b0 + 32 * k), idesc,
                                   (kb | k) != 0);
                    tc_commit(&empty[stage]);   // frees the smem slot once these MMAs complete
                    if (++stage == VSA_STAGES) { stage = 0; phase ^= 1; }
                }
                tc_commit(&tfull[as]);          // accumulator ready for the epilogue
                if (++as == 2) { as = 0; aphase ^= 1; }
            }
        }
    } else {
        // epilogue warps 2..5: warp w may access TMEM lanes [32 (w%4), 32 (w%4) + 32)
        const int quarter = warp & 3;
        const int row_in_tile = quarter * 32 + lane;
        uint32_t as = 0, aphase = 0;
        for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
            const int mb = tile % num_m, nb = tile / num_m;
            mbar_wait(&tfull[as], aphase);
            tc_fence_after();
            const int m = mb * VSA_BM + row_in_tile;
#pragma unroll 1
            for (int cc = 0; cc < VSA_BN / 32; ++cc) {
                uint32_t v[32];
                const uint32_t taddr = tmem_base + ((uint32_t)(quarter * 32) << 16) + as * VSA_BN + cc * 32;
                TMEM_LD_32x32b_X32(taddr, v);
                tmem_ld_wait();
                epilogue_chunk<MODE>(v, m, nb * VSA_BN + cc * 32, M, N, epi);
            }
            tc_fence_before();
            mbar_arrive(&tempty[as]);
            if (++as == 2) { as = 0; aphase ^= 1; }
        }
    }

    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(TMEM_COLS)
                     : "memory");
    }
}

// ------------------------------------------------------------------ 2-CTA kernel
template <int MODE, int BN>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(GEMM_THREADS, 1)
    k_decode_gemm2(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, int M, int N,
                   int K, uint32_t idesc, Epi epi)
{
    constexpr uint32_t A_BYTES = 128 * VSA_BK * 2;          // this CTA's 128 rows of A
    constexpr uint32_t BH_BYTES = (BN / 2) * VSA_BK * 2;    // this CTA's half of B
    constexpr uint32_t ST_BYTES = A_BYTES + BH_BYTES;
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw_addr = smem_u32(smem_raw);
    uint8_t *smem = smem_raw + ((1024 - (raw_addr & 1023)) & 1023);
    uint8_t *sA = smem;
    uint8_t *sB = smem + STAGES2 * A_BYTES;
    uint64_t *bars = reinterpret_cast<uint64_t *>(sB + STAGES2 * BH_BYTES);
    uint64_t *full = bars;                  // used in CTA 0: TMA bytes of both CTAs
    uint64_t *empty = bars + STAGES2;       // both CTAs: slot free (multicast commit)
    uint64_t *tfull = bars + 2 * STAGES2;   // both CTAs: accumulator ready (multicast commit)
    uint64_t *tempty = tfull + 2;           // used in CTA 0: 8 epilogue warps of the pair
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tempty + 2);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const uint32_t rank = cluster_ctarank();
    const int pair = blockIdx.x >> 1, num_pairs = gridDim.x >> 1;
    const int num_m = (M + 255) / 256;
    const int num_n = (N + BN - 1) / BN;
    const int num_tiles = num_m * num_n;
    const int num_kb = K / VSA_BK;
    const int S = epi.splits;                 // split-K factor (1 = none)

    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES2; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(&tfull[s], 1);
            mbar_init(&tempty[s], 8);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(TMEM_COLS)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    cluster_sync_all();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {
            asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
            asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
            uint32_t stage = 0, phase = 0;
            for (int u = pair; u < num_tiles * S; u += num_pairs) {
                const int tile = u / S, sk = u - tile * S;
                const int nb = tile % num_n, mb = tile / num_n;   // n-fastest: a wave reads A once
                const int arow = mb * 256 + (int)rank * 128;
                const int brow = nb * BN + (int)rank * (BN / 2);
                const int kb0 = sk * epi.kb_per, kb1 = min(num_kb, kb0 + epi.kb_per);
                for (int kb = kb0; kb < kb1; ++kb) {
                    mbar_wait_cluster(&empty[stage], phase ^ 1);
                    if (rank == 0) mbar_expect_tx(&full[stage], 2 * ST_BYTES);
                    tma_load_2d_2sm(sA + stage * A_BYTES, &tmA, &full[stage], kb * VSA_BK, arow);
                    tma_load_2d_2sm(sB + stage * BH_BYTES, &tmB, &full[stage], kb * VSA_BK, brow);
                    if (++stage == STAGES2) { stage = 0; phase ^= 1; }
                }
            }
        }
    } else if (warp == 1) {
        if (rank == 0 && lane == 0) {
            uint32_t stage = 0, phase = 0, as = 0, aphase = 0;
            for (int u = pair; u < num_tiles * S; u += num_pairs) {
                const int sk = u % S;
                const int kb0 = sk * epi.kb_per, kb1 = min(num_kb, kb0 + epi.kb_per);
                mbar_wait_cluster(&tempty[as], aphase ^ 1);
                tc_fence_after();
                const uint32_t d = tmem_base + as * 256;
                for (int kb = kb0; kb < kb1; ++kb) {
                    mbar_wait(&full[stage], phase);
                    tc_fence_after();
                    const uint32_t a0 = smem_u32(sA + stage * A_BYTES);
                    const uint32_t b0 = smem_u32(sB + stage * BH_BYTES);
#pragma unroll
                    for (int k = 0; k < VSA_BK / 16; ++k)
                        tc_mma2_f16(d, sw128_kmajor_desc(a0 + 32 * k), sw128_kmajor_desc(b0 + 32 * k), idesc,
                                    (kb != kb0) || (k != 0));
                    tc_commit2_mc(&empty[stage]);
                    if (++stage == STAGES2) { stage = 0; phase ^= 1; }
                }
                tc_commit2_mc(&tfull[as]);
                if (++as == 2) { as = 0; aphase ^= 1; }
            }
        }
    } else {
        const int quarter = warp & 3;
        const int row_in_tile = (int)rank * 128 + quarter * 32 + lane;
        uint32_t as = 0, aphase = 0;
        Epi part = epi;                       // split-K: raw fp32 partial sums to the workspace
        for (int u = pair; u < num_tiles * S; u += num_pairs) {
            const int tile = u / S, sk = u - tile * S;
            const int nb = tile % num_n, mb = tile / num_n;
            mbar_wait_cluster(&tfull[as], aphase);
            tc_fence_after();
            const int m = mb * 256 + row_in_tile;
            part.C = epi.ws + (size_t)sk * M * N;
#pragma unroll 1
            for (int cc = 0; cc < BN / 32; ++cc) {
                uint32_t v[32];
                const uint32_t taddr = tmem_base + ((uint32_t)(quarter * 32) << 16) + as * 256 + cc * 32;
                TMEM_LD_32x32b_X32(taddr, v);
                tmem_ld_wait();
                if (S == 1) epilogue_chunk<MODE>(v, m, nb * BN + cc * 32, M, N, epi);
                else epilogue_chunk<0>(v, m, nb * BN + cc * 32, M, N, part);
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_cluster(&tempty[as], 0);
            if (++as == 2) { as = 0; aphase ^= 1; }
        }
    }

    tc_fence_before();
    cluster_sync_all();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(TMEM_COLS)
                     : "memory");
    }
}

// split-K: sum the partial accumulators in split order (deterministic), then the epilogue
template <int MODE>
__global__ void __launch_bounds__(256) k_splitk_reduce(int M, int N, Epi epi)
{
    const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    const size_t MN = (size_t)M * N;
    if (idx >= MN) return;
    float acc = 0.f;
    for (int s = 0; s < epi.splits; ++s) acc += epi.ws[(size_t)s * MN + idx];
    if (MODE == 0) {
        epi.C[idx] = acc;
        return;
    }
    const int m = (int)(idx / N), n = (int)(idx - (size_t)m * N);
    const float q = acc * epi.inv_scale;
    epi.hb[(size_t)m * epi.ldh + n] = hb_of_p(fminf(q * q, 1.f));
    const int cls = m / epi.r_ext, i = m - cls * epi.r_ext;
    if (epi.q && i >= epi.band_off && i < epi.band_off + epi.band_rows)
        epi.q[((size_t)cls * epi.band_rows + (i - epi.band_off)) * N + n] = q;
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn()
{
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    return fn;
}

// 2-D K-major tensor map: dims {K, rows}, box {64, box_rows}, 128-byte swizzle,
// out-of-bounds rows are zero-filled (so M, N need no padding).
int make_map(CUtensorMap *map, const void *ptr, int rows, int K, int box_rows, int prec)
{
    auto fn = encode_fn();
    if (!fn) return VSAOGM_ECUDA;
    cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)K * 2};
    cuuint32_t box[2] = {VSA_BK, (cuuint32_t)box_rows};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = fn(map, prec == VSAOGM_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2,
                    const_cast<void *>(ptr), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? VSAOGM_OK : VSAOGM_ECUDA;
}

template <int MODE>
int launch1(const void *A, const void *B, int M, int N, int K, int prec, const Epi &epi, cudaStream_t s, int num_sms)
{
    CUtensorMap ta, tb;
    int rc = make_map(&ta, A, M, K, VSA_BM, prec);
    if (rc) return rc;
    rc = make_map(&tb, B, N, K, VSA_BN, prec);
    if (rc) return rc;
    VSA_CUDA_TRY(cudaFuncSetAttribute(k_decode_gemm<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)GEMM_SMEM));
    const int tiles = ((M + VSA_BM - 1) / VSA_BM) * ((N + VSA_BN - 1) / VSA_BN);
    const int grid = tiles < num_sms ? tiles : num_sms;
    const uint32_t idesc = make_idesc_f16(prec == VSAOGM_BF16, VSA_BM, VSA_BN);
    k_decode_gemm<MODE><<<grid, GEMM_THREADS, GEMM_SMEM, s>>>(ta, tb, M, N, K, idesc, epi);
    VSA_CUDA_TRY(cudaGetLastError());
    return VSAOGM_OK;
}

template <int MODE, int BN>
int launch2_bn(const void *A, const void *B, int M, int N, int K, int prec, Epi epi, cudaStream_t s, int num_sms)
{
    CUtensorMap ta, tb;
    int rc = make_map(&ta, A, M, K, 128, prec);
    if (rc) return rc;
    rc = make_map(&tb, B, N, K, BN / 2, prec);
    if (rc) return rc;
    const size_t smem = 1024 + (size_t)STAGES2 * (128 + BN / 2) * VSA_BK * 2 + 256;
    VSA_CUDA_TRY(cudaFuncSetAttribute(k_decode_gemm2<MODE, BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const int units = ((M + 255) / 256) * ((N + BN - 1) / BN) * epi.splits;
    const int pairs = num_sms / 2;
    const int grid = 2 * (units < pairs ? units : pairs);
    const uint32_t idesc = make_idesc_f16(prec == VSAOGM_BF16, 256, BN);
    k_decode_gemm2<MODE, BN><<<grid, GEMM_THREADS, smem, s>>>(ta, tb, M, N, K, idesc, epi);
    VSA_CUDA_TRY(cudaGetLastError());
    if (epi.splits > 1) {
        const size_t MN = (size_t)M * N;
        k_splitk_reduce<MODE><<<(unsigned)((MN + 255) / 256), 256, 0, s>>>(M, N, epi);
        VSA_CUDA_TRY(cudaGetLastError());
    }
    return VSAOGM_OK;
}

// BN minimising (waves x BN): the MMA time of a tile is proportional to BN.
int pick_bn(int M, int N, int num_sms)
{
    static const int cands[] = {256, 224, 192, 160, 128};
    const int pairs = num_sms / 2;
    const int num_m = (M + 255) / 256;
    int best = 256;
    long best_cost = -1;
    for (int bn : cands) {
        const long tiles = (long)num_m * ((N + bn - 1) / bn);
        const long cost = ((tiles + pairs - 1) / pairs) * bn;
        if (best_cost < 0 || cost < best_cost) { best_cost = cost; best = bn; }
    }
    return best;
}

// Split-K factor for short problems (few tiles for 74 SM pairs, e.g. the row band of one
// rank of 8): model time = waves * tile_time / S + partial-sum traffic, tile_time from the
// measured ~16 TFLOP/s per SM pair, traffic at ~5 TB/s.  S = 1 when the tiles fill the GPU.
int pick_splits(int M, int N, int K, int bn, int num_sms)
{
    const int pairs = num_sms / 2;
    const long tiles = (long)((M + 255) / 256) * ((N + bn - 1) / bn);
    const int num_kb = K / VSA_BK;
    const double t_tile = 2.0 * 256 * bn * (double)K / 16e12 * 1e6;   // us
    double best_t = -1;
    int best = 1;
    for (int S = 1; S <= 16 && S <= num_kb / 4; ++S) {
        const double waves = (double)((tiles * S + pairs - 1) / pairs);
        double t = waves * t_tile / S;
        if (S > 1) t += 2.0 * S * (double)M * N * 4 / 5e12 * 1e6 + 3.0;
        if (best_t < 0 || t < best_t * 0.97) { best_t = t; best = S; }
    }
    return best;
}

template <int MODE>
int launch2(const void *A, const void *B, int M, int N, int K, int prec, const Epi &epi, cudaStream_t s, int num_sms,
            int bn)
{
    switch (bn) {
    case 224: return launch2_bn<MODE, 224>(A, B, M, N, K, prec, epi, s, num_sms);
    case 192: return launch2_bn<MODE, 192>(A, B, M, N, K, prec, epi, s, num_sms);
    case 160: return launch2_bn<MODE, 160>(A, B, M, N, K, prec, epi, s, num_sms);
    case 128: return launch2_bn<MODE, 128>(A, B, M, N, K, prec, epi, s, num_sms);
    default: return launch2_bn<MODE, 256>(A, B, M, N, K, prec, epi, s, num_sms);
    }
}

// variant: 0 = 2-CTA (default), 1 = 1-CTA; env VSAOGM_GEMM=1cta selects the latter,
// VSAOGM_GEMM_BN=<n> pins the 2-CTA tile width, VSAOGM_GEMM_SPLITS=<s> the split-K factor.
// *ws / *ws_cap: a caller-owned growable workspace for split-K partials.
template <int MODE>
int launch(const void *A, const void *B, int M, int N, int K, int prec, Epi epi, cudaStream_t s, int num_sms,
           int variant, float **ws, size_t *ws_cap)
{
    if (variant < 0) {
        const char *e = getenv("VSAOGM_GEMM");
        variant = (e && strcmp(e, "1cta") == 0) ? 1 : 0;
    }
    if (variant == 1) return launch1<MODE>(A, B, M, N, K, prec, epi, s, num_sms);
    int bn = pick_bn(M, N, num_sms);
    if (const char *e = getenv("VSAOGM_GEMM_BN")) bn = atoi(e);
    int S = pick_splits(M, N, K, bn, num_sms);
    if (const char *e = getenv("VSAOGM_GEMM_SPLITS")) S = atoi(e);
    const int num_kb = K / VSA_BK;
    S = std::max(1, std::min(S, num_kb));
    epi.kb_per = (num_kb + S - 1) / S;
    epi.splits = (num_kb + epi.kb_per - 1) / epi.kb_per;   // no empty split
    if (epi.splits > 1) {
        const size_t need = (size_t)epi.splits * M * N * sizeof(float);
        if (need > *ws_cap) {
            if (*ws) cudaFree(*ws);
            *ws = nullptr;
            *ws_cap = 0;
            if (cudaMalloc(ws, need) != cudaSuccess) { *ws = nullptr; return VSAOGM_ENOMEM; }
            *ws_cap = need;
        }
        epi.ws = *ws;
    }
    return launch2<MODE>(A, B, M, N, K, prec, epi, s, num_sms, bn);
}

}  // namespace

int vsa_launch_decode_gemm(vsaogm_ctx *c, int32_t M, int32_t N, int prec, float inv_scale, float *hb, float *q,
                           int32_t r_ext, int32_t band_off, int32_t band_rows)
{
    Epi e{};
    e.inv_scale = inv_scale;
    e.hb = hb;
    e.q = q;
    e.r_ext = r_ext;
    e.band_off = band_off;
    e.band_rows = band_rows;
    e.ldh = (N + 7) / 8 * 8;
    e.splits = 1;
    e.kb_per = c->Kp / VSA_BK;
    cudaEvent_t ev;
    vsa_prof_begin(c, VSAOGM_K_DECODE_GEMM, &ev);
    int rc = launch<1>(c->d_A, c->d_B, M, N, c->Kp, prec, e, c->stream, c->num_sms, -1, &c->d_ws, &c->ws_cap);
    if (rc) return rc;
    vsa_prof_end(c, VSAOGM_K_DECODE_GEMM, ev);
    c->launches++;
    return VSAOGM_OK;
}

int vsa_gemm_raw(const void *A, const void *B, int32_t M, int32_t N, int32_t K, int prec, float *C, cudaStream_t s,
                 int num_sms, int variant)
{
    Epi e{};
    e.C = C;
    e.splits = 1;
    e.kb_per = K / VSA_BK;
    float *ws = nullptr;
    size_t cap = 0;
    int rc = launch<0>(A, B, M, N, K, prec, e, s, num_sms, variant, &ws, &cap);
    if (ws) {
        cudaStreamSynchronize(s);
        cudaFree(ws);
    }
    return rc;
}
