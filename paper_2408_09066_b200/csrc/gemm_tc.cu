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
// Grouped problem (quadrant memories, delta > 1, sec. III-B-4): the
// cells of quadrant (i, j) query that quadrant's memories, so the contraction
// is a set of GEMMs, one per quadrant: A rows of the quadrant's (class, row)
// block x B rows (= grid columns) of the quadrant's column range.  `Groups`
// (passed by value) lists them; delta = 1 is the single group.
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
//   waves x BN on the 74 SM pairs; split-K (fixed-order reduction) when the
//   tiles cannot fill the GPU.
// k_decode_gemm (1-CTA, M=128 x N=256, single group): the first version, kept as
//   a measured comparison point (VSAOGM_GEMM=1cta) and for the test hook.
#include <cudaTypedefs.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <stdlib.h>
#include <string.h>

#include "common.cuh"

PFN_cuTensorMapEncodeTiled_v12000 vsa_tmap_encode_fn()
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

namespace {

constexpr int GEMM_THREADS = 192;
constexpr uint32_t A_TILE_BYTES = VSA_BM * VSA_BK * 2;   // 16 KB
constexpr uint32_t B_TILE_BYTES = VSA_BN * VSA_BK * 2;   // 32 KB
constexpr uint32_t STAGE_BYTES = A_TILE_BYTES + B_TILE_BYTES;
constexpr uint32_t TMEM_COLS = 512;                       // double-buffered fp32 accumulator
constexpr size_t GEMM_SMEM = 1024 + (size_t)VSA_STAGES * STAGE_BYTES + 256;
constexpr int STAGES2 = 6;                                // 2-CTA ring depth (32 KB / stage at BN=256)

struct Epi {
    float *C;          // MODE 0: raw output, row = group A row, ldc = total columns
    int ldc;
    float inv_scale;   // VSA: q = acc * inv_scale
    float *hb;         // VSA: hb[(c * r_ext + row) * ldh + col]
    uint8_t *code;     // VSA, histogram estimator: 8-bit p code at the same index (hb unused)
    int ldh, r_ext;
    float *q;          // VSA: q[(c * band_rows + row + q_off) * qcols + col] for band rows, or null
    int q_off, band_rows, qcols;
    float *ws;         // split-K partials ws[(s * ws_rows + a_row) * ws_cols + col]
    int ws_rows, ws_cols;
    int splits, kb_per;
    int l2_hints;      // TMA L2 eviction hints: 0 none, 1 A evict-first + B evict-last, 2 B evict-last
    // A tiles generated on the fly (AGEN kernels): a = s_c Ey_k(y) conj(m_ck), stored as
    // conj(a) = e^{-i 2 pi ty_k y} mhat_ck = (Re a, -Im a)  (tables.cu layout, no table A)
    const double *ag_ty;     // theta_y / (2 pi l), turns per metre [Dp]
    const float2 *ag_mhat;   // sqrt(D) m / ||m|| per slot [S][Dp]
    double ag_y0, ag_res;    // first grid row's lower edge minus the phase origin c_y; cell size
    int ag_rlo, ag_Dp, ag_bf16;
    int ag_slot0[VSA_MAX_GROUPS];   // memory slot of class 0 per group
};

__device__ __forceinline__ float hb_of_p(float p)
{
    // binary entropy in bits, 0 log 0 = 0; log1p keeps (1-p) log(1-p) accurate for small p
    float h = 0.f;
    if (p > 0.f) h = -p * log2f(p);
    if (p < 1.f) h -= (1.f - p) * log1pf(-p) * 1.44269504088896341f;
    return h;
}

// 8-bit grey level of a probability: floor(255 p + 1/2) with separately rounded fp32 multiply
// and add (no FMA contraction), clipped to [0, 255] -- DESIGN.md NEXT #2
__device__ __forceinline__ uint8_t code8(float p)
{
    const int c = __float2int_rd(__fadd_rn(__fmul_rn(p, 255.0f), 0.5f));
    return (uint8_t)min(255, max(0, c));
}

__device__ __forceinline__ void store32(float *dst, const float *v, int nvalid, bool vec_ok)
{
    if (nvalid == 32 && vec_ok) {
#pragma unroll
        for (int j = 0; j < 32; j += 4)
            *reinterpret_cast<float4 *>(dst + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
    } else {
#pragma unroll
        for (int j = 0; j < 32; ++j)
            if (j < nvalid) dst[j] = v[j];
    }
}

// One thread's 32 consecutive accumulator columns of local row m_l of group g,
// starting at local column n0.  MODE 0: raw; MODE 1: VSA; MODE 2: split-K partial of split sk.
template <int MODE>
__device__ __forceinline__ void epilogue_chunk(const uint32_t (&v)[32], const Groups &G, int g, int m_l, int n0,
                                               int sk, const Epi &e)
{
    if (m_l >= G.mrows[g] || n0 >= G.ncols[g]) return;
    const int nvalid = min(32, G.ncols[g] - n0);
    const int col = G.col0[g] + n0;
    float f[32];
    if (MODE != 1) {
#pragma unroll
        for (int j = 0; j < 32; ++j) f[j] = __uint_as_float(v[j]);
        const int a_row = G.a_row0[g] + m_l;
        float *dst = MODE == 0 ? e.C + (size_t)a_row * e.ldc + col
                               : e.ws + ((size_t)sk * e.ws_rows + a_row) * e.ws_cols + col;
        const int ld = MODE == 0 ? e.ldc : e.ws_cols;
        store32(dst, f, nvalid, ((col | ld) & 3) == 0);
        return;
    }
    const int nr = G.nrows[g];
    const int cls = m_l >= nr;
    const int row = G.row0[g] + m_l - cls * nr;
    if (e.code) {   // histogram estimator: 8-bit grey level of p (NEXT #2)
#pragma unroll
        for (int j = 0; j < 32; ++j) f[j] = __uint_as_float(v[j]) * e.inv_scale;
        uint8_t *cdst = e.code + ((size_t)cls * e.r_ext + row) * e.ldh + col;
#pragma unroll
        for (int j = 0; j < 32; ++j)
            if (j < nvalid) cdst[j] = code8(fminf(f[j] * f[j], 1.f));
    } else {
        float hv[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) {
            f[j] = __uint_as_float(v[j]) * e.inv_scale;
            hv[j] = hb_of_p(fminf(f[j] * f[j], 1.f));
        }
        store32(e.hb + ((size_t)cls * e.r_ext + row) * e.ldh + col, hv, nvalid, (col & 3) == 0);
    }
    const int br = row + e.q_off;
    if (e.q && br >= 0 && br < e.band_rows)
        store32(e.q + ((size_t)cls * e.band_rows + br) * e.qcols + col, f, nvalid, ((col | e.qcols) & 3) == 0);
}

// ------------------------------------------------------------------ 1-CTA kernel (single group)
template <int MODE>   // 0 = raw fp32 store (test hook), 1 = VSA epilogue
__global__ void __launch_bounds__(GEMM_THREADS, 1)
    k_decode_gemm(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                  const __grid_constant__ Groups G, int K, uint32_t idesc, Epi epi)
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
    const int num_m = (G.mrows[0] + VSA_BM - 1) / VSA_BM;
    const int num_n = (G.ncols[0] + VSA_BN - 1) / VSA_BN;
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
                    tma_load_2d(sA + stage * A_TILE_BYTES, &tmA, &full[stage], kb * VSA_BK,
                                G.a_row0[0] + mb * VSA_BM);
                    tma_load_2d(sB + stage * B_TILE_BYTES, &tmB, &full[stage], kb * VSA_BK,
                                G.col0[0] + nb * VSA_BN);
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
#pragma unroll 1
            for (int cc = 0; cc < VSA_BN / 32; ++cc) {
                uint32_t v[32];
                const uint32_t taddr = tmem_base + ((uint32_t)(quarter * 32) << 16) + as * VSA_BN + cc * 32;
                TMEM_LD_32x32b_X32(taddr, v);
                tmem_ld_wait();
                epilogue_chunk<MODE>(v, G, 0, mb * VSA_BM + row_in_tile, nb * VSA_BN + cc * 32, 0, epi);
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

// ------------------------------------------------------------------ phasor tiles on the fly
// One k-block (32 phasor dimensions = 64 K elements) of this CTA's 128 A rows, written straight
// into the stage's SWIZZLE_128B K-major tile (the layout the TMA would produce: 16-byte chunk
// index XOR row % 8 inside 1024-byte atoms).  128 threads (4 warps); thread t: dimension pair
// kp = t % 16, and two row sequences r = b + 16 i (i = 0..7), b = o + 8 s (s = 0, 1),
// o = {0, 4, 1, 5, 2, 6, 3, 7}[t / 16] (the two half-warps of a warp write rows 4 apart:
// disjoint bank halves).  Along a sequence the row phasor advances by a rotation,
// c(y + 16 res) = c(y) e^{-i 2 pi ty 16 res}; the start of each sequence (and a class change
// inside it) is evaluated directly from the fp64 turn count, as tables.cu does (7 rotation steps
// at most: ~1e-6 relative, far below 16-bit rounding).  The per-dimension inputs (turn rates,
// scaled memories of both classes) are loaded one k-block ahead (AgenIn).
struct AgenIn {
    double ty0, ty1;
    float2 m[2][2];   // [class][dimension k0, k0 + 1]
};

// prefetch a later k-block's inputs into L1 (no register dependence: the generator never waits on it)
__device__ __forceinline__ void agen_prefetch(int kb, int t, int g, const Epi &e)
{
    const int k0 = kb * 32 + 2 * (t & 15);
    if (k0 >= e.ag_Dp) return;
    asm volatile("prefetch.global.L1 [%0];" ::"l"(e.ag_ty + k0));
    asm volatile("prefetch.global.L1 [%0];" ::"l"(e.ag_mhat + (size_t)e.ag_slot0[g] * e.ag_Dp + k0));
    asm volatile("prefetch.global.L1 [%0];" ::"l"(e.ag_mhat + (size_t)(e.ag_slot0[g] + 1) * e.ag_Dp + k0));
}

__device__ __forceinline__ AgenIn agen_load(int kb, int t, int g, const Epi &e)
{
    const int k0 = kb * 32 + 2 * (t & 15);
    AgenIn in;
    in.ty0 = k0 < e.ag_Dp ? e.ag_ty[k0] : 0.0;
    in.ty1 = k0 + 1 < e.ag_Dp ? e.ag_ty[k0 + 1] : 0.0;
#pragma unroll
    for (int cls = 0; cls < 2; ++cls) {
        const float2 *mh = e.ag_mhat + (size_t)(e.ag_slot0[g] + cls) * e.ag_Dp;
        in.m[cls][0] = k0 < e.ag_Dp ? mh[k0] : make_float2(0.f, 0.f);
        in.m[cls][1] = k0 + 1 < e.ag_Dp ? mh[k0 + 1] : make_float2(0.f, 0.f);
    }
    return in;
}

template <bool BF>
__device__ __forceinline__ uint32_t agen_pack(float a, float b)
{
    if (BF) {
        __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
        return *reinterpret_cast<uint32_t *>(&h);
    }
    __half2 h = __floats2half2_rn(a, b);
    return *reinterpret_cast<uint32_t *>(&h);
}

__device__ __forceinline__ float2 agen_expm(double turns_per_m, double coord)
{
    // e^{-i 2 pi f}, f = turns - rint(turns) in [-1/2, 1/2]
    const double t = turns_per_m * coord;
    const double r = __dsub_rn(__dadd_rn(t, 6755399441055744.0), 6755399441055744.0);
    float sv, cv;
    __sincosf(6.28318530717958648f * (float)__dsub_rn(t, r), &sv, &cv);
    return make_float2(cv, -sv);
}

template <bool BF>
__device__ __forceinline__ void agen_kblock(uint8_t *tile, int t, const AgenIn &in, const Groups &G, int g,
                                            int m_base, const Epi &e)
{
    const int kp = t & 15;
    const int q = t >> 4;
    const int o = (q >> 1) + 4 * (q & 1);
    const float2 rot0 = agen_expm(in.ty0, 16.0 * e.ag_res), rot1 = agen_expm(in.ty1, 16.0 * e.ag_res);
    const int nr = G.nrows[g], mrows = G.mrows[g];
    const uint32_t col_re = (uint32_t)(kp >> 2), col_im = 4u + (uint32_t)(kp >> 2);   // logical 16-byte chunks
    const uint32_t inchunk = (uint32_t)(kp & 3) * 4u;
    const double ybase = e.ag_y0 + ((double)(e.ag_rlo + G.row0[g]) + 0.5) * e.ag_res;
#pragma unroll
    for (int sq = 0; sq < 2; ++sq) {
        const int b = o + 8 * sq;                       // first row of the sequence (tile-local)
        float cr0 = 0.f, ci0 = 0.f, cr1 = 0.f, ci1 = 0.f;
        int cls_prev = -1;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const int r = b + 16 * i;
            const int m_l = m_base + r;                 // group-local A row
            uint32_t pre = 0u, pim = 0u;
            if (m_l < mrows) {
                const int cls = m_l >= nr;
                if (cls != cls_prev) {                  // sequence start or class change: direct
                    const double y = ybase + (double)(m_l - cls * nr) * e.ag_res;
                    const float2 p0 = agen_expm(in.ty0, y), p1 = agen_expm(in.ty1, y);
                    const float2 m0 = in.m[cls][0], m1 = in.m[cls][1];
                    cr0 = p0.x * m0.x - p0.y * m0.y;
                    ci0 = p0.x * m0.y + p0.y * m0.x;
                    cr1 = p1.x * m1.x - p1.y * m1.y;
                    ci1 = p1.x * m1.y + p1.y * m1.x;
                    cls_prev = cls;
                } else {                                // advance by 16 rows
                    const float a0 = cr0 * rot0.x - ci0 * rot0.y, b0 = cr0 * rot0.y + ci0 * rot0.x;
                    const float a1 = cr1 * rot1.x - ci1 * rot1.y, b1 = cr1 * rot1.y + ci1 * rot1.x;
                    cr0 = a0; ci0 = b0; cr1 = a1; ci1 = b1;
                }
                pre = agen_pack<BF>(cr0, cr1);
                pim = agen_pack<BF>(ci0, ci1);
            }
            uint8_t *row = tile + (uint32_t)r * 128u;
            const uint32_t sw = (uint32_t)(r & 7);
            *reinterpret_cast<uint32_t *>(row + (((col_re ^ sw) << 4) | inchunk)) = pre;
            *reinterpret_cast<uint32_t *>(row + (((col_im ^ sw) << 4) | inchunk)) = pim;
        }
    }
}

// ------------------------------------------------------------------ 2-CTA kernel (grouped, split-K)
// work unit u -> (tile t = u / S, split sk = u % S); tile t -> group g (prefix of the
// groups' tile counts) -> n-fastest (mb, nb) inside the group.
__device__ __forceinline__ void unit_coords(int tile, const int *s_pref, const int *s_tn, int ng, int &g, int &mb,
                                            int &nb)
{
    g = 0;
    while (g + 1 < ng && tile >= s_pref[g + 1]) ++g;
    const int lt = tile - s_pref[g];
    nb = lt % s_tn[g];
    mb = lt / s_tn[g];
}

// register cap: <= 80 per thread (15 K per CTA) so that a GEMM CTA and three 8-warp encode
// blocks fit one SM's register file when the streaming pipeline overlaps them (bench: §10)
// AGEN: the A tiles are generated in shared memory by four extra warps per CTA (agen_kblock) instead
// of TMA-loaded from table A (north_star: "phasor tiles generated on the fly"); the full barrier then
// counts the B bytes plus the eight generator warps' arrivals of the pair.
// Pipeline waits poll with CTA-scope acquire (mbar_wait), as CUTLASS's cluster pipelines do: the
// arrivals are tcgen05.commit completions (async proxy, ordered by the tcgen05 fences) and the
// epilogue's remote release arrivals after tcgen05.wait::ld; a cluster-scope acquire on every
// poll compiled to an L1 invalidation (CCTL.IVALL) per iteration -- 3.2 M per launch at C4.
// CL = 4: clusters of two CTA pairs; the pairs take m-blocks 2 mp and 2 mp + 1 of the same
// n-block, so both need the same B rows: each CTA TMA-loads half of its B half (BN/4 rows) and
// multicasts it to itself and the same-rank CTA of the other pair -- 23 % fewer L2 -> SM bytes
// per flop at BN = 224.  A slot is then written by two CTAs' producers, so "slot free" needs both
// pairs' MMA commits (count 2, commits multicast to all four CTAs).
template <int MODE, int BN, bool AGEN = false, int CL = 2>
__global__ void __cluster_dims__(CL, 1, 1) __launch_bounds__(AGEN ? GEMM_THREADS + 128 : GEMM_THREADS, AGEN ? 2 : 4)
    k_decode_gemm2(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   const __grid_constant__ Groups G, int K, uint32_t idesc, Epi epi)
{
    static_assert(CL == 2 || (CL == 4 && !AGEN), "4-CTA clusters: TMA-loaded A only");
    constexpr uint32_t A_BYTES = 128 * VSA_BK * 2;          // this CTA's 128 rows of A
    constexpr uint32_t BH_BYTES = (BN / 2) * VSA_BK * 2;    // this CTA's half of B
    constexpr uint32_t ST_BYTES = A_BYTES + BH_BYTES;
    extern __shared__ uint8_t smem_raw[];
    __shared__ int s_pref[VSA_MAX_GROUPS + 1], s_tn[VSA_MAX_GROUPS];
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
    const uint32_t rp = rank & 1, pr = rank >> 1;   // rank in the CTA pair, pair in the cluster
    const int wid = blockIdx.x / CL, num_w = gridDim.x / CL;   // cluster = work-unit owner
    constexpr uint16_t ALL_MASK = CL == 4 ? 0xF : 0x3;
    const uint16_t pair_mask = (uint16_t)(3u << (2 * pr));
    const int num_kb = K / VSA_BK;
    const int S = epi.splits;                 // split-K factor (1 = none)
    const int ng = G.n;

    if (threadIdx.x == 0) {
        int t = 0;
        for (int g = 0; g < ng; ++g) {
            s_pref[g] = t;
            s_tn[g] = (G.ncols[g] + BN - 1) / BN;
            t += (((G.mrows[g] + 255) / 256 + CL / 2 - 1) / (CL / 2)) * s_tn[g];
        }
        s_pref[ng] = t;
        for (int s = 0; s < STAGES2; ++s) {
            mbar_init(&full[s], AGEN ? 9 : 1);   // AGEN: + 4 generator warps x 2 CTAs
            mbar_init(&empty[s], CL / 2);   // CL = 4: both pairs' MMAs read this CTA's B rows
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
    const int num_units = s_pref[ng] * S;

    if (warp == 0) {
        if (lane == 0) {
            asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
            asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
            uint32_t stage = 0, phase = 0;
            for (int u = wid; u < num_units; u += num_w) {
                const int tile = u / S, sk = u - tile * S;
                int g, mb, nb;
                unit_coords(tile, s_pref, s_tn, ng, g, mb, nb);
                if (CL == 4) mb = 2 * mb + (int)pr;
                const int arow = G.a_row0[g] + mb * 256 + (int)rp * 128;
                const int brow = G.col0[g] + nb * BN + (int)rp * (BN / 2);
                const int kb0 = sk * epi.kb_per, kb1 = min(num_kb, kb0 + epi.kb_per);
                for (int kb = kb0; kb < kb1; ++kb) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    if (AGEN) {
                        if (rp == 0) mbar_expect_tx(&full[stage], 2 * BH_BYTES);
                        tma_load_2d_2sm(sB + stage * BH_BYTES, &tmB, &full[stage], kb * VSA_BK, brow);
                        if (++stage == STAGES2) { stage = 0; phase ^= 1; }
                        continue;
                    }
                    if (rp == 0) mbar_expect_tx(&full[stage], 2 * ST_BYTES);
                    if (CL == 4) {
                        tma_load_2d_2sm(sA + stage * A_BYTES, &tmA, &full[stage], kb * VSA_BK, arow);
                        tma_load_2d_2sm_mc(sB + stage * BH_BYTES + pr * (BN / 4) * 128, &tmB, &full[stage], kb * VSA_BK,
                                           brow + (int)pr * (BN / 4), (uint16_t)((1u << rank) | (1u << (rank ^ 2))));
                    } else if (epi.l2_hints == 2) {
                        // B (every panel re-read by the next wave, 66 MB at C4 < 126 MB L2)
                        // evict-last; A normal (an A panel is shared by the concurrent tiles of its
                        // m-block row: n-fastest order)
                        tma_load_2d_2sm(sA + stage * A_BYTES, &tmA, &full[stage], kb * VSA_BK, arow);
                        tma_load_2d_2sm_hint(sB + stage * BH_BYTES, &tmB, &full[stage], kb * VSA_BK, brow,
                                             VSA_L2_EVICT_LAST);
                    } else if (epi.l2_hints == 1) {   // A evict-first as well (measured: A re-read)
                        tma_load_2d_2sm_hint(sA + stage * A_BYTES, &tmA, &full[stage], kb * VSA_BK, arow,
                                             VSA_L2_EVICT_FIRST);
                        tma_load_2d_2sm_hint(sB + stage * BH_BYTES, &tmB, &full[stage], kb * VSA_BK, brow,
                                             VSA_L2_EVICT_LAST);
                    } else {
                        tma_load_2d_2sm(sA + stage * A_BYTES, &tmA, &full[stage], kb * VSA_BK, arow);
                        tma_load_2d_2sm(sB + stage * BH_BYTES, &tmB, &full[stage], kb * VSA_BK, brow);
                    }
                    if (++stage == STAGES2) { stage = 0; phase ^= 1; }
                }
            }
        }
    } else if (warp == 1) {
        if (rp == 0 && lane == 0) {
            uint32_t stage = 0, phase = 0, as = 0, aphase = 0;
            for (int u = wid; u < num_units; u += num_w) {
                const int sk = u % S;
                const int kb0 = sk * epi.kb_per, kb1 = min(num_kb, kb0 + epi.kb_per);
                mbar_wait(&tempty[as], aphase ^ 1);
                tc_fence_after();
                const uint32_t d = tmem_base + as * 256;
                for (int kb = kb0; kb < kb1; ++kb) {
                    mbar_wait(&full[stage], phase);   // (AGEN: + the generators' release.cluster arrivals)
                    tc_fence_after();
                    const uint32_t a0 = smem_u32(sA + stage * A_BYTES);
                    const uint32_t b0 = smem_u32(sB + stage * BH_BYTES);
#pragma unroll
                    for (int k = 0; k < VSA_BK / 16; ++k)
                        tc_mma2_f16(d, sw128_kmajor_desc(a0 + 32 * k), sw128_kmajor_desc(b0 + 32 * k), idesc,
                                    (kb != kb0) || (k != 0));
                    tc_commit2_mc(&empty[stage], ALL_MASK);
                    if (++stage == STAGES2) { stage = 0; phase ^= 1; }
                }
                tc_commit2_mc(&tfull[as], pair_mask);
                if (++as == 2) { as = 0; aphase ^= 1; }
            }
        }
    } else if (AGEN && warp >= 6) {
        // phasor-tile generators: this CTA's 128 A rows of every k-block of every unit; the
        // inputs of the next k-block are loaded while this one is generated
        const int t = (warp - 6) * 32 + lane;
        uint32_t stage = 0, phase = 0;
        for (int u = wid; u < num_units; u += num_w) {
            const int tile = u / S, sk = u - tile * S;
            int g, mb, nb;
            unit_coords(tile, s_pref, s_tn, ng, g, mb, nb);
            const int m_base = mb * 256 + (int)rp * 128;
            const int kb0 = sk * epi.kb_per, kb1 = min(num_kb, kb0 + epi.kb_per);
            for (int j = 1; j <= 3 && kb0 + j < kb1; ++j) agen_prefetch(kb0 + j, t, g, epi);
            AgenIn cur = agen_load(kb0, t, g, epi);
            for (int kb = kb0; kb < kb1; ++kb) {
                if (kb + 4 < kb1) agen_prefetch(kb + 4, t, g, epi);
                const AgenIn nxt = agen_load(kb + 1 < kb1 ? kb + 1 : kb, t, g, epi);   // L1 hit
                // slot free: one lane polls (the arrival is the MMA's commit; a CTA-scope acquire
                // suffices for the write-after-read, and a cluster-scope acquire per thread would
                // invalidate L1 on every poll)
                if (lane == 0) mbar_wait(&empty[stage], phase ^ 1);
                __syncwarp();
                if (epi.ag_bf16) agen_kblock<true>(sA + stage * A_BYTES, t, cur, G, g, m_base, epi);
                else agen_kblock<false>(sA + stage * A_BYTES, t, cur, G, g, m_base, epi);
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic writes -> UMMA reads
                __syncwarp();
                if (lane == 0) {
                    if (rp == 0) mbar_arrive(&full[stage]);
                    else mbar_arrive_cluster(&full[stage], 0);
                }
                if (++stage == STAGES2) { stage = 0; phase ^= 1; }
                cur = nxt;
            }
        }
    } else {
        const int quarter = warp & 3;
        const int row_in_tile = (int)rp * 128 + quarter * 32 + lane;
        uint32_t as = 0, aphase = 0;
        for (int u = wid; u < num_units; u += num_w) {
            const int tile = u / S, sk = u - tile * S;
            int g, mb, nb;
            unit_coords(tile, s_pref, s_tn, ng, g, mb, nb);
            if (CL == 4) mb = 2 * mb + (int)pr;
            mbar_wait(&tfull[as], aphase);
            tc_fence_after();
            const int m_l = mb * 256 + row_in_tile;
#pragma unroll 1
            for (int cc = 0; cc < BN / 32; ++cc) {
                uint32_t v[32];
                const uint32_t taddr = tmem_base + ((uint32_t)(quarter * 32) << 16) + as * 256 + cc * 32;
                TMEM_LD_32x32b_X32(taddr, v);
                tmem_ld_wait();
                if (S == 1) epilogue_chunk<MODE>(v, G, g, m_l, nb * BN + cc * 32, 0, epi);
                else epilogue_chunk<2>(v, G, g, m_l, nb * BN + cc * 32, sk, epi);
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_cluster(&tempty[as], rank & ~1u);
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
__global__ void __launch_bounds__(256) k_splitk_reduce(const __grid_constant__ Groups G, Epi e)
{
    const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    const size_t RC = (size_t)e.ws_rows * e.ws_cols;
    if (idx >= RC) return;
    const int a_row = (int)(idx / e.ws_cols), col = (int)(idx - (size_t)a_row * e.ws_cols);
    int g = -1;
    for (int k = 0; k < G.n; ++k)
        if (a_row >= G.a_row0[k] && a_row < G.a_row0[k] + G.mrows[k] && col >= G.col0[k] &&
            col < G.col0[k] + G.ncols[k]) { g = k; break; }
    if (g < 0) return;
    float acc = 0.f;
    for (int s = 0; s < e.splits; ++s) acc += e.ws[(size_t)s * RC + idx];
    if (MODE == 0) {
        e.C[(size_t)a_row * e.ldc + col] = acc;
        return;
    }
    const int m_l = a_row - G.a_row0[g];
    const int nr = G.nrows[g];
    const int cls = m_l >= nr;
    const int row = G.row0[g] + m_l - cls * nr;
    const float q = acc * e.inv_scale;
    if (e.code) e.code[((size_t)cls * e.r_ext + row) * e.ldh + col] = code8(fminf(q * q, 1.f));
    else e.hb[((size_t)cls * e.r_ext + row) * e.ldh + col] = hb_of_p(fminf(q * q, 1.f));
    const int br = row + e.q_off;
    if (e.q && br >= 0 && br < e.band_rows) e.q[((size_t)cls * e.band_rows + br) * e.qcols + col] = q;
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() { return vsa_tmap_encode_fn(); }

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
int launch1(const void *A, const void *B, int a_rows, int b_rows, int K, int prec, const Groups &G, const Epi &epi,
            cudaStream_t s, int num_sms)
{
    if (G.n != 1) return VSAOGM_EINVAL_ARG;
    CUtensorMap ta, tb;
    int rc = make_map(&ta, A, a_rows, K, VSA_BM, prec);
    if (rc) return rc;
    rc = make_map(&tb, B, b_rows, K, VSA_BN, prec);
    if (rc) return rc;
    VSA_CUDA_TRY(cudaFuncSetAttribute(k_decode_gemm<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)GEMM_SMEM));
    const int tiles = ((G.mrows[0] + VSA_BM - 1) / VSA_BM) * ((G.ncols[0] + VSA_BN - 1) / VSA_BN);
    const int grid = tiles < num_sms ? tiles : num_sms;
    const uint32_t idesc = make_idesc_f16(prec == VSAOGM_BF16, VSA_BM, VSA_BN);
    k_decode_gemm<MODE><<<grid, GEMM_THREADS, GEMM_SMEM, s>>>(ta, tb, G, K, idesc, epi);
    VSA_CUDA_TRY(cudaGetLastError());
    return VSAOGM_OK;
}

long group_tiles(const Groups &G, int bn, int cl = 2)
{
    long t = 0;
    for (int g = 0; g < G.n; ++g)
        t += (long)(((G.mrows[g] + 255) / 256 + cl / 2 - 1) / (cl / 2)) * ((G.ncols[g] + bn - 1) / bn);
    return t;
}

// co-resident 4-CTA clusters of k_decode_gemm2<MODE, BN, false, 4> (a cluster must fit one GPC)
template <int MODE, int BN>
int max_clusters4(size_t smem, int num_sms)
{
    static int cached[2] = {0, 0};
    int &n = cached[MODE ? 1 : 0];
    if (n) return n;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(4 * (num_sms / 4));
    cfg.blockDim = dim3(GEMM_THREADS);
    cfg.dynamicSmemBytes = smem;
    int q = 0;
    if (cudaOccupancyMaxActiveClusters(&q, (void *)k_decode_gemm2<MODE, BN, false, 4>, &cfg) != cudaSuccess || q <= 0) {
        cudaGetLastError();
        q = num_sms / 4 - 2;   // conservative: GPC sizes need not be multiples of 4
    }
    n = q;
    return n;
}

template <int MODE, int BN>
int launch2_bn(const void *A, const void *B, int a_rows, int b_rows, int K, int prec, const Groups &G, Epi epi,
               cudaStream_t s, int num_sms, bool agen, int cl)
{
    CUtensorMap ta, tb;
    if (cl == 4 && !agen) {   // two CTA pairs per cluster, B multicast
        int rc = make_map(&tb, B, b_rows, K, BN / 4, prec);
        if (rc) return rc;
        if ((rc = make_map(&ta, A, a_rows, K, 128, prec))) return rc;
        const size_t smem = 1024 + (size_t)STAGES2 * (128 + BN / 2) * VSA_BK * 2 + 256;
        VSA_CUDA_TRY(cudaFuncSetAttribute(k_decode_gemm2<MODE, BN, false, 4>,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        const long units = group_tiles(G, BN, 4) * epi.splits;
        const int ncl = max_clusters4<MODE, BN>(smem, num_sms);
        const int grid = 4 * (int)(units < ncl ? units : ncl);
        if (grid == 0) return VSAOGM_OK;
        const uint32_t idesc = make_idesc_f16(prec == VSAOGM_BF16, 256, BN);
        k_decode_gemm2<MODE, BN, false, 4><<<grid, GEMM_THREADS, smem, s>>>(ta, tb, G, K, idesc, epi);
        VSA_CUDA_TRY(cudaGetLastError());
        if (epi.splits > 1) {
            const size_t RC = (size_t)epi.ws_rows * epi.ws_cols;
            k_splitk_reduce<MODE><<<(unsigned)((RC + 255) / 256), 256, 0, s>>>(G, epi);
            VSA_CUDA_TRY(cudaGetLastError());
        }
        return VSAOGM_OK;
    }
    int rc = make_map(&tb, B, b_rows, K, BN / 2, prec);
    if (rc) return rc;
    if (agen) ta = tb;   // unused: the A tiles are generated in shared memory
    else if ((rc = make_map(&ta, A, a_rows, K, 128, prec))) return rc;
    const size_t smem = 1024 + (size_t)STAGES2 * (128 + BN / 2) * VSA_BK * 2 + 256;
    const long units = group_tiles(G, BN) * epi.splits;
    const int pairs = num_sms / 2;
    const int grid = 2 * (int)(units < pairs ? units : pairs);
    if (grid == 0) return VSAOGM_OK;
    const uint32_t idesc = make_idesc_f16(prec == VSAOGM_BF16, 256, BN);
    if (agen) {
        VSA_CUDA_TRY(cudaFuncSetAttribute(k_decode_gemm2<MODE, BN, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)smem));
        k_decode_gemm2<MODE, BN, true><<<grid, GEMM_THREADS + 128, smem, s>>>(ta, tb, G, K, idesc, epi);
    } else {
        VSA_CUDA_TRY(cudaFuncSetAttribute(k_decode_gemm2<MODE, BN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)smem));
        k_decode_gemm2<MODE, BN><<<grid, GEMM_THREADS, smem, s>>>(ta, tb, G, K, idesc, epi);
    }
    VSA_CUDA_TRY(cudaGetLastError());
    if (epi.splits > 1) {
        const size_t RC = (size_t)epi.ws_rows * epi.ws_cols;
        k_splitk_reduce<MODE><<<(unsigned)((RC + 255) / 256), 256, 0, s>>>(G, epi);
        VSA_CUDA_TRY(cudaGetLastError());
    }
    return VSAOGM_OK;
}

// BN minimising (waves x BN): the MMA time of a tile is proportional to BN.  When the widest
// tile already fits one wave, it is kept: narrower tiles would fill more pairs but move more
// operand bytes per flop from L2 (measured at C3: BN 256 59 us, BN 128 68 us).
int pick_bn(const Groups &G, int num_sms)
{
    static const int cands[] = {256, 224, 192, 160, 128};
    const int pairs = num_sms / 2;
    if (group_tiles(G, 256) <= pairs) return 256;
    int best = 256;
    long best_cost = -1;
    for (int bn : cands) {
        const long tiles = group_tiles(G, bn);
        const long cost = ((tiles + pairs - 1) / pairs) * bn;
        if (best_cost < 0 || cost < best_cost) { best_cost = cost; best = bn; }
    }
    return best;
}

// Split-K factor for short problems (few tiles for 74 SM pairs, e.g. the row band of one
// rank of 8): model time = waves * tile_time / S + partial-sum traffic, tile_time from the
// measured ~16 TFLOP/s per SM pair, traffic at ~5 TB/s.  S = 1 when the tiles fill the GPU.
int pick_splits(const Groups &G, int ws_rows, int ws_cols, int K, int bn, int num_sms)
{
    const int pairs = num_sms / 2;
    const long tiles = group_tiles(G, bn);
    const int num_kb = K / VSA_BK;
    const double t_tile = 2.0 * 256 * bn * (double)K / 16e12 * 1e6;   // us
    double best_t = -1;
    int best = 1;
    for (int S = 1; S <= 16 && S <= num_kb / 4; ++S) {
        const double waves = (double)((tiles * S + pairs - 1) / pairs);
        double t = waves * t_tile / S;
        if (S > 1) t += 2.0 * S * (double)ws_rows * ws_cols * 4 / 5e12 * 1e6 + 3.0;
        if (best_t < 0 || t < best_t * 0.97) { best_t = t; best = S; }
    }
    return best;
}

template <int MODE>
int launch2(const void *A, const void *B, int a_rows, int b_rows, int K, int prec, const Groups &G, const Epi &epi,
            cudaStream_t s, int num_sms, int bn, bool agen, int cl)
{
    switch (bn) {
    case 224: return launch2_bn<MODE, 224>(A, B, a_rows, b_rows, K, prec, G, epi, s, num_sms, agen, cl);
    case 192: return launch2_bn<MODE, 192>(A, B, a_rows, b_rows, K, prec, G, epi, s, num_sms, agen, cl);
    case 160: return launch2_bn<MODE, 160>(A, B, a_rows, b_rows, K, prec, G, epi, s, num_sms, agen, cl);
    case 128: return launch2_bn<MODE, 128>(A, B, a_rows, b_rows, K, prec, G, epi, s, num_sms, agen, cl);
    default: return launch2_bn<MODE, 256>(A, B, a_rows, b_rows, K, prec, G, epi, s, num_sms, agen, cl);
    }
}

// variant: -1 / 0 = 2-CTA (default), 1 = 1-CTA (single group only), 2 = 4-CTA clusters (two
// pairs, B multicast); bn_force > 0 pins the
// 2-CTA tile width, splits_force > 0 the split-K factor (vsaogm_set_tuning).  *ws / *ws_cap:
// a caller-owned growable workspace for split-K partials.
template <int MODE>
int launch(const void *A, const void *B, int a_rows, int b_rows, int K, int prec, const Groups &G, Epi epi,
           cudaStream_t s, int num_sms, int variant, float **ws, size_t *ws_cap, int bn_force = 0,
           int splits_force = 0, bool agen = false)
{
    if (variant == 1 && G.n == 1 && !agen) return launch1<MODE>(A, B, a_rows, b_rows, K, prec, G, epi, s, num_sms);
    int bn = pick_bn(G, num_sms);
    if (bn_force > 0) bn = bn_force;
    epi.ws_rows = a_rows;
    epi.ws_cols = b_rows;
    int S = pick_splits(G, a_rows, b_rows, K, bn, num_sms);
    if (splits_force > 0) S = splits_force;
    const int num_kb = K / VSA_BK;
    S = std::max(1, std::min(S, num_kb));
    epi.kb_per = (num_kb + S - 1) / S;
    epi.splits = (num_kb + epi.kb_per - 1) / epi.kb_per;   // no empty split
    if (epi.splits > 1) {
        const size_t need = (size_t)epi.splits * a_rows * b_rows * sizeof(float);
        if (need > *ws_cap) {
            if (*ws) cudaFree(*ws);
            *ws = nullptr;
            *ws_cap = 0;
            if (cudaMalloc(ws, need) != cudaSuccess) { *ws = nullptr; return VSAOGM_ENOMEM; }
            *ws_cap = need;
        }
        epi.ws = *ws;
    }
    return launch2<MODE>(A, B, a_rows, b_rows, K, prec, G, epi, s, num_sms, bn, agen, variant == 2 ? 4 : 2);
}

}  // namespace

int vsa_launch_decode_gemm(vsaogm_ctx *c, const Groups &G, int32_t a_rows, int32_t N, int prec, float inv_scale,
                           float *hb, float *q, int32_t r_ext, int32_t q_off, int32_t band_rows, const int *slot0,
                           double y0, double res, int32_t r_lo)
{
    Epi e{};
    e.inv_scale = inv_scale;
    e.hb = hb;
    e.code = c->estimator == 1 ? c->d_code : nullptr;
    e.ldh = (N + 7) / 8 * 8;
    e.r_ext = r_ext;
    e.q = q;
    e.q_off = q_off;
    e.band_rows = band_rows;
    e.qcols = N;
    e.splits = 1;
    e.kb_per = c->Kp / VSA_BK;
    e.l2_hints = c->gemm_l2_hints;
    const bool agen = c->gemm_agen != 0;
    if (agen) {
        int rc0 = vsa_launch_mhat(c);
        if (rc0) return rc0;
        e.ag_ty = c->d_ty_turns;
        e.ag_mhat = c->d_mhat;
        e.ag_y0 = y0 - c->cy;
        e.ag_res = res;
        e.ag_rlo = r_lo;
        e.ag_Dp = c->Dp;
        e.ag_bf16 = prec == VSAOGM_BF16;
        for (int g = 0; g < G.n; ++g) e.ag_slot0[g] = slot0[g];
    }
    cudaEvent_t ev;
    vsa_prof_begin(c, VSAOGM_K_DECODE_GEMM, &ev);
    int rc = launch<1>(c->d_A, c->d_B, a_rows, N, c->Kp, prec, G, e, c->stream, c->num_sms, c->gemm_variant, &c->d_ws,
                       &c->ws_cap, c->gemm_bn, c->gemm_splits, agen);
    if (rc) return rc;
    vsa_prof_end(c, VSAOGM_K_DECODE_GEMM, ev);
    c->launches++;
    return VSAOGM_OK;
}

int vsa_gemm_raw(const void *A, const void *B, int32_t M, int32_t N, int32_t K, int prec, float *C, cudaStream_t s,
                 int num_sms, int variant, int bn, int splits)
{
    Groups G{};
    G.n = 1;
    G.a_row0[0] = 0;
    G.mrows[0] = M;
    G.nrows[0] = M;
    G.row0[0] = 0;
    G.col0[0] = 0;
    G.ncols[0] = N;
    Epi e{};
    e.C = C;
    e.ldc = N;
    e.splits = 1;
    e.kb_per = K / VSA_BK;
    float *ws = nullptr;
    size_t cap = 0;
    int rc = launch<0>(A, B, M, N, K, prec, G, e, s, num_sms, variant, &ws, &cap, bn, splits);
    if (ws) {
        cudaStreamSynchronize(s);
        cudaFree(ws);
    }
    return rc;
}
