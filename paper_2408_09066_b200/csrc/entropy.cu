// entropy.cu -- K6: local Shannon entropy, global entropy and labels.
//
//   S_c(r, col) = mean of H_b(p_c) over the window footprint clipped to the full grid
//                 (Alg. 2; per-class radii r(psi=1), r(psi=0);
//                  estimator and clipping per DESIGN.md L10, L11, L13)
//   S = S_1 - S_0                                   (Alg. 2)
//   label = 1 occupied if S >= rho_occ, 0 empty if S < rho_emp, else 2 unknown
//                                                   (Eq. 12 PAPER.md:320-328 + L14)
//
// Input is the per-cell H_b(q_c^2) written by the decode epilogue for the band
// plus halo rows ([2][R_ext][ldh] fp32).  Input outside the decoded rows /
// grid columns reads as zero, which is exactly the border clipping of the
// window sums (L13); clipped counts are closed-form.  A box window
// forms row sums of width 2h+1 then sums 2h+1 of them down the column; a disk
// sums each footprint row segment directly.  Kernels: k_entropy_stream (box,
// equal radii h <= 4: the BASELINE windows; TMA-streamed warps, register
// rings), k_entropy (any radii / disks, cp.async-staged tile), k_entropy_hist
// (the histogram estimator).  HBM-bound: 8 B read + 1 B written per cell.
#include <cudaTypedefs.h>

#include "common.cuh"

namespace {

constexpr int TR = 32;    // output rows per CTA
constexpr int TC = 128;   // output cols per CTA
constexpr int HMAX = 16;
constexpr int ENT_THREADS = 2 * TC;   // two threads per column, each owning half of the output rows

__device__ __forceinline__ int isqrt_floor(int t)
{
    int w = (int)sqrtf((float)t);
    while ((w + 1) * (w + 1) <= t) ++w;
    while (w * w > t) --w;
    return w;
}


// Box window, equal radii h1 = h0 = H <= 4 (every BASELINE config: 3x3 / 5x5 / 7x7), labels
// only (the streaming step's output; a request for the S maps takes the generic kernel).
// HBM-bound: 8 B read + 1 B written per cell.  Persistent warps take work items from a device
// queue; an item is one 128-column strip x `rw` output rows of the band, streamed top to
// bottom:
//   * lane 0 keeps a private ring of NST = 2H+1 TMA stages of RS = 2 rows in flight
//     (cp.async.bulk.tensor.3d, box 136 columns x 2 rows x both classes, 4 halo columns on
//     each side; the tensor map's bounds are the decoded rows x grid columns, so the TMA
//     zero-fill IS the window clipping of DESIGN.md L13) on per-stage mbarriers -- no block
//     barriers, every warp independent;
//   * rows go in blocks of U = RS NST rows (a multiple of W = 2H+1), so the stage slot, the
//     row inside the stage and the register-ring slot of every row are compile-time;
//   * each lane owns 4 adjacent columns: per staged row and class it reads its float4 and the
//     H neighbour columns on each side straight from the staged row (no shuffles: shared
//     memory has the bandwidth, the issue slots are the limit), forms the first horizontal
//     (2H+1)-sum in order and the next three by sliding, and the class difference
//     d = h_occ - h_emp; a running vertical sum V += d_new - d_old (the last W differences in
//     registers) gives S = S_occ - S_emp = V / count for the row 2H above, then the label.
// Against the fp64 definition the fp32 rounding of these sums is <= 2e-6 in S (DESIGN.md
// section 7).
constexpr int ST_WARPS = 4;                       // warps per block
constexpr int ST_COLS = 128;                      // output columns per strip (4 per lane)
constexpr int ST_W = ST_COLS + 8;                 // staged floats per row (4 + 128 + 4)

template <int H>
struct StCfg {
    static constexpr int W = 2 * H + 1;
    static constexpr int RS = 2;                              // rows per stage
    static constexpr int NST = W;                             // stages per ring
    static constexpr int U = RS * NST;                        // rows per block (multiple of W)
    static constexpr int STAGE_FLOATS = (2 * RS * ST_W + 31) / 32 * 32;   // [class][row][col], 128 B aligned
    static constexpr int STAGE_BYTES = 2 * RS * ST_W * 4;     // TMA box bytes
    static constexpr int WARP_BYTES = NST * STAGE_FLOATS * 4;
    static constexpr int BLOCK_SMEM = ST_WARPS * WARP_BYTES;
    static constexpr int BLOCKS_PER_SM = 200 * 1024 / BLOCK_SMEM < 4 ? 200 * 1024 / BLOCK_SMEM : 4;
};

struct StreamArgs {
    int R, C, r_lo;            // full grid; first decoded row (tensor-map row 0)
    int r0, band_rows;         // band: full-grid rows [r0, r0 + band_rows)
    int strips, chunks, rw;    // work items = strips x chunks of rw output rows
    float rho_occ, rho_emp;
    uint8_t *lab;
    int *ctr;                  // [0] next item, [1] warps done (reset by the last warp)
};

__device__ __forceinline__ void tma_load_3d(void *dst, const CUtensorMap *map, uint64_t *bar, int c0, int c1, int c2)
{
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
            smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
        : "memory");
}

// label of one cell (Eq. 12 + L14): 1 occupied if S >= rho_occ, 0 empty if S < rho_emp, else 2
__device__ __forceinline__ uint32_t label_of(float g, float rho_occ, float rho_emp)
{
    return g >= rho_occ ? 1u : (g < rho_emp ? 0u : 2u);
}

template <int H>
__global__ void __launch_bounds__(ST_WARPS * 32, StCfg<H>::BLOCKS_PER_SM)
    k_entropy_stream(const __grid_constant__ CUtensorMap tm, const StreamArgs a)
{
    static_assert(H >= 1 && H <= 4, "halo within one float4 per side");
    using Cfg = StCfg<H>;
    constexpr int W = Cfg::W, RS = Cfg::RS, NST = Cfg::NST, U = Cfg::U;
    extern __shared__ __align__(128) float sm_st[];
    __shared__ __align__(8) uint64_t bars[ST_WARPS][NST];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    float *ring_smem = sm_st + (size_t)warp * NST * Cfg::STAGE_FLOATS;
    uint64_t *bar = bars[warp];
    if (lane == 0) {
        for (int s = 0; s < NST; ++s) mbar_init(&bar[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncwarp();
    vsa_pdl();   // the barrier set-up above overlaps the decode's tail; H_b is read only from here on
    const int items = a.strips * a.chunks;
    uint32_t blk = 0;   // row blocks this warp has consumed: every slot is used once per block
    const float *lane_base = ring_smem + 4 + 4 * lane;        // this lane's 4 columns
    for (;;) {
        int it = 0;
        if (lane == 0) it = atomicAdd(&a.ctr[0], 1);
        it = __shfl_sync(0xffffffffu, it, 0);
        if (it >= items) break;
        const int strip = it % a.strips, chunk = it / a.strips;
        const int col0 = strip * ST_COLS;
        const int oA = chunk * a.rw;                          // band-relative output rows [oA, oB)
        const int oB = min(a.band_rows, oA + a.rw);
        const int rA = a.r0 + oA;                             // full-grid row of output oA
        const int nblk = ((oB - oA) + 2 * H + U - 1) / U;     // staged rows rA - H ..., padded
        auto issue = [&](int b, int s) {                      // block b, stage s -> slot s
            mbar_expect_tx(&bar[s], Cfg::STAGE_BYTES);
            tma_load_3d(ring_smem + s * Cfg::STAGE_FLOATS, &tm, &bar[s], col0 - 4,
                        rA - H + b * U + s * RS - a.r_lo, 0);
        };
        if (lane == 0)
            for (int s = 0; s < NST; ++s) issue(0, s);
        const int c0 = col0 + 4 * lane;
        // column clip counts and the interior-row reciprocals 1 / (W nc)
        float ncf[4], inv_in[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            ncf[j] = (float)(min(c0 + j + H, a.C - 1) - max(c0 + j - H, 0) + 1);
            inv_in[j] = 1.0f / ((float)W * ncf[j]);
        }
        const bool full4 = c0 + 3 < a.C && (a.C & 3) == 0;
        uint8_t *lab_item = a.lab + (size_t)oA * a.C + c0;
        float ring[W][4];                                     // d = h_occ - h_emp of the last W rows
        float V[4] = {0.f, 0.f, 0.f, 0.f};                    // running vertical sums of d
        uint8_t *lp = lab_item - (size_t)2 * H * a.C;         // label row of staged row i: lp + i C
        for (int b = 0; b < nblk; ++b, ++blk) {
            const uint32_t par = blk & 1u;
#pragma unroll
            for (int uu = 0; uu < U; ++uu) {
                const int s = uu / RS, rr = uu % RS, u = uu % W;
                if (rr == 0) mbar_wait(&bar[s], par);
                const int soff = s * Cfg::STAGE_FLOATS + rr * ST_W;
                float hs[2][4];
#pragma unroll
                for (int cls = 0; cls < 2; ++cls) {
                    // columns c0-H .. c0+3+H straight from the staged row (halo included: no shuffles)
                    const float *rp = lane_base + soff + cls * RS * ST_W;
                    float x[12];                              // x[4 + j] = column c0 + j
                    const float4 v = *reinterpret_cast<const float4 *>(rp);
                    x[4] = v.x; x[5] = v.y; x[6] = v.z; x[7] = v.w;
                    if (H <= 2) {
                        const float2 l2 = *reinterpret_cast<const float2 *>(rp - 2);
                        const float2 r2 = *reinterpret_cast<const float2 *>(rp + 4);
                        x[2] = l2.x; x[3] = l2.y; x[8] = r2.x; x[9] = r2.y;
                    } else {
                        const float4 l4 = *reinterpret_cast<const float4 *>(rp - 4);
                        const float4 r4 = *reinterpret_cast<const float4 *>(rp + 4);
                        x[0] = l4.x; x[1] = l4.y; x[2] = l4.z; x[3] = l4.w;
                        x[8] = r4.x; x[9] = r4.y; x[10] = r4.z; x[11] = r4.w;
                    }
                    // horizontal (2H+1)-sums: the first in order, the next three sliding
                    float h0 = x[4 - H];
#pragma unroll
                    for (int dv = -H + 1; dv <= H; ++dv) h0 += x[4 + dv];
                    hs[cls][0] = h0;
#pragma unroll
                    for (int j = 1; j < 4; ++j) hs[cls][j] = (hs[cls][j - 1] - x[3 + j - H]) + x[4 + j + H];
                }
                if (rr == RS - 1) {                           // stage s consumed: refill for block b+1
                    // every lane's reads of the stage have completed (their values were consumed
                    // by the sums above), so the TMA may overwrite it once the warp reconverges
                    __syncwarp();
                    if (lane == 0 && b + 1 < nblk) issue(b + 1, s);
                }
                const int i = b * U + uu;                     // staged row
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const float d = hs[1][j] - hs[0][j];     // h_occ - h_emp
                    V[j] += d;
                    if (i >= W) V[j] -= ring[u][j];           // drop row i - W
                    ring[u][j] = d;
                }
                const int o = oA + i - 2 * H;                 // band-relative output row
                if (i >= 2 * H && o < oB) {                   // warp-uniform
                    const int row = a.r0 + o;
                    float g4[4];
#pragma unroll
                    for (int j = 0; j < 4; ++j) g4[j] = V[j] * inv_in[j];
                    if (row < H || row >= a.R - H) {          // clipped rows (grid top / bottom)
                        const float cntr = (float)(min(row + H, a.R - 1) - max(row - H, 0) + 1);
#pragma unroll
                        for (int j = 0; j < 4; ++j) g4[j] = V[j] * (1.0f / (cntr * ncf[j]));
                    }
                    const uint32_t l4 = label_of(g4[0], a.rho_occ, a.rho_emp) | label_of(g4[1], a.rho_occ, a.rho_emp) << 8 |
                                        label_of(g4[2], a.rho_occ, a.rho_emp) << 16 |
                                        label_of(g4[3], a.rho_occ, a.rho_emp) << 24;
                    uint8_t *lrow = lp + (size_t)i * a.C;
                    if (full4) *reinterpret_cast<uint32_t *>(lrow) = l4;
                    else
                        for (int j = 0; j < 4 && c0 + j < a.C; ++j) lrow[j] = (uint8_t)(l4 >> (8 * j));
                }
            }
        }
    }
    // the last warp to finish resets the queue for the next launch
    if (lane == 0) {
        __threadfence();
        if (atomicAdd(&a.ctr[1], 1) == (int)(gridDim.x * ST_WARPS) - 1) {
            a.ctr[0] = 0;
            a.ctr[1] = 0;
        }
    }
}

__global__ void __launch_bounds__(ENT_THREADS) k_entropy(const float *__restrict__ hb, int ldh, int r_ext, int R,
                                                         int C, int r_lo, int r0, int band_rows, int h1, int h0,
                                                         int disk, float rho_occ, float rho_emp,
                                                         float *__restrict__ S, uint8_t *__restrict__ lab)
{
    extern __shared__ float sm[];
    __shared__ int s_w[2][2 * HMAX + 1];   // footprint half-width of each window row
    const int H = max(h1, h0);
    const int TW = TC + 2 * H, TH = TR + 2 * H;
    float *tile = sm;                      // [2][TH][TW]
    float *hs = sm + 2 * TH * TW;          // [2][TH][TC] (box: row sums)
    const int orow0 = r0 + blockIdx.y * TR;
    const int ocol0 = blockIdx.x * TC;
    const int tid = threadIdx.x & (TC - 1);     // column lane
    const int half = threadIdx.x / TC;          // which half of the output rows

    if (threadIdx.x < 2 * (2 * HMAX + 1)) {
        const int cls = threadIdx.x / (2 * HMAX + 1), j = threadIdx.x % (2 * HMAX + 1);
        const int h = cls == 1 ? h1 : h0;
        const int du = j - HMAX;
        s_w[cls][j] = (du < -h || du > h) ? -1 : (disk ? isqrt_floor(h * h - du * du) : h);
    }
    // stage both classes with cp.async (4-byte, zero-fill outside the decoded rows / grid
    // columns = the window clipping): every element is an independent request in flight
    {
        const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
        for (int cr = warp; cr < 2 * TH; cr += ENT_THREADS / 32) {
            const int cls = cr >= TH, row = cr - cls * TH;
            const int rr = orow0 - H + row;               // full-grid row
            const bool rin = rr >= 0 && rr < R && rr - r_lo < r_ext;
            const float *srow = hb + ((size_t)cls * r_ext + (size_t)(rin ? rr - r_lo : 0)) * ldh;
            float *t = tile + cr * TW;
            for (int cc = lane; cc < TW; cc += 32) {
                const int gc = ocol0 - H + cc;
                const bool ok = rin && gc >= 0 && gc < C;
                asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(smem_u32(t + cc)),
                             "l"(srow + (ok ? gc : 0)), "r"(ok ? 4 : 0)
                             : "memory");
            }
        }
        asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
    }
    __syncthreads();

    const int col = ocol0 + tid;
    if (!disk) {
#pragma unroll
        for (int cls = 0; cls < 2; ++cls) {
            const int h = cls == 1 ? h1 : h0;
            const float *t = tile + cls * TH * TW + H + tid;
            float *o = hs + cls * TH * TC + tid;
            for (int row = H - h + half; row < TR + H + h; row += 2) {
                float s = 0.f;
                for (int dv = -h; dv <= h; ++dv) s += t[row * TW + dv];
                o[row * TC] = s;
            }
        }
        __syncthreads();
    }
    const int nc1 = min(col + h1, C - 1) - max(col - h1, 0) + 1;
    const int nc0 = min(col + h0, C - 1) - max(col - h0, 0) + 1;
    for (int r = half * (TR / 2); r < (half + 1) * (TR / 2); ++r) {
        const int row = orow0 + r;
        const int br = row - r0;
        if (br >= band_rows) break;
        float Sc[2];
#pragma unroll
        for (int cls = 0; cls < 2; ++cls) {
            const int h = cls == 1 ? h1 : h0;
            float s = 0.f;
            float cnt;
            if (!disk) {
                const float *o = hs + cls * TH * TC + tid;
                for (int du = -h; du <= h; ++du) s += o[(r + H + du) * TC];
                const int nr = min(row + h, R - 1) - max(row - h, 0) + 1;
                cnt = (float)(nr * (cls == 1 ? nc1 : nc0));
            } else {
                const float *t = tile + cls * TH * TW + H + tid;
                int n = 0;
                for (int du = -h; du <= h; ++du) {
                    const int w = s_w[cls][du + HMAX];
                    const float *tr = t + (r + H + du) * TW;
                    for (int dv = -w; dv <= w; ++dv) s += tr[dv];
                    if (row + du >= 0 && row + du < R) n += min(col + w, C - 1) - max(col - w, 0) + 1;
                }
                cnt = (float)n;
            }
            Sc[cls] = __fmul_rn(s, 1.0f / cnt);   // as the streamed kernel (no contraction): bit-identical

        }
        if (col < C) {
            const float g = __fsub_rn(Sc[1], Sc[0]);
            const size_t o = (size_t)br * C + col;
            if (S) {
                S[o] = Sc[1];
                S[(size_t)band_rows * C + o] = Sc[0];
                S[(size_t)2 * band_rows * C + o] = g;
            }
            if (lab) lab[o] = g >= rho_occ ? 1 : (g < rho_emp ? 0 : 2);
        }
    }
}

// Histogram estimator (NEXT #2): S_c = Shannon entropy (bits) of the 8-bit grey-level
// histogram of p_c in the clipped footprint.  One thread per output column walks TR rows;
// each thread owns a 256-bin uint16 histogram in shared memory (bins interleaved across
// threads: bin b of thread t at [b][t], conflict-free for equal bins), counts the window,
// then sums n log2 n over the window's bins (table) while clearing them:
// S = log2 N - (1/N) sum_b n_b log2 n_b.
constexpr int HT = 128;   // threads (= output columns) per block
constexpr int HR = 16;    // output rows per block
__global__ void __launch_bounds__(HT) k_entropy_hist(const uint8_t *__restrict__ code, int ldh, int r_ext, int R, int C,
                                                     int r_lo, int r0, int band_rows, int h1, int h0, int disk,
                                                     float rho_occ, float rho_emp, float *__restrict__ S,
                                                     uint8_t *__restrict__ lab)
{
    extern __shared__ uint8_t smh[];
    const int H = max(h1, h0);
    const int TW = HT + 2 * H, TH = HR + 2 * H;
    const int NMAX = (2 * H + 1) * (2 * H + 1);
    uint16_t *hist = reinterpret_cast<uint16_t *>(smh);                       // [256][HT]
    float *nlogn = reinterpret_cast<float *>(smh + 256 * HT * 2);             // [NMAX + 1]
    uint8_t *tile = smh + 256 * HT * 2 + 4 * (NMAX + 1);                      // [2][TH][TW]
    __shared__ int s_w[2][2 * HMAX + 1];
    const int tid = threadIdx.x;
    const int orow0 = r0 + blockIdx.y * HR, ocol0 = blockIdx.x * HT;
    for (int n = tid; n <= NMAX; n += HT) nlogn[n] = n > 0 ? (float)n * log2f((float)n) : 0.f;
    for (int k = 0; k < 256; ++k) hist[k * HT + tid] = 0;   // each thread clears its own bins
    if (tid < 2 * (2 * HMAX + 1)) {
        const int cls = tid / (2 * HMAX + 1), j = tid % (2 * HMAX + 1);
        const int h = cls == 1 ? h1 : h0, du = j - HMAX;
        s_w[cls][j] = (du < -h || du > h) ? -1 : (disk ? isqrt_floor(h * h - du * du) : h);
    }
    for (int idx = tid; idx < 2 * TH * TW; idx += HT) {
        const int cls = idx / (TH * TW), rem = idx - cls * TH * TW;
        const int row = rem / TW, cc = rem - row * TW;
        const int rr = orow0 - H + row, gc = ocol0 - H + cc;
        const bool ok = rr >= 0 && rr < R && rr - r_lo < r_ext && gc >= 0 && gc < C;
        tile[idx] = ok ? code[((size_t)cls * r_ext + (rr - r_lo)) * ldh + gc] : 0;
    }
    __syncthreads();
    const int col = ocol0 + tid;
    for (int r = 0; r < HR; ++r) {
        const int row = orow0 + r;
        const int br = row - r0;
        if (br >= band_rows) break;
        float Sc[2];
        for (int cls = 0; cls < 2; ++cls) {
            const uint8_t *t = tile + cls * TH * TW;
            int n = 0;
            // count (only cells inside the full grid belong to the clipped footprint)
            for (int du = -H; du <= H; ++du) {
                const int w = s_w[cls][du + HMAX];
                if (w < 0 || row + du < 0 || row + du >= R) continue;
                const uint8_t *tr = t + (r + H + du) * TW + tid + H;
                for (int dv = -w; dv <= w; ++dv) {
                    if (col + dv < 0 || col + dv >= C) continue;
                    hist[tr[dv] * HT + tid]++;
                    ++n;
                }
            }
            // sum n log n over the occupied bins, clearing them
            float s = 0.f;
            for (int du = -H; du <= H; ++du) {
                const int w = s_w[cls][du + HMAX];
                if (w < 0 || row + du < 0 || row + du >= R) continue;
                const uint8_t *tr = t + (r + H + du) * TW + tid + H;
                for (int dv = -w; dv <= w; ++dv) {
                    if (col + dv < 0 || col + dv >= C) continue;
                    uint16_t &hb = hist[tr[dv] * HT + tid];
                    s += nlogn[hb];
                    hb = 0;
                }
            }
            Sc[cls] = n > 0 ? log2f((float)n) - s / (float)n : 0.f;
        }
        if (col < C) {
            const float g = Sc[1] - Sc[0];
            const size_t o = (size_t)br * C + col;
            if (S) {
                S[o] = Sc[1];
                S[(size_t)band_rows * C + o] = Sc[0];
                S[(size_t)2 * band_rows * C + o] = g;
            }
            if (lab) lab[o] = g >= rho_occ ? 1 : (g < rho_emp ? 0 : 2);
        }
    }
}

// Box window, equal radii H <= 4, labels only -- the same contract as k_entropy_stream, without
// shared memory, TMA or barriers: a thread owns 4 adjacent columns of one chunk of `rw` output rows
// and walks down the rw + 2H input rows.  Per row it loads its float4 and the HL = 2 (H <= 2) or 4
// halo columns on each side of both classes straight from global memory (the H_b map was written by
// the decode just before and is L2-resident; the halos are its neighbours' float4s: L1 hits),
// forms d = h_occ - h_emp per column, the four horizontal (2H+1)-sums of d (the first in order,
// the next three sliding) and the running vertical sum V += s_new - s_old over the last 2H+1 rows
// (a register ring, rows unrolled by 2H+1 so that the ring slot is compile-time and the loads of
// 2H+1 rows are in flight together): S = V / count for the row 2H above, then the label.  Rows and
// columns outside the grid contribute 0 and the count is the clipped one (L13).
template <int H>
__global__ void __launch_bounds__(128) k_entropy_cols(const float *__restrict__ hb, int ldh, int r_ext, int R, int C, int r_lo,
                                                      int r0, int band_rows, int rw, float rho_occ, float rho_emp,
                                                      uint8_t *__restrict__ lab)
{
    vsa_pdl();
    constexpr int W = 2 * H + 1;
    constexpr int HL = H <= 2 ? 2 : 4;             // halo columns loaded per side
    const int c0 = (blockIdx.x * 128 + threadIdx.x) * 4;
    if (c0 >= C) return;
    const int oA = blockIdx.y * rw, oB = min(band_rows, oA + rw);   // band-relative output rows
    const int rA = r0 + oA;                                         // full-grid row of output oA
    const int nrows = (oB - oA) + 2 * H;                            // input rows rA - H .. rA - H + nrows - 1
    float ncf[4], inv_in[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        ncf[j] = (float)(min(c0 + j + H, C - 1) - max(c0 + j - H, 0) + 1);
        inv_in[j] = 1.0f / ((float)W * ncf[j]);
    }
    const bool fast = c0 - HL >= 0 && c0 + 4 + HL <= C;             // every loaded column is inside the grid
    const bool full4 = c0 + 3 < C && (C & 3) == 0;
    const float *p0 = hb + c0, *p1 = hb + (size_t)r_ext * ldh + c0;
    float ring[W][4];
#pragma unroll
    for (int u = 0; u < W; ++u)
#pragma unroll
        for (int j = 0; j < 4; ++j) ring[u][j] = 0.f;
    float V[4] = {0.f, 0.f, 0.f, 0.f};
    constexpr int NV = 4 + 2 * HL;                                  // columns loaded per row and class
    constexpr int G = H <= 2 ? W : 4;                               // rows whose loads are in flight together
    for (int ib = 0; ib < nrows; ib += W) {
#pragma unroll
        for (int ug = 0; ug < W; ug += G) {
            // phase 1: every load of the group's rows, unconditionally (rows outside the grid or the
            // chunk read a clamped row and are masked below), so that they are all in flight at once
            float x1[G][NV], x0[G][NV];
            bool rv[G];
#pragma unroll
            for (int g = 0; g < G; ++g) {
                const int u = ug + g;
                if (u >= W) continue;                               // compile time
                const int i = ib + u;
                const int gr = rA - H + i, dr = gr - r_lo;
                rv[g] = i < nrows && gr >= 0 && gr < R && dr >= 0 && dr < r_ext;
                const size_t off = (size_t)min(max(dr, 0), r_ext - 1) * ldh;
                if (fast) {
                    const float4 a1 = __ldg(reinterpret_cast<const float4 *>(p1 + off));
                    const float4 a0 = __ldg(reinterpret_cast<const float4 *>(p0 + off));
                    x1[g][HL] = a1.x; x1[g][HL + 1] = a1.y; x1[g][HL + 2] = a1.z; x1[g][HL + 3] = a1.w;
                    x0[g][HL] = a0.x; x0[g][HL + 1] = a0.y; x0[g][HL + 2] = a0.z; x0[g][HL + 3] = a0.w;
                    if (HL == 2) {
                        const float2 l1 = __ldg(reinterpret_cast<const float2 *>(p1 + off - 2));
                        const float2 l0 = __ldg(reinterpret_cast<const float2 *>(p0 + off - 2));
                        const float2 r1 = __ldg(reinterpret_cast<const float2 *>(p1 + off + 4));
                        const float2 r0v = __ldg(reinterpret_cast<const float2 *>(p0 + off + 4));
                        x1[g][0] = l1.x; x1[g][1] = l1.y; x1[g][HL + 4] = r1.x; x1[g][HL + 5] = r1.y;
                        x0[g][0] = l0.x; x0[g][1] = l0.y; x0[g][HL + 4] = r0v.x; x0[g][HL + 5] = r0v.y;
                    } else {
                        const float4 l1 = __ldg(reinterpret_cast<const float4 *>(p1 + off - 4));
                        const float4 l0 = __ldg(reinterpret_cast<const float4 *>(p0 + off - 4));
                        const float4 r1 = __ldg(reinterpret_cast<const float4 *>(p1 + off + 4));
                        const float4 r0v = __ldg(reinterpret_cast<const float4 *>(p0 + off + 4));
                        x1[g][0] = l1.x; x1[g][1] = l1.y; x1[g][2] = l1.z; x1[g][3] = l1.w;
                        x0[g][0] = l0.x; x0[g][1] = l0.y; x0[g][2] = l0.z; x0[g][3] = l0.w;
                        x1[g][8] = r1.x; x1[g][9] = r1.y; x1[g][10] = r1.z; x1[g][11] = r1.w;
                        x0[g][8] = r0v.x; x0[g][9] = r0v.y; x0[g][10] = r0v.z; x0[g][11] = r0v.w;
                    }
                } else {
#pragma unroll
                    for (int e = 0; e < NV; ++e) {
                        const int col = c0 + e - HL;
                        const bool in = col >= 0 && col < C;
                        x1[g][e] = in ? __ldg(p1 + off + e - HL) : 0.f;
                        x0[g][e] = in ? __ldg(p0 + off + e - HL) : 0.f;
                    }
                }
            }
            // phase 2: class difference, horizontal sums, running vertical sum, labels
#pragma unroll
            for (int g = 0; g < G; ++g) {
                const int u = ug + g;
                if (u >= W) continue;                               // compile time
                const int i = ib + u;
                float d[NV];                                        // d[HL + j] = column c0 + j
#pragma unroll
                for (int e = 0; e < NV; ++e) d[e] = rv[g] ? x1[g][e] - x0[g][e] : 0.f;
                float hs[4];
                float h0 = d[HL - H];
#pragma unroll
                for (int dv = -H + 1; dv <= H; ++dv) h0 += d[HL + dv];
                hs[0] = h0;
#pragma unroll
                for (int j = 1; j < 4; ++j) hs[j] = (hs[j - 1] - d[HL + j - 1 - H]) + d[HL + j + H];
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    V[j] += hs[j];
                    V[j] -= ring[u][j];                             // row i - W (0 for the first W rows)
                    ring[u][j] = hs[j];
                }
                const int o = oA + i - 2 * H;                       // band-relative output row
                if (i >= 2 * H && o < oB) {                         // warp-uniform
                    const int row = r0 + o;
                    float g4[4];
#pragma unroll
                    for (int j = 0; j < 4; ++j) g4[j] = V[j] * inv_in[j];
                    if (row < H || row >= R - H) {                  // clipped rows (grid top / bottom)
                        const float cntr = (float)(min(row + H, R - 1) - max(row - H, 0) + 1);
#pragma unroll
                        for (int j = 0; j < 4; ++j) g4[j] = V[j] * (1.0f / (cntr * ncf[j]));
                    }
                    const uint32_t l4 = label_of(g4[0], rho_occ, rho_emp) | label_of(g4[1], rho_occ, rho_emp) << 8 |
                                        label_of(g4[2], rho_occ, rho_emp) << 16 | label_of(g4[3], rho_occ, rho_emp) << 24;
                    uint8_t *lrow = lab + (size_t)o * C + c0;
                    if (full4) *reinterpret_cast<uint32_t *>(lrow) = l4;
                    else
                        for (int j = 0; j < 4 && c0 + j < C; ++j) lrow[j] = (uint8_t)(l4 >> (8 * j));
                }
            }
        }
    }
}

template <int H>
int launch_cols(vsaogm_ctx *c, const vsaogm_entropy_params *p, int band, int ldh, uint8_t *lab, cudaEvent_t *ev)
{
    // chunks of rw output rows: 20 by default (C4: 4 x 100 blocks of 128 threads, one wave of 3 blocks per SM)
    const int rw = c->entropy_rw > 0 ? c->entropy_rw : 20;
    dim3 grid((c->g_cols + 511) / 512, (band + rw - 1) / rw);
    vsa_prof_begin(c, VSAOGM_K_ENTROPY, ev);
    VSA_CUDA_TRY(vsa_launch(c, k_entropy_cols<H>, grid, dim3(128), 0, (const float *)c->d_hb, ldh, c->g_rext, c->g_rows, c->g_cols,
                            c->g_rlo, c->g_r0, band, rw, p->rho_occ, p->rho_emp, lab));
    return VSAOGM_OK;
}

template <int H>
int launch_stream(vsaogm_ctx *c, const CUtensorMap &tm, StreamArgs sa, int band, cudaEvent_t *ev)
{
    using Cfg = StCfg<H>;
    // items of rw output rows (default 16: the 2H halo rows stay a modest fraction of the
    // staged rows), taken dynamically by all resident warps
    sa.rw = c->entropy_rw > 0 ? c->entropy_rw : 16;
    sa.chunks = (band + sa.rw - 1) / sa.rw;
    sa.ctr = c->d_ent_ctr;
    const int blocks = c->num_sms * Cfg::BLOCKS_PER_SM;
    VSA_CUDA_TRY(cudaFuncSetAttribute(k_entropy_stream<H>, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::BLOCK_SMEM));
    vsa_prof_begin(c, VSAOGM_K_ENTROPY, ev);
    VSA_CUDA_TRY(vsa_launch(c, k_entropy_stream<H>, dim3(blocks), dim3(ST_WARPS * 32), (size_t)Cfg::BLOCK_SMEM, tm, sa));
    return VSAOGM_OK;
}

}  // namespace

int vsa_launch_entropy(vsaogm_ctx *c, const vsaogm_entropy_params *p, float *S, uint8_t *lab)
{
    if (c->g_estimator == 1) {
        const int H = p->half_occ > p->half_emp ? p->half_occ : p->half_emp;
        const int TW = HT + 2 * H, TH = HR + 2 * H, NMAX = (2 * H + 1) * (2 * H + 1);
        const size_t smem = 256 * HT * 2 + 4 * (size_t)(NMAX + 1) + 2 * (size_t)TH * TW;
        VSA_CUDA_TRY(cudaFuncSetAttribute(k_entropy_hist, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        const int band = c->g_r1 - c->g_r0;
        dim3 grid((c->g_cols + HT - 1) / HT, (band + HR - 1) / HR);
        cudaEvent_t ev;
        vsa_prof_begin(c, VSAOGM_K_ENTROPY, &ev);
        k_entropy_hist<<<grid, HT, smem, c->stream>>>(c->d_code, (c->g_cols + 7) / 8 * 8, c->g_rext, c->g_rows,
                                                      c->g_cols, c->g_rlo, c->g_r0, band, p->half_occ, p->half_emp,
                                                      p->disk, p->rho_occ, p->rho_emp, S, lab);
        VSA_CUDA_TRY(cudaGetLastError());
        vsa_prof_end(c, VSAOGM_K_ENTROPY, ev);
        c->launches++;
        return VSAOGM_OK;
    }
    const int H = p->half_occ > p->half_emp ? p->half_occ : p->half_emp;
    const int band = c->g_r1 - c->g_r0;
    const int ldh = (c->g_cols + 7) / 8 * 8;
    cudaEvent_t ev;
    const bool stream_k =
        p->half_occ == p->half_emp && !p->disk && H <= 4 && lab && !S && c->entropy_kernel != 1;
    if (stream_k && c->entropy_kernel != 2) {   // default: the column-walk kernel; 2: the TMA-streamed one
        int rc = VSAOGM_OK;
        switch (H) {
        case 1: rc = launch_cols<1>(c, p, band, ldh, lab, &ev); break;
        case 2: rc = launch_cols<2>(c, p, band, ldh, lab, &ev); break;
        case 3: rc = launch_cols<3>(c, p, band, ldh, lab, &ev); break;
        default: rc = launch_cols<4>(c, p, band, ldh, lab, &ev); break;
        }
        if (rc) return rc;
    } else if (stream_k) {
        // tensor map over the decoded H_b rows: dims {cols, r_ext, 2 classes}; out-of-bounds
        // boxes are zero-filled (the window clipping)
        auto fn = vsa_tmap_encode_fn();
        if (!fn) return VSAOGM_ECUDA;
        CUtensorMap tm;
        cuuint64_t dims[3] = {(cuuint64_t)c->g_cols, (cuuint64_t)c->g_rext, 2};
        cuuint64_t strides[2] = {(cuuint64_t)ldh * 4, (cuuint64_t)c->g_rext * ldh * 4};
        cuuint32_t box[3] = {(cuuint32_t)ST_W, 2 /* StCfg<H>::RS */, 2};
        cuuint32_t estr[3] = {1, 1, 1};
        if (fn(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, c->d_hb, dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return VSAOGM_ECUDA;
        StreamArgs sa;
        sa.R = c->g_rows;
        sa.C = c->g_cols;
        sa.r_lo = c->g_rlo;
        sa.r0 = c->g_r0;
        sa.band_rows = band;
        sa.strips = (c->g_cols + ST_COLS - 1) / ST_COLS;
        sa.rho_occ = p->rho_occ;
        sa.rho_emp = p->rho_emp;
        sa.lab = lab;
        int rc = VSAOGM_OK;
        switch (H) {
        case 1: rc = launch_stream<1>(c, tm, sa, band, &ev); break;
        case 2: rc = launch_stream<2>(c, tm, sa, band, &ev); break;
        case 3: rc = launch_stream<3>(c, tm, sa, band, &ev); break;
        default: rc = launch_stream<4>(c, tm, sa, band, &ev); break;
        }
        if (rc) return rc;
    } else {
        const int TW = TC + 2 * H, TH = TR + 2 * H;
        const size_t smem = sizeof(float) * (2 * (size_t)TH * TW + 2 * (size_t)TH * TC);
        dim3 grid((c->g_cols + TC - 1) / TC, (band + TR - 1) / TR);
        VSA_CUDA_TRY(cudaFuncSetAttribute(k_entropy, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        vsa_prof_begin(c, VSAOGM_K_ENTROPY, &ev);
        k_entropy<<<grid, ENT_THREADS, smem, c->stream>>>(c->d_hb, ldh, c->g_rext, c->g_rows, c->g_cols, c->g_rlo,
                                                          c->g_r0, band, p->half_occ, p->half_emp, p->disk,
                                                          p->rho_occ, p->rho_emp, S, lab);
    }
    VSA_CUDA_TRY(cudaGetLastError());
    vsa_prof_end(c, VSAOGM_K_ENTROPY, ev);
    c->launches++;
    return VSAOGM_OK;
}
