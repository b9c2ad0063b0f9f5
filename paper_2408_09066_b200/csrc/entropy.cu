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


// Box window, equal radii h1 = h0 = H <= 4 (every BASELINE config: 3x3 / 5x5 / 7x7), the
// HBM-bound hot kernel.  Persistent warps, each streaming a work item = one 128-column strip x
// `rw` output rows of the band from top to bottom:
//   * lane 0 keeps a private ring of ST_NST TMA stages in flight (cp.async.bulk.tensor.3d, box
//     136 columns x ST_RS rows x both classes, 4 halo columns on each side; the tensor map's
//     bounds are the decoded rows x grid columns, so the TMA zero-fill IS the window clipping of
//     DESIGN.md L13) on per-stage mbarriers -- no block barriers, every warp independent;
//   * each lane owns 4 adjacent columns: per staged row and class it reads its own float4,
//     gets the H neighbour columns on each side by warp shuffles (the strip's edge lanes read
//     the staged halo), forms the 4 horizontal (2H+1)-sums and keeps the last 2H+1 of them in a
//     register ring; each output row is the in-order sum of its ring (the additions and their
//     order of the generic kernel, so the result is bit-identical to it);
//   * labels leave as one 4-byte store per lane (128 B per warp row), S as float4s.
// Each staged row is read from shared memory once per class (16 B per lane); halo rows of
// neighbouring items are re-read from L2, not DRAM (items run concurrently).
constexpr int ST_RS = 4;                          // staged rows per TMA stage
constexpr int ST_NST = 4;                         // stages per warp ring
constexpr int ST_W = 136;                         // staged floats per row (4 + 128 + 4)
constexpr int ST_WARPS = 4;                       // warps per block
constexpr int ST_BLOCKS_PER_SM = 2;
constexpr int ST_STAGE_FLOATS = 2 * ST_RS * ST_W; // [class][row][col]
constexpr int ST_STAGE_BYTES = ST_STAGE_FLOATS * 4;
constexpr size_t ST_SMEM = (size_t)ST_WARPS * ST_NST * ST_STAGE_BYTES;

struct StreamArgs {
    int R, C, r_lo;            // full grid; first decoded row (tensor-map row 0)
    int r0, band_rows;         // band: full-grid rows [r0, r0 + band_rows)
    int strips, chunks, rw;    // work items = strips x chunks of rw output rows
    float rho_occ, rho_emp;
    float *S;
    uint8_t *lab;
};

__device__ __forceinline__ void tma_load_3d(void *dst, const CUtensorMap *map, uint64_t *bar, int c0, int c1, int c2)
{
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
            smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
        : "memory");
}

template <int H>
__global__ void __launch_bounds__(ST_WARPS * 32, ST_BLOCKS_PER_SM)
    k_entropy_stream(const __grid_constant__ CUtensorMap tm, const StreamArgs a)
{
    static_assert(H >= 1 && H <= 4, "halo within one float4 per side");
    constexpr int W = 2 * H + 1;
    extern __shared__ __align__(128) float sm_st[];
    __shared__ __align__(8) uint64_t bars[ST_WARPS][ST_NST];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    float *ring_smem = sm_st + (size_t)warp * ST_NST * ST_STAGE_FLOATS;
    uint64_t *bar = bars[warp];
    if (lane == 0) {
        for (int s = 0; s < ST_NST; ++s) mbar_init(&bar[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncwarp();
    const int items = a.strips * a.chunks;
    const int nwarps = gridDim.x * ST_WARPS;
    uint32_t g = 0;   // stages this warp has consumed (slot g % ST_NST, phase (g / ST_NST) & 1)
    for (int it = blockIdx.x * ST_WARPS + warp; it < items; it += nwarps) {
        const int strip = it % a.strips, chunk = it / a.strips;
        const int col0 = strip * 128;
        const int oA = chunk * a.rw;                          // band-relative output rows [oA, oB)
        const int oB = min(a.band_rows, oA + a.rw);
        const int rA = a.r0 + oA;                             // full-grid row of output oA
        const int nstaged = (oB - oA) + 2 * H;                // staged rows rA - H .. rB - 1 + H
        const int nst = (nstaged + ST_RS - 1) / ST_RS;
        auto issue = [&](int t) {                             // local stage t -> slot (g + t) % ST_NST
            const uint32_t slot = (g + t) % ST_NST;
            mbar_expect_tx(&bar[slot], ST_STAGE_BYTES);
            tma_load_3d(ring_smem + slot * ST_STAGE_FLOATS, &tm, &bar[slot], col0 - 4,
                        rA - H + t * ST_RS - a.r_lo, 0);
        };
        if (lane == 0)
            for (int t = 0; t < min(nst, ST_NST); ++t) issue(t);
        const int c0 = col0 + 4 * lane;
        int nc[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) nc[j] = min(c0 + j + H, a.C - 1) - max(c0 + j - H, 0) + 1;
        const bool cols_live = c0 < a.C;
        const bool full4 = c0 + 3 < a.C && (a.C & 3) == 0;
        float ring[2][W][4];
        for (int ib = 0; ib < nstaged; ib += W) {
#pragma unroll
            for (int u = 0; u < W; ++u) {
                const int i = ib + u;                         // staged row (ring slot u = i % W)
                if (i < nstaged) {
                    const int t = i / ST_RS, rr = i - t * ST_RS;
                    const uint32_t slot = (g + t) % ST_NST;
                    if (rr == 0) mbar_wait(&bar[slot], ((g + t) / ST_NST) & 1u);
                    const float *stage = ring_smem + slot * ST_STAGE_FLOATS;
#pragma unroll
                    for (int cls = 0; cls < 2; ++cls) {
                        const float *rp = stage + (cls * ST_RS + rr) * ST_W;
                        const float4 v = *reinterpret_cast<const float4 *>(rp + 4 + 4 * lane);
                        float4 L, Rt;
                        L.x = __shfl_up_sync(0xffffffffu, v.x, 1);
                        L.y = __shfl_up_sync(0xffffffffu, v.y, 1);
                        L.z = __shfl_up_sync(0xffffffffu, v.z, 1);
                        L.w = __shfl_up_sync(0xffffffffu, v.w, 1);
                        Rt.x = __shfl_down_sync(0xffffffffu, v.x, 1);
                        Rt.y = __shfl_down_sync(0xffffffffu, v.y, 1);
                        Rt.z = __shfl_down_sync(0xffffffffu, v.z, 1);
                        Rt.w = __shfl_down_sync(0xffffffffu, v.w, 1);
                        if (lane == 0) L = *reinterpret_cast<const float4 *>(rp);
                        if (lane == 31) Rt = *reinterpret_cast<const float4 *>(rp + 132);
                        const float x[12] = {L.x, L.y, L.z, L.w, v.x, v.y, v.z, v.w, Rt.x, Rt.y, Rt.z, Rt.w};
#pragma unroll
                        for (int j = 0; j < 4; ++j) {
                            float sh = 0.f;
#pragma unroll
                            for (int dv = -H; dv <= H; ++dv) sh += x[4 + j + dv];
                            ring[cls][u][j] = sh;
                        }
                    }
                    if (rr == ST_RS - 1 || i == nstaged - 1) {   // stage consumed: refill its slot
                        __syncwarp();
                        if (lane == 0 && t + ST_NST < nst) {
                            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                            issue(t + ST_NST);
                        }
                    }
                    if (i >= 2 * H && cols_live) {
                        const int o = oA + i - 2 * H;             // band-relative output row
                        const int row = a.r0 + o;
                        const float cntr = (float)(min(row + H, a.R - 1) - max(row - H, 0) + 1);
                        float g4[4], s14[4], s04[4];
#pragma unroll
                        for (int j = 0; j < 4; ++j) {
                            float sc[2];
#pragma unroll
                            for (int cls = 0; cls < 2; ++cls) {
                                float sv = 0.f;
#pragma unroll
                                for (int du = 0; du < W; ++du) sv += ring[cls][(u + 1 + du) % W][j];
                                sc[cls] = sv;
                            }
                            const float inv = 1.0f / (cntr * (float)nc[j]);
                            s14[j] = sc[1] * inv;
                            s04[j] = sc[0] * inv;
                            g4[j] = s14[j] - s04[j];
                        }
                        const size_t off = (size_t)o * a.C + c0;
                        if (a.lab) {
                            uint8_t l4[4];
#pragma unroll
                            for (int j = 0; j < 4; ++j) l4[j] = g4[j] >= a.rho_occ ? 1 : (g4[j] < a.rho_emp ? 0 : 2);
                            if (full4) *reinterpret_cast<uchar4 *>(a.lab + off) = make_uchar4(l4[0], l4[1], l4[2], l4[3]);
                            else
                                for (int j = 0; j < 4 && c0 + j < a.C; ++j) a.lab[off + j] = l4[j];
                        }
                        if (a.S) {
                            float *S1 = a.S + off, *S0 = a.S + (size_t)a.band_rows * a.C + off,
                                  *SG = a.S + (size_t)2 * a.band_rows * a.C + off;
                            if (full4) {
                                *reinterpret_cast<float4 *>(S1) = make_float4(s14[0], s14[1], s14[2], s14[3]);
                                *reinterpret_cast<float4 *>(S0) = make_float4(s04[0], s04[1], s04[2], s04[3]);
                                *reinterpret_cast<float4 *>(SG) = make_float4(g4[0], g4[1], g4[2], g4[3]);
                            } else {
                                for (int j = 0; j < 4 && c0 + j < a.C; ++j) {
                                    S1[j] = s14[j];
                                    S0[j] = s04[j];
                                    SG[j] = g4[j];
                                }
                            }
                        }
                    }
                }
            }
        }
        g += nst;
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
            Sc[cls] = s * (1.0f / cnt);   // as the streamed kernel: bit-identical box results
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
    const bool stream_k = p->half_occ == p->half_emp && !p->disk && H <= 4 && c->entropy_kernel != 1;
    if (stream_k) {
        // tensor map over the decoded H_b rows: dims {cols, r_ext, 2 classes}; out-of-bounds
        // boxes are zero-filled (the window clipping)
        auto fn = vsa_tmap_encode_fn();
        if (!fn) return VSAOGM_ECUDA;
        CUtensorMap tm;
        cuuint64_t dims[3] = {(cuuint64_t)c->g_cols, (cuuint64_t)c->g_rext, 2};
        cuuint64_t strides[2] = {(cuuint64_t)ldh * 4, (cuuint64_t)c->g_rext * ldh * 4};
        cuuint32_t box[3] = {(cuuint32_t)ST_W, (cuuint32_t)ST_RS, 2};
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
        sa.strips = (c->g_cols + 127) / 128;
        // one wave of work items over the resident warps; at least 16 output rows per item so
        // that the 2H halo rows stay a small fraction of the staged rows
        const int warps = c->num_sms * ST_BLOCKS_PER_SM * ST_WARPS;
        sa.rw = std::max(16, (int)(((int64_t)band * sa.strips + warps - 1) / warps));
        if (c->entropy_rw > 0) sa.rw = c->entropy_rw;
        sa.chunks = (band + sa.rw - 1) / sa.rw;
        sa.rho_occ = p->rho_occ;
        sa.rho_emp = p->rho_emp;
        sa.S = S;
        sa.lab = lab;
        const int items = sa.strips * sa.chunks;
        const int blocks = std::min((items + ST_WARPS - 1) / ST_WARPS, c->num_sms * ST_BLOCKS_PER_SM);
        vsa_prof_begin(c, VSAOGM_K_ENTROPY, &ev);
        switch (H) {
#define VSA_ST(HH)                                                                                                 \
    case HH:                                                                                                       \
        VSA_CUDA_TRY(cudaFuncSetAttribute(k_entropy_stream<HH>, cudaFuncAttributeMaxDynamicSharedMemorySize,        \
                                          (int)ST_SMEM));                                                          \
        k_entropy_stream<HH><<<blocks, ST_WARPS * 32, ST_SMEM, c->stream>>>(tm, sa);                               \
        break;
            VSA_ST(1)
            VSA_ST(2)
            VSA_ST(3)
            VSA_ST(4)
#undef VSA_ST
        }
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
