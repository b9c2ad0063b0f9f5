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
// sums each footprint row segment directly.  Kernels: k_entropy_box4 (box,
// h <= 4, register rings, no shared memory), k_entropy_fixed (equal radii
// h <= 8, cp.async-staged tile), k_entropy (any radii).
// HBM-bound: 8 B read + 1 B written per cell.
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

__host__ __device__ constexpr int cisqrt(int t, int w = 0) { return (w + 1) * (w + 1) <= t ? cisqrt(t, w + 1) : w; }

// Equal radii h1 = h0 = H <= 8 (every BASELINE config): H and the footprint
// are compile-time, the tile is staged with 16-byte cp.async (zero-filled
// outside the decoded rows / grid columns), and each thread keeps the row
// sums of its 16 output rows (+2H) in registers: no second shared buffer,
// no barrier between the two passes.
template <int H, bool DISK>
__global__ void __launch_bounds__(ENT_THREADS) k_entropy_fixed(const float *__restrict__ hb, int ldh, int r_ext,
                                                               int R, int C, int r_lo, int r0, int band_rows,
                                                               float rho_occ, float rho_emp, float *__restrict__ S,
                                                               uint8_t *__restrict__ lab)
{
    constexpr int PADC = (H + 3) / 4 * 4;          // column halo rounded to 16 bytes
    constexpr int TW = TC + 2 * PADC;              // floats per staged row
    constexpr int TH = TR + 2 * H;
    constexpr int CH = TW / 4;                     // 16-byte chunks per staged row
    constexpr int RPT = TR / 2;                    // output rows per thread
    extern __shared__ float4 sm4[];
    float *tile = reinterpret_cast<float *>(sm4);  // [2][TH][TW]
    const int orow0 = r0 + blockIdx.y * TR;
    const int ocol0 = blockIdx.x * TC;

    for (int idx = threadIdx.x; idx < 2 * TH * CH; idx += ENT_THREADS) {
        const int cr = idx / CH, j = idx - cr * CH;
        const int cls = cr >= TH, row = cr - cls * TH;
        const int rr = orow0 - H + row;            // full-grid row
        const int gc = ocol0 - PADC + 4 * j;       // multiple of 4
        const bool ok = rr >= 0 && rr < R && rr - r_lo < r_ext && gc >= 0 && gc < C;
        const int nbytes = ok ? 4 * min(4, C - gc) : 0;
        const float *src = hb + ((size_t)cls * r_ext + (size_t)(ok ? rr - r_lo : 0)) * ldh + (ok ? gc : 0);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(tile + cr * TW + 4 * j)),
                     "l"(src), "r"(nbytes)
                     : "memory");
    }
    asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
    __syncthreads();

    const int tid = threadIdx.x & (TC - 1);
    const int half = threadIdx.x / TC;
    const int col = ocol0 + tid;
    float Sc[2][RPT];
#pragma unroll
    for (int cls = 0; cls < 2; ++cls) {
        const float *t = tile + cls * TH * TW + (half * RPT) * TW + PADC + tid;
        if (!DISK) {
            float hs[RPT + 2 * H];
#pragma unroll
            for (int i = 0; i < RPT + 2 * H; ++i) {
                float s = 0.f;
#pragma unroll
                for (int dv = -H; dv <= H; ++dv) s += t[i * TW + dv];
                hs[i] = s;
            }
#pragma unroll
            for (int r = 0; r < RPT; ++r) {
                float s = 0.f;
#pragma unroll
                for (int du = 0; du <= 2 * H; ++du) s += hs[r + du];
                Sc[cls][r] = s;
            }
        } else {
#pragma unroll
            for (int r = 0; r < RPT; ++r) {
                float s = 0.f;
#pragma unroll
                for (int du = -H; du <= H; ++du) {
                    constexpr int dummy = 0;
                    (void)dummy;
                    const int w = cisqrt(H * H - du * du);
#pragma unroll
                    for (int dv = -w; dv <= w; ++dv) s += t[(r + H + du) * TW + dv];
                }
                Sc[cls][r] = s;
            }
        }
    }
    // clipped counts (closed form) and outputs
    const int nc = min(col + H, C - 1) - max(col - H, 0) + 1;
#pragma unroll
    for (int r = 0; r < RPT; ++r) {
        const int row = orow0 + half * RPT + r;
        const int br = row - r0;
        float cnt;
        if (!DISK) {
            cnt = (float)((min(row + H, R - 1) - max(row - H, 0) + 1) * nc);
        } else {
            int n = 0;
#pragma unroll
            for (int du = -H; du <= H; ++du) {
                const int w = cisqrt(H * H - du * du);
                if (row + du >= 0 && row + du < R) n += min(col + w, C - 1) - max(col - w, 0) + 1;
            }
            cnt = (float)n;
        }
        const float inv = 1.0f / cnt;
        if (col < C && br < band_rows) {
            const float s1 = Sc[1][r] * inv, s0 = Sc[0][r] * inv;
            const float g = s1 - s0;
            const size_t o = (size_t)br * C + col;
            if (S) {
                S[o] = s1;
                S[(size_t)band_rows * C + o] = s0;
                S[(size_t)2 * band_rows * C + o] = g;
            }
            if (lab) lab[o] = g >= rho_occ ? 1 : (g < rho_emp ? 0 : 2);
        }
    }
}

// Box window, H <= 4 (the BASELINE configs' 3x3 / 5x5 / 7x7): the TR x TC tile (+ halo) of
// both classes is staged with 16-byte cp.async exactly as in k_entropy_fixed; then a thread
// owns 4 adjacent output columns of BOX_RPT rows: per staged row and class it reads the 12
// floats c0-4 .. c0+7 (three 16-byte shared loads), forms the 4 horizontal (2H+1)-sums, and
// keeps the last 2H+1 of them per column in a register ring; each output row is the in-order
// sum of its ring -- the same additions in the same order as k_entropy_fixed<H, false>, so the
// result is bit-identical, with ~4x fewer shared-memory instructions.  Labels leave as one
// 4-byte store, S as float4s.
constexpr int BOX_RPT = 4;                       // output rows per thread
constexpr int BOX_CG = TC / 4;                   // column groups (threads across)
static_assert(BOX_CG * (TR / BOX_RPT) == ENT_THREADS, "one thread per (column group, row strip)");

template <int H>
__global__ void __launch_bounds__(ENT_THREADS) k_entropy_box4(const float *__restrict__ hb, int ldh, int r_ext,
                                                             int R, int C, int r_lo, int r0, int band_rows,
                                                             float rho_occ, float rho_emp, float *__restrict__ S,
                                                             uint8_t *__restrict__ lab)
{
    static_assert(H >= 1 && H <= 4, "halo within one 16-byte chunk");
    constexpr int W = 2 * H + 1;
    constexpr int PADC = 4;
    constexpr int TW = TC + 2 * PADC;
    constexpr int TH = TR + 2 * H;
    constexpr int CH = TW / 4;
    extern __shared__ float4 sm4[];
    float *tile = reinterpret_cast<float *>(sm4);  // [2][TH][TW]
    const int orow0 = r0 + blockIdx.y * TR;
    const int ocol0 = blockIdx.x * TC;
    for (int idx = threadIdx.x; idx < 2 * TH * CH; idx += ENT_THREADS) {
        const int cr = idx / CH, j = idx - cr * CH;
        const int cls = cr >= TH, row = cr - cls * TH;
        const int rr = orow0 - H + row;
        const int gc = ocol0 - PADC + 4 * j;
        const bool ok = rr >= 0 && rr < R && rr - r_lo < r_ext && gc >= 0 && gc < C;
        const int nbytes = ok ? 4 * min(4, C - gc) : 0;
        const float *src = hb + ((size_t)cls * r_ext + (size_t)(ok ? rr - r_lo : 0)) * ldh + (ok ? gc : 0);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(tile + cr * TW + 4 * j)),
                     "l"(src), "r"(nbytes)
                     : "memory");
    }
    asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
    __syncthreads();

    const int cgi = threadIdx.x % BOX_CG, strip = threadIdx.x / BOX_CG;
    const int c0 = ocol0 + 4 * cgi;
    if (c0 >= C) return;
    int nc[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) nc[j] = min(c0 + j + H, C - 1) - max(c0 + j - H, 0) + 1;
    float ring[2][W][4];
#pragma unroll
    for (int i = 0; i < BOX_RPT + 2 * H; ++i) {
#pragma unroll
        for (int cls = 0; cls < 2; ++cls) {
            const float4 *t4 = reinterpret_cast<const float4 *>(tile + (cls * TH + strip * BOX_RPT + i) * TW + 4 * cgi);
            const float4 a = t4[0], b = t4[1], d = t4[2];   // columns c0-4 .. c0+7
            const float x[12] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w, d.x, d.y, d.z, d.w};
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                float sh = 0.f;
#pragma unroll
                for (int dv = -H; dv <= H; ++dv) sh += x[4 + j + dv];
                ring[cls][i % W][j] = sh;
            }
        }
        if (i >= 2 * H) {
            const int row = orow0 + strip * BOX_RPT + i - 2 * H;
            const int br = row - r0;
            if (br < band_rows) {
                const float cntr = (float)(min(row + H, R - 1) - max(row - H, 0) + 1);
                float g4[4], s14[4], s04[4];
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    float sc[2];
#pragma unroll
                    for (int cls = 0; cls < 2; ++cls) {
                        float sv = 0.f;
#pragma unroll
                        for (int du = 0; du < W; ++du) sv += ring[cls][(i - 2 * H + du) % W][j];
                        sc[cls] = sv;
                    }
                    const float inv = 1.0f / (cntr * (float)nc[j]);
                    s14[j] = sc[1] * inv;
                    s04[j] = sc[0] * inv;
                    g4[j] = s14[j] - s04[j];
                }
                const size_t o = (size_t)br * C + c0;
                const bool full = c0 + 3 < C && (C & 3) == 0;
                if (lab) {
                    uint8_t l4[4];
#pragma unroll
                    for (int j = 0; j < 4; ++j) l4[j] = g4[j] >= rho_occ ? 1 : (g4[j] < rho_emp ? 0 : 2);
                    if (full) *reinterpret_cast<uchar4 *>(lab + o) = make_uchar4(l4[0], l4[1], l4[2], l4[3]);
                    else
                        for (int j = 0; j < 4 && c0 + j < C; ++j) lab[o + j] = l4[j];
                }
                if (S) {
                    float *S1 = S + o, *S0 = S + (size_t)band_rows * C + o, *SG = S + (size_t)2 * band_rows * C + o;
                    if (full) {
                        *reinterpret_cast<float4 *>(S1) = make_float4(s14[0], s14[1], s14[2], s14[3]);
                        *reinterpret_cast<float4 *>(S0) = make_float4(s04[0], s04[1], s04[2], s04[3]);
                        *reinterpret_cast<float4 *>(SG) = make_float4(g4[0], g4[1], g4[2], g4[3]);
                    } else {
                        for (int j = 0; j < 4 && c0 + j < C; ++j) {
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

template <int H, bool DISK>
int launch_fixed(vsaogm_ctx *c, const vsaogm_entropy_params *p, float *S, uint8_t *lab, int ldh, dim3 grid)
{
    constexpr int PADC = (H + 3) / 4 * 4;
    const size_t smem = sizeof(float) * 2 * (TR + 2 * H) * (TC + 2 * PADC);
    VSA_CUDA_TRY(cudaFuncSetAttribute(k_entropy_fixed<H, DISK>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_entropy_fixed<H, DISK><<<grid, ENT_THREADS, smem, c->stream>>>(c->d_hb, ldh, c->g_rext, c->g_rows, c->g_cols,
                                                                     c->g_rlo, c->g_r0, c->g_r1 - c->g_r0, p->rho_occ,
                                                                     p->rho_emp, S, lab);
    return VSAOGM_OK;
}

template <bool DISK>
int dispatch_fixed(int H, vsaogm_ctx *c, const vsaogm_entropy_params *p, float *S, uint8_t *lab, int ldh, dim3 grid)
{
    switch (H) {
    case 1: return launch_fixed<1, DISK>(c, p, S, lab, ldh, grid);
    case 2: return launch_fixed<2, DISK>(c, p, S, lab, ldh, grid);
    case 3: return launch_fixed<3, DISK>(c, p, S, lab, ldh, grid);
    case 4: return launch_fixed<4, DISK>(c, p, S, lab, ldh, grid);
    case 5: return launch_fixed<5, DISK>(c, p, S, lab, ldh, grid);
    case 6: return launch_fixed<6, DISK>(c, p, S, lab, ldh, grid);
    case 7: return launch_fixed<7, DISK>(c, p, S, lab, ldh, grid);
    default: return launch_fixed<8, DISK>(c, p, S, lab, ldh, grid);
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
            Sc[cls] = s / cnt;
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
    const int TW = TC + 2 * H, TH = TR + 2 * H;
    const int band = c->g_r1 - c->g_r0;
    const int ldh = (c->g_cols + 7) / 8 * 8;
    const size_t smem = sizeof(float) * (2 * (size_t)TH * TW + 2 * (size_t)TH * TC);
    dim3 grid((c->g_cols + TC - 1) / TC, (band + TR - 1) / TR);
    const bool fixed = p->half_occ == p->half_emp && H <= 8 && c->entropy_kernel != 1;
    if (!fixed)
        VSA_CUDA_TRY(cudaFuncSetAttribute(k_entropy, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    cudaEvent_t ev;
    vsa_prof_begin(c, VSAOGM_K_ENTROPY, &ev);
    if (fixed && !p->disk && H <= 4 && c->entropy_kernel != 2) {
#define VSA_BOX(HH)                                                                                                \
    do {                                                                                                           \
        const size_t bsm = sizeof(float) * 2 * (TR + 2 * (HH)) * (TC + 8);                                          \
        VSA_CUDA_TRY(cudaFuncSetAttribute(k_entropy_box4<HH>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bsm)); \
        k_entropy_box4<HH><<<grid, ENT_THREADS, bsm, c->stream>>>(c->d_hb, ldh, c->g_rext, c->g_rows, c->g_cols,     \
                                                                  c->g_rlo, c->g_r0, band, p->rho_occ, p->rho_emp,  \
                                                                  S, lab);                                          \
    } while (0)
        switch (H) {
        case 1: VSA_BOX(1); break;
        case 2: VSA_BOX(2); break;
        case 3: VSA_BOX(3); break;
        default: VSA_BOX(4); break;
        }
#undef VSA_BOX
    } else if (fixed) {
        int rc = p->disk ? dispatch_fixed<true>(H, c, p, S, lab, ldh, grid)
                         : dispatch_fixed<false>(H, c, p, S, lab, ldh, grid);
        if (rc) return rc;
    } else {
        k_entropy<<<grid, ENT_THREADS, smem, c->stream>>>(c->d_hb, ldh, c->g_rext, c->g_rows, c->g_cols, c->g_rlo,
                                                          c->g_r0, band, p->half_occ, p->half_emp, p->disk,
                                                          p->rho_occ, p->rho_emp, S, lab);
    }
    VSA_CUDA_TRY(cudaGetLastError());
    vsa_prof_end(c, VSAOGM_K_ENTROPY, ev);
    c->launches++;
    return VSAOGM_OK;
}
