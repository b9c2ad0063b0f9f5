// nufft.cu -- the encode (K2, Eq. 9 + Eq. 5, Alg. 1 with delta = 1) as a type-3 non-uniform FFT.
//
//   pending_{c,k} += sum_{i : psi_i = c} exp(i (w^x_k x_i + w^y_k y_i)),  w = theta / l,
//   (x_i, y_i) centred on the bounds centre (PAPER.md:252-258 Eq. 9, :216-219 Eq. 5).
//
// The direct encode evaluates N x D phasors (k_encode_pairs1: 1.5 MUFU ops each).  The same sums
// are a 2-D type-3 NUFFT: points x_i (in the world box) to frequencies s_k = w_k (|s| <= pi / l).
// Following the gridding formulation (Dutt & Rokhlin; Greengard & Lee 2004; Lee & Greengard 2005):
//   1. spread: b(g) = sum_i phi(g h - x_i) on a fine grid of spacing h = pi / (sigma S) = l / 2
//      (sigma = 2, S = pi / l), Gaussian phi(u) = exp(-|u|^2 / (4 tau)), 14 x 14 cells per point,
//      accumulated in 32.32 fixed point (int64 atomics: exact, so the result does not depend on
//      the order of the additions -- the L16 reproducibility of the fp64 reductions);
//   2. B(s) = h^2 sum_g b(g) e^{i s.g h} is a type-2 NUFFT at the targets t_k = s_k h in
//      [-pi/2, pi/2]^2: pre-correct b by 1 / psi^(l) (the Gaussian psi of the interpolation),
//      zero-pad to n2 = 2^p >= 2 n1 and take a 2-D FFT (own mixed radix-4 Stockham kernels, rows
//      then columns, both classes in one complex transform), then interpolate at t_k over 13 x 13
//      grid points;
//   3. pending += B(s_k) / Phi(s_k), Phi = 4 pi tau exp(-|s|^2 tau) (the FT of phi).
// Accuracy (Gaussian gridding, msp = 6 both steps): ~1e-6 relative in l2 over k, below the fp32
// direct encode's ~1.5e-5.
// Points outside the grid (world bounds + margin) are bundled by the direct pair kernel
// (k_encode_nufft_outliers), chunk by chunk.
#include <math.h>

#include <algorithm>
#include <vector>

#include "common.cuh"
#include "fft.cuh"

namespace {

constexpr int NU_MSP = 6;               // spreading half-width: cells ix-6 .. ix+7 (14)
constexpr int NU_W = 2 * NU_MSP + 2;    // 14
constexpr int NU_MSP2 = 6;              // interpolation half-width: m0-6 .. m0+6 (13)
constexpr double NU_FIX = 4294967296.0; // 2^32: fixed-point scale of the spread grid

// ---- 1. spreading --------------------------------------------------------------------------
// The fine grid is cut into NU_TS x NU_TS tiles; a point belongs to the tile of its cell and
// spreads into the tile's window (the tile plus 6 cells before and 7 after, per axis).
// (a) k_nu_bin: class / validity, cell, tile; per-(class, tile) counts (the atomic's return
//     value is the point's slot inside its bin, warp-aggregated); outliers (support off the grid) counted per
//     chunk for the direct fallback; valid points counted per class (integer sums: exact).
// (b) k_nu_scan: exclusive prefix of the bin counts (one block).
// (c) k_nu_place: each point to its bin's range (the order inside a bin is arbitrary -- the
//     accumulation below is in integers, so the result is not).
// (d) k_nu_spread_tiles: block = (tile, class) work unit, one warp per point: the 196 weights of
//     a point (14 x 14 separable Gaussian) are added into the block's shared window with 32-bit
//     shared-memory atomics in integer fixed point (exact), then the window's nonzero cells into
//     the class's dense 32.32 fixed-point grid with 64-bit integer atomics (exact: the result does
//     not depend on the order).  The row FFT reads and re-zeroes the grid.
constexpr int NU_TS = 32;                      // tile side (cells): ~180 points per unit at C4 (16: 38; the window's zeroing and flush are per unit)
constexpr int NU_WIN = NU_TS + NU_W - 1;       // 45: window side
constexpr int NU_WST = 48;                     // window row stride (words): the half-warps' rows, 7 apart, are 16 banks apart
static_assert(NU_WST >= NU_WIN && (7 * NU_WST) % 32 >= 14 && (7 * NU_WST) % 32 <= 18, "half-warps on disjoint banks");
constexpr int NU_WOFF = NU_MSP;                // window starts 6 cells before the tile

// NU_PT points per thread in k_nu_bin / k_nu_place (their loads in flight together): 4 for large batches
// (C5's 10M points: 93 + 52 -> 64 + 40 us), 1 for small ones (C4's 204k: more blocks than SMs)
template <int NU_PT>
__global__ void __launch_bounds__(256) k_nu_bin(const float2 *__restrict__ xy, const uint8_t *__restrict__ lab, int64_t n,
                                                double cx, double cy, double lo, double inv_h, int n1, int ntx,
                                                int *__restrict__ bin_cnt, int2 *__restrict__ pkey, int64_t chunk_pts,
                                                int *__restrict__ out_cnt, double *__restrict__ pcount,
                                                int *__restrict__ bcnt, int *__restrict__ err)
{
    vsa_pdl();
    __shared__ int s_cnt[4];   // class counts: all valid points, grid points
    if (threadIdx.x < 4) s_cnt[threadIdx.x] = 0;
    __syncthreads();
    const int64_t base_i = (int64_t)blockIdx.x * (256 * NU_PT) + threadIdx.x;
    float2 v[NU_PT];
    int L[NU_PT];
#pragma unroll
    for (int p = 0; p < NU_PT; ++p) {   // coalesced: point base + 256 p + thread
        const int64_t i = base_i + 256 * p;
        v[p] = i < n ? xy[i] : make_float2(0.f, 0.f);
        L[p] = i < n ? (int)lab[i] : -1;
    }
    int my_err = 0;
    int cnt[4] = {0, 0, 0, 0};   // this thread's class counts: valid points, grid points
#pragma unroll
    for (int p = 0; p < NU_PT; ++p) {
        const int64_t i = base_i + 256 * p;
        int2 key = make_int2(-1, 0);
        if (L[p] >= 0) {
            if (L[p] > 1) my_err |= VSA_ERRBIT_LABEL;
            else if (!(isfinite(v[p].x) && isfinite(v[p].y))) my_err |= VSA_ERRBIT_NONFINITE;
            else {
                cnt[0] += L[p] == 0;
                cnt[1] += L[p] == 1;
                const int ix = (int)floor(((double)v[p].x - cx - lo) * inv_h), iy = (int)floor(((double)v[p].y - cy - lo) * inv_h);
                if (ix - NU_MSP < 0 || iy - NU_MSP < 0 || ix + NU_MSP + 1 >= n1 || iy + NU_MSP + 1 >= n1)
                    atomicAdd(&out_cnt[i / chunk_pts], 1);       // outlier: direct fallback
                else {
                    key.x = (L[p] * ntx + iy / NU_TS) * ntx + ix / NU_TS;
                    cnt[2] += L[p] == 0;
                    cnt[3] += L[p] == 1;
                }
            }
        }
        // warp-aggregated slot allocation: one atomic per distinct bin in the warp (neighbouring
        // points of a scan share bins; a hot bin would otherwise serialise thousands of atomics)
        const unsigned peers = __match_any_sync(0xffffffffu, key.x);
        if (key.x >= 0) {
            const int leader = __ffs(peers) - 1;
            const int rank = __popc(peers & ((1u << (threadIdx.x & 31)) - 1u));
            int base = 0;
            if ((int)(threadIdx.x & 31) == leader) base = atomicAdd(&bin_cnt[key.x], __popc(peers));
            base = __shfl_sync(peers, base, leader);
            key.y = base + rank;
        }
        if (i < n) pkey[i] = key;
    }
    if (my_err) atomicOr(err, my_err);
    // class counts: warp sums (integer: exact), one shared atomic per warp and counter
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const int w = __reduce_add_sync(0xffffffffu, cnt[k]);
        if ((threadIdx.x & 31) == 0 && w) atomicAdd(&s_cnt[k], w);
    }
    __syncthreads();
    if (threadIdx.x < 2 && s_cnt[threadIdx.x]) atomicAdd(&pcount[threadIdx.x], (double)s_cnt[threadIdx.x]);
    if (threadIdx.x >= 2 && threadIdx.x < 4 && s_cnt[threadIdx.x]) atomicAdd(&bcnt[threadIdx.x - 2], s_cnt[threadIdx.x]);
}

__global__ void __launch_bounds__(256) k_nu_zero(int *__restrict__ a, int na, int *__restrict__ b, int nb)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < na) a[i] = 0;
    if (i < nb) b[i] = 0;
}

// exclusive prefix of the bin counts and of the bins' work units (NU_UNIT points each): unit u
// is NU_UNIT points of the bin b with unit_off[b] <= u < unit_off[b + 1] (k_nu_spread_tiles finds b);
// *n_units = the total
constexpr int NU_UNIT = 256;
__global__ void __launch_bounds__(1024) k_nu_scan(const int *__restrict__ bin_cnt, int nbins, int *__restrict__ bin_off,
                                                  int *__restrict__ unit_off, int *__restrict__ n_units)
{
    vsa_pdl();
    // chunks of 1024 bins, one per thread (coalesced); up to CH chunks' counts loaded at once;
    // each chunk scanned by warp shuffles (two barriers) on top of the running carry
    constexpr int CH = 8;
    __shared__ int s_w[2][32], s_uw[2][32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int carry = 0, ucarry = 0;
    for (int base = 0; base < nbins; base += CH * 1024) {
        int v[CH];
#pragma unroll
        for (int q = 0; q < CH; ++q) {
            const int b = base + q * 1024 + threadIdx.x;
            v[q] = b < nbins ? __ldcg(bin_cnt + b) : 0;
        }
#pragma unroll
        for (int q = 0; q < CH; ++q) {
            if (base + q * 1024 >= nbins) break;   // block-uniform
            const int b = base + q * 1024 + threadIdx.x;
            const int nu = (v[q] + NU_UNIT - 1) / NU_UNIT;
            int inc = v[q], uinc = nu;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int t = __shfl_up_sync(0xffffffffu, inc, o), ut = __shfl_up_sync(0xffffffffu, uinc, o);
                if (lane >= o) {
                    inc += t;
                    uinc += ut;
                }
            }
            const int pb = q & 1;   // double-buffered warp totals: one barrier per chunk suffices
            if (lane == 31) {
                s_w[pb][warp] = inc;
                s_uw[pb][warp] = uinc;
            }
            __syncthreads();
            int wi = s_w[pb][lane], uwi = s_uw[pb][lane];   // every warp scans the 32 totals
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int t = __shfl_up_sync(0xffffffffu, wi, o), ut = __shfl_up_sync(0xffffffffu, uwi, o);
                if (lane >= o) {
                    wi += t;
                    uwi += ut;
                }
            }
            const int wpre = __shfl_sync(0xffffffffu, wi, (warp + 31) & 31), uwpre = __shfl_sync(0xffffffffu, uwi, (warp + 31) & 31);
            const int run = carry + inc - v[q] + (warp ? wpre : 0), urun = ucarry + uinc - nu + (warp ? uwpre : 0);
            if (b < nbins) {
                bin_off[b] = run;
                unit_off[b] = urun;
            }
            carry += __shfl_sync(0xffffffffu, wi, 31);
            ucarry += __shfl_sync(0xffffffffu, uwi, 31);
        }
    }
    if (threadIdx.x == 0) {
        bin_off[nbins] = carry;
        unit_off[nbins] = ucarry;
        *n_units = ucarry;
    }
}

template <int NU_PT>
__global__ void __launch_bounds__(256) k_nu_place(const float2 *__restrict__ xy, int64_t n, const int2 *__restrict__ pkey,
                                                  const int *__restrict__ bin_off, float2 *__restrict__ sorted)
{
    vsa_pdl();
    const int64_t base_i = (int64_t)blockIdx.x * (256 * NU_PT) + threadIdx.x;
    int2 key[NU_PT];
    float2 v[NU_PT];
    int off[NU_PT];
#pragma unroll
    for (int p = 0; p < NU_PT; ++p) {
        const int64_t i = base_i + 256 * p;
        key[p] = i < n ? pkey[i] : make_int2(-1, 0);
        v[p] = i < n ? xy[i] : make_float2(0.f, 0.f);
    }
#pragma unroll
    for (int p = 0; p < NU_PT; ++p) off[p] = key[p].x >= 0 ? bin_off[key[p].x] : 0;
    // the raw coordinates: k_nu_spread_tiles recomputes the cell with k_nu_bin's fp64 expression
#pragma unroll
    for (int p = 0; p < NU_PT; ++p)
        if (key[p].x >= 0) sorted[off[p] + key[p].y] = v[p];
}

__device__ __forceinline__ float nu_ex2(float x)
{
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

__global__ void __launch_bounds__(256) k_nu_spread_tiles(const float2 *__restrict__ sorted, const int *__restrict__ bin_off,
                                                         const int *__restrict__ unit_off,
                                                         const int *__restrict__ n_units, int ntx, int n1, double cx,
                                                         double cy, double lo, double h, double inv_h, double tau,
                                                         unsigned long long *__restrict__ grid)
{
    vsa_pdl();
    __shared__ unsigned int s_win[NU_WIN * NU_WST];   // the block's window (row stride NU_WST)
    __shared__ int s_bin;
    const int unit = blockIdx.x;
    if (unit >= *n_units) return;                     // block-uniform (the grid is an upper bound)
    // the unit's bin: the b with unit_off[b] <= unit < unit_off[b + 1] (two parallel steps: the thread
    // whose segment of the prefix array brackets the unit scans it -- no per-unit lists to build)
    {
        const int nbins = 2 * ntx * ntx, step = (nbins + 255) / 256;
        const int b0 = threadIdx.x * step, b1 = min(b0 + step, nbins);
        if (b0 < nbins && unit_off[b0] <= unit && unit < unit_off[b1]) {
            int b = b0;
            while (unit_off[b + 1] <= unit) ++b;      // < step iterations
            s_bin = b;
        }
    }
    __syncthreads();
    const int bin = s_bin;                            // (class, tile_y, tile_x)
    const int first = bin_off[bin] + (unit - unit_off[bin]) * NU_UNIT;
    const int cnt = min(NU_UNIT, bin_off[bin + 1] - first);
    // fixed point 2^20 per unit weight: a cell sums at most NU_UNIT weights <= 1 (< 2^28, no 32-bit
    // overflow); written as 32.32 fixed point (an exact shift)
    constexpr int sh = 20;
    const float qscale = (float)(1u << sh);
    for (int q = threadIdx.x; q < NU_WIN * NU_WST; q += blockDim.x) s_win[q] = 0u;
    __syncthreads();
    const int t = bin % (ntx * ntx);
    const int tx = t % ntx, ty = t / ntx;
    const int gx0 = tx * NU_TS - NU_WOFF, gy0 = ty * NU_TS - NU_WOFF;   // window origin (cells)
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    // Gaussian in cell units: phi = exp(-c u^2), c = h^2 / (4 tau), u = support index - 6 - offset.
    // Lane = support column dx (lanes 14, 15 of each half idle), half-warp = rows 7 half .. +6;
    // the row weights by the recurrence exp(-c (u+1)^2) = exp(-c u^2) r, r = exp(-c (2u + 1)),
    // r <- r exp(-2c) (Greengard & Lee's fast Gaussian gridding): 3 exponentials per lane and point.
    // in base 2: ex2.approx directly (arguments within [-30, 6]: no range guard needed)
    const float c2 = (float)(h * h / (4.0 * tau) * 1.4426950408889634);
    const float e2 = nu_ex2(-2.f * c2);
    const f32x2 e13 = pk2(e2, e2 * e2 * e2), e44 = bc2((e2 * e2) * (e2 * e2));
    const int dx = lane & 15, half = lane >> 4;
    const bool col_ok = dx < NU_W;
    const float2 *pts = sorted + first;
    // the warp's points (p = warp + 8 j): 32 at a time, one per lane, which computes the point's
    // cell with k_nu_bin's fp64 expression and its fractional offset in the cell; broadcast
    const int nmine = (cnt - warp + 7) / 8;
    for (int j0 = 0; j0 < nmine; j0 += 32) {
        const float2 raw = j0 + lane < nmine ? pts[warp + 8 * (j0 + lane)] : make_float2(0.f, 0.f);
        const double gxd = ((double)raw.x - cx - lo) * inv_h, gyd = ((double)raw.y - cy - lo) * inv_h;
        const double flx = floor(gxd), fly = floor(gyd);
        const int mcell = ((int)fly << 16) | (int)flx;       // 0 <= ix, iy < n1 <= 4096
        const float mfx = (float)(gxd - flx), mfy = (float)(gyd - fly);
        const int jn = min(32, nmine - j0);
        for (int jj = 0; jj < jn; ++jj) {
            const int cell = __shfl_sync(0xffffffffu, mcell, jj);
            const float fx = __shfl_sync(0xffffffffu, mfx, jj), fy = __shfl_sync(0xffffffffu, mfy, jj);
            const int ix = cell & 0xffff, iy = cell >> 16;
            const float ux = (float)(dx - NU_MSP) - fx, uy = (float)(7 * half - NU_MSP) - fy;
            const float wx = nu_ex2(-c2 * ux * ux) * qscale;   // the x weight carries the scale
            float wy = nu_ex2(-c2 * uy * uy), r = nu_ex2(-c2 * (2.f * uy + 1.f));
            unsigned int *wb = s_win + (iy - NU_MSP - gy0 + 7 * half) * NU_WST + (ix - NU_MSP - gx0 + dx);
            if (col_ok) {
                // the 7 rows two at a time in packed fp32x2 (the kernel is issue-bound): P = (wy_k, wy_k+1)
                // advances two rows by rho = (r_k r_k+1, r_k+1 r_k+2) = r_k^2 (e2, e2^3), rho <- rho e2^4.
                // Rounding to the nearest integer by the 1.5 * 2^23 bias (wx wy <= 2^20 < 2^22): ALU ops
                // instead of a conversion on the XU pipe; shared-memory integer atomics: exact
                const f32x2 wxb = bc2(wx), bias = bc2(12582912.f);
                f32x2 P = pk2(wy, wy * r);
                f32x2 rho = mul2(bc2(r * r), e13);
                float v0, v1;
#pragma unroll
                for (int k = 0; k < 6; k += 2) {
                    upk2(fma2(wxb, P, bias), v0, v1);
                    atomicAdd(wb + k * NU_WST, __float_as_uint(v0) - 0x4B400000u);
                    atomicAdd(wb + (k + 1) * NU_WST, __float_as_uint(v1) - 0x4B400000u);
                    P = mul2(P, rho);
                    if (k < 4) rho = mul2(rho, e44);
                }
                upk2(P, v0, v1);                     // row 6
                atomicAdd(wb + 6 * NU_WST, __float_as_uint(fmaf(wx, v0, 12582912.f)) - 0x4B400000u);
            }
        }
    }
    __syncthreads();
    // the nonzero cells (all inside the grid: a point's whole support is) into the class's
    // dense 32.32 grid: integer atomics, so the sum does not depend on the order of the units
    unsigned long long *gc = grid + (size_t)(bin / (ntx * ntx)) * n1 * n1;
    for (int q = threadIdx.x; q < NU_WIN * NU_WST; q += blockDim.x) {
        const unsigned int v = s_win[q];
        if (v) {
            const int wy = q / NU_WST, wx = q - wy * NU_WST;
            atomicAdd(gc + (size_t)(gy0 + wy) * n1 + (gx0 + wx), (unsigned long long)v << (32 - sh));
        }
    }
}

// ---- 2. FFTs ------------------------------------------------------------------------------
// Both classes go through ONE complex transform: Z = b_0 + i alpha b_1 (the grids are real), and
// the interpolation separates them by the conjugate symmetry of real transforms,
//   B_0(m) = (Z^(m) + conj Z^(-m)) / 2,   B_1(m) = (Z^(m) - conj Z^(-m)) / (2 i alpha),
// which halves the FFT work.  alpha = 2^e (exact) balances the classes' magnitudes (the fp32
// transform error is relative to |Z|): e = round(log2(n_0 / n_1)) over this batch's grid points.
__device__ __forceinline__ float nu_alpha(const int *__restrict__ bcnt)
{
    const int n0 = bcnt[0], n1 = bcnt[1];
    if (n0 <= 0 || n1 <= 0) return 1.f;
    const int e = max(-12, min(12, (int)rintf(log2f((float)n0 / (float)n1))));
    return ldexpf(1.f, e);
}

// row pass: block = one grid row gy.  Reads the row of both classes' fixed-point grids (and
// zeroes what it read: the grid is clean for the next encode), pre-corrects (psi_inv[gx]
// psi_inv[gy]), packs Z = b_0 + i alpha b_1, zero-pads to N, transforms along x, and writes the
// row-major intermediate F1[gy][mx] (compact mx; coalesced stores -- the column pass reads it
// strided, all of a thread's loads in flight together: measured 12.7 + 7.5 us with the transposed
// layout, 9.2 + 10.4 us with this one).
template <int LOGN, int T>
__global__ void __launch_bounds__(T) k_nu_rowfft(unsigned long long *__restrict__ grid, int n1,
                                                 const int *__restrict__ bcnt, const float *__restrict__ psi_inv,
                                                 const float2 *__restrict__ tw, float2 *__restrict__ f1t)
{
    vsa_pdl();
    constexpr int N = 1 << LOGN;
    extern __shared__ float2 sm_fft[];
    const int gy = blockIdx.x;
    const float py = psi_inv[gy], alpha = nu_alpha(bcnt);
    unsigned long long *row0 = grid + (size_t)gy * n1, *row1 = grid + ((size_t)n1 + gy) * n1;
    // only the frequencies the interpolation reads: |m| < K2 = N/4 + 8 (|t| <= pi/2 plus the
    // 6-point reach), stored compactly at m + K2
    constexpr int K2 = N / 4 + 8;
    fftr::fft<LOGN, T, 8>(
        sm_fft, tw,
        [&](int j, int) {
            // loads only (no store between them: the first pass's loads are all in flight together;
            // the row is re-zeroed below)
            if (j >= n1) return make_float2(0.f, 0.f);
            const unsigned long long v0 = __ldcg(row0 + j), v1 = __ldcg(row1 + j);
            const float s = __ldg(psi_inv + j) * py;
            return make_float2((float)((double)v0 * (1.0 / NU_FIX)) * s, (float)((double)v1 * (1.0 / NU_FIX)) * s * alpha);
        },
        [&](int, int m, float2 v) {
            if (m < K2) f1t[(size_t)gy * (2 * K2) + (m + K2)] = v;
            else if (m >= N - K2) f1t[(size_t)gy * (2 * K2) + (m - N + K2)] = v;
        });
    // the grid is clean for the next encode (every thread's loads of the row completed in the first pass)
    for (int j = threadIdx.x; j < n1; j += T) {
        row0[j] = 0ull;
        row1[j] = 0ull;
    }
}

// column pass: block = one (compact) x-frequency; transforms along y and writes the compact
// Z^[mx + K2][my + K2] (|mx|, |my| < K2).
template <int LOGN, int T>
__global__ void __launch_bounds__(T) k_nu_colfft(const float2 *__restrict__ f1t, int n1, const float2 *__restrict__ tw,
                                                 float2 *__restrict__ G)
{
    vsa_pdl();
    constexpr int N = 1 << LOGN;
    extern __shared__ float2 sm_fft[];
    constexpr int K2 = N / 4 + 8;
    const int cx = blockIdx.x;
    const float2 *in = f1t + cx;   // row-major F1[gy][cx]: this column's values are 2 K2 apart
    float2 *out = G + (size_t)cx * 2 * K2;
    fftr::fft<LOGN, T, 8>(
        sm_fft, tw, [&](int j, int) { return j < n1 ? __ldg(in + (size_t)j * (2 * K2)) : make_float2(0.f, 0.f); },
        [&](int, int m, float2 v) {
            if (m < K2) out[m + K2] = v;
            else if (m >= N - K2) out[m - N + K2] = v;
        });
}

// ---- 3. interpolation + deconvolution ------------------------------------------------------
// one warp per dimension k: g_c(t) = hs^2 sum_{m near t} psi(t - t_m) B_c(t_m) e^{-i n1/2 t_m}
// over the 13 x 13 grid points nearest t (the grid index l runs from 0 while the coefficients are
// centred at n1/2), B_c separated from Z^(m), Z^(-m) (above); lanes take the points in a fixed
// order and the warp sums them in a fixed tree (deterministic); then pending_c += h^2 g_c / Phi(s)
// for each class with grid points in this batch (an empty class stays exactly zero).
struct NuKpar {          // per dimension k (fixed per context: theta and the grid geometry), host-built
    int m0x, m0y;        // nearest transform grid point to t_k = s_k h
    float ftx, fty;      // offset from it in grid units, in [-1/2, 1/2]
    double scale;        // h^2 hs^2 / Phi(s_k)
};

__global__ void __launch_bounds__(256) k_nu_interp(const float2 *__restrict__ G, int logn, int n1, int D, int Dp,
                                                   const NuKpar *__restrict__ kpar, double tau2,
                                                   const float2 *__restrict__ ph, const int *__restrict__ bcnt,
                                                   double *__restrict__ pending)
{
    vsa_pdl();
    constexpr int NP = 2 * NU_MSP2 + 1;   // 13
    const int lane = threadIdx.x & 31;
    const int k = blockIdx.x * 8 + (threadIdx.x >> 5);
    if (k >= D) return;   // warp-uniform
    const int N = 1 << logn;
    const NuKpar kp = kpar[k];
    const int m0x = kp.m0x, m0y = kp.m0y;
    const float ftx = kp.ftx, fty = kp.fty;
    const float hsf = (float)(2.0 * 3.14159265358979323846 / N);
    const float inv4t2 = (float)(1.0 / (4.0 * tau2));
    const float inv2a = 0.5f / nu_alpha(bcnt);
    const int K2 = N / 4 + 8;                // compact frequency range (k_nu_colfft); |m| <= N/4 + 7
    float a0r = 0.f, a0i = 0.f, a1r = 0.f, a1i = 0.f;
#pragma unroll
    for (int it = 0; it < (NP * NP + 31) / 32; ++it) {   // all loads of the warp's points in flight
        const int idx = lane + 32 * it;
        if (idx >= NP * NP) break;
        const int dx = idx / NP, dy = idx - dx * NP;
        const int mx = m0x - NU_MSP2 + dx, my = m0y - NU_MSP2 + dy;
        const float ux = (ftx - (float)(dx - NU_MSP2)) * hsf, uy = (fty - (float)(dy - NU_MSP2)) * hsf;
        const float w = __expf(-(ux * ux + uy * uy) * inv4t2);
        const float2 px = ph[mx & (N - 1)], py = ph[my & (N - 1)];
        const float2 p = make_float2(w * (px.x * py.x - px.y * py.y), w * (px.x * py.y + px.y * py.x));
        const float2 g = G[(size_t)(mx + K2) * 2 * K2 + (my + K2)];
        const float2 gm = G[(size_t)(K2 - mx) * 2 * K2 + (K2 - my)];
        const float2 b0 = make_float2(0.5f * (g.x + gm.x), 0.5f * (g.y - gm.y));
        const float2 b1 = make_float2(inv2a * (g.y + gm.y), -inv2a * (g.x - gm.x));
        a0r += b0.x * p.x - b0.y * p.y;
        a0i += b0.x * p.y + b0.y * p.x;
        a1r += b1.x * p.x - b1.y * p.y;
        a1i += b1.x * p.y + b1.y * p.x;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        a0r += __shfl_xor_sync(0xffffffffu, a0r, o);
        a0i += __shfl_xor_sync(0xffffffffu, a0i, o);
        a1r += __shfl_xor_sync(0xffffffffu, a1r, o);
        a1i += __shfl_xor_sync(0xffffffffu, a1i, o);
    }
    if (lane == 0) {
        const double scale = kp.scale;
        if (bcnt[0] > 0) {
            double *pd = pending + 2 * (size_t)k;
            pd[0] += scale * a0r;
            pd[1] += scale * a0i;
        }
        if (bcnt[1] > 0) {
            double *pd = pending + 2 * ((size_t)Dp + k);
            pd[0] += scale * a1r;
            pd[1] += scale * a1i;
        }
    }
}

}  // namespace

// ---- plan and launch -----------------------------------------------------------------------
// grid geometry only (host): h, tau, n1, N = 2^logn; no allocation
int vsa_nufft_geometry(vsaogm_ctx *c)
{
    if (c->nu_n1) return VSAOGM_OK;
    const double S = 3.14159265358979323846 / c->l;   // |w| <= pi / l
    const double sigma = 2.0;
    const double h = 3.14159265358979323846 / (sigma * S);
    const double W = c->bounds.x_max - c->bounds.x_min, Hh = c->bounds.y_max - c->bounds.y_min;
    const double margin = 1.0 + 0.05 * std::max(W, Hh);   // metres beyond the bounds on the grid
    const double X = 0.5 * std::max(W, Hh) + margin;       // half-width of the covered square (centred)
    const double n1d = 2.0 * ceil((X + (NU_MSP + 2) * h) / h);
    if (!(n1d <= 4096.0)) return VSAOGM_EINVAL_ARG;        // N <= 8192 (shared-memory transform)
    int n1 = (int)n1d;
    int logn = 1;
    while ((1 << logn) < 2 * n1) ++logn;
    c->nu_h = h;
    c->nu_n1 = n1;
    c->nu_logn = logn;
    c->nu_lo = -(n1 / 2) * h;
    return VSAOGM_OK;
}

// encode method for a batch of n points (vsa_launch_encode): the NUFFT when its modelled time
// is below the direct pair kernel's (measured at C2 / C4 / C5: FFTs ~90 us at N = 2048 scaling
// with N^2, spreading ~60 us per 204k points, ~20 us of launches; direct ~N D / 3.5e12 s)
bool vsa_nufft_wanted(vsaogm_ctx *c, int64_t n)
{
    if (c->nslots != 2 || c->Dp < 2048 || c->enc_method == 0) return false;
    if (vsa_nufft_geometry(c)) return false;
    if (c->enc_method == 1) return true;
    const double N = (double)(1 << c->nu_logn);
    const double t_nufft = 90e-6 * (N / 2048.0) * (N / 2048.0) + 60e-6 * (double)n / 204000.0 + 20e-6;
    const double t_direct = (double)n * c->D / 3.5e12;
    return t_nufft < t_direct;
}

int vsa_nufft_plan(vsaogm_ctx *c)
{
    if (c->nu_ready) return VSAOGM_OK;
    int rc;
    if ((rc = vsa_nufft_geometry(c))) return rc;
    const double sigma = 2.0;
    const double h = c->nu_h;
    const int n1 = c->nu_n1, logn = c->nu_logn;
    const int N = 1 << logn;
    const double R = (double)N / n1;
    c->nu_tau = NU_MSP * h * h / (3.14159265358979323846 * sigma * (sigma - 0.5));
    c->nu_tau2 = 3.14159265358979323846 * NU_MSP2 / ((double)n1 * n1 * R * (R - 0.5));
    std::vector<float> psi(n1);
    for (int l = 0; l < n1; ++l) {
        const double lc = l - n1 / 2;
        psi[l] = (float)(1.0 / (sqrt(4.0 * 3.14159265358979323846 * c->nu_tau2) * exp(-lc * lc * c->nu_tau2)));
    }
    // per-k interpolation parameters (fp64 frequencies w = theta / l from the turn rates of vsaogm_create)
    std::vector<NuKpar> kpar(c->D);
    {
        const double hs = 2.0 * 3.14159265358979323846 / N;
        for (int k = 0; k < c->D; ++k) {
            const double sx = 2.0 * 3.14159265358979323846 * (c->thx[k] / (2.0 * 3.14159265358979323846 * c->l));
            const double sy = 2.0 * 3.14159265358979323846 * (c->thy[k] / (2.0 * 3.14159265358979323846 * c->l));
            const double tx = sx * h, ty = sy * h;
            kpar[k].m0x = (int)rint(tx / hs);
            kpar[k].m0y = (int)rint(ty / hs);
            kpar[k].ftx = (float)(tx / hs - kpar[k].m0x);
            kpar[k].fty = (float)(ty / hs - kpar[k].m0y);
            const double s2 = sx * sx + sy * sy;
            kpar[k].scale = h * h * hs * hs / (4.0 * 3.14159265358979323846 * c->nu_tau * exp(-s2 * c->nu_tau));
        }
    }
    std::vector<float2> tw(N), ph(N);
    for (int p = 1; p < N; p <<= 1)
        for (int k = 0; k < p; ++k) {
            const double a = 3.14159265358979323846 * k / p;   // 2 pi k / (2p)
            tw[p - 1 + k] = make_float2((float)cos(a), (float)sin(a));
        }
    for (int m = 0; m < N; ++m) {
        const double a = -2.0 * 3.14159265358979323846 * (double)(n1 / 2) * m / N;
        ph[m] = make_float2((float)cos(a), (float)sin(a));
    }
    const int ntx = (n1 + NU_TS - 1) / NU_TS;
    c->nu_ntx = ntx;
    const int nbins = 2 * ntx * ntx;
    const size_t K2 = N / 4 + 8;
    // dense fixed-point grids of both classes (zeroed once; the row FFT re-zeroes what it reads),
    // the packed transform's intermediate and compact output
    const size_t grid_bytes = 2 * (size_t)n1 * n1 * 8, f1_bytes = 2 * K2 * n1 * 8, g_bytes = 4 * K2 * K2 * 8;
    if (cudaMalloc(&c->d_nu_bins, (3 * (size_t)nbins + 5) * sizeof(int)) != cudaSuccess) return VSAOGM_ENOMEM;
    VSA_CUDA_TRY(cudaMemset(c->d_nu_bins, 0, (3 * (size_t)nbins + 5) * sizeof(int)));
    if (cudaMalloc(&c->d_nu_grid, grid_bytes) != cudaSuccess) return VSAOGM_ENOMEM;
    VSA_CUDA_TRY(cudaMemset(c->d_nu_grid, 0, grid_bytes));
    if (cudaMalloc(&c->d_nu_f1, f1_bytes) != cudaSuccess ||
        cudaMalloc(&c->d_nu_G, g_bytes) != cudaSuccess || cudaMalloc(&c->d_nu_psi, n1 * 4) != cudaSuccess ||
        cudaMalloc(&c->d_nu_tw, N * 8) != cudaSuccess || cudaMalloc(&c->d_nu_ph, N * 8) != cudaSuccess ||
        cudaMalloc(&c->d_nu_kpar, kpar.size() * sizeof(NuKpar)) != cudaSuccess)
        return VSAOGM_ENOMEM;
    VSA_CUDA_TRY(cudaMemcpy(c->d_nu_kpar, kpar.data(), kpar.size() * sizeof(NuKpar), cudaMemcpyHostToDevice));
    VSA_CUDA_TRY(cudaMemcpy(c->d_nu_psi, psi.data(), n1 * 4, cudaMemcpyHostToDevice));
    VSA_CUDA_TRY(cudaMemcpy(c->d_nu_tw, tw.data(), N * 8, cudaMemcpyHostToDevice));
    VSA_CUDA_TRY(cudaMemcpy(c->d_nu_ph, ph.data(), N * 8, cudaMemcpyHostToDevice));
    c->nu_ready = true;
    return VSAOGM_OK;
}

namespace {
template <int LOGN>
int launch_ffts(vsaogm_ctx *c, const int *bcnt)
{
    // register radix-16 passes (fft.cuh, fftr): one butterfly per thread and pass, one padded
    // shared buffer of N + N/16 values (17 KB at N = 2048; ping-pong buffers measured slower:
    // column pass 7.6 -> 8.5 us)
    constexpr int N = 1 << LOGN;
    constexpr int T = N / 16 < 32 ? 32 : N / 16;
    const size_t smem = (size_t)(N + N / 16) * sizeof(float2);
    VSA_CUDA_TRY(cudaFuncSetAttribute(k_nu_rowfft<LOGN, T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    VSA_CUDA_TRY(cudaFuncSetAttribute(k_nu_colfft<LOGN, T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    VSA_CUDA_TRY(vsa_launch(c, k_nu_rowfft<LOGN, T>, dim3(c->nu_n1), dim3(T), smem, (unsigned long long *)c->d_nu_grid, c->nu_n1,
                            bcnt, (const float *)c->d_nu_psi, (const float2 *)c->d_nu_tw, (float2 *)c->d_nu_f1));
    VSA_CUDA_TRY(vsa_launch(c, k_nu_colfft<LOGN, T>, dim3(2 * (N / 4 + 8)), dim3(T), smem, (const float2 *)c->d_nu_f1, c->nu_n1,
                            (const float2 *)c->d_nu_tw, (float2 *)c->d_nu_G));
    return VSAOGM_OK;
}
}  // namespace

int vsa_launch_encode_nufft(vsaogm_ctx *c, const float *xy, const uint8_t *lab, int64_t n, int64_t chunk_pts,
                            int chunks)
{
    int rc;
    if ((rc = vsa_nufft_plan(c))) return rc;
    if ((size_t)chunks > c->nu_out_cap) {
        if (c->d_nu_out) cudaFree(c->d_nu_out);
        if (cudaMalloc(&c->d_nu_out, chunks * sizeof(int)) != cudaSuccess) { c->d_nu_out = nullptr; c->nu_out_cap = 0; return VSAOGM_ENOMEM; }
        c->nu_out_cap = chunks;
    }
    const int ntx = c->nu_ntx, nbins = 2 * ntx * ntx;
    const size_t max_units = (size_t)n / NU_UNIT + nbins;   // sum over bins of ceil(cnt / NU_UNIT)
    if ((size_t)n > c->nu_pts_cap) {
        if (c->d_nu_key) cudaFree(c->d_nu_key);
        if (c->d_nu_sorted) cudaFree(c->d_nu_sorted);
        c->d_nu_key = c->d_nu_sorted = nullptr;
        c->nu_pts_cap = 0;
        const size_t cap = (size_t)n + (size_t)n / 4;   // headroom: batch sizes vary
        if (cudaMalloc(&c->d_nu_key, cap * sizeof(int2)) != cudaSuccess ||
            cudaMalloc(&c->d_nu_sorted, cap * sizeof(float2)) != cudaSuccess)
            return VSAOGM_ENOMEM;
        c->nu_pts_cap = cap;
    }
    // d_nu_bins: bin counts [nbins], grid-point class counts [2], bin offsets [nbins + 1], unit
    // offsets [nbins + 1], unit count
    int *bin_cnt = c->d_nu_bins, *bcnt = c->d_nu_bins + nbins, *bin_off = bcnt + 2, *unit_off = bin_off + nbins + 1;
    int *n_units = unit_off + nbins + 1;
    // one small kernel instead of two memsets (a memset may be queued on a copy engine behind a
    // pipelined host upload: the encode's start would wait for the whole batch copy)
    const int nz = std::max(chunks, nbins + 2);
    k_nu_zero<<<(nz + 255) / 256, 256, 0, c->stream>>>(c->d_nu_out, chunks, bin_cnt, nbins + 2);
    const int pt = n >= (int64_t)1 << 21 ? 4 : 1;   // points per thread of the bin / place kernels
    const unsigned pblocks = (unsigned)((n + 256 * pt - 1) / (256 * pt));
    const double inv_h = 1.0 / c->nu_h;
    VSA_CUDA_TRY(vsa_launch(c, pt == 4 ? k_nu_bin<4> : k_nu_bin<1>, dim3(pblocks), dim3(256), 0, (const float2 *)xy, lab, n, c->cx,
                            c->cy, c->nu_lo, inv_h, c->nu_n1, ntx, bin_cnt, (int2 *)c->d_nu_key, chunk_pts, c->d_nu_out,
                            c->d_pcounts, bcnt, c->d_err));
    VSA_CUDA_TRY(vsa_launch(c, k_nu_scan, dim3(1), dim3(1024), 0, (const int *)bin_cnt, nbins, bin_off, unit_off, n_units));
    VSA_CUDA_TRY(vsa_launch(c, pt == 4 ? k_nu_place<4> : k_nu_place<1>, dim3(pblocks), dim3(256), 0, (const float2 *)xy, n,
                            (const int2 *)c->d_nu_key, (const int *)bin_off, (float2 *)c->d_nu_sorted));
    VSA_CUDA_TRY(vsa_launch(c, k_nu_spread_tiles, dim3((unsigned)max_units), dim3(256), 0, (const float2 *)c->d_nu_sorted,
                            (const int *)bin_off, (const int *)unit_off, (const int *)n_units, ntx,
                            c->nu_n1, c->cx, c->cy, c->nu_lo, c->nu_h, inv_h, c->nu_tau, (unsigned long long *)c->d_nu_grid));
    VSA_CUDA_TRY(cudaGetLastError());
    switch (c->nu_logn) {
    case 8: rc = launch_ffts<8>(c, bcnt); break;
    case 9: rc = launch_ffts<9>(c, bcnt); break;
    case 10: rc = launch_ffts<10>(c, bcnt); break;
    case 11: rc = launch_ffts<11>(c, bcnt); break;
    case 12: rc = launch_ffts<12>(c, bcnt); break;
    case 13: rc = launch_ffts<13>(c, bcnt); break;
    default: rc = launch_ffts<7>(c, bcnt); break;
    }
    if (rc) return rc;
    VSA_CUDA_TRY(cudaGetLastError());
    VSA_CUDA_TRY(vsa_launch(c, k_nu_interp, dim3((c->D + 7) / 8), dim3(256), 0, (const float2 *)c->d_nu_G, c->nu_logn, c->nu_n1,
                            c->D, c->Dp, (const NuKpar *)c->d_nu_kpar, c->nu_tau2, (const float2 *)c->d_nu_ph, (const int *)bcnt,
                            c->d_pending));
    VSA_CUDA_TRY(cudaGetLastError());
    c->launches += 8;
    return VSAOGM_OK;
}
