// nudecode.cu -- the decode (Eq. 11 + Born rule + H_b) as a type-1 NUFFT.
//
//   q_c(x, y) = Re sum_k conj(m_ck) exp(2 pi i (tx_k (x - cx) + ty_k (y - cy))) / (sqrt(D) ||m_c||)
//
// (Eq. 11 after the Eq. 10 normalisation; t = theta / (2 pi l) turns per
// metre; the phase origin (cx, cy) is the bounds centre, a rotation that cancels in q).  On the cells
// of a regular grid, x_j = x0 + (j + 1/2) res, this is a 2-D trigonometric sum with D off-grid
// frequencies: the decode GEMM (gemm_tc.cu) evaluates it densely (8 R C D flops); here it is a
// type-1 non-uniform FFT (Dutt & Rokhlin 1993; Greengard & Lee 2004, Gaussian gridding):
//
//   0. with centred output indices j' = j - jc, r' = r - rc (jc = C / 2, rc = R_ext / 2) and the
//      shift folded into the strengths, s_ck = a_ck e^{2 pi i (tx_k U0 + ty_k V0)}, a_ck =
//      conj(m_ck) / (sqrt(D) ||m_c||) (0 for an empty class, L8), U0 = x_jc - cx, V0 = y_rc - cy,
//      f_c(r', j') = sum_k s_ck e^{i (xi^x_k j' + xi^y_k r')},  xi = 2 pi t res  (radians per cell);
//   1. both classes in ONE complex sum whose real and imaginary parts are q_0 and q_1 (q_c = Re f_c):
//      q_0 + i q_1 = sum_k [ c_k e^{+i xi_k . (j', r')} + d_k e^{-i xi_k . (j', r')} ],
//      c_k = (s_0k + i s_1k) / 2,  d_k = (conj s_0k + i conj s_1k) / 2  (2 D points at +-xi_k);
//   2. spread: G(m) = sum_p st_p g_x(m_x h_x - xi^x_p) g_y(m_y h_y - xi^y_p) on the periodic fine
//      grid of M_x x M_y points (h = 2 pi / M, M = 2^p >= 2 x outputs: oversampling sigma >= 2),
//      Gaussian g(u) = exp(-u^2 / (4 tau)), tau = pi msp / (n^2 sigma (sigma - 1/2)), msp = 5;
//      only the band |m| <= B = ceil(max |xi| / h) + 6 is nonzero (xi <= pi res / l: B ~ M res / 2l);
//   3. F(t) = (1 / M_x M_y) sum_m G(m) e^{+2 pi i m . t / M}: a pruned 2-D FFT -- along y for each of
//      the W_x = 2 B_x + 1 band columns (zero-padded: the band is shifted to the start, the shift's
//      phase e^{-2 pi i B t / M} folded into the output factor), then along x for each decoded row;
//      only the outputs |t| < M / 4 (the centred rows / columns) are formed in the fused last stage;
//   4. deconvolve: f(r', j') = (pi / tau) e^{j'^2 tau_x + r'^2 tau_y} F(r', j'); q_0 = Re, q_1 = Im;
//      the epilogue is the GEMM's: p = min(q^2, 1) (Born rule), H_b(p) for Alg. 2
//      or the 8-bit p code of the histogram estimator, q for the band's own rows.
// Accuracy: ~1e-6 of the peak |q| (Gaussian gridding with msp = 5, fp32 transforms), against the
// fp16-operand GEMM's ~1e-4..1e-3.
//
// Kernels (one decode): k_nd_spread (block = 16 x 16 tile of the band grid; gathers the points of
// the 4 x 4 neighbouring bins in a fixed host-sorted order: deterministic, no atomics),
// k_nd_colfft (persistent over band columns), k_nd_rowfft (persistent over decoded rows).  The binning
// of the 2 D points depends only on theta and the grid geometry: it is built on the host once per
// geometry (a plan) and cached.
#include <math.h>

#include <algorithm>
#include <vector>

#include "common.cuh"
#include "fft.cuh"

namespace {

constexpr int ND_TS = 16;          // spread tile side (cells): 2 x 2 cells per thread, 64 threads per tile (10.5 us at C4; 32-cell
                                   // tiles: 14.7 us -- a point is evaluated on (side + 16)^2 cells)
constexpr int ND_BS = 8;           // point bin side (cells)
constexpr int ND_CH = 64;          // points staged per pass in the spread kernel (~34 per tile at C4: one pass)
constexpr double ND_MSP = 5.0;     // Gaussian width parameter (accuracy ~1e-6)
constexpr int ND_MARGIN = 6;       // band half-width beyond max |xi| / h (cells)
constexpr int ND_LOGN_MAX = 13;    // shared-memory transforms up to 8192 points
constexpr double kPi = 3.14159265358979323846;

struct NdPlan {
    // geometry key
    double x0 = 0, y0 = 0, res = 0;
    int cols = 0, r_lo = 0, r_ext = 0;
    // transform geometry
    int logx = 0, logy = 0, Mx = 0, My = 0;
    int Bx = 0, By = 0, Wx = 0, Wy = 0, nbx = 0, nby = 0, ntx = 0, nty = 0;
    int jc = 0, rc = 0, ldt = 0;
    double U0 = 0, V0 = 0;
    float ax = 0, ay = 0;              // h^2 / (4 tau) per axis
    int *d_kid = nullptr;              // point ids (k, or D + k for -xi_k) in bin order [2 D]
    float2 *d_pos = nullptr;           // per slot: position relative to its bin's first cell (cells)
    int *d_binx = nullptr;             // per slot: its bin's column
    int *d_bin_off = nullptr;          // [nbx nby + 1]
    float2 *d_Px = nullptr;            // output factors per column [cols]
    float2 *d_Py = nullptr;            // output factors per decoded row [r_ext]
    int64_t used = 0;                  // LRU tick
};

// per decode: the strength of every point, in bin order (slot s holds point kid[s]: k, or D + k
// for the mirrored point at -xi_k)
__global__ void __launch_bounds__(256) k_nd_strength(const int *__restrict__ kid, int npts, int D, int Dp,
                                                     const double2 *__restrict__ m, const double *__restrict__ mscale,
                                                     double inv_D, const double *__restrict__ tx_t,
                                                     const double *__restrict__ ty_t, double U0, double V0,
                                                     float2 *__restrict__ st)
{
    vsa_pdl();
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= npts) return;
    const int pt = kid[s];
    const bool neg = pt >= D;
    const int k = neg ? pt - D : pt;
    const double t = tx_t[k] * U0 + ty_t[k] * V0;   // turns of the centring shift
    const float f = (float)(t - rint(t));            // in [-1/2, 1/2]
    float sn, cs;
    sincospif(2.f * f, &sn, &cs);
    const double sc0 = mscale[0] * inv_D, sc1 = mscale[1] * inv_D;   // 1 / (sqrt(D) ||m_c||), 0 if empty
    const double2 m0 = m[k], m1 = m[Dp + k];
    // a_c = conj(m_c) sc_c; s_c = a_c e^{i phi}
    const float a0r = (float)(m0.x * sc0), a0i = (float)(-m0.y * sc0);
    const float a1r = (float)(m1.x * sc1), a1i = (float)(-m1.y * sc1);
    const float s0r = a0r * cs - a0i * sn, s0i = a0r * sn + a0i * cs;
    const float s1r = a1r * cs - a1i * sn, s1i = a1r * sn + a1i * cs;
    // c = (s0 + i s1) / 2 at +xi; d = (conj s0 + i conj s1) / 2 at -xi
    st[s] = neg ? make_float2(0.5f * (s0r + s1i), 0.5f * (s1r - s0i)) : make_float2(0.5f * (s0r - s1i), 0.5f * (s0i + s1r));
}

struct NdSpread {
    const float2 *st;        // strengths per slot
    const float2 *pos;       // position per slot relative to its bin's first cell (cells, fp32)
    const int *binx;         // bin column per slot
    const int *bin_off;      // [nbx nby + 1]
    int Wx, Wy, nbx, nby;
    float ax, ay;            // h^2 / (4 tau)
    float2 *Gt;              // compact band grid, x-major: Gt[ux][uy]
};

// block = one ND_TS x ND_TS tile of the band grid (16 x 16), 2 x 2 cells per thread (x = tx, tx + ND_TS/2;
// y = ty, ty + ND_TS/2); gathers the points binned (8 x 8 bins) within 8 cells of it -- the bins covering
// [ND_TS b - 8, ND_TS b + ND_TS + 8) per axis (4 x 4 of them), one contiguous slot range per bin row, where
// a point farther than 8 cells has weight < e^-31 --, up to ND_CH per pass.  One thread per staged point
// computes its position relative to the tile (bin column from the plan: no search); then all threads
// compute the ND_TS x-weights g_x and the ND_TS strength-scaled y-weights h_y = g_y st of every staged
// point, and every thread sums g_x[q][x] h_y[q][y] for its four cells over the points in slot order
// (deterministic).  ~34 points per tile at C4, 1936 blocks of 64 threads.
constexpr int ND_NT = ND_TS * ND_TS / 4;   // threads per tile: 2 x 2 cells each
__global__ void __launch_bounds__(ND_NT, 1024 / ND_NT) k_nd_spread(const __grid_constant__ NdSpread p)
{
    vsa_pdl_launch();
    constexpr int CH = ND_CH, NB = ND_TS / ND_BS + 2;   // staged points per pass; bin rows / columns gathered
    constexpr int HT = ND_TS / 2;                       // a thread's cells: x = cxl, cxl + HT; y = cyl, cyl + HT
    __shared__ float2 s_st[CH];
    __shared__ float2 s_u[CH];   // the point's position relative to this tile's first cell
    __shared__ float s_gx[CH][ND_TS];
    __shared__ float2 s_hy[CH][ND_TS];
    const int bx = blockIdx.x, by = blockIdx.y, tid = threadIdx.x;
    const int cxl = tid / HT, cyl = tid % HT;   // consecutive threads = consecutive rows (contiguous stores)
    constexpr int BPT = ND_TS / ND_BS;          // bins per tile side
    const int xb0 = max(BPT * bx - 1, 0), xb1 = min(BPT * bx + BPT, p.nbx - 1);
    int beg[NB], len[NB], total = 0;
#pragma unroll
    for (int r = 0; r < NB; ++r) {
        const int yb = BPT * by - 1 + r;
        const bool in = yb >= 0 && yb < p.nby;
        beg[r] = in ? __ldg(p.bin_off + yb * p.nbx + xb0) : 0;
        len[r] = in ? __ldg(p.bin_off + yb * p.nbx + xb1 + 1) - beg[r] : 0;
        total += len[r];
    }
    vsa_pdl_wait();   // the plan's bin offsets above are not the predecessor's output (the strengths are)
    float2 acc[2][2] = {{make_float2(0.f, 0.f), make_float2(0.f, 0.f)}, {make_float2(0.f, 0.f), make_float2(0.f, 0.f)}};
    for (int c0 = 0; c0 < total; c0 += CH) {
        const int nc = min(CH, total - c0);
        if (c0) __syncthreads();   // the previous pass is consumed
        for (int t = tid; t < nc; t += ND_NT) {
            int i = c0 + t, slot = 0, yb = 0;
            bool found = false;
#pragma unroll
            for (int r = 0; r < NB; ++r) {   // the bin row of staged point i (registers only)
                if (!found && i < len[r]) {
                    slot = beg[r] + i;
                    yb = BPT * by - 1 + r;
                    found = true;
                }
                i -= len[r];
            }
            const float2 ps = __ldg(p.pos + slot);
            const int xbp = __ldg(p.binx + slot);
            s_u[t] = make_float2((float)(xbp * ND_BS - bx * ND_TS) + ps.x, (float)(yb * ND_BS - by * ND_TS) + ps.y);
            s_st[t] = __ldg(p.st + slot);
        }
        __syncthreads();
        for (int e = tid; e < nc * 2 * ND_TS; e += ND_NT) {
            const int q = e / (2 * ND_TS), r = e % (2 * ND_TS);
            const float2 u = s_u[q];
            if (r < ND_TS) {
                const float d = (float)r - u.x;
                s_gx[q][r] = __expf(-d * d * p.ax);
            } else {
                const float d = (float)(r - ND_TS) - u.y;
                const float g = __expf(-d * d * p.ay);
                const float2 st = s_st[q];
                s_hy[q][r - ND_TS] = make_float2(g * st.x, g * st.y);
            }
        }
        __syncthreads();
#pragma unroll 4
        for (int q = 0; q < nc; ++q) {   // four independent accumulator pairs, each summed in slot order
            const float g0 = s_gx[q][cxl], g1 = s_gx[q][cxl + HT];
            const float2 h0 = s_hy[q][cyl], h1 = s_hy[q][cyl + HT];
            acc[0][0].x = fmaf(g0, h0.x, acc[0][0].x);
            acc[0][0].y = fmaf(g0, h0.y, acc[0][0].y);
            acc[0][1].x = fmaf(g0, h1.x, acc[0][1].x);
            acc[0][1].y = fmaf(g0, h1.y, acc[0][1].y);
            acc[1][0].x = fmaf(g1, h0.x, acc[1][0].x);
            acc[1][0].y = fmaf(g1, h0.y, acc[1][0].y);
            acc[1][1].x = fmaf(g1, h1.x, acc[1][1].x);
            acc[1][1].y = fmaf(g1, h1.y, acc[1][1].y);
        }
    }
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int b = 0; b < 2; ++b) {
            const int ux = bx * ND_TS + cxl + HT * a, uy = by * ND_TS + cyl + HT * b;
            if (ux < p.Wx && uy < p.Wy) p.Gt[(size_t)ux * p.Wy + uy] = acc[a][b];
        }
}

__device__ __forceinline__ float2 cmulf(float2 a, float2 b)
{
    return make_float2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}

// transforms along y of the band columns (fftr::fft: register radix-16 passes), persistent over
// columns ux = blockIdx.x, += gridDim.x; output rows r in [0, r_ext) (r' = r - rc, the centred modes
// |r'| < M / 4), times Py[r] (each thread's rows are fixed: their factors are loaded once)
template <int LOGN, int T, int NZ, bool DB>
__global__ void __launch_bounds__(T, (768 / T < 1 ? 1 : 768 / T)) k_nd_colfft(const float2 *__restrict__ Gt, int Wx, int Wy,
                                                                           const float2 *__restrict__ tw,
                                                                           const float2 *__restrict__ Py, int r_ext, int rc,
                                                                           int ldt, float2 *__restrict__ Tt)
{
    vsa_pdl_launch();
    constexpr int N = 1 << LOGN, NS = N / 16;
    extern __shared__ float2 sm_fft[];
    const int j = threadIdx.x;
    float2 py[16];
    int rq[16];
#pragma unroll
    for (int q = 0; q < 16; ++q) {
        const int m = j + q * NS;
        const int r = rc + (m < N / 2 ? m : m - N);
        rq[q] = (j < NS && (q < 4 || q >= 12) && r >= 0 && r < r_ext) ? r : -1;
        py[q] = rq[q] >= 0 ? __ldg(Py + r) : make_float2(0.f, 0.f);
    }
    vsa_pdl_wait();   // the plan's factors above are not the predecessor's output
    for (int ux = blockIdx.x; ux < Wx; ux += gridDim.x) {
        const float2 *in = Gt + (size_t)ux * Wy;
        float2 *out = Tt + (size_t)ux * ldt;
        if (!(DB && fftr::chained<LOGN>())) __syncthreads();   // the previous column's transform consumed the buffer
        fftr::fft<LOGN, T, NZ, true, DB, true>(
            sm_fft, tw, [&](int i, int) { return i < Wy ? __ldg(in + i) : make_float2(0.f, 0.f); },
            [&](int q, int, float2 v) {
                if (rq[q] >= 0) out[rq[q]] = cmulf(py[q], v);
            });
    }
}

struct NdEpi {
    const double *mscale;   // sqrt(D) / ||m_c|| [2]: 0 for an empty class
    float *hb;        // hb[(c * r_ext + row) * ldh + col]
    uint8_t *code;    // histogram estimator: 8-bit p code at the same index (hb unused)
    int ldh, r_ext;
    float *q;         // q[(c * band_rows + row + q_off) * cols + col] for band rows, or null
    int q_off, band_rows, cols;
};

__device__ __forceinline__ float nd_hb_of_p(float p)
{
    // binary entropy in bits of p in [0, 1], 0 log 0 = 0, branch-free with MUFU log2:
    // -p log2 p + (1 - p) L, L = -log2(1 - p).  For p < 1/32, L = (p + p^2/2 + p^3/3 + p^4/4) / ln 2
    // (truncation p^5/5: < 6e-8 of H_b): 1 - p in fp32 would lose log2(1/p) bits of p, the
    // cancellation log1pf avoids in the GEMM epilogue.  The clamps make 0 x log2(0) = 0 x finite.
    const float lp = __log2f(fmaxf(p, 1e-37f));
    const float om = 1.f - p;
    const float ser = p * fmaf(p, fmaf(p, fmaf(p, 0.36067376f, 0.48089835f), 0.72134752f), 1.44269504f);
    const float lg = -__log2f(fmaxf(om, 1e-37f));
    const float L = p < 0.03125f ? ser : lg;
    return fmaf(om, L, -p * lp);
}

__device__ __forceinline__ uint8_t nd_code8(float p)
{
    const int c = __float2int_rd(__fadd_rn(__fmul_rn(p, 255.0f), 0.5f));
    return (uint8_t)min(255, max(0, c));
}

// transforms along x of the decoded rows, persistent over rows row = blockIdx.x, += gridDim.x; the
// first pass reads the column-transformed Tt[ux][row] (strided: neighbouring rows, on other blocks,
// share the sectors in L2); thread j < N / 16 holds the last pass's outputs m = j + q N / 16, of which
// the centred ones (q < 4: j' = m, q >= 12: j' = m - N) are columns col0 + off_s, col0 = jc + j,
// off_s = (s < 4 ? s : s - 8) N / 16, s = 0..7: each thread's columns are fixed (their factors Px are
// loaded once, their validity is a bit mask) and every store address is one per-row pointer plus a
// compile-time offset.  FAST: H_b only (no q output, no histogram codes) -- the streaming step.
template <int LOGN, int T, int NZ, bool FAST, bool DB>
__global__ void __launch_bounds__(T, (768 / T < 1 ? 1 : 768 / T)) k_nd_rowfft(const float2 *__restrict__ Tt, int ldt, int Wx,
                                                                           const float2 *__restrict__ tw,
                                                                           const float2 *__restrict__ Px, int cols, int jc,
                                                                           const NdEpi e)
{
    vsa_pdl_launch();
    constexpr int N = 1 << LOGN, NS = N / 16;
    extern __shared__ float2 sm_fft[];
    const int j = threadIdx.x;
    const int col0 = jc + j;
    float2 px[8];
    unsigned ok = 0;
#pragma unroll
    for (int s = 0; s < 8; ++s) {
        const int col = col0 + (s < 4 ? s : s - 8) * NS;
        const bool v = j < NS && col >= 0 && col < cols;
        px[s] = v ? __ldg(Px + col) : make_float2(0.f, 0.f);
        ok |= (unsigned)v << s;
    }
    vsa_pdl_wait();   // the plan's factors above are not the predecessor's output
    // an empty class decodes to exactly 0 (L8), not to the other class's transform rounding: bit masks
    const unsigned live0 = e.mscale[0] != 0.0 ? 0xffffffffu : 0u, live1 = e.mscale[1] != 0.0 ? 0xffffffffu : 0u;
    const size_t cls_h = (size_t)e.r_ext * e.ldh, cls_q = (size_t)e.band_rows * e.cols;
    // a pruned radix-16 first pass reads NZ <= 4 values per thread: the next row's are loaded
    // before this row's passes (the strided loads' latency is hidden behind a whole transform)
    constexpr bool PF = (LOGN & 3) == 0 && NZ <= 4;
    auto ld = [&](int i, int row) { return i < Wx ? __ldg(Tt + (size_t)i * ldt + row) : make_float2(0.f, 0.f); };
    float2 nxt[PF ? NZ : 1], cur[PF ? NZ : 1];
    if (PF) {
#pragma unroll
        for (int r = 0; r < NZ; ++r) nxt[r] = ld(j + r * NS, blockIdx.x);
    }
    for (int row = blockIdx.x; row < e.r_ext; row += gridDim.x) {
        if (PF) {
            const int nrow = row + gridDim.x;
#pragma unroll
            for (int r = 0; r < NZ; ++r) {
                cur[r] = nxt[r];
                if (nrow < e.r_ext) nxt[r] = ld(j + r * NS, nrow);
            }
        }
        // per-row pointers at this thread's column col0 (class 0; class 1 at + cls_*)
        float *h0 = e.hb + (size_t)row * e.ldh + col0, *h1 = h0 + cls_h;
        uint8_t *c0 = e.code + (size_t)row * e.ldh + col0, *c1 = c0 + cls_h;
        const int br = row + e.q_off;
        float *q0 = (!FAST && e.q && br >= 0 && br < e.band_rows) ? e.q + (size_t)br * e.cols + col0 : nullptr;
        float *q1 = q0 + cls_q;
        if (!(DB && fftr::chained<LOGN>())) __syncthreads();   // the previous row's transform consumed the buffer
        fftr::fft<LOGN, T, NZ, true, DB, true>(
            sm_fft, tw, [&](int i, int slot) { return PF ? cur[PF ? slot : 0] : ld(i, row); },
            [&](int qi, int, float2 v) {
                const int s = qi < 4 ? qi : qi - 8;              // qi in {0..3, 12..15} (ENDS)
                const int off = (qi < 4 ? qi : qi - 16) * NS;    // compile time after unrolling
                if (!(ok >> s & 1)) return;
                const float2 g = cmulf(px[s], v);
                const float qa = __uint_as_float(__float_as_uint(g.x) & live0), qb = __uint_as_float(__float_as_uint(g.y) & live1);
                const float pa = fminf(qa * qa, 1.f), pb = fminf(qb * qb, 1.f);   // Born rule
                if (FAST || !e.code) {
                    h0[off] = nd_hb_of_p(pa);
                    h1[off] = nd_hb_of_p(pb);
                } else {
                    c0[off] = nd_code8(pa);
                    c1[off] = nd_code8(pb);
                }
                if (!FAST && q0) {
                    q0[off] = qa;
                    q1[off] = qb;
                }
            });
    }
}

int nd_grow(void **p, size_t *cap, size_t need)
{
    if (need <= *cap) return VSAOGM_OK;
    if (*p) cudaFree(*p);
    *p = nullptr;
    *cap = 0;
    if (cudaMalloc(p, need) != cudaSuccess) { *p = nullptr; return VSAOGM_ENOMEM; }
    *cap = need;
    return VSAOGM_OK;
}

int ilog2_ceil(int64_t v)
{
    int l = 0;
    while (((int64_t)1 << l) < v) ++l;
    return l;
}

void free_plan(NdPlan *p)
{
    if (!p) return;
    void *ptrs[] = {p->d_kid, p->d_pos, p->d_binx, p->d_bin_off, p->d_Px, p->d_Py};
    for (void *q : ptrs)
        if (q) cudaFree(q);
    delete p;
}

// the geometry of a decode (no allocation); false if the NUFFT does not apply
bool nd_geometry(const vsaogm_ctx *c, double x0, double y0, double res, int cols, int r_lo, int r_ext, NdPlan &P)
{
    if (c->nslots != 2 || cols < 1 || r_ext < 1) return false;
    P.x0 = x0;
    P.y0 = y0;
    P.res = res;
    P.cols = cols;
    P.r_lo = r_lo;
    P.r_ext = r_ext;
    P.logx = std::max(8, ilog2_ceil(2 * (int64_t)cols));
    P.logy = std::max(8, ilog2_ceil(2 * (int64_t)r_ext));
    if (P.logx > ND_LOGN_MAX || P.logy > ND_LOGN_MAX) return false;
    P.Mx = 1 << P.logx;
    P.My = 1 << P.logy;
    double amx = 0.0, amy = 0.0;   // max |turns per metre|
    for (int k = 0; k < c->D; ++k) {
        amx = std::max(amx, fabs(c->thx[k] / (2.0 * kPi * c->l)));
        amy = std::max(amy, fabs(c->thy[k] / (2.0 * kPi * c->l)));
    }
    P.Bx = (int)ceil(amx * res * P.Mx) + ND_MARGIN;
    P.By = (int)ceil(amy * res * P.My) + ND_MARGIN;
    P.Wx = 2 * P.Bx + 1;
    P.Wy = 2 * P.By + 1;
    if (P.Wx > P.Mx / 2 || P.Wy > P.My / 2) return false;   // band wider than the zero-padded half
    P.nbx = (P.Wx + ND_BS - 1) / ND_BS;   // point bins
    P.nby = (P.Wy + ND_BS - 1) / ND_BS;
    P.ntx = (P.Wx + ND_TS - 1) / ND_TS;   // spread tiles
    P.nty = (P.Wy + ND_TS - 1) / ND_TS;
    P.jc = cols / 2;
    P.rc = r_ext / 2;
    P.ldt = (r_ext + 3) / 4 * 4;
    P.U0 = x0 + ((double)P.jc + 0.5) * res - c->cx;
    P.V0 = y0 + ((double)(r_lo + P.rc) + 0.5) * res - c->cy;
    return true;
}

double nd_tau(int n, int M) { const double s = (double)M / n; return kPi * ND_MSP / ((double)n * n * s * (s - 0.5)); }

int nd_build(vsaogm_ctx *c, NdPlan &P)
{
    const int D = c->D;
    const double sx = P.res * P.Mx, sy = P.res * P.My;
    const int nb = P.nbx * P.nby;
    std::vector<int> bin(2 * (size_t)D), cnt(nb + 1, 0);
    std::vector<double> fxa(2 * (size_t)D), fya(2 * (size_t)D);
    for (int pt = 0; pt < 2 * D; ++pt) {
        const int k = pt % D;
        const double sg = pt < D ? 1.0 : -1.0;
        // fine-grid position in cells from the band's first cell (the device's turns per metre,
        // computed the same way as in vsaogm_create)
        const double fx = sg * (c->thx[k] / (2.0 * kPi * c->l)) * sx + P.Bx, fy = sg * (c->thy[k] / (2.0 * kPi * c->l)) * sy + P.By;
        fxa[pt] = fx;
        fya[pt] = fy;
        const int ux = std::min(P.Wx - 1, std::max(0, (int)floor(fx)));
        const int uy = std::min(P.Wy - 1, std::max(0, (int)floor(fy)));
        bin[pt] = (uy / ND_BS) * P.nbx + ux / ND_BS;
        cnt[bin[pt] + 1]++;
    }
    for (int b = 0; b < nb; ++b) cnt[b + 1] += cnt[b];
    std::vector<int> off(cnt.begin(), cnt.end()), kid(2 * (size_t)D);
    std::vector<float2> pos(2 * (size_t)D);
    std::vector<int> binx(2 * (size_t)D);
    for (int pt = 0; pt < 2 * D; ++pt) {   // stable: ascending point id per bin
        const int s = off[bin[pt]]++;
        kid[s] = pt;
        const int bxp = bin[pt] % P.nbx, byp = bin[pt] / P.nbx;
        pos[s] = make_float2((float)(fxa[pt] - ND_BS * bxp), (float)(fya[pt] - ND_BS * byp));
        binx[s] = bxp;
    }
    const double tx_ = nd_tau(P.cols, P.Mx), ty_ = nd_tau(P.r_ext, P.My);
    const double hx = 2.0 * kPi / P.Mx, hy = 2.0 * kPi / P.My;
    P.ax = (float)(hx * hx / (4.0 * tx_));
    P.ay = (float)(hy * hy / (4.0 * ty_));
    std::vector<float2> px(P.cols), py(P.r_ext);
    for (int j = 0; j < P.cols; ++j) {
        const double jp = j - P.jc;
        const double mag = sqrt(kPi / tx_) * exp(jp * jp * tx_) / P.Mx;
        // e^{-2 pi i B j' / M} with the integer product reduced exactly
        const double turns = (double)(((int64_t)P.Bx * (int64_t)(j - P.jc)) % P.Mx) / P.Mx;
        px[j] = make_float2((float)(mag * cos(-2.0 * kPi * turns)), (float)(mag * sin(-2.0 * kPi * turns)));
    }
    for (int r = 0; r < P.r_ext; ++r) {
        const double rp = r - P.rc;
        const double mag = sqrt(kPi / ty_) * exp(rp * rp * ty_) / P.My;
        const double turns = (double)(((int64_t)P.By * (int64_t)(r - P.rc)) % P.My) / P.My;
        py[r] = make_float2((float)(mag * cos(-2.0 * kPi * turns)), (float)(mag * sin(-2.0 * kPi * turns)));
    }
    if (cudaMalloc(&P.d_kid, kid.size() * sizeof(int)) != cudaSuccess ||
        cudaMalloc(&P.d_pos, pos.size() * sizeof(float2)) != cudaSuccess ||
        cudaMalloc(&P.d_binx, binx.size() * sizeof(int)) != cudaSuccess ||
        cudaMalloc(&P.d_bin_off, cnt.size() * sizeof(int)) != cudaSuccess ||
        cudaMalloc(&P.d_Px, px.size() * sizeof(float2)) != cudaSuccess ||
        cudaMalloc(&P.d_Py, py.size() * sizeof(float2)) != cudaSuccess)
        return VSAOGM_ENOMEM;
    VSA_CUDA_TRY(cudaMemcpy(P.d_kid, kid.data(), kid.size() * sizeof(int), cudaMemcpyHostToDevice));
    VSA_CUDA_TRY(cudaMemcpy(P.d_pos, pos.data(), pos.size() * sizeof(float2), cudaMemcpyHostToDevice));
    VSA_CUDA_TRY(cudaMemcpy(P.d_binx, binx.data(), binx.size() * sizeof(int), cudaMemcpyHostToDevice));
    VSA_CUDA_TRY(cudaMemcpy(P.d_bin_off, cnt.data(), cnt.size() * sizeof(int), cudaMemcpyHostToDevice));
    VSA_CUDA_TRY(cudaMemcpy(P.d_Px, px.data(), px.size() * sizeof(float2), cudaMemcpyHostToDevice));
    VSA_CUDA_TRY(cudaMemcpy(P.d_Py, py.data(), py.size() * sizeof(float2), cudaMemcpyHostToDevice));
    return VSAOGM_OK;
}

// the cached plan of this geometry (at most VSA_ND_PLANS; the least recently used is replaced)
int nd_plan(vsaogm_ctx *c, double x0, double y0, double res, int cols, int r_lo, int r_ext, NdPlan **out)
{
    ++c->nd_tick;
    for (int i = 0; i < c->nd_nplans; ++i) {
        NdPlan *p = static_cast<NdPlan *>(c->nd_plans[i]);
        if (p->x0 == x0 && p->y0 == y0 && p->res == res && p->cols == cols && p->r_lo == r_lo && p->r_ext == r_ext) {
            p->used = c->nd_tick;
            *out = p;
            return VSAOGM_OK;
        }
    }
    NdPlan G;
    if (!nd_geometry(c, x0, y0, res, cols, r_lo, r_ext, G)) return VSAOGM_EINVAL_ARG;
    if (!c->d_nd_tw) {   // universal twiddle table (fft.cuh): tw[p - 1 + k] = e^{i pi k / p}
        const int n = 1 << ND_LOGN_MAX;
        std::vector<float2> tw(n);
        for (int p = 1; p < n; p <<= 1)
            for (int k = 0; k < p; ++k) {
                const double a = kPi * k / p;
                tw[p - 1 + k] = make_float2((float)cos(a), (float)sin(a));
            }
        if (cudaMalloc(&c->d_nd_tw, n * sizeof(float2)) != cudaSuccess) { c->d_nd_tw = nullptr; return VSAOGM_ENOMEM; }
        VSA_CUDA_TRY(cudaMemcpy(c->d_nd_tw, tw.data(), n * sizeof(float2), cudaMemcpyHostToDevice));
    }
    int slot = c->nd_nplans;
    if (slot == VSA_ND_PLANS) {   // evict the least recently used plan (its buffers may be in flight)
        slot = 0;
        for (int i = 1; i < VSA_ND_PLANS; ++i)
            if (static_cast<NdPlan *>(c->nd_plans[i])->used < static_cast<NdPlan *>(c->nd_plans[slot])->used) slot = i;
        VSA_CUDA_TRY(cudaDeviceSynchronize());
        free_plan(static_cast<NdPlan *>(c->nd_plans[slot]));
        c->nd_plans[slot] = nullptr;
    } else {
        ++c->nd_nplans;
    }
    NdPlan *p = new NdPlan(G);
    c->nd_plans[slot] = p;
    int rc = nd_build(c, *p);
    if (rc) {
        free_plan(p);
        c->nd_plans[slot] = c->nd_plans[--c->nd_nplans];
        c->nd_plans[c->nd_nplans] = nullptr;
        return rc;
    }
    p->used = c->nd_tick;
    *out = p;
    return VSAOGM_OK;
}

// nonzero input groups of N / 16 values (the first radix-16 pass skips the others), rounded up
// to an instantiated count (transforms whose first pass is radix 16: LOGN = 8, 12)
int nz_of(int W, int logn)
{
    if ((logn & 3) > 1) return 16;
    // sizes 16^p: groups of N / 16 inputs; sizes 2 x 16^p: the skipped radix-2 pass doubles every input
    // (fft.cuh, ZP), so a group holds N / 32 distinct ones
    const int per = (logn & 3) == 0 ? (1 << logn) / 16 : (1 << logn) / 32;
    const int g = (W + per - 1) / per;
    return g <= 3 ? 3 : g <= 4 ? 4 : g <= 8 ? 8 : 16;
}

template <typename K>
int persistent_grid(vsaogm_ctx *c, K kernel, int T, size_t smem, int work)
{
    int per_sm = 0;
    VSA_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, T, smem));
    if (c->nd_bps > 0) per_sm = std::min(per_sm, c->nd_bps);
    return std::max(1, std::min(work, c->num_sms * std::max(1, per_sm)));
}

template <int LOGN, int NZ>
int launch_colfft_nz(vsaogm_ctx *c, const NdPlan &P)
{
    constexpr int N = 1 << LOGN;
    constexpr int T = N / 16 < 32 ? 32 : N / 16;
    // ping-pong buffers (fft.cuh DB: one barrier per pass) measured slower -- 209 KB of shared memory
    // per SM leaves no L1 for the twiddle and Tt loads (row pass 30.4 -> 37.4 us at C4): off
    constexpr bool DB = false;
    const size_t smem = (size_t)(N + N / 16) * sizeof(float2) * (DB ? 2 : 1);
    auto kern = k_nd_colfft<LOGN, T, NZ, DB>;
    VSA_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const int grid = persistent_grid(c, kern, T, smem, P.Wx);
    VSA_CUDA_TRY(vsa_launch(c, kern, dim3(grid), dim3(T), smem, (const float2 *)c->d_nd_G, P.Wx, P.Wy, (const float2 *)c->d_nd_tw,
                            (const float2 *)P.d_Py, P.r_ext, P.rc, P.ldt, (float2 *)c->d_nd_T));
    return VSAOGM_OK;
}

template <int LOGN, int NZ, bool FAST>
int launch_rowfft_nz(vsaogm_ctx *c, const NdPlan &P, const NdEpi &e)
{
    constexpr int N = 1 << LOGN;
    constexpr int T = N / 16 < 32 ? 32 : N / 16;
    constexpr bool DB = false;   // see launch_colfft_nz
    const size_t smem = (size_t)(N + N / 16) * sizeof(float2) * (DB ? 2 : 1);
    auto kern = k_nd_rowfft<LOGN, T, NZ, FAST, DB>;
    VSA_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const int grid = persistent_grid(c, kern, T, smem, P.r_ext);
    VSA_CUDA_TRY(vsa_launch(c, kern, dim3(grid), dim3(T), smem, (const float2 *)c->d_nd_T, P.ldt, P.Wx, (const float2 *)c->d_nd_tw,
                            (const float2 *)P.d_Px, P.cols, P.jc, e));
    return VSAOGM_OK;
}

template <int LOGN>
int launch_colfft(vsaogm_ctx *c, const NdPlan &P)
{
    if constexpr ((LOGN & 3) <= 1) {
        switch (nz_of(P.Wy, LOGN)) {
        case 3: return launch_colfft_nz<LOGN, 3>(c, P);
        case 4: return launch_colfft_nz<LOGN, 4>(c, P);
        case 8: return launch_colfft_nz<LOGN, 8>(c, P);
        default: break;
        }
    }
    return launch_colfft_nz<LOGN, 16>(c, P);
}

template <int LOGN, bool FAST>
int launch_rowfft_f(vsaogm_ctx *c, const NdPlan &P, const NdEpi &e)
{
    if constexpr ((LOGN & 3) <= 1) {
        switch (nz_of(P.Wx, LOGN)) {
        case 3: return launch_rowfft_nz<LOGN, 3, FAST>(c, P, e);
        case 4: return launch_rowfft_nz<LOGN, 4, FAST>(c, P, e);
        case 8: return launch_rowfft_nz<LOGN, 8, FAST>(c, P, e);
        default: break;
        }
    }
    return launch_rowfft_nz<LOGN, 16, FAST>(c, P, e);
}

template <int LOGN>
int launch_rowfft(vsaogm_ctx *c, const NdPlan &P, const NdEpi &e)
{
    // the streaming step (H_b only) runs the lean kernel; q outputs / histogram codes the generic one
    return (!e.q && !e.code) ? launch_rowfft_f<LOGN, true>(c, P, e) : launch_rowfft_f<LOGN, false>(c, P, e);
}

}  // namespace

bool vsa_nudecode_applies(vsaogm_ctx *c, double x0, double y0, double res, int32_t cols, int32_t r_lo, int32_t r_ext)
{
    if (c->dec_method == 0 || c->nslots != 2) return false;
    NdPlan G;
    if (!nd_geometry(c, x0, y0, res, cols, r_lo, r_ext, G)) return false;
    if (c->dec_method == 1) return true;
    // auto: modelled times, fitted to profiles/r5z_configs.json.  GEMM: 8 R C D
    // flops at ~1.1 PF/s plus the tables plus ~35 us of fixed cost (table A build + a one-wave GEMM:
    // 45 us at C2, 78 at C3, 249 at C4); NUFFT: transform work (point-stages, 0.32 ps each: 132 M in
    // 41 us at C4), the gather (1.1 ns per point: 15-18 us for 2 D = 16384), ~22 us for the four
    // launches and the short kernels' latency (32 us at C2, 40 at C3, 68 at C4).
    const double t_gemm = 8.0 * r_ext * (double)cols * c->D / 1.1e15 + 2.0 * (r_ext + 0.5 * cols) * (double)c->Dp * 2.0 / 4e12 + 35e-6;
    const double work = (double)G.Wx * G.My * G.logy + (double)r_ext * G.Mx * G.logx;
    const double t_nufft = work * 0.32e-12 + 2.0 * c->D * 1.1e-9 + 22e-6;
    return t_nufft < t_gemm;
}

int vsa_launch_decode_nufft(vsaogm_ctx *c, double x0, double y0, double res, int32_t cols, int32_t r_lo, int32_t r_ext,
                            float *hb, uint8_t *code, size_t ldh, float *q, int32_t q_off, int32_t band_rows,
                            bool mark_main)
{
    NdPlan *P = nullptr;
    int rc;
    if ((rc = nd_plan(c, x0, y0, res, cols, r_lo, r_ext, &P))) return rc;
    if ((rc = nd_grow(&c->d_nd_G, &c->nd_G_cap, (size_t)P->Wx * P->Wy * sizeof(float2)))) return rc;
    if ((rc = nd_grow(&c->d_nd_T, &c->nd_T_cap, (size_t)P->Wx * P->ldt * sizeof(float2)))) return rc;
    if ((rc = nd_grow(&c->d_nd_st, &c->nd_st_cap, 2 * (size_t)c->D * sizeof(float2)))) return rc;
    cudaEvent_t ev;
    vsa_prof_begin(c, VSAOGM_K_ND_SPREAD, &ev);
    const int npts = 2 * c->D;
    VSA_CUDA_TRY(vsa_launch(c, k_nd_strength, dim3((npts + 255) / 256), dim3(256), 0, (const int *)P->d_kid, npts, c->D, c->Dp,
                            (const double2 *)c->d_m, (const double *)(c->d_norm2 + c->nslots), 1.0 / c->D,
                            (const double *)c->d_tx_turns, (const double *)c->d_ty_turns, P->U0, P->V0, (float2 *)c->d_nd_st));
    // the memories are consumed: the next encode (encode stream) may start
    if (mark_main && (rc = vsa_mark_main(c))) return rc;
    NdSpread sp;
    sp.st = (const float2 *)c->d_nd_st;
    sp.pos = P->d_pos;
    sp.binx = P->d_binx;
    sp.bin_off = P->d_bin_off;
    sp.Wx = P->Wx;
    sp.Wy = P->Wy;
    sp.nbx = P->nbx;
    sp.nby = P->nby;
    sp.ax = P->ax;
    sp.ay = P->ay;
    sp.Gt = (float2 *)c->d_nd_G;
    VSA_CUDA_TRY(vsa_launch(c, k_nd_spread, dim3(P->ntx, P->nty), dim3(ND_NT), 0, sp));
    vsa_prof_end(c, VSAOGM_K_ND_SPREAD, ev);
    vsa_prof_begin(c, VSAOGM_K_ND_COLFFT, &ev);
    switch (P->logy) {
    case 8: rc = launch_colfft<8>(c, *P); break;
    case 9: rc = launch_colfft<9>(c, *P); break;
    case 10: rc = launch_colfft<10>(c, *P); break;
    case 11: rc = launch_colfft<11>(c, *P); break;
    case 12: rc = launch_colfft<12>(c, *P); break;
    default: rc = launch_colfft<13>(c, *P); break;
    }
    if (rc) return rc;
    VSA_CUDA_TRY(cudaGetLastError());
    vsa_prof_end(c, VSAOGM_K_ND_COLFFT, ev);
    vsa_prof_begin(c, VSAOGM_K_ND_ROWFFT, &ev);
    NdEpi e;
    e.mscale = c->d_norm2 + c->nslots;
    e.hb = hb;
    e.code = code;
    e.ldh = (int)ldh;
    e.r_ext = r_ext;
    e.q = q;
    e.q_off = q_off;
    e.band_rows = band_rows;
    e.cols = cols;
    switch (P->logx) {
    case 8: rc = launch_rowfft<8>(c, *P, e); break;
    case 9: rc = launch_rowfft<9>(c, *P, e); break;
    case 10: rc = launch_rowfft<10>(c, *P, e); break;
    case 11: rc = launch_rowfft<11>(c, *P, e); break;
    case 12: rc = launch_rowfft<12>(c, *P, e); break;
    default: rc = launch_rowfft<13>(c, *P, e); break;
    }
    if (rc) return rc;
    VSA_CUDA_TRY(cudaGetLastError());
    vsa_prof_end(c, VSAOGM_K_ND_ROWFFT, ev);
    c->launches += 4;
    return VSAOGM_OK;
}

void vsa_nudecode_free(vsaogm_ctx *c)
{
    for (int i = 0; i < c->nd_nplans; ++i) free_plan(static_cast<NdPlan *>(c->nd_plans[i]));
    c->nd_nplans = 0;
    if (c->d_nd_tw) cudaFree(c->d_nd_tw);
    if (c->d_nd_G) cudaFree(c->d_nd_G);
    if (c->d_nd_T) cudaFree(c->d_nd_T);
    if (c->d_nd_st) cudaFree(c->d_nd_st);
    c->d_nd_tw = c->d_nd_G = c->d_nd_T = c->d_nd_st = nullptr;
}
