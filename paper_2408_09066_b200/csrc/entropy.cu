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
// plus halo rows ([2][R_ext][cols] fp32).  Shared-memory tiled: a CTA stages a
// (TR + 2H) x (TC + 2H) tile of both classes (zeros outside the grid), then
// box windows use separable sums (row sums in shared memory, then column sums),
// disk windows sum each footprint row segment directly.  HBM-bound.
#include "common.cuh"

namespace {

constexpr int TR = 16;    // output rows per CTA
constexpr int TC = 128;   // output cols per CTA (one thread per column)

__global__ void __launch_bounds__(TC) k_entropy(const float *__restrict__ hb, int R, int C, int r_lo, int r_ext,
                                                int r0, int band_rows, int h1, int h0, int disk, float rho_occ,
                                                float rho_emp, float *__restrict__ S, uint8_t *__restrict__ lab)
{
    extern __shared__ float sm[];
    const int H = max(h1, h0);
    const int TW = TC + 2 * H, TH = TR + 2 * H;
    float *tile[2] = {sm, sm + TH * TW};
    float *hs = sm + 2 * TH * TW;   // [TH][TC] row sums (box)
    const int orow0 = r0 + blockIdx.y * TR;   // first output row (full-grid index)
    const int ocol0 = blockIdx.x * TC;
    const int tid = threadIdx.x;

    for (int cls = 0; cls < 2; ++cls) {
        const float *src = hb + (size_t)cls * r_ext * C;
        for (int idx = tid; idx < TH * TW; idx += TC) {
            const int rr = orow0 - H + idx / TW;
            const int cc = ocol0 - H + idx % TW;
            float v = 0.f;
            if (rr >= 0 && rr < R && cc >= 0 && cc < C) v = src[(size_t)(rr - r_lo) * C + cc];
            tile[cls][idx] = v;
        }
    }
    __syncthreads();

    const int col = ocol0 + tid;
    float Sc[2][TR];
#pragma unroll
    for (int cls = 0; cls < 2; ++cls) {
        const int h = cls == 1 ? h1 : h0;
        const float *t = tile[cls];
        if (!disk) {
            __syncthreads();
            for (int idx = tid; idx < TH * TC; idx += TC) {
                const int row = idx / TC, cc = idx % TC;
                float s = 0.f;
                for (int dv = -h; dv <= h; ++dv) s += t[row * TW + cc + H + dv];
                hs[idx] = s;
            }
            __syncthreads();
            const int nc = min(col + h, C - 1) - max(col - h, 0) + 1;
#pragma unroll
            for (int r = 0; r < TR; ++r) {
                float s = 0.f;
                for (int du = -h; du <= h; ++du) s += hs[(r + H + du) * TC + tid];
                const int row = orow0 + r;
                const int nr = min(row + h, R - 1) - max(row - h, 0) + 1;
                Sc[cls][r] = s / (float)(nr * nc);
            }
        } else {
#pragma unroll
            for (int r = 0; r < TR; ++r) {
                const int row = orow0 + r;
                float s = 0.f;
                int cnt = 0;
                for (int du = -h; du <= h; ++du) {
                    const int t2 = h * h - du * du;   // exact integer floor(sqrt(t2))
                    int w = (int)sqrtf((float)t2);
                    while ((w + 1) * (w + 1) <= t2) ++w;
                    while (w * w > t2) --w;
                    const float *tr = t + (r + H + du) * TW + tid + H;
                    for (int dv = -w; dv <= w; ++dv) s += tr[dv];
                    if (row + du >= 0 && row + du < R) cnt += min(col + w, C - 1) - max(col - w, 0) + 1;
                }
                Sc[cls][r] = cnt > 0 ? s / (float)cnt : 0.f;
            }
        }
    }

    if (col < C) {
#pragma unroll
        for (int r = 0; r < TR; ++r) {
            const int row = orow0 + r;
            const int br = row - r0;
            if (br >= band_rows) break;
            const float s1 = Sc[1][r], s0 = Sc[0][r];
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

}  // namespace

int vsa_launch_entropy(vsaogm_ctx *c, const vsaogm_entropy_params *p, float *S, uint8_t *lab)
{
    const int H = p->half_occ > p->half_emp ? p->half_occ : p->half_emp;
    const int band = c->g_r1 - c->g_r0;
    const size_t smem = sizeof(float) * (2 * (size_t)(TR + 2 * H) * (TC + 2 * H) + (size_t)(TR + 2 * H) * TC);
    if (smem > 48 * 1024) VSA_CUDA_TRY(cudaFuncSetAttribute(k_entropy, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    dim3 grid((c->g_cols + TC - 1) / TC, (band + TR - 1) / TR);
    cudaEvent_t ev;
    vsa_prof_begin(c, VSAOGM_K_ENTROPY, &ev);
    k_entropy<<<grid, TC, smem, c->stream>>>(c->d_hb, c->g_rows, c->g_cols, c->g_rlo, c->g_rext, c->g_r0, band,
                                             p->half_occ, p->half_emp, p->disk, p->rho_occ, p->rho_emp, S, lab);
    VSA_CUDA_TRY(cudaGetLastError());
    vsa_prof_end(c, VSAOGM_K_ENTROPY, ev);
    c->launches++;
    return VSAOGM_OK;
}
