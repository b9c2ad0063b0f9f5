// tables.cu -- K4: phasor tables, the two operands of the decode contraction.
//
// Because the encoding is separable, exp(i (w^x x + w^y y)) = Ex(x) Ey(y)
// (Eq. 9 binds the x- and y- fractional powers by an
// element-wise product, Eq. 6), the query of Eq. 11 over a grid is
//     H_c[r, col] = sum_k Re( Ey_k(y_r) conj(m_{c,k}) * Ex_k(x_col) )
// = a real GEMM with contraction length 2 Dp ("precalculating a
// matrix of location vectors", factorised here into row and column tables).
//
// K layout (shared by A and B, 16-bit, K-major rows of Kp = 2 Dp elements):
// k-groups of 32 phasor dimensions; group g occupies elements [64 g, 64 g+64):
// the 32 real parts then the 32 imaginary parts.  One 64-element group is one
// 128-byte TMA/UMMA swizzle row.
//   B[col][.] = ( Re Ex_k(x_col) | Im Ex_k(x_col) )                (cached per grid)
//   A[c*R_ext + i][.] = ( Re a | -Im a ),  a = s_c Ey_k(y_{r_lo+i}) conj(m_{c,k}),
//   s_c = sqrt(D) / ||m_c|| (Eq. 10; 0 for an empty class, L8),
// so that sum_j A[m][j] B[n][j] = s_c H_c = D q_c: the GEMM epilogue multiplies by 1/D.
// The sqrt(D) keeps |A| ~ 1 on average (16-bit operands stay normal numbers).
//
// Phases are reduced in fp64 (w * (x - c) in turns, minus the nearest integer)
// and evaluated by fp32 sincospi on the reduced argument.
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "common.cuh"

namespace {

template <typename T2>
__device__ __forceinline__ T2 pack2(float a, float b);
template <>
__device__ __forceinline__ __half2 pack2<__half2>(float a, float b) { return __floats2half2_rn(a, b); }
template <>
__device__ __forceinline__ __nv_bfloat162 pack2<__nv_bfloat162>(float a, float b) { return __floats2bfloat162_rn(a, b); }

__device__ __forceinline__ void phasor64(double w, double d, float *s, float *c)
{
    const double t = w * d * 0.15915494309189533577;   // turns
    const double f = t - rint(t);                        // in [-1/2, 1/2]
    sincospif((float)(2.0 * f), s, c);
}

// One thread = one row x one pair of consecutive k (same 32-group).
template <typename T2>
__global__ void k_table_B(T2 *__restrict__ B, int cols, int Dp, int D, int Kp, const double *__restrict__ wx,
                          double x0, double res, double cx)
{
    const int halfD = Dp >> 1;
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= (int64_t)cols * halfD) return;
    const int col = (int)(idx / halfD);
    const int k = 2 * (int)(idx - (int64_t)col * halfD);
    const double x = x0 + ((double)col + 0.5) * res - cx;
    float s0 = 0.f, c0 = 0.f, s1 = 0.f, c1 = 0.f;
    if (k < D) phasor64(wx[k], x, &s0, &c0);
    if (k + 1 < D) phasor64(wx[k + 1], x, &s1, &c1);
    const int g = k >> 5, w = k & 31;
    T2 *row = B + ((size_t)col * Kp >> 1);
    row[(64 * g + w) >> 1] = pack2<T2>(c0, c1);
    row[(64 * g + 32 + w) >> 1] = pack2<T2>(s0, s1);
}

template <typename T2>
__global__ void k_table_A(T2 *__restrict__ A, int r_ext, int Dp, int D, int Kp, const double *__restrict__ wy,
                          double y0, double res, int r_lo, double cy, const double *__restrict__ m,
                          const double *__restrict__ norm2, double sqrtD)
{
    const int halfD = Dp >> 1;
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= (int64_t)r_ext * halfD) return;
    const int i = (int)(idx / halfD);
    const int k = 2 * (int)(idx - (int64_t)i * halfD);
    const double y = y0 + ((double)(r_lo + i) + 0.5) * res - cy;
    float s[2] = {0.f, 0.f}, c[2] = {0.f, 0.f};
    if (k < D) phasor64(wy[k], y, &s[0], &c[0]);
    if (k + 1 < D) phasor64(wy[k + 1], y, &s[1], &c[1]);
    const int g = k >> 5, w = k & 31;
#pragma unroll
    for (int cls = 0; cls < 2; ++cls) {
        const double n2 = norm2[cls];
        const float sc = n2 > 0.0 ? (float)(sqrtD / sqrt(n2)) : 0.f;
        float re[2], nim[2];
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            const float mr = (float)m[2 * ((size_t)cls * Dp + k + e)] * sc;
            const float mi = (float)m[2 * ((size_t)cls * Dp + k + e) + 1] * sc;
            // a = (c + i s)(mr - i mi): Re a = c mr + s mi, -Im a = c mi - s mr
            re[e] = c[e] * mr + s[e] * mi;
            nim[e] = c[e] * mi - s[e] * mr;
        }
        T2 *row = A + (((size_t)cls * r_ext + i) * Kp >> 1);
        row[(64 * g + w) >> 1] = pack2<T2>(re[0], re[1]);
        row[(64 * g + 32 + w) >> 1] = pack2<T2>(nim[0], nim[1]);
    }
}

int grow(void **p, size_t *cap, size_t need)
{
    if (need <= *cap) return VSAOGM_OK;
    if (*p) cudaFree(*p);
    *p = nullptr;
    *cap = 0;
    if (cudaMalloc(p, need) != cudaSuccess) { *p = nullptr; return VSAOGM_ENOMEM; }
    *cap = need;
    return VSAOGM_OK;
}

}  // namespace

int vsa_launch_table_B(vsaogm_ctx *c, double x0, double res, int32_t cols, int prec)
{
    if (c->B_valid && c->B_x0 == x0 && c->B_res == res && c->B_cols == cols && c->B_prec == prec) return VSAOGM_OK;
    c->B_valid = false;
    const size_t bytes = (size_t)cols * c->Kp * 2;
    int rc = grow(&c->d_B, &c->B_cap, bytes);
    if (rc) return rc;
    const int64_t nthr = (int64_t)cols * (c->Dp / 2);
    const int bs = 256;
    cudaEvent_t ev;
    vsa_prof_begin(c, VSAOGM_K_TABLE_B, &ev);
    if (prec == VSAOGM_BF16)
        k_table_B<__nv_bfloat162><<<(unsigned)((nthr + bs - 1) / bs), bs, 0, c->stream>>>(
            (__nv_bfloat162 *)c->d_B, cols, c->Dp, c->D, c->Kp, c->d_wx64, x0, res, c->cx);
    else
        k_table_B<__half2><<<(unsigned)((nthr + bs - 1) / bs), bs, 0, c->stream>>>(
            (__half2 *)c->d_B, cols, c->Dp, c->D, c->Kp, c->d_wx64, x0, res, c->cx);
    VSA_CUDA_TRY(cudaGetLastError());
    vsa_prof_end(c, VSAOGM_K_TABLE_B, ev);
    c->launches++;
    c->B_valid = true;
    c->B_x0 = x0; c->B_res = res; c->B_cols = cols; c->B_prec = prec;
    return VSAOGM_OK;
}

int vsa_launch_table_A(vsaogm_ctx *c, double y0, double res, int32_t r_lo, int32_t r_ext, int prec)
{
    const size_t bytes = (size_t)2 * r_ext * c->Kp * 2;
    int rc = grow(&c->d_A, &c->A_cap, bytes);
    if (rc) return rc;
    const int64_t nthr = (int64_t)r_ext * (c->Dp / 2);
    const int bs = 256;
    cudaEvent_t ev;
    vsa_prof_begin(c, VSAOGM_K_TABLE_A, &ev);
    const double sqrtD = sqrt((double)c->D);
    if (prec == VSAOGM_BF16)
        k_table_A<__nv_bfloat162><<<(unsigned)((nthr + bs - 1) / bs), bs, 0, c->stream>>>(
            (__nv_bfloat162 *)c->d_A, r_ext, c->Dp, c->D, c->Kp, c->d_wy64, y0, res, r_lo, c->cy, c->d_m,
            c->d_norm2, sqrtD);
    else
        k_table_A<__half2><<<(unsigned)((nthr + bs - 1) / bs), bs, 0, c->stream>>>(
            (__half2 *)c->d_A, r_ext, c->Dp, c->D, c->Kp, c->d_wy64, y0, res, r_lo, c->cy, c->d_m, c->d_norm2,
            sqrtD);
    VSA_CUDA_TRY(cudaGetLastError());
    vsa_prof_end(c, VSAOGM_K_TABLE_A, ev);
    c->launches++;
    return VSAOGM_OK;
}
