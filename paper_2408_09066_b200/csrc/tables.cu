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
// One thread owns 8 consecutive k (16-byte stores) and walks table_rows rows,
// so theta and the scaled memory are loaded once per thread.  Phases are
// reduced in fp64 (turns = tau_k * coordinate, minus the nearest integer) and
// evaluated with MUFU sin/cos on the reduced argument |2 pi f| <= pi.
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "common.cuh"

namespace {

constexpr int TAB_THREADS = 128;
constexpr int TAB_KT = 8;

template <typename T2>
__device__ __forceinline__ T2 pack2(float a, float b);
template <>
__device__ __forceinline__ __half2 pack2<__half2>(float a, float b) { return __floats2half2_rn(a, b); }
template <>
__device__ __forceinline__ __nv_bfloat162 pack2<__nv_bfloat162>(float a, float b) { return __floats2bfloat162_rn(a, b); }

template <typename T2>
__device__ __forceinline__ uint4 pack8(const float *v)
{
    T2 p[4] = {pack2<T2>(v[0], v[1]), pack2<T2>(v[2], v[3]), pack2<T2>(v[4], v[5]), pack2<T2>(v[6], v[7])};
    return *reinterpret_cast<uint4 *>(p);
}

__device__ __forceinline__ void phasor_turns(double tau, double coord, float *s, float *c)
{
    const double t = tau * coord;                                               // turns
    const double r = __dsub_rn(__dadd_rn(t, 6755399441055744.0), 6755399441055744.0);   // rint(t)
    const float f = (float)__dsub_rn(t, r);                                     // in [-1/2, 1/2]
    __sincosf(6.28318530717958648f * f, s, c);
}

// IS_A = false: B[row][.] = (Re E | Im E), E = exp(2 pi i tau_k coord_row)
// IS_A = true : A[c*rows + row][.] = (Re a | -Im a), a = E conj(s_c m_c,k)
template <typename T2, bool IS_A>
__global__ void __launch_bounds__(TAB_THREADS) k_table(uint4 *__restrict__ out, int rows, int Dp, int D, int Kp,
                                                       const double *__restrict__ tau, double base, double res,
                                                       int row0, int tab_rows, const double2 *__restrict__ m,
                                                       const double *__restrict__ mscale)
{
    const int kq = blockIdx.x * TAB_THREADS + threadIdx.x;
    const int k0 = kq * TAB_KT;
    if (k0 >= Dp) return;
    const int g = k0 >> 5, w = k0 & 31;
    double tk[TAB_KT];
#pragma unroll
    for (int e = 0; e < TAB_KT; ++e) tk[e] = k0 + e < D ? tau[k0 + e] : 0.0;
    float mr[2][TAB_KT], mi[2][TAB_KT];
    if (IS_A) {
#pragma unroll
        for (int cls = 0; cls < 2; ++cls) {
            const double sc = mscale[cls];   // sqrt(D) / ||m_c||, 0 for an empty class (k_commit_norms)
#pragma unroll
            for (int e = 0; e < TAB_KT; ++e) {
                const double2 v = m[(size_t)cls * Dp + k0 + e];   // sqrt(D) m / ||m||, rounded to fp32
                mr[cls][e] = (float)(v.x * sc);
                mi[cls][e] = (float)(v.y * sc);
            }
        }
    }
    const int i0 = blockIdx.y * tab_rows;
    const int i1 = min(rows, i0 + tab_rows);
    // element offsets (in 16-byte units) of this thread's Re and Im octets within a row
    const size_t re_off = (size_t)(64 * g + w) / 8, im_off = (size_t)(64 * g + 32 + w) / 8;
    const size_t row_u4 = (size_t)Kp / 8;
    for (int i = i0; i < i1; ++i) {
        const double coord = base + ((double)(row0 + i) + 0.5) * res;
        float cs[TAB_KT], sn[TAB_KT];
#pragma unroll
        for (int e = 0; e < TAB_KT; ++e) {
            phasor_turns(tk[e], coord, &sn[e], &cs[e]);
            if (k0 + e >= D) cs[e] = sn[e] = 0.f;
        }
        if (!IS_A) {
            uint4 *row = out + (size_t)i * row_u4;
            row[re_off] = pack8<T2>(cs);
            row[im_off] = pack8<T2>(sn);
        } else {
#pragma unroll
            for (int cls = 0; cls < 2; ++cls) {
                float re[TAB_KT], nim[TAB_KT];
#pragma unroll
                for (int e = 0; e < TAB_KT; ++e) {
                    // a = (c + i s)(mr - i mi): Re a = c mr + s mi, -Im a = c mi - s mr
                    re[e] = cs[e] * mr[cls][e] + sn[e] * mi[cls][e];
                    nim[e] = cs[e] * mi[cls][e] - sn[e] * mr[cls][e];
                }
                uint4 *row = out + ((size_t)cls * rows + i) * row_u4;
                row[re_off] = pack8<T2>(re);
                row[im_off] = pack8<T2>(nim);
            }
        }
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

template <bool IS_A>
void launch_table(vsaogm_ctx *c, void *out, int rows, const double *tau, double base, double res, int row0, int prec,
                  const double2 *m, const double *mscale)
{
    dim3 grid((c->Dp / TAB_KT + TAB_THREADS - 1) / TAB_THREADS, (rows + c->table_rows - 1) / c->table_rows);
    if (prec == VSAOGM_BF16)
        k_table<__nv_bfloat162, IS_A><<<grid, TAB_THREADS, 0, c->stream>>>((uint4 *)out, rows, c->Dp, c->D, c->Kp,
                                                                            tau, base, res, row0, c->table_rows, m, mscale);
    else
        k_table<__half2, IS_A><<<grid, TAB_THREADS, 0, c->stream>>>((uint4 *)out, rows, c->Dp, c->D, c->Kp, tau,
                                                                     base, res, row0, c->table_rows, m, mscale);
}

}  // namespace

int vsa_launch_table_B(vsaogm_ctx *c, double x0, double res, int32_t cols, int prec)
{
    if (c->B_valid && c->B_x0 == x0 && c->B_res == res && c->B_cols == cols && c->B_prec == prec) return VSAOGM_OK;
    c->B_valid = false;
    const size_t bytes = (size_t)cols * c->Kp * 2;
    int rc = grow(&c->d_B, &c->B_cap, bytes);
    if (rc) return rc;
    cudaEvent_t ev;
    vsa_prof_begin(c, VSAOGM_K_TABLE_B, &ev);
    launch_table<false>(c, c->d_B, cols, c->d_tx_turns, x0 - c->cx, res, 0, prec, nullptr, nullptr);
    VSA_CUDA_TRY(cudaGetLastError());
    vsa_prof_end(c, VSAOGM_K_TABLE_B, ev);
    c->launches++;
    c->B_valid = true;
    c->B_x0 = x0; c->B_res = res; c->B_cols = cols; c->B_prec = prec;
    return VSAOGM_OK;
}

// One A block per decode group (quadrant): rows [a_row0, a_row0 + 2 nrows) hold the
// class-0 then class-1 rows of the group's decoded grid rows, built from the group's
// memory slots slot0[g], slot0[g] + 1 (delta = 1: one group, slots 0 and 1).
int vsa_launch_table_A(vsaogm_ctx *c, const Groups &G, double y0, double res, int32_t r_lo, int prec,
                       const int *slot0)
{
    size_t rows = 0;
    for (int g = 0; g < G.n; ++g) rows = std::max(rows, (size_t)(G.a_row0[g] + G.mrows[g]));
    int rc = grow(&c->d_A, &c->A_cap, rows * c->Kp * 2);
    if (rc) return rc;
    cudaEvent_t ev;
    vsa_prof_begin(c, VSAOGM_K_TABLE_A, &ev);
    for (int g = 0; g < G.n; ++g) {
        launch_table<true>(c, (uint8_t *)c->d_A + (size_t)G.a_row0[g] * c->Kp * 2, G.nrows[g], c->d_ty_turns,
                           y0 - c->cy, res, r_lo + G.row0[g], prec,
                           (const double2 *)c->d_m + (size_t)slot0[g] * c->Dp, c->d_norm2 + c->nslots + slot0[g]);
        c->launches++;
    }
    VSA_CUDA_TRY(cudaGetLastError());
    vsa_prof_end(c, VSAOGM_K_TABLE_A, ev);
    return VSAOGM_OK;
}
