// fft.cuh -- shared-memory complex FFTs used by the NUFFT encode (nufft.cu) and the NUFFT
// decode (nudecode.cu).
//
// Mixed radix Stockham (self-sorting) transform of N = 2^LOGN complex values in shared memory
// with the positive exponent, G_m = sum_j x_j e^{+2 pi i j m / N}, of an input whose upper half
// is zero (the zero padding: only x_j, j < N / 2, can be nonzero): the first stage is folded into
// the load -- x_j = load(j), j < N / 2 -- (radix 2 for odd LOGN: (x_j, x_j); radix 4 for even
// LOGN: the 4-point DFT of (x_j, x_{j + N/4}, 0, 0)), then radix-4 stages (sub-transform size
// Ns x4 per stage).  Radix-4 twiddles e^{+2 pi i k / (4 Ns)}, k < Ns: tw[2 Ns - 1 + k] of the
// per-stage table tw[p - 1 + k] = e^{+2 pi i k / (2p)}, k < p, p = 1, 2, 4, ... (the entries for
// p depend on p and k only, so one table built for the largest N serves every smaller N);
// w^2, w^3 by products.
//
// stockham_zp runs every stage and returns the buffer holding G.  stockham_zp_front stops before
// the last radix-4 stage (Ns = N / 4) so that the caller can fuse that stage with its epilogue
// and evaluate only the outputs it needs (fft_last_r4: outputs m = j and m = j + 3 N / 4 of
// thread j < N / 4, the two ends of the spectrum that a centred set of |m| < N / 4 modes uses).
#pragma once

#include <cuda_runtime.h>

template <int LOGN, int T, bool LAST, class Load>
__device__ __forceinline__ float2 *stockham_zp_impl(float2 *a, float2 *b, const float2 *__restrict__ tw, Load load)
{
    constexpr int N = 1 << LOGN;
    int ns;
    if (LOGN & 1) {
#pragma unroll
        for (int jj = 0; jj < N / 2; jj += T) {
            const int j = jj + threadIdx.x;
            if (N / 2 < T && j >= N / 2) break;   // small transforms: fewer values than threads
            const float2 v = load(j);
            *reinterpret_cast<float4 *>(a + 2 * j) = make_float4(v.x, v.y, v.x, v.y);
        }
        ns = 2;
    } else {
#pragma unroll
        for (int jj = 0; jj < N / 4; jj += T) {
            const int j = jj + threadIdx.x;
            if (N / 4 < T && j >= N / 4) break;
            const float2 x0 = load(j), x1 = load(j + N / 4);
            *reinterpret_cast<float4 *>(a + 4 * j) = make_float4(x0.x + x1.x, x0.y + x1.y, x0.x - x1.y, x0.y + x1.x);
            *reinterpret_cast<float4 *>(a + 4 * j + 2) = make_float4(x0.x - x1.x, x0.y - x1.y, x0.x + x1.y, x0.y - x1.x);
        }
        ns = 4;
    }
    constexpr int NST = (LOGN - 1) / 2 - (LAST ? 0 : 1);   // radix-4 stages run here
#pragma unroll
    for (int st = 0; st < NST; ++st) {
        __syncthreads();
#pragma unroll
        for (int jj = 0; jj < N / 4; jj += T) {
            const int j = jj + threadIdx.x;
            if (N / 4 < T && j >= N / 4) break;
            const int k = j & (ns - 1);
            float2 x0 = a[j], x1 = a[j + N / 4], x2 = a[j + N / 2], x3 = a[j + 3 * N / 4];
            const float2 w1 = __ldg(tw + 2 * ns - 1 + k);
            const float2 w2 = make_float2(w1.x * w1.x - w1.y * w1.y, 2.f * w1.x * w1.y);
            const float2 w3 = make_float2(w2.x * w1.x - w2.y * w1.y, w2.x * w1.y + w2.y * w1.x);
            x1 = make_float2(w1.x * x1.x - w1.y * x1.y, w1.x * x1.y + w1.y * x1.x);
            x2 = make_float2(w2.x * x2.x - w2.y * x2.y, w2.x * x2.y + w2.y * x2.x);
            x3 = make_float2(w3.x * x3.x - w3.y * x3.y, w3.x * x3.y + w3.y * x3.x);
            // 4-point DFT with the + sign: i^q
            const float2 s02 = make_float2(x0.x + x2.x, x0.y + x2.y), d02 = make_float2(x0.x - x2.x, x0.y - x2.y);
            const float2 s13 = make_float2(x1.x + x3.x, x1.y + x3.y), d13 = make_float2(x1.x - x3.x, x1.y - x3.y);
            const int o = ((j - k) << 2) + k;
            b[o] = make_float2(s02.x + s13.x, s02.y + s13.y);
            b[o + ns] = make_float2(d02.x - d13.y, d02.y + d13.x);           // + i d13
            b[o + 2 * ns] = make_float2(s02.x - s13.x, s02.y - s13.y);
            b[o + 3 * ns] = make_float2(d02.x + d13.y, d02.y - d13.x);       // - i d13
        }
        float2 *c = a;
        a = b;
        b = c;
        ns <<= 2;
    }
    __syncthreads();
    return a;
}

template <int LOGN, int T, class Load>
__device__ __forceinline__ float2 *stockham_zp(float2 *a, float2 *b, const float2 *__restrict__ tw, Load load)
{
    return stockham_zp_impl<LOGN, T, true>(a, b, tw, load);
}

template <int LOGN, int T, class Load>
__device__ __forceinline__ float2 *stockham_zp_front(float2 *a, float2 *b, const float2 *__restrict__ tw, Load load)
{
    static_assert(LOGN >= 3, "the fused last stage needs one radix-4 stage after the load");
    return stockham_zp_impl<LOGN, T, false>(a, b, tw, load);
}

// the last radix-4 stage (Ns = N / 4, so k = j) of thread j < N / 4 on the buffer returned by
// stockham_zp_front: y0 = G_j, y3 = G_{j + 3N/4} (= G_{j - N/4}, the negative modes)
template <int LOGN>
__device__ __forceinline__ void fft_last_r4(const float2 *a, const float2 *__restrict__ tw, int j, float2 &y0,
                                            float2 &y3)
{
    constexpr int N = 1 << LOGN;
    float2 x0 = a[j], x1 = a[j + N / 4], x2 = a[j + N / 2], x3 = a[j + 3 * N / 4];
    const float2 w1 = __ldg(tw + N / 2 - 1 + j);
    const float2 w2 = make_float2(w1.x * w1.x - w1.y * w1.y, 2.f * w1.x * w1.y);
    const float2 w3 = make_float2(w2.x * w1.x - w2.y * w1.y, w2.x * w1.y + w2.y * w1.x);
    x1 = make_float2(w1.x * x1.x - w1.y * x1.y, w1.x * x1.y + w1.y * x1.x);
    x2 = make_float2(w2.x * x2.x - w2.y * x2.y, w2.x * x2.y + w2.y * x2.x);
    x3 = make_float2(w3.x * x3.x - w3.y * x3.y, w3.x * x3.y + w3.y * x3.x);
    const float2 s02 = make_float2(x0.x + x2.x, x0.y + x2.y), d02 = make_float2(x0.x - x2.x, x0.y - x2.y);
    const float2 s13 = make_float2(x1.x + x3.x, x1.y + x3.y), d13 = make_float2(x1.x - x3.x, x1.y - x3.y);
    y0 = make_float2(s02.x + s13.x, s02.y + s13.y);
    y3 = make_float2(d02.x + d13.y, d02.y - d13.x);   // - i d13
}

// ---------------------------------------------------------------------------------------------
// Register-blocked Stockham FFT (the same transform, G_m = sum_j x_j e^{+2 pi i j m / N}): radix-16
// passes with the 16 values of a butterfly in registers (16 = 4 x 4, the quarter turns exact), a
// first pass of radix 2^(LOGN mod 4) when LOGN is not a multiple of 4; the first pass reads its
// inputs through load(j, slot) (global memory, zero padding inside load; slot = b R + r, the compile-time
// index of the value within the thread's first-pass inputs, for callers that prefetch them into registers), the last pass hands its
// outputs to store(i, m, G_m) from registers (i = the output's compile-time index within the thread's
// last-pass outputs, b R + q, for per-thread tables the caller keeps in registers), and the passes between exchange through ONE shared
// buffer of N + N/16 values (pad(i) = i + i/16 makes every pass's reads and writes conflict-free
// for 8-byte values).  T = max(32, N / 16) threads: one radix-16 butterfly per thread and pass.
// Twiddles e^{+2 pi i k / (R Ns)} from the universal table (tw[p - 1 + k] = e^{i pi k / p}), their
// powers by products (depth <= 7).
namespace fftr {

__device__ __forceinline__ int pad(int i) { return i + (i >> 4); }

__device__ __forceinline__ float2 cmul(float2 a, float2 b)
{
    return make_float2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}

// complex add / subtract as ONE packed fp32x2 instruction (FADD2: both lanes round to nearest, so the
// results are those of two scalar adds; the kernels are issue-bound, and the butterflies' adds are a
// third of their instructions: 128 FADD -> 32 FADD + 48 FADD2 per radix-16 butterfly, no moves -- a
// float2 already lives in an aligned register pair)
__device__ __forceinline__ float2 cadd(float2 a, float2 b)
{
    unsigned long long pa, pb, pr;
    asm("mov.b64 %0, {%1, %2};" : "=l"(pa) : "f"(a.x), "f"(a.y));
    asm("mov.b64 %0, {%1, %2};" : "=l"(pb) : "f"(b.x), "f"(b.y));
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(pr) : "l"(pa), "l"(pb));
    float2 r;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(pr));
    return r;
}
__device__ __forceinline__ float2 csub(float2 a, float2 b)
{
    unsigned long long pa, pb, pr;
    asm("mov.b64 %0, {%1, %2};" : "=l"(pa) : "f"(a.x), "f"(a.y));
    asm("mov.b64 %0, {%1, %2};" : "=l"(pb) : "f"(b.x), "f"(b.y));
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(pr) : "l"(pa), "l"(pb));
    float2 r;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(pr));
    return r;
}

// x e^{2 pi i m / 16}, the quarter turns exact
__device__ __forceinline__ float2 rot16(float2 x, int m)
{
    constexpr float C[16] = {1.f, 0.923879532511287f, 0.707106781186548f, 0.382683432365090f, 0.f,
                             -0.382683432365090f, -0.707106781186548f, -0.923879532511287f, -1.f,
                             -0.923879532511287f, -0.707106781186548f, -0.382683432365090f, 0.f,
                             0.382683432365090f, 0.707106781186548f, 0.923879532511287f};
    m &= 15;
    if (m == 0) return x;
    if (m == 4) return make_float2(-x.y, x.x);
    if (m == 8) return make_float2(-x.x, -x.y);
    if (m == 12) return make_float2(x.y, -x.x);
    return cmul(x, make_float2(C[m], C[(m + 12) & 15]));   // sin(a) = cos(a - pi/2)
}

template <int R>
struct Dft;
template <>
struct Dft<1> {
    __device__ __forceinline__ static void run(float2 *) {}
};
template <>
struct Dft<2> {
    __device__ __forceinline__ static void run(float2 *x)
    {
        const float2 a = x[0], b = x[1];
        x[0] = cadd(a, b);
        x[1] = csub(a, b);
    }
};
template <>
struct Dft<4> {
    __device__ __forceinline__ static void run(float2 *x)
    {
        const float2 s02 = cadd(x[0], x[2]), d02 = csub(x[0], x[2]);
        const float2 s13 = cadd(x[1], x[3]), d13 = csub(x[1], x[3]);
        x[0] = cadd(s02, s13);
        x[1] = make_float2(d02.x - d13.y, d02.y + d13.x);   // + i d13
        x[2] = csub(s02, s13);
        x[3] = make_float2(d02.x + d13.y, d02.y - d13.x);   // - i d13
    }
};
// 4-point DFT whose inputs t[i], i >= NZ, are known zeros (NZ = 1..4)
template <int NZ>
__device__ __forceinline__ void dft4z(float2 *t)
{
    if constexpr (NZ == 1) {
        t[1] = t[2] = t[3] = t[0];
    } else if constexpr (NZ == 2) {
        const float2 a = t[0], b = t[1];
        t[0] = cadd(a, b);
        t[1] = make_float2(a.x - b.y, a.y + b.x);
        t[2] = csub(a, b);
        t[3] = make_float2(a.x + b.y, a.y - b.x);
    } else if constexpr (NZ == 3) {
        const float2 s02 = cadd(t[0], t[2]), d02 = csub(t[0], t[2]), d13 = t[1];
        t[0] = cadd(s02, d13);
        t[1] = make_float2(d02.x - d13.y, d02.y + d13.x);
        t[2] = csub(s02, d13);
        t[3] = make_float2(d02.x + d13.y, d02.y - d13.x);
    } else {
        Dft<4>::run(t);
    }
}

// R = A B: r = B r1 + r2, q = q1 + A q2; y_q = DFT_B over r2 of (w_R^{r2 q1} DFT_A over r1).
// NZ: inputs x_r, r >= NZ, are known zeros (the zero padding of a first pass); ENDS (R = 16):
// only the outputs q2 in {0, B - 1} are formed (the others are left undefined).
template <int A, int B, int NZ = A * B, bool ENDS = false>
__device__ __forceinline__ void dft_ab(float2 *x)
{
    constexpr int R = A * B;
    float2 u[R];
#pragma unroll
    for (int r2 = 0; r2 < B; ++r2) {
        if (r2 >= NZ) continue;   // an all-zero group (compile time)
        float2 t[A];
#pragma unroll
        for (int r1 = 0; r1 < A; ++r1) t[r1] = x[B * r1 + r2];
        constexpr int dummy = 0;
        (void)dummy;
        // nonzero inputs of this group: r1 < ceil((NZ - r2) / B)
        if (A == 4) {
            const int nzg = (NZ - r2 + B - 1) / B;
            if (nzg == 1) dft4z<1>(t);
            else if (nzg == 2) dft4z<2>(t);
            else if (nzg == 3) dft4z<3>(t);
            else Dft<4>::run(t);
        } else {
            Dft<A>::run(t);
        }
#pragma unroll
        for (int q1 = 0; q1 < A; ++q1) u[r2 * A + q1] = rot16(t[q1], r2 * q1 * (16 / R));
    }
    constexpr int NG = NZ < B ? NZ : B;   // nonzero groups
#pragma unroll
    for (int q1 = 0; q1 < A; ++q1) {
        float2 t[B];
#pragma unroll
        for (int r2 = 0; r2 < B; ++r2) t[r2] = r2 < NG ? u[r2 * A + q1] : make_float2(0.f, 0.f);
        if constexpr (B == 4 && ENDS) {
            // outputs q2 = 0 and 3 only: t0 + t1 + t2 + t3 and t0 - i t1 - t2 + i t3
            const float2 s02 = cadd(t[0], t[2]), d02 = csub(t[0], t[2]);
            const float2 s13 = cadd(t[1], t[3]), d13 = csub(t[1], t[3]);
            x[q1] = cadd(s02, s13);
            x[q1 + 3 * A] = make_float2(d02.x + d13.y, d02.y - d13.x);
        } else if constexpr (B == 4) {
            dft4z<NG>(t);
#pragma unroll
            for (int q2 = 0; q2 < B; ++q2) x[q1 + A * q2] = t[q2];
        } else {
            Dft<B>::run(t);
#pragma unroll
            for (int q2 = 0; q2 < B; ++q2) x[q1 + A * q2] = t[q2];
        }
    }
}
template <>
struct Dft<8> {
    __device__ __forceinline__ static void run(float2 *x) { dft_ab<2, 4>(x); }
};
template <>
struct Dft<16> {
    __device__ __forceinline__ static void run(float2 *x) { dft_ab<4, 4>(x); }
};

// x_r *= w^r, r = 1 .. R-1
template <int R>
__device__ __forceinline__ void twiddle(float2 *x, float2 w)
{
    float2 p[R];
    p[1] = w;
#pragma unroll
    for (int r = 2; r < R; ++r) p[r] = (r & 1) ? cmul(p[r - 1], w) : cmul(p[r / 2], p[r / 2]);
#pragma unroll
    for (int r = 1; r < R; ++r) x[r] = cmul(x[r], p[r]);
}

// one radix-R pass on sub-transforms of length NS: butterfly j < N / R, k = j mod NS,
// x_r = in[j + r N / R] w^{r k} (w = e^{2 pi i / (R NS)}), y = DFT_R(x), out[(j - k) R + k + q NS] = y_q.
// SRC 0: load(i); 1: shared buf.  DST 0: shared buf; 1: store(b R + q, m, y).  NZ (first pass, R = 16): the
// inputs of groups r >= NZ are zero padding (not loaded).  ENDS (last pass, R = 16): only the
// outputs q < 4 and q >= 12 (|m| < N / 4, the centred modes) are formed and stored.
// DB: the pass reads bin and writes bout != bin (ping-pong buffers: no barrier between its reads and writes).
template <int LOGN, int R, int NS, int T, int SRC, int DST, int NZ, bool ENDS, bool DB, class Load, class Store>
__device__ __forceinline__ void pass(float2 *bin, float2 *bout, const float2 *__restrict__ tw, Load &load, Store &store)
{
    constexpr int N = 1 << LOGN;
    constexpr int NB = N / R;                         // butterflies
    constexpr int PER = (NB + T - 1) / T;            // per thread
    float2 x[PER][R];
    float2 wb[PER];                                   // twiddle bases, loaded before the data (latency overlap)
#pragma unroll
    for (int b = 0; b < PER; ++b)
        wb[b] = NS > 1 ? __ldg(tw + R * NS / 2 - 1 + ((threadIdx.x + b * T) & (NS - 1))) : make_float2(1.f, 0.f);
#pragma unroll
    for (int b = 0; b < PER; ++b) {
        const int j = threadIdx.x + b * T;
        if (NB % T == 0 || j < NB) {
#pragma unroll
            for (int r = 0; r < R; ++r) {
                if (r < NZ) x[b][r] = SRC == 0 ? load(j + r * NB, b * R + r) : bin[pad(j + r * NB)];
                else x[b][r] = make_float2(0.f, 0.f);   // zero padding (never read by the pruned butterfly)
            }
        }
    }
    if (SRC == 1 && DST == 0 && !DB) __syncthreads();   // every read of the buffer precedes the first write
#pragma unroll
    for (int b = 0; b < PER; ++b) {
        const int j = threadIdx.x + b * T;
        if (NB % T == 0 || j < NB) {
            const int k = j & (NS - 1);
            if (NS > 1) twiddle<R>(x[b], wb[b]);
            if constexpr (R == 16) dft_ab<4, 4, NZ, ENDS>(x[b]);
            else Dft<R>::run(x[b]);
            const int o = (j - k) * R + k;
#pragma unroll
            for (int q = 0; q < R; ++q) {
                if (ENDS && q >= 4 && q < 12) continue;
                if (DST == 0) bout[pad(o + q * NS)] = x[b][q];
                else store(b * R + q, o + q * NS, x[b][q]);
            }
        }
    }
    if (DST == 0) __syncthreads();
}

template <int LOGN, int P, int T, bool ENDS, bool DB, class Load, class Store>
__device__ __forceinline__ void passes16(float2 *bin, float2 *bout, const float2 *__restrict__ tw, Load &load, Store &store)
{
    // radix-16 pass P (NS = RF 16^P) and the ones after it
    constexpr int RF = 1 << (LOGN & 3);
    constexpr int NP16 = LOGN >> 2;
    if constexpr (P < NP16) {
        constexpr int NS = RF * (1 << (4 * P));
        constexpr bool LASTP = P == NP16 - 1;
        pass<LOGN, 16, NS, T, 1, LASTP ? 1 : 0, 16, LASTP && ENDS, DB>(bin, bout, tw, load, store);
        passes16<LOGN, P + 1, T, ENDS, DB>(bout, bin, tw, load, store);
    }
}

// the whole transform; buf: shared memory of N + N/16 float2 (DB: twice that -- the passes ping-pong
// between the halves, one barrier per pass instead of two, and a caller that runs transform after
// transform needs no barrier between them when there are exactly two exchanges (chained<LOGN>():
// the last pass then reads the second half while the next first pass writes the first)); otherwise
// the caller synchronises before reusing the buffer for another transform.  NZ: only x_j,
// j < NZ N / 16, can be nonzero (a radix-16 first
// pass skips the zero groups; NZ = 16: dense).  ENDS: only the outputs |m| < N / 4 are needed.
template <int LOGN>
__host__ __device__ constexpr bool chained()
{
    return (LOGN >> 2) + ((LOGN & 3) ? 1 : 0) == 3;   // three passes: two exchanges (without the ZP skip)
}

// ZP: the caller's input is zero-padded, x_j = 0 for j >= N / 2.  For odd-by-one sizes (LOGN = 4 p + 1) the
// radix-2 first pass would then only duplicate its inputs, buf[i] = x_{i >> 1}: it is skipped, and the
// first radix-16 pass (sub-transform length 2) reads load(i >> 1) itself, with NZ counting ITS nonzero
// input groups (x_{(j + r N/16) >> 1}: r < ceil(2 W / (N / 16)) for W nonzero values).
template <int LOGN, int T, int NZ = 16, bool ENDS = false, bool DB = false, bool ZP = false, class Load, class Store>
__device__ __forceinline__ void fft(float2 *buf, const float2 *__restrict__ tw, Load load, Store store)
{
    static_assert(LOGN >= 5, "at least one radix-16 pass after the first");
    constexpr int RF = 1 << (LOGN & 3);
    constexpr int NP16 = LOGN >> 2;
    float2 *b0 = buf, *b1 = DB ? buf + (1 << LOGN) + (1 << LOGN) / 16 : buf;
    if constexpr (RF == 2 && ZP && NP16 >= 2) {
        auto load2 = [&](int i, int slot) { return load(i >> 1, slot); };
        pass<LOGN, 16, 2, T, 0, 0, NZ, false, DB>(b0, b0, tw, load2, store);
        passes16<LOGN, 1, T, ENDS, DB>(b0, b1, tw, load2, store);
    } else if constexpr (RF > 1) {
        pass<LOGN, RF, 1, T, 0, 0, RF, false, DB>(b0, b0, tw, load, store);
        passes16<LOGN, 0, T, ENDS, DB>(b0, b1, tw, load, store);
    } else {
        pass<LOGN, 16, 1, T, 0, (NP16 == 1) ? 1 : 0, NZ, ENDS && NP16 == 1, DB>(b0, b0, tw, load, store);
        passes16<LOGN, 1, T, ENDS, DB>(b0, b1, tw, load, store);
    }
}

}  // namespace fftr
