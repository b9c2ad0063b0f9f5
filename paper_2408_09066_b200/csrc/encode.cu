// encode.cu -- K2 encode/bundle, K3 partial reduction, commit and norms.
//
// K2 computes, for every point i (label psi_i) and phasor dimension k,
//     E_k(x_i, y_i) = exp(i (w^x_k (x_i - c_x) + w^y_k (y_i - c_y))),  w = theta / l,
// (Eq. 9, length scale Eq. 8 :232-235) and bundles it into
// class memory psi_i by addition (Eq. 5 :216-219; Alg. 1 :260-285 with delta=1).
// The phase origin (c_x, c_y) is the bounds centre: a per-k rotation common to
// every point that cancels in the decode (Eq. 11) and keeps the fp32 phase
// small.  The kernel is bound by the MUFU (XU) and FMA pipes together: a phasor
// costs either one MUFU sin + one MUFU cos, or a packed FMA-pipe polynomial
// (sincos_fma2_lite); the default kernel k_encode_bundle_x2 runs all-MUFU warps
// beside polynomial warps.  k_encode_bundle (scalar) and
// k_encode_slots remain as measured variants / the small-D path.
//
// Layout: threads own phasor dimensions k (KT per thread, strided by the block
// size so the w loads and partial stores are coalesced); the points of the
// block's chunk are staged through shared memory and read as warp-uniform
// broadcasts, so the per-point label branch is uniform across the warp.  Each
// block writes its chunk's fp32 partial sums; K3 adds chunks in a fixed order
// in fp64 (deterministic, no float atomics).
#include <cooperative_groups.h>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace {

constexpr int ENC_THREADS = 128;
constexpr int ENC_TILE = 256;   // points staged per shared-memory tile

__device__ __forceinline__ void sincos_poly(float phi, float *s_out, float *c_out) { sincos_fma(phi, s_out, c_out); }

// Phasor j of KT: the last NPOLY of each thread's KT dimensions use the
// polynomial, the others MUFU.SIN / MUFU.COS (__sincosf).
template <int KT, int NPOLY>
__device__ __forceinline__ void phasor(int j, float phi, float *s, float *c)
{
    if (j >= KT - NPOLY) sincos_poly(phi, s, c);
    else __sincosf(phi, s, c);
}

template <int KT, int NPOLY, int MINB = 6>
__global__ void __launch_bounds__(ENC_THREADS, MINB) k_encode_bundle(
    const float2 *__restrict__ xy, const uint8_t *__restrict__ lab, int64_t n, int64_t chunk_pts,
    const float *__restrict__ wx, const float *__restrict__ wy, double cx, double cy, int Dp,
    float2 *__restrict__ part, long long *__restrict__ part_cnt, int *__restrict__ err)
{
    constexpr int NW = ENC_THREADS / 32;
    constexpr int ROUNDS = ENC_TILE / ENC_THREADS;
    __shared__ float4 s_p0[ENC_TILE], s_p1[ENC_TILE];   // the tile's class-0 / class-1 points, in point order
    __shared__ int s_g0[ROUNDS * NW], s_g1[ROUNDS * NW];
    const int tid = threadIdx.x;
    const int lane = tid & 31, warp = tid >> 5;
    const int kb = blockIdx.x;
    const int64_t chunk = blockIdx.y;
    const int kbase = kb * ENC_THREADS * KT + tid;

    float fx[KT], fy[KT];
    float a0r[KT], a0i[KT], a1r[KT], a1i[KT];
#pragma unroll
    for (int j = 0; j < KT; ++j) {
        const int k = kbase + j * ENC_THREADS;
        fx[j] = k < Dp ? wx[k] : 0.f;
        fy[j] = k < Dp ? wy[k] : 0.f;
        a0r[j] = a0i[j] = a1r[j] = a1i[j] = 0.f;
    }
    long long c0 = 0, c1 = 0;
    int my_err = 0;
    const int64_t p0 = chunk * chunk_pts;
    const int64_t p1 = min(n, p0 + chunk_pts);

    for (int64_t base = p0; base < p1; base += ENC_TILE) {
        const int cnt = (int)min((int64_t)ENC_TILE, p1 - base);
        __syncthreads();
        // stage the tile split by label with a deterministic, order-preserving compaction
        // (ballot + block prefix), so the inner loops carry no per-point label branch
        float4 rec[ROUNDS];
        int code_r[ROUNDS];
        unsigned b0[ROUNDS], b1[ROUNDS];
#pragma unroll
        for (int r = 0; r < ROUNDS; ++r) {
            const int t = tid + r * ENC_THREADS;
            int code = 2;
            rec[r] = make_float4(0.f, 0.f, 0.f, 0.f);
            if (t < cnt) {
                const float2 v = xy[base + t];
                const int L = lab[base + t];
                code = L;
                if (L > 1) { code = 2; my_err |= VSA_ERRBIT_LABEL; }
                if (!(isfinite(v.x) && isfinite(v.y))) { code = 2; my_err |= VSA_ERRBIT_NONFINITE; }
                // centred coordinates: fp64 subtraction, one rounding to fp32
                rec[r] = make_float4((float)((double)v.x - cx), (float)((double)v.y - cy), 0.f, 0.f);
            }
            code_r[r] = code;
            b0[r] = __ballot_sync(0xffffffffu, code == 0);
            b1[r] = __ballot_sync(0xffffffffu, code == 1);
            if (lane == 0) {
                s_g0[r * NW + warp] = __popc(b0[r]);
                s_g1[r * NW + warp] = __popc(b1[r]);
            }
        }
        __syncthreads();
        int n0 = 0, n1 = 0, o0[ROUNDS], o1[ROUNDS];
#pragma unroll
        for (int g = 0; g < ROUNDS * NW; ++g) {
#pragma unroll
            for (int r = 0; r < ROUNDS; ++r)
                if (g == r * NW + warp) { o0[r] = n0; o1[r] = n1; }
            n0 += s_g0[g];
            n1 += s_g1[g];
        }
        const unsigned lt = (1u << lane) - 1u;
#pragma unroll
        for (int r = 0; r < ROUNDS; ++r) {
            if (code_r[r] == 0) s_p0[o0[r] + __popc(b0[r] & lt)] = rec[r];
            else if (code_r[r] == 1) s_p1[o1[r] + __popc(b1[r] & lt)] = rec[r];
        }
        c0 += n0;   // block totals (every thread has them; thread 0 reports)
        c1 += n1;
        __syncthreads();
#pragma unroll 2
        for (int p = 0; p < n0; ++p) {
            const float4 P = s_p0[p];                   // warp-uniform broadcast
#pragma unroll
            for (int j = 0; j < KT; ++j) {
                float s, c;
                phasor<KT, NPOLY>(j, fmaf(fx[j], P.x, fy[j] * P.y), &s, &c);
                a0r[j] += c;
                a0i[j] += s;
            }
        }
#pragma unroll 2
        for (int p = 0; p < n1; ++p) {
            const float4 P = s_p1[p];
#pragma unroll
            for (int j = 0; j < KT; ++j) {
                float s, c;
                phasor<KT, NPOLY>(j, fmaf(fx[j], P.x, fy[j] * P.y), &s, &c);
                a1r[j] += c;
                a1i[j] += s;
            }
        }
    }
#pragma unroll
    for (int j = 0; j < KT; ++j) {
        const int k = kbase + j * ENC_THREADS;
        if (k < Dp) {
            part[((size_t)chunk * 2 + 0) * Dp + k] = make_float2(a0r[j], a0i[j]);
            part[((size_t)chunk * 2 + 1) * Dp + k] = make_float2(a1r[j], a1i[j]);
        }
    }
    if (kb == 0) {   // counts and deferred errors once per chunk
        if (my_err) atomicOr(err, my_err);
        if (tid == 0) {
            part_cnt[chunk * 2 + 0] = c0;
            part_cnt[chunk * 2 + 1] = c1;
        }
    }
}

// Packed variant of K2: the same label-split staging and loop as k_encode_bundle, with
// each thread's 8 dimensions processed as 4 pairs in fp32x2 instructions (PhasorAcc,
// common.cuh): the angles, the accumulation and the polynomial phasors take one issue
// slot per two lanes, and the register footprint is the scalar kernel's.
//
// Warp roles: the first half of the block's warps evaluate NPA of their 8 dimensions by
// polynomial, the second half NPB.  With NPA = 0 (all MUFU) and NPB = 4 (the default), every SM
// sub-partition (warps w and w + 4 of each block) runs one MUFU-bound warp beside one
// FMA-bound warp: two homogeneous instruction streams that the warp scheduler
// interleaves, rather than one stream whose MUFU and polynomial phases alternate and
// stall on each other's latencies.  Each dimension still sums its points in point
// order with the scalar per-lane arithmetic (only which dimensions use the polynomial
// differs from k_encode_bundle).
template <int THREADS, int NPA, int NPB, int MINB>
__global__ void __launch_bounds__(THREADS, MINB) k_encode_bundle_x2(
    const float2 *__restrict__ xy, const uint8_t *__restrict__ lab, int64_t n, int64_t chunk_pts,
    const float *__restrict__ wx, const float *__restrict__ wy, double cx, double cy, int Dp,
    float2 *__restrict__ part, long long *__restrict__ part_cnt, int *__restrict__ err)
{
    constexpr int KT = 8;
    constexpr int NW = THREADS / 32;
    constexpr int TILE = THREADS >= ENC_TILE ? THREADS : ENC_TILE;
    constexpr int ROUNDS = TILE / THREADS;
    __shared__ float2 s_p0[TILE], s_p1[TILE];
    __shared__ int s_g0[ROUNDS * NW], s_g1[ROUNDS * NW];
    const int tid = threadIdx.x;
    const int lane = tid & 31, warp = tid >> 5;
    const bool role_b = warp >= NW / 2;   // warp-uniform
    const int kb = blockIdx.x;
    const int64_t chunk = blockIdx.y;
    const int kbase = kb * THREADS * KT + tid;

    float fx[KT], fy[KT];
#pragma unroll
    for (int j = 0; j < KT; ++j) {
        const int k = kbase + j * THREADS;
        fx[j] = k < Dp ? wx[k] : 0.f;
        fy[j] = k < Dp ? wy[k] : 0.f;
    }
    long long c0 = 0, c1 = 0;
    int my_err = 0;
    const int64_t p0 = chunk * chunk_pts;
    const int64_t p1 = min(n, p0 + chunk_pts);

    // the tile loop, per role (the staging code is common; the bundle loops differ)
    auto run = [&](auto acc0, auto acc1) {
        acc0.init(fx, fy);
        acc1.init(fx, fy);
        for (int64_t base = p0; base < p1; base += TILE) {
            const int cnt = (int)min((int64_t)TILE, p1 - base);
            block_sync_any();
            float2 rec[ROUNDS];
            int code_r[ROUNDS];
            unsigned b0[ROUNDS], b1[ROUNDS];
#pragma unroll
            for (int r = 0; r < ROUNDS; ++r) {
                const int t = tid + r * THREADS;
                int code = 2;
                rec[r] = make_float2(0.f, 0.f);
                if (t < cnt) {
                    const float2 v = xy[base + t];
                    const int L = lab[base + t];
                    code = L;
                    if (L > 1) { code = 2; my_err |= VSA_ERRBIT_LABEL; }
                    if (!(isfinite(v.x) && isfinite(v.y))) { code = 2; my_err |= VSA_ERRBIT_NONFINITE; }
                    rec[r] = make_float2((float)((double)v.x - cx), (float)((double)v.y - cy));
                }
                code_r[r] = code;
                b0[r] = __ballot_sync(0xffffffffu, code == 0);
                b1[r] = __ballot_sync(0xffffffffu, code == 1);
                if (lane == 0) {
                    s_g0[r * NW + warp] = __popc(b0[r]);
                    s_g1[r * NW + warp] = __popc(b1[r]);
                }
            }
            block_sync_any();
            int n0 = 0, n1 = 0, o0[ROUNDS], o1[ROUNDS];
#pragma unroll
            for (int g = 0; g < ROUNDS * NW; ++g) {
#pragma unroll
                for (int r = 0; r < ROUNDS; ++r)
                    if (g == r * NW + warp) { o0[r] = n0; o1[r] = n1; }
                n0 += s_g0[g];
                n1 += s_g1[g];
            }
            const unsigned lt = (1u << lane) - 1u;
#pragma unroll
            for (int r = 0; r < ROUNDS; ++r) {
                if (code_r[r] == 0) s_p0[o0[r] + __popc(b0[r] & lt)] = rec[r];
                else if (code_r[r] == 1) s_p1[o1[r] + __popc(b1[r] & lt)] = rec[r];
            }
            c0 += n0;
            c1 += n1;
            block_sync_any();
#pragma unroll 2
            for (int p = 0; p < n0; ++p) {
                const float2 P = s_p0[p];   // warp-uniform broadcast
                acc0.point(P.x, P.y);
            }
#pragma unroll 2
            for (int p = 0; p < n1; ++p) {
                const float2 P = s_p1[p];
                acc1.point(P.x, P.y);
            }
        }
#pragma unroll
        for (int j = 0; j < KT; ++j) {
            const int k = kbase + j * THREADS;
            if (k < Dp) {
                part[((size_t)chunk * 2 + 0) * Dp + k] = acc0.get(j);
                part[((size_t)chunk * 2 + 1) * Dp + k] = acc1.get(j);
            }
        }
    };
    if (role_b) run(PhasorAcc<KT, NPB>{}, PhasorAcc<KT, NPB>{});
    else run(PhasorAcc<KT, NPA>{}, PhasorAcc<KT, NPA>{});
    if (kb == 0) {
        if (my_err) atomicOr(err, my_err);
        if (tid == 0) {
            part_cnt[chunk * 2 + 0] = c0;
            part_cnt[chunk * 2 + 1] = c1;
        }
    }
}

// Pair (half-angle) variant of K2, the default for delta = 1 and D >= 2048: the label-split
// staging of k_encode_bundle_x2, with the coordinates kept centred in fp64 in shared memory;
// consecutive points of one class in the tile form pairs whose mean and half-difference
// (xbar, ybar, dx, dy) are computed in fp64 and rounded once to fp32; the bundle loop then
// adds 2 cos(delta) e^{i sigma} per pair (PairAcc, common.cuh): 1.5 MUFU ops per phasor
// instead of 2.  An odd last point of a class in a tile is added on its own.  Warp roles as in
// k_encode_bundle_x2 (warps 0-3: NPA, warps 4-7: NPB of 8 dimensions on the FMA pipe).  Every
// block barrier is the non-.aligned barrier.sync, reached from both roles' code.
template <int THREADS, int NPA, int NPB, int MINB>
__global__ void __launch_bounds__(THREADS, MINB) k_encode_pairs(
    const float2 *__restrict__ xy, const uint8_t *__restrict__ lab, int64_t n, int64_t chunk_pts,
    const float *__restrict__ wx, const float *__restrict__ wy, double cx, double cy, int Dp,
    float2 *__restrict__ part, long long *__restrict__ part_cnt, int *__restrict__ err)
{
    constexpr int KT = 8;
    constexpr int NW = THREADS / 32;
    constexpr int TILE = THREADS;
    __shared__ double2 s_p[2][TILE];          // the tile's centred points, split by class, in order
    __shared__ float4 s_q[2][TILE / 2];       // pair records (xbar, ybar, dx, dy)
    __shared__ int s_g0[NW], s_g1[NW];
    const int tid = threadIdx.x;
    const int lane = tid & 31, warp = tid >> 5;
    const bool role_b = warp >= NW / 2;   // warp-uniform
    const int kb = blockIdx.x;
    const int64_t chunk = blockIdx.y;
    const int kbase = kb * THREADS * KT + tid;

    float fx[KT], fy[KT];
#pragma unroll
    for (int j = 0; j < KT; ++j) {
        const int k = kbase + j * THREADS;
        fx[j] = k < Dp ? wx[k] : 0.f;
        fy[j] = k < Dp ? wy[k] : 0.f;
    }
    long long c0 = 0, c1 = 0;
    int my_err = 0;
    const int64_t p0 = chunk * chunk_pts;
    const int64_t p1 = min(n, p0 + chunk_pts);

    PairW<KT> w;
    w.init(fx, fy);
    auto run = [&](auto acc0, auto acc1) {
        acc0.init();
        acc1.init();
        for (int64_t base = p0; base < p1; base += TILE) {
            const int cnt = (int)min((int64_t)TILE, p1 - base);
            block_sync_any();
            int code = 2;
            double2 rec = make_double2(0.0, 0.0);
            if (tid < cnt) {
                const float2 v = xy[base + tid];
                const int L = lab[base + tid];
                code = L;
                if (L > 1) { code = 2; my_err |= VSA_ERRBIT_LABEL; }
                if (!(isfinite(v.x) && isfinite(v.y))) { code = 2; my_err |= VSA_ERRBIT_NONFINITE; }
                rec = make_double2((double)v.x - cx, (double)v.y - cy);
            }
            const unsigned b0 = __ballot_sync(0xffffffffu, code == 0);
            const unsigned b1 = __ballot_sync(0xffffffffu, code == 1);
            if (lane == 0) {
                s_g0[warp] = __popc(b0);
                s_g1[warp] = __popc(b1);
            }
            block_sync_any();
            int n0 = 0, n1 = 0, o0 = 0, o1 = 0;
#pragma unroll
            for (int g = 0; g < NW; ++g) {
                if (g == warp) { o0 = n0; o1 = n1; }
                n0 += s_g0[g];
                n1 += s_g1[g];
            }
            const unsigned lt = (1u << lane) - 1u;
            if (code == 0) s_p[0][o0 + __popc(b0 & lt)] = rec;
            else if (code == 1) s_p[1][o1 + __popc(b1 & lt)] = rec;
            c0 += n0;
            c1 += n1;
            block_sync_any();
            const int np0 = n0 >> 1, np1 = n1 >> 1;
            if (tid < np0 + np1) {                            // pair records, fp64 then one rounding
                const int cls = tid >= np0, i = cls ? tid - np0 : tid;
                const double2 a = s_p[cls][2 * i], b = s_p[cls][2 * i + 1];
                s_q[cls][i] = make_float4((float)(0.5 * (a.x + b.x)), (float)(0.5 * (a.y + b.y)),
                                          (float)(0.5 * (a.x - b.x)), (float)(0.5 * (a.y - b.y)));
            }
            block_sync_any();
#pragma unroll 1
            for (int p = 0; p < np0; ++p) acc0.pair(w, s_q[0][p]);   // warp-uniform broadcasts
            if (n0 & 1) {
                const double2 a = s_p[0][n0 - 1];
                acc0.single(w, (float)a.x, (float)a.y);
            }
#pragma unroll 1
            for (int p = 0; p < np1; ++p) acc1.pair(w, s_q[1][p]);
            if (n1 & 1) {
                const double2 a = s_p[1][n1 - 1];
                acc1.single(w, (float)a.x, (float)a.y);
            }
        }
#pragma unroll
        for (int j = 0; j < KT; ++j) {
            const int k = kbase + j * THREADS;
            if (k < Dp) {
                part[((size_t)chunk * 2 + 0) * Dp + k] = acc0.get(j);
                part[((size_t)chunk * 2 + 1) * Dp + k] = acc1.get(j);
            }
        }
    };
    if (role_b) run(PairAcc<KT, NPB>{}, PairAcc<KT, NPB>{});
    else run(PairAcc<KT, NPA>{}, PairAcc<KT, NPA>{});
    if (kb == 0) {
        if (my_err) atomicOr(err, my_err);
        if (tid == 0) {
            part_cnt[chunk * 2 + 0] = c0;
            part_cnt[chunk * 2 + 1] = c1;
        }
    }
}

// One class per block (grid.z = class): the pair kernel with a single accumulator set, 16
// registers lighter (64 registers, 4 blocks per SM without spills, so that three blocks fit
// beside a decode-GEMM CTA in the pipelined schedule).  Every block stages the whole tile and
// keeps its class's points (in order), so the per-dimension sums are those of k_encode_pairs.
// OUTL (NUFFT fallback, nufft.cu): only the points outside the NUFFT grid are bundled, a chunk
// without such points exits at once, and the block's sums are added to the pending memories
// directly (fp64 atomics: the order of the chunks' additions is not fixed, L16).
struct NuOutl {
    double lo, inv_h;
    int n1;
    const int *out_cnt;
    double *pending;
    int D;
};

template <int THREADS, int NPA, int NPB, int MINB, bool OUTL = false>
__global__ void __launch_bounds__(THREADS, MINB) k_encode_pairs1(
    const float2 *__restrict__ xy, const uint8_t *__restrict__ lab, int64_t n, int64_t chunk_pts,
    const float *__restrict__ wx, const float *__restrict__ wy, double cx, double cy, int Dp,
    float2 *__restrict__ part, long long *__restrict__ part_cnt, int *__restrict__ err, NuOutl nu = NuOutl{})
{
    vsa_pdl();
    if (OUTL && nu.out_cnt[blockIdx.y] == 0) return;   // block-uniform
    constexpr int KT = 8;
    constexpr int NW = THREADS / 32;
    constexpr int TILE = THREADS;
    __shared__ double2 s_p[TILE];             // the tile's centred points of this class, in order
    __shared__ float4 s_q[TILE / 2];          // pair records (xbar, ybar, dx, dy)
    __shared__ int s_g[NW];
    const int tid = threadIdx.x;
    const int lane = tid & 31, warp = tid >> 5;
    const bool role_b = warp >= NW / 2;   // warp-uniform
    const int kb = blockIdx.x;
    const int64_t chunk = blockIdx.y;
    const int cls = blockIdx.z;
    const int kbase = kb * THREADS * KT + tid;

    float fx[KT], fy[KT];
#pragma unroll
    for (int j = 0; j < KT; ++j) {
        const int k = kbase + j * THREADS;
        fx[j] = k < Dp ? wx[k] : 0.f;
        fy[j] = k < Dp ? wy[k] : 0.f;
    }
    long long cn = 0;
    int my_err = 0;
    const int64_t p0 = chunk * chunk_pts;
    const int64_t p1 = min(n, p0 + chunk_pts);
    PairW<KT> w;
    w.init(fx, fy);

    auto run = [&](auto acc) {
        acc.init();
        for (int64_t base = p0; base < p1; base += TILE) {
            const int cnt = (int)min((int64_t)TILE, p1 - base);
            block_sync_any();
            bool mine = false;
            double2 rec = make_double2(0.0, 0.0);
            if (tid < cnt) {
                const float2 v = xy[base + tid];
                const int L = lab[base + tid];
                int code = L;
                if (L > 1) { code = 2; my_err |= VSA_ERRBIT_LABEL; }
                if (!(isfinite(v.x) && isfinite(v.y))) { code = 2; my_err |= VSA_ERRBIT_NONFINITE; }
                mine = code == cls;
                rec = make_double2((double)v.x - cx, (double)v.y - cy);
                if (OUTL && mine) {   // the same fp64 expression as k_nu_spread's grid test
                    const int ix = (int)floor((rec.x - nu.lo) * nu.inv_h), iy = (int)floor((rec.y - nu.lo) * nu.inv_h);
                    mine = ix - 6 < 0 || iy - 6 < 0 || ix + 7 >= nu.n1 || iy + 7 >= nu.n1;
                }
            }
            const unsigned b = __ballot_sync(0xffffffffu, mine);
            if (lane == 0) s_g[warp] = __popc(b);
            block_sync_any();
            int nc = 0, o = 0;
#pragma unroll
            for (int g = 0; g < NW; ++g) {
                if (g == warp) o = nc;
                nc += s_g[g];
            }
            if (mine) s_p[o + __popc(b & ((1u << lane) - 1u))] = rec;
            cn += nc;
            block_sync_any();
            const int np = nc >> 1;
            if (tid < np) {                                   // pair records, fp64 then one rounding
                const double2 a = s_p[2 * tid], bb = s_p[2 * tid + 1];
                s_q[tid] = make_float4((float)(0.5 * (a.x + bb.x)), (float)(0.5 * (a.y + bb.y)),
                                       (float)(0.5 * (a.x - bb.x)), (float)(0.5 * (a.y - bb.y)));
            }
            block_sync_any();
#pragma unroll 1
            for (int p = 0; p < np; ++p) acc.pair(w, s_q[p]);     // warp-uniform broadcasts
            if (nc & 1) {
                const double2 a = s_p[nc - 1];
                acc.single(w, (float)a.x, (float)a.y);
            }
        }
#pragma unroll
        for (int j = 0; j < KT; ++j) {
            const int k = kbase + j * THREADS;
            if (OUTL) {
                if (k < nu.D) {
                    const float2 v = acc.get(j);
                    atomicAdd(nu.pending + 2 * ((size_t)cls * Dp + k), (double)v.x);
                    atomicAdd(nu.pending + 2 * ((size_t)cls * Dp + k) + 1, (double)v.y);
                }
            } else if (k < Dp) {
                part[((size_t)chunk * 2 + cls) * Dp + k] = acc.get(j);
            }
        }
    };
    if (role_b) run(PairAcc<KT, NPB>{});
    else run(PairAcc<KT, NPA>{});
    if (!OUTL && kb == 0) {
        if (my_err && cls == 0) atomicOr(err, my_err);
        if (tid == 0) part_cnt[chunk * 2 + cls] = cn;
    }
}


// Quadrant routing (delta > 1; Alg. 1): slot = 2 beta + psi with
// beta the nearest quadrant centre in fp64 squared distance, ties to the lowest
// index -- the expression, operation order and rounding DESIGN.md fixes for the decision
// (explicit _rn intrinsics: no FMA contraction).  255 = invalid point (deferred error).
__global__ void k_route(const float2 *__restrict__ xy, const uint8_t *__restrict__ lab, int64_t n,
                        const double *__restrict__ qc, int nq, uint8_t *__restrict__ slot, int *__restrict__ err)
{
    __shared__ double s_qc[2 * VSAOGM_MAX_DELTA * VSAOGM_MAX_DELTA];
    for (int k = threadIdx.x; k < 2 * nq; k += blockDim.x) s_qc[k] = qc[k];
    __syncthreads();
    int my_err = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const float2 v = xy[i];
        const int L = lab[i];
        uint8_t s = 255;
        if (L > 1) my_err |= VSA_ERRBIT_LABEL;
        else if (!(isfinite(v.x) && isfinite(v.y))) my_err |= VSA_ERRBIT_NONFINITE;
        else {
            const double x = (double)v.x, y = (double)v.y;
            int best = 0;
            double bd = 0.0;
            for (int k = 0; k < nq; ++k) {
                const double dx = __dsub_rn(x, s_qc[2 * k]), dy = __dsub_rn(y, s_qc[2 * k + 1]);
                const double d = __dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy));
                if (k == 0 || d < bd) { bd = d; best = k; }
            }
            s = (uint8_t)(2 * best + L);
        }
        slot[i] = s;
    }
    if (my_err) atomicOr(err, my_err);
}

// Slot-filtered encode: block (kb, chunk, z) bundles the points of its chunk whose
// memory slot is z (slot = label for delta = 1, else the routed 2 beta + psi), so
// every block keeps one accumulator set.  Same phasor arithmetic as k_encode_bundle;
// points of other slots are only staged (cost ~0.3 % per slot).
template <int KT, int NPOLY, int MINB = 6>
__global__ void __launch_bounds__(ENC_THREADS, MINB) k_encode_slots(
    const float2 *__restrict__ xy, const uint8_t *__restrict__ lab, const uint8_t *__restrict__ slot, int64_t n,
    int64_t chunk_pts, const float *__restrict__ wx, const float *__restrict__ wy, double cx, double cy, int Dp,
    int nslots, float2 *__restrict__ part, long long *__restrict__ part_cnt, int *__restrict__ err)
{
    constexpr int NW = ENC_THREADS / 32;
    constexpr int ROUNDS = ENC_TILE / ENC_THREADS;
    __shared__ float4 s_p[ENC_TILE];
    __shared__ int s_g[ROUNDS * NW];
    const int tid = threadIdx.x;
    const int lane = tid & 31, warp = tid >> 5;
    const int kb = blockIdx.x;
    const int64_t chunk = blockIdx.y;
    const int z = blockIdx.z;
    const int kbase = kb * ENC_THREADS * KT + tid;

    float fx[KT], fy[KT], ar[KT], ai[KT];
#pragma unroll
    for (int j = 0; j < KT; ++j) {
        const int k = kbase + j * ENC_THREADS;
        fx[j] = k < Dp ? wx[k] : 0.f;
        fy[j] = k < Dp ? wy[k] : 0.f;
        ar[j] = ai[j] = 0.f;
    }
    long long cnt_z = 0;
    int my_err = 0;
    const int64_t p0 = chunk * chunk_pts;
    const int64_t p1 = min(n, p0 + chunk_pts);

    for (int64_t base = p0; base < p1; base += ENC_TILE) {
        const int cnt = (int)min((int64_t)ENC_TILE, p1 - base);
        __syncthreads();
        float4 rec[ROUNDS];
        bool mine[ROUNDS];
        unsigned b[ROUNDS];
#pragma unroll
        for (int r = 0; r < ROUNDS; ++r) {
            const int t = tid + r * ENC_THREADS;
            mine[r] = false;
            rec[r] = make_float4(0.f, 0.f, 0.f, 0.f);
            if (t < cnt) {
                const float2 v = xy[base + t];
                int sl;
                if (slot) {
                    sl = slot[base + t];
                } else {
                    const int L = lab[base + t];
                    sl = L;
                    if (L > 1) { sl = 255; my_err |= VSA_ERRBIT_LABEL; }
                    if (!(isfinite(v.x) && isfinite(v.y))) { sl = 255; my_err |= VSA_ERRBIT_NONFINITE; }
                }
                mine[r] = sl == z;
                rec[r] = make_float4((float)((double)v.x - cx), (float)((double)v.y - cy), 0.f, 0.f);
            }
            b[r] = __ballot_sync(0xffffffffu, mine[r]);
            if (lane == 0) s_g[r * NW + warp] = __popc(b[r]);
        }
        __syncthreads();
        int nz = 0, o[ROUNDS];
#pragma unroll
        for (int g = 0; g < ROUNDS * NW; ++g) {
#pragma unroll
            for (int r = 0; r < ROUNDS; ++r)
                if (g == r * NW + warp) o[r] = nz;
            nz += s_g[g];
        }
        const unsigned lt = (1u << lane) - 1u;
#pragma unroll
        for (int r = 0; r < ROUNDS; ++r)
            if (mine[r]) s_p[o[r] + __popc(b[r] & lt)] = rec[r];
        cnt_z += nz;
        __syncthreads();
#pragma unroll 2
        for (int p = 0; p < nz; ++p) {
            const float4 P = s_p[p];                    // warp-uniform broadcast
#pragma unroll
            for (int j = 0; j < KT; ++j) {
                float sv, cv;
                phasor<KT, NPOLY>(j, fmaf(fx[j], P.x, fy[j] * P.y), &sv, &cv);
                ar[j] += cv;
                ai[j] += sv;
            }
        }
    }
#pragma unroll
    for (int j = 0; j < KT; ++j) {
        const int k = kbase + j * ENC_THREADS;
        if (k < Dp) part[((size_t)chunk * nslots + z) * Dp + k] = make_float2(ar[j], ai[j]);
    }
    if (kb == 0) {
        if (my_err && z == 0) atomicOr(err, my_err);
        if (tid == 0) part_cnt[chunk * nslots + z] = cnt_z;
    }
}

// K3: pending[c][k] += sum over chunks of the partials, fp64, fixed order: block =
// 32 column lanes (two k each: one 16-byte load per chunk row) x RED_SLICES chunk slices;
// slice s sums chunks s, s+S, ... in order, then the slice sums are added in slice order
// (deterministic).  Bandwidth-bound: 16 slices keep ~8 loads per thread in flight.
constexpr int RED_SLICES = 16;
__global__ void __launch_bounds__(32 * RED_SLICES) k_reduce_partials(
    const float2 *__restrict__ part, const long long *__restrict__ part_cnt, int chunks, int nslots, int Dp, int D,
    double *__restrict__ pending, double *__restrict__ pcount)
{
    __shared__ double4 s_acc[RED_SLICES][32];
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    const int ncol = nslots * Dp / 2;               // float4 columns: (slot, k pair)
    const int col = blockIdx.x * 32 + tx;
    const bool live = col < ncol;
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    if (live) {
        const float4 *p = reinterpret_cast<const float4 *>(part) + col;
#pragma unroll 8
        for (int ch = ty; ch < chunks; ch += RED_SLICES) {
            const float4 v = __ldcs(p + (size_t)ch * ncol);   // read once: evict-first
            a0 += v.x;
            a1 += v.y;
            a2 += v.z;
            a3 += v.w;
        }
    }
    s_acc[ty][tx] = make_double4(a0, a1, a2, a3);
    __syncthreads();
    if (ty == 0 && live) {
        double4 r = s_acc[0][tx];
#pragma unroll
        for (int s = 1; s < RED_SLICES; ++s) {
            const double4 v = s_acc[s][tx];
            r.x += v.x;
            r.y += v.y;
            r.z += v.z;
            r.w += v.w;
        }
        const int idx = 2 * col;                    // (slot, k) of the first of the pair
        const int c = idx / Dp, k = idx - c * Dp;
        // padding dimensions (w = 0 accumulate cos 0 = 1) stay exactly zero
        if (k < D) {
            pending[2 * (size_t)idx] += r.x;
            pending[2 * (size_t)idx + 1] += r.y;
        }
        if (k + 1 < D) {
            pending[2 * (size_t)idx + 2] += r.z;
            pending[2 * (size_t)idx + 3] += r.w;
        }
    }
    if (blockIdx.x == 0) {   // counts: integer sums (exact in any order: integer-valued fp64 < 2^53)
        for (int sl = 0; sl < nslots; ++sl) {
            long long s = 0;
            for (int ch = threadIdx.x; ch < chunks; ch += blockDim.x) s += part_cnt[ch * nslots + sl];
            if (s) atomicAdd(&pcount[sl], (double)s);
        }
    }
}

// Commit: m += pending, pending = 0 (Alg. 3 result folded into the memories).
__global__ void k_commit(double *__restrict__ m, double *__restrict__ pending, long long *__restrict__ cnt,
                         double *__restrict__ pcnt, int n, int nslots)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) {
        m[i] += pending[i];
        pending[i] = 0.0;
    }
    if (blockIdx.x == 0 && threadIdx.x < nslots) {
        cnt[threadIdx.x] += (long long)pcnt[threadIdx.x];
        pcnt[threadIdx.x] = 0.0;
    }
}

// Optional commit (m += pending, pending = 0), then ||m_c||^2 per memory slot (Eq. 10): grid
// (slot, nb <= NORM_BLOCKS k-ranges, nb fixed per Dp); each block commits its range and reduces
// it with a fixed tree into normpart[slot][b]; the last block of a slot to finish (atomic
// ticket) adds the slot's nb partials in a fixed order (deterministic) into norm2 -- an ordinary
// launch, no grid barrier.  The table-A kernel scales m by sqrt(D) / ||m|| itself (k_mhat
// writes the scaled fp32 copy only for the on-the-fly phasor-tile GEMM, gemm_agen).
constexpr int NORM_THREADS = 256, NORM_BLOCKS = 16;
__global__ void __launch_bounds__(NORM_THREADS) k_commit_norms(double *__restrict__ m, double *__restrict__ pending,
                                                               long long *__restrict__ cnt, double *__restrict__ pcnt,
                                                               int do_commit, int Dp, int D, double *__restrict__ normpart,
                                                               unsigned int *__restrict__ ticket,
                                                               double *__restrict__ norm2)
{
    vsa_pdl();
    __shared__ double s[NORM_THREADS];
    __shared__ bool s_last;
    const int c = blockIdx.x, b = blockIdx.y, nb = gridDim.y;
    const int per = (Dp + nb - 1) / nb;
    const int k1 = min(Dp, (b + 1) * per);
    double acc = 0.0;
    for (int k = b * per + threadIdx.x; k < k1; k += NORM_THREADS) {
        const size_t o = 2 * ((size_t)c * Dp + k);
        double re = m[o], im = m[o + 1];
        if (do_commit) {
            re += pending[o];
            im += pending[o + 1];
            m[o] = re;
            m[o + 1] = im;
            pending[o] = 0.0;
            pending[o + 1] = 0.0;
        }
        acc += re * re + im * im;
    }
    s[threadIdx.x] = acc;
    __syncthreads();
    for (int o = NORM_THREADS / 2; o > 0; o >>= 1) {
        if (threadIdx.x < o) s[threadIdx.x] += s[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        normpart[c * NORM_BLOCKS + b] = s[0];
        __threadfence();   // the partial and this block's m are visible before the ticket
        s_last = atomicAdd(ticket + c, 1u) == (unsigned)nb - 1;
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    __shared__ double s_n2;
    if (threadIdx.x < 32) {   // fixed order: lane-strided, then a butterfly
        double v = 0.0;
        for (int i = threadIdx.x; i < nb; i += 32) v += __ldcg(normpart + c * NORM_BLOCKS + i);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (threadIdx.x == 0) {
            s_n2 = v;
            ticket[c] = 0u;   // ready for the next launch (stream-ordered)
        }
    }
    __syncthreads();
    const double n2 = s_n2;
    if (threadIdx.x == 0) {
        norm2[c] = n2;
        norm2[gridDim.x + c] = n2 > 0.0 ? sqrt((double)D / n2) : 0.0;   // the table-A scale
        if (do_commit) {
            cnt[c] += (long long)pcnt[c];
            pcnt[c] = 0.0;
        }
    }
}

// mhat_c = sqrt(D) m_c / ||m_c|| (0 for an empty class, L8) in fp32: the same expression as the
// table-A kernel's
__global__ void __launch_bounds__(256) k_mhat(const double2 *__restrict__ m, const double *__restrict__ norm2, int D,
                                              int Dp, int n, float2 *__restrict__ mhat)
{
    const int i = blockIdx.x * 256 + threadIdx.x;
    if (i >= n) return;
    const double n2 = norm2[i / Dp];
    const double sc = n2 > 0.0 ? sqrt((double)D / n2) : 0.0;
    const double2 v = m[i];
    mhat[i] = make_float2((float)(v.x * sc), (float)(v.y * sc));
}

}  // namespace

int vsa_launch_nufft_outliers(vsaogm_ctx *c, const float *xy, const uint8_t *lab, int64_t n, int64_t chunk_pts,
                              int chunks)
{
    NuOutl nu{c->nu_lo, 1.0 / c->nu_h, c->nu_n1, c->d_nu_out, c->d_pending, c->D};
    const int kblocks = (c->Dp + 2047) / 2048;
    VSA_CUDA_TRY(vsa_launch(c, k_encode_pairs1<256, 0, 4, 4, true>, dim3(kblocks, chunks, 2), dim3(256), 0, (const float2 *)xy, lab, n,
                            chunk_pts, (const float *)c->d_wx, (const float *)c->d_wy, c->cx, c->cy, c->Dp, (float2 *)nullptr,
                            (long long *)nullptr, c->d_err, nu));
    c->launches++;
    return VSAOGM_OK;
}

int vsa_launch_encode(vsaogm_ctx *c, const float *xy, const uint8_t *lab, int64_t n)
{
    // default (enc_path 0): counting sort by slot + equal runs (encode_sorted.cu).
    // Measured alternatives kept as tuning variants: enc_path 1 = label-split blocks
    // (delta = 1) / slot-filtered blocks (delta > 1); enc_path 2 = slot-filtered always.
    if (c->enc_path == 0 || (c->enc_path < 0 && c->nslots > 2)) return vsa_launch_encode_sorted(c, xy, lab, n);
    if (vsa_nufft_wanted(c, n)) {
        // type-3 NUFFT (nufft.cu) + direct fallback for the points outside its grid; the chunks
        // are those of the direct kernel (4 waves of 4 blocks per SM over the k-blocks)
        const int kblocks = (c->Dp + 2047) / 2048;
        int64_t chunks = std::max<int64_t>(1, std::min<int64_t>((int64_t)c->num_sms * 4 * 4 / (2 * kblocks), (n + 63) / 64));
        const int64_t chunk_pts = (n + chunks - 1) / chunks;
        chunks = (n + chunk_pts - 1) / chunk_pts;
        cudaEvent_t ev;
        vsa_prof_begin(c, VSAOGM_K_ENCODE, &ev);
        int rc = vsa_launch_encode_nufft(c, xy, lab, n, chunk_pts, (int)chunks);
        if (!rc) rc = vsa_launch_nufft_outliers(c, xy, lab, n, chunk_pts, (int)chunks);
        vsa_prof_end(c, VSAOGM_K_ENCODE, ev);
        return rc;
    }
    const bool slots_path = c->nslots > 2 || c->enc_path == 2;
    const int KT = (!slots_path && c->enc_kt == 16 && c->Dp >= 2048) ? 16 : (c->Dp >= 1024 ? 8 : 4);
    // packed kernel: 128 threads (enc_x2 = 1) or 8-warp role variants (2, 3: 2048 dims per block)
    const bool x2 = !slots_path && KT == 8 && c->enc_x2 && (c->enc_x2 == 1 || c->Dp >= 2048);
    const int x2_threads = (x2 && c->enc_x2 >= 2) ? 256 : ENC_THREADS;
    const int kblocks = (c->Dp + x2_threads * KT - 1) / (x2_threads * KT);
    // one full wave at ~6 resident blocks per SM (3 for the 256-thread variants), at least 64
    // points per chunk; 7 or 8 resident blocks as tuning variants of the scalar kernel
    const int minb = x2 ? (x2_threads == 256 ? (c->enc_x2 == 4 ? c->enc_pairs_minb : (c->enc_x2_minb == 4 ? 4 : 3)) : 6)
                     : KT == 16 ? 4
                     : (!slots_path && KT == 8 && (c->enc_npoly == 1 || c->enc_npoly == 2) &&
                        (c->enc_minb == 7 || c->enc_minb == 8))
                         ? c->enc_minb
                         : 6;
    const int zslots = slots_path ? c->nslots : 1;     // grid.z
    // slot-filtered blocks carry unequal work (slots hold different point counts): several
    // waves of smaller blocks even the tail out
    const bool split1 = x2 && c->enc_x2 == 4 && c->enc_pairs_split;   // grid.z = 2 classes
    const int minb_eff = split1 ? 4 : minb;
    const int64_t target_blocks =
        (int64_t)c->num_sms * minb_eff * (slots_path ? c->enc_waves : x2 ? c->enc_x2_waves : 1);
    int64_t chunks = (target_blocks + (int64_t)kblocks * zslots * (split1 ? 2 : 1) - 1) /
                     ((int64_t)kblocks * zslots * (split1 ? 2 : 1));
    chunks = std::max<int64_t>(1, std::min<int64_t>(chunks, (n + 63) / 64));
    const int64_t chunk_pts = (n + chunks - 1) / chunks;
    chunks = (n + chunk_pts - 1) / chunk_pts;
    const size_t need = (size_t)chunks * c->nslots * c->Dp;
    if (need > c->part_cap) {
        if (c->d_part) cudaFree(c->d_part);
        if (cudaMalloc(&c->d_part, need * sizeof(float2)) != cudaSuccess) { c->d_part = nullptr; c->part_cap = 0; return VSAOGM_ENOMEM; }
        c->part_cap = need;
    }
    if ((size_t)chunks * c->nslots > c->part_cnt_cap) {
        if (c->d_part_cnt) cudaFree(c->d_part_cnt);
        if (cudaMalloc(&c->d_part_cnt, chunks * c->nslots * sizeof(long long)) != cudaSuccess) { c->d_part_cnt = nullptr; c->part_cnt_cap = 0; return VSAOGM_ENOMEM; }
        c->part_cnt_cap = chunks * c->nslots;
    }
    cudaEvent_t ev;
    const uint8_t *slot = nullptr;
    if (c->nslots > 2) {
        if ((size_t)n > c->slot_cap) {
            if (c->d_slot) cudaFree(c->d_slot);
            if (cudaMalloc(&c->d_slot, n) != cudaSuccess) { c->d_slot = nullptr; c->slot_cap = 0; return VSAOGM_ENOMEM; }
            c->slot_cap = n;
        }
        vsa_prof_begin(c, VSAOGM_K_ENCODE, &ev);
        const int rblocks = (int)std::min<int64_t>((n + 255) / 256, (int64_t)c->num_sms * 8);
        k_route<<<rblocks, 256, 0, c->stream>>>((const float2 *)xy, lab, n, c->d_qc, c->nq, c->d_slot, c->d_err);
        VSA_CUDA_TRY(cudaGetLastError());
        vsa_prof_end(c, VSAOGM_K_ENCODE, ev);
        c->launches++;
        slot = c->d_slot;
    }
    vsa_prof_begin(c, VSAOGM_K_ENCODE, &ev);
    if (slots_path) {
        dim3 grid(kblocks, (unsigned)chunks, (unsigned)zslots);
#define VSA_ENC_SLOTS(KT_, NP_)                                                                                     \
    k_encode_slots<KT_, NP_><<<grid, ENC_THREADS, 0, c->stream>>>((const float2 *)xy, lab, slot, n, chunk_pts,       \
                                                                  c->d_wx, c->d_wy, c->cx, c->cy, c->Dp, c->nslots, \
                                                                  c->d_part, c->d_part_cnt, c->d_err)
        if (KT == 8) {
            if (c->enc_npoly == 2) VSA_ENC_SLOTS(8, 2);
            else if (c->enc_npoly == 0) VSA_ENC_SLOTS(8, 0);
            else VSA_ENC_SLOTS(8, 1);
        } else {
            if (c->enc_npoly == 0) VSA_ENC_SLOTS(4, 0);
            else VSA_ENC_SLOTS(4, 1);
        }
#undef VSA_ENC_SLOTS
    } else {
    dim3 grid(kblocks, (unsigned)chunks);
#define VSA_ENC_X2(T_, NPA_, NPB_, MB_)                                                                            \
    k_encode_bundle_x2<T_, NPA_, NPB_, MB_><<<grid, T_, 0, c->stream>>>(                                          \
        (const float2 *)xy, lab, n, chunk_pts, c->d_wx, c->d_wy, c->cx, c->cy, c->Dp, c->d_part, c->d_part_cnt,  \
        c->d_err)
#define VSA_ENC_LAUNCH(KT_, NP_, ...)                                                                             \
    k_encode_bundle<KT_, NP_, ##__VA_ARGS__><<<grid, ENC_THREADS, 0, c->stream>>>(                                \
        (const float2 *)xy, lab, n, chunk_pts, c->d_wx, c->d_wy, c->cx, c->cy, c->Dp, c->d_part, c->d_part_cnt,  \
        c->d_err)
#define VSA_ENC_PAIRS(NPB_, MB_)                                                                                   \
    k_encode_pairs<256, 0, NPB_, MB_><<<grid, 256, 0, c->stream>>>(                                               \
        (const float2 *)xy, lab, n, chunk_pts, c->d_wx, c->d_wy, c->cx, c->cy, c->Dp, c->d_part, c->d_part_cnt,  \
        c->d_err)
#define VSA_ENC_PAIRS1(NPB_, MB_)                                                                                  \
    k_encode_pairs1<256, 0, NPB_, MB_><<<dim3(grid.x, grid.y, 2), 256, 0, c->stream>>>(                            \
        (const float2 *)xy, lab, n, chunk_pts, c->d_wx, c->d_wy, c->cx, c->cy, c->Dp, c->d_part, c->d_part_cnt,  \
        c->d_err)
    if (x2 && c->enc_x2 == 4 && c->enc_pairs_split) {   // pairs, one class per block
        switch (c->enc_pairs_npoly) {
        case 0: VSA_ENC_PAIRS1(0, 4); break;
        case 2: VSA_ENC_PAIRS1(2, 4); break;
        case 6: VSA_ENC_PAIRS1(6, 4); break;
        case 8: VSA_ENC_PAIRS1(8, 4); break;
        default: VSA_ENC_PAIRS1(4, 4); break;
        }
    } else if (x2 && c->enc_x2 == 4) {   // pairs (half-angle): all-MUFU warps beside NPOLY-FMA-pipe warps
        const bool mb4 = c->enc_pairs_minb == 4;
        switch (c->enc_pairs_npoly) {
        case 0: if (mb4) VSA_ENC_PAIRS(0, 4); else VSA_ENC_PAIRS(0, 3); break;
        case 2: if (mb4) VSA_ENC_PAIRS(2, 4); else VSA_ENC_PAIRS(2, 3); break;
        case 6: if (mb4) VSA_ENC_PAIRS(6, 4); else VSA_ENC_PAIRS(6, 3); break;
        case 8: if (mb4) VSA_ENC_PAIRS(8, 4); else VSA_ENC_PAIRS(8, 3); break;
        default: if (mb4) VSA_ENC_PAIRS(4, 4); else VSA_ENC_PAIRS(4, 3); break;
        }
    } else if (x2 && c->enc_x2 == 1) {   // uniform roles, 4 warps
        switch (c->enc_x2_npoly) {
        case 1: VSA_ENC_X2(128, 1, 1, 6); break;
        case 3: VSA_ENC_X2(128, 3, 3, 6); break;
        case 4: VSA_ENC_X2(128, 4, 4, 6); break;
        default: VSA_ENC_X2(128, 2, 2, 6); break;
        }
    } else if (x2 && c->enc_x2 == 2) {   // all-MUFU warps beside NPOLY-polynomial warps (default: 4)
        switch (c->enc_x2_npoly) {
        case 4:
            if (c->enc_x2_minb == 4) VSA_ENC_X2(256, 0, 4, 4);
            else VSA_ENC_X2(256, 0, 4, 3);
            break;
        case 5:
            if (c->enc_x2_minb == 4) VSA_ENC_X2(256, 0, 5, 4);
            else VSA_ENC_X2(256, 0, 5, 3);
            break;
        case 7: VSA_ENC_X2(256, 0, 7, 3); break;
        case 8: VSA_ENC_X2(256, 0, 8, 3); break;
        default:
            if (c->enc_x2_minb == 4) VSA_ENC_X2(256, 0, 6, 4);
            else VSA_ENC_X2(256, 0, 6, 3);
            break;
        }
    } else if (x2) {   // 1-polynomial warps beside NPOLY-polynomial warps
        switch (c->enc_x2_npoly) {
        case 4: VSA_ENC_X2(256, 1, 4, 3); break;
        default: VSA_ENC_X2(256, 1, 5, 3); break;
        }
    } else if (KT == 8) {
        switch (c->enc_npoly) {
        case 0: VSA_ENC_LAUNCH(8, 0); break;
        case 2:
            if (minb == 8) VSA_ENC_LAUNCH(8, 2, 8);
            else if (minb == 7) VSA_ENC_LAUNCH(8, 2, 7);
            else VSA_ENC_LAUNCH(8, 2);
            break;
        case 3: VSA_ENC_LAUNCH(8, 3); break;
        case 4: VSA_ENC_LAUNCH(8, 4); break;
        default:
            if (minb == 8) VSA_ENC_LAUNCH(8, 1, 8);
            else if (minb == 7) VSA_ENC_LAUNCH(8, 1, 7);
            else VSA_ENC_LAUNCH(8, 1);
            break;
        }
    } else if (KT == 16) {   // tuning variant: 16 dimensions per thread (4 blocks per SM)
        switch (c->enc_npoly) {
        case 2: VSA_ENC_LAUNCH(16, 2, 4); break;
        case 4: VSA_ENC_LAUNCH(16, 4, 4); break;
        default: VSA_ENC_LAUNCH(16, 3, 4); break;
        }
    } else {
        if (c->enc_npoly == 0) VSA_ENC_LAUNCH(4, 0);
        else VSA_ENC_LAUNCH(4, 1);
    }
#undef VSA_ENC_LAUNCH
#undef VSA_ENC_X2
#undef VSA_ENC_PAIRS
#undef VSA_ENC_PAIRS1
    }
    VSA_CUDA_TRY(cudaGetLastError());
    vsa_prof_end(c, VSAOGM_K_ENCODE, ev);
    c->launches++;

    vsa_prof_begin(c, VSAOGM_K_REDUCE, &ev);
    k_reduce_partials<<<(c->nslots * c->Dp / 2 + 31) / 32, 32 * RED_SLICES, 0, c->stream>>>(
        c->d_part, c->d_part_cnt, (int)chunks, c->nslots, c->Dp, c->D, c->d_pending, c->d_pcounts);
    VSA_CUDA_TRY(cudaGetLastError());
    vsa_prof_end(c, VSAOGM_K_REDUCE, ev);
    c->launches++;
    return VSAOGM_OK;
}

int vsa_launch_commit(vsaogm_ctx *c)
{
    cudaEvent_t ev;
    vsa_prof_begin(c, VSAOGM_K_COMMIT, &ev);
    const int n = 2 * c->nslots * c->Dp;
    k_commit<<<(n + 255) / 256, 256, 0, c->stream>>>(c->d_m, c->d_pending, c->d_counts, c->d_pcounts, n, c->nslots);
    VSA_CUDA_TRY(cudaGetLastError());
    vsa_prof_end(c, VSAOGM_K_COMMIT, ev);
    c->launches++;
    return VSAOGM_OK;
}

int vsa_launch_norms(vsaogm_ctx *c, int do_commit)
{
    cudaEvent_t ev;
    vsa_prof_begin(c, VSAOGM_K_NORMS, &ev);
    {
        double *m = c->d_m, *pend = c->d_pending, *np = c->d_normpart, *n2 = c->d_norm2;
        long long *cnt = c->d_counts;
        double *pcnt = c->d_pcounts;
        // nb fixed per Dp (so the norm's summation order is too); tickets after the partials
        const int nb = std::max(1, std::min(NORM_BLOCKS, (c->Dp + 2 * NORM_THREADS - 1) / (2 * NORM_THREADS)));
        VSA_CUDA_TRY(vsa_launch(c, k_commit_norms, dim3(c->nslots, nb), dim3(NORM_THREADS), 0, m, pend, cnt, pcnt, do_commit, c->Dp,
                                c->D, np, reinterpret_cast<unsigned int *>(np + (size_t)c->nslots * NORM_BLOCKS), n2));

    }
    VSA_CUDA_TRY(cudaGetLastError());
    vsa_prof_end(c, VSAOGM_K_NORMS, ev);
    c->launches++;
    return VSAOGM_OK;
}

// the scaled fp32 memories for the on-the-fly phasor-tile GEMM (gemm_agen), from the committed
// memories and the norms of the last vsa_launch_norms
int vsa_launch_mhat(vsaogm_ctx *c)
{
    const int n = c->nslots * c->Dp;
    k_mhat<<<(n + 255) / 256, 256, 0, c->stream>>>((const double2 *)c->d_m, c->d_norm2, c->D, c->Dp, n, c->d_mhat);
    VSA_CUDA_TRY(cudaGetLastError());
    c->launches++;
    return VSAOGM_OK;
}
