// encode_sorted.cu -- encode/bundle through a stable counting sort of the points by memory slot.
//
// Alg. 1 sends point i to memory omega_{2 beta + psi_i}; with
// delta > 1 there are 2 delta^2 memories (sec. III-B-4).  A
// block can only keep one memory's accumulators in registers, and the memories
// hold very different numbers of points, so the points are first sorted by slot
// (stable, deterministic) and cut into equal-size runs of one slot each; the
// encode blocks then carry equal work (one wave) and the partial sums stay small.
//
//   k_route_hist  slot per point (delta = 1: the label; else the nearest quadrant
//                 centre in fp64, ties to the lowest index), per-block histograms
//   k_sort_plan   per-slot totals, per-(block, slot) offsets, the table of runs
//   k_scatter     stable scatter of the centred coordinates into slot order
//   k_encode_runs one run per block row: E_k = exp(i (w^x x + w^y y)), summed (Eq. 9, 5)
//   k_reduce_runs pending[slot][k] += sum of the slot's runs, fp64, fixed order
#include "common.cuh"

namespace {

constexpr int RT_THREADS = 256;
constexpr int RT_PTS = 4096;                 // points per routing / scatter block
constexpr int ENC_T = 128;                   // encode threads
constexpr int ENC_TILE_S = 512;              // staged points per tile
constexpr int MAX_SLOTS = 2 * VSAOGM_MAX_DELTA * VSAOGM_MAX_DELTA;

// meta layout (int): total[MAX_SLOTS], slot_start[MAX_SLOTS+1], run_start[MAX_SLOTS+1], n_runs
__host__ __device__ constexpr int META_TOTAL() { return 0; }
__host__ __device__ constexpr int META_SSTART() { return MAX_SLOTS; }
__host__ __device__ constexpr int META_RSTART() { return 2 * MAX_SLOTS + 1; }
__host__ __device__ constexpr int META_NRUNS() { return 3 * MAX_SLOTS + 2; }
__host__ __device__ constexpr int META_INTS() { return 3 * MAX_SLOTS + 3; }

__global__ void __launch_bounds__(RT_THREADS) k_route_hist(const float2 *__restrict__ xy, const uint8_t *__restrict__ lab,
                                                           int64_t n, const double *__restrict__ qc, int nq,
                                                           int nslots, uint8_t *__restrict__ slot,
                                                           int *__restrict__ bhist, int *__restrict__ err)
{
    __shared__ double s_qc[2 * VSAOGM_MAX_DELTA * VSAOGM_MAX_DELTA];
    __shared__ int s_h[MAX_SLOTS];
    for (int k = threadIdx.x; k < 2 * nq; k += RT_THREADS) s_qc[k] = qc[k];
    for (int k = threadIdx.x; k < nslots; k += RT_THREADS) s_h[k] = 0;
    __syncthreads();
    int my_err = 0;
    const int64_t b0 = (int64_t)blockIdx.x * RT_PTS;
    for (int t = threadIdx.x; t < RT_PTS; t += RT_THREADS) {
        const int64_t i = b0 + t;
        if (i >= n) break;
        const float2 v = xy[i];
        const int L = lab[i];
        int s = 255;
        if (L > 1) my_err |= VSA_ERRBIT_LABEL;
        else if (!(isfinite(v.x) && isfinite(v.y))) my_err |= VSA_ERRBIT_NONFINITE;
        else {
            int best = 0;
            if (nq > 1) {   // Alg. 1 argmin, fp64, no FMA contraction, ties to the lowest index
                const double x = (double)v.x, y = (double)v.y;
                double bd = 0.0;
                for (int k = 0; k < nq; ++k) {
                    const double dx = __dsub_rn(x, s_qc[2 * k]), dy = __dsub_rn(y, s_qc[2 * k + 1]);
                    const double d = __dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy));
                    if (k == 0 || d < bd) { bd = d; best = k; }
                }
            }
            s = 2 * best + L;
            atomicAdd(&s_h[s], 1);
        }
        slot[i] = (uint8_t)s;
    }
    if (my_err) atomicOr(err, my_err);
    __syncthreads();
    for (int k = threadIdx.x; k < nslots; k += RT_THREADS) bhist[(size_t)blockIdx.x * nslots + k] = s_h[k];
}

// single block: per-slot totals and per-(block, slot) exclusive offsets (in place in
// bhist), slot starts, and runs of at most `run_pts` points of one slot
__global__ void __launch_bounds__(1024) k_sort_plan(int *__restrict__ bhist, int nblk, int nslots, int run_pts,
                                                    int *__restrict__ meta, int4 *__restrict__ runs)
{
    const int s = threadIdx.x;
    if (s < nslots) {
        int run = 0;
        for (int b = 0; b < nblk; ++b) {
            const int h = bhist[(size_t)b * nslots + s];
            bhist[(size_t)b * nslots + s] = run;
            run += h;
        }
        meta[META_TOTAL() + s] = run;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        int ss = 0, rs = 0;
        for (int k = 0; k < nslots; ++k) {
            meta[META_SSTART() + k] = ss;
            meta[META_RSTART() + k] = rs;
            const int t = meta[META_TOTAL() + k];
            ss += t;
            rs += (t + run_pts - 1) / run_pts;
        }
        meta[META_SSTART() + nslots] = ss;
        meta[META_RSTART() + nslots] = rs;
        meta[META_NRUNS()] = rs;
    }
    __syncthreads();
    if (s < nslots) {
        const int t = meta[META_TOTAL() + s], base = meta[META_SSTART() + s];
        int r = meta[META_RSTART() + s];
        for (int p = 0; p < t; p += run_pts, ++r) runs[r] = make_int4(s, base + p, base + min(t, p + run_pts), 0);
    }
}

// stable scatter: within a block, points keep their index order inside each slot
__global__ void __launch_bounds__(RT_THREADS) k_scatter(const float2 *__restrict__ xy, const uint8_t *__restrict__ slot,
                                                        int64_t n, int nslots, const int *__restrict__ boff,
                                                        const int *__restrict__ meta, double cx, double cy,
                                                        double2 *__restrict__ sorted)
{
    constexpr int NW = RT_THREADS / 32;
    __shared__ int s_run[MAX_SLOTS];
    __shared__ int s_w[NW][MAX_SLOTS];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int k = threadIdx.x; k < nslots; k += RT_THREADS) s_run[k] = 0;
    for (int k = threadIdx.x; k < NW * MAX_SLOTS; k += RT_THREADS) (&s_w[0][0])[k] = 0;
    __syncthreads();
    const int64_t b0 = (int64_t)blockIdx.x * RT_PTS;
    const unsigned lt = (1u << lane) - 1u;
    for (int base = 0; base < RT_PTS; base += RT_THREADS) {
        const int64_t i = b0 + base + threadIdx.x;
        const int s = i < n ? slot[i] : 255;
        const unsigned peers = __match_any_sync(0xffffffffu, s);
        const int rank = __popc(peers & lt);
        if (s != 255 && rank == 0) s_w[warp][s] = __popc(peers);
        __syncthreads();
        if (s != 255) {
            int off = s_run[s];
            for (int w = 0; w < warp; ++w) off += s_w[w][s];
            const int pos = meta[META_SSTART() + s] + boff[(size_t)blockIdx.x * nslots + s] + off + rank;
            const float2 v = xy[i];
            sorted[pos] = make_double2((double)v.x - cx, (double)v.y - cy);
        }
        __syncthreads();
        for (int k = threadIdx.x; k < nslots; k += RT_THREADS) {
            int t = 0;
            for (int w = 0; w < NW; ++w) { t += s_w[w][k]; s_w[w][k] = 0; }
            s_run[k] += t;
        }
        __syncthreads();
    }
}

template <int KT, int NPOLY>
__global__ void __launch_bounds__(ENC_T, 6) k_encode_runs(const double2 *__restrict__ sorted, const int4 *__restrict__ runs,
                                                          const int *__restrict__ meta, const float *__restrict__ wx,
                                                          const float *__restrict__ wy, int Dp,
                                                          float2 *__restrict__ part)
{
    __shared__ float2 s_p[ENC_TILE_S];
    const int r = blockIdx.y;
    if (r >= meta[META_NRUNS()]) return;
    const int4 run = runs[r];
    const int tid = threadIdx.x;
    const int kbase = blockIdx.x * ENC_T * KT + tid;
    float fx[KT], fy[KT], ar[KT], ai[KT];
#pragma unroll
    for (int j = 0; j < KT; ++j) {
        const int k = kbase + j * ENC_T;
        fx[j] = k < Dp ? wx[k] : 0.f;
        fy[j] = k < Dp ? wy[k] : 0.f;
        ar[j] = ai[j] = 0.f;
    }
    for (int base = run.y; base < run.z; base += ENC_TILE_S) {
        const int cnt = min(ENC_TILE_S, run.z - base);
        __syncthreads();
        for (int t = tid; t < cnt; t += ENC_T) {
            const double2 v = sorted[base + t];
            s_p[t] = make_float2((float)v.x, (float)v.y);
        }
        __syncthreads();
#pragma unroll 2
        for (int p = 0; p < cnt; ++p) {
            const float2 P = s_p[p];
#pragma unroll
            for (int j = 0; j < KT; ++j) {
                float sv, cv;
                const float phi = fmaf(fx[j], P.x, fy[j] * P.y);
                if (j >= KT - NPOLY) sincos_fma(phi, &sv, &cv);
                else __sincosf(phi, &sv, &cv);
                ar[j] += cv;
                ai[j] += sv;
            }
        }
    }
#pragma unroll
    for (int j = 0; j < KT; ++j) {
        const int k = kbase + j * ENC_T;
        if (k < Dp) part[(size_t)r * Dp + k] = make_float2(ar[j], ai[j]);
    }
}

// Packed variant (delta > 1 default for D >= 2048): 8 warps, the first four all-MUFU, the
// other four with NPB of their 8 dimensions on the polynomial (PhasorAcc, as
// k_encode_bundle_x2 in encode.cu); one run of one slot per block row.
template <int NPA, int NPB>
__global__ void __launch_bounds__(256, 3) k_encode_runs_x2(const double2 *__restrict__ sorted,
                                                          const int4 *__restrict__ runs,
                                                          const int *__restrict__ meta, const float *__restrict__ wx,
                                                          const float *__restrict__ wy, int Dp,
                                                          float2 *__restrict__ part)
{
    constexpr int T = 256, KT = 8;
    __shared__ float2 s_p[ENC_TILE_S];
    const int r = blockIdx.y;
    if (r >= meta[META_NRUNS()]) return;
    const int4 run = runs[r];
    const int tid = threadIdx.x;
    const int kbase = blockIdx.x * T * KT + tid;
    float fx[KT], fy[KT];
#pragma unroll
    for (int j = 0; j < KT; ++j) {
        const int k = kbase + j * T;
        fx[j] = k < Dp ? wx[k] : 0.f;
        fy[j] = k < Dp ? wy[k] : 0.f;
    }
    auto go = [&](auto acc) {
        acc.init(fx, fy);
        for (int base = run.y; base < run.z; base += ENC_TILE_S) {
            const int cnt = min(ENC_TILE_S, run.z - base);
            block_sync_any();   // reached from both warp roles: non-.aligned
            for (int t = tid; t < cnt; t += T) {
                const double2 v = sorted[base + t];
                s_p[t] = make_float2((float)v.x, (float)v.y);
            }
            block_sync_any();   // reached from both warp roles: non-.aligned
#pragma unroll 2
            for (int p = 0; p < cnt; ++p) {
                const float2 P = s_p[p];
                acc.point(P.x, P.y);
            }
        }
#pragma unroll
        for (int j = 0; j < KT; ++j) {
            const int k = kbase + j * T;
            if (k < Dp) part[(size_t)r * Dp + k] = acc.get(j);
        }
    };
    if ((tid >> 5) >= 4) go(PhasorAcc<KT, NPB>{});
    else go(PhasorAcc<KT, NPA>{});
}

// Pair (half-angle) variant, the default for D >= 2048 (PairAcc,
// common.cuh): a run holds points of one slot in index order; consecutive points form pairs
// whose mean and half-difference are computed from the fp64 centred coordinates and rounded
// once; an odd last point of a run is added on its own.  8 warps, the first four all-MUFU, the
// other four NPB of 8 dimensions on the FMA pipe; 64 registers, 4 blocks per SM.
template <int NPB>
__global__ void __launch_bounds__(256, 4) k_encode_runs_pairs(const double2 *__restrict__ sorted,
                                                              const int4 *__restrict__ runs,
                                                              const int *__restrict__ meta, const float *__restrict__ wx,
                                                              const float *__restrict__ wy, int Dp,
                                                              float2 *__restrict__ part)
{
    constexpr int T = 256, KT = 8;
    __shared__ float4 s_q[ENC_TILE_S / 2];
    __shared__ double2 s_last;
    const int r = blockIdx.y;
    if (r >= meta[META_NRUNS()]) return;
    const int4 run = runs[r];
    const int tid = threadIdx.x;
    const int kbase = blockIdx.x * T * KT + tid;
    float fx[KT], fy[KT];
#pragma unroll
    for (int j = 0; j < KT; ++j) {
        const int k = kbase + j * T;
        fx[j] = k < Dp ? wx[k] : 0.f;
        fy[j] = k < Dp ? wy[k] : 0.f;
    }
    PairW<KT> w;
    w.init(fx, fy);
    auto go = [&](auto acc) {
        acc.init();
        for (int base = run.y; base < run.z; base += ENC_TILE_S) {
            const int cnt = min(ENC_TILE_S, run.z - base);
            const int np = cnt >> 1;
            block_sync_any();   // reached from both warp roles: non-.aligned
            for (int t = tid; t < np; t += T) {
                const double2 a = sorted[base + 2 * t], b = sorted[base + 2 * t + 1];
                s_q[t] = make_float4((float)(0.5 * (a.x + b.x)), (float)(0.5 * (a.y + b.y)),
                                     (float)(0.5 * (a.x - b.x)), (float)(0.5 * (a.y - b.y)));
            }
            if (tid == 0 && (cnt & 1)) s_last = sorted[base + cnt - 1];
            block_sync_any();
#pragma unroll 1
            for (int p = 0; p < np; ++p) acc.pair(w, s_q[p]);
            if (cnt & 1) acc.single(w, (float)s_last.x, (float)s_last.y);
        }
#pragma unroll
        for (int j = 0; j < KT; ++j) {
            const int k = kbase + j * T;
            if (k < Dp) part[(size_t)r * Dp + k] = acc.get(j);
        }
    };
    if ((tid >> 5) >= 4) go(PairAcc<KT, NPB>{});
    else go(PairAcc<KT, 0>{});
}

// pending[s][k] += sum over the slot's runs (fixed order, fp64): 32 k-lanes x 8 run slices
__global__ void __launch_bounds__(256) k_reduce_runs(const float2 *__restrict__ part, const int *__restrict__ meta,
                                                     int nslots, int Dp, int D, double *__restrict__ pending,
                                                     double *__restrict__ pcount)
{
    __shared__ double s_re[8][32], s_im[8][32];
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    const int idx = blockIdx.x * 32 + tx;          // (slot, k)
    const bool live = idx < nslots * Dp;
    const int s = live ? idx / Dp : 0, k = idx - s * Dp;
    double re = 0.0, im = 0.0;
    if (live) {
        const int r0 = meta[META_RSTART() + s], r1 = meta[META_RSTART() + s + 1];
        for (int r = r0 + ty; r < r1; r += 8) {
            const float2 v = part[(size_t)r * Dp + k];
            re += v.x;
            im += v.y;
        }
    }
    s_re[ty][tx] = re;
    s_im[ty][tx] = im;
    __syncthreads();
    if (ty == 0 && live && k < D) {   // padding dimensions stay exactly zero
        double a = 0.0, b = 0.0;
#pragma unroll
        for (int w = 0; w < 8; ++w) { a += s_re[w][tx]; b += s_im[w][tx]; }
        pending[2 * (size_t)idx] += a;
        pending[2 * (size_t)idx + 1] += b;
    }
    if (blockIdx.x == 0 && threadIdx.x < nslots) pcount[threadIdx.x] += (double)meta[META_TOTAL() + threadIdx.x];
}

template <typename T>
int grow_t(T **p, size_t *cap, size_t need)
{
    if (need <= *cap) return VSAOGM_OK;
    if (*p) cudaFree(*p);
    *p = nullptr;
    *cap = 0;
    need += need / 4;   // headroom: batch sizes vary, and a reallocation synchronises the device
    if (cudaMalloc(p, need * sizeof(T)) != cudaSuccess) { *p = nullptr; return VSAOGM_ENOMEM; }
    *cap = need;
    return VSAOGM_OK;
}

}  // namespace

int vsa_launch_encode_sorted(vsaogm_ctx *c, const float *xy, const uint8_t *lab, int64_t n)
{
    const int ns = c->nslots;
    const int nblk = (int)((n + RT_PTS - 1) / RT_PTS);
    const int KT = c->Dp >= 1024 ? 8 : 4;
    const bool pairs = c->enc_x2 == 4 && c->Dp >= 2048;  // pair kernel (default)
    const bool x2 = c->enc_x2 >= 2 && c->Dp >= 2048;     // packed 8-warp role kernels
    const int T = x2 ? 256 : ENC_T, per_sm = pairs ? 4 : x2 ? 3 : 6;
    const int kblocks = (c->Dp + T * KT - 1) / (T * KT);
    // runs per k-block column so that all blocks fit whole waves of `per_sm` per SM; each slot's
    // last run may be short, so size runs for (target - nslots) and the total never exceeds it
    const int64_t target_runs = (int64_t)c->num_sms * per_sm * c->enc_runs_waves / kblocks;
    const int run_pts =
        (int)std::max<int64_t>(64, (n + std::max<int64_t>(1, target_runs - ns) - 1) / std::max<int64_t>(1, target_runs - ns));
    const int64_t max_runs = (n + run_pts - 1) / run_pts + ns;
    int rc;
    size_t cap_meta = c->d_sortmeta ? (size_t)META_INTS() : 0;
    if ((rc = grow_t(&c->d_slot, &c->slot_cap, (size_t)n))) return rc;
    if ((rc = grow_t(&c->d_bhist, &c->bhist_cap, (size_t)nblk * ns))) return rc;
    if ((rc = grow_t(&c->d_sortmeta, &cap_meta, (size_t)META_INTS()))) return rc;
    if ((rc = grow_t(&c->d_sorted, &c->sorted_cap, (size_t)n))) return rc;
    if ((rc = grow_t(&c->d_runs, &c->runs_cap, (size_t)max_runs))) return rc;
    if ((rc = grow_t(&c->d_part, &c->part_cap, (size_t)max_runs * c->Dp))) return rc;

    cudaEvent_t ev;
    vsa_prof_begin(c, VSAOGM_K_ENCODE, &ev);
    k_route_hist<<<nblk, RT_THREADS, 0, c->stream>>>((const float2 *)xy, lab, n, c->d_qc, c->nq, ns, c->d_slot,
                                                      c->d_bhist, c->d_err);
    k_sort_plan<<<1, 1024, 0, c->stream>>>(c->d_bhist, nblk, ns, run_pts, c->d_sortmeta, c->d_runs);
    k_scatter<<<nblk, RT_THREADS, 0, c->stream>>>((const float2 *)xy, c->d_slot, n, ns, c->d_bhist, c->d_sortmeta,
                                                  c->cx, c->cy, c->d_sorted);
    dim3 grid(kblocks, (unsigned)max_runs);
#define VSA_RUNS(KT_, NP_)                                                                                         \
    k_encode_runs<KT_, NP_><<<grid, ENC_T, 0, c->stream>>>(c->d_sorted, c->d_runs, c->d_sortmeta, c->d_wx, c->d_wy, \
                                                          c->Dp, c->d_part)
    if (pairs) {
        switch (c->enc_pairs_npoly) {
        case 0: k_encode_runs_pairs<0><<<grid, 256, 0, c->stream>>>(c->d_sorted, c->d_runs, c->d_sortmeta, c->d_wx,
                                                                    c->d_wy, c->Dp, c->d_part); break;
        case 2: k_encode_runs_pairs<2><<<grid, 256, 0, c->stream>>>(c->d_sorted, c->d_runs, c->d_sortmeta, c->d_wx,
                                                                    c->d_wy, c->Dp, c->d_part); break;
        case 6: k_encode_runs_pairs<6><<<grid, 256, 0, c->stream>>>(c->d_sorted, c->d_runs, c->d_sortmeta, c->d_wx,
                                                                    c->d_wy, c->Dp, c->d_part); break;
        default: k_encode_runs_pairs<4><<<grid, 256, 0, c->stream>>>(c->d_sorted, c->d_runs, c->d_sortmeta, c->d_wx,
                                                                     c->d_wy, c->Dp, c->d_part); break;
        }
    } else if (x2) {
        switch (c->enc_x2_npoly) {
        case 4: k_encode_runs_x2<0, 4><<<grid, 256, 0, c->stream>>>(c->d_sorted, c->d_runs, c->d_sortmeta, c->d_wx,
                                                                    c->d_wy, c->Dp, c->d_part); break;
        default: k_encode_runs_x2<0, 6><<<grid, 256, 0, c->stream>>>(c->d_sorted, c->d_runs, c->d_sortmeta, c->d_wx,
                                                                     c->d_wy, c->Dp, c->d_part); break;
        }
    } else if (KT == 8) {
        if (c->enc_npoly == 2) VSA_RUNS(8, 2);
        else if (c->enc_npoly == 0) VSA_RUNS(8, 0);
        else VSA_RUNS(8, 1);
    } else {
        if (c->enc_npoly == 0) VSA_RUNS(4, 0);
        else VSA_RUNS(4, 1);
    }
#undef VSA_RUNS
    VSA_CUDA_TRY(cudaGetLastError());
    vsa_prof_end(c, VSAOGM_K_ENCODE, ev);
    c->launches += 4;

    vsa_prof_begin(c, VSAOGM_K_REDUCE, &ev);
    k_reduce_runs<<<(ns * c->Dp + 31) / 32, 256, 0, c->stream>>>(c->d_part, c->d_sortmeta, ns, c->Dp, c->D,
                                                                  c->d_pending, c->d_pcounts);
    VSA_CUDA_TRY(cudaGetLastError());
    vsa_prof_end(c, VSAOGM_K_REDUCE, ev);
    c->launches++;
    return VSAOGM_OK;
}
