// api.cu -- the C ABI of include/vsaogm.h: context, theta, state machine,
// argument checks, launch sequencing, profiling and test hooks.
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <new>

#include "common.cuh"

namespace {

// splitmix64 (Steele, Lea & Flood 2014): theta draw order x axis then y axis,
// u = (z >> 11) 2^-53 in [0,1), theta = pi (1 - 2u) in (-pi, pi]   (L2)
uint64_t splitmix64(uint64_t &s)
{
    uint64_t z = (s += 0x9E3779B97F4A7C15ULL);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

constexpr double kPi = 3.14159265358979323846;

template <typename T>
int dev_alloc_zero(T **p, size_t n)
{
    if (cudaMalloc(p, n * sizeof(T)) != cudaSuccess) { *p = nullptr; return VSAOGM_ENOMEM; }
    if (cudaMemset(*p, 0, n * sizeof(T)) != cudaSuccess) return VSAOGM_ECUDA;
    return VSAOGM_OK;
}

int grow_bytes(void **p, size_t *cap, size_t need)
{
    if (need <= *cap) return VSAOGM_OK;
    if (*p) cudaFree(*p);
    *p = nullptr;
    *cap = 0;
    if (cudaMalloc(p, need) != cudaSuccess) { *p = nullptr; return VSAOGM_ENOMEM; }
    *cap = need;
    return VSAOGM_OK;
}

bool finite_all(double a, double b, double c, double d) { return isfinite(a) && isfinite(b) && isfinite(c) && isfinite(d); }

}  // namespace

void vsa_report_cuda_error(cudaError_t e, const char *expr, const char *file, int line)
{
    static const bool on = getenv("VSAOGM_DEBUG") != nullptr;
    if (on) fprintf(stderr, "vsaogm: %s failed: %s (%s:%d)\n", expr, cudaGetErrorString(e), file, line);
}

// ------------------------------------------------------------------ profiling

int vsa_prof_begin(vsaogm_ctx *c, int kid, cudaEvent_t *a)
{
    (void)kid;
    *a = nullptr;
    if (!c->prof) return 0;
    if (c->ev_pool.empty()) {
        cudaEvent_t e;
        if (cudaEventCreate(&e) != cudaSuccess) return 0;
        c->ev_pool.push_back(e);
    }
    *a = c->ev_pool.back();
    c->ev_pool.pop_back();
    cudaEventRecord(*a, c->stream);
    return 0;
}

void vsa_prof_end(vsaogm_ctx *c, int kid, cudaEvent_t a)
{
    if (!c->prof || !a) return;
    cudaEvent_t b;
    if (c->ev_pool.empty()) {
        if (cudaEventCreate(&b) != cudaSuccess) return;
    } else {
        b = c->ev_pool.back();
        c->ev_pool.pop_back();
    }
    cudaEventRecord(b, c->stream);
    c->prof_live.push_back({kid, a, b});
}

static void prof_harvest(vsaogm_ctx *c)
{
    for (auto &r : c->prof_live) {
        float ms = 0.f;
        cudaEventSynchronize(r.b);
        if (cudaEventElapsedTime(&ms, r.a, r.b) == cudaSuccess) {
            c->prof_ms[r.kid] += ms;
            c->prof_n[r.kid] += 1;
        }
        c->ev_pool.push_back(r.a);
        c->ev_pool.push_back(r.b);
    }
    c->prof_live.clear();
}

// ------------------------------------------------------------------ ABI

extern "C" {

const char *vsaogm_strerror(int code)
{
    switch (code) {
    case VSAOGM_OK: return "ok";
    case VSAOGM_EINVAL_DIM: return "invalid dimension (D < 1)";
    case VSAOGM_EINVAL_ARG: return "invalid argument";
    case VSAOGM_EEMPTY: return "empty point set (n < 1)";
    case VSAOGM_ELABEL: return "a point label is not in {0, 1}";
    case VSAOGM_ENONFINITE: return "a point coordinate is not finite";
    case VSAOGM_ENOMEM: return "out of memory";
    case VSAOGM_ECUDA: return "CUDA error";
    case VSAOGM_ESTATE: return "call not valid in the current state";
    case VSAOGM_EPRECOND: return "fusion precondition violated (axis vectors, classes, delta, D, length scale or bounds differ)";
    default: return "unknown error";
    }
}

int vsaogm_create(int32_t D, uint64_t seed, double length_scale, vsaogm_bounds b, vsaogm_ctx **out)
{
    return vsaogm_create_quadrants(D, seed, length_scale, b, 1, out);
}

int vsaogm_create_quadrants(int32_t D, uint64_t seed, double length_scale, vsaogm_bounds b, int32_t delta,
                            vsaogm_ctx **out)
{
    VSA_NVTX();
    if (!out) return VSAOGM_EINVAL_ARG;
    *out = nullptr;
    if (D < 1) return VSAOGM_EINVAL_DIM;
    if (!(length_scale > 0.0) || !isfinite(length_scale)) return VSAOGM_EINVAL_ARG;
    if (!finite_all(b.x_min, b.y_min, b.x_max, b.y_max) || !(b.x_max > b.x_min) || !(b.y_max > b.y_min))
        return VSAOGM_EINVAL_ARG;
    if (delta < 1 || delta > VSAOGM_MAX_DELTA) return VSAOGM_EINVAL_ARG;
    vsaogm_ctx *c = new (std::nothrow) vsaogm_ctx();
    if (!c) return VSAOGM_ENOMEM;
    int rc = VSAOGM_OK;
    do {
        if (cudaGetDevice(&c->device) != cudaSuccess) { rc = VSAOGM_ECUDA; break; }
        cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, c->device);
        c->seed = seed;
        c->delta = delta;
        c->nq = delta * delta;
        c->nslots = 2 * c->nq;
        // getQuadrantCenters() of Alg. 1, expression order fixed by DESIGN.md (fp64)
        c->qcx.resize(c->nq);
        c->qcy.resize(c->nq);
        for (int j = 0; j < delta; ++j)
            for (int i = 0; i < delta; ++i) {
                c->qcx[j * delta + i] = b.x_min + ((double)i + 0.5) * (b.x_max - b.x_min) / (double)delta;
                c->qcy[j * delta + i] = b.y_min + ((double)j + 0.5) * (b.y_max - b.y_min) / (double)delta;
            }
        c->D = D;
        c->Dp = (D + 31) / 32 * 32;
        c->Kp = 2 * c->Dp;
        c->l = length_scale;
        c->bounds = b;
        c->cx = 0.5 * (b.x_min + b.x_max);
        c->cy = 0.5 * (b.y_min + b.y_max);
        c->thx.resize(D);
        c->thy.resize(D);
        uint64_t s = seed;
        for (int k = 0; k < D; ++k) c->thx[k] = kPi * (1.0 - 2.0 * ((double)(splitmix64(s) >> 11) * 0x1.0p-53));
        for (int k = 0; k < D; ++k) c->thy[k] = kPi * (1.0 - 2.0 * ((double)(splitmix64(s) >> 11) * 0x1.0p-53));
        std::vector<float> wx(c->Dp, 0.f), wy(c->Dp, 0.f);
        std::vector<double> tx(c->Dp, 0.0), ty(c->Dp, 0.0);
        for (int k = 0; k < D; ++k) {
            wx[k] = (float)(c->thx[k] / length_scale);             // rad per metre (encode)
            wy[k] = (float)(c->thy[k] / length_scale);
            tx[k] = c->thx[k] / (2.0 * kPi * length_scale);       // turns per metre (tables)
            ty[k] = c->thy[k] / (2.0 * kPi * length_scale);
        }
        if ((rc = dev_alloc_zero(&c->d_wx, c->Dp))) break;
        if ((rc = dev_alloc_zero(&c->d_wy, c->Dp))) break;
        if ((rc = dev_alloc_zero(&c->d_tx_turns, c->Dp))) break;
        if ((rc = dev_alloc_zero(&c->d_ty_turns, c->Dp))) break;
        if ((rc = dev_alloc_zero(&c->d_m, 2 * (size_t)c->nslots * c->Dp))) break;
        if ((rc = dev_alloc_zero(&c->d_pending, 2 * (size_t)c->nslots * c->Dp + c->nslots))) break;
        c->d_pcounts = c->d_pending + 2 * (size_t)c->nslots * c->Dp;
        if ((rc = dev_alloc_zero(&c->d_counts, c->nslots))) break;
        if ((rc = dev_alloc_zero(&c->d_norm2, 2 * (size_t)c->nslots))) break;
        if ((rc = dev_alloc_zero(&c->d_mhat, (size_t)c->nslots * c->Dp))) break;
        if ((rc = dev_alloc_zero(&c->d_normpart, (size_t)c->nslots * 17))) break;
        if ((rc = dev_alloc_zero(&c->d_qc, 2 * (size_t)c->nq))) break;
        {
            std::vector<double> qc(2 * c->nq);
            for (int k = 0; k < c->nq; ++k) { qc[2 * k] = c->qcx[k]; qc[2 * k + 1] = c->qcy[k]; }
            if (cudaMemcpy(c->d_qc, qc.data(), qc.size() * sizeof(double), cudaMemcpyHostToDevice) != cudaSuccess) {
                rc = VSAOGM_ECUDA;
                break;
            }
        }
        if ((rc = dev_alloc_zero(&c->d_err, 1))) break;
        if ((rc = dev_alloc_zero(&c->d_ent_ctr, 2))) break;
        if (cudaMemcpy(c->d_wx, wx.data(), c->Dp * sizeof(float), cudaMemcpyHostToDevice) != cudaSuccess ||
            cudaMemcpy(c->d_wy, wy.data(), c->Dp * sizeof(float), cudaMemcpyHostToDevice) != cudaSuccess ||
            cudaMemcpy(c->d_tx_turns, tx.data(), c->Dp * sizeof(double), cudaMemcpyHostToDevice) != cudaSuccess ||
            cudaMemcpy(c->d_ty_turns, ty.data(), c->Dp * sizeof(double), cudaMemcpyHostToDevice) != cudaSuccess) {
            rc = VSAOGM_ECUDA;
            break;
        }
    } while (0);
    if (rc) {
        vsaogm_destroy(c);
        return rc;
    }
    *out = c;
    return VSAOGM_OK;
}

void vsaogm_destroy(vsaogm_ctx *c)
{
    VSA_NVTX();
    if (!c) return;
    cudaStreamSynchronize(c->stream);
    if (c->enc_stream) cudaStreamSynchronize(c->enc_stream);
    if (c->ev_enc) cudaEventDestroy(c->ev_enc);
    if (c->ev_main) cudaEventDestroy(c->ev_main);
    void *ptrs[] = {c->d_wx, c->d_wy, c->d_tx_turns, c->d_ty_turns, c->d_m, c->d_pending, c->d_counts,
                    c->d_norm2, c->d_mhat, c->d_normpart, c->d_err, c->d_ent_ctr, c->d_part, c->d_part_cnt, c->d_stage_xy, c->d_stage_lab, c->d_A,
                    c->d_B, c->d_hb, c->d_ws, c->d_S, c->d_lab, c->d_qc, c->d_slot, c->d_bhist,
                    c->d_sortmeta, c->d_sorted, c->d_runs, c->d_code, c->d_nu_grid, c->d_nu_f1, c->d_nu_G,
                    c->d_nu_psi, c->d_nu_tw, c->d_nu_ph, c->d_nu_kpar, c->d_nu_out, c->d_nu_bins,
                    c->d_nu_key, c->d_nu_sorted};
    for (void *p : ptrs)
        if (p) cudaFree(p);
    vsa_nudecode_free(c);
    for (auto &r : c->prof_live) { cudaEventDestroy(r.a); cudaEventDestroy(r.b); }
    for (auto e : c->ev_pool) cudaEventDestroy(e);
    if (c->up) {
        cudaStreamSynchronize(c->up);
        cudaStreamSynchronize(c->down);
        for (int s = 0; s < VSA_IO_SLOTS; ++s) {
            void *q[] = {c->d_in_xy[s], c->d_in_lab[s], c->d_out_S[s], c->d_out_lab[s]};
            for (void *p : q)
                if (p) cudaFree(p);
            cudaEvent_t e[] = {c->ev_up[s], c->ev_used[s], c->ev_out[s], c->ev_down[s]};
            for (cudaEvent_t x : e)
                if (x) cudaEventDestroy(x);
        }
        cudaStreamDestroy(c->up);
        cudaStreamDestroy(c->down);
        if (c->h_err) cudaFreeHost(c->h_err);
    }
    delete c;
}

int vsaogm_set_stream(vsaogm_ctx *c, void *stream)
{
    if (!c) return VSAOGM_EINVAL_ARG;
    c->stream = (cudaStream_t)stream;
    return VSAOGM_OK;
}

int vsa_join_encode(vsaogm_ctx *c)
{
    if (c->enc_stream && c->enc_inflight) {
        VSA_CUDA_TRY(cudaStreamWaitEvent(c->stream, c->ev_enc, 0));
        c->enc_inflight = false;
    }
    return VSAOGM_OK;
}

int vsa_mark_main(vsaogm_ctx *c)
{
    if (c->enc_stream) {
        VSA_CUDA_TRY(cudaEventRecord(c->ev_main, c->stream));
        c->main_mark = true;
    }
    return VSAOGM_OK;
}

int vsaogm_set_encode_stream(vsaogm_ctx *c, void *stream)
{
    VSA_NVTX();
    if (!c) return VSAOGM_EINVAL_ARG;
    int rc;
    if ((rc = vsa_join_encode(c))) return rc;
    if (c->enc_stream && (cudaStream_t)stream != c->enc_stream) {
        // encodes already queued on the old stream must precede anything queued after this call
        VSA_CUDA_TRY(cudaStreamSynchronize(c->enc_stream));
    }
    // the pipelined host I/O orders slot reuse differently with and without an encode stream
    // (api.cu: vsaogm_*_host_async); drain its copy streams so that no slot's previous user is
    // left unordered across the switch
    if (c->up && (cudaStream_t)stream != c->enc_stream) {
        VSA_CUDA_TRY(cudaStreamSynchronize(c->stream));
        VSA_CUDA_TRY(cudaStreamSynchronize(c->up));
        VSA_CUDA_TRY(cudaStreamSynchronize(c->down));
    }
    if (stream && !c->ev_enc) {
        VSA_CUDA_TRY(cudaEventCreateWithFlags(&c->ev_enc, cudaEventDisableTiming));
        VSA_CUDA_TRY(cudaEventCreateWithFlags(&c->ev_main, cudaEventDisableTiming));
    }
    c->enc_stream = (cudaStream_t)stream;
    c->enc_inflight = false;
    c->main_mark = false;
    if (c->enc_stream) {   // the new encode stream starts after everything queued so far
        VSA_CUDA_TRY(cudaEventRecord(c->ev_main, c->stream));
        c->main_mark = true;
    }
    return VSAOGM_OK;
}

int vsaogm_encode_bundle(vsaogm_ctx *c, const float *xy, const uint8_t *lab, int64_t n)
{
    VSA_NVTX();
    if (!c) return VSAOGM_EINVAL_ARG;
    if (n < 1) return VSAOGM_EEMPTY;
    if (!xy || !lab) return VSAOGM_EINVAL_ARG;
    int rc;
    if (!c->enc_stream) {
        if ((rc = vsa_launch_encode(c, xy, lab, n))) return rc;
    } else {
        if (c->main_mark) {
            VSA_CUDA_TRY(cudaStreamWaitEvent(c->enc_stream, c->ev_main, 0));
            c->main_mark = false;
        }
        cudaStream_t main = c->stream;
        c->stream = c->enc_stream;
        rc = vsa_launch_encode(c, xy, lab, n);
        c->stream = main;
        if (rc) return rc;
        VSA_CUDA_TRY(cudaEventRecord(c->ev_enc, c->enc_stream));
        c->enc_inflight = true;
    }
    c->dirty = true;
    return VSAOGM_OK;
}

int vsaogm_encode_bundle_host(vsaogm_ctx *c, const float *xy, const uint8_t *lab, int64_t n)
{
    VSA_NVTX();
    if (!c) return VSAOGM_EINVAL_ARG;
    if (n < 1) return VSAOGM_EEMPTY;
    if (!xy || !lab) return VSAOGM_EINVAL_ARG;
    if ((size_t)n > c->stage_cap) {
        if (c->d_stage_xy) cudaFree(c->d_stage_xy);
        if (c->d_stage_lab) cudaFree(c->d_stage_lab);
        c->d_stage_xy = nullptr;
        c->d_stage_lab = nullptr;
        c->stage_cap = 0;
        if (cudaMalloc(&c->d_stage_xy, n * sizeof(float2)) != cudaSuccess ||
            cudaMalloc(&c->d_stage_lab, n) != cudaSuccess)
            return VSAOGM_ENOMEM;
        c->stage_cap = n;
    }
    // the copies go on the stream the encode runs on: with an encode stream, after its wait for
    // the context stream's last mark (a previous reader of the staging buffers may be an encode
    // queued on the context stream before the encode stream was set); consecutive host encodes
    // then reuse the buffers in stream order
    cudaStream_t es = c->stream;
    if (c->enc_stream) {
        es = c->enc_stream;
        if (c->main_mark) {
            VSA_CUDA_TRY(cudaStreamWaitEvent(c->enc_stream, c->ev_main, 0));
            c->main_mark = false;
        }
    }
    VSA_CUDA_TRY(cudaMemcpyAsync(c->d_stage_xy, xy, n * sizeof(float2), cudaMemcpyHostToDevice, es));
    VSA_CUDA_TRY(cudaMemcpyAsync(c->d_stage_lab, lab, n, cudaMemcpyHostToDevice, es));
    return vsaogm_encode_bundle(c, (const float *)c->d_stage_xy, c->d_stage_lab, n);
}

namespace {
// lazily create the copy streams and slot events of the pipelined host path
int ensure_pipeline(vsaogm_ctx *c)
{
    if (c->up) return VSAOGM_OK;
    VSA_CUDA_TRY(cudaStreamCreateWithFlags(&c->up, cudaStreamNonBlocking));
    VSA_CUDA_TRY(cudaStreamCreateWithFlags(&c->down, cudaStreamNonBlocking));
    VSA_CUDA_TRY(cudaHostAlloc((void **)&c->h_err, VSA_IO_SLOTS * sizeof(int), cudaHostAllocDefault));
    for (int s = 0; s < VSA_IO_SLOTS; ++s) c->h_err[s] = 0;
    for (int s = 0; s < VSA_IO_SLOTS; ++s) {
        VSA_CUDA_TRY(cudaEventCreateWithFlags(&c->ev_up[s], cudaEventDisableTiming));
        VSA_CUDA_TRY(cudaEventCreateWithFlags(&c->ev_used[s], cudaEventDisableTiming));
        VSA_CUDA_TRY(cudaEventCreateWithFlags(&c->ev_out[s], cudaEventDisableTiming));
        VSA_CUDA_TRY(cudaEventCreateWithFlags(&c->ev_down[s], cudaEventDisableTiming));
    }
    return VSAOGM_OK;
}

// grow a slot buffer (with 25 % headroom: batch sizes vary a little from step to step, and a
// reallocation synchronises the device); the previous user of the slot must be done first
int grow_slot(void **p, size_t *cap, size_t need, cudaEvent_t busy, bool recorded)
{
    if (need <= *cap) return VSAOGM_OK;
    if (recorded) VSA_CUDA_TRY(cudaEventSynchronize(busy));
    return grow_bytes(p, cap, need + need / 4);
}
}  // namespace

int vsaogm_encode_bundle_host_async(vsaogm_ctx *c, const float *xy, const uint8_t *lab, int64_t n)
{
    VSA_NVTX();
    if (!c) return VSAOGM_EINVAL_ARG;
    if (n < 1) return VSAOGM_EEMPTY;
    if (!xy || !lab) return VSAOGM_EINVAL_ARG;
    int rc;
    if ((rc = ensure_pipeline(c))) return rc;
    const int s = (int)(c->in_seq % VSA_IO_SLOTS);
    const bool used = c->in_seq >= VSA_IO_SLOTS;   // slot s was consumed by an earlier encode
    if ((rc = grow_slot((void **)&c->d_in_xy[s], &c->in_xy_cap[s], n * sizeof(float2), c->ev_used[s], used))) return rc;
    if ((rc = grow_slot((void **)&c->d_in_lab[s], &c->in_lab_cap[s], (size_t)n, c->ev_used[s], used))) return rc;
    cudaStream_t es = c->enc_stream ? c->enc_stream : c->stream;
    // upload on the upload stream, after the slot's previous encode; the encode (on the encode
    // stream when one is set) waits for it.  Not on the encode stream itself: between two encodes
    // that stream is on the step's critical path (encode -> norms -> strengths -> next encode), and
    // the 36 us copy of a C4 batch would sit in it
    if (used) VSA_CUDA_TRY(cudaStreamWaitEvent(c->up, c->ev_used[s], 0));
    VSA_CUDA_TRY(cudaMemcpyAsync(c->d_in_xy[s], xy, n * sizeof(float2), cudaMemcpyHostToDevice, c->up));
    VSA_CUDA_TRY(cudaMemcpyAsync(c->d_in_lab[s], lab, n, cudaMemcpyHostToDevice, c->up));
    VSA_CUDA_TRY(cudaEventRecord(c->ev_up[s], c->up));
    VSA_CUDA_TRY(cudaStreamWaitEvent(es, c->ev_up[s], 0));
    if ((rc = vsaogm_encode_bundle(c, (const float *)c->d_in_xy[s], c->d_in_lab[s], n))) return rc;
    VSA_CUDA_TRY(cudaEventRecord(c->ev_used[s], es));
    c->in_seq++;
    return VSAOGM_OK;
}

int vsaogm_pending(vsaogm_ctx *c, double **p, int64_t *n)
{
    VSA_NVTX();
    if (!c || !p) return VSAOGM_EINVAL_ARG;
    if (int rc = vsa_join_encode(c)) return rc;
    *p = c->d_pending;
    if (n) *n = 2 * (int64_t)c->nslots * c->Dp + c->nslots;
    c->pending_taken = true;
    return VSAOGM_OK;
}

int vsaogm_commit(vsaogm_ctx *c)
{
    VSA_NVTX();
    if (!c) return VSAOGM_EINVAL_ARG;
    int rc;
    if ((rc = vsa_join_encode(c))) return rc;
    if ((rc = vsa_launch_commit(c))) return rc;
    c->dirty = false;
    return vsa_mark_main(c);
}

int vsaogm_reset(vsaogm_ctx *c)
{
    VSA_NVTX();
    if (!c) return VSAOGM_EINVAL_ARG;
    if (int rc = vsa_join_encode(c)) return rc;
    VSA_CUDA_TRY(cudaMemsetAsync(c->d_m, 0, 2 * (size_t)c->nslots * c->Dp * sizeof(double), c->stream));
    VSA_CUDA_TRY(cudaMemsetAsync(c->d_pending, 0, (2 * (size_t)c->nslots * c->Dp + c->nslots) * sizeof(double), c->stream));
    VSA_CUDA_TRY(cudaMemsetAsync(c->d_counts, 0, c->nslots * sizeof(long long), c->stream));
    c->dirty = false;
    c->decoded = false;
    return vsa_mark_main(c);
}

int vsaogm_decode(vsaogm_ctx *c, const vsaogm_grid *g, vsaogm_precision prec, float *q)
{
    VSA_NVTX();
    if (!c || !g) return VSAOGM_EINVAL_ARG;
    if (!(g->res > 0.0) || !isfinite(g->res) || !isfinite(g->x0) || !isfinite(g->y0) || g->rows < 1 ||
        g->cols < 1 || g->row_begin < 0 || g->row_end > g->rows || g->row_begin >= g->row_end || g->halo < 0 ||
        (prec != VSAOGM_F16 && prec != VSAOGM_BF16))
        return VSAOGM_EINVAL_ARG;
    int rc;
    const int do_commit = c->dirty ? 1 : 0;   // single-rank: implicit commit, fused into the norms kernel
    if (c->dirty && c->pending_taken) return VSAOGM_ESTATE;
    const int32_t r_lo = std::max(0, g->row_begin - g->halo);
    const int32_t r_hi = std::min(g->rows, g->row_end + g->halo);
    const int32_t r_ext = r_hi - r_lo;
    const int64_t M = 2 * (int64_t)r_ext;
    if (M * c->delta > (int64_t)1 << 30 || (int64_t)g->cols > (int64_t)1 << 30) return VSAOGM_EINVAL_ARG;
    // Decode groups: one per quadrant with decoded cells.  A cell's quadrant is the nearest
    // centre (fp64, ties to the lower index) along each axis: cell rows of quadrant row j and
    // cell columns of quadrant column i are contiguous ranges (delta = 1: one group).
    Groups G{};
    int slot0[VSA_MAX_GROUPS];
    {
        const int dl = c->delta;
        auto nearest = [&](double v, bool is_y) {
            int best = 0;
            double bd = 0.0;
            for (int k = 0; k < dl; ++k) {
                const double cc = is_y ? c->qcy[k * dl] : c->qcx[k];
                const double d = (v - cc) * (v - cc);
                if (k == 0 || d < bd) { bd = d; best = k; }
            }
            return best;
        };
        std::vector<int> rlo(dl, INT32_MAX), rhi(dl, -1), clo(dl, INT32_MAX), chi(dl, -1);
        for (int r = r_lo; r < r_hi; ++r) {
            const int j = dl == 1 ? 0 : nearest(g->y0 + ((double)r + 0.5) * g->res, true);
            rlo[j] = std::min(rlo[j], r);
            rhi[j] = std::max(rhi[j], r);
        }
        for (int col = 0; col < g->cols; ++col) {
            const int i = dl == 1 ? 0 : nearest(g->x0 + ((double)col + 0.5) * g->res, false);
            clo[i] = std::min(clo[i], col);
            chi[i] = std::max(chi[i], col);
        }
        int a_rows = 0;
        for (int j = 0; j < dl; ++j) {
            if (rhi[j] < 0) continue;
            for (int i = 0; i < dl; ++i) {
                if (chi[i] < 0) continue;
                const int k = G.n++;
                G.nrows[k] = rhi[j] - rlo[j] + 1;
                G.mrows[k] = 2 * G.nrows[k];
                G.row0[k] = rlo[j] - r_lo;
                G.col0[k] = clo[i];
                G.ncols[k] = chi[i] - clo[i] + 1;
                G.a_row0[k] = a_rows;
                slot0[k] = 2 * (j * dl + i);
                a_rows += G.mrows[k];
            }
        }
    }
    int a_rows = 0;
    for (int k = 0; k < G.n; ++k) a_rows = std::max(a_rows, G.a_row0[k] + G.mrows[k]);
    const size_t ldh = ((size_t)g->cols + 7) / 8 * 8;   // H_b row stride (16-byte multiple)
    if (c->estimator == 1) {
        if ((rc = grow_bytes((void **)&c->d_code, &c->code_cap, (size_t)M * ldh))) return rc;
    } else if ((rc = grow_bytes((void **)&c->d_hb, &c->hb_cap, (size_t)M * ldh * sizeof(float)))) {
        return rc;
    }
    if ((rc = vsa_join_encode(c))) return rc;
    if ((rc = vsa_launch_norms(c, do_commit))) return rc;
    c->dirty = false;
    if (c->delta == 1 && vsa_nudecode_applies(c, g->x0, g->y0, g->res, g->cols, r_lo, r_ext)) {
        // the type-1 NUFFT decode (nudecode.cu): no phasor tables; fp32 throughout (prec unused)
        if ((rc = vsa_launch_decode_nufft(c, g->x0, g->y0, g->res, g->cols, r_lo, r_ext, c->d_hb, c->d_code, ldh,
                                          q, r_lo - g->row_begin, g->row_end - g->row_begin, true)))
            return rc;
    } else {
    const bool early = c->pipe_early != 0;   // tuning variant
    if (early && (rc = vsa_mark_main(c))) return rc;
    if ((rc = vsa_launch_table_B(c, g->x0, g->res, g->cols, prec))) return rc;
    // table A, unless the GEMM generates its A tiles on the fly (gemm_agen)
    if (!c->gemm_agen && (rc = vsa_launch_table_A(c, G, g->y0, g->res, r_lo, prec, slot0))) return rc;
    // the next encode (encode stream) may start now: pending is committed and the scaled
    // memories are consumed (by table A, or read by the GEMM: the next norms kernel, which
    // rewrites them, is queued after this GEMM on this stream); it then shares the SMs with
    // this decode's GEMM
    if (!early && (rc = vsa_mark_main(c))) return rc;
    if ((rc = vsa_launch_decode_gemm(c, G, a_rows, g->cols, prec, 1.0f / (float)c->D, c->d_hb, q, r_ext,
                                     r_lo - g->row_begin, g->row_end - g->row_begin, slot0, g->y0, g->res, r_lo)))
        return rc;
    }
    c->decoded = true;
    c->g_estimator = c->estimator;
    c->g_rows = g->rows;
    c->g_cols = g->cols;
    c->g_r0 = g->row_begin;
    c->g_r1 = g->row_end;
    c->g_rlo = r_lo;
    c->g_rext = r_ext;
    c->g_halo = g->halo;
    return VSAOGM_OK;
}

int vsaogm_set_estimator(vsaogm_ctx *c, int32_t estimator)
{
    if (!c || (estimator != 0 && estimator != 1)) return VSAOGM_EINVAL_ARG;
    c->estimator = estimator;
    return VSAOGM_OK;
}

static int tuning_knob(vsaogm_ctx *c, const char *key, int64_t value, int64_t *get);

int vsaogm_set_tuning(vsaogm_ctx *c, const char *key, int64_t value) { return tuning_knob(c, key, value, nullptr); }

int vsaogm_get_tuning(vsaogm_ctx *c, const char *key, int64_t *value)
{
    if (!value) return VSAOGM_EINVAL_ARG;
    return tuning_knob(c, key, 0, value);
}

static int tuning_knob(vsaogm_ctx *c, const char *key, int64_t value, int64_t *get)
{
    if (!c || !key) return VSAOGM_EINVAL_ARG;
    struct Knob {
        const char *name;
        int *field;
        int lo, hi;
    } knobs[] = {
        {"enc_x2", &c->enc_x2, 0, 4},
        {"enc_x2_npoly", &c->enc_x2_npoly, 0, 8},
        {"enc_pairs_npoly", &c->enc_pairs_npoly, 0, 8},
        {"enc_pairs_minb", &c->enc_pairs_minb, 3, 4},
        {"enc_pairs_split", &c->enc_pairs_split, 0, 1},
        {"enc_method", &c->enc_method, -1, 1},
        {"enc_x2_minb", &c->enc_x2_minb, 3, 4},
        {"enc_x2_waves", &c->enc_x2_waves, 1, 64},
        {"enc_npoly", &c->enc_npoly, 0, 4},
        {"enc_minb", &c->enc_minb, 6, 8},
        {"enc_kt", &c->enc_kt, 8, 16},
        {"enc_path", &c->enc_path, -1, 2},
        {"enc_waves", &c->enc_waves, 1, 64},
        {"enc_runs_waves", &c->enc_runs_waves, 1, 64},
        {"gemm_variant", &c->gemm_variant, -1, 2},
        {"gemm_bn", &c->gemm_bn, 0, 256},
        {"gemm_splits", &c->gemm_splits, 0, 64},
        {"gemm_l2_hints", &c->gemm_l2_hints, 0, 2},
        {"gemm_agen", &c->gemm_agen, 0, 1},
        {"pipe_early", &c->pipe_early, 0, 1},
        {"entropy_kernel", &c->entropy_kernel, 0, 2},
        {"entropy_rw", &c->entropy_rw, 0, 1 << 20},
        {"table_rows", &c->table_rows, 1, 256},
        {"dec_method", &c->dec_method, -1, 1},
        {"pdl", &c->pdl, 0, 1},
        {"nd_bps", &c->nd_bps, 0, 8},
    };
    for (const Knob &k : knobs)
        if (strcmp(k.name, key) == 0) {
            if (get) {
                *get = *k.field;
                return VSAOGM_OK;
            }
            if (value < k.lo || value > k.hi) return VSAOGM_EINVAL_ARG;
            *k.field = (int)value;
            return VSAOGM_OK;
        }
    return VSAOGM_EINVAL_ARG;
}

static int check_entropy(vsaogm_ctx *c, const vsaogm_entropy_params *p)
{
    if (!c || !p) return VSAOGM_EINVAL_ARG;
    if (!c->decoded || c->g_estimator != c->estimator) return VSAOGM_ESTATE;   // decode again after a switch
    if (p->half_occ < 1 || p->half_emp < 1 || p->half_occ > 16 || p->half_emp > 16 || (p->disk != 0 && p->disk != 1) ||
        !isfinite(p->rho_occ) || !isfinite(p->rho_emp) || p->rho_emp > p->rho_occ)
        return VSAOGM_EINVAL_ARG;
    const int H = std::max(p->half_occ, p->half_emp);
    // every window row inside the full grid must have been decoded
    if (std::max(0, c->g_r0 - H) < c->g_rlo || std::min(c->g_rows, c->g_r1 + H) > c->g_rlo + c->g_rext)
        return VSAOGM_EINVAL_ARG;
    return VSAOGM_OK;
}

int vsaogm_entropy(vsaogm_ctx *c, const vsaogm_entropy_params *p, float *S, uint8_t *lab)
{
    VSA_NVTX();
    int rc = check_entropy(c, p);
    if (rc) return rc;
    return vsa_launch_entropy(c, p, S, lab);
}

int vsaogm_entropy_host(vsaogm_ctx *c, const vsaogm_entropy_params *p, float *S_host, uint8_t *lab_host)
{
    VSA_NVTX();
    int rc = check_entropy(c, p);
    if (rc) return rc;
    const size_t cells = (size_t)(c->g_r1 - c->g_r0) * c->g_cols;
    if (S_host && (rc = grow_bytes((void **)&c->d_S, &c->S_cap, 3 * cells * sizeof(float)))) return rc;
    if (lab_host && (rc = grow_bytes((void **)&c->d_lab, &c->lab_cap, cells))) return rc;
    if ((rc = vsa_launch_entropy(c, p, S_host ? c->d_S : nullptr, lab_host ? c->d_lab : nullptr))) return rc;
    if (S_host) VSA_CUDA_TRY(cudaMemcpyAsync(S_host, c->d_S, 3 * cells * sizeof(float), cudaMemcpyDeviceToHost, c->stream));
    if (lab_host) VSA_CUDA_TRY(cudaMemcpyAsync(lab_host, c->d_lab, cells, cudaMemcpyDeviceToHost, c->stream));
    VSA_CUDA_TRY(cudaStreamSynchronize(c->stream));
    return VSAOGM_OK;
}

int vsaogm_entropy_host_async(vsaogm_ctx *c, const vsaogm_entropy_params *p, float *S_host, uint8_t *lab_host,
                              int64_t *ticket)
{
    VSA_NVTX();
    int rc = check_entropy(c, p);
    if (rc) return rc;
    if (!ticket) return VSAOGM_EINVAL_ARG;
    if ((rc = ensure_pipeline(c))) return rc;
    const size_t cells = (size_t)(c->g_r1 - c->g_r0) * c->g_cols;
    const int s = (int)(c->out_seq % VSA_IO_SLOTS);
    const bool used = c->out_seq >= VSA_IO_SLOTS;   // slot s was downloaded by an earlier call
    if (S_host && (rc = grow_slot((void **)&c->d_out_S[s], &c->out_S_cap[s], 3 * cells * sizeof(float), c->ev_down[s], used)))
        return rc;
    if (lab_host && (rc = grow_slot((void **)&c->d_out_lab[s], &c->out_lab_cap[s], cells, c->ev_down[s], used)))
        return rc;
    // the download runs on the download stream so that it overlaps the next step's kernels (at C4
    // the 4 MB of labels take ~75 us over PCIe, half a step: on the context stream they would
    // delay the next decode by that much)
    cudaStream_t ds = c->down;
    if (used) VSA_CUDA_TRY(cudaStreamWaitEvent(c->stream, c->ev_down[s], 0));
    if ((rc = vsa_launch_entropy(c, p, S_host ? c->d_out_S[s] : nullptr, lab_host ? c->d_out_lab[s] : nullptr))) return rc;
    VSA_CUDA_TRY(cudaEventRecord(c->ev_out[s], c->stream));
    VSA_CUDA_TRY(cudaStreamWaitEvent(c->down, c->ev_out[s], 0));
    if (S_host) VSA_CUDA_TRY(cudaMemcpyAsync(S_host, c->d_out_S[s], 3 * cells * sizeof(float), cudaMemcpyDeviceToHost, ds));
    if (lab_host) VSA_CUDA_TRY(cudaMemcpyAsync(lab_host, c->d_out_lab[s], cells, cudaMemcpyDeviceToHost, ds));
    // deferred error bits as of this step (sticky until vsaogm_sync clears them)
    VSA_CUDA_TRY(cudaMemcpyAsync(c->h_err + s, c->d_err, sizeof(int), cudaMemcpyDeviceToHost, ds));
    VSA_CUDA_TRY(cudaEventRecord(c->ev_down[s], ds));
    *ticket = c->out_seq++;
    return VSAOGM_OK;
}

int vsaogm_wait(vsaogm_ctx *c, int64_t ticket)
{
    VSA_NVTX();
    if (!c || ticket < 0 || ticket >= c->out_seq) return VSAOGM_EINVAL_ARG;
    // the slot's event was recorded for this ticket or a later one (later downloads
    // complete after earlier ones: one download stream)
    VSA_CUDA_TRY(cudaEventSynchronize(c->ev_down[ticket % VSA_IO_SLOTS]));
    const int err = c->h_err[ticket % VSA_IO_SLOTS];
    if (err) return (err & VSA_ERRBIT_LABEL) ? VSAOGM_ELABEL : VSAOGM_ENONFINITE;
    return VSAOGM_OK;
}

int vsaogm_sync(vsaogm_ctx *c)
{
    VSA_NVTX();
    if (!c) return VSAOGM_EINVAL_ARG;
    if (int rc = vsa_join_encode(c)) return rc;
    int err = 0;
    VSA_CUDA_TRY(cudaMemcpyAsync(&err, c->d_err, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    VSA_CUDA_TRY(cudaStreamSynchronize(c->stream));
    if (err) {
        VSA_CUDA_TRY(cudaMemsetAsync(c->d_err, 0, sizeof(int), c->stream));
        VSA_CUDA_TRY(cudaStreamSynchronize(c->stream));
        return (err & VSA_ERRBIT_LABEL) ? VSAOGM_ELABEL : VSAOGM_ENONFINITE;
    }
    return VSAOGM_OK;
}

int vsaogm_get_memory(vsaogm_ctx *c, double *host, int64_t *counts)
{
    VSA_NVTX();
    if (!c) return VSAOGM_EINVAL_ARG;
    if (int rc = vsa_join_encode(c)) return rc;
    const int ns = c->nslots;
    const size_t n = 2 * (size_t)ns * c->Dp;
    std::vector<double> m(n), pd(n);
    std::vector<long long> cnt(ns);
    std::vector<double> pcnt(ns);
    VSA_CUDA_TRY(cudaStreamSynchronize(c->stream));
    VSA_CUDA_TRY(cudaMemcpy(m.data(), c->d_m, n * sizeof(double), cudaMemcpyDeviceToHost));
    VSA_CUDA_TRY(cudaMemcpy(pd.data(), c->d_pending, n * sizeof(double), cudaMemcpyDeviceToHost));
    VSA_CUDA_TRY(cudaMemcpy(cnt.data(), c->d_counts, ns * sizeof(long long), cudaMemcpyDeviceToHost));
    VSA_CUDA_TRY(cudaMemcpy(pcnt.data(), c->d_pcounts, ns * sizeof(double), cudaMemcpyDeviceToHost));
    if (host) {
        // undo the centring rotation: m_raw,k = m_centred,k * exp(+i (thx_k c_x + thy_k c_y) / l)
        for (int s = 0; s < ns; ++s)
            for (int k = 0; k < c->D; ++k) {
                const double psi = (c->thx[k] * c->cx + c->thy[k] * c->cy) / c->l;
                const double cr = cos(psi), si = sin(psi);
                const size_t o = 2 * ((size_t)s * c->Dp + k);
                const double re = m[o] + pd[o], im = m[o + 1] + pd[o + 1];
                host[2 * ((size_t)s * c->D + k)] = re * cr - im * si;
                host[2 * ((size_t)s * c->D + k) + 1] = re * si + im * cr;
            }
    }
    if (counts)
        for (int s = 0; s < ns; ++s) counts[s] = cnt[s] + (long long)pcnt[s];
    return VSAOGM_OK;
}

int vsaogm_get_phases(vsaogm_ctx *c, double *host)
{
    if (!c || !host) return VSAOGM_EINVAL_ARG;
    memcpy(host, c->thx.data(), c->D * sizeof(double));
    memcpy(host + c->D, c->thy.data(), c->D * sizeof(double));
    return VSAOGM_OK;
}

int vsaogm_profile_enable(vsaogm_ctx *c, int enable)
{
    if (!c) return VSAOGM_EINVAL_ARG;
    c->prof = enable != 0;
    return VSAOGM_OK;
}

int vsaogm_profile_read(vsaogm_ctx *c, double *ms, int64_t *launches)
{
    if (!c) return VSAOGM_EINVAL_ARG;
    if (int rc = vsa_join_encode(c)) return rc;
    VSA_CUDA_TRY(cudaStreamSynchronize(c->stream));
    prof_harvest(c);
    for (int i = 0; i < VSAOGM_NKERNELS; ++i) {
        if (ms) ms[i] = c->prof_ms[i];
        if (launches) launches[i] = c->prof_n[i];
        c->prof_ms[i] = 0;
        c->prof_n[i] = 0;
    }
    return VSAOGM_OK;
}

int64_t vsaogm_launch_count(const vsaogm_ctx *c) { return c ? c->launches : 0; }

int vsaogm_test_gemm(const void *A, const void *B, int32_t M, int32_t N, int32_t K, vsaogm_precision prec,
                     int32_t kernel, int32_t bn, int32_t splits, float *C, void *stream)
{
    if (!A || !B || !C || M < 1 || N < 1 || K < 64 || K % 64 != 0 || kernel < -1 || kernel > 2)
        return VSAOGM_EINVAL_ARG;
    if (bn != 0 && (bn < 128 || bn > 256 || bn % 32 != 0)) return VSAOGM_EINVAL_ARG;
    if (splits < 0) return VSAOGM_EINVAL_ARG;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    int rc = vsa_gemm_raw(A, B, M, N, K, prec, C, (cudaStream_t)stream, sms, kernel, bn, splits);
    if (rc) return rc;
    VSA_CUDA_TRY(cudaStreamSynchronize((cudaStream_t)stream));
    return VSAOGM_OK;
}

}  // extern "C"
