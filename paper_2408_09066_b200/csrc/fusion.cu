// fusion.cu -- multi-agent fusion (Alg. 3): export / import of the
// memory state with the paper's fusion preconditions (same axis vectors,
// same classes, same delta; plus D, length scale and bounds) checked on import.
//
// Container (little-endian): 8-byte magic "VSAOGM1\0", a "key=value\n" header ended by an
// empty line (doubles as C99 hex floats, exact round trip), int64 counts[S], fp64
// memories [S][D][2] in the raw-coordinate convention of Eq. 9 (the centring rotation of
// the device state undone), S = 2 delta^2 slots.
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <string>

#include "common.cuh"

namespace {

const char kMagic[8] = {'V', 'S', 'A', 'O', 'G', 'M', '1', '\0'};

std::string header(const vsaogm_ctx *c)
{
    char buf[512];
    snprintf(buf, sizeof buf, "D=%d\nseed=%llu\nl=%a\ndelta=%d\nslots=%d\nbounds=%a,%a,%a,%a\n\n", c->D,
             (unsigned long long)c->seed, c->l, c->delta, c->nslots, c->bounds.x_min, c->bounds.y_min,
             c->bounds.x_max, c->bounds.y_max);
    return std::string(buf);
}

__global__ void k_fuse(double *__restrict__ m, double *__restrict__ pending, const double *__restrict__ src, size_t n,
                       int replace)
{
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    if (replace) {
        m[i] = src[i];
        pending[i] = 0.0;
    } else {
        m[i] += src[i];   // Alg. 3: Omega{omega_j} = Omega{omega_j} + omega_j (Eq. 5 bundling)
    }
}

}  // namespace

extern "C" {

int vsaogm_export(vsaogm_ctx *c, void *buf, int64_t *size)
{
    VSA_NVTX();
    if (!c || !size) return VSAOGM_EINVAL_ARG;
    if (int rc = vsa_join_encode(c)) return rc;
    const std::string h = header(c);
    const int S = c->nslots;
    const int64_t need = 8 + (int64_t)h.size() + 8 * (int64_t)S + 16 * (int64_t)S * c->D;
    if (!buf) {
        *size = need;
        return VSAOGM_OK;
    }
    if (*size < need) return VSAOGM_EINVAL_ARG;
    uint8_t *p = (uint8_t *)buf;
    memcpy(p, kMagic, 8);
    memcpy(p + 8, h.data(), h.size());
    int64_t *counts = (int64_t *)malloc(8 * (size_t)S);
    double *mem = (double *)malloc(16 * (size_t)S * c->D);
    if (!counts || !mem) { free(counts); free(mem); return VSAOGM_ENOMEM; }
    int rc = vsaogm_get_memory(c, mem, counts);
    if (rc == VSAOGM_OK) {
        memcpy(p + 8 + h.size(), counts, 8 * (size_t)S);
        memcpy(p + 8 + h.size() + 8 * (size_t)S, mem, 16 * (size_t)S * c->D);
        *size = need;
    }
    free(counts);
    free(mem);
    return rc;
}

static int import_impl(vsaogm_ctx *c, const void *buf, int64_t size, int32_t mode);

int vsaogm_import(vsaogm_ctx *c, const void *buf, int64_t size, int32_t mode)
{
    VSA_NVTX();
    if (!c || !buf || size < 10 || (mode != 0 && mode != 1)) return VSAOGM_EINVAL_ARG;
    if (int rc = vsa_join_encode(c)) return rc;
    const int rc_import = import_impl(c, buf, size, mode);
    if (rc_import == VSAOGM_OK) return vsa_mark_main(c);
    return rc_import;
}

static int import_impl(vsaogm_ctx *c, const void *buf, int64_t size, int32_t mode)
{
    const char *p = (const char *)buf;
    if (memcmp(p, kMagic, 8) != 0) return VSAOGM_EINVAL_ARG;
    const char *end = (const char *)memmem(p + 8, (size_t)size - 8, "\n\n", 2);
    if (!end) return VSAOGM_EINVAL_ARG;
    const std::string h(p + 8, end + 2);
    // parse key=value lines
    long long D = -1, delta = -1, slots = -1;
    unsigned long long seed = 0;
    double l = NAN, b[4] = {NAN, NAN, NAN, NAN};
    size_t pos = 0;
    while (pos < h.size()) {
        size_t nl = h.find('\n', pos);
        if (nl == std::string::npos || nl == pos) break;
        const std::string line = h.substr(pos, nl - pos);
        pos = nl + 1;
        const size_t eq = line.find('=');
        if (eq == std::string::npos) return VSAOGM_EINVAL_ARG;
        const std::string k = line.substr(0, eq), v = line.substr(eq + 1);
        if (k == "D") D = strtoll(v.c_str(), nullptr, 10);
        else if (k == "seed") seed = strtoull(v.c_str(), nullptr, 10);
        else if (k == "l") l = strtod(v.c_str(), nullptr);
        else if (k == "delta") delta = strtoll(v.c_str(), nullptr, 10);
        else if (k == "slots") slots = strtoll(v.c_str(), nullptr, 10);
        else if (k == "bounds") {
            if (sscanf(v.c_str(), "%la,%la,%la,%la", &b[0], &b[1], &b[2], &b[3]) != 4) return VSAOGM_EINVAL_ARG;
        }
    }
    if (D < 1 || delta < 1 || slots < 2) return VSAOGM_EINVAL_ARG;
    const int64_t need = 8 + (int64_t)h.size() + 8 * slots + 16 * slots * D;
    if (size < need) return VSAOGM_EINVAL_ARG;
    // Alg. 3 preconditions + D, l, bounds (the phase convention)
    if (D != c->D || seed != c->seed || delta != c->delta || slots != c->nslots || !(l == c->l) ||
        !(b[0] == c->bounds.x_min && b[1] == c->bounds.y_min && b[2] == c->bounds.x_max && b[3] == c->bounds.y_max))
        return VSAOGM_EPRECOND;
    const int S = c->nslots;
    const int64_t *counts_in = (const int64_t *)(p + 8 + h.size());
    const double *mem_in = (const double *)(p + 8 + h.size() + 8 * (size_t)S);
    // raw -> centred convention of the device state: m_c,k = m_raw,k exp(-i (thx c_x + thy c_y) / l)
    const size_t n = 2 * (size_t)S * c->Dp;
    double *cent = (double *)calloc(n, sizeof(double));
    if (!cent) return VSAOGM_ENOMEM;
    for (int s = 0; s < S; ++s)
        for (int k = 0; k < c->D; ++k) {
            const double psi = (c->thx[k] * c->cx + c->thy[k] * c->cy) / c->l;
            const double cr = cos(psi), si = sin(psi);
            const double re = mem_in[2 * ((size_t)s * c->D + k)], im = mem_in[2 * ((size_t)s * c->D + k) + 1];
            cent[2 * ((size_t)s * c->Dp + k)] = re * cr + im * si;
            cent[2 * ((size_t)s * c->Dp + k) + 1] = im * cr - re * si;
        }
    double *d_src = nullptr;
    int rc = VSAOGM_OK;
    do {
        if (cudaStreamSynchronize(c->stream) != cudaSuccess) { rc = VSAOGM_ECUDA; break; }
        if (cudaMalloc(&d_src, n * sizeof(double)) != cudaSuccess) { d_src = nullptr; rc = VSAOGM_ENOMEM; break; }
        if (cudaMemcpy(d_src, cent, n * sizeof(double), cudaMemcpyHostToDevice) != cudaSuccess) { rc = VSAOGM_ECUDA; break; }
        k_fuse<<<(unsigned)((n + 255) / 256), 256, 0, c->stream>>>(c->d_m, c->d_pending, d_src, n, mode == 0);
        c->launches++;
        std::vector<long long> cnt(S);
        if (cudaMemcpy(cnt.data(), c->d_counts, S * sizeof(long long), cudaMemcpyDeviceToHost) != cudaSuccess) {
            rc = VSAOGM_ECUDA;
            break;
        }
        for (int s = 0; s < S; ++s) cnt[s] = (mode == 0 ? 0 : cnt[s]) + counts_in[s];
        if (cudaMemcpy(c->d_counts, cnt.data(), S * sizeof(long long), cudaMemcpyHostToDevice) != cudaSuccess) {
            rc = VSAOGM_ECUDA;
            break;
        }
        if (mode == 0 && cudaMemset(c->d_pcounts, 0, S * sizeof(double)) != cudaSuccess) { rc = VSAOGM_ECUDA; break; }
        if (cudaStreamSynchronize(c->stream) != cudaSuccess) { rc = VSAOGM_ECUDA; break; }
        if (mode == 0) c->dirty = false;
    } while (0);
    if (d_src) cudaFree(d_src);
    free(cent);
    return rc;
}

}  // extern "C"
