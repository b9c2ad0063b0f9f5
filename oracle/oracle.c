/*
 * oracle.c -- plain, slow, fp64 CPU oracle for the VSA-OGM hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * It shares no code, header, table or constant generator with the CUDA
 * product path (paper_2408_09066_b200/csrc); neither includes the other.
 *
 * Citations: "P:n" = /root/reference/PAPER.md line n (arXiv 2408.09066
 * LaTeX source), "S:n" = SPEC.md line n.  Readings of ambiguous passages are
 * the ledger items L1..L17 of SURVEY.md section 8(c), restated in DESIGN.md.
 *
 * What it computes -- the plain definitions, no factorisation, no blocking:
 *   theta      : phases of the two axis vectors, uniform on (-pi, pi]
 *                (Eq. 3, sec. III-B-3; L2).
 *   encode     : m_{c,k} = sum_{i : psi_i = c} exp(i (thx_k x_i + thy_k y_i) / l)
 *                (Eq. 9 with Eq. 8 length scale P:232-235;
 *                 bundling = addition P:216-219 Eq. 5; Alg. 1 P:260-285 with
 *                 delta = 1 so the memory slot is the label psi; L1, L6).
 *   decode     : n_c = ||m_c||_2 (Eq. 10); per cell centre (x, y)
 *                H_c = sum_k Re(conj(m_{c,k}) exp(i (thx_k x + thy_k y)/l)),
 *                q_c = H_c / (sqrt(D) n_c), 0 if n_c = 0 (Eq. 11; L5, L7, L8),
 *                p_c = q_c^2 (Born rule; L9).
 *   entropy    : hb(p) = -p log2 p - (1-p) log2 (1-p), 0 log 0 = 0;
 *                S_c(r,c) = mean of hb(p_c) over the window footprint clipped
 *                to the full grid; S = S_1 - S_0 (Alg. 2, P:330-356, P:318;
 *                L10, L11, L12, L13).
 *   labels     : occupied (1) if S >= rho_occ, empty (0) if S < rho_emp,
 *                unknown (2) otherwise (Eq. 12; L14).
 *   quadrants  : delta > 1 (sec. III-B-4, Alg. 1): 2 delta^2
 *                memories; a point goes to slot 2 beta + psi, beta = the
 *                nearest quadrant centre (ties to the lowest index); a cell
 *                queries its own quadrant's two memories.
 *
 * Parallelism: pthreads split points (encode; per-thread partial sums added in
 * thread order) or cells (decode).  Results are deterministic for a fixed
 * thread count.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_PI 3.14159265358979323846

/* ------------------------------------------------------------------ theta */
/* splitmix64 (Steele, Lea, Flood 2014; Vigna's public-domain splitmix64.c).
 * Draw order (L2): thx_0 .. thx_{D-1}, then thy_0 .. thy_{D-1} from one
 * stream seeded with `seed`; u = (z >> 11) * 2^-53 in [0,1);
 * theta = pi (1 - 2u) in (-pi, pi].                                        */
static uint64_t orc_splitmix64(uint64_t *state)
{
    uint64_t z = (*state += 0x9E3779B97F4A7C15ULL);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

uint64_t oracle_splitmix64_stream(uint64_t seed, int64_t n, uint64_t *out)
{
    uint64_t s = seed;
    for (int64_t i = 0; i < n; ++i) out[i] = orc_splitmix64(&s);
    return s;
}

int oracle_theta(uint64_t seed, int32_t D, double *theta_x, double *theta_y)
{
    if (D < 1) return -1;
    uint64_t s = seed;
    for (int32_t k = 0; k < D; ++k) {
        double u = (double)(orc_splitmix64(&s) >> 11) * 0x1.0p-53;
        theta_x[k] = ORC_PI * (1.0 - 2.0 * u);
    }
    for (int32_t k = 0; k < D; ++k) {
        double u = (double)(orc_splitmix64(&s) >> 11) * 0x1.0p-53;
        theta_y[k] = ORC_PI * (1.0 - 2.0 * u);
    }
    return 0;
}

/* ------------------------------------------------------------------ encode */
typedef struct {
    int32_t D;
    const double *tx, *ty;
    double l;
    const float *xy;
    const uint8_t *lab;
    int64_t i0, i1;
    double *m;          /* [2][D][2] partial for this thread */
    int64_t cnt[2];
    int64_t bad;
} enc_job;

static void *enc_worker(void *arg)
{
    enc_job *j = (enc_job *)arg;
    memset(j->m, 0, sizeof(double) * 4 * (size_t)j->D);
    j->cnt[0] = j->cnt[1] = 0;
    j->bad = 0;
    for (int64_t i = j->i0; i < j->i1; ++i) {
        double x = (double)j->xy[2 * i], y = (double)j->xy[2 * i + 1];
        int c = j->lab[i];
        if (c > 1 || !isfinite(x) || !isfinite(y)) { j->bad++; continue; }
        j->cnt[c]++;
        double *mc = j->m + (size_t)c * 2 * j->D;
        for (int32_t k = 0; k < j->D; ++k) {
            /* Eq. 9: phase of the bound x- and y- fractional powers, Eq. 8 scaling by l */
            double a = (j->tx[k] * x + j->ty[k] * y) / j->l;
            mc[2 * k] += cos(a);
            mc[2 * k + 1] += sin(a);
        }
    }
    return NULL;
}

/* m: [2][D][2] (class, k, re/im), ADDED to (bundling is addition, Eq. 5).
 * counts[2] added to.  Returns the number of skipped invalid points. */
int64_t oracle_encode(int32_t D, const double *tx, const double *ty, double l,
                      int64_t n, const float *xy, const uint8_t *labels,
                      double *m, int64_t *counts, int32_t nthreads)
{
    if (nthreads < 1) nthreads = 1;
    if (n < (int64_t)nthreads) nthreads = n > 0 ? (int32_t)n : 1;
    enc_job *jobs = (enc_job *)calloc((size_t)nthreads, sizeof(enc_job));
    pthread_t *th = (pthread_t *)calloc((size_t)nthreads, sizeof(pthread_t));
    double *parts = (double *)malloc(sizeof(double) * 4 * (size_t)D * (size_t)nthreads);
    for (int t = 0; t < nthreads; ++t) {
        jobs[t].D = D; jobs[t].tx = tx; jobs[t].ty = ty; jobs[t].l = l;
        jobs[t].xy = xy; jobs[t].lab = labels;
        jobs[t].i0 = n * t / nthreads; jobs[t].i1 = n * (t + 1) / nthreads;
        jobs[t].m = parts + (size_t)t * 4 * D;
        pthread_create(&th[t], NULL, enc_worker, &jobs[t]);
    }
    int64_t bad = 0;
    for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
    for (int t = 0; t < nthreads; ++t) {            /* fixed thread order */
        for (int64_t e = 0; e < 4 * (int64_t)D; ++e) m[e] += jobs[t].m[e];
        counts[0] += jobs[t].cnt[0];
        counts[1] += jobs[t].cnt[1];
        bad += jobs[t].bad;
    }
    free(parts); free(th); free(jobs);
    return bad;
}

/* ------------------------------------------------------------------ norms */
/* Eq. 10: n_c = ||m_c||_2 over the D complex components. */
void oracle_norms(int32_t D, const double *m, double *norms)
{
    for (int c = 0; c < 2; ++c) {
        double s = 0.0;
        for (int32_t k = 0; k < D; ++k) {
            double re = m[(size_t)c * 2 * D + 2 * k], im = m[(size_t)c * 2 * D + 2 * k + 1];
            s += re * re + im * im;
        }
        norms[c] = sqrt(s);
    }
}

/* ------------------------------------------------------------------ decode */
typedef struct {
    int32_t D;
    const double *tx, *ty;
    double l;
    const double *m;
    double norms[2];
    double x0, y0, res;
    const int32_t *rows, *cols;
    int64_t c0, c1, ncell;
    double *q;     /* [2][ncell] */
    int64_t range_violations;
} dec_job;

static void *dec_worker(void *arg)
{
    dec_job *j = (dec_job *)arg;
    j->range_violations = 0;
    for (int64_t e = j->c0; e < j->c1; ++e) {
        /* L7: query points are cell centres, row index grows along +y */
        double x = j->x0 + ((double)j->cols[e] + 0.5) * j->res;
        double y = j->y0 + ((double)j->rows[e] + 0.5) * j->res;
        for (int c = 0; c < 2; ++c) {
            double q = 0.0;
            if (j->norms[c] > 0.0) {                        /* L8: empty class decodes to 0 */
                const double *mc = j->m + (size_t)c * 2 * j->D;
                double H = 0.0;
                for (int32_t k = 0; k < j->D; ++k) {
                    double a = (j->tx[k] * x + j->ty[k] * y) / j->l;
                    /* Re(conj(m) * e^{ia}) = Re m cos a + Im m sin a   (Eq. 11) */
                    H += mc[2 * k] * cos(a) + mc[2 * k + 1] * sin(a);
                }
                q = H / (sqrt((double)j->D) * j->norms[c]);
                if (fabs(q) > 1.0 + 1e-12) j->range_violations++;   /* Cauchy-Schwarz */
            }
            j->q[(size_t)c * j->ncell + e] = q;
        }
    }
    return NULL;
}

/* Signed similarity q for a list of cells (rows[e], cols[e]) of the grid with
 * lower-left corner (x0, y0) and cell size res.  q: [2][ncell].
 * Returns the number of |q| > 1 + 1e-12 violations (must be 0). */
int64_t oracle_decode_cells(int32_t D, const double *tx, const double *ty, double l,
                            const double *m, double x0, double y0, double res,
                            int64_t ncell, const int32_t *rows, const int32_t *cols,
                            double *q, int32_t nthreads)
{
    double norms[2];
    oracle_norms(D, m, norms);
    if (nthreads < 1) nthreads = 1;
    if (ncell < (int64_t)nthreads) nthreads = ncell > 0 ? (int32_t)ncell : 1;
    dec_job *jobs = (dec_job *)calloc((size_t)nthreads, sizeof(dec_job));
    pthread_t *th = (pthread_t *)calloc((size_t)nthreads, sizeof(pthread_t));
    for (int t = 0; t < nthreads; ++t) {
        dec_job *j = &jobs[t];
        j->D = D; j->tx = tx; j->ty = ty; j->l = l; j->m = m;
        j->norms[0] = norms[0]; j->norms[1] = norms[1];
        j->x0 = x0; j->y0 = y0; j->res = res; j->rows = rows; j->cols = cols;
        j->c0 = ncell * t / nthreads; j->c1 = ncell * (t + 1) / nthreads;
        j->ncell = ncell; j->q = q;
        pthread_create(&th[t], NULL, dec_worker, j);
    }
    int64_t viol = 0;
    for (int t = 0; t < nthreads; ++t) { pthread_join(th[t], NULL); viol += jobs[t].range_violations; }
    free(th); free(jobs);
    return viol;
}

/* ------------------------------------------------------------------ quadrants (delta > 1) */
/* Space discretisation (sec. III-B-4): delta x delta equal chunks of
 * the bounds, 2 delta^2 memories.  getQuadrantCenters() of Alg. 1:
 * mu_{i,j} = (x_min + (i + 1/2) W / delta, y_min + (j + 1/2) H / delta),
 * index beta = j delta + i (row-major, x fastest). */
void oracle_quadrant_centers(double x_min, double y_min, double x_max, double y_max, int32_t delta,
                             double *cx, double *cy)
{
    for (int32_t j = 0; j < delta; ++j)
        for (int32_t i = 0; i < delta; ++i) {
            cx[j * delta + i] = x_min + ((double)i + 0.5) * (x_max - x_min) / (double)delta;
            cy[j * delta + i] = y_min + ((double)j + 0.5) * (y_max - y_min) / (double)delta;
        }
}

/* Alg. 1: beta = argmin_k d_L2(point, mu_k) over all delta^2 centres,
 * ties to the lowest index (coordinate-space distance). */
static int32_t nearest_quadrant(double x, double y, const double *cx, const double *cy, int32_t nq)
{
    int32_t best = 0;
    double bd = 0.0;
    for (int32_t k = 0; k < nq; ++k) {
        double dx = x - cx[k], dy = y - cy[k];
        double d = dx * dx + dy * dy;
        if (k == 0 || d < bd) { bd = d; best = k; }
    }
    return best;
}

void oracle_assign_quadrants(double x_min, double y_min, double x_max, double y_max, int32_t delta, int64_t n,
                             const double *x, const double *y, int32_t *beta)
{
    int32_t nq = delta * delta;
    double *cx = (double *)malloc(sizeof(double) * nq), *cy = (double *)malloc(sizeof(double) * nq);
    oracle_quadrant_centers(x_min, y_min, x_max, y_max, delta, cx, cy);
    for (int64_t i = 0; i < n; ++i) beta[i] = nearest_quadrant(x[i], y[i], cx, cy, nq);
    free(cx);
    free(cy);
}

typedef struct {
    int32_t D;
    const double *tx, *ty;
    double l;
    const float *xy;
    const uint8_t *lab;
    const double *cx, *cy;
    int32_t nq;
    int64_t i0, i1;
    double *m;          /* [2 nq][D][2] partial */
    int64_t *cnt;       /* [2 nq] */
    int64_t bad;
} encq_job;

static void *encq_worker(void *arg)
{
    encq_job *j = (encq_job *)arg;
    memset(j->m, 0, sizeof(double) * 4 * (size_t)j->nq * (size_t)j->D);
    memset(j->cnt, 0, sizeof(int64_t) * 2 * (size_t)j->nq);
    j->bad = 0;
    for (int64_t i = j->i0; i < j->i1; ++i) {
        double x = (double)j->xy[2 * i], y = (double)j->xy[2 * i + 1];
        int c = j->lab[i];
        if (c > 1 || !isfinite(x) || !isfinite(y)) { j->bad++; continue; }
        int32_t beta = nearest_quadrant(x, y, j->cx, j->cy, j->nq);
        int32_t slot = 2 * beta + c;                     /* Alg. 1: omega_{2 beta + psi} (0-based, L6) */
        j->cnt[slot]++;
        double *ms = j->m + (size_t)slot * 2 * j->D;
        for (int32_t k = 0; k < j->D; ++k) {
            double a = (j->tx[k] * x + j->ty[k] * y) / j->l;   /* Eq. 9 */
            ms[2 * k] += cos(a);
            ms[2 * k + 1] += sin(a);
        }
    }
    return NULL;
}

/* Alg. 1 with delta >= 1: m [2 delta^2][D][2] and counts [2 delta^2] ADDED to. */
int64_t oracle_encode_quadrants(int32_t D, const double *tx, const double *ty, double l, double x_min,
                                double y_min, double x_max, double y_max, int32_t delta, int64_t n,
                                const float *xy, const uint8_t *labels, double *m, int64_t *counts,
                                int32_t nthreads)
{
    int32_t nq = delta * delta;
    double *cx = (double *)malloc(sizeof(double) * nq), *cy = (double *)malloc(sizeof(double) * nq);
    oracle_quadrant_centers(x_min, y_min, x_max, y_max, delta, cx, cy);
    if (nthreads < 1) nthreads = 1;
    if (n < (int64_t)nthreads) nthreads = n > 0 ? (int32_t)n : 1;
    encq_job *jobs = (encq_job *)calloc((size_t)nthreads, sizeof(encq_job));
    pthread_t *th = (pthread_t *)calloc((size_t)nthreads, sizeof(pthread_t));
    size_t msz = 4 * (size_t)nq * (size_t)D;
    double *parts = (double *)malloc(sizeof(double) * msz * (size_t)nthreads);
    int64_t *cparts = (int64_t *)malloc(sizeof(int64_t) * 2 * (size_t)nq * (size_t)nthreads);
    for (int t = 0; t < nthreads; ++t) {
        encq_job *j = &jobs[t];
        j->D = D; j->tx = tx; j->ty = ty; j->l = l; j->xy = xy; j->lab = labels;
        j->cx = cx; j->cy = cy; j->nq = nq;
        j->i0 = n * t / nthreads; j->i1 = n * (t + 1) / nthreads;
        j->m = parts + (size_t)t * msz;
        j->cnt = cparts + (size_t)t * 2 * nq;
        pthread_create(&th[t], NULL, encq_worker, j);
    }
    int64_t bad = 0;
    for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
    for (int t = 0; t < nthreads; ++t) {          /* fixed thread order */
        for (size_t e = 0; e < msz; ++e) m[e] += jobs[t].m[e];
        for (int32_t s = 0; s < 2 * nq; ++s) counts[s] += jobs[t].cnt[s];
        bad += jobs[t].bad;
    }
    free(parts); free(cparts); free(th); free(jobs); free(cx); free(cy);
    return bad;
}

typedef struct {
    int32_t D;
    const double *tx, *ty;
    double l;
    const double *m;
    const double *norms;     /* [2 nq] */
    const double *cx, *cy;
    int32_t nq;
    double x0, y0, res;
    const int32_t *rows, *cols;
    int64_t c0, c1, ncell;
    double *q;
    int32_t *beta_out;
    int64_t viol;
} decq_job;

static void *decq_worker(void *arg)
{
    decq_job *j = (decq_job *)arg;
    j->viol = 0;
    for (int64_t e = j->c0; e < j->c1; ++e) {
        double x = j->x0 + ((double)j->cols[e] + 0.5) * j->res;
        double y = j->y0 + ((double)j->rows[e] + 0.5) * j->res;
        int32_t beta = nearest_quadrant(x, y, j->cx, j->cy, j->nq);   /* the cell's own quadrant */
        if (j->beta_out) j->beta_out[e] = beta;
        for (int c = 0; c < 2; ++c) {
            int32_t slot = 2 * beta + c;
            double q = 0.0;
            if (j->norms[slot] > 0.0) {
                const double *ms = j->m + (size_t)slot * 2 * j->D;
                double H = 0.0;
                for (int32_t k = 0; k < j->D; ++k) {
                    double a = (j->tx[k] * x + j->ty[k] * y) / j->l;
                    H += ms[2 * k] * cos(a) + ms[2 * k + 1] * sin(a);     /* Eq. 11 */
                }
                q = H / (sqrt((double)j->D) * j->norms[slot]);
                if (fabs(q) > 1.0 + 1e-12) j->viol++;
            }
            j->q[(size_t)c * j->ncell + e] = q;
        }
    }
    return NULL;
}

/* Eq. 11 with delta >= 1: each cell queries the memories 2 beta + {0,1} of the
 * quadrant beta nearest to its centre.  q [2][ncell]; beta_out [ncell] or NULL. */
int64_t oracle_decode_cells_quadrants(int32_t D, const double *tx, const double *ty, double l, const double *m,
                                      double x_min, double y_min, double x_max, double y_max, int32_t delta,
                                      double x0, double y0, double res, int64_t ncell, const int32_t *rows,
                                      const int32_t *cols, double *q, int32_t *beta_out, int32_t nthreads)
{
    int32_t nq = delta * delta;
    double *cx = (double *)malloc(sizeof(double) * nq), *cy = (double *)malloc(sizeof(double) * nq);
    oracle_quadrant_centers(x_min, y_min, x_max, y_max, delta, cx, cy);
    double *norms = (double *)malloc(sizeof(double) * 2 * nq);
    for (int32_t s = 0; s < 2 * nq; ++s) {                 /* Eq. 10 per memory */
        double acc = 0.0;
        for (int32_t k = 0; k < D; ++k) {
            double re = m[(size_t)s * 2 * D + 2 * k], im = m[(size_t)s * 2 * D + 2 * k + 1];
            acc += re * re + im * im;
        }
        norms[s] = sqrt(acc);
    }
    if (nthreads < 1) nthreads = 1;
    if (ncell < (int64_t)nthreads) nthreads = ncell > 0 ? (int32_t)ncell : 1;
    decq_job *jobs = (decq_job *)calloc((size_t)nthreads, sizeof(decq_job));
    pthread_t *th = (pthread_t *)calloc((size_t)nthreads, sizeof(pthread_t));
    for (int t = 0; t < nthreads; ++t) {
        decq_job *j = &jobs[t];
        j->D = D; j->tx = tx; j->ty = ty; j->l = l; j->m = m; j->norms = norms;
        j->cx = cx; j->cy = cy; j->nq = nq; j->x0 = x0; j->y0 = y0; j->res = res;
        j->rows = rows; j->cols = cols; j->c0 = ncell * t / nthreads; j->c1 = ncell * (t + 1) / nthreads;
        j->ncell = ncell; j->q = q; j->beta_out = beta_out;
        pthread_create(&th[t], NULL, decq_worker, j);
    }
    int64_t viol = 0;
    for (int t = 0; t < nthreads; ++t) { pthread_join(th[t], NULL); viol += jobs[t].viol; }
    free(th); free(jobs); free(norms); free(cx); free(cy);
    return viol;
}

/* ------------------------------------------------------------------ entropy */
/* Binary Shannon entropy in bits with 0 log 0 = 0. */
double oracle_hb(double p)
{
    double h = 0.0;
    if (p > 0.0) h -= p * log2(p);
    if (p < 1.0) h -= (1.0 - p) * log2(1.0 - p);
    return h;
}

/* Footprint membership (L11): box |du|,|dv| <= h, or disk du^2 + dv^2 <= h^2. */
static int in_footprint(int du, int dv, int h, int disk)
{
    if (disk) return du * du + dv * dv <= h * h;
    return abs(du) <= h && abs(dv) <= h;
}

/* ---- histogram ("rank") entropy estimator (SPEC.md:375 open question) ----
 * The paper passes "a disk filter across the heat map image" and applies Shannon
 * entropy (Alg. 2) without writing the estimator; the
 * image-processing reading is the entropy of the grey-level histogram inside the
 * footprint: the probability image is quantised to 8 bits, code = floor(255 p + 1/2)
 * clipped to [0, 255], and S = -sum_b (n_b/N) log2 (n_b/N) over the N footprint
 * cells inside the grid.  Codes are taken in fp32 (the kernel's precision) from the
 * given fp32-representable p: both sides then take the same integer decisions. */
static int code8(double p)
{
    float f = (float)p * 255.0f + 0.5f;
    int c = (int)floorf(f);
    return c < 0 ? 0 : (c > 255 ? 255 : c);
}

/* S [3][n] and labels for target cells from p_region [2][rb-ra][cb-ca] (probabilities,
 * i.e. already q^2), as oracle_entropy_cells does for the mean estimator. */
int64_t oracle_entropy_hist_cells(int32_t R, int32_t C, int32_t ra, int32_t rb, int32_t ca, int32_t cb,
                                  const double *p_region, int32_t h_occ, int32_t h_emp, int32_t disk,
                                  double rho_occ, double rho_emp, int64_t n, const int32_t *rows,
                                  const int32_t *cols, double *S, uint8_t *labels)
{
    int32_t W = cb - ca, Hh = rb - ra;
    for (int64_t e = 0; e < n; ++e) {
        int32_t r = rows[e], c = cols[e];
        double Sc[2];
        for (int cls = 0; cls < 2; ++cls) {
            int h = cls == 1 ? h_occ : h_emp;
            int64_t hist[256];
            memset(hist, 0, sizeof hist);
            int64_t N = 0;
            for (int du = -h; du <= h; ++du)
                for (int dv = -h; dv <= h; ++dv) {
                    if (!in_footprint(du, dv, h, disk)) continue;
                    int rr = r + du, cc = c + dv;
                    if (rr < 0 || rr >= R || cc < 0 || cc >= C) continue;   /* L13 */
                    if (rr < ra || rr >= rb || cc < ca || cc >= cb) return -1;
                    hist[code8(p_region[(size_t)cls * Hh * W + (size_t)(rr - ra) * W + (cc - ca)])]++;
                    N++;
                }
            double s = 0.0;
            for (int b = 0; b < 256; ++b)
                if (hist[b] > 0) {
                    double f = (double)hist[b] / (double)N;
                    s -= f * log2(f);
                }
            Sc[cls] = s;
        }
        double g = Sc[1] - Sc[0];
        S[e] = Sc[1];
        S[n + e] = Sc[0];
        S[2 * n + e] = g;
        labels[e] = g >= rho_occ ? 1 : (g < rho_emp ? 0 : 2);
    }
    return 0;
}

/* Entropy maps and labels for a list of target cells.
 * q_region: [2][rb-ra][cb-ca] signed similarities of the full-grid region
 * rows [ra, rb) x cols [ca, cb) of an R x C grid.  For each target cell
 * (rows[e], cols[e]) every footprint offset that lands inside the full grid
 * must land inside the region (else returns -1).
 * Class 1 (occupied) uses half-width h_occ, class 0 (empty) h_emp (Alg. 2 r(psi)).
 * S: [3][n] = (S_occ, S_emp, S_occ - S_emp); labels[n] in {0 empty, 1 occupied, 2 unknown}.
 * Returns the number of |q| > 1 + 1e-12 violations seen, or -1 on a region error. */
int64_t oracle_entropy_cells(int32_t R, int32_t C, int32_t ra, int32_t rb, int32_t ca, int32_t cb,
                             const double *q_region, int32_t h_occ, int32_t h_emp, int32_t disk,
                             double rho_occ, double rho_emp, int64_t n,
                             const int32_t *rows, const int32_t *cols,
                             double *S, uint8_t *labels)
{
    int32_t W = cb - ca, Hh = rb - ra;
    int64_t viol = 0;
    for (int64_t e = 0; e < n; ++e) {
        int32_t r = rows[e], c = cols[e];
        double Sc[2];
        for (int cls = 0; cls < 2; ++cls) {
            int h = cls == 1 ? h_occ : h_emp;
            double sum = 0.0;
            int64_t cnt = 0;
            for (int du = -h; du <= h; ++du)
                for (int dv = -h; dv <= h; ++dv) {
                    if (!in_footprint(du, dv, h, disk)) continue;
                    int rr = r + du, cc = c + dv;
                    if (rr < 0 || rr >= R || cc < 0 || cc >= C) continue;   /* L13: clip to full grid */
                    if (rr < ra || rr >= rb || cc < ca || cc >= cb) return -1;
                    double q = q_region[(size_t)cls * Hh * W + (size_t)(rr - ra) * W + (cc - ca)];
                    if (fabs(q) > 1.0 + 1e-12) viol++;
                    sum += oracle_hb(q * q);      /* Born rule p = q^2 */
                    cnt++;
                }
            Sc[cls] = sum / (double)cnt;
        }
        double s = Sc[1] - Sc[0];          /* S(psi=1) - S(psi=0), Alg. 2 */
        S[e] = Sc[1];
        S[n + e] = Sc[0];
        S[2 * n + e] = s;
        labels[e] = s >= rho_occ ? 1 : (s < rho_emp ? 0 : 2);   /* Eq. 12 + L14 */
    }
    return viol;
}
