// common.cuh -- context layout, error plumbing and sm_100a PTX helpers shared
// by the library's translation units.  Product code only (the oracle never
// includes anything from here).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <vector>

#include "vsaogm.h"

// NVTX range per C-ABI call (header-only NVTX v3: a no-op unless a profiler is attached), so
// nsys / ncu timelines show vsaogm_encode_bundle, vsaogm_decode, ... around their kernels.
#include <nvtx3/nvToolsExt.h>
struct VsaNvtxRange {
    explicit VsaNvtxRange(const char *name) { nvtxRangePushA(name); }
    ~VsaNvtxRange() { nvtxRangePop(); }
};
#define VSA_NVTX() VsaNvtxRange vsa_nvtx_range_(__func__)

// VSAOGM_DEBUG=1 in the environment prints the failing CUDA call to stderr.
void vsa_report_cuda_error(cudaError_t e, const char *expr, const char *file, int line);
#define VSA_CUDA_TRY(expr)                                                       \
    do {                                                                         \
        cudaError_t _e = (expr);                                                 \
        if (_e != cudaSuccess) {                                                 \
            vsa_report_cuda_error(_e, #expr, __FILE__, __LINE__);                \
            return VSAOGM_ECUDA;                                                 \
        }                                                                        \
    } while (0)

// Device error-flag bits set by the encode kernel (deferred errors).
#define VSA_ERRBIT_LABEL 1
#define VSA_ERRBIT_NONFINITE 2

// Decode GEMM tiling (tcgen05, cta_group::1): 128 x 256 output tile, K chunk
// of 64 16-bit elements (one 128-byte swizzle row), 4-stage TMA ring.
#define VSA_BM 128
#define VSA_BN 256
#define VSA_BK 64
#define VSA_STAGES 4

#define VSA_MAX_GROUPS (VSAOGM_MAX_DELTA * VSAOGM_MAX_DELTA)

// staging / output slots of the pipelined host I/O (vsaogm_*_host_async): VSAOGM_IO_SLOTS of each; a slot
// is reused VSA_IO_SLOTS calls later, so the host may keep VSA_IO_SLOTS - 1 steps in flight
#define VSA_IO_SLOTS VSAOGM_IO_SLOTS
#define VSA_ND_PLANS 4   // cached NUFFT-decode plans (decode geometries)

// Decode GEMM problem groups (one per quadrant with decoded cells; delta = 1: one group).
// Group g: A-table rows [a_row0, a_row0 + mrows) = class 0 then class 1 blocks of nrows grid
// rows each (decoded rows row0 .. row0+nrows-1, relative to the first decoded row), times the
// grid columns [col0, col0 + ncols).
struct Groups {
    int n;
    int a_row0[VSA_MAX_GROUPS], mrows[VSA_MAX_GROUPS], nrows[VSA_MAX_GROUPS], row0[VSA_MAX_GROUPS];
    int col0[VSA_MAX_GROUPS], ncols[VSA_MAX_GROUPS];
};

struct ProfRec {
    int kid;
    cudaEvent_t a, b;
};

struct vsaogm_ctx {
    int device = 0;
    int num_sms = 148;
    int32_t D = 0;      // phasor dimensions
    int32_t Dp = 0;     // D rounded up to 32 (k-group of the interleaved K layout)
    int32_t Kp = 0;     // 2 * Dp: real contraction length of the decode GEMM
    double l = 1.0;
    uint64_t seed = 0;   // theta seed (fusion precondition: same axis vectors)
    int32_t delta = 1;   // quadrants per axis (sec. III-B-4); delta^2 quadrants
    int32_t nq = 1;      // delta^2
    int32_t nslots = 2;  // 2 delta^2 memories, slot = 2 beta + psi
    std::vector<double> qcx, qcy;                  // quadrant centres (host, fp64)
    double *d_qc = nullptr;                        // quadrant centres (device) [nq][2]
    uint8_t *d_slot = nullptr; size_t slot_cap = 0;   // per-point slot (sorted encode)
    int *d_bhist = nullptr; size_t bhist_cap = 0;     // per-block slot histograms
    int *d_sortmeta = nullptr;                     // slot totals / starts / vchunk table
    double2 *d_sorted = nullptr; size_t sorted_cap = 0;   // centred fp64 coordinates in slot order
    int4 *d_runs = nullptr; size_t runs_cap = 0;      // runs of one slot (sorted encode)
    // encode path: -1 auto (delta = 1: label-split blocks, measured fastest; delta > 1: sorted
    // runs); 0 sorted runs; 1 label-split / slot-filtered; 2 slot-filtered (tuning knob)
    int enc_path = -1;
    int enc_waves = 16;   // waves of slot-filtered encode blocks (tuning knob)
    int enc_runs_waves = 4;   // waves of sorted-run encode blocks (tuning knob)
    int enc_npoly = 1;  // phasors per 8 evaluated by the FMA polynomial instead of MUFU (tuning knob)
    int enc_minb = 6;   // encode blocks resident per SM (6: 80 regs, 8: <= 64 regs) (tuning knob)
    // packed fp32x2 encode (k_encode_bundle_x2, delta = 1, D >= 2048): 0 off (scalar kernel),
    // 1 uniform 4-warp blocks, 2 all-MUFU warps beside enc_x2_npoly-polynomial warps (default,
    // measured fastest in the pipelined schedule: (0 | 4), 4 blocks/SM), 3 one-polynomial warps
    // beside enc_x2_npoly-polynomial warps
    // 4: the pair (half-angle) kernel k_encode_pairs, all-MUFU warps beside enc_x2_npoly-FMA warps
    int enc_x2 = 4;
    int enc_pairs_npoly = 4;  // FMA-pipe dimensions of 8 in the pair kernel's second warp role
    int enc_pairs_minb = 3;   // resident pair-kernel blocks per SM (3: 80 registers, no spills)
    int enc_pairs_split = 1;
    // encode method: -1 auto (the NUFFT where its modelled time is lower), 0 direct (pair kernels),
    // 1 type-3 NUFFT (nufft.cu; delta = 1, D >= 2048)
    int enc_method = -1;
    bool nu_ready = false;
    double nu_h = 0, nu_tau = 0, nu_tau2 = 0, nu_lo = 0;
    int nu_n1 = 0, nu_logn = 0, nu_ntx = 0;
    void *d_nu_grid = nullptr, *d_nu_f1 = nullptr, *d_nu_G = nullptr;   // u64 32.32 grids [2][n1][n1], packed f32x2 [n1][2 K2], [2 K2][2 K2]
    int *d_nu_bins = nullptr;   // bin counts [nb], offsets [nb + 1], unit offsets [nb + 1], unit count [1]
    void *d_nu_key = nullptr, *d_nu_sorted = nullptr; size_t nu_pts_cap = 0;   // per-point (bin, slot); binned points
    float *d_nu_psi = nullptr;                                         // 1 / psi^(l - n1/2)
    void *d_nu_tw = nullptr, *d_nu_ph = nullptr;                       // twiddles, centring phases
    int nd_bps = 0;                                                    // NUFFT decode FFTs: resident blocks per SM cap (0 = occupancy limit; tuning)
    int pdl = 1;                                                       // programmatic dependent launch of the step's kernels (tuning)
    void *d_nu_kpar = nullptr;                                         // per-k interpolation parameters (NuKpar [D])
    int *d_nu_out = nullptr; size_t nu_out_cap = 0;                    // outliers per chunk  // 1 (default): one class per block (k_encode_pairs1, 64 registers, 4 per SM)
    int enc_x2_npoly = 4;   // polynomial dimensions of 8 in the second warp role
    int enc_x2_waves = 4;   // waves of packed encode blocks (dynamic SM balance vs partials)
    int enc_x2_minb = 4;    // resident 8-warp blocks per SM (4: 64 registers, the default; 3: 80)
    int enc_kt = 8;     // phasor dimensions per encode thread (8, or 16 as a tuning variant)
    // decode / pipeline / entropy tuning variants (vsaogm_set_tuning; defaults = measured best)
    int gemm_variant = -1;  // -1 auto (CTA pair), 0 CTA pair, 1 single CTA (one group only)
    int gemm_bn = 0;        // 0 auto, else the CTA-pair tile width (128..256, multiple of 32)
    int gemm_splits = 0;    // 0 auto, else the split-K factor
    int gemm_agen = 0;      // 1: A phasor tiles generated in the GEMM (no table A)
    int gemm_l2_hints = 0;  // TMA L2 eviction hints in the decode GEMM: 0 none (default: no measured gain), 1 A first + B last, 2 B last
    int pipe_early = 0;     // 1: release the next encode before table A (measured slower)
    int entropy_kernel = 0; // 0 auto (column-walk box kernel where it applies); 1 generic kernel; 2 TMA-streamed box kernel
    int entropy_rw = 0;     // 0 auto, else output rows per streamed work item (test hook)
    int table_rows = 32;    // table rows per thread of k_table (setup amortised over them)
    // decode method: -1 auto (the type-1 NUFFT of nudecode.cu where it applies and its modelled
    // time is lower), 0 the tcgen05 GEMM over phasor tables, 1 the NUFFT (delta = 1)
    int dec_method = -1;
    void *nd_plans[VSA_ND_PLANS] = {};   // cached NUFFT-decode plans (nudecode.cu), one per geometry
    int nd_nplans = 0;
    int64_t nd_tick = 0;
    void *d_nd_tw = nullptr;                          // twiddles for transforms up to 8192 points
    void *d_nd_G = nullptr; size_t nd_G_cap = 0;      // compact spread grid [Wx][Wy] complex fp32
    void *d_nd_T = nullptr; size_t nd_T_cap = 0;      // column-transformed band [Wx][ldt] complex fp32
    void *d_nd_st = nullptr; size_t nd_st_cap = 0;    // point strengths in bin order [2 D] complex fp32
    vsaogm_bounds bounds{};
    double cx = 0, cy = 0;            // phase origin = bounds centre
    std::vector<double> thx, thy;     // host fp64 theta

    // device state
    float *d_wx = nullptr, *d_wy = nullptr;        // theta / l, fp32 rad/m [Dp] (0-padded)
    double *d_tx_turns = nullptr, *d_ty_turns = nullptr;   // theta / (2 pi l), fp64 turns per metre [Dp]
    double *d_m = nullptr;                         // committed memories [2][Dp][2]
    // pending memories [S][Dp][2] followed by the S pending point counts (integer-valued fp64),
    // one contiguous buffer so that a multi-rank job sums both with ONE all-reduce (Alg. 3)
    double *d_pending = nullptr;
    long long *d_counts = nullptr;                 // [S]
    double *d_pcounts = nullptr;                   // = d_pending + 2 S Dp (not a separate allocation)
    double *d_norm2 = nullptr;                     // ||m_c||^2 [S], then sqrt(D) / ||m_c|| [S]
    float2 *d_mhat = nullptr;                      // sqrt(D) m_c / ||m_c||, fp32 [S][Dp]
    double *d_normpart = nullptr;                  // per-block partial ||m_c||^2 [S][16], then S u32 tickets
    int *d_err = nullptr;                          // deferred error bits
    int *d_ent_ctr = nullptr;                      // streamed entropy work queue [2]: next item, warps done
    float2 *d_part = nullptr;                      // encode chunk partials
    size_t part_cap = 0;                           // in float2
    long long *d_part_cnt = nullptr;
    size_t part_cnt_cap = 0;
    float2 *d_stage_xy = nullptr;                  // host-encode staging
    uint8_t *d_stage_lab = nullptr;
    size_t stage_cap = 0;

    // decode tables and buffers
    void *d_A = nullptr;  size_t A_cap = 0;        // bytes
    void *d_B = nullptr;  size_t B_cap = 0;
    bool B_valid = false;
    double B_x0 = 0, B_res = 0; int32_t B_cols = 0; int B_prec = -1;
    float *d_hb = nullptr; size_t hb_cap = 0;      // [2][R_ext][ldh] fp32
    float *d_ws = nullptr; size_t ws_cap = 0;      // split-K partial sums (bytes)
    int estimator = 0;                             // 0: window mean of H_b(p); 1: 8-bit histogram entropy
    uint8_t *d_code = nullptr; size_t code_cap = 0;   // [2][R_ext][ldh] 8-bit p (histogram estimator)
    int g_estimator = 0;                           // estimator of the last decode
    float *d_S = nullptr; size_t S_cap = 0;        // host-entropy scratch
    uint8_t *d_lab = nullptr; size_t lab_cap = 0;

    // pipelined host I/O (vsaogm_*_host_async): VSA_IO_SLOTS staging / output slots each, copy streams
    cudaStream_t up = nullptr, down = nullptr;     // upload (H2D) / download (D2H) streams
    float2 *d_in_xy[VSA_IO_SLOTS] = {}; size_t in_xy_cap[VSA_IO_SLOTS] = {};
    uint8_t *d_in_lab[VSA_IO_SLOTS] = {}; size_t in_lab_cap[VSA_IO_SLOTS] = {};
    float *d_out_S[VSA_IO_SLOTS] = {}; size_t out_S_cap[VSA_IO_SLOTS] = {};
    uint8_t *d_out_lab[VSA_IO_SLOTS] = {}; size_t out_lab_cap[VSA_IO_SLOTS] = {};
    cudaEvent_t ev_up[VSA_IO_SLOTS] = {};       // upload of slot done
    cudaEvent_t ev_used[VSA_IO_SLOTS] = {};     // encode has consumed staging slot
    cudaEvent_t ev_out[VSA_IO_SLOTS] = {};      // entropy wrote output slot
    cudaEvent_t ev_down[VSA_IO_SLOTS] = {};     // download of output slot done
    int64_t in_seq = 0, out_seq = 0;            // calls so far (slot = seq % VSA_IO_SLOTS)
    int *h_err = nullptr;                            // pinned [VSA_IO_SLOTS]: deferred error bits per output slot

    // encode stream (vsaogm_set_encode_stream): encodes run there and overlap the previous
    // decode; ev_enc orders the next commit after them, ev_main orders them after the last
    // commit / reset / table-A build on the context stream
    cudaStream_t enc_stream = nullptr;
    cudaEvent_t ev_enc = nullptr, ev_main = nullptr;
    bool enc_inflight = false, main_mark = false;

    // last decode geometry
    bool decoded = false;
    int32_t g_rows = 0, g_cols = 0, g_r0 = 0, g_r1 = 0, g_rlo = 0, g_rext = 0, g_halo = 0;

    cudaStream_t stream = nullptr;
    bool pending_taken = false;   // multi-rank mode
    bool dirty = false;           // pending holds uncommitted work

    // profiling
    bool prof = false;
    std::vector<ProfRec> prof_live;
    std::vector<cudaEvent_t> ev_pool;
    double prof_ms[VSAOGM_NKERNELS] = {0};
    int64_t prof_n[VSAOGM_NKERNELS] = {0};
    int64_t launches = 0;
};

// ---- encode-stream ordering (api.cu) -----------------------------------------
extern "C" int vsa_join_encode(vsaogm_ctx *c);   // context stream waits for in-flight encodes
extern "C" int vsa_mark_main(vsaogm_ctx *c);     // later encodes wait for the context stream's work so far

// ---- profiling brackets (api.cu) -------------------------------------------
int vsa_prof_begin(vsaogm_ctx *c, int kid, cudaEvent_t *a);
void vsa_prof_end(vsaogm_ctx *c, int kid, cudaEvent_t a);

// ---- launchers implemented in the kernel translation units -----------------
int vsa_launch_encode(vsaogm_ctx *c, const float *xy, const uint8_t *lab, int64_t n);
int vsa_launch_encode_sorted(vsaogm_ctx *c, const float *xy, const uint8_t *lab, int64_t n);
int vsa_launch_encode_nufft(vsaogm_ctx *c, const float *xy, const uint8_t *lab, int64_t n, int64_t chunk_pts,
                            int chunks);
int vsa_launch_mhat(vsaogm_ctx *c);
int vsa_launch_nufft_outliers(vsaogm_ctx *c, const float *xy, const uint8_t *lab, int64_t n, int64_t chunk_pts,
                              int chunks);
bool vsa_nufft_wanted(vsaogm_ctx *c, int64_t n);
int vsa_launch_commit(vsaogm_ctx *c);
int vsa_launch_norms(vsaogm_ctx *c, int do_commit);   // [commit +] norms + scaled memory mhat
int vsa_launch_table_B(vsaogm_ctx *c, double x0, double res, int32_t cols, int prec);
int vsa_launch_table_A(vsaogm_ctx *c, const Groups &G, double y0, double res, int32_t r_lo, int prec,
                       const int *slot0);
int vsa_launch_decode_gemm(vsaogm_ctx *c, const Groups &G, int32_t a_rows, int32_t N, int prec, float inv_scale,
                           float *hb, float *q, int32_t r_ext, int32_t q_off, int32_t band_rows, const int *slot0,
                           double y0, double res, int32_t r_lo);
bool vsa_nudecode_applies(vsaogm_ctx *c, double x0, double y0, double res, int32_t cols, int32_t r_lo, int32_t r_ext);
int vsa_launch_decode_nufft(vsaogm_ctx *c, double x0, double y0, double res, int32_t cols, int32_t r_lo, int32_t r_ext,
                            float *hb, uint8_t *code, size_t ldh, float *q, int32_t q_off, int32_t band_rows,
                            bool mark_main);
void vsa_nudecode_free(vsaogm_ctx *c);
int vsa_launch_entropy(vsaogm_ctx *c, const vsaogm_entropy_params *p, float *S, uint8_t *lab);
int vsa_gemm_raw(const void *A, const void *B, int32_t M, int32_t N, int32_t K, int prec, float *C,
                 cudaStream_t s, int num_sms, int variant, int bn = 0, int splits = 0);
// staged host-encode / I/O helpers: comments in api.cu

// cuTensorMapEncodeTiled from the driver (gemm_tc.cu), nullptr if unavailable
#include <cudaTypedefs.h>
PFN_cuTensorMapEncodeTiled_v12000 vsa_tmap_encode_fn();

// ---- PTX helpers (sm_100a) ---------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void *p)
{
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t *bar)
{
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity)
{
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ void tma_load_2d(void *dst, const CUtensorMap *map, uint64_t *bar, int c0, int c1)
{
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void tc_commit(uint64_t *bar)
{
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}

__device__ __forceinline__ void tc_mma_f16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                           uint32_t accumulate)
{
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}

// K-major operand tile in shared memory, 128-byte swizzle (matches the TMA
// SWIZZLE_128B box of 64 16-bit elements per row): 8-row atoms of 1024 B.
// Descriptor fields (tcgen05 shared-memory matrix descriptor): start address
// >> 4 in [0,14), leading byte offset >> 4 in [16,30) (unused for swizzled
// K-major, 1), stride byte offset >> 4 in [32,46) (1024 B between 8-row
// groups), version 1 in [46,48), swizzle mode 2 (128B) in [61,64).
__device__ __forceinline__ uint64_t sw128_kmajor_desc(uint32_t smem_addr)
{
    return (uint64_t)((smem_addr & 0x3FFFFu) >> 4) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
           ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}

// Instruction descriptor, kind::f16: D fp32 (bits 4-5 = 1), A/B format
// (bits 7-9, 10-12: 0 = f16, 1 = bf16), both K-major, N >> 3 at bit 17,
// M >> 4 at bit 24.
__host__ __device__ __forceinline__ uint32_t make_idesc_f16(int bf16, int M, int N)
{
    return (1u << 4) | ((uint32_t)bf16 << 7) | ((uint32_t)bf16 << 10) | ((uint32_t)(N >> 3) << 17) |
           ((uint32_t)(M >> 4) << 24);
}

#define TMEM_LD_32x32b_X32(taddr, v)                                                                          \
    asm volatile(                                                                                             \
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "                                                             \
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"                                             \
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"                            \
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),     \
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),            \
          "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]),          \
          "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]),          \
          "=r"(v[29]), "=r"(v[30]), "=r"(v[31])                                                               \
        : "r"(taddr))

__device__ __forceinline__ void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// sin/cos on the FMA + ALU pipes (no MUFU), 18 instructions: half-turn
// reduction phi = q pi + r (q by the magic-number rint, 2-term Cody-Waite pi;
// |q| < 2^12 keeps q * 3.140625 exact), then near-minimax polynomials on
// [-pi/2, pi/2] (odd degree 9 / even degree 10, fitted by tools/fit_sincos.py;
// fp32 Horner max error 1.2e-7, i.e. as accurate as MUFU.SIN/COS), and the
// sign (-1)^q applied to both by one shift and two xors.  Used for a
// fraction of the phasors so that the XU (MUFU) pipe and the issue slots are
// both busy: the encode is SFU-bound otherwise.
__device__ __forceinline__ void sincos_fma(float phi, float *s_out, float *c_out)
{
    const float magic = 12582912.f;                 // 1.5 * 2^23: x + magic rounds x to an integer
    const float tq = fmaf(phi, 0.318309886183790672f, magic);   // phi / pi + magic
    const int qi = __float_as_int(tq);              // low bits hold q mod 2^22
    const float q = tq - magic;
    float r = fmaf(q, -3.140625f, phi);             // exact (8-bit constant)
    r = fmaf(q, -9.67653589793e-4f, r);             // pi - 3.140625
    const float r2 = r * r;
    float p = fmaf(r2, 2.600054358e-06f, -1.980661473e-04f);
    p = fmaf(p, r2, 8.333017118e-03f);
    p = fmaf(p, r2, -1.666665673e-01f);
    const float s = fmaf(p * r2, r, r);
    float c = fmaf(r2, -2.607710314e-07f, 2.476188638e-05f);
    c = fmaf(c, r2, -1.388840377e-03f);
    c = fmaf(c, r2, 4.166664183e-02f);
    c = fmaf(c, r2, -5.000000000e-01f);
    c = fmaf(c, r2, 1.0f);
    const int sign = qi << 31;                      // (-1)^q
    *s_out = __int_as_float(__float_as_int(s) ^ sign);
    *c_out = __int_as_float(__float_as_int(c) ^ sign);
}

// ---- programmatic dependent launch (PDL) -------------------------------------------------------
// The streaming step is a chain of 15 short dependent kernels; an ordinary launch starts a kernel
// only after its predecessor has drained (~2 us of launch latency per link on the step's critical
// path).  vsa_launch_pdl launches with programmatic stream serialization: the kernel's blocks are
// scheduled as the predecessor's blocks exit, and wait at vsa_pdl_wait() -- griddepcontrol.wait
// returns when the predecessor grid has completed and its writes are visible -- so the launch
// latency, the block scheduling and the plan-constant prologues overlap the predecessor's tail.
// Every kernel launched this way calls vsa_pdl() / vsa_pdl_wait() before it touches global memory
// written by its predecessor; launched ordinarily the instruction is a no-op.
// The trigger is the implicit one, at each block's exit: an explicit griddepcontrol.launch_dependents at
// the start of every kernel (the first version) made the dependent grid's blocks resident -- holding
// registers, shared memory and thread slots while they wait -- for the whole run of their predecessor,
// which starved the other stream's kernels in the pipelined schedule (C4 step 0.129 -> 0.113 ms, end
// to end 0.136 -> 0.126 ms without it; the serial step is unchanged).
__device__ __forceinline__ void vsa_pdl_launch() {}
__device__ __forceinline__ void vsa_pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void vsa_pdl()
{
    vsa_pdl_launch();
    vsa_pdl_wait();
}

template <typename... KArgs, typename... Args>
inline cudaError_t vsa_launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args &&...args)
{
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

// launch on the context's current stream: PDL unless the tuning knob `pdl` is 0
template <typename... KArgs, typename... Args>
inline cudaError_t vsa_launch(const vsaogm_ctx *c, void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, Args &&...args)
{
    if (c->pdl) return vsa_launch_pdl(kern, grid, block, smem, c->stream, static_cast<Args &&>(args)...);
    kern<<<grid, block, smem, c->stream>>>(static_cast<KArgs>(args)...);
    return cudaGetLastError();
}

// ---- packed fp32x2 arithmetic (FFMA2 / FMUL2 / FADD2, sm_100a) ----------------
// Two fp32 lanes in one 64-bit register pair; each lane rounds exactly as the
// scalar fmaf / __fmul_rn / __fadd_rn would.  One issue slot per two lanes: the
// encode is bound by the MUFU pipe and the issue slots together, so packing the
// angle, accumulation and polynomial arithmetic frees issue for more phasors
// (DESIGN.md section 6).  A scalar operand broadcast as pk2(f, f) compiles to
// the R.F32 / immediate broadcast form of the packed instruction.
typedef unsigned long long f32x2;

__device__ __forceinline__ f32x2 pk2(float a, float b)
{
    f32x2 r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ f32x2 bc2(float a) { return pk2(a, a); }
__device__ __forceinline__ void upk2(f32x2 v, float &a, float &b) { asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v)); }
__device__ __forceinline__ f32x2 fma2(f32x2 a, f32x2 b, f32x2 c)
{
    f32x2 r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
    return r;
}
__device__ __forceinline__ f32x2 mul2(f32x2 a, f32x2 b)
{
    f32x2 r;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ f32x2 add2(f32x2 a, f32x2 b)
{
    f32x2 r;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}

// sincos_fma on two angles at once: the same operations in the same order per
// lane (bit-identical to two sincos_fma calls), 15 packed FMA-pipe instructions
// plus the per-lane sign xors.
__device__ __forceinline__ void sincos_fma2(f32x2 phi, f32x2 &s_out, f32x2 &c_out)
{
    const float magic = 12582912.f;
    const f32x2 tq = fma2(phi, bc2(0.318309886183790672f), bc2(magic));
    const f32x2 q = add2(tq, bc2(-magic));
    f32x2 r = fma2(q, bc2(-3.140625f), phi);
    r = fma2(q, bc2(-9.67653589793e-4f), r);
    const f32x2 r2 = mul2(r, r);
    f32x2 p = fma2(r2, bc2(2.600054358e-06f), bc2(-1.980661473e-04f));
    p = fma2(p, r2, bc2(8.333017118e-03f));
    p = fma2(p, r2, bc2(-1.666665673e-01f));
    const f32x2 s = fma2(mul2(p, r2), r, r);
    f32x2 c = fma2(r2, bc2(-2.607710314e-07f), bc2(2.476188638e-05f));
    c = fma2(c, r2, bc2(-1.388840377e-03f));
    c = fma2(c, r2, bc2(4.166664183e-02f));
    c = fma2(c, r2, bc2(-5.000000000e-01f));
    c = fma2(c, r2, bc2(1.0f));
    float ta, tb, sa, sb, ca, cb;
    upk2(tq, ta, tb);
    upk2(s, sa, sb);
    upk2(c, ca, cb);
    const int ga = __float_as_int(ta) << 31, gb = __float_as_int(tb) << 31;
    s_out = pk2(__int_as_float(__float_as_int(sa) ^ ga), __int_as_float(__float_as_int(sb) ^ gb));
    c_out = pk2(__int_as_float(__float_as_int(ca) ^ ga), __int_as_float(__float_as_int(cb) ^ gb));
}

// Cheaper packed sin/cos for the encode's polynomial phasors: one-constant reduction
// r = phi - q fl(pi) (its error q |pi - fl(pi)| <= |phi| 2.8e-8 is below the fp32 rounding
// of phi itself, |phi| 6e-8, and below MUFU.SIN's |phi| 3e-8 x 2pi of the RZ turn
// conversion), odd degree-7 sin (fp32 max error 9.7e-7, MUFU-class) and even degree-8 cos
// (1.6e-7) near-minimax fits (tools/fit_sincos.py --lite): 12 packed FMA-pipe instructions
// instead of 15 per two phasors.
__device__ __forceinline__ void sincos_fma2_lite(f32x2 phi, f32x2 &s_out, f32x2 &c_out)
{
    const float magic = 12582912.f;
    const f32x2 tq = fma2(phi, bc2(0.318309886183790672f), bc2(magic));
    const f32x2 q = add2(tq, bc2(-magic));
    const f32x2 r = fma2(q, bc2(-3.14159274101257324f), phi);
    const f32x2 r2 = mul2(r, r);
    f32x2 p = fma2(r2, bc2(-1.849217806e-04f), bc2(8.312365972e-03f));
    p = fma2(p, r2, bc2(-1.666568071e-01f));
    const f32x2 s = fma2(mul2(p, r2), r, r);
    f32x2 c = fma2(r2, bc2(2.319438317e-05f), bc2(-1.385592739e-03f));
    c = fma2(c, r2, bc2(4.166398942e-02f));
    c = fma2(c, r2, bc2(-4.999993145e-01f));
    c = fma2(c, r2, bc2(1.0f));
    float ta, tb, sa, sb, ca, cb;
    upk2(tq, ta, tb);
    upk2(s, sa, sb);
    upk2(c, ca, cb);
    const int ga = __float_as_int(ta) << 31, gb = __float_as_int(tb) << 31;
    s_out = pk2(__int_as_float(__float_as_int(sa) ^ ga), __int_as_float(__float_as_int(sb) ^ gb));
    c_out = pk2(__int_as_float(__float_as_int(ca) ^ ga), __int_as_float(__float_as_int(cb) ^ gb));
}

// Per-thread phasor accumulators of the packed encode: KT dimensions (KT even) held
// as KT/2 dimension pairs (j, j+1), the last NPOLY dimensions on the polynomial.
// One point at a time: the pair's two angles come from one FMUL2 + FFMA2 with the
// point coordinates broadcast, and the pair's cos / sin sums are two FADD2.  Every
// dimension sums its points in point order; MUFU dimensions use the scalar kernel's
// per-lane arithmetic, polynomial pairs the cheaper sincos_fma2_lite.
template <int KT, int NPOLY>
struct PhasorAcc {
    static_assert(KT % 2 == 0, "dimension pairs");
    static constexpr int NP = KT / 2;
    f32x2 wx[NP], wy[NP];   // (w_j, w_j+1) per pair
    f32x2 re[NP], im[NP];   // (sum cos_j, sum cos_j+1), (sum sin_j, sum sin_j+1)

    __device__ __forceinline__ void init(const float *fx, const float *fy)
    {
#pragma unroll
        for (int q = 0; q < NP; ++q) {
            wx[q] = pk2(fx[2 * q], fx[2 * q + 1]);
            wy[q] = pk2(fy[2 * q], fy[2 * q + 1]);
            re[q] = im[q] = pk2(0.f, 0.f);
        }
    }

    __device__ __forceinline__ void point(float x, float y)
    {
        const f32x2 X = bc2(x), Y = bc2(y);
#pragma unroll
        for (int q = 0; q < NP; ++q) {
            const f32x2 phi = fma2(wx[q], X, mul2(wy[q], Y));   // fmaf(w^x, x, w^y * y) per lane
            constexpr int J0 = 0;
            const int j0 = J0 + 2 * q;
            if (j0 + 1 < KT - NPOLY) {                    // both on MUFU
                float pa, pb, sa, ca, sb, cb;
                upk2(phi, pa, pb);
                __sincosf(pa, &sa, &ca);
                __sincosf(pb, &sb, &cb);
                re[q] = add2(re[q], pk2(ca, cb));
                im[q] = add2(im[q], pk2(sa, sb));
            } else if (j0 >= KT - NPOLY) {                // both on the polynomial
                f32x2 S, C;
                sincos_fma2_lite(phi, S, C);
                re[q] = add2(re[q], C);
                im[q] = add2(im[q], S);
            } else {                                      // MUFU, polynomial
                float pa, pb, sa, ca, sb, cb;
                upk2(phi, pa, pb);
                __sincosf(pa, &sa, &ca);
                sincos_fma(pb, &sb, &cb);
                re[q] = add2(re[q], pk2(ca, cb));
                im[q] = add2(im[q], pk2(sa, sb));
            }
        }
    }

    __device__ __forceinline__ float2 get(int j) const
    {
        float a, b, c, d;
        upk2(re[j >> 1], a, b);
        upk2(im[j >> 1], c, d);
        return (j & 1) ? make_float2(b, d) : make_float2(a, c);
    }
};

// Packed cos only, same reduction and cos polynomial as sincos_fma2_lite: 8 packed FMA-pipe
// instructions plus the sign xors, for the half-difference factor of the pair encode.
__device__ __forceinline__ f32x2 cos_fma2_lite(f32x2 phi)
{
    const float magic = 12582912.f;
    const f32x2 tq = fma2(phi, bc2(0.318309886183790672f), bc2(magic));
    const f32x2 q = add2(tq, bc2(-magic));
    const f32x2 r = fma2(q, bc2(-3.14159274101257324f), phi);
    const f32x2 r2 = mul2(r, r);
    f32x2 c = fma2(r2, bc2(2.319438317e-05f), bc2(-1.385592739e-03f));
    c = fma2(c, r2, bc2(4.166398942e-02f));
    c = fma2(c, r2, bc2(-4.999993145e-01f));
    c = fma2(c, r2, bc2(1.0f));
    float ta, tb, ca, cb;
    upk2(tq, ta, tb);
    upk2(c, ca, cb);
    return pk2(__int_as_float(__float_as_int(ca) ^ (__float_as_int(ta) << 31)),
               __int_as_float(__float_as_int(cb) ^ (__float_as_int(tb) << 31)));
}

// Block barrier without .aligned (PTX barrier.sync): legal when the warps of a block reach it
// from different (warp-uniform) code paths, e.g. the role-templated loops of the encode.
__device__ __forceinline__ void block_sync_any() { asm volatile("barrier.sync 0;" ::: "memory"); }

// Pair accumulators of the half-angle encode: two points a, b of one
// class contribute
//     e^{i phi_a} + e^{i phi_b} = 2 cos(delta) e^{i sigma},
//     sigma = w^x xbar + w^y ybar,  delta = w^x dx + w^y dy,
//     xbar = (x_a + x_b) / 2,  dx = (x_a - x_b) / 2  (same for y),
// i.e. three sin/cos evaluations per two phasors instead of four.  A thread holds KT
// dimensions as KT/2 packed pairs; re/im accumulate cos(delta) (cos sigma, sin sigma), i.e.
// HALF the sum (the factor 2 is applied once, exactly, when the partials are stored).  The
// last NPOLY dimensions evaluate all three on the FMA pipe (sincos_fma2_lite, cos_fma2_lite),
// the others on MUFU.  A single leftover point adds (1/2) e^{i phi}.
// The thread's KT phase rates (w^x, w^y) as KT/2 packed pairs, shared by its accumulators.
template <int KT>
struct PairW {
    f32x2 wx[KT / 2], wy[KT / 2];
    __device__ __forceinline__ void init(const float *fx, const float *fy)
    {
#pragma unroll
        for (int q = 0; q < KT / 2; ++q) {
            wx[q] = pk2(fx[2 * q], fx[2 * q + 1]);
            wy[q] = pk2(fy[2 * q], fy[2 * q + 1]);
        }
    }
};

template <int KT, int NPOLY>
struct PairAcc {
    static_assert(KT % 2 == 0, "dimension pairs");
    static constexpr int NP = KT / 2;
    f32x2 re[NP], im[NP];

    __device__ __forceinline__ void init()
    {
#pragma unroll
        for (int q = 0; q < NP; ++q) re[q] = im[q] = pk2(0.f, 0.f);
    }

    // P = (xbar, ybar, dx, dy), centred metres
    __device__ __forceinline__ void pair(const PairW<KT> &w, float4 P)
    {
        const f32x2 X = bc2(P.x), Y = bc2(P.y), DX = bc2(P.z), DY = bc2(P.w);
#pragma unroll
        for (int q = 0; q < NP; ++q) {
            const f32x2 sg = fma2(w.wx[q], X, mul2(w.wy[q], Y));    // sigma per lane
            const f32x2 dl = fma2(w.wx[q], DX, mul2(w.wy[q], DY));  // delta per lane
            const int j0 = 2 * q;
            if (j0 + 1 < KT - NPOLY) {                            // both on MUFU
                float sa, sb, da, db, ssa, csa, ssb, csb;
                upk2(sg, sa, sb);
                upk2(dl, da, db);
                __sincosf(sa, &ssa, &csa);
                __sincosf(sb, &ssb, &csb);
                const f32x2 cd = pk2(__cosf(da), __cosf(db));
                re[q] = fma2(cd, pk2(csa, csb), re[q]);
                im[q] = fma2(cd, pk2(ssa, ssb), im[q]);
            } else if (j0 >= KT - NPOLY) {                        // both on the FMA pipe
                f32x2 S, C;
                sincos_fma2_lite(sg, S, C);
                const f32x2 cd = cos_fma2_lite(dl);
                re[q] = fma2(cd, C, re[q]);
                im[q] = fma2(cd, S, im[q]);
            } else {                                              // MUFU, FMA pipe
                float sa, sb, da, db, ssa, csa, ssb, csb;
                upk2(sg, sa, sb);
                upk2(dl, da, db);
                __sincosf(sa, &ssa, &csa);
                sincos_fma(sb, &ssb, &csb);
                float sdb, cdb;
                sincos_fma(db, &sdb, &cdb);
                const f32x2 cd = pk2(__cosf(da), cdb);
                re[q] = fma2(cd, pk2(csa, csb), re[q]);
                im[q] = fma2(cd, pk2(ssa, ssb), im[q]);
            }
        }
    }

    // a single (leftover) point: + (1/2) e^{i phi}, MUFU
    __device__ __forceinline__ void single(const PairW<KT> &w, float x, float y)
    {
        const f32x2 X = bc2(x), Y = bc2(y), H = bc2(0.5f);
#pragma unroll
        for (int q = 0; q < NP; ++q) {
            float pa, pb, sa, ca, sb, cb;
            upk2(fma2(w.wx[q], X, mul2(w.wy[q], Y)), pa, pb);
            __sincosf(pa, &sa, &ca);
            __sincosf(pb, &sb, &cb);
            re[q] = fma2(H, pk2(ca, cb), re[q]);
            im[q] = fma2(H, pk2(sa, sb), im[q]);
        }
    }

    // the dimension's full sum (2 x the half sum; exact scaling)
    __device__ __forceinline__ float2 get(int j) const
    {
        float a, b, c, d;
        upk2(re[j >> 1], a, b);
        upk2(im[j >> 1], c, d);
        return (j & 1) ? make_float2(2.f * b, 2.f * d) : make_float2(2.f * a, 2.f * c);
    }
};

// ---- CTA-pair (cta_group::2) helpers -----------------------------------------
__device__ __forceinline__ uint32_t cluster_ctarank()
{
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}

__device__ __forceinline__ void cluster_sync_all()
{
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// wait with cluster-scope acquire (arrivals may come from the peer CTA)
__device__ __forceinline__ void mbar_wait_cluster(uint64_t *bar, uint32_t parity)
{
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAITC_%=:\n\t"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAITC_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

// arrive on the barrier at the same shared-memory offset in CTA `cta` of the cluster
__device__ __forceinline__ void mbar_arrive_cluster(uint64_t *bar, uint32_t cta)
{
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(bar)), "r"(cta));
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(r) : "memory");
}

// 2-SM TMA load: data lands in this CTA's shared memory, the transaction bytes
// are counted on the barrier of CTA 0 of the pair (peer bit 24 cleared).
__device__ __forceinline__ void tma_load_2d_2sm(void *dst, const CUtensorMap *map, uint64_t *bar, int c0, int c1)
{
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
        "%3}], [%4];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar) & 0xFEFFFFFFu)
        : "memory");
}

// as tma_load_2d_2sm, multicast: the box lands at the same offset in every CTA of ctaMask, and
// each destination's bytes are counted on the barrier of its own pair's CTA 0
__device__ __forceinline__ void tma_load_2d_2sm_mc(void *dst, const CUtensorMap *map, uint64_t *bar, int c0, int c1,
                                                   uint16_t mask)
{
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster "
        "[%0], [%1, {%2, %3}], [%4], %5;" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar) & 0xFEFFFFFFu), "h"(mask)
        : "memory");
}

// as tma_load_2d_2sm with an L2 eviction-priority hint (64-bit cache policy: the encodings of
// createpolicy.fractional evict_first / evict_last with fraction 1.0)
constexpr uint64_t VSA_L2_EVICT_FIRST = 0x12F0000000000000ull;
constexpr uint64_t VSA_L2_EVICT_LAST = 0x14F0000000000000ull;
__device__ __forceinline__ void tma_load_2d_2sm_hint(void *dst, const CUtensorMap *map, uint64_t *bar, int c0, int c1,
                                                     uint64_t policy)
{
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], "
        "[%1, {%2, %3}], [%4], %5;" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar) & 0xFEFFFFFFu), "l"(policy)
        : "memory");
}

__device__ __forceinline__ void tc_mma2_f16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                            uint32_t accumulate)
{
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}

// commit the issuing thread's prior tcgen05 ops to the barrier at this offset in both CTAs
__device__ __forceinline__ void tc_commit2_mc(uint64_t *bar, uint16_t mask = 3)
{
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            smem_u32(bar)),
        "h"(mask)
        : "memory");
}
