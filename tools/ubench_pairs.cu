// ubench_pairs.cu -- measured ALU ceiling of the pair (half-angle) encode.
//
// Runs the exact bundle loop of k_encode_pairs1 (PairAcc<8, NPOLY>::pair on pair records read
// from shared memory as warp-uniform broadcasts, the kernel's warp roles: warps 0-3 all-MUFU,
// warps 4-7 NPOLY of 8 dimensions on the FMA pipe) with no staging, no global traffic and no
// tail: 4 blocks of 256 threads per SM (64 registers), every SM busy for ~50 ms.  Prints one
// JSON line per NPOLY with phasors per clock per SM and per second; the best of them is the
// measured ceiling the bench divides by.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Iinclude \
//        -Ipaper_2408_09066_b200/csrc -o /tmp/ubench_pairs tools/ubench_pairs.cu && /tmp/ubench_pairs
#include <cstdio>

#include "common.cuh"

constexpr int NREC = 128;     // pair records in shared memory
constexpr int PASSES = 64;    // passes over the records per block

template <int NPB>
__global__ void __launch_bounds__(256, 4) k_pairs_loop(const float *__restrict__ wx, const float *__restrict__ wy,
                                                       float2 *__restrict__ out, long long *__restrict__ clk)
{
    __shared__ float4 s_q[NREC];
    const int tid = threadIdx.x;
    if (tid < NREC) {
        const float t = 0.37f * (float)(tid + 1) + 0.001f * (float)blockIdx.x;
        s_q[tid] = make_float4(20.f * __sinf(t), 20.f * __cosf(1.3f * t), 9.f * __sinf(2.1f * t), 7.f * __cosf(0.7f * t));
    }
    __syncthreads();
    float fx[8], fy[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        fx[j] = wx[(tid * 8 + j) & 1023];
        fy[j] = wy[(tid * 8 + j) & 1023];
    }
    PairW<8> w;
    w.init(fx, fy);
    const long long t0 = clock64();
    auto run = [&](auto acc) {
        acc.init();
        for (int pass = 0; pass < PASSES; ++pass) {
#pragma unroll 1
            for (int p = 0; p < NREC; ++p) acc.pair(w, s_q[p]);
        }
        float2 sum = make_float2(0.f, 0.f);
#pragma unroll
        for (int j = 0; j < 8; ++j) {   // every dimension's sum is live
            const float2 g = acc.get(j);
            sum.x += g.x;
            sum.y += g.y;
        }
        out[blockIdx.x * 256 + tid] = sum;
    };
    if ((tid >> 5) >= 4) run(PairAcc<8, NPB>{});
    else run(PairAcc<8, 0>{});
    const long long t1 = clock64();
    if (tid == 0) clk[blockIdx.x] = t1 - t0;
}

template <int NPB>
void run(const float *wx, const float *wy, float2 *out, long long *clk, int sms, int mhz)
{
    const int blocks = sms * 4;
    k_pairs_loop<NPB><<<blocks, 256>>>(wx, wy, out, clk);   // warm-up
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    const int reps = 5;
    for (int r = 0; r < reps; ++r) k_pairs_loop<NPB><<<blocks, 256>>>(wx, wy, out, clk);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, b);
    ms /= reps;
    // phasors: every thread evaluates 8 dimensions x 2 points per pair record
    const double phasors = (double)blocks * 256 * 8 * 2 * NREC * PASSES;
    const double per_s = phasors / (ms * 1e-3);
    const double per_clk_sm = per_s / (sms * (double)mhz * 1e6);
    printf("{\"npoly_role_b\": %d, \"ms\": %.4f, \"phasors_per_s\": %.4e, \"phasors_per_clk_per_sm_at_%d_mhz\": %.3f, "
           "\"fma_pipe_fraction\": %.4f, \"err\": \"%s\"}\n",
           NPB, ms, per_s, mhz, per_clk_sm, NPB / 16.0, cudaGetErrorString(cudaGetLastError()));
}

int main()
{
    int dev = 0, sms = 0, khz = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, dev);
    const int mhz = khz / 1000;
    float *wx, *wy;
    float2 *out;
    long long *clk;
    cudaMalloc(&wx, 1024 * 4);
    cudaMalloc(&wy, 1024 * 4);
    cudaMalloc(&out, (size_t)sms * 4 * 256 * sizeof(float2));
    cudaMalloc(&clk, (size_t)sms * 4 * sizeof(long long));
    float h[1024];
    for (int i = 0; i < 1024; ++i) h[i] = 10.47f * (((i * 2654435761u) >> 8) / 16777216.f - 0.5f) * 2.f;
    cudaMemcpy(wx, h, sizeof h, cudaMemcpyHostToDevice);
    for (int i = 0; i < 1024; ++i) h[i] = 10.47f * (((i * 40503u + 7u) * 2654435761u >> 8) / 16777216.f - 0.5f) * 2.f;
    cudaMemcpy(wy, h, sizeof h, cudaMemcpyHostToDevice);
    run<0>(wx, wy, out, clk, sms, mhz);
    run<2>(wx, wy, out, clk, sms, mhz);
    run<4>(wx, wy, out, clk, sms, mhz);
    run<6>(wx, wy, out, clk, sms, mhz);
    run<8>(wx, wy, out, clk, sms, mhz);
    return 0;
}
