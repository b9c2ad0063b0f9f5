// ubench_pipes.cu -- issue/pipe throughput probe for the encode design:
// FFMA vs packed FFMA2 (fma.rn.f32x2) vs MUFU.SIN/COS, alone and mixed, in lane-ops per
// clock per SM.  Standalone: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ubench tools/ubench_pipes.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define ITERS 4096
#define CH 8

__device__ __forceinline__ unsigned long long f2u(float2 v) { return *reinterpret_cast<unsigned long long *>(&v); }
__device__ __forceinline__ float2 u2f(unsigned long long v) { return *reinterpret_cast<float2 *>(&v); }

__device__ __forceinline__ unsigned long long ffma2(unsigned long long a, unsigned long long b, unsigned long long c)
{
    unsigned long long r;
    asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
    return r;
}

// mode 0: FFMA only; 1: FFMA2 only; 2: MUFU sin+cos only; 3: 2 MUFU + 2 FFMA2 per step;
// 4: 2 MUFU + 4 FFMA (scalar)
template <int MODE>
__global__ void k(float *out, float seed, long long *clk)
{
    float a[CH], b[CH];
    unsigned long long p[CH];
    for (int i = 0; i < CH; ++i) {
        a[i] = seed * (threadIdx.x + i);
        b[i] = seed + i;
        p[i] = f2u(make_float2(a[i], b[i]));
    }
    const unsigned long long m = f2u(make_float2(0.999f, 0.998f)), c = f2u(make_float2(1e-3f, 2e-3f));
    long long t0 = clock64();
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < CH; ++i) {
            if (MODE == 0) { a[i] = fmaf(a[i], 0.999f, 1e-3f); b[i] = fmaf(b[i], 0.998f, 2e-3f); }
            if (MODE == 1) { p[i] = ffma2(p[i], m, c); }
            if (MODE == 2) { float s, co; __sincosf(a[i], &s, &co); a[i] = s + co; }
            if (MODE == 3) { float s, co; __sincosf(a[i], &s, &co); a[i] = s; b[i] += co; p[i] = ffma2(p[i], m, c); p[i] = ffma2(p[i], m, c); }
            if (MODE == 4) { float s, co; __sincosf(a[i], &s, &co); a[i] = s; b[i] += co; b[i] = fmaf(b[i], 0.999f, 1e-3f); b[i] = fmaf(b[i], 0.999f, 1e-3f); b[i] = fmaf(b[i], 0.999f, 1e-3f); }
        }
    }
    long long t1 = clock64();
    float acc = 0.f;
    for (int i = 0; i < CH; ++i) { float2 q = u2f(p[i]); acc += a[i] + b[i] + q.x + q.y; }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    if (threadIdx.x == 0 && blockIdx.x == 0) *clk = t1 - t0;
}

template <int MODE>
void run(const char *name, double lane_ops_per_step, int blocks_per_sm)
{
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int threads = blocks_per_sm == 1 ? 1024 : 256, blocks = sms * blocks_per_sm;
    float *out;
    long long *clk;
    cudaMalloc(&out, sizeof(float) * threads * blocks);
    cudaMalloc(&clk, sizeof(long long));
    k<MODE><<<blocks, threads>>>(out, 1e-3f, clk);
    cudaDeviceSynchronize();
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k<MODE><<<blocks, threads>>>(out, 1e-3f, clk);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    long long c = 0;
    cudaMemcpy(&c, clk, sizeof c, cudaMemcpyDeviceToHost);
    int khz = 0;
    cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, 0);
    const double cycles = ms * 1e-3 * khz * 1e3;
    // per SM per clock over the whole kernel (events, max clock)
    const double per_clk = (double)threads * blocks_per_sm * ITERS * CH * lane_ops_per_step / cycles;
    printf("%-34s %.3f ms, block0 %lld cyc -> %.1f per clk per SM (%s)\n", name, ms, c, per_clk, cudaGetErrorString(cudaGetLastError()));
    cudaFree(out);
    cudaFree(clk);
}

int main()
{
    run<0>("FFMA (lane-ops)", 2, 4);
    run<0>("FFMA (lane-ops) 1x1024", 2, 1);
    run<1>("FFMA2 (lane-ops, x2)", 2, 4);
    run<1>("FFMA2 (instr)", 1, 4);
    run<2>("MUFU sin+cos (lane-ops)", 2, 4);
    run<3>("2 MUFU + 2 FFMA2 (steps)", 1, 4);
    run<4>("2 MUFU + 3 FFMA +1 FADD (steps)", 1, 4);
    return 0;
}
