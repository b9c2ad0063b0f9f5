// ubench_mix.cu -- does MUFU sin/cos overlap with packed FMA work?  Per step: one __sincosf
// plus K independent FFMA2; reports steps/clk/SM (MUFU ceiling 8) and FMA lane-ops/clk/SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2408_09066_b200/csrc -Iinclude -o tools/ubench_mix tools/ubench_mix.cu
#include <cstdio>
#include "common.cuh"

#define ITERS 2048
#define CH 8

template <int K>
__global__ void __launch_bounds__(256) k(float *out, float seed)
{
    float a[CH], acc[CH];
    f32x2 f[CH];
    for (int i = 0; i < CH; ++i) {
        a[i] = seed * (threadIdx.x + 3 * i);
        acc[i] = 0.f;
        f[i] = pk2(a[i], a[i] + 1.f);
    }
    const f32x2 m = pk2(0.999f, 0.998f), c = pk2(1e-3f, 2e-3f);
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < CH; ++i) {
            a[i] += 0.37f;
            float s, co;
            __sincosf(a[i], &s, &co);
            acc[i] += s + co;
#pragma unroll
            for (int q = 0; q < K; ++q) f[i] = fma2(f[i], m, c);
        }
    }
    float r = 0.f;
    for (int i = 0; i < CH; ++i) { float u, v; upk2(f[i], u, v); r += acc[i] + u + v; }
    out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}

template <int K>
void run(int bps)
{
    int sms = 0, khz = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, 0);
    const int threads = 256, blocks = sms * bps;
    float *out;
    cudaMalloc(&out, sizeof(float) * threads * blocks);
    k<K><<<blocks, threads>>>(out, 1e-3f);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k<K><<<blocks, threads>>>(out, 1e-3f);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    const double steps = (double)CH * ITERS * threads * blocks / (ms * 1e-3 * khz * 1e3) / sms;
    // FMA-pipe lane-ops per step: 2K (FFMA2) + 1 (FMUL.RZ) + 2 (FADD) + 1 (angle add)
    printf("K=%2d FFMA2/sincos  %d blk/SM  %.2f steps/clk/SM  %.1f FMA lane-ops/clk/SM\n", K, bps, steps,
           steps * (2 * K + 4));
    cudaFree(out);
}

int main()
{
    run<0>(3); run<2>(3); run<4>(3); run<6>(3); run<8>(3); run<10>(3); run<12>(3); run<16>(3);
    return 0;
}
