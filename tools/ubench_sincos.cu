// ubench_sincos.cu -- throughput of the encode's phasor evaluators in isolation:
// MUFU __sincosf, scalar sincos_fma, packed sincos_fma2 -- phasors per clock per SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2408_09066_b200/csrc -Iinclude -o tools/ubench_sincos tools/ubench_sincos.cu
#include <cstdio>
#include "common.cuh"

#define ITERS 2048
#define CH 8   // independent phasor pairs per thread

template <int MODE>
__global__ void __launch_bounds__(256) k(float *out, float seed)
{
    f32x2 ph[CH], acc[CH];
    for (int i = 0; i < CH; ++i) {
        ph[i] = pk2(seed * (threadIdx.x + 3 * i), seed * (threadIdx.x + 3 * i + 1));
        acc[i] = pk2(0.f, 0.f);
    }
    const f32x2 step = pk2(0.37f, 0.41f);
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < CH; ++i) {
            ph[i] = add2(ph[i], step);
            if (MODE == 0) {   // MUFU, two phasors
                float a, b, sa, ca, sb, cb;
                upk2(ph[i], a, b);
                __sincosf(a, &sa, &ca);
                __sincosf(b, &sb, &cb);
                acc[i] = add2(acc[i], pk2(ca + sb, sa + cb));
            } else if (MODE == 1) {   // scalar polynomial, two phasors
                float a, b, sa, ca, sb, cb;
                upk2(ph[i], a, b);
                sincos_fma(a, &sa, &ca);
                sincos_fma(b, &sb, &cb);
                acc[i] = add2(acc[i], pk2(ca + sb, sa + cb));
            } else {   // packed polynomial, two phasors
                f32x2 S, C;
                sincos_fma2(ph[i], S, C);
                acc[i] = add2(acc[i], add2(S, C));
            }
        }
    }
    float r = 0.f;
    for (int i = 0; i < CH; ++i) { float a, b; upk2(acc[i], a, b); r += a + b; }
    out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}

template <int MODE>
void run(const char *name, int bps)
{
    int sms = 0, khz = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, 0);
    const int threads = 256, blocks = sms * bps;
    float *out;
    cudaMalloc(&out, sizeof(float) * threads * blocks);
    k<MODE><<<blocks, threads>>>(out, 1e-3f);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k<MODE><<<blocks, threads>>>(out, 1e-3f);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    const double phasors = 2.0 * CH * ITERS * threads * (double)blocks;
    printf("%-22s %d blk/SM  %.3f ms  %.2f phasors/clk/SM (%s)\n", name, bps, ms,
           phasors / (ms * 1e-3 * khz * 1e3) / sms, cudaGetErrorString(cudaGetLastError()));
    cudaFree(out);
}

int main()
{
    for (int b : {2, 3, 4}) {
        run<0>("MUFU __sincosf", b);
        run<1>("scalar sincos_fma", b);
        run<2>("packed sincos_fma2", b);
    }
    return 0;
}
