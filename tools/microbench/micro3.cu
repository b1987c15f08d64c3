// Pipe-throughput microbenchmarks for the round-2 pass design on sm_100a:
// FFMA vs packed FFMA2, conversions (F2I / I2F / FRND) vs the magic-number
// equivalents, FMNMX, and int32 shared ATOMS with the rotated-entry pattern
// of the line tables.  Each kernel runs 148 x 4 CTAs of 512 threads; the
// reported figure is warp-instructions per clock per SM.
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s @%d\n",cudaGetErrorString(e),__LINE__); exit(1);}}while(0)

constexpr int ITERS = 4096;

__global__ void k_ffma(float *out, float a, float b) {
    float x[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = threadIdx.x + i;
    for (int it = 0; it < ITERS; ++it)
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = fmaf(x[i], a, b);
    float s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += x[i];
    if (s == 1.2345f) out[0] = s;
}
__global__ void k_ffma2(float *out, float a, float b) {
    float2 x[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = make_float2(threadIdx.x + i, i);
    const float2 A = make_float2(a, a), B = make_float2(b, b);
    for (int it = 0; it < ITERS; ++it)
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = __ffma2_rn(x[i], A, B);
    float s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += x[i].x + x[i].y;
    if (s == 1.2345f) out[0] = s;
}
// FFMA and IADD interleaved (dual pipe)
__global__ void k_ffma_iadd(float *out, float a, float b) {
    float x[8];
    int y[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) { x[i] = threadIdx.x + i; y[i] = threadIdx.x * i; }
    for (int it = 0; it < ITERS; ++it)
#pragma unroll
        for (int i = 0; i < 8; ++i) { x[i] = fmaf(x[i], a, b); y[i] = (y[i] ^ it) + 7; }
    float s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += x[i] + y[i];
    if (s == 1.2345f) out[0] = s;
}
__global__ void k_f2i(float *out, float a, float b) {
    float x[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = threadIdx.x + i;
    for (int it = 0; it < ITERS; ++it)
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = (float)(int)(x[i] * a) ;
    float s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += x[i];
    if (s == 1.2345f) out[0] = s;
}
__global__ void k_frnd(float *out, float a, float b) {
    float x[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = threadIdx.x + i;
    for (int it = 0; it < ITERS; ++it)
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = floorf(x[i]) + b;
    float s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += x[i];
    if (s == 1.2345f) out[0] = s;
}
// magic-number floor: FADD.RM + FADD
__global__ void k_magic(float *out, float a, float b) {
    float x[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = threadIdx.x + i;
    for (int it = 0; it < ITERS; ++it)
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = (__fadd_rd(x[i], 12582912.f) - 12582912.f) + b;
    float s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += x[i];
    if (s == 1.2345f) out[0] = s;
}
__global__ void k_fmnmx(float *out, float a, float b) {
    float x[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = threadIdx.x + i;
    for (int it = 0; it < ITERS; ++it)
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = fminf(fmaxf(x[i], a), b);
    float s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += x[i];
    if (s == 1.2345f) out[0] = s;
}
// int32 shared atomics: MODE 0 lane-distinct banks; 1: 8 lanes per address group with
// rotated entries (the line-table pattern: 4 slots x 8 entries per instruction); 2: all
// lanes one address; 3: random over 41 slots x 9 words
template <int MODE>
__global__ void k_atoms(int *out) {
    __shared__ int t[16 * 41 * 9];
    for (int i = threadIdx.x; i < 16 * 41 * 9; i += blockDim.x) t[i] = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int *tw = t + warp * 41 * 9;
    unsigned h = lane * 2654435761u + warp;
    for (int it = 0; it < ITERS / 8; ++it) {
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            int a;
            if (MODE == 0) a = lane;
            else if (MODE == 1) a = ((lane >> 3) + 4 * (it & 7)) * 9 + ((lane + e) & 7);
            else if (MODE == 2) a = 0;
            else { h = h * 1664525u + 1013904223u; a = ((h >> 16) % 41) * 9 + e; }
            atomicAdd(tw + a, it);
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) out[blockIdx.x] = t[7];
}

template <typename K>
static void run(const char *name, K kern, int instr_per_iter, int nsm) {
    float *o;
    CK(cudaMalloc(&o, 4096));
    const int grid = nsm * 4, block = 512;
    kern<<<grid, block>>>(o, 1.0001f, 0.5f);
    CK(cudaDeviceSynchronize());
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    kern<<<grid, block>>>(o, 1.0001f, 0.5f);
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    int clk;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const double warps = (double)grid * block / 32;
    const double winst = warps * ITERS * instr_per_iter;
    const double cyc = ms * 1e-3 * clk * 1e3;   // at max clock
    printf("%-12s %8.3f ms  %6.3f warp-inst/clk/SM (at %d MHz nominal)\n", name, ms, winst / cyc / nsm, clk / 1000);
    cudaFree(o);
}
template <int MODE>
static void run_atoms(const char *name, int nsm) {
    int *o;
    CK(cudaMalloc(&o, 4096 * 4));
    const int grid = nsm * 2, block = 512;
    k_atoms<MODE><<<grid, block>>>(o);
    CK(cudaDeviceSynchronize());
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    k_atoms<MODE><<<grid, block>>>(o);
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    int clk;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const double lanes = (double)grid * block * ITERS;
    printf("%-12s %8.3f ms  %6.2f lane-ops/clk/SM\n", name, ms, lanes / (ms * 1e-3 * clk * 1e3) / nsm);
    cudaFree(o);
}

int main() {
    int nsm;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    run("ffma", k_ffma, 8, nsm);
    run("ffma2", k_ffma2, 8, nsm);
    run("ffma+iadd", k_ffma_iadd, 16, nsm);
    run("f2i+i2f+fmul", k_f2i, 24, nsm);
    run("frnd+fadd", k_frnd, 16, nsm);
    run("magic floor", k_magic, 24, nsm);
    run("fmnmx x2", k_fmnmx, 16, nsm);
    run_atoms<0>("atoms lane", nsm);
    run_atoms<1>("atoms rot8", nsm);
    run_atoms<2>("atoms same", nsm);
    run_atoms<3>("atoms rand", nsm);
    return 0;
}
