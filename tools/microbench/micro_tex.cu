// Gather microbenchmark for the warped sample of M (pass 1): per voxel the 8 corners of
// the trilinear cell, (a) 8 scalar LDG (the current passes) vs (b) 2 TLD4 (textureGather
// of a 2-D layered texture, layer = z: one 2x2 footprint per z-layer).  Access pattern as
// in pass 1 (C5 512 x 512 x 320): a warp marches z along one row; lane = x; the sample
// point is the voxel plus a smooth displacement of a few voxels.  Reports ms per pass over
// the volume and checks that both read identical corner values.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s @%d\n",cudaGetErrorString(e),__LINE__); exit(1);}}while(0)

constexpr int NX = 512, NY = 512, NZ = 320;

__device__ __forceinline__ void disp(int x, int y, int z, float &ux, float &uy, float &uz) {
    ux = 2.5f * __sinf(0.031f * y + 0.017f * z) + 0.37f;
    uy = 2.0f * __sinf(0.023f * x + 0.029f * z) - 0.21f;
    uz = 1.5f * __sinf(0.019f * x + 0.027f * y) + 0.13f;
}

__device__ __forceinline__ void cellof(int x, int y, int z, int &cx, int &cy, int &cz, float &tx, float &ty, float &tz) {
    float ux, uy, uz;
    disp(x, y, z, ux, uy, uz);
    const float px = x + ux, py = y + uy, pz = z + uz;
    cx = min(max((int)floorf(px), 0), NX - 2);
    cy = min(max((int)floorf(py), 0), NY - 2);
    cz = min(max((int)floorf(pz), 0), NZ - 2);
    tx = px - floorf(px); ty = py - floorf(py); tz = pz - floorf(pz);
}

__device__ __forceinline__ float tri(const float c[8], float tx, float ty, float tz) {
    const float e00 = fmaf(tx, c[1] - c[0], c[0]), e10 = fmaf(tx, c[3] - c[2], c[2]);
    const float e01 = fmaf(tx, c[5] - c[4], c[4]), e11 = fmaf(tx, c[7] - c[6], c[6]);
    const float f0 = fmaf(ty, e10 - e00, e00), f1 = fmaf(ty, e11 - e01, e01);
    return fmaf(tz, f1 - f0, f0);
}

// one warp per (y) row, marching z; grid-stride over rows
__global__ void __launch_bounds__(512) k_ldg(const float *__restrict__ M, float *out) {
    const int lane = threadIdx.x & 31;
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
    float acc = 0.f;
    for (int row = warp; row < NY * (NX / 32); row += nw) {
        const int y = row / (NX / 32), x = (row % (NX / 32)) * 32 + lane;
        for (int z = 0; z < NZ; ++z) {
            int cx, cy, cz;
            float tx, ty, tz;
            cellof(x, y, z, cx, cy, cz, tx, ty, tz);
            const int o = (cz * NY + cy) * NX + cx;
            float c[8];
            c[0] = __ldg(M + o); c[1] = __ldg(M + o + 1);
            c[2] = __ldg(M + o + NX); c[3] = __ldg(M + o + NX + 1);
            c[4] = __ldg(M + o + NX * NY); c[5] = __ldg(M + o + NX * NY + 1);
            c[6] = __ldg(M + o + NX * NY + NX); c[7] = __ldg(M + o + NX * NY + NX + 1);
            acc += tri(c, tx, ty, tz);
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

__device__ __forceinline__ float4 gather4(cudaTextureObject_t t, int layer, float x, float y) {
    float4 r;
    asm volatile("tld4.r.a2d.v4.f32.f32 {%0, %1, %2, %3}, [%4, {%5, %6, %7, %7}];"
                 : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
                 : "l"(t), "r"(layer), "f"(x), "f"(y));
    return r;
}

// corners from the 2x2 footprint centred on the cell's (x+1, y+1) texel corner: the
// footprint is texels (cx, cy) .. (cx+1, cy+1) exactly (integer + 1 coordinates)
template <int ORDER>
__device__ __forceinline__ void corners_tex(cudaTextureObject_t t, int cx, int cy, int cz, float c[8]) {
    const float fx = (float)(cx + 1), fy = (float)(cy + 1);
    const float4 a = gather4(t, cz, fx, fy), b = gather4(t, cz + 1, fx, fy);
    // textureGather order: (x0,y1), (x1,y1), (x1,y0), (x0,y0)
    c[0] = a.w; c[1] = a.z; c[2] = a.x; c[3] = a.y;
    c[4] = b.w; c[5] = b.z; c[6] = b.x; c[7] = b.y;
}

__global__ void __launch_bounds__(512) k_tex(cudaTextureObject_t t, float *out) {
    const int lane = threadIdx.x & 31;
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
    float acc = 0.f;
    for (int row = warp; row < NY * (NX / 32); row += nw) {
        const int y = row / (NX / 32), x = (row % (NX / 32)) * 32 + lane;
        for (int z = 0; z < NZ; ++z) {
            int cx, cy, cz;
            float tx, ty, tz;
            cellof(x, y, z, cx, cy, cz, tx, ty, tz);
            float c[8];
            corners_tex<0>(t, cx, cy, cz, c);
            acc += tri(c, tx, ty, tz);
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

// correctness: both corner sets for a sample of voxels
__global__ void k_check(const float *M, cudaTextureObject_t t, int *bad) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int x = i % NX, y = (i / NX) % NY, z = (i / (NX * NY)) * 7 % NZ;
    int cx, cy, cz;
    float tx, ty, tz;
    cellof(x, y, z, cx, cy, cz, tx, ty, tz);
    const int o = (cz * NY + cy) * NX + cx;
    const float r[8] = {M[o], M[o + 1], M[o + NX], M[o + NX + 1], M[o + NX * NY], M[o + NX * NY + 1],
                        M[o + NX * NY + NX], M[o + NX * NY + NX + 1]};
    float c[8];
    corners_tex<0>(t, cx, cy, cz, c);
    for (int k = 0; k < 8; ++k)
        if (c[k] != r[k]) atomicAdd(bad, 1);
}

int main() {
    const size_t n = (size_t)NX * NY * NZ;
    std::vector<float> h(n);
    unsigned s = 12345;
    for (size_t i = 0; i < n; ++i) { s = s * 1664525u + 1013904223u; h[i] = (s >> 8) * (1.0f / 16777216.f) * 127.f; }
    float *M, *out;
    CK(cudaMalloc(&M, n * 4));
    CK(cudaMemcpy(M, h.data(), n * 4, cudaMemcpyHostToDevice));
    CK(cudaMalloc(&out, 148 * 4 * 512 * 4));
    cudaArray_t arr;
    cudaChannelFormatDesc cd = cudaCreateChannelDesc<float>();
    CK(cudaMalloc3DArray(&arr, &cd, make_cudaExtent(NX, NY, NZ), cudaArrayLayered));
    cudaMemcpy3DParms p{};
    p.srcPtr = make_cudaPitchedPtr(h.data(), NX * 4, NX, NY);
    p.dstArray = arr;
    p.extent = make_cudaExtent(NX, NY, NZ);
    p.kind = cudaMemcpyHostToDevice;
    CK(cudaMemcpy3D(&p));
    cudaResourceDesc rd{};
    rd.resType = cudaResourceTypeArray;
    rd.res.array.array = arr;
    cudaTextureDesc td{};
    td.addressMode[0] = td.addressMode[1] = td.addressMode[2] = cudaAddressModeClamp;
    td.filterMode = cudaFilterModePoint;
    td.readMode = cudaReadModeElementType;
    td.normalizedCoords = 0;
    cudaTextureObject_t t;
    CK(cudaCreateTextureObject(&t, &rd, &td, nullptr));
    int *bad;
    CK(cudaMalloc(&bad, 4));
    CK(cudaMemset(bad, 0, 4));
    k_check<<<(NX * NY * 4) / 256, 256>>>(M, t, bad);
    int hb;
    CK(cudaMemcpy(&hb, bad, 4, cudaMemcpyDeviceToHost));
    printf("mismatching corners: %d of %d\n", hb, NX * NY * 4 * 8);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int occ = 1; occ <= 4; occ *= 2) {
        const int grid = 148 * occ, block = 512;
        for (int rep = 0; rep < 2; ++rep) {
            float ms1, ms2;
            cudaEventRecord(a);
            k_ldg<<<grid, block>>>(M, out);
            cudaEventRecord(b);
            CK(cudaEventSynchronize(b));
            cudaEventElapsedTime(&ms1, a, b);
            cudaEventRecord(a);
            k_tex<<<grid, block>>>(t, out);
            cudaEventRecord(b);
            CK(cudaEventSynchronize(b));
            cudaEventElapsedTime(&ms2, a, b);
            if (rep) printf("CTAs/SM %d (x512 threads): ldg %.3f ms   tex-gather %.3f ms\n", occ, ms1, ms2);
        }
    }
    CK(cudaGetLastError());
    return 0;
}
