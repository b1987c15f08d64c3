// Microbenchmarks that decide the histogram / gather design of the SRWCR passes
// on sm_100a: shared-memory atomic and RMW throughput, HBM streaming, gathers.
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s @%d\n",cudaGetErrorString(e),__LINE__); exit(1);}}while(0)

__device__ __forceinline__ unsigned hash32(unsigned x){ x ^= x>>16; x*=0x7feb352dU; x^=x>>15; x*=0x846ca68bU; x^=x>>16; return x; }

// mode 0: lane-distinct conflict-free (addr = warp*32*8 + (it&7)*32 + lane)
// mode 1: random in 8192-word table
// mode 2: all lanes of a warp same address
// mode 3: groups of 4 lanes share an address (8 distinct, distinct banks)
// mode 4: 16-way groups (2 distinct)
template<int MODE>
__device__ __forceinline__ int addr_of(int it, int lane, int warp){
  if (MODE==0) return (warp*8 + (it&7))*32 + lane;
  if (MODE==1) return hash32(it*1024 + warp*32 + lane) & 8191;
  if (MODE==2) return (warp*8 + (it&7))*32;
  if (MODE==3) return (warp*8 + (it&7))*32 + (lane>>2);
  return (warp*8 + (it&7))*32 + (lane>>4);
}

template<int MODE>
__global__ void k_atoms_i32(int iters, int* out){
  __shared__ int t[8192];
  for (int i=threadIdx.x;i<8192;i+=blockDim.x) t[i]=0;
  __syncthreads();
  int lane=threadIdx.x&31, warp=threadIdx.x>>5;
  for (int it=0; it<iters; ++it){ atomicAdd(&t[addr_of<MODE>(it,lane,warp)&8191], it|1); }
  __syncthreads();
  if (threadIdx.x==0) out[blockIdx.x]=t[5];
}
template<int MODE>
__global__ void k_atoms_f32(int iters, float* out){
  __shared__ float t[8192];
  for (int i=threadIdx.x;i<8192;i+=blockDim.x) t[i]=0;
  __syncthreads();
  int lane=threadIdx.x&31, warp=threadIdx.x>>5;
  for (int it=0; it<iters; ++it){ atomicAdd(&t[addr_of<MODE>(it,lane,warp)&8191], 1.0f); }
  __syncthreads();
  if (threadIdx.x==0) out[blockIdx.x]=t[5];
}
// lane-private plain RMW: t[(k)*32+lane] += v   (no atomics, conflict-free)
__global__ void k_rmw_f32(int iters, float* out){
  __shared__ float t[8192];
  for (int i=threadIdx.x;i<8192;i+=blockDim.x) t[i]=0;
  __syncthreads();
  int lane=threadIdx.x&31, warp=threadIdx.x>>5;
  float* base = t + warp*1024 + lane;
  for (int it=0; it<iters; ++it){ int k = hash32(it*64+warp) & 31; base[k*32] += 1.0f; }
  __syncthreads();
  if (threadIdx.x==0) out[blockIdx.x]=t[5];
}
// streaming read of n floats with float4, grid-stride
__global__ void k_stream(const float4* __restrict__ a, size_t n4, float* out){
  float s=0;
  for (size_t i=blockIdx.x*(size_t)blockDim.x+threadIdx.x; i<n4; i+=(size_t)gridDim.x*blockDim.x){ float4 v=__ldg(a+i); s+=v.x+v.y+v.z+v.w; }
  if (s==12345.f) out[0]=s;
}
// gather: per "voxel" 8 corner loads around (x+dx, y+dy, z+dz) with smooth small displacement
__global__ void k_gather8(const float* __restrict__ M, int nx, int ny, int nz, float* out, float amp){
  size_t nvox=(size_t)nx*ny*nz; float s=0;
  for (size_t i=blockIdx.x*(size_t)blockDim.x+threadIdx.x; i<nvox; i+=(size_t)gridDim.x*blockDim.x){
    int x=i%nx; int y=(i/nx)%ny; int z=i/((size_t)nx*ny);
    float ux = amp*__sinf(0.05f*y+0.03f*z), uy=amp*__sinf(0.04f*x+0.02f*z), uz=amp*__sinf(0.03f*x+0.05f*y);
    int cx=min(max(x+(int)floorf(ux),0),nx-2), cy=min(max(y+(int)floorf(uy),0),ny-2), cz=min(max(z+(int)floorf(uz),0),nz-2);
    size_t b=((size_t)cz*ny+cy)*nx+cx;
    s += __ldg(M+b)+__ldg(M+b+1)+__ldg(M+b+nx)+__ldg(M+b+nx+1)+__ldg(M+b+(size_t)nx*ny)+__ldg(M+b+(size_t)nx*ny+1)+__ldg(M+b+(size_t)nx*ny+nx)+__ldg(M+b+(size_t)nx*ny+nx+1);
  }
  if (s==12345.f) out[0]=s;
}

int main(){
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p,0));
  int clk=0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("dev %s SMs %d smemPerSM %zu smemOptin %zu L2 %d clock(kHz) %d\n", p.name, p.multiProcessorCount, p.sharedMemPerMultiprocessor, p.sharedMemPerBlockOptin, p.l2CacheSize, clk);
  int nsm=p.multiProcessorCount;
  int* oi; float* of; CK(cudaMalloc(&oi, 1<<20)); CK(cudaMalloc(&of, 1<<20));
  cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int iters=4096, blocks=nsm*4, threads=256; float ms;
  double ops=(double)blocks*threads*iters;
#define RUN(name, launch) { launch; CK(cudaDeviceSynchronize()); cudaEventRecord(e0); launch; cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms,e0,e1); \
   printf("%-28s %8.3f ms  %8.2f Glane-op/s  %6.3f lane-op/clk/SM (at 1.9GHz)\n", name, ms, ops/ms/1e6, ops/(ms*1e-3)/nsm/1.9e9); }
  RUN("atoms_i32 distinct", (k_atoms_i32<0><<<blocks,threads>>>(iters,oi)));
  RUN("atoms_i32 random8k", (k_atoms_i32<1><<<blocks,threads>>>(iters,oi)));
  RUN("atoms_i32 same-addr/warp", (k_atoms_i32<2><<<blocks,threads>>>(iters,oi)));
  RUN("atoms_i32 4-lane groups", (k_atoms_i32<3><<<blocks,threads>>>(iters,oi)));
  RUN("atoms_i32 16-lane groups", (k_atoms_i32<4><<<blocks,threads>>>(iters,oi)));
  RUN("atoms_f32 distinct", (k_atoms_f32<0><<<blocks,threads>>>(iters,of)));
  RUN("atoms_f32 random8k", (k_atoms_f32<1><<<blocks,threads>>>(iters,of)));
  RUN("atoms_f32 4-lane groups", (k_atoms_f32<3><<<blocks,threads>>>(iters,of)));
  RUN("rmw_f32 lane-private", (k_rmw_f32<<<blocks,threads>>>(iters,of)));
  size_t n = (size_t)1<<28; float* a; CK(cudaMalloc(&a, n*4)); CK(cudaMemset(a,0,n*4));
  for (int rep=0; rep<3; ++rep){
    k_stream<<<nsm*8,512>>>((const float4*)a, n/4, of); CK(cudaDeviceSynchronize());
    cudaEventRecord(e0); k_stream<<<nsm*8,512>>>((const float4*)a, n/4, of); cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms,e0,e1);
    printf("stream read 1GiB: %.3f ms  %.1f GB/s\n", ms, n*4/ms/1e6);
  }
  int nx=512, ny=512, nz=320; 
  for (float amp : {0.0f, 2.0f, 15.0f}){
    k_gather8<<<nsm*8,256>>>(a,nx,ny,nz,of,amp); CK(cudaDeviceSynchronize());
    cudaEventRecord(e0); k_gather8<<<nsm*8,256>>>(a,nx,ny,nz,of,amp); cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms,e0,e1);
    double vox=(double)nx*ny*nz;
    printf("gather8 amp %.0f: %.3f ms  %.1f Gvox/s  (%.1f GB/s at 4B/vox)\n", amp, ms, vox/ms/1e6, vox*4/ms/1e6);
  }
  return 0;
}
