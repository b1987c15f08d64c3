// Second microbenchmark set: warp-aggregation primitives (match/redux/shfl) and
// clean 3-D trilinear gathers (LDG vs smem), used to size the pass-1 histogram design.
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s @%d\n",cudaGetErrorString(e),__LINE__); exit(1);}}while(0)
__device__ __forceinline__ unsigned hash32(unsigned x){ x ^= x>>16; x*=0x7feb352dU; x^=x>>15; x*=0x846ca68bU; x^=x>>16; return x; }

// NB distinct keys per warp (1,4,8,32): match_any + 16 redux + leader ATOMS (int32 fixed-point)
template<int NB>
__global__ void k_match_redux(int iters, int* out){
  __shared__ int t[8][1024];
  for (int i=threadIdx.x;i<8*1024;i+=blockDim.x) (&t[0][0])[i]=0;
  __syncthreads();
  int lane=threadIdx.x&31, warp=threadIdx.x>>5;
  float w0=0.1f*lane, w1=0.2f, w2=0.3f, w3=0.4f;
  for (int it=0; it<iters; ++it){
    int key = (hash32(it*32 + (lane*NB>>5)) & 127);
    float v0 = 1.0f+it*1e-3f, v1=v0*0.5f, v2=v0*v0, v3=v2*0.5f;
    unsigned m = __match_any_sync(0xffffffffu, key);
    int leader = __ffs(m)-1;
    int* row = &t[warp][(key&31)*32];
    float ws[4]={w0,w1,w2,w3}, vs[4]={v0,v1,v2,v3};
    #pragma unroll
    for (int l=0;l<4;++l)
      #pragma unroll
      for (int v=0; v<4; ++v){
        int q = __float2int_rn(ws[l]*vs[v]*4096.f);
        int s = __reduce_add_sync(m, q);
        if (lane==leader) atomicAdd(&row[l*4+v], s);
      }
  }
  __syncthreads();
  if (threadIdx.x==0) out[blockIdx.x]=t[0][5];
}
// baseline: 16 direct int atomics per lane, NB distinct keys per warp
template<int NB>
__global__ void k_direct16(int iters, int* out){
  __shared__ int t[8][1024];
  for (int i=threadIdx.x;i<8*1024;i+=blockDim.x) (&t[0][0])[i]=0;
  __syncthreads();
  int lane=threadIdx.x&31, warp=threadIdx.x>>5;
  float w0=0.1f*lane, w1=0.2f, w2=0.3f, w3=0.4f;
  for (int it=0; it<iters; ++it){
    int key = (hash32(it*32 + (lane*NB>>5)) & 127);
    float v0 = 1.0f+it*1e-3f, v1=v0*0.5f, v2=v0*v0, v3=v2*0.5f;
    int* row = &t[warp][(key&31)*32];
    float ws[4]={w0,w1,w2,w3}, vs[4]={v0,v1,v2,v3};
    #pragma unroll
    for (int l=0;l<4;++l)
      #pragma unroll
      for (int v=0; v<4; ++v) atomicAdd(&row[l*4+v], __float2int_rn(ws[l]*vs[v]*4096.f));
  }
  __syncthreads();
  if (threadIdx.x==0) out[blockIdx.x]=t[0][5];
}
// 3-D trilinear gather, tile 32x8 threads marching z, smooth displacement (amp voxels)
__global__ void k_tri_ldg(const float* __restrict__ M, int nx, int ny, int nz, int tz, float amp, float* out){
  int x = blockIdx.x*32 + (threadIdx.x&31), y = blockIdx.y*8 + (threadIdx.x>>5); int z0 = blockIdx.z*tz;
  float s=0; size_t sxy=(size_t)nx*ny;
  float ux = amp*__sinf(0.05f*y), uy=amp*__sinf(0.04f*x);
  for (int z=z0; z<z0+tz; ++z){
    float uz = amp*__sinf(0.03f*x+0.05f*y+0.07f*z);
    float fx=floorf(ux), fy=floorf(uy), fz=floorf(uz);
    int cx=min(max(x+(int)fx,0),nx-2), cy=min(max(y+(int)fy,0),ny-2), cz=min(max(z+(int)fz,0),nz-2);
    float tx=ux-fx, ty=uy-fy, tzz=uz-fz;
    const float* b=M+((size_t)cz*ny+cy)*nx+cx;
    float c00=b[0]+tx*(b[1]-b[0]), c10=b[nx]+tx*(b[nx+1]-b[nx]);
    float c01=b[sxy]+tx*(b[sxy+1]-b[sxy]), c11=b[sxy+nx]+tx*(b[sxy+nx+1]-b[sxy+nx]);
    float c0=c00+ty*(c10-c00), c1=c01+ty*(c11-c01);
    s += c0+tzz*(c1-c0);
  }
  if (s==12345.f) out[0]=s;
}
// streaming 8B/voxel read (F + M) with the same tiling, no gather
__global__ void k_two_stream(const float* __restrict__ F, const float* __restrict__ M, int nx, int ny, int nz, int tz, float* out){
  int x = blockIdx.x*32 + (threadIdx.x&31), y = blockIdx.y*8 + (threadIdx.x>>5); int z0 = blockIdx.z*tz;
  float s=0; size_t sxy=(size_t)nx*ny;
  for (int z=z0; z<z0+tz; ++z){ size_t i=z*sxy+(size_t)y*nx+x; s += __ldg(F+i)*__ldg(M+i); }
  if (s==12345.f) out[0]=s;
}
__global__ void k_shfl(int iters, float* out){
  float v=threadIdx.x; int lane=threadIdx.x&31;
  for (int it=0; it<iters; ++it){ v += __shfl_sync(0xffffffffu, v, (lane+it)&31); }
  if (v==12345.f) out[0]=v;
}
int main(){
  int nsm=148;
  int* oi; float* of; CK(cudaMalloc(&oi, 1<<20)); CK(cudaMalloc(&of, 1<<20));
  cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1); float ms;
  int iters=2048, blocks=nsm*4, threads=256;
  double lines=(double)blocks*8*iters; // warp-iterations (32 voxels each)
#define RUN(name, launch, denom, unit) { launch; CK(cudaDeviceSynchronize()); cudaEventRecord(e0); launch; cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms,e0,e1); \
   printf("%-30s %8.3f ms  %8.3f clk/SM per %s (at 1.9GHz)\n", name, ms, (ms*1e-3)*1.9e9*nsm/(denom), unit); }
  RUN("match+redux16 NB=1", (k_match_redux<1><<<blocks,threads>>>(iters,oi)), lines*32, "voxel");
  RUN("match+redux16 NB=4", (k_match_redux<4><<<blocks,threads>>>(iters,oi)), lines*32, "voxel");
  RUN("match+redux16 NB=8", (k_match_redux<8><<<blocks,threads>>>(iters,oi)), lines*32, "voxel");
  RUN("match+redux16 NB=32", (k_match_redux<32><<<blocks,threads>>>(iters,oi)), lines*32, "voxel");
  RUN("direct16 NB=1", (k_direct16<1><<<blocks,threads>>>(iters,oi)), lines*32, "voxel");
  RUN("direct16 NB=4", (k_direct16<4><<<blocks,threads>>>(iters,oi)), lines*32, "voxel");
  RUN("direct16 NB=8", (k_direct16<8><<<blocks,threads>>>(iters,oi)), lines*32, "voxel");
  RUN("direct16 NB=32", (k_direct16<32><<<blocks,threads>>>(iters,oi)), lines*32, "voxel");
  RUN("shfl", (k_shfl<<<blocks,threads>>>(iters*8,of)), lines*8, "warp-shfl");
  int nx=512, ny=512, nz=320; size_t n=(size_t)nx*ny*nz; float *F,*M; CK(cudaMalloc(&F,n*4)); CK(cudaMalloc(&M,n*4)); cudaMemset(F,0,n*4); cudaMemset(M,0,n*4);
  for (int tz : {8, 40}) for (float amp : {0.0f, 2.0f, 15.0f}){
    dim3 g(nx/32, ny/8, nz/tz);
    for (int r=0;r<2;++r){ k_tri_ldg<<<g,256>>>(M,nx,ny,nz,tz,amp,of);} CK(cudaDeviceSynchronize());
    cudaEventRecord(e0); k_tri_ldg<<<g,256>>>(M,nx,ny,nz,tz,amp,of); cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms,e0,e1);
    printf("tri_ldg tz=%d amp=%4.1f: %.3f ms  %.1f Gvox/s  (x8B=%.0f GB/s)\n", tz, amp, ms, n/ms/1e6, n*8/ms/1e6);
  }
  for (int tz : {8, 40}) { dim3 g(nx/32, ny/8, nz/tz);
    k_two_stream<<<g,256>>>(F,M,nx,ny,nz,tz,of); CK(cudaDeviceSynchronize());
    cudaEventRecord(e0); k_two_stream<<<g,256>>>(F,M,nx,ny,nz,tz,of); cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms,e0,e1);
    printf("two_stream tz=%d: %.3f ms  %.1f GB/s\n", tz, ms, n*8/ms/1e6); }
  return 0;
}
