// Hardware probe: global atomic throughput (f64, f32, v4.f32), gather bandwidth, device props.
#include <cstdio>
#include <cuda_runtime.h>
#include <cstdint>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); return 1;}}while(0)
__global__ void red_f64(double* g, const uint32_t* idx, int n, int G){
  int i = blockIdx.x*blockDim.x+threadIdx.x; if(i>=n) return;
  uint32_t b = idx[i] % G;
  #pragma unroll
  for(int k=0;k<27;k++) atomicAdd(&g[(b*27+k)%(G*27)], 1.0);
}
__global__ void red_f32(float* g, const uint32_t* idx, int n, int G){
  int i = blockIdx.x*blockDim.x+threadIdx.x; if(i>=n) return;
  uint32_t b = idx[i] % G;
  #pragma unroll
  for(int k=0;k<27;k++) atomicAdd(&g[(b*27+k)%(G*27)], 1.0f);
}
__global__ void red_v4(float4* g, const uint32_t* idx, int n, int G){
  int i = blockIdx.x*blockDim.x+threadIdx.x; if(i>=n) return;
  uint32_t b = idx[i] % G;
  #pragma unroll
  for(int k=0;k<9;k++) atomicAdd(&g[(b*9+k)%(G*9)], make_float4(1.f,1.f,1.f,0.f));
}
__global__ void red_u64(unsigned long long* g, const uint32_t* idx, int n, int G){
  int i = blockIdx.x*blockDim.x+threadIdx.x; if(i>=n) return;
  uint32_t b = idx[i] % G;
  #pragma unroll
  for(int k=0;k<27;k++) atomicAdd(&g[(b*27+k)%(G*27)], 1ull);
}
__global__ void smem_f32(float* out, int n){
  __shared__ float s[4096];
  for(int i=threadIdx.x;i<4096;i+=blockDim.x) s[i]=0;
  __syncthreads();
  uint32_t h = blockIdx.x*7919u + threadIdx.x*104729u;
  for(int k=0;k<256;k++){ h = h*1664525u+1013904223u; atomicAdd(&s[(h>>8)&4095], 1.0f);}
  __syncthreads();
  if(threadIdx.x==0) out[blockIdx.x]=s[5];
}
__global__ void smem_f64(double* out, int n){
  __shared__ double s[4096];
  for(int i=threadIdx.x;i<4096;i+=blockDim.x) s[i]=0;
  __syncthreads();
  uint32_t h = blockIdx.x*7919u + threadIdx.x*104729u;
  for(int k=0;k<256;k++){ h = h*1664525u+1013904223u; atomicAdd(&s[(h>>8)&4095], 1.0);}
  __syncthreads();
  if(threadIdx.x==0) out[blockIdx.x]=s[5];
}
__global__ void gather2(const float2* __restrict__ y, const int* __restrict__ col, float* out, long n){
  long i = blockIdx.x*(long)blockDim.x+threadIdx.x; if(i>=n) return;
  float2 v = y[col[i]]; out[i] = v.x+v.y;
}
__global__ void init_idx(uint32_t* idx, int n, uint32_t seed){
  int i = blockIdx.x*blockDim.x+threadIdx.x; if(i>=n) return;
  uint32_t h = (i+1)*2654435761u ^ seed; h ^= h>>15; h*=2246822519u; h^=h>>13; idx[i]=h;
}
__global__ void init_col(int* c, long n, int N, int mode){
  long i = blockIdx.x*(long)blockDim.x+threadIdx.x; if(i>=n) return;
  uint32_t h = (uint32_t)(i+1)*2654435761u; h ^= h>>15; h*=2246822519u; h^=h>>13;
  if(mode==0) c[i] = h % N; else { long row = i/137; c[i] = (int)((row + (long)(h%4096) - 2048 + N) % N); }
}
__global__ void stream_rd(const int4* __restrict__ a, int4* out, long n){
  long i = blockIdx.x*(long)blockDim.x+threadIdx.x; long st = (long)gridDim.x*blockDim.x;
  int4 acc = make_int4(0,0,0,0);
  for(; i<n; i+=st){ int4 v = a[i]; acc.x^=v.x; acc.y^=v.y; acc.z^=v.z; acc.w^=v.w;}
  if(acc.x==12345) out[0]=acc;
}
int main(){
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p,0));
  printf("name=%s SMs=%d L2=%d MB smem/block optin=%zu KB, smem/SM=%zu KB, clock=%d kHz memclk=%d kHz bus=%d\n", p.name, p.multiProcessorCount, p.l2CacheSize>>20, p.sharedMemPerBlockOptin>>10, p.sharedMemPerMultiprocessor>>10, p.clockRate, p.memoryClockRate, p.memoryBusWidth);
  int n = 1300000; int Gs[3] = {4, 8100, 90000};
  uint32_t* idx; CK(cudaMalloc(&idx, n*4)); init_idx<<<(n+255)/256,256>>>(idx,n,123);
  double* g64; float* g32; float4* g4; unsigned long long* gu;
  CK(cudaMalloc(&g64, 90000*27*8)); CK(cudaMalloc(&g32, 90000*27*4)); CK(cudaMalloc(&g4, 90000*9*16)); CK(cudaMalloc(&gu, 90000*27*8));
  cudaEvent_t a,b; cudaEventCreate(&a); cudaEventCreate(&b); float ms;
  for(int gi=0; gi<3; gi++){ int G=Gs[gi];
    for(int rep=0;rep<3;rep++){
    cudaEventRecord(a); red_f64<<<(n+255)/256,256>>>(g64,idx,n,G); cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms,a,b);
    if(rep==2) printf("G=%d boxes: red f64 x27/pt: %.1f us\n", G, ms*1e3);
    cudaEventRecord(a); red_f32<<<(n+255)/256,256>>>(g32,idx,n,G); cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms,a,b);
    if(rep==2) printf("G=%d boxes: red f32 x27/pt: %.1f us\n", G, ms*1e3);
    cudaEventRecord(a); red_v4<<<(n+255)/256,256>>>(g4,idx,n,G); cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms,a,b);
    if(rep==2) printf("G=%d boxes: red v4f32 x9/pt: %.1f us\n", G, ms*1e3);
    cudaEventRecord(a); red_u64<<<(n+255)/256,256>>>(gu,idx,n,G); cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms,a,b);
    if(rep==2) printf("G=%d boxes: red u64 x27/pt: %.1f us\n", G, ms*1e3);
    }
  }
  float* o; CK(cudaMalloc(&o, 1<<20)); double* od; CK(cudaMalloc(&od, 1<<20));
  for(int rep=0;rep<3;rep++){
  cudaEventRecord(a); smem_f32<<<148*8,256>>>(o,0); cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms,a,b);
  if(rep==2) printf("smem f32 atomics: %.2f Gop/s\n", 148.0*8*256*256/(ms*1e-3)/1e9);
  cudaEventRecord(a); smem_f64<<<148*8,256>>>(od,0); cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms,a,b);
  if(rep==2) printf("smem f64 atomics: %.2f Gop/s\n", 148.0*8*256*256/(ms*1e-3)/1e9);
  }
  long nnz = 178000000L; int N=1300000; int* col; float2* y; float* out;
  CK(cudaMalloc(&col, nnz*4)); CK(cudaMalloc(&y, N*8)); CK(cudaMalloc(&out, nnz*4));
  for(int mode=0;mode<2;mode++){
    init_col<<<(nnz+255)/256,256>>>(col,nnz,N,mode);
    for(int rep=0;rep<3;rep++){
      cudaEventRecord(a); gather2<<<(nnz+255)/256,256>>>(y,col,out,nnz); cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms,a,b);
      if(rep==2) printf("gather mode=%d (0 random,1 local +-2048): %.1f us, col+out stream %.0f GB/s\n", mode, ms*1e3, nnz*8.0/(ms*1e-3)/1e9);
    }
  }
  for(int rep=0;rep<3;rep++){
    cudaEventRecord(a); stream_rd<<<148*16,512>>>((const int4*)col,(int4*)out,nnz/4); cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms,a,b);
    if(rep==2) printf("stream read %.2f GB: %.1f us = %.0f GB/s\n", nnz*4/1e9, ms*1e3, nnz*4.0/(ms*1e-3)/1e9);
  }
  CK(cudaDeviceSynchronize());
  return 0;
}
