// Day-1 microbenchmarks: ChaCha20 keystream rate, int ALU rate, copy GB/s.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s @%d\n",cudaGetErrorString(e),__LINE__);return 1;}}while(0)
__device__ __forceinline__ uint32_t rotl(uint32_t x, int n){ return __funnelshift_l(x,x,n); }
#define QR(a,b,c,d) a+=b; d^=a; d=rotl(d,16); c+=d; b^=c; b=rotl(b,12); a+=b; d^=a; d=rotl(d,8); c+=d; b^=c; b=rotl(b,7);
__device__ __forceinline__ void chacha_block(const uint32_t k[8], uint32_t ctr, uint32_t o[16]){
  uint32_t x0=0x61707865u,x1=0x3320646eu,x2=0x79622d32u,x3=0x6b206574u;
  uint32_t x4=k[0],x5=k[1],x6=k[2],x7=k[3],x8=k[4],x9=k[5],x10=k[6],x11=k[7];
  uint32_t x12=ctr,x13=0,x14=0,x15=0;
  #pragma unroll
  for(int i=0;i<10;i++){ QR(x0,x4,x8,x12) QR(x1,x5,x9,x13) QR(x2,x6,x10,x14) QR(x3,x7,x11,x15)
                         QR(x0,x5,x10,x15) QR(x1,x6,x11,x12) QR(x2,x7,x8,x13) QR(x3,x4,x9,x14) }
  o[0]=x0+0x61707865u;o[1]=x1+0x3320646eu;o[2]=x2+0x79622d32u;o[3]=x3+0x6b206574u;
  o[4]=x4+k[0];o[5]=x5+k[1];o[6]=x6+k[2];o[7]=x7+k[3];o[8]=x8+k[4];o[9]=x9+k[5];o[10]=x10+k[6];o[11]=x11+k[7];
  o[12]=x12+ctr;o[13]=x13;o[14]=x14;o[15]=x15;
}
__global__ void ks_reduce(uint32_t* out, int nblk, uint32_t seed){
  uint32_t k[8]; for(int i=0;i<8;i++) k[i]=seed*(i+1);
  uint32_t acc=0; uint32_t t=blockIdx.x*blockDim.x+threadIdx.x, T=gridDim.x*blockDim.x;
  for(int i=0;i<nblk;i++){ uint32_t o[16]; chacha_block(k,t+i*T,o);
    #pragma unroll
    for(int j=0;j<16;j++) acc^=o[j]; }
  out[t]=acc;
}
__global__ void ks_write(uint4* out, int nblk){
  uint32_t k[8]; for(int i=0;i<8;i++) k[i]=0x1234567u*(i+1);
  size_t t=blockIdx.x*(size_t)blockDim.x+threadIdx.x, T=(size_t)gridDim.x*blockDim.x;
  for(int i=0;i<nblk;i++){ uint32_t o[16]; size_t c=t+i*T; chacha_block(k,(uint32_t)c,o);
    uint4* p=out+c*4; p[0]=make_uint4(o[0],o[1],o[2],o[3]);p[1]=make_uint4(o[4],o[5],o[6],o[7]);
    p[2]=make_uint4(o[8],o[9],o[10],o[11]);p[3]=make_uint4(o[12],o[13],o[14],o[15]); }
}
__global__ void copyk(const uint4* __restrict__ a, uint4* __restrict__ b, size_t n){
  size_t t=blockIdx.x*(size_t)blockDim.x+threadIdx.x, T=(size_t)gridDim.x*blockDim.x;
  for(size_t i=t;i<n;i+=T) b[i]=a[i];
}
__global__ void alu_lop(uint32_t* out, int n){ uint32_t a=threadIdx.x,b=blockIdx.x,c=a^0x5555,d=b+7;
  for(int i=0;i<n;i++){ a=(a^b)|c; b=(b^c)&d; c=(c^d)|a; d=(d^a)&b; a=(a^b)|c; b=(b^c)&d; c=(c^d)|a; d=(d^a)&b;} out[blockIdx.x*blockDim.x+threadIdx.x]=a^b^c^d; }
int main(){
  int dev=0; cudaDeviceProp p; CK(cudaGetDeviceProperties(&p,dev));
  int l2; CK(cudaDeviceGetAttribute(&l2,cudaDevAttrL2CacheSize,dev));
  int clk; CK(cudaDeviceGetAttribute(&clk,cudaDevAttrClockRate,dev));
  printf("{\"name\":\"%s\",\"sms\":%d,\"l2_bytes\":%d,\"clock_khz\":%d,\"persist_max\":%d}\n",p.name,p.multiProcessorCount,l2,clk,p.persistingL2CacheMaxSize);
  cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1); float ms;
  uint32_t* out; CK(cudaMalloc(&out, 1<<26));
  int sms=p.multiProcessorCount;
  for(int bs: {128,256,512}) for(int per: {4,8}){
    int grid=sms*per*(1024/bs)/ (bs>=512?1:1); int nblk=64;
    ks_reduce<<<grid,bs>>>(out,4,1); cudaDeviceSynchronize();
    cudaEventRecord(e0); ks_reduce<<<grid,bs>>>(out,nblk,2); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms,e0,e1); double bytes=64.0*nblk*grid*bs;
    printf("{\"test\":\"chacha_reduce\",\"bs\":%d,\"grid\":%d,\"GBps\":%.1f}\n",bs,grid,bytes/ms/1e6);
  }
  uint4* ks; size_t ksb=(size_t)1<<30; CK(cudaMalloc(&ks,ksb));
  { int bs=256, grid=sms*8; int nblk=(int)(ksb/64/(grid*bs)); ks_write<<<grid,bs>>>(ks,nblk); cudaDeviceSynchronize();
    cudaEventRecord(e0); ks_write<<<grid,bs>>>(ks,nblk); cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms,e0,e1);
    printf("{\"test\":\"chacha_write\",\"GBps\":%.1f}\n",64.0*nblk*grid*bs/ms/1e6); }
  uint4* b2; CK(cudaMalloc(&b2,ksb));
  for(int per: {2,4,8}){ int bs=256, grid=sms*per; copyk<<<grid,bs>>>(ks,b2,ksb/16); cudaDeviceSynchronize();
    cudaEventRecord(e0); for(int r=0;r<5;r++) copyk<<<grid,bs>>>(ks,b2,ksb/16); cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms,e0,e1);
    printf("{\"test\":\"copy\",\"grid\":%d,\"GBps\":%.1f}\n",grid,5*2.0*ksb/ms/1e6); }
  { int bs=256, grid=sms*8, n=4096; alu_lop<<<grid,bs>>>(out,16); cudaDeviceSynchronize();
    cudaEventRecord(e0); alu_lop<<<grid,bs>>>(out,n); cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms,e0,e1);
    double ops=8.0*n*grid*bs; printf("{\"test\":\"alu_lop\",\"Gops\":%.1f,\"per_clk_sm_at_1965\":%.1f}\n",ops/ms/1e6, ops/ms/1e6/1.965/sms); }
  return 0;
}
