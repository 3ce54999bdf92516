// microbenchmark: per-SM throughput of MUFU.EX2, F2FP.BF16 pack, and their mix
#include <cstdio>
#include <cuda_bf16.h>
__device__ __forceinline__ float ex2(float x){float y;asm volatile("ex2.approx.ftz.f32 %0,%1;":"=f"(y):"f"(x));return y;}
__device__ __forceinline__ unsigned pk(float a,float b){unsigned r;asm volatile("cvt.rn.bf16x2.f32 %0,%1,%2;":"=r"(r):"f"(b),"f"(a));return r;}
__device__ __forceinline__ unsigned ex2h(unsigned x){unsigned y;asm volatile("ex2.approx.f16x2 %0,%1;":"=r"(y):"r"(x));return y;}
__device__ __forceinline__ unsigned long long f2(float a,float b){unsigned long long r;asm("mov.b64 %0,{%1,%2};":"=l"(r):"f"(a),"f"(b));return r;}
__device__ __forceinline__ void uf2(unsigned long long r,float&a,float&b){asm("mov.b64 {%0,%1},%2;":"=f"(a),"=f"(b):"l"(r));}
__device__ __forceinline__ unsigned long long fma2(unsigned long long a,unsigned long long b,unsigned long long c){unsigned long long d;asm("fma.rn.f32x2 %0,%1,%2,%3;":"=l"(d):"l"(a),"l"(b),"l"(c));return d;}
__device__ __forceinline__ unsigned long long add2(unsigned long long a,unsigned long long b){unsigned long long d;asm("add.rn.f32x2 %0,%1,%2;":"=l"(d):"l"(a),"l"(b));return d;}
__device__ __forceinline__ unsigned long long pexp2(unsigned long long x){
  const unsigned long long M=f2(12582912.f,12582912.f), NM=f2(-12582912.f,-12582912.f), NEG=f2(-1.f,-1.f);
  unsigned long long t=add2(x,M); unsigned long long r=add2(t,NM); unsigned long long f=fma2(r,NEG,x);
  unsigned long long p=fma2(f2(0.0545961f,0.0545961f),f,f2(0.2422184f,0.2422184f));
  p=fma2(p,f,f2(0.6933680f,0.6933680f)); p=fma2(p,f,f2(1.f,1.f));
  unsigned tl=(unsigned)t, th=(unsigned)(t>>32), pl=(unsigned)p, ph=(unsigned)(p>>32);
  return ((unsigned long long)((th<<23)+ph)<<32) | (unsigned)((tl<<23)+pl);
}
template<int MODE> __global__ void k(float* out, int iters){
  float v[8]; unsigned u[8];
  for(int i=0;i<8;i++){v[i]=-(threadIdx.x+i)*1e-3f; u[i]=0x3c003c00u+i;}
  for(int it=0;it<iters;it++){
#pragma unroll
    for(int i=0;i<8;i++){
      if(MODE==0) v[i]=ex2(v[i])-1.0f;
      if(MODE==1) u[i]^=pk(v[i],v[(i+1)&7]);
      if(MODE==2){ v[i]=ex2(v[i])-1.0f; if(i&1) u[i]^=pk(v[i],v[i-1]); }
      if(MODE==3) u[i]=ex2h(u[i]);
      if(MODE==4 && (i&1)){ unsigned long long x=f2(v[i-1],v[i]); x=pexp2(x); float a,b; uf2(x,a,b); v[i-1]=a-1.0f; v[i]=b-1.0f; }
      if(MODE==5 && (i&1)){ unsigned a=__float_as_uint(v[i-1])+0x8000u, b=__float_as_uint(v[i])+0x8000u; unsigned r; asm volatile("prmt.b32 %0,%1,%2,0x7632;":"=r"(r):"r"(a),"r"(b)); u[i]^=r; v[i]+=1.0f; }
    }
  }
  float s=0; for(int i=0;i<8;i++) s+=v[i]+u[i];
  if(s==123.f) out[0]=s;
}
template<int MODE> void run(const char* name, int threads){
  float* o; cudaMalloc(&o,4); int iters=4096; int blocks=148;
  k<MODE><<<blocks,threads>>>(o,16);
  cudaEvent_t a,b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a); k<MODE><<<blocks,threads>>>(o,iters); cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms,a,b);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double ops=(double)blocks*threads*iters*8; // per-element ops
  printf("%-10s threads %4d: %.3f ms, %.2f ops/clk/SM (clock %.0f MHz assumed)\n", name, threads, ms, ops/148/(ms*1e-3*clk*1e3), clk/1e3);
}
int main(){
  for(int t: {256, 512, 1024}){ run<0>("ex2",t); run<1>("f2fp",t); run<2>("ex2+f2fp/2",t); run<3>("ex2.f16x2",t); run<4>("polyexp2",t); run<5>("intpack",t);}
  return 0;
}
