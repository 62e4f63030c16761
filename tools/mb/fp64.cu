#include <cstdio>
__global__ void dadd_k(double* out, int n) {
  double a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0+4, a5=a0+5, a6=a0+6, a7=a0+7;
  const double b = 1e-9;
  for (int i = 0; i < n; ++i) {
    a0 += b; a1 += b; a2 += b; a3 += b; a4 += b; a5 += b; a6 += b; a7 += b;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}
__global__ void fadd_k(float* out, int n) {
  float a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0+4, a5=a0+5, a6=a0+6, a7=a0+7;
  const float b = 1e-9f;
  for (int i = 0; i < n; ++i) {
    a0 += b; a1 += b; a2 += b; a3 += b; a4 += b; a5 += b; a6 += b; a7 += b;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}
__global__ void dmma_k(double* out, int n) {
  double d[8][2] = {};
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};" : "+d"(d[k][0]), "+d"(d[k][1]) : "d"(a), "d"(b));
  }
  double s = 0; for (int k = 0; k < 8; ++k) s += d[k][0] + d[k][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main2();
int main() {
  main2();
  double* o; cudaMalloc(&o, 148 * 8 * 1024 * 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int n = 1 << 16; float ms;
  for (int rep = 0; rep < 2; ++rep) {
  cudaEventRecord(e0); dadd_k<<<148 * 4, 256>>>(o, n); cudaEventRecord(e1); cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  double ops = 148.0 * 4 * 256 * n * 8;
  printf("DADD: %.3f ms  %.1f Gop/s  %.1f per clk per SM @1.9GHz\n", ms, ops / ms / 1e6, ops / (ms * 1e-3) / 1.9e9 / 148);
  cudaEventRecord(e0); fadd_k<<<148 * 4, 256>>>((float*)o, n); cudaEventRecord(e1); cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  printf("FADD: %.3f ms  %.1f per clk per SM\n", ms, ops / (ms * 1e-3) / 1.9e9 / 148);
  cudaEventRecord(e0); dmma_k<<<148 * 4, 256>>>(o, n / 8); cudaEventRecord(e1); cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  double fma = 148.0 * 4 * 8 * (n / 8) * 8 * 256;  // warps * iters * 8 mma * 256 FMA
  printf("DMMA: %.3f ms  %.2f TFLOP/s  %.1f FMA per clk per SM\n", ms, 2 * fma / ms / 1e9, fma / (ms * 1e-3) / 1.9e9 / 148);
  }
  return 0;
}
// appended: conversion throughput
__global__ void f2f_k(double* out, int n) {
  float x0 = threadIdx.x * 1e-3f, x1 = x0 + 1.f, x2 = x0 + 2.f, x3 = x0 + 3.f;
  double a0 = 0, a1 = 0, a2 = 0, a3 = 0;
  for (int i = 0; i < n; ++i) {
    a0 += (double)x0; a1 += (double)x1; a2 += (double)x2; a3 += (double)x3;
    x0 += 1e-7f; x1 += 1e-7f; x2 += 1e-7f; x3 += 1e-7f;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3;
}
__device__ __forceinline__ double f2d_int(float f) {
  const unsigned u = __float_as_uint(f);
  const unsigned e = (u >> 23) & 0xff;
  const unsigned long long hi = (unsigned long long)((u & 0x80000000u) | (e ? ((e + 896u) << 20) : 0u) | ((u & 0x7fffffu) >> 3));
  const unsigned lo = e ? (u << 29) : 0u;
  return __hiloint2double((int)hi, (int)lo);
}
__global__ void f2i_k(double* out, int n) {
  float x0 = threadIdx.x * 1e-3f + 1.f, x1 = x0 + 1.f, x2 = x0 + 2.f, x3 = x0 + 3.f;
  double a0 = 0, a1 = 0, a2 = 0, a3 = 0;
  for (int i = 0; i < n; ++i) {
    a0 += f2d_int(x0); a1 += f2d_int(x1); a2 += f2d_int(x2); a3 += f2d_int(x3);
    x0 += 1e-7f; x1 += 1e-7f; x2 += 1e-7f; x3 += 1e-7f;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3;
}
int main2() {
  double* o; cudaMalloc(&o, 148 * 8 * 1024 * 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int n = 1 << 16; float ms;
  for (int rep = 0; rep < 2; ++rep) {
    double ops = 148.0 * 4 * 256 * n * 4;
    cudaEventRecord(e0); f2f_k<<<148 * 4, 256>>>(o, n); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("F2F+DADD: %.3f ms  %.1f conv+add per clk per SM\n", ms, ops / (ms * 1e-3) / 1.9e9 / 148);
    cudaEventRecord(e0); f2i_k<<<148 * 4, 256>>>(o, n); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("INTCONV+DADD: %.3f ms  %.1f conv+add per clk per SM\n", ms, ops / (ms * 1e-3) / 1.9e9 / 148);
  }
  return 0;
}
