// Throughput of the conversions / f64 ops the exact predictor and norm passes use, per SM
// per clock (B200).  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/cvt_bench tools/cvt_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int MODE>
__global__ void k(float* out, int iters, long long* cyc) {
  float f[8];
  double dd[8];
  uint32_t u[8];
  for (int i = 0; i < 8; ++i) {
    f[i] = 1.0f + threadIdx.x * 1e-3f + i;
    dd[i] = f[i];
    u[i] = __float_as_uint(f[i]);
  }
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (MODE == 0) {  // F2F.F64.F32
        dd[i] += (double)f[i];
        f[i] = __uint_as_float(__float_as_uint(f[i]) ^ 1u);
      } else if (MODE == 1) {  // F2F.F32.F64
        f[i] += (float)dd[i];
        dd[i] = __longlong_as_double(__double_as_longlong(dd[i]) + 1ull);
      } else if (MODE == 2) {  // DFMA
        dd[i] = fma(dd[i], 0.999, 1e-3);
      } else if (MODE == 3) {  // FFMA
        f[i] = fmaf(f[i], 0.999f, 1e-3f);
      } else if (MODE == 4) {  // bf16 -> f64 via PTX cvt
        double t;
        unsigned short h = (unsigned short)(u[i] >> 16);
        asm volatile("{ .reg .b16 hb; mov.b16 hb, %1; cvt.f64.bf16 %0, hb; }" : "=d"(t) : "h"(h));
        dd[i] += t;
        u[i] ^= 0x10000u;
      }
    }
  }
  long long t1 = clock64();
  float s = 0;
  for (int i = 0; i < 8; ++i) s += f[i] + (float)dd[i] + u[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

template <int MODE>
void run(const char* name) {
  float* o;
  long long* c;
  cudaMalloc(&o, 148 * 1024 * 4 * 4);
  cudaMalloc(&c, 8);
  const int iters = 2000;
  k<MODE><<<148 * 8, 256>>>(o, 10, c);
  cudaDeviceSynchronize();
  k<MODE><<<148 * 8, 256>>>(o, iters, c);
  long long cyc;
  cudaMemcpy(&cyc, c, 8, cudaMemcpyDeviceToHost);
  // per SM: 8 CTAs x 256 threads x iters x 8 ops over cyc cycles
  printf("%-22s %6.1f ops/clk/SM   (%s)\n", name, 8.0 * 256 * iters * 8 / cyc,
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(o);
  cudaFree(c);
}

int main() {
  run<0>("F2F.F64.F32");
  run<1>("F2F.F32.F64");
  run<2>("DFMA");
  run<3>("FFMA");
  run<4>("cvt.f64.bf16");
  return 0;
}
