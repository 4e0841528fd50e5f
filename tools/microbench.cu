// Pipe-throughput microbenchmarks on the B200 SM (tools/, not product code). Measures per-SM
// throughput in lane-ops/clk for the instruction mixes the pose-search kernel is built from:
// FFMA (3-register form), FFMA2 (f32x2), PRMT, FMNMX, random LDS.32 / LDS.128 (smem gathers),
// broadcast LDS.128. One 1024-thread CTA per SM, 8 independent chains per thread.
#include <cstdio>
#include <cuda_runtime.h>

#define CH 8
__device__ unsigned long long g_cycles[1024];

template <int OP>
__global__ void __launch_bounds__(1024, 1) bench(float* out, const float* in, int iters) {
  extern __shared__ uint4 tab[];
  const int t = threadIdx.x;
  for (int i = t; i < 8192; i += blockDim.x) tab[i] = make_uint4(i, i * 3, i * 5, i * 7);
  __syncthreads();
  float a[CH], b[CH], c[CH];
  float2 a2[CH], b2[CH], c2[CH];
  unsigned u[CH];
#pragma unroll
  for (int j = 0; j < CH; ++j) {
    a[j] = in[(t + j) & 255];
    b[j] = in[(t + 2 * j + 1) & 255];
    c[j] = in[(t + 3 * j + 2) & 255];
    a2[j] = make_float2(a[j], b[j]);
    b2[j] = make_float2(b[j], c[j]);
    c2[j] = make_float2(c[j], a[j]);
    u[j] = (t * 2654435761u) ^ (j * 40503u);
  }
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < CH; ++j) {
      if (OP == 0) a[j] = fmaf(a[j], b[j], c[j]);
      if (OP == 1) a2[j] = __ffma2_rn(a2[j], b2[j], c2[j]);
      if (OP == 2) u[j] = __byte_perm(u[j], (unsigned)i, 0x5410 + j);
      if (OP == 3) a[j] = fmaxf(fabsf(a[j]), c[j]) ;
      if (OP == 4) {  // random LDS.32 over 128 KB
        u[j] = u[j] * 1664525u + 1013904223u;
        a[j] += __uint_as_float(reinterpret_cast<const unsigned*>(tab)[(u[j] >> 9) & 32767]);
      }
      if (OP == 5) {  // random LDS.128 over 128 KB
        u[j] = u[j] * 1664525u + 1013904223u;
        const uint4 v = tab[(u[j] >> 11) & 8191];
        a[j] += __uint_as_float(v.x ^ v.y ^ v.z ^ v.w);
      }
      if (OP == 6) {  // broadcast LDS.128 (whole warp same address)
        const uint4 v = tab[(i * CH + j) & 8191];
        a[j] += __uint_as_float(v.x ^ v.y ^ v.z ^ v.w);
      }
      if (OP == 7) {  // address arithmetic only (baseline for 4/5)
        u[j] = u[j] * 1664525u + 1013904223u;
        a[j] += __uint_as_float((u[j] >> 11) & 8191);
      }
    }
  }
  long long t1 = clock64();
  float s = 0.f;
#pragma unroll
  for (int j = 0; j < CH; ++j) s += a[j] + a2[j].x + a2[j].y + __uint_as_float(u[j]);
  out[blockIdx.x * blockDim.x + t] = s;
  if (t == 0) g_cycles[blockIdx.x] = (unsigned long long)(t1 - t0);
}

template <int OP>
void run(const char* name, float* out, float* in, int sms, double lane_ops_per_iter) {
  const int iters = 4096;
  cudaFuncSetAttribute(bench<OP>, cudaFuncAttributeMaxDynamicSharedMemorySize, 8192 * 16);
  bench<OP><<<sms, 1024, 8192 * 16>>>(out, in, 16);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  bench<OP><<<sms, 1024, 8192 * 16>>>(out, in, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long cyc[1024];
  cudaMemcpyFromSymbol(cyc, g_cycles, sizeof(unsigned long long) * sms);
  double mean = 0;
  for (int i = 0; i < sms; ++i) mean += cyc[i];
  mean /= sms;
  const double ops = 1024.0 * iters * CH * lane_ops_per_iter;  // per SM
  printf("%-28s %8.1f lane-ops/clk/SM  (%.3f ms, %.0f MHz effective)\n", name, ops / mean, ms,
         mean / (ms * 1e3));
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float *out, *in;
  cudaMalloc(&out, sizeof(float) * sms * 1024);
  cudaMalloc(&in, sizeof(float) * 256);
  float h[256];
  for (int i = 0; i < 256; ++i) h[i] = 0.5f + i * 1e-3f;
  cudaMemcpy(in, h, sizeof h, cudaMemcpyHostToDevice);
  printf("SMs %d\n", sms);
  run<0>("FFMA r,r,r,r", out, in, sms, 1);
  run<1>("FFMA2 (f32x2, 2 ops/lane)", out, in, sms, 2);
  run<2>("PRMT", out, in, sms, 1);
  run<3>("FMNMX |a|", out, in, sms, 1);
  run<7>("IMAD+LOP (addr only)", out, in, sms, 1);
  run<4>("LDS.32 random (per load)", out, in, sms, 1);
  run<5>("LDS.128 random (per load)", out, in, sms, 1);
  run<6>("LDS.128 broadcast", out, in, sms, 1);
  cudaError_t e = cudaGetLastError();
  printf("status %s\n", cudaGetErrorString(e));
  return 0;
}
