// FP32 FFMA peak of the B200 SM (tools/, not product code): the denominator of bench.py's FP32
// roofline. Each thread runs 16 independent FFMA chains whose multiplier and addend are kernel
// parameters (constant-bank operands: no register-bank conflicts), 8x unrolled (128 FFMA per loop
// trip, loop overhead < 3%); 2 CTAs x 1024 threads per SM. The SM clock comes from clock64 deltas
// over the kernel's CUDA-event time, so lane-ops/clk/SM does not depend on the clock the GPU ran.
// Also: the f32x2 form (FFMA2, 2 lane-ops per lane) with the same structure.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp32_peak fp32_peak.cu && ./fp32_peak
#include <cstdio>
#include <cuda_runtime.h>

__device__ unsigned long long g_cyc[4096];

template <bool PAIR>
__global__ void __launch_bounds__(1024, 2) ffma_kernel(float* out, float b, float c, int iters) {
  float x[16];
  float2 y[8];
#pragma unroll
  for (int j = 0; j < 16; ++j) x[j] = threadIdx.x * 1e-3f + j;
#pragma unroll
  for (int j = 0; j < 8; ++j) y[j] = make_float2(x[2 * j], x[2 * j + 1]);
  const float2 b2 = make_float2(b, b), c2 = make_float2(c, c);
  __syncthreads();
  const long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      if (PAIR) {
#pragma unroll
        for (int j = 0; j < 8; ++j) y[j] = __ffma2_rn(y[j], b2, c2);
      } else {
#pragma unroll
        for (int j = 0; j < 16; ++j) x[j] = fmaf(x[j], b, c);
      }
    }
  }
  const long long t1 = clock64();
  float s = 0.f;
#pragma unroll
  for (int j = 0; j < 16; ++j) s += x[j];
#pragma unroll
  for (int j = 0; j < 8; ++j) s += y[j].x + y[j].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) g_cyc[blockIdx.x] = (unsigned long long)(t1 - t0);
}

template <bool PAIR>
void run(const char* name, float* out, int sms, bool last) {
  const int iters = 1 << 14, blocks = 2 * sms, threads = 1024;
  ffma_kernel<PAIR><<<blocks, threads>>>(out, 0.999f, 1e-3f, 64);  // warm-up
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  double best = 0.0, best_ms = 0.0, best_mhz = 0.0;
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(e0);
    ffma_kernel<PAIR><<<blocks, threads>>>(out, 0.999f, 1e-3f, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    static unsigned long long cyc[4096];
    cudaMemcpyFromSymbol(cyc, g_cyc, sizeof(unsigned long long) * blocks);
    double mx = 0.0;
    for (int i = 0; i < blocks; ++i) mx = cyc[i] > mx ? double(cyc[i]) : mx;
    // lane-ops per SM: 2 CTAs x 1024 threads x iters x 128 FFMA (x 1: both forms are 128 lane-ops)
    const double lane_ops = 2.0 * threads * double(iters) * 128.0;
    const double per_clk = lane_ops / mx;
    if (per_clk > best) {
      best = per_clk;
      best_ms = ms;
      best_mhz = mx / (ms * 1e3);
    }
  }
  const double tflops = best * sms * best_mhz * 1e6 / 1e12;
  std::printf("  \"%s\": {\"lane_ops_per_clk_per_sm\": %.2f, \"ms\": %.3f, \"sm_mhz_effective\": %.0f, "
              "\"lane_ops_per_s_T\": %.2f}%s\n",
              name, best, best_ms, best_mhz, tflops, last ? "" : ",");
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* out = nullptr;
  cudaMalloc(&out, sizeof(float) * 2 * sms * 1024);
  std::printf("{\n  \"sms\": %d,\n", sms);
  run<false>("ffma", out, sms, false);
  run<true>("ffma2_f32x2", out, sms, true);
  std::printf("}\n");
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) std::fprintf(stderr, "error: %s\n", cudaGetErrorString(e));
  return e == cudaSuccess ? 0 : 1;
}
