// Texture-unit trilinear throughput on B200 (tools/, not product code): R32F 3D texture, linear
// filtering, unnormalised coordinates, random points inside a 24^3 grid. Reports filtered samples
// per clock per SM, plus the same loop with explicit 8-corner smem gathers for comparison.
#include <cstdio>
#include <cuda_runtime.h>

__device__ unsigned long long g_cyc[1024];

__global__ void __launch_bounds__(1024, 1) tex_kernel(cudaTextureObject_t tex, float* out, int iters, float span) {
  unsigned u = threadIdx.x * 2654435761u + blockIdx.x * 97u;
  float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  float px[8], py[8], pz[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    u = u * 1664525u + 1013904223u; px[j] = 0.5f + span * (u >> 8) * (1.0f / 16777216.0f);
    u = u * 1664525u + 1013904223u; py[j] = 0.5f + span * (u >> 8) * (1.0f / 16777216.0f);
    u = u * 1664525u + 1013904223u; pz[j] = 0.5f + span * (u >> 8) * (1.0f / 16777216.0f);
  }
  const float step = 0.37f;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      acc[j] += tex3D<float>(tex, px[j], py[j], pz[j]);
      px[j] += step; if (px[j] > span) px[j] -= span;
      py[j] += 0.61f * step; if (py[j] > span) py[j] -= span;
    }
  }
  long long t1 = clock64();
  float s = 0; for (int j = 0; j < 8; ++j) s += acc[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) g_cyc[blockIdx.x] = t1 - t0;
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int n = 24;
  float* h = new float[n * n * n];
  for (int i = 0; i < n * n * n; ++i) h[i] = (i % 97) / 97.0f;
  cudaArray_t arr; cudaChannelFormatDesc cd = cudaCreateChannelDesc<float>();
  cudaMalloc3DArray(&arr, &cd, make_cudaExtent(n, n, n));
  cudaMemcpy3DParms p = {}; p.srcPtr = make_cudaPitchedPtr(h, n * 4, n, n); p.dstArray = arr;
  p.extent = make_cudaExtent(n, n, n); p.kind = cudaMemcpyHostToDevice; cudaMemcpy3D(&p);
  cudaResourceDesc rd = {}; rd.resType = cudaResourceTypeArray; rd.res.array.array = arr;
  float* out; cudaMalloc(&out, sizeof(float) * sms * 1024);
  for (int mode = 0; mode < 2; ++mode) {
    cudaTextureDesc td = {}; td.addressMode[0] = td.addressMode[1] = td.addressMode[2] = cudaAddressModeClamp;
    td.filterMode = mode ? cudaFilterModePoint : cudaFilterModeLinear; td.readMode = cudaReadModeElementType; td.normalizedCoords = 0;
    cudaTextureObject_t tex; cudaCreateTextureObject(&tex, &rd, &td, nullptr);
    for (float span : {23.0f, 4.0f}) {
      const int iters = 2048;
      tex_kernel<<<sms, 1024>>>(tex, out, 16, span);
      cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
      cudaEventRecord(e0); tex_kernel<<<sms, 1024>>>(tex, out, iters, span); cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      unsigned long long c[1024]; cudaMemcpyFromSymbol(c, g_cyc, sizeof(unsigned long long) * sms);
      double mean = 0; for (int i = 0; i < sms; ++i) mean += c[i]; mean /= sms;
      printf("%s span %5.1f: %.2f samples/clk/SM  (%.3f ms)\n", mode ? "point " : "linear", span, 1024.0 * iters * 8 / mean, ms);
    }
    cudaDestroyTextureObject(tex);
  }
  printf("status %s\n", cudaGetErrorString(cudaGetLastError()));
}
