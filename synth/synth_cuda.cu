// synth_cuda.cu -- CUDA twin of the synthetic input generator (test/bench infrastructure).
// Same integer per-pixel functions as the CPU twin (synth.h), same host-built LUTs and
// per-frame parameters, so the caps it writes are bit-identical to sy_gen_host().
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>
#include "synth.h"

static sy_luts* g_dev_luts = nullptr;
static int g_dev_luts_device = -1;

__global__ void sy_gen_kernel(const sy_luts* __restrict__ L, const sy_frame* __restrict__ frames, int n, int H,
                              int W, int K, int garbage, int32_t* cs, int32_t* ct, int32_t* cnb) {
  __shared__ sy_frame f;
  int i = blockIdx.z;
  if (threadIdx.x == 0 && threadIdx.y == 0) f = frames[i];
  __syncthreads();
  int x = blockIdx.x * blockDim.x + threadIdx.x;
  int y = blockIdx.y * blockDim.y + threadIdx.y;
  if (x >= W || y >= H) return;
  int64_t plane = (int64_t)H * W;
  int64_t o = (int64_t)y * W + x;
  sy_pixel(L, &f, K, garbage, y, x, cs + (int64_t)i * plane + o, ct + (int64_t)i * plane + o,
           cnb + (int64_t)i * plane * K + o, plane);
}

extern "C" int sy_gen_cuda(int kind, uint64_t seed, int t0, int n, int H, int W, int K, int garbage, int seq_len,
                           int32_t* cs, int32_t* ct, int32_t* cnb, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 1;
  if (g_dev_luts == nullptr || g_dev_luts_device != dev) {
    sy_luts* h = (sy_luts*)malloc(sizeof(sy_luts));
    sy_build_luts(h);
    if (cudaMalloc(&g_dev_luts, sizeof(sy_luts)) != cudaSuccess) { free(h); return 2; }
    cudaMemcpy(g_dev_luts, h, sizeof(sy_luts), cudaMemcpyHostToDevice);
    free(h);
    g_dev_luts_device = dev;
  }
  if (n <= 0) return 0;
  // per-frame parameters: computed on the host, chunked to bound the staging buffer
  const int CH = 65535;
  for (int base = 0; base < n; base += CH) {
    int m = n - base < CH ? n - base : CH;
    sy_frame* hf = (sy_frame*)malloc(sizeof(sy_frame) * m);
    for (int i = 0; i < m; ++i) {
      int t = t0 + base + i;
      int seq_t = seq_len > 0 ? (t % seq_len) : t;
      sy_make_frame(&hf[i], kind, seed, H, W, t, seq_t);
    }
    sy_frame* df = nullptr;
    if (cudaMalloc(&df, sizeof(sy_frame) * m) != cudaSuccess) { free(hf); return 2; }
    cudaMemcpyAsync(df, hf, sizeof(sy_frame) * m, cudaMemcpyHostToDevice, st);
    dim3 blk(32, 8, 1);
    dim3 grd((W + 31) / 32, (H + 7) / 8, m);
    int64_t plane = (int64_t)H * W;
    sy_gen_kernel<<<grd, blk, 0, st>>>(g_dev_luts, df, m, H, W, K, garbage, cs + base * plane, ct + base * plane,
                                       cnb + base * plane * K);
    cudaError_t e = cudaGetLastError();
    cudaStreamSynchronize(st);
    cudaFree(df);
    free(hf);
    if (e != cudaSuccess) { fprintf(stderr, "sy_gen_cuda: %s\n", cudaGetErrorString(e)); return 3; }
  }
  return 0;
}

__global__ void sy_energy_kernel(const sy_luts* __restrict__ L, const sy_frame* __restrict__ frames, int H, int W,
                                 uint8_t* rgb, uint16_t* prior) {
  __shared__ sy_frame f;
  int i = blockIdx.z;
  if (threadIdx.x == 0 && threadIdx.y == 0) f = frames[i];
  __syncthreads();
  int x = blockIdx.x * blockDim.x + threadIdx.x;
  int y = blockIdx.y * blockDim.y + threadIdx.y;
  if (x >= W || y >= H) return;
  int64_t o = (int64_t)i * H * W + (int64_t)y * W + x;
  sy_energy_pixel(L, &f, y, x, rgb + 3 * o, prior + o);
}

extern "C" int sy_gen_energy_cuda(uint64_t seed, int t0, int n, int H, int W, int seq_len, uint8_t* rgb,
                                  uint16_t* prior, void* stream) {
  int32_t dummy;
  (void)dummy;
  if (sy_gen_cuda(SY_KIND_BLOB, seed, t0, 0, H, W, 4, 0, seq_len, nullptr, nullptr, nullptr, stream) != 0) return 2;
  cudaStream_t st = (cudaStream_t)stream;
  if (n <= 0) return 0;
  const int CH = 65535;
  for (int base = 0; base < n; base += CH) {
    int m = n - base < CH ? n - base : CH;
    sy_frame* hf = (sy_frame*)malloc(sizeof(sy_frame) * m);
    for (int i = 0; i < m; ++i) {
      int t = t0 + base + i;
      int seq_t = seq_len > 0 ? (t % seq_len) : t;
      sy_make_frame(&hf[i], SY_KIND_BLOB, seed, H, W, t, seq_t);
    }
    sy_frame* df = nullptr;
    if (cudaMalloc(&df, sizeof(sy_frame) * m) != cudaSuccess) { free(hf); return 2; }
    cudaMemcpyAsync(df, hf, sizeof(sy_frame) * m, cudaMemcpyHostToDevice, st);
    dim3 blk(32, 8, 1);
    dim3 grd((W + 31) / 32, (H + 7) / 8, m);
    int64_t plane = (int64_t)H * W;
    sy_energy_kernel<<<grd, blk, 0, st>>>(g_dev_luts, df, H, W, rgb + base * plane * 3, prior + base * plane);
    cudaError_t e = cudaGetLastError();
    cudaStreamSynchronize(st);
    cudaFree(df);
    free(hf);
    if (e != cudaSuccess) { fprintf(stderr, "sy_gen_energy_cuda: %s\n", cudaGetErrorString(e)); return 3; }
  }
  return 0;
}
