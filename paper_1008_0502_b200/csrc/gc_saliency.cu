// gc_saliency.cu -- NEXT-4: the Itti-style saliency map of PAPER.md §3 /
// §7.2 on the device ("fundamental feature extraction such as intensity, color
// opponents, edge orientation and optical flow, Gaussian pyramid construction, a special
// normalization function utilizing the global and local [extrema] of pixel values, and
// weighted addition of images" -- pixel-wise computation, filter convolution and local
// extrema detection).  Every step is float32 with the operation order written out and no
// FMA contraction (this file is compiled with -fmad=false), reductions are exact (min / max,
// and an int64 fixed-point sum for the mean of local maxima), so the numpy float32 oracle
// (oracle/saliency.py) reproduces every value bit for bit.  Readings: DESIGN.md c18-c23.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <string.h>

#include <string>
#include <vector>

#include "gc.h"

// gc_solver.cu: the context's grow-only device scratch (library-internal)
extern "C" void* gc_ctx_scratch(gc_ctx* c, int i, size_t bytes);
extern "C" void gc_ctx_set_launches(gc_ctx* c, long long n);

namespace {

constexpr int NLEV = 9;      // pyramid levels 0..8
constexpr int LMR = 7;       // local-maximum window radius
constexpr int GABOR = 9;     // 9 x 9 orientation filters
constexpr int NORI = 4;      // 0, 45, 90, 135 degrees
const int CENTERS[3] = {2, 3, 4};
const int DELTAS[2] = {3, 4};

__constant__ float c_gabor[NORI][GABOR * GABOR];

int half_up(int v) { return (v + 1) / 2; }

// level-0 features: I = (r + g + b) / 3, RG = (r - g) / I, BY = (b - (r + g) / 2) / I (zero
// where I < 0.1), M = |I - I_prev| (zero without a previous frame); r, g, b = byte / 255
__global__ void k_features(int n, int HW, const uint8_t* img, const uint8_t* prev, float* I, float* RG, float* BY,
                           float* M) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (size_t)n * HW) return;
  const float k255 = 255.0f;
  const float r = img[3 * i] / k255, g = img[3 * i + 1] / k255, b = img[3 * i + 2] / k255;
  const float in = ((r + g) + b) / 3.0f;
  I[i] = in;
  float rg = 0.0f, by = 0.0f;
  if (in >= 0.1f) {
    rg = (r - g) / in;
    by = (b - (r + g) / 2.0f) / in;
  }
  RG[i] = rg;
  BY[i] = by;
  float m = 0.0f;
  if (prev) {
    const float pr = prev[3 * i] / k255, pg = prev[3 * i + 1] / k255, pb = prev[3 * i + 2] / k255;
    const float pin = ((pr + pg) + pb) / 3.0f;
    m = fabsf(in - pin);
  }
  M[i] = m;
}

// blur with [1 4 6 4 1] / 16 (separable, clamped border) and decimate by 2:
// out(y, x) = sum_j w_j (sum_i w_i in(clamp(2y + j - 2), clamp(2x + i - 2))), i, j ascending
__global__ void k_down(int n, int h, int w, int h2, int w2, const float* in, float* out) {
  const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (size_t)n * h2 * w2) return;
  const int f = (int)(idx / ((size_t)h2 * w2));
  const int r = (int)(idx % ((size_t)h2 * w2));
  const int y = r / w2, x = r % w2;
  const float wt[5] = {1.0f / 16.0f, 4.0f / 16.0f, 6.0f / 16.0f, 4.0f / 16.0f, 1.0f / 16.0f};
  const float* src = in + (size_t)f * h * w;
  float acc = 0.0f;
  for (int j = 0; j < 5; ++j) {
    const int yy = min(max(2 * y + j - 2, 0), h - 1);
    float row = 0.0f;
    for (int i = 0; i < 5; ++i) {
      const int xx = min(max(2 * x + i - 2, 0), w - 1);
      row = row + wt[i] * src[(size_t)yy * w + xx];
    }
    acc = acc + wt[j] * row;
  }
  out[idx] = acc;
}

// orientation response |gabor_theta * I| (9 x 9, clamped border, row-major summation order)
__global__ void k_gabor(int n, int h, int w, int th, const float* in, float* out) {
  const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (size_t)n * h * w) return;
  const int f = (int)(idx / ((size_t)h * w));
  const int r = (int)(idx % ((size_t)h * w));
  const int y = r / w, x = r % w;
  const float* src = in + (size_t)f * h * w;
  float acc = 0.0f;
  for (int j = 0; j < GABOR; ++j) {
    const int yy = min(max(y + j - GABOR / 2, 0), h - 1);
    for (int i = 0; i < GABOR; ++i) {
      const int xx = min(max(x + i - GABOR / 2, 0), w - 1);
      acc = acc + c_gabor[th][j * GABOR + i] * src[(size_t)yy * w + xx];
    }
  }
  out[idx] = fabsf(acc);
}

// bilinear sample of a (hs x ws) map at the centre of pixel (y, x) of an (hc x wc) grid
__device__ __forceinline__ float bilinear(const float* s, int hs, int ws, int hc, int wc, int y, int x) {
  const float sy = ((float)y + 0.5f) * ((float)hs / (float)hc) - 0.5f;
  const float sx = ((float)x + 0.5f) * ((float)ws / (float)wc) - 0.5f;
  const float fy0 = floorf(sy), fx0 = floorf(sx);
  const float ay = sy - fy0, ax = sx - fx0;
  const int y0 = min(max((int)fy0, 0), hs - 1), y1 = min(max((int)fy0 + 1, 0), hs - 1);
  const int x0 = min(max((int)fx0, 0), ws - 1), x1 = min(max((int)fx0 + 1, 0), ws - 1);
  const float top = (1.0f - ax) * s[(size_t)y0 * ws + x0] + ax * s[(size_t)y0 * ws + x1];
  const float bot = (1.0f - ax) * s[(size_t)y1 * ws + x0] + ax * s[(size_t)y1 * ws + x1];
  return (1.0f - ay) * top + ay * bot;
}

// center-surround: |center - upsample(surround)| at the center level's size
__global__ void k_cs(int n, int hc, int wc, int hs, int ws, const float* cen, const float* sur, float* out) {
  const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (size_t)n * hc * wc) return;
  const int f = (int)(idx / ((size_t)hc * wc));
  const int r = (int)(idx % ((size_t)hc * wc));
  const int y = r / wc, x = r % wc;
  out[idx] = fabsf(cen[idx] - bilinear(sur + (size_t)f * hs * ws, hs, ws, hc, wc, y, x));
}

// per-frame min / max (float bits: non-negative maps only -> unsigned order = float order)
__global__ void k_minmax(int n, int hw, const float* v, unsigned* mn, unsigned* mx) {
  const int f = blockIdx.y;
  unsigned lo = 0x7f800000u, hi = 0u;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < hw; i += gridDim.x * blockDim.x) {
    const unsigned b = __float_as_uint(v[(size_t)f * hw + i]);
    lo = min(lo, b);
    hi = max(hi, b);
  }
  for (int o = 16; o > 0; o >>= 1) {
    lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMin(mn + f, lo);
    atomicMax(mx + f, hi);
  }
}

// rescale to [0, 1]: (v - min) / (max - min), all 0 for a constant map
__global__ void k_rescale(int n, int hw, float* v, const unsigned* mn, const unsigned* mx) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (size_t)n * hw) return;
  const int f = (int)(i / hw);
  const float lo = __uint_as_float(mn[f]), hi = __uint_as_float(mx[f]);
  v[i] = hi > lo ? (v[i] - lo) / (hi - lo) : 0.0f;
}

// separable window maximum, radius LMR (clamped): rows then columns
__global__ void k_rowmax(int n, int h, int w, const float* v, float* o) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (size_t)n * h * w) return;
  const int x = (int)(i % w);
  const float* row = v + (i - x);
  float m = row[x];
  for (int d = 1; d <= LMR; ++d) m = fmaxf(m, fmaxf(row[max(x - d, 0)], row[min(x + d, w - 1)]));
  o[i] = m;
}
__global__ void k_colmax_localmax(int n, int h, int w, const float* v, const float* rm, unsigned long long* cnt,
                                  unsigned long long* sum) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  unsigned long long c = 0, s = 0;
  int f = 0;
  if (i < (size_t)n * h * w) {
    f = (int)(i / ((size_t)h * w));
    const int r = (int)(i % ((size_t)h * w));
    const int y = r / w, x = r % w;
    const float* col = rm + (size_t)f * h * w + x;
    float m = col[(size_t)y * w];
    for (int d = 1; d <= LMR; ++d) m = fmaxf(m, fmaxf(col[(size_t)max(y - d, 0) * w], col[(size_t)min(y + d, h - 1) * w]));
    const float val = v[i];
    if (val > 0.0f && val == m) {  // a local maximum: >= every pixel of its window
      c = 1;
      s = (unsigned long long)floor((double)val * 16777216.0);  // fixed point 2^-24, exact sum
    }
  }
  // frames do not mix inside a warp only if h*w is a multiple of 32: reduce per frame atomically
  if (c) {
    atomicAdd(cnt + f, 1ull);
    atomicAdd(sum + f, s);
  }
}

// N(.): multiply by (1 - mbar)^2, mbar = mean of the local maxima except one instance of the
// global maximum (1 after rescaling); mbar = 0 with fewer than two local maxima
__global__ void k_nscale(int n, int hw, float* v, const unsigned long long* cnt, const unsigned long long* sum,
                         const unsigned* mx, const unsigned* mn) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (size_t)n * hw) return;
  const int f = (int)(i / hw);
  float fac = 1.0f;
  if (__uint_as_float(mx[f]) > __uint_as_float(mn[f]) && cnt[f] > 1) {
    const double mb = (double)(sum[f] - 16777216ull) / 16777216.0 / (double)(cnt[f] - 1);
    const float m = (float)mb;
    fac = (1.0f - m) * (1.0f - m);
  }
  v[i] = v[i] * fac;
}

__global__ void k_accum(size_t total, const float* a, float* acc) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < total) acc[i] = acc[i] + a[i];
}

__global__ void k_final(size_t total, const float* a, const float* b, const float* c, const float* d, float* out) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < total) out[i] = (((a[i] + b[i]) + c[i]) + d[i]) / 4.0f;
}

// saliency at level 4 -> full-resolution prior code floor(65535 s + 0.5) (bilinear)
__global__ void k_upcode(int n, int H, int W, int h4, int w4, const float* s, uint16_t* q) {
  const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (size_t)n * H * W) return;
  const int f = (int)(idx / ((size_t)H * W));
  const int r = (int)(idx % ((size_t)H * W));
  const float v = bilinear(s + (size_t)f * h4 * w4, h4, w4, H, W, r / W, r % W);
  const float c = floorf(65535.0f * v + 0.5f);
  q[idx] = (uint16_t)(c < 0.0f ? 0.0f : (c > 65535.0f ? 65535.0f : c));
}

unsigned nblk(size_t total) { return (unsigned)((total + 255) / 256); }

}  // namespace

extern "C" {

gc_status gc_gabor_kernels(float* out) {
  if (!out) return GC_ERR_ARG;
  // 9 x 9 even Gabor, sigma 2, wavelength 6, aspect 0.5, zero mean (reading c19)
  const double PI = 3.14159265358979323846;
  for (int t = 0; t < NORI; ++t) {
    const double th = t * PI / 4.0;
    double g[GABOR * GABOR], mean = 0.0;
    for (int j = 0; j < GABOR; ++j)
      for (int i = 0; i < GABOR; ++i) {
        const double x = i - GABOR / 2, y = j - GABOR / 2;
        const double xr = x * cos(th) + y * sin(th), yr = -x * sin(th) + y * cos(th);
        g[j * GABOR + i] = exp(-(xr * xr + 0.25 * yr * yr) / (2.0 * 2.0 * 2.0)) * cos(2.0 * PI * xr / 6.0);
        mean += g[j * GABOR + i];
      }
    mean /= GABOR * GABOR;
    for (int k = 0; k < GABOR * GABOR; ++k) out[t * GABOR * GABOR + k] = (float)(g[k] - mean);
  }
  return GC_OK;
}

gc_status gc_saliency_dims(int H, int W, int* h4, int* w4) {
  if (H <= 0 || W <= 0 || !h4 || !w4) return GC_ERR_ARG;
  int h = H, w = W;
  for (int l = 0; l < 4; ++l) { h = half_up(h); w = half_up(w); }
  *h4 = h;
  *w4 = w;
  return GC_OK;
}

gc_status gc_saliency(gc_ctx* ctx, const gc_saliency_batch* b, void* stream) {
  if (!ctx || !b) return GC_ERR_ARG;
  const int n = b->n, H = b->H, W = b->W;
  if (n < 0 || H <= 0 || W <= 0 || (n > 0 && (!b->image || (!b->sal_out && !b->q_out)))) return GC_ERR_ARG;
  if (n == 0) return GC_OK;
  cudaStream_t st = (cudaStream_t)stream;
  {
    float k[NORI * GABOR * GABOR];
    gc_gabor_kernels(k);
    if (cudaMemcpyToSymbolAsync(c_gabor, k, sizeof(k), 0, cudaMemcpyHostToDevice, st) != cudaSuccess) return GC_ERR_CUDA;
  }
  int hl[NLEV], wl[NLEV];
  hl[0] = H; wl[0] = W;
  for (int l = 1; l < NLEV; ++l) { hl[l] = half_up(hl[l - 1]); wl[l] = half_up(wl[l - 1]); }
  std::vector<size_t> off(NLEV + 1, 0);
  for (int l = 0; l < NLEV; ++l) off[l + 1] = off[l] + (size_t)n * hl[l] * wl[l];
  const size_t pyr = off[NLEV];
  const size_t n4 = (size_t)n * hl[4] * wl[4];
  const size_t nc = (size_t)n * hl[2] * wl[2];  // largest feature map
  // scratch: 4 feature pyramids + 4 orientation pyramids, feature map + temps, class sums
  const size_t fl = 8 * pyr + 3 * nc + 6 * n4 + 16;
  // the context's grow-only scratch (no allocation per call once it has grown)
  float* buf = static_cast<float*>(gc_ctx_scratch(ctx, 0, fl * sizeof(float)));
  void* red = gc_ctx_scratch(ctx, 1, (size_t)n * 32);
  if (!buf || !red) return GC_ERR_OOM;
  float* P[8];
  for (int c = 0; c < 8; ++c) P[c] = buf + c * pyr;  // I, RG, BY, M, O0..O3
  float* fm = buf + 8 * pyr;   // feature map
  float* tmp = fm + nc;        // row maxima / downsampling
  float* tmp2 = tmp + nc;
  float* cls[4];
  for (int c = 0; c < 4; ++c) cls[c] = tmp2 + nc + c * n4;  // class sums at level 4
  float* acc = cls[3] + n4;                                  // per-orientation sum
  float* sal = acc + n4;
  unsigned* mn = (unsigned*)red;
  unsigned* mx = mn + n;
  unsigned long long* cnt = (unsigned long long*)(mx + n);  // 8n bytes in: aligned
  unsigned long long* sum = cnt + n;
  const size_t HW = (size_t)H * W;
  long long nl = 0;  // kernel launches of this call (gc_last_launches)
  k_features<<<nblk(n * HW), 256, 0, st>>>(n, (int)HW, b->image, b->prev, P[0], P[1], P[2], P[3]); ++nl;
  for (int c = 0; c < 4; ++c)
    for (int l = 1; l < NLEV; ++l)
      k_down<<<nblk((size_t)n * hl[l] * wl[l]), 256, 0, st>>>(n, hl[l - 1], wl[l - 1], hl[l], wl[l], P[c] + off[l - 1],
                                                              P[c] + off[l]); ++nl;
  for (int t = 0; t < NORI; ++t)
    for (int l = 2; l < NLEV; ++l)
      k_gabor<<<nblk((size_t)n * hl[l] * wl[l]), 256, 0, st>>>(n, hl[l], wl[l], t, P[0] + off[l], P[4 + t] + off[l]); ++nl;
  cudaMemsetAsync(cls[0], 0, 4 * n4 * sizeof(float), st);
  // N(.) of a map at level l (in place), then added into `dst` at level 4
  auto normalize = [&](float* v, int l) {
    const size_t hw = (size_t)hl[l] * wl[l];
    cudaMemsetAsync(mn, 0xff, (size_t)n * 4, st);  // > +inf bits: every value lowers it
    cudaMemsetAsync(mx, 0, (size_t)n * 4, st);
    cudaMemsetAsync(cnt, 0, (size_t)n * 16, st);
    k_minmax<<<dim3(64, n), 256, 0, st>>>(n, (int)hw, v, mn, mx); ++nl;
    k_rescale<<<nblk(n * hw), 256, 0, st>>>(n, (int)hw, v, mn, mx); ++nl;
    k_rowmax<<<nblk(n * hw), 256, 0, st>>>(n, hl[l], wl[l], v, tmp); ++nl;
    k_colmax_localmax<<<nblk(n * hw), 256, 0, st>>>(n, hl[l], wl[l], v, tmp, cnt, sum); ++nl;
    k_nscale<<<nblk(n * hw), 256, 0, st>>>(n, (int)hw, v, cnt, sum, mx, mn); ++nl;
  };
  auto add_at4 = [&](const float* v, int l, float* dst) {
    const float* cur = v;
    for (int k = l; k < 4; ++k) {  // blur-decimate down to level 4
      float* o = (k % 2 == l % 2) ? tmp : tmp2;
      k_down<<<nblk((size_t)n * hl[k + 1] * wl[k + 1]), 256, 0, st>>>(n, hl[k], wl[k], hl[k + 1], wl[k + 1], cur, o); ++nl;
      cur = o;
    }
    k_accum<<<nblk(n4), 256, 0, st>>>(n4, cur, dst); ++nl;
  };
  // classes: 0 intensity, 1 colour (RG and BY), 2 orientation, 3 motion
  const int chan_class[8] = {0, 1, 1, 3, 2, 2, 2, 2};
  for (int ch = 0; ch < 8; ++ch) {
    float* dst = cls[chan_class[ch]];
    if (ch >= 4) {  // orientation: N(sum over c, s of N(O_theta(c, s))) per theta
      cudaMemsetAsync(acc, 0, n4 * sizeof(float), st);
      dst = acc;
    }
    for (int ci = 0; ci < 3; ++ci)
      for (int di = 0; di < 2; ++di) {
        const int c = CENTERS[ci], s = c + DELTAS[di];
        k_cs<<<nblk((size_t)n * hl[c] * wl[c]), 256, 0, st>>>(n, hl[c], wl[c], hl[s], wl[s], P[ch] + off[c],
                                                              P[ch] + off[s], fm); ++nl;
        normalize(fm, c);
        add_at4(fm, c, dst);
      }
    if (ch >= 4) {
      normalize(acc, 4);
      k_accum<<<nblk(n4), 256, 0, st>>>(n4, acc, cls[2]); ++nl;
    }
  }
  for (int c = 0; c < 4; ++c) normalize(cls[c], 4);
  k_final<<<nblk(n4), 256, 0, st>>>(n4, cls[0], cls[1], cls[2], cls[3], sal); ++nl;
  normalize(sal, 4);  // rescaled to [0, 1] (and the same N(.) as every stage)
  if (b->sal_out) cudaMemcpyAsync(b->sal_out, sal, n4 * sizeof(float), cudaMemcpyDeviceToDevice, st);
  if (b->q_out) k_upcode<<<nblk((size_t)n * HW), 256, 0, st>>>(n, H, W, hl[4], wl[4], sal, b->q_out); ++nl;
  const cudaError_t e = cudaGetLastError();
  const cudaError_t e2 = cudaStreamSynchronize(st);
  gc_ctx_set_launches(ctx, nl);
  return (e != cudaSuccess || e2 != cudaSuccess) ? GC_ERR_CUDA : GC_OK;
}

}  // extern "C"
