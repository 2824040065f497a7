/* synth_host.c -- host side of the synthetic input generator (test/bench infrastructure).
 * Builds the integer LUTs in double precision, computes per-frame integer parameters
 * (trajectories, jitter, Sec. 6 Kalman weights), and runs the CPU twin of the per-pixel
 * generator.  See synth.h for the frame model and citations. */
#include "synth.h"
#include <math.h>
#include <string.h>

static int g_rmax_t = 1000, g_rmax_n = 1000, g_rzero = 20;
static int g_lane = 64, g_big = 1 << 20;

void sy_set_random_params(int rmax_t, int rmax_n, int rzero_pct) {
  g_rmax_t = rmax_t; g_rmax_n = rmax_n; g_rzero = rzero_pct;
}
void sy_set_serp_params(int lane, int big) { g_lane = lane; g_big = big; }

static int32_t quant(double x) { /* reading c11: floor(S x + 0.5), clamped to [0, CAP_MAX] */
  double v = floor(64.0 * x + 0.5);
  if (v < 0) v = 0;
  if (v > SY_CAP_MAX) v = SY_CAP_MAX;
  return (int32_t)v;
}

void sy_build_luts(sy_luts* L) {
  const double PI = 3.14159265358979323846;
  for (int i = 0; i <= SY_NP; ++i) {
    double p = (i == SY_NP) ? 1e-6 : 0.95 * (i + 0.5) / SY_NP; /* eps_p = 1e-6 (reading c9) */
    L->tl0_p[i] = quant(-log(1.0 - p));
    L->tl1_p[i] = quant(-log(p));
  }
  for (int I = 0; I < 256; ++I) {
    double d0 = (I - 100.0) / 30.0, d1 = (I - 200.0) / 25.0;
    L->tl0_I[I] = quant(log(30.0 * sqrt(2 * PI)) + 0.5 * d0 * d0);
    L->tl1_I[I] = quant(log(25.0 * sqrt(2 * PI)) + 0.5 * d1 * d1);
  }
  const double lambda = 10.0, sigma = 0.1, kappa = 0.05; /* S:447 defaults, reading c5 */
  for (int d = 0; d < 256; ++d) {
    double g = (d / 255.0);
    double e = exp(-(g * g) / (2 * sigma * sigma));
    L->nl[0][d] = quant(lambda * e / 1.0 + kappa);
    L->nl[1][d] = quant(lambda * e / sqrt(2.0) + kappa);
  }
  for (int i = 0; i < SY_NQ; ++i) L->q_lut[i] = (int32_t)floor(65535.0 * exp(-i / 64.0) + 0.5);
  for (int i = 0; i < SY_NF; ++i) {
    double rho = sqrt(i / 256.0);
    L->f_lut[i] = (int32_t)floor(65535.0 / (1.0 + exp(8.0 * (rho - 1.0))) + 0.5);
  }
}

/* Sec. 6 prior update as printed (reading c10):
 *   w_f = s1^2/(s1^2+s2^2+v),  w_q = (s2^2+v)/(s1^2+s2^2+v),
 *   v(t) = s1^2 (s2^2+v(t-1)) / (s1^2+s2^2+v(t-1)),  v(0) = 0, s1=0.03, s2=0.035. */
void sy_kalman_weights(int seq_t, double* wf, double* wq, double* var_out) {
  const double s1 = 0.03 * 0.03, s2 = 0.035 * 0.035;
  double v = 0.0;
  for (int t = 1; t < seq_t; ++t) v = s1 * (s2 + v) / (s1 + s2 + v);
  double den = s1 + s2 + v;
  if (wf) *wf = s1 / den;
  if (wq) *wq = (s2 + v) / den;
  if (var_out) *var_out = v;
}

void sy_make_frame(sy_frame* f, int kind, uint64_t seed, int H, int W, int t, int seq_t) {
  memset(f, 0, sizeof(*f));
  f->kind = kind; f->H = H; f->W = W; f->seed = seed; f->frame = (uint32_t)t;
  f->lane = g_lane; f->big = g_big;
  f->rmax_t = g_rmax_t; f->rmax_n = g_rmax_n; f->rzero_pct = g_rzero;
  if (kind != SY_KIND_BLOB) return;
  /* objects: count and motion constants from the seed (static per sequence) */
  uint64_t h0 = sy_mix64(seed ^ 0x51u);
  f->nobj = 1 + (int)(h0 % 3u);
  const double omega = 2.0 * 3.14159265358979323846 / 96.0; /* one loop per 8 s at 12 fps */
  int mind = H < W ? H : W;
  double rs_y = 0, rs_x = 0;
  for (int j = 0; j < f->nobj; ++j) {
    uint64_t hj = sy_mix64(seed ^ (0x100u + (uint64_t)j));
    double u0 = (hj & 0xffff) / 65535.0, u1 = ((hj >> 16) & 0xffff) / 65535.0;
    double u2 = ((hj >> 32) & 0xffff) / 65535.0, u3 = ((hj >> 48) & 0xffff) / 65535.0;
    double ry = H * (0.10 + 0.10 * u0), rx = ry * (0.8 + 0.5 * u1);
    if (ry < 2) ry = 2;
    if (rx < 2) rx = 2;
    if (rx > 0.3 * W) rx = 0.3 * W;
    double ph = 6.283185307179586 * u2, ph2 = 6.283185307179586 * u3;
    double ay = 0.5 * H - ry - 1, ax = 0.5 * W - rx - 1;
    if (ay < 0) ay = 0;
    if (ax < 0) ax = 0;
    for (int back = 0; back <= 1; ++back) {
      double tt = (double)(t - back);
      double cy = 0.5 * H + 0.6 * ay * sin(omega * tt + ph);
      double cx = 0.5 * W + 0.6 * ax * sin(0.7 * omega * tt + ph2);
      int32_t icy = (int32_t)floor(cy * 16.0 + 0.5), icx = (int32_t)floor(cx * 16.0 + 0.5);
      if (back == 0) { f->cy[j] = icy; f->cx[j] = icx; }
      else { f->py[j] = icy; f->px[j] = icx; }
    }
    f->ry[j] = (int32_t)floor(ry + 0.5);
    f->rx[j] = (int32_t)floor(rx + 0.5);
    rs_y += ry; rs_x += rx;
  }
  /* saliency blob around object 0's centre with per-frame +-3 px jitter */
  uint64_t hq = sy_hash(seed, (uint32_t)t, -1, -1, 3);
  f->qy = (int32_t)floor(f->cy[0] / 16.0 + 0.5) + (int)(hq % 7u) - 3;
  f->qx = (int32_t)floor(f->cx[0] / 16.0 + 0.5) + (int)((hq >> 8) % 7u) - 3;
  double sig = 0.5 * (rs_y + rs_x) / f->nobj;
  if (sig < 1) sig = 1;
  (void)mind;
  /* LUT index = s*64 with s = d2/(2 sig^2)  ->  index = d2 * (64/(2 sig^2)) */
  f->q_scale = (int32_t)floor(65536.0 * 64.0 / (2.0 * sig * sig) + 0.5);
  f->has_prev = seq_t > 0;
  double wf, wq;
  sy_kalman_weights(seq_t > 0 ? seq_t : 1, &wf, &wq, 0);
  if (!f->has_prev) { wf = 0.0; wq = 1.0; }
  f->wf = (int32_t)floor(wf * 32768.0 + 0.5);
  f->wq = 32768 - f->wf;
}

void sy_gen_host(int kind, uint64_t seed, int t0, int n, int H, int W, int K, int garbage, int seq_len,
                 int32_t* cs, int32_t* ct, int32_t* cnb) {
  static sy_luts L;
  static int built = 0;
  if (!built) { sy_build_luts(&L); built = 1; }
  int64_t plane = (int64_t)H * W;
  for (int i = 0; i < n; ++i) {
    int t = t0 + i;
    int seq_t = seq_len > 0 ? (t % seq_len) : t;
    sy_frame f;
    sy_make_frame(&f, kind, seed, H, W, t, seq_t);
    int32_t* ocs = cs + (int64_t)i * plane;
    int32_t* oct = ct + (int64_t)i * plane;
    int32_t* onb = cnb + (int64_t)i * plane * K;
    for (int y = 0; y < H; ++y)
      for (int x = 0; x < W; ++x) {
        int64_t o = (int64_t)y * W + x;
        sy_pixel(&L, &f, K, garbage, y, x, ocs + o, oct + o, onb + o, plane);
      }
  }
}

void sy_gen_energy_host(uint64_t seed, int t0, int n, int H, int W, int seq_len, uint8_t* rgb, uint16_t* prior) {
  static sy_luts L;
  static int built = 0;
  if (!built) { sy_build_luts(&L); built = 1; }
  int64_t plane = (int64_t)H * W;
  for (int i = 0; i < n; ++i) {
    int t = t0 + i;
    int seq_t = seq_len > 0 ? (t % seq_len) : t;
    sy_frame f;
    sy_make_frame(&f, SY_KIND_BLOB, seed, H, W, t, seq_t);
    for (int y = 0; y < H; ++y)
      for (int x = 0; x < W; ++x) {
        int64_t o = (int64_t)i * plane + (int64_t)y * W + x;
        sy_energy_pixel(&L, &f, y, x, rgb + 3 * o, prior + o);
      }
  }
}
