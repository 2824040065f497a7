/* synth.h -- seeded synthetic INPUT generator for the grid min-cut path.
 *
 * This module is test/bench infrastructure.  It produces int32 t-link and n-link
 * capacities shaped like the paper's saliency-driven frames; it contains NONE of the
 * method's arithmetic (no flow, no cut, no labels).  Both the CPU oracle's tests and the
 * CUDA path's tests/bench draw their inputs from here, so the per-pixel functions are
 * integer-only and shared by the host build (synth_host.c) and the CUDA twin
 * (synth_cuda.cu): the two twins are bit-identical by construction.  Every floating-point
 * quantity (log-likelihoods, exp() of contrasts, Kalman weights, trajectories) is
 * evaluated ONCE on the host in double precision into integer look-up tables or
 * per-frame integer parameters (SURVEY.md §8(c) reading c11).
 *
 * Frame model:
 *   - intensity I in [0,255]: background ~100 + static low-frequency value noise +
 *     per-frame pixel noise; 1..3 moving ellipses ~200 (P:608-611 clip shape, 12 fps);
 *   - saliency q: Gaussian blob around a per-frame jittered object centre;
 *   - f(A_{t-1}): smoothed previous-frame ellipse;
 *   - prior p = w_f f + w_q q with the Sec. 6 weights as printed, x0.95,
 *     frame-edge band of 8 px -> eps;
 *   - t-links: c(s,v) = q(-ln(1-p) - ln N(I;100,30^2)),
 *                          c(v,t) = q(-ln p   - ln N(I;200,25^2));
 *   - n-links: B = q(lambda exp(-(dI/255)^2/(2 sigma^2))/dist + kappa),
 *     lambda=10, sigma=0.1, kappa=0.05 (SPEC S:447 defaults), q(x) = floor(64 x + 0.5).
 *   Off-grid n-link entries are filled with hash garbage when requested, because the
 *   boundary contract says they are ignored.
 *
 * Direction order: k: 0 E(0,+1) 1 W(0,-1) 2 S(+1,0) 3 N(-1,0)
 *                                   4 SE(+1,+1) 5 NW(-1,-1) 6 SW(+1,-1) 7 NE(-1,+1).
 */
#ifndef SYNTH_H
#define SYNTH_H
#include <stdint.h>

#ifdef __CUDACC__
#define SY_HD __host__ __device__ __forceinline__
#else
#define SY_HD static inline
#endif

#define SY_CAP_MAX ((1 << 26) - 1)
#define SY_NP 1024   /* prior quantisation steps; index SY_NP = edge-band eps */
#define SY_NQ 1024   /* saliency Gaussian LUT: s = d^2/(2 sigma^2) in steps of 1/64 */
#define SY_NF 4096   /* smoothed-mask LUT over normalised radius^2 in steps of 1/256 */
#define SY_MAXOBJ 3

enum { SY_KIND_BLOB = 0, SY_KIND_SERPENTINE = 1, SY_KIND_RANDOM = 2 };

typedef struct {
  int32_t tl0_p[SY_NP + 1]; /* q(-ln(1-p)) : cost of label 0 from the prior */
  int32_t tl1_p[SY_NP + 1]; /* q(-ln p)    : cost of label 1 from the prior */
  int32_t tl0_I[256];       /* q(-ln N(I;100,30^2)) background likelihood */
  int32_t tl1_I[256];       /* q(-ln N(I;200,25^2)) object likelihood */
  int32_t nl[2][256];       /* n-link cap by |dI|, [0]=axial dist 1, [1]=diagonal dist sqrt2 */
  int32_t q_lut[SY_NQ];     /* 65535*exp(-s) */
  int32_t f_lut[SY_NF];     /* 65535/(1+exp(8(rho-1))) */
} sy_luts;

typedef struct {
  int32_t kind;
  int32_t H, W;
  int32_t nobj;
  int32_t cy[SY_MAXOBJ], cx[SY_MAXOBJ];   /* object centres, 1/16 px */
  int32_t ry[SY_MAXOBJ], rx[SY_MAXOBJ];   /* radii, px (>=2) */
  int32_t py[SY_MAXOBJ], px[SY_MAXOBJ];   /* previous-frame centres, 1/16 px */
  int32_t qy, qx;                         /* jittered saliency centre, px */
  int32_t q_scale;                        /* LUT index = d2 * q_scale >> 16 */
  int32_t wf, wq;                         /* prior weights, fixed point, wf+wq = 1<<15 */
  int32_t has_prev;                       /* 0 on the first frame: prior = q only */
  /* serpentine (adversarial) parameters */
  int32_t lane;                           /* lane width (px) */
  int32_t big;                            /* strong capacity (2^20) */
  /* random kind parameters */
  int32_t rmax_t, rmax_n;                 /* t-link / n-link caps uniform in [0, rmax] */
  int32_t rzero_pct;                      /* % of n-links forced to 0 */
  uint32_t frame;                         /* absolute frame index (hash input) */
  uint32_t pad_;
  uint64_t seed;
} sy_frame;

SY_HD uint64_t sy_mix64(uint64_t z) {
  z += 0x9e3779b97f4a7c15ULL;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

SY_HD uint64_t sy_hash(uint64_t seed, uint32_t frame, int32_t y, int32_t x, uint32_t stream) {
  uint64_t h = sy_mix64(seed ^ ((uint64_t)stream << 48));
  h = sy_mix64(h ^ (uint64_t)frame);
  h = sy_mix64(h ^ (((uint64_t)(uint32_t)y << 32) | (uint64_t)(uint32_t)x));
  return h;
}

SY_HD int sy_dy(int k) { return (k == 2 || k == 4 || k == 6) ? 1 : ((k == 3 || k == 5 || k == 7) ? -1 : 0); }
SY_HD int sy_dx(int k) { return (k == 0 || k == 4 || k == 7) ? 1 : ((k == 1 || k == 5 || k == 6) ? -1 : 0); }

/* ---- blob frames ------------------------------------------------------------ */

SY_HD int sy_inside(const sy_frame* f, const int32_t* cy, const int32_t* cx, int y, int x) {
  for (int j = 0; j < f->nobj; ++j) {
    int64_t dy = (int64_t)y * 16 + 8 - cy[j];
    int64_t dx = (int64_t)x * 16 + 8 - cx[j];
    int64_t ry = f->ry[j], rx = f->rx[j];
    int64_t lhs = dy * dy * rx * rx + dx * dx * ry * ry;
    int64_t r = 16 * ry * rx;
    if (lhs <= r * r) return 1;
  }
  return 0;
}

SY_HD int sy_intensity(const sy_frame* f, int y, int x) {
  uint64_t hn = sy_hash(f->seed, f->frame, y, x, 2);
  int noise = (int)(hn % 11u) - 5;
  if (sy_inside(f, f->cy, f->cx, y, x)) {
    int v = 200 + noise;
    return v < 0 ? 0 : (v > 255 ? 255 : v);
  }
  /* static value noise on a 16-px lattice, bilinear, corner values in [0,40] */
  int gy = y >> 4, gx = x >> 4, fy = y & 15, fx = x & 15;
  int c00 = (int)(sy_hash(f->seed, 0u, gy, gx, 1) % 41u);
  int c01 = (int)(sy_hash(f->seed, 0u, gy, gx + 1, 1) % 41u);
  int c10 = (int)(sy_hash(f->seed, 0u, gy + 1, gx, 1) % 41u);
  int c11 = (int)(sy_hash(f->seed, 0u, gy + 1, gx + 1, 1) % 41u);
  int vn = (c00 * (16 - fy) * (16 - fx) + c01 * (16 - fy) * fx + c10 * fy * (16 - fx) + c11 * fy * fx) >> 8;
  int v = 80 + vn + noise;
  return v < 0 ? 0 : (v > 255 ? 255 : v);
}

/* prior index in [0, SY_NP] (SY_NP = edge band) */
SY_HD int sy_prior_index(const sy_luts* L, const sy_frame* f, int y, int x) {
  if (y < 8 || x < 8 || y >= f->H - 8 || x >= f->W - 8) return SY_NP;
  int64_t dy = y - f->qy, dx = x - f->qx;
  int64_t qi = ((dy * dy + dx * dx) * (int64_t)f->q_scale) >> 16;
  int32_t q = L->q_lut[qi < SY_NQ - 1 ? qi : SY_NQ - 1];
  int32_t fv = 0;
  if (f->has_prev) {
    for (int j = 0; j < f->nobj; ++j) {
      int64_t ddy = (int64_t)y * 16 + 8 - f->py[j];
      int64_t ddx = (int64_t)x * 16 + 8 - f->px[j];
      int64_t ry = f->ry[j], rx = f->rx[j];
      int64_t num = (ddy * ddy * rx * rx + ddx * ddx * ry * ry) * 256;
      int64_t den = (16 * ry * rx) * (16 * ry * rx);
      int64_t ri = num / den;
      int32_t v = L->f_lut[ri < SY_NF - 1 ? ri : SY_NF - 1];
      if (v > fv) fv = v;
    }
  } else {
    fv = q;
  }
  int64_t p16 = ((int64_t)f->wf * fv + (int64_t)f->wq * q) >> 15; /* [0,65535] */
  int pi = (int)((p16 * SY_NP) >> 16);
  return pi < SY_NP - 1 ? pi : SY_NP - 1;
}

SY_HD int32_t sy_garbage(const sy_frame* f, int y, int x, int k) {
  return (int32_t)(uint32_t)sy_hash(f->seed, f->frame, y, x, 16u + (uint32_t)k);
}

/* ---- serpentine (adversarial, C5) ---------------------------------------------
 * Horizontal lanes of width `lane` separated by 1-px wall rows.  Wall pixels carry no
 * n-links except in the gap (alternating ends), so the only s-t connection snakes
 * through every lane.  In-lane n-links are bimodal {1, big} by hash ("high
 * contrast"); cs = big on the first 64 columns of lane 0, ct = big on the last 64
 * columns of the last lane (at the far end), 0..3 noise t-links everywhere.          */
SY_HD int sy_serp_is_wall(const sy_frame* f, int y, int x) {
  int period = f->lane + 1;
  int r = y % period;
  if (r != f->lane) return 0;
  int wi = y / period;                 /* wall index below lane wi */
  int gap_right = (wi % 2) == 0;
  if (gap_right) return x < f->W - f->lane;
  return x >= f->lane;
}

SY_HD int32_t sy_serp_nlink(const sy_frame* f, int y, int x, int k) {
  int y2 = y + sy_dy(k), x2 = x + sy_dx(k);
  if (sy_serp_is_wall(f, y, x) || sy_serp_is_wall(f, y2, x2)) return 0;
  /* symmetric: hash the unordered pair */
  int ya = y, xa = x, yb = y2, xb = x2;
  if (ya > yb || (ya == yb && xa > xb)) { ya = y2; xa = x2; yb = y; xb = x; }
  uint64_t h = sy_hash(f->seed, f->frame, ya * 4 + (yb - ya + 1), xa * 4 + (xb - xa + 1), 7);
  return (h & 7u) == 0 ? 1 : f->big;
}

SY_HD void sy_serp_tlinks(const sy_frame* f, int y, int x, int32_t* cs, int32_t* ct) {
  uint64_t h = sy_hash(f->seed, f->frame, y, x, 8);
  int32_t ns = (int32_t)(h & 3u), nt = (int32_t)((h >> 2) & 3u);
  int period = f->lane + 1;
  int lane_i = y / period;
  int is_wall = (y % period) == f->lane;
  if (!is_wall && lane_i == 0 && x < 64) ns += f->big;
  int last = (f->H - 1) / period;
  int far_right = (last % 2) == 0; /* lane 0 flows left->right, so even lanes end at the right */
  if (!is_wall && lane_i == last && (far_right ? (x >= f->W - 64) : (x < 64))) nt += f->big;
  *cs = ns;
  *ct = nt;
}

/* ---- random (stress) -------------------------------------------------------------- */
SY_HD void sy_rand_tlinks(const sy_frame* f, int y, int x, int32_t* cs, int32_t* ct) {
  uint64_t h = sy_hash(f->seed, f->frame, y, x, 9);
  *cs = (int32_t)((h & 0xffffffffu) % (uint32_t)(f->rmax_t + 1));
  *ct = (int32_t)((h >> 32) % (uint32_t)(f->rmax_t + 1));
}
SY_HD int32_t sy_rand_nlink(const sy_frame* f, int y, int x, int k) {
  uint64_t h = sy_hash(f->seed, f->frame, y, x, 24u + (uint32_t)k);
  if ((int)((h >> 40) % 100u) < f->rzero_pct) return 0;
  return (int32_t)((h & 0xffffffffu) % (uint32_t)(f->rmax_n + 1));
}

/* ---- one pixel of one frame: all outputs ----------------------------------------- */
/* cnb points at plane 0 of this pixel; plane stride = H*W. */
SY_HD void sy_pixel(const sy_luts* L, const sy_frame* f, int K, int garbage, int y, int x,
                    int32_t* cs, int32_t* ct, int32_t* cnb, int64_t plane) {
  if (f->kind == SY_KIND_BLOB) {
    int I = sy_intensity(f, y, x);
    int pi = sy_prior_index(L, f, y, x);
    int64_t a = (int64_t)L->tl0_p[pi] + L->tl0_I[I];
    int64_t b = (int64_t)L->tl1_p[pi] + L->tl1_I[I];
    *cs = (int32_t)(a > SY_CAP_MAX ? SY_CAP_MAX : a);
    *ct = (int32_t)(b > SY_CAP_MAX ? SY_CAP_MAX : b);
    for (int k = 0; k < K; ++k) {
      int y2 = y + sy_dy(k), x2 = x + sy_dx(k);
      int32_t c;
      if (y2 < 0 || y2 >= f->H || x2 < 0 || x2 >= f->W) {
        c = garbage ? sy_garbage(f, y, x, k) : 0;
      } else {
        int I2 = sy_intensity(f, y2, x2);
        int d = I > I2 ? I - I2 : I2 - I;
        c = L->nl[k >= 4][d];
      }
      cnb[(int64_t)k * plane] = c;
    }
  } else if (f->kind == SY_KIND_SERPENTINE) {
    sy_serp_tlinks(f, y, x, cs, ct);
    for (int k = 0; k < K; ++k) {
      int y2 = y + sy_dy(k), x2 = x + sy_dx(k);
      int32_t c;
      if (y2 < 0 || y2 >= f->H || x2 < 0 || x2 >= f->W) c = garbage ? sy_garbage(f, y, x, k) : 0;
      else c = sy_serp_nlink(f, y, x, k);
      cnb[(int64_t)k * plane] = c;
    }
  } else {
    sy_rand_tlinks(f, y, x, cs, ct);
    for (int k = 0; k < K; ++k) {
      int y2 = y + sy_dy(k), x2 = x + sy_dx(k);
      int32_t c;
      if (y2 < 0 || y2 >= f->H || x2 < 0 || x2 >= f->W) c = garbage ? sy_garbage(f, y, x, k) : 0;
      else c = sy_rand_nlink(f, y, x, k);
      cnb[(int64_t)k * plane] = c;
    }
  }
}

/* ---- energy inputs (NEXT-1, gc_solve_energy): the same blob frame as RGB + prior code --------
 * RGB = the frame intensity I (sy_intensity) plus per-channel hash noise in [-4, 4]; prior code
 * u = round(0.95 (i + 0.5) / SY_NP x 65535) of the frame's prior index i (the value the cap
 * generator's t-link LUT uses), 0 in the frame-edge band.  Integer only.          */
SY_HD void sy_energy_pixel(const sy_luts* L, const sy_frame* f, int y, int x, uint8_t* rgb, uint16_t* prior) {
  int I = sy_intensity(f, y, x);
  uint64_t h = sy_hash(f->seed, f->frame, y, x, 40);
  for (int c = 0; c < 3; ++c) {
    int v = I + (int)((h >> (8 * c)) % 9u) - 4;
    rgb[c] = (uint8_t)(v < 0 ? 0 : (v > 255 ? 255 : v));
  }
  int pi = sy_prior_index(L, f, y, x);
  *prior = pi >= SY_NP ? (uint16_t)0 : (uint16_t)(((int64_t)(2 * pi + 1) * 62258 + SY_NP) / (2 * SY_NP));
}

#ifdef __cplusplus
extern "C" {
#endif
/* host API (synth_host.c) */
void sy_build_luts(sy_luts* L);
void sy_make_frame(sy_frame* f, int kind, uint64_t seed, int H, int W, int t, int seq_t);
void sy_kalman_weights(int seq_t, double* wf, double* wq, double* var_out);
void sy_gen_host(int kind, uint64_t seed, int t0, int n, int H, int W, int K, int garbage, int seq_len,
                 int32_t* cs, int32_t* ct, int32_t* cnb);
void sy_set_random_params(int rmax_t, int rmax_n, int rzero_pct);
void sy_set_serp_params(int lane, int big);
void sy_gen_energy_host(uint64_t seed, int t0, int n, int H, int W, int seq_len, uint8_t* rgb, uint16_t* prior);
int sy_gen_energy_cuda(uint64_t seed, int t0, int n, int H, int W, int seq_len, uint8_t* rgb, uint16_t* prior,
                       void* stream);
/* CUDA twin (synth_cuda.cu): device pointers, returns 0 on success */
int sy_gen_cuda(int kind, uint64_t seed, int t0, int n, int H, int W, int K, int garbage, int seq_len,
                int32_t* cs, int32_t* ct, int32_t* cnb, void* stream);
#ifdef __cplusplus
}
#endif

#endif
