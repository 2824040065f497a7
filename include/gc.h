/* gc.h -- C ABI of the B200 grid min-cut library (libgc.so).
 *
 * Operation (§4):
 *   For each frame, the graph of P:331-357 -- one vertex per pixel, a source s and a
 *   sink t, t-links c(s,v) = cap_s (the cost of label 0) and c(v,t) = cap_t
 *   (the cost of label 1), and for every pixel p and direction k an n-link
 *   p -> p+d_k of capacity cap_nb[k] (the "pair of mutually connected directed edges"
 *   of footnote P:336-338; the two directions may differ).  The library computes the
 *   maximum s-t flow value F* (= the minimum cut capacity) and the canonical minimum
 *   cut: mask[v] = 1 iff v is reachable from s in the residual graph of a maximum
 *   flow.  "The minimum cut ... provides the MAP configuration": mask = 1 is
 *   label 1 (object, source side), mask = 0 is label 0 (background); among several
 *   minimum cuts the mask is the inclusion-minimal one, i.e. ties go to label 0
 *   (readings c1, c2).  Both outputs are unique functions of the input, so
 *   they are compared bit-exactly with the CPU oracle.
 *
 * Direction order (k, (dy,dx)):  0 E(0,+1) 1 W(0,-1) 2 S(+1,0) 3 N(-1,0)
 *                                4 SE(+1,+1) 5 NW(-1,-1) 6 SW(+1,-1) 7 NE(-1,+1);
 *   opp(k) = k ^ 1.  4-neighbour frames use k = 0..3, 8-neighbour frames k = 0..7.
 *   "Forward" directions (warm-start flow planes) are the even k: E, S[, SE, SW].
 *
 * Layout: every plane is row-major [H][W] (x fastest), int32 unless noted; a batch is
 *   n frames back to back.  No alignment beyond the element size is required.
 *
 * Ownership: all I/O buffers belong to the caller.  gc_solve_batch takes CUDA DEVICE
 *   pointers (e.g. torch tensors on the context's device); gc_solve_batch_host takes
 *   HOST pointers (pinned memory recommended) and copies through the context's
 *   staging buffers.  The context owns all scratch.  One context serves one device and
 *   one caller at a time (not thread-safe); distinct contexts may run concurrently.
 *
 * Errors: host-checkable argument errors (NULL required pointer, n/H/W <= 0 or
 *   H > max_h or W > max_w, bad neighbourhood) return GC_ERR_ARG before any launch.
 *   Capacities are checked on the device: any in-grid capacity < 0 or > GC_CAP_MAX
 *   makes that frame's flow_out = -1, its mask all 0, its stats status GC_ERR_RANGE,
 *   and the call returns GC_ERR_RANGE (other frames are still solved).  n-link entries
 *   that point off the grid are IGNORED (any value, reading c7).  If the solve needs
 *   more than max_launches x (tiles in flight) tile tasks, or runs longer than the
 *   context's wall-clock bound (GC_TIMEOUT_S, default 300 s), the unfinished frames get
 *   flow_out = -1 and the call returns GC_ERR_NOCONV.  CUDA failures return GC_ERR_CUDA; the message is
 *   available from gc_last_error().  Calls return after all work on `stream` for this
 *   call has completed.
 */
#ifndef GC_H
#define GC_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct gc_ctx gc_ctx;

typedef enum {
  GC_OK = 0,
  GC_ERR_ARG = 1,
  GC_ERR_RANGE = 2,
  GC_ERR_OOM = 3,
  GC_ERR_CUDA = 4,
  GC_ERR_NOCONV = 5
} gc_status;

#define GC_CAP_MAX ((1 << 26) - 1)

/* 0 in any field selects the default -- except `device`, where 0 is device 0.  A NULL
 * config selects every default (the current device). */
typedef struct {
  int device;            /* CUDA device ordinal (0 = device 0); < 0: the calling thread's
                            current device                                                */
  int neighborhood;      /* 4 or 8 (default 4)                                            */
  int max_h, max_w;      /* largest frame the context will accept (default 1080 x 1920)  */
  int max_batch;         /* frames solved concurrently per device pass (default: as many
                            as a scratch budget of min(8 GB, 1/16 device memory) holds) */
  int rounds_per_launch; /* push/relabel rounds inside a tile per push task (default 16) */
  int relabel_period;    /* reserved (global relabels follow Goldberg's heuristic)       */
  long long max_launches;/* watchdog: a call may run max_launches x (tiles in flight) tile
                            tasks; exceeded -> GC_ERR_NOCONV (default 1,000,000)          */
} gc_config;

/* Allocates the context and its device scratch.  *out is NULL on failure. */
gc_status gc_create(const gc_config* cfg, gc_ctx** out);

/* Frees the context and its scratch.  NULL is a no-op. */
void gc_destroy(gc_ctx* ctx);

typedef struct {
  int n, H, W;
  const int32_t* cap_s;      /* [n][H][W]   c(s->v): cost of label 0            */
  const int32_t* cap_t;      /* [n][H][W]   c(v->t): cost of label 1            */
  const int32_t* cap_nb;     /* [n][K][H][W] c(p -> p+d_k); off-grid entries ignored        */
  const int32_t* warm_flow;  /* NULL, or [n][K/2][H][W]: net flow on the forward arcs
                                (E, S[, SE, SW]) from any earlier solve (Kohli-Torr-style
                                reuse); it is clamped to the new capacities, so
                                any int32 values are accepted and the result is unchanged */
  int64_t* flow_out;         /* [n] max-flow value of the graph as given                   */
  uint8_t* mask_out;         /* [n][H][W] 1 iff reachable from s in the final residual     */
  int32_t* flow_state_out;   /* NULL, or [n][K/2][H][W]: this solve's forward-arc flows
                                (n-link flows of the final maximum preflow; 0 on off-grid
                                arcs; F = sum c(v,t) - sum max(0, -e) holds; unspecified for a
                                frame that reports GC_ERR_RANGE)                           */
  int32_t* stats_out;        /* NULL, or [n][4]: push tile tasks, global relabels, BFS relax
                                tile tasks, status (gc_status of the frame)                */
} gc_batch;

/* Device-pointer entry point.  `stream` is a cudaStream_t (NULL = legacy default). */
gc_status gc_solve_batch(gc_ctx* ctx, const gc_batch* batch, void* stream);

/* Video sequences (BASELINE config C3; Kohli-Torr-style dynamic cuts): S sequences of
 * L frames each, frame index f = j * L + t (sequence j, time t), every array laid out like
 * gc_batch's with n = S * L.  The whole set is ONE device pass: a frame slot holds a sequence
 * and, when frame t is solved, takes frame t+1 of the same sequence -- warm-started (warm != 0)
 * from the forward-arc flows frame t just exported, which the context keeps on the device
 * (clamped to the new capacities exactly as gc_batch.warm_flow is, so F and mask equal a cold
 * solve of every frame); warm == 0 runs the same schedule cold.  Results are F and the
 * canonical mask of every frame, as gc_solve_batch defines them.  Device pointers; errors as
 * gc_solve_batch (GC_ERR_ARG: S < 0, L <= 0, bad H/W, NULL required pointer). */
typedef struct {
  int S, L, H, W;
  const int32_t* cap_s;      /* [S][L][H][W]                                                 */
  const int32_t* cap_t;      /* [S][L][H][W]                                                 */
  const int32_t* cap_nb;     /* [S][L][K][H][W]                                              */
  const int32_t* warm_flow;  /* NULL, or [S][K/2][H][W]: warm start of each sequence's frame 0 */
  int64_t* flow_out;         /* [S][L]                                                       */
  uint8_t* mask_out;         /* [S][L][H][W]                                                 */
  int32_t* flow_state_out;   /* NULL, or [S][K/2][H][W]: the flows of each sequence's last
                                frame (to continue the sequences in a later call)           */
  int32_t* stats_out;        /* NULL, or [S][L][4] as gc_batch.stats_out                     */
  int warm;                  /* 1: frame t >= 1 warm-started from frame t-1; 0: all cold     */
} gc_seq_batch;
gc_status gc_solve_sequences(gc_ctx* ctx, const gc_seq_batch* batch, void* stream);

/* Host-pointer entry point: same semantics; the library copies inputs to the device and
 * results back, in chunks, on `stream`.  All pointers in *batch are host pointers. */
gc_status gc_solve_batch_host(gc_ctx* ctx, const gc_batch* batch, void* stream);

/* Per-frame digest of solved frames -- the statistics the frame-sharded multi-GPU path
 * gathers: out[i] = { flow[i], popcount(mask_i), H(mask_i), 0 }
 * with H(m) = sum over pixels p = y*W + x with m[p] != 0 of splitmix64(p + 1), mod 2^64
 * (splitmix64: z += 0x9e3779b97f4a7c15; z = (z ^ z>>30) * 0xbf58476d1ce4e5b9;
 * z = (z ^ z>>27) * 0x94d049bb133111eb; z ^ z>>31), stored as int64 bits.  flow [n] int64,
 * mask [n][H][W] uint8 and out [n][4] int64 are DEVICE pointers on the context's device.
 * GC_ERR_ARG for n < 0, H or W <= 0, or a NULL pointer with n > 0; returns after the work on
 * `stream` completed. */
gc_status gc_frame_digest(gc_ctx* ctx, int n, int H, int W, const int64_t* flow, const uint8_t* mask,
                          int64_t* out, void* stream);

/* ---- NEXT-1: the energy of PAPER.md §4 -> capacities, built inside the
 * solve's init pass (no cap arrays in HBM or over PCIe: 5 B/px of input instead of 4(2+K)).
 *
 * Colour likelihood p(C|A) of one label: a Gaussian mixture over RGB with
 * M <= GC_GMM_MAX components; lognorm[m] = log w_m - 1/2 log((2 pi)^3 det S_m) is computed on
 * the host ("only the normalization term of each Gaussian density is calculated on CPU",
 * P:584-585) by gc_gmm_prepare, prec[m] = S_m^-1 as (xx, xy, xz, yy, yz, zz). */
#define GC_GMM_MAX 4
typedef struct {
  int M, pad;
  double lognorm[GC_GMM_MAX];
  double mean[GC_GMM_MAX][3];
  double prec[GC_GMM_MAX][6];
} gc_gmm;

/* Host helper: fills *out from M weights (> 0), means [M][3] and full covariances [M][3][3]
 * (symmetric positive definite) in double precision.  GC_ERR_ARG on M outside 1..GC_GMM_MAX,
 * a non-positive weight or a covariance that is not positive definite.  No device work. */
gc_status gc_gmm_prepare(int M, const double* weights, const double* means, const double* covs, gc_gmm* out);

/* Energy parameters (per call).  For frame f, pixel v with colour C = (R,G,B) and prior code
 * u = prior[f][v]: p = clamp(u / 65535, eps, 1 - eps) (p(A=1) from the prior),
 *   c(s,v) = q(-log p(C|A=0) - log(1 - p))     (psi1 + xi1 of label 0)
 *   c(v,t) = q(-log p(C|A=1) - log p)           (psi1 + xi1 of label 1)
 * and for the n-link of direction k (distance 1, or sqrt 2 for diagonals), with the integer
 * luma I = (77 R + 150 G + 29 B + 128) >> 8 ("I_x denotes the intensity"):
 *   c_k(v) = q(lambda exp(-((I_v - I_{v+d_k}) / 255)^2 / (2 sigma^2)) / dist + kappa)
 * (psi2 + xi2; reading c5), q(x) = floor(scale x + 0.5)
 * clamped to [0, GC_CAP_MAX].  Evaluated in double precision.  n-links are symmetric. */
typedef struct {
  double lambda, sigma, kappa, eps, scale;
} gc_energy_params;

typedef struct {
  int n, H, W;
  const uint8_t* image;      /* [n][H][W][3] RGB (device)                                    */
  const uint16_t* prior;     /* [n][H][W] prior code u: p(A=1) = u / 65535 (device)          */
  const gc_gmm* gmm;         /* [n][2] colour GMMs of label 0 and label 1 (device)           */
  gc_energy_params params;
  const int32_t* warm_flow;  /* as gc_batch                                                   */
  int64_t* flow_out;         /* [n]                                                           */
  uint8_t* mask_out;         /* [n][H][W]                                                     */
  int32_t* flow_state_out;   /* NULL or [n][K/2][H][W]                                        */
  int32_t* stats_out;        /* NULL or [n][4]                                                */
  int32_t* caps_out;         /* NULL, or [n][2+K][H][W]: the capacities the solve used (cs, ct,
                                n-link planes; off-grid entries 0), for inspection / parity   */
} gc_energy_batch;

/* Solves every frame of the energy batch exactly as gc_solve_batch solves the capacities
 * defined above (same outputs, errors and semantics; GC_ERR_ARG also for NULL image / prior /
 * gmm, sigma <= 0, eps outside (0, 0.5) or scale <= 0).  Device pointers. */
gc_status gc_solve_energy(gc_ctx* ctx, const gc_energy_batch* batch, void* stream);

/* ---- NEXT-2: the prior update of PAPER.md §6 on the device.
 * For frame t: f(A_{t-1}, x) = the previous segmentation mask smoothed by a separable Gaussian
 * (P:420-424), fused with the saliency prior q(A_t = 1) by the Kalman-style estimate as printed
 * (reading c10):
 *   p(A_t = 1) = w_f f + (1 - w_f) q,  w_f = s1 / (s1 + s2 + v(t-1)),
 *   v(t) = s1 (s2 + v(t-1)) / (s1 + s2 + v(t-1))          (s1 = sigma_1^2, s2 = sigma_2^2)
 * and p = 0 in a frame-edge band.  Exact integer arithmetic on the device:
 *   R(y,x) = sum_i taps[|i|] mask(y, clamp(x+i)),  S(y,x) = sum_j taps[|j|] R(clamp(y+j), x)
 *   (replicated border), G = sum_{|i|<=radius} taps[|i|], f = S / G^2,
 *   prior(y,x) = 0 in the band, else (wf S 65535 + (4096 - wf) q G^2 + 2048 G^2) / (4096 G^2)
 *   (integer division) -- i.e. round(65535 (w_f f + (1 - w_f) q / 65535)) with w_f = wf / 4096.
 * wf comes from gc_kalman_step, taps from gc_gauss_taps (host helpers, double precision). */
#define GC_PRIOR_RMAX 16
typedef struct {
  int radius;                      /* 0..GC_PRIOR_RMAX                                        */
  int taps[GC_PRIOR_RMAX + 1];     /* taps[0..radius] >= 0, taps[0] > 0, each <= 1024           */
  int band;                        /* >= 0 px                                                 */
} gc_prior_params;

/* taps[i] = floor(1024 exp(-i^2 / (2 sigma^2)) + 0.5), i = 0..radius; GC_ERR_ARG for sigma <= 0
 * or radius outside 0..GC_PRIOR_RMAX.  Host only. */
gc_status gc_gauss_taps(double sigma, int radius, int* taps);

/* One step of the §6 recursion: *wf_q12 = floor(4096 s1 / (s1 + s2 + v_prev) + 0.5), *v_next as
 * above.  GC_ERR_ARG unless s1 > 0, s2 >= 0, v_prev >= 0.  Host only. */
gc_status gc_kalman_step(double s1, double s2, double v_prev, int* wf_q12, double* v_next);

/* n frames: mask_prev [n][H][W] uint8 (0/1; nonzero counts as 1), q [n][H][W] uint16 saliency
 * prior codes, wf [n] int32 (0..4096) -> prior_out [n][H][W] uint16 codes for gc_solve_energy.
 * Device pointers; GC_ERR_ARG for bad dims, NULL pointers or bad params. */
gc_status gc_prior_update(gc_ctx* ctx, int n, int H, int W, const uint8_t* mask_prev, const uint16_t* q,
                          const int32_t* wf, const gc_prior_params* params, uint16_t* prior_out, void* stream);

/* ---- NEXT-4: the Itti-style saliency map of PAPER.md §3 / §7.2 on the
 * device: level-0 features I = (r+g+b)/3, RG = (r-g)/I, BY = (b-(r+g)/2)/I (0 where
 * I < 0.1), M = |I - I_prev| (r, g, b = byte / 255); Gaussian pyramids (levels 0..8, [1 4 6 4 1]/16
 * separable blur with clamped border, decimation by 2 rounding up); orientation maps |G_theta * I|
 * with the four 9 x 9 filters of gc_gabor_kernels on I's levels 2..8; centre-surround maps
 * |L_c - up(L_s)| for c in {2,3,4}, s = c + {3,4} (bilinear, pixel centres); the normalisation
 * N(.) = rescale to [0,1], times (1 - m)^2 with m the mean of the local maxima (window radius 7)
 * other than the global one ("global and local [extrema]", DESIGN.md c21); each map
 * brought to level 4 by blur-decimation and summed per class (intensity, colour, orientation --
 * N of each orientation's sum first --, motion); saliency = N(mean of the four N(class)).
 * Float32 with the operation order fixed and no fused multiply-add, exact reductions: the result
 * is a deterministic function of the input (the oracle reproduces it bit for bit).
 * image / prev: [n][H][W][3] RGB (prev NULL: no motion); sal_out: NULL or [n][h4][w4] float at
 * level 4 (gc_saliency_dims); q_out: NULL or [n][H][W] uint16 = floor(65535 s + 0.5) of the
 * bilinearly upsampled saliency (a prior code for gc_prior_update).  Device pointers;
 * GC_ERR_ARG for bad dims / NULL pointers, GC_ERR_OOM if the pyramids (~88 MB per 1080p frame)
 * do not fit. */
typedef struct {
  int n, H, W;
  const uint8_t* image;
  const uint8_t* prev;
  float* sal_out;
  uint16_t* q_out;
} gc_saliency_batch;
gc_status gc_saliency(gc_ctx* ctx, const gc_saliency_batch* batch, void* stream);
/* Level-4 size: h4 = H rounded up 4 times by halving, likewise w4.  Host only. */
gc_status gc_saliency_dims(int H, int W, int* h4, int* w4);
/* The four orientation filters [4][9][9] float (theta = 0, 45, 90, 135 degrees): even Gabor,
 * sigma 2, wavelength 6, aspect 0.5, mean removed (DESIGN.md c19).  Host only. */
gc_status gc_gabor_kernels(float* out);

/* NEXT-3 (per-pixel time vs resolution): band
 * partition of every frame's tiles for the next solves on this context.  The tile rows of a
 * frame are split into `parts` horizontal bands of ceil(tile rows / parts) rows; every task of
 * band b (init group, relabel, push, closure) is queued on band b's own ring and run only by
 * the persistent CTAs with blockIdx % parts == b, so band b's state is only ever written by its
 * own CTAs except across the band border (border flow counters, requests, reach marks, halo
 * reads) -- the owner-computes schedule of a parts-GPU domain decomposition of one frame,
 * EMULATED in one kernel on one device (the bands share the device's memory; nothing here
 * spans GPUs).  Results are identical for every `parts`; profiling counts the cross-band
 * requests and task hand-offs (development counter 19).  parts = 1 (default) turns it off; 1 <= parts <=
 * GC_PARTS_MAX, else GC_ERR_ARG.  Host only. */
#define GC_PARTS_MAX 8
gc_status gc_set_partitions(gc_ctx* ctx, int parts);

/* Message for the last failing call on this context ("" if none).  Never NULL. */
const char* gc_last_error(const gc_ctx* ctx);

/* Number of kernel launches the last call issued (for the bench's gpu_launches): a solve
 * issues a clear kernel (the call's initial state), a setup kernel and one persistent k_solve
 * per chunk of frames (+ k_abort after a watchdog stop); gc_saliency its ~440 stage kernels. */
long long gc_last_launches(const gc_ctx* ctx);

/* Profiling: when enabled, the persistent kernel times every tile task (globaltimer) and
 * the host brackets every k_solve launch with CUDA events on the launching stream.
 * Task classes: 0 init, 1 bfs (seed + relax), 2 push, 3 scheduler (waiting for a task,
 * phase transitions), 4 closure, 5 export (flow_state_out).
 * Off by default (the timers add a few atomics per task). */
void gc_set_profiling(gc_ctx* ctx, int enable);
/* Fills launches[6] (k_solve launches, the same in every class), ms[6] (CTA time spent in
 * the class, averaged over the CTAs of the persistent grid, so the six add up to the
 * kernel's duration) and tiles[6] (32x32 tiles the class processed; an init task covers a
 * group of tiles), accumulated since the last
 * reset; any pointer may be NULL; resets the counters if reset != 0. */
void gc_get_profile(gc_ctx* ctx, long long* launches, double* ms, long long* tiles, int reset);
/* Device time (ms, CUDA events on the launching stream) of the k_solve launches since the
 * last reset; always measured (launches[] of gc_get_profile counts them). */
double gc_get_kernel_ms(gc_ctx* ctx, int reset);

#ifdef __cplusplus
}
#endif
#endif /* GC_H */
