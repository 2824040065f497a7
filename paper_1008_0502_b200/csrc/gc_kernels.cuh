// gc_kernels.cuh -- sm_100a kernels of the grid min-cut hot path.
//
// Algorithm: push-relabel (Goldberg-Tarjan) on the pixel grid graph of P:331-357, run as
// asynchronous 32x32-tile region discharges, with exact global relabels (BFS from the sink)
// as the termination certificate, and the canonical mask taken as the residual closure of
// the excess nodes.  The paper's GPU solver is "CUDA Cuts";
// this is a fresh B200 design, not a translation of it.  This header holds the tile-level
// building blocks; gc_phases.cuh holds the task bodies and the persistent scheduler.
//
// State (tile-major, 32x32 tiles, frame padded to whole tiles):
//   fl [slot][tile][1024] u16  bit k: r_k > 0 (arc open), bit 8: e > 0, bit 9: e < 0.
//                              Everything the BFS and closure phases need (2 B/px).
//   h  [slot][tile][1024]      height / distance label (HINF = cannot reach the sink)
//   e  [slot][tile][1024]      signed net excess e = cs - ct + inflow - outflow      } only for
//   r  [slot][k][tile][1024]   residual capacity of arc v -> v + d_k                 } "materialised"
//                              tiles (mat = 1): a tile's e, r are computed from the caps
//                              (+ warm flows) the first time a push touches it, so tiles
//                              the push phase never visits are never written.
//   hedge [slot][tile][4][32]  copy of the tile's border heights (top, bottom, left, right)
//   sent/got [slot][tile][k][64] cumulative flow pushed INTO the tile across its border, by
//                              arc direction and receiver edge slot: `sent` written only by
//                              the sending tile, `got` only by the receiver (no atomics)
//   reach [slot][tile][k][64]  min-cut reach marks arriving across the border (closure epoch)
// A tile is processed by at most one CTA at a time (gc_phases.cuh); all mutable state is
// read through L2 (the library is compiled with -dlcm=cg), the caps through the read-only
// path.
#pragma once
#include <cuda.h>  // CUtensorMap (the TMA descriptors of the init stream)
#include <cuda_runtime.h>
#include <stdint.h>

namespace gcb {

constexpr int TS = 32;       // tile side
constexpr int TPX = 1024;    // pixels per tile
constexpr int NTH = 256;     // threads per CTA; thread t owns pixels (t/32 + 8j, t%32), j<4
constexpr int HINF = 0x3fffffff;
constexpr int CAPMAX = (1 << 26) - 1;
constexpr int HS = 34;       // halo'd height tile side
constexpr int FL_POS = 1 << 8;
constexpr int FL_NEG = 1 << 9;

__host__ __device__ constexpr int DYk(int k) {
  return (k == 2 || k == 4 || k == 6) ? 1 : ((k == 3 || k == 5 || k == 7) ? -1 : 0);
}
__host__ __device__ constexpr int DXk(int k) {
  return (k == 0 || k == 4 || k == 7) ? 1 : ((k == 1 || k == 5 || k == 6) ? -1 : 0);
}

struct Dev {
  int H, W, TY, TX, T, nslot;
  int initg;  // tiles per init task
  int bulkg;  // tiles per seed / closure-seed task (1, 2, 4 or 8)
  int hmax;  // relabel cap: heights >= hmax are unreachable (HINF)
  int32_t* e;
  int32_t* h;
  int32_t* r;
  uint16_t* fl;
  int32_t* hedge;
  uint32_t* sent;   // [NS][K][64] cumulative flow pushed INTO the tile across its border, by
                    //             arc direction and receiver edge slot (written by the sender)
  uint32_t* got;    // [NS][K][64] cumulative flow the tile has absorbed from `sent` (receiver)
  uint8_t* reach;
  long long* neg0;  // [NS] the tile's share of sumneg: sum max(0,-e) as initialised, updated
                    //      by each closure seed of a materialised tile
  int32_t* tsrc;    // [NS]   uniform source tile: every in-frame pixel has e > 0 (all in the
                    //        closure; the init pass wrote its mask bytes = 1)
  int32_t* tss;     // [NS]   global relabel (fbe) in which the seed of this uniform source tile
                    //        was skipped: its stored h / hedge are stale, read as HINF, until a
                    //        relax or push task of that relabel writes them (and clears it)
  int32_t* tmk;     // [NS]   epoch of the closure attempt in which the tile's mask bytes got a
                    //        1 beyond its excess pixels (rewritten by the next attempt)
  int32_t* mat;     // [NS]   e, r of the tile are materialised
  int32_t* tact;    // [NS]   tile has an active node (e > 0, h < HINF)
  int32_t* flag;    // [NS]   tile is in the first task set of the next phase (seed -> BFS, cseed -> closure)
  int32_t* recv1;   // [NS]   tile has inbound flow not yet absorbed
  int32_t* treq;    // [NS]   requests for the tile in the running phase (> 0: queued or running)
  int32_t* tuni;    // [NS]   uniform sink tile: every in-frame pixel has e < 0 and h = 1 (h is not
                    //        stored; hedge is); such a tile is neither seeded nor relaxed
  int32_t* tfix;    // [NS]   a BFS relax of the tile cannot change it (every pixel with an
                    //        open arc has h = 1)
  int32_t* tph;     // [NS]   push-phase id of the tile's last push task
  int32_t* tminh;   // [NS]   lowest height of an active pixel of the tile (HINF if none)
  int32_t* tsk;     // [NS]   global relabel (fbe) in which the tile's seed was skipped (its
                    //        border heights, all 1 in frame, are final for that relabel)
  // per frame slot (state machine): zero-initialised by one memset
  const int32_t** scs;  // [nslot] the slot's frame's cap planes: c(s,v) [H][W], c(v,t) [H][W] and
  const int32_t** sct;  //         the n-links [K][H][W] -- the caller's arrays, or (energy mode)
  const int32_t** snb;  //         the slot's cap buffer the init pass builds them into
  int32_t* capbuf;      // energy mode: [nslot][2+K][H][W] capacities built from the energy, or
  int capbyframe;       //   (capbyframe) the caller's caps_out [n][2+K][H][W], indexed by frame
  const int32_t** swf;  // [nslot] warm-start flows of the slot's frame ([K/2][H][W]) or NULL
  int32_t** sfs;        // [nslot] where the slot's frame exports its flows ([K/2][H][W]) or NULL
  int32_t* fbuf;        // sequence mode, warm: [nslot][2][K/2][H][W] ping-pong flow buffers (frame
                        // t exports into buffer t & 1, frame t+1 starts from it)
  int32_t* fmode;   // [nslot] M_INIT, M_SEED, M_BFS, M_PUSH, M_CSEED, M_CLOS, M_IDLE
  int32_t* sfr;     // [nslot] batch frame index held by the slot
  int32_t* fout;    // [nslot] tasks of the running phase queued or running
  int32_t* gctr;    // [4] next frame to start, frames finished, range-error frames, -
  int32_t* ferr;    // [nslot] capacity out of range
  int32_t* fph;     // [nslot] global relabels so far (push-phase id)
  int32_t* fvis;    // [nslot] push tasks in the current push phase
  int32_t* fprog;   // [nslot] value of fvis after the last push task that made progress
  int32_t* cep;     // [nslot] closure attempts so far (epoch = cep % 255 + 1)
  int32_t* cfail;   // [nslot] the running closure attempt reached a node with e < 0
  int32_t* fdrain;  // [nslot] the running push phase drains (no new requests)
  int32_t* fhmin;   // [nslot] lowest height of an active pixel seen in the running push phase
  int32_t* fbe;     // [nslot] global relabels started (BFS epoch)
  int32_t* fcap;    // [nslot] height cap of the running push phase (higher pixels are frozen)
  int32_t* fbnd;    // [nslot] distance bound of the running global relabel (HINF: exact)
  int32_t* sep;     // [nslot] closure attempts of the slot in this call (all its frames): the
                    //         reach-mark epoch is sep % 255 + 1; the slot's marks are cleared
                    //         when it wraps, so a mark never aliases an earlier attempt's
  int32_t* fflag;   // [nslot] a task of the running phase flagged a tile for the next one
  int32_t* fstat;   // [nslot][4] push tasks, global relabels, BFS relax tasks, -
  unsigned long long* frel;   // [nslot] relabel operations in the current push phase
  unsigned long long* sumct;  // [nslot]
  unsigned long long* sumneg; // [nslot]
  // work queues: rings of task entries, ticketed by two 64-bit counters each.
  // q holds the latency-critical tasks (relabel, push, closure: dependency chains), qi the
  // init groups (HBM streaming); an idle CTA serves q first.
  uint32_t* q;
  uint32_t qmask;
  unsigned long long* qhead;   // qhead, qtail adjacent and 16-byte aligned (read as one)
  unsigned long long* qtail;
  uint32_t* qi;
  uint32_t qimask;
  unsigned long long* qihead;  // likewise
  unsigned long long* qitail;
  int32_t* done;    // [0] every frame finished, [1] aborted
  unsigned long long* ntask;  // tasks executed (watchdog)
  // NEXT-3 band partition (gc_set_partitions): a frame's tile rows split into nparts bands of
  // prow rows; band b's tasks go to ring b (q / qi + b x capacity, head / tail pairs at
  // qhead + 2b, qihead + 2b) and run only on CTAs with blockIdx % nparts == b -- the owner-
  // computes schedule of an nparts-GPU domain decomposition, emulated in one kernel.  1: off.
  int nparts;
  int prow;
  const volatile int32_t* hostabort;  // mapped host word: the host asks the kernel to stop
  unsigned long long* ptiles;  // [6] tasks per class (profiling only, else NULL)
  unsigned long long* pns;     // [6] ns per class summed over CTAs (profiling only)
  unsigned long long* pdbg;    // [16] development counters (profiling only)
  // development trace (profiling level 2 only, else NULL): one record of 4 u64 per task --
  // globaltimer start, duration ns, (md << 56 | gcnt << 48 | cta << 32 | frame), tile
  unsigned long long* trace;
  unsigned long long* trace_n;
  unsigned long long trace_cap;
};

enum { M_INIT = 0, M_SEED = 1, M_BFS = 2, M_PUSH = 3, M_CSEED = 4, M_CLOS = 5, M_IDLE = 8 };

// NEXT-1 energy mode (gc_solve_energy): colour GMM of one label, as include/gc.h's gc_gmm.
constexpr int GMM_MAX = 4;
struct Gmm {
  int M, pad_;
  double lognorm[GMM_MAX];  // log w_m - 1/2 log((2 pi)^3 det S_m)   (computed on the host)
  double mean[GMM_MAX][3];
  double prec[GMM_MAX][6];  // S_m^-1: xx, xy, xz, yy, yz, zz
};

struct IO {
  const int32_t* cs;
  const int32_t* ct;
  const int32_t* nb;
  const int32_t* wf;
  int64_t* flow;
  uint8_t* mask;
  int32_t* fstate;
  int32_t* stats;
  // energy mode (NULL img: the caller gives the caps): the init pass builds every frame's caps
  // from its RGB image, prior and colour GMMs into the slot's cap buffer
  const uint8_t* img;     // [n][H][W][3]
  const uint16_t* prior;  // [n][H][W]: p(A=1) = prior / 65535
  const Gmm* gmm;         // [n][2]: label 0 (background), label 1 (object)
  const int32_t* nlut;    // [2][256]: quantised n-link cap by |dI| (axial, diagonal), built per call
  double eps, scale;      // prior clamp, quantisation scale
};

__device__ __forceinline__ size_t NS(const Dev& d) { return (size_t)d.nslot * d.T; }

// Checked builds (make CHECKS=1; compute-sanitizer is not available on the GPU pool): device
// invariants that guard every index the scheduler derives from shared state.  A failed check
// records its source line in gctr[3] (>= 2) and stops the kernel through the abort flag; the
// host returns GC_ERR_CUDA "device check failed at line N".  Compiled out otherwise.
#ifdef GC_CHECKS
#define GC_CHECK(d, cond)                                              \
  do {                                                                 \
    if (!(cond)) {                                                     \
      atomicCAS(&(d).gctr[3], 0, 2 + __LINE__);                        \
      *(volatile int*)&(d).done[1] = 1;                                \
    }                                                                  \
  } while (0)
#else
#define GC_CHECK(d, cond) \
  do {                    \
  } while (0)
#endif
__device__ __forceinline__ int32_t* Rp(const Dev& d, int K, size_t gt, int k) {
  const size_t s = (unsigned)gt / (unsigned)d.T, tile = gt - s * d.T;
  return d.r + ((s * K + k) * d.T + tile) * TPX;
}
__device__ __forceinline__ uint32_t* SENTp(const Dev& d, int K, size_t gt, int k) { return d.sent + (gt * K + k) * 64; }
__device__ __forceinline__ uint32_t* GOTp(const Dev& d, int K, size_t gt, int k) { return d.got + (gt * K + k) * 64; }

// Does arc (iy,ix) -> (iy,ix)+d_k leave the tile?
__device__ __forceinline__ bool crosses(int k, int iy, int ix) {
  const int y2 = iy + DYk(k), x2 = ix + DXk(k);
  return (unsigned)y2 >= 32u || (unsigned)x2 >= 32u;
}

// Receiver-side inbox slot of the arc arriving at receiver pixel (uy,ux) along direction k,
// for arcs whose sender u - d_k lies in another tile.  Unique per (k, receiver pixel).
__device__ __forceinline__ int recv_slot(int k, int uy, int ux) {
  switch (k) {
    case 0: return uy;                        // E arrives at the left column
    case 1: return uy;                        // W arrives at the right column
    case 2: return ux;                        // S arrives at the top row
    case 3: return ux;                        // N arrives at the bottom row
    case 4: return uy == 0 ? ux : 32 + uy;    // SE: top row, else left column
    case 5: return uy == 31 ? ux : 32 + uy;   // NW: bottom row, else right column
    case 6: return uy == 0 ? ux : 32 + uy;    // SW: top row, else right column
    default: return uy == 31 ? ux : 32 + uy;  // NE: bottom row, else left column
  }
}

// Sender-side view of the receiver slots: the tile (offset dy, dx from the sending tile)
// that owns slot `sl` of direction k (inverse of recv_slot; unused slots are never written).
__device__ __forceinline__ void recv_tile_offset(int k, int sl, int& dy, int& dx) {
  switch (k) {
    case 0: dy = 0; dx = 1; break;                                           // E
    case 1: dy = 0; dx = -1; break;                                          // W
    case 2: dy = 1; dx = 0; break;                                           // S
    case 3: dy = -1; dx = 0; break;                                          // N
    case 4: if (sl < 32) { dy = 1; dx = sl == 0 ? 1 : 0; } else { dy = 0; dx = 1; } break;     // SE
    case 5: if (sl < 32) { dy = -1; dx = sl == 31 ? -1 : 0; } else { dy = 0; dx = -1; } break; // NW
    case 6: if (sl < 32) { dy = 1; dx = sl == 31 ? -1 : 0; } else { dy = 0; dx = -1; } break;  // SW
    default: if (sl < 32) { dy = -1; dx = sl == 0 ? 1 : 0; } else { dy = 0; dx = 1; } break;   // NE
  }
}

// Receiver pixel (in the receiver tile) of slot `sl` of direction k (inverse of recv_slot).
__device__ __forceinline__ void recv_pixel(int k, int sl, int& uy, int& ux) {
  switch (k) {
    case 0: uy = sl; ux = 0; break;
    case 1: uy = sl; ux = 31; break;
    case 2: uy = 0; ux = sl; break;
    case 3: uy = 31; ux = sl; break;
    case 4: if (sl < 32) { uy = 0; ux = sl; } else { uy = sl - 32; ux = 0; } break;
    case 5: if (sl < 32) { uy = 31; ux = sl; } else { uy = sl - 32; ux = 31; } break;
    case 6: if (sl < 32) { uy = 0; ux = sl; } else { uy = sl - 32; ux = 31; } break;
    default: if (sl < 32) { uy = 31; ux = sl; } else { uy = sl - 32; ux = 0; } break;
  }
}

__device__ __forceinline__ int hidx(int iy, int ix) { return (iy + 1) * HS + (ix + 1); }
__device__ __forceinline__ bool on_border(int iy, int ix) { return iy == 0 || iy == 31 || ix == 0 || ix == 31; }

// Load the 34x34 halo ring of heights from the neighbours' border copies (HINF off-frame, and
// HINF for a neighbour whose seed was skipped in relabel `ep` as a uniform source tile and
// that no task has relabelled since: its stored copy is stale).
__device__ __forceinline__ void load_halo(const Dev& d, int s, int ty, int tx, int* hs, int t, int ep) {
  if (t < 128) {
    const int side = t >> 5, i = t & 31;
    int nty = ty, ntx = tx, esd, pos;
    if (side == 0) { nty = ty - 1; esd = 1; pos = hidx(-1, i); }
    else if (side == 1) { nty = ty + 1; esd = 0; pos = hidx(32, i); }
    else if (side == 2) { ntx = tx - 1; esd = 3; pos = hidx(i, -1); }
    else { ntx = tx + 1; esd = 2; pos = hidx(i, 32); }
    int v = HINF;
    if (nty >= 0 && nty < d.TY && ntx >= 0 && ntx < d.TX) {
      const size_t n = (size_t)s * d.T + nty * d.TX + ntx;
      const int hv = d.hedge[(n * 4 + esd) * 32 + i];
      v = __ldcg(d.tss + n) == ep ? HINF : hv;
    }
    hs[pos] = v;
  } else if (t < 132) {
    const int c = t - 128;
    const int dy = (c < 2) ? -1 : 1, dx = (c & 1) ? 1 : -1;
    const int nty = ty + dy, ntx = tx + dx;
    int v = HINF;
    if (nty >= 0 && nty < d.TY && ntx >= 0 && ntx < d.TX) {
      const size_t n = (size_t)s * d.T + nty * d.TX + ntx;
      const int hv = d.hedge[(n * 4 + (dy < 0 ? 1 : 0)) * 32 + (dx < 0 ? 31 : 0)];
      v = __ldcg(d.tss + n) == ep ? HINF : hv;
    }
    hs[hidx(dy < 0 ? -1 : 32, dx < 0 ? -1 : 32)] = v;
  }
}

// Halo from the neighbours selected by `sides` (side bits as side_bit: 0 N, 1 S, 2 W, 3 E,
// 4 NW, 5 NE, 6 SW, 7 SE); INF elsewhere.
__device__ __forceinline__ void load_halo_sides(const Dev& d, int s, int ty, int tx, int* hs, int t, int sides) {
  if (t < 128) {
    const int side = t >> 5, i = t & 31;
    int nty = ty, ntx = tx, esd, pos, bit;
    if (side == 0) { nty = ty - 1; esd = 1; pos = hidx(-1, i); bit = 0; }
    else if (side == 1) { nty = ty + 1; esd = 0; pos = hidx(32, i); bit = 1; }
    else if (side == 2) { ntx = tx - 1; esd = 3; pos = hidx(i, -1); bit = 2; }
    else { ntx = tx + 1; esd = 2; pos = hidx(i, 32); bit = 3; }
    int v = HINF;
    if (((sides >> bit) & 1) && nty >= 0 && nty < d.TY && ntx >= 0 && ntx < d.TX)
      v = d.hedge[(((size_t)s * d.T + nty * d.TX + ntx) * 4 + esd) * 32 + i];
    hs[pos] = v;
  } else if (t < 132) {
    const int c = t - 128;
    const int dy = (c < 2) ? -1 : 1, dx = (c & 1) ? 1 : -1;
    const int bit = dy < 0 ? (dx < 0 ? 4 : 5) : (dx < 0 ? 6 : 7);
    const int nty = ty + dy, ntx = tx + dx;
    int v = HINF;
    if (((sides >> bit) & 1) && nty >= 0 && nty < d.TY && ntx >= 0 && ntx < d.TX)
      v = d.hedge[(((size_t)s * d.T + nty * d.TX + ntx) * 4 + (dy < 0 ? 1 : 0)) * 32 + (dx < 0 ? 31 : 0)];
    hs[hidx(dy < 0 ? -1 : 32, dx < 0 ? -1 : 32)] = v;
  }
}

// fl words of the 34x34 halo ring (the neighbours' border pixels; 0 off-frame), hidx layout.
__device__ __forceinline__ void load_fl_halo(const Dev& d, int s, int ty, int tx, uint16_t* flh, int t) {
  if (t < 128) {
    const int side = t >> 5, i = t & 31;
    int nty = ty, ntx = tx, py, px, pos;
    if (side == 0) { nty = ty - 1; py = 31; px = i; pos = hidx(-1, i); }
    else if (side == 1) { nty = ty + 1; py = 0; px = i; pos = hidx(32, i); }
    else if (side == 2) { ntx = tx - 1; py = i; px = 31; pos = hidx(i, -1); }
    else { ntx = tx + 1; py = i; px = 0; pos = hidx(i, 32); }
    uint16_t v = 0;
    if (nty >= 0 && nty < d.TY && ntx >= 0 && ntx < d.TX)
      v = d.fl[((size_t)s * d.T + nty * d.TX + ntx) * TPX + py * TS + px];
    flh[pos] = v;
  } else if (t < 132) {
    const int c = t - 128;
    const int dy = (c < 2) ? -1 : 1, dx = (c & 1) ? 1 : -1;
    const int nty = ty + dy, ntx = tx + dx;
    uint16_t v = 0;
    if (nty >= 0 && nty < d.TY && ntx >= 0 && ntx < d.TX)
      v = d.fl[((size_t)s * d.T + nty * d.TX + ntx) * TPX + (dy < 0 ? 31 : 0) * TS + (dx < 0 ? 31 : 0)];
    flh[hidx(dy < 0 ? -1 : 32, dx < 0 ? -1 : 32)] = v;
  }
}

__device__ __forceinline__ void store_hedge(const Dev& d, size_t gt, const int (&h)[4], int t) {
  const int ix = t & 31, iy0 = t >> 5;
  int32_t* he = d.hedge + gt * 128;
  if (iy0 == 0) he[0 * 32 + ix] = h[0];
  if (iy0 == 7) he[1 * 32 + ix] = h[3];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    if (ix == 0) he[2 * 32 + iy0 + 8 * j] = h[j];
    if (ix == 31) he[3 * 32 + iy0 + 8 * j] = h[j];
  }
}

template <int K>
__device__ __forceinline__ int make_fl(int e, const int (&r)[K]) {
  int f = (e > 0 ? FL_POS : 0) | (e < 0 ? FL_NEG : 0);
#pragma unroll
  for (int k = 0; k < K; ++k) f |= (r[k] > 0) << k;
  return f;
}

// a1 / a1w: the tile's initial e and r from the caps (and the clamped warm flows).
// e = cs - ct pre-cancels min(cs,ct) along s -> v -> t; arcs pointing off the grid get
// r = 0 whatever the caller stored there (reading c7).
template <int K>
__device__ __forceinline__ void tile_from_caps(const Dev& d, const IO& io, int s, int ty, int tx, int (&e)[4],
                                               int (&r)[4][K], int& bad, long long& sct) {
  const int t = threadIdx.x, ix = t & 31, iy0 = t >> 5;
  const int H = d.H, W = d.W;
  const size_t plane = (size_t)H * W;
  const size_t f = (size_t)d.sfr[s];  // batch frame held by this slot
  const int32_t* cs = d.scs[s];
  const int32_t* ct = d.sct[s];
  const int32_t* nb = d.snb[s];
  const int32_t* wf = d.swf[s];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int y = ty * TS + iy0 + 8 * j, x = tx * TS + ix;
    int ev = 0;
#pragma unroll
    for (int k = 0; k < K; ++k) r[j][k] = 0;
    if (y < H && x < W) {
      const size_t o = (size_t)y * W + x;
      const int a = __ldg(cs + o), b = __ldg(ct + o);
      bad |= (a < 0) | (a > CAPMAX) | (b < 0) | (b > CAPMAX);
      ev = a - b;
      sct += b;
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const int y2 = y + DYk(k), x2 = x + DXk(k);
        if (y2 < 0 || y2 >= H || x2 < 0 || x2 >= W) continue;
        const int c = __ldg(nb + k * plane + o);
        bad |= (c < 0) | (c > CAPMAX);
        if (!wf) {
          r[j][k] = c;
        } else {
          const size_t oq = (size_t)y2 * W + x2;
          const int cq = __ldg(nb + (k ^ 1) * plane + oq);
          if ((k & 1) == 0) {  // forward arc p -> q; its flow is stored at p
            const int f = max(-cq, min(c, __ldg(wf + (k >> 1) * plane + o)));  // a1w clamp
            r[j][k] = c - f;
            ev -= f;
          } else {  // reverse arc of the forward arc q -> p; its flow is stored at q
            const int f = max(-c, min(cq, __ldg(wf + ((k ^ 1) >> 1) * plane + oq)));
            r[j][k] = c + f;
            ev += f;
          }
        }
      }
    }
    e[j] = ev;
  }
}

template <int K>
__device__ __forceinline__ void load_er(const Dev& d, size_t gt, int (&e)[4], int (&r)[4][K]) {
  const int t = threadIdx.x, ix = t & 31, iy0 = t >> 5;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int lp = (iy0 + 8 * j) * TS + ix;
    e[j] = d.e[gt * TPX + lp];
#pragma unroll
    for (int k = 0; k < K; ++k) r[j][k] = Rp(d, K, gt, k)[lp];
  }
}

template <int K>
__device__ __forceinline__ void store_er(const Dev& d, size_t gt, const int (&e)[4], const int (&r)[4][K]) {
  const int t = threadIdx.x, ix = t & 31, iy0 = t >> 5;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int lp = (iy0 + 8 * j) * TS + ix;
    d.e[gt * TPX + lp] = e[j];
#pragma unroll
    for (int k = 0; k < K; ++k) Rp(d, K, gt, k)[lp] = r[j][k];
    d.fl[gt * TPX + lp] = (uint16_t)make_fl<K>(e[j], r[j]);
  }
}

// e, r of a tile: from the materialised state, else recomputed from the caps.
template <int K>
__device__ __forceinline__ void get_er(const Dev& d, const IO& io, size_t gt, int (&e)[4], int (&r)[4][K]) {
  if (d.mat[gt]) {
    load_er<K>(d, gt, e, r);
  } else {
    const int s = (int)((unsigned)gt / (unsigned)d.T), tile = (int)(gt - (size_t)s * d.T);
    const int ty = tile / d.TX, tx = tile - ty * d.TX;
    int bad = 0;
    long long sct = 0;
    tile_from_caps<K>(d, io, s, ty, tx, e, r, bad, sct);
  }
}

// Tile-local BFS fixpoint: h(v) = min(h(v), 1 + min{h(v+d_k) : arc k open}) until stable,
// for distances up to `bnd` (a bounded global relabel; HINF: exact distances everywhere).
// hs holds the halo'd heights (halo fixed); updates are written in place (monotone, so a
// racing reader sees an old or a new upper bound -- both valid).
template <int K>
__device__ __forceinline__ void bfs_fixpoint(volatile int* hs, const int (&fl)[4], int (&h)[4], int bnd) {
  const int t = threadIdx.x, ix = t & 31, iy0 = t >> 5;
  for (;;) {
    int changed = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int iy = iy0 + 8 * j;
      if (h[j] > 1) {
        int mn = HINF;
#pragma unroll
        for (int k = 0; k < K; ++k)
          if ((fl[j] >> k) & 1) mn = min(mn, hs[hidx(iy + DYk(k), ix + DXk(k))]);
        if (mn < bnd && mn + 1 < h[j]) {  // distances beyond the relabel's bound stay HINF
          h[j] = mn + 1;
          hs[hidx(iy, ix)] = h[j];
          changed = 1;
        }
      }
    }
    if (!__syncthreads_or(changed)) break;
  }
}

// One pixel's current e and r: from the materialised state, else recomputed from the caps
// (+ clamped warm flows) exactly as tile_from_caps does.  (y, x) are frame coordinates.
template <int K>
__device__ __forceinline__ void px_er(const Dev& d, const IO& io, size_t gt, int lp, int y, int x, int& e,
                                      int (&r)[K]) {
  if (d.mat[gt]) {
    e = d.e[gt * TPX + lp];
#pragma unroll
    for (int k = 0; k < K; ++k) r[k] = Rp(d, K, gt, k)[lp];
    return;
  }
  const int s = (int)((unsigned)gt / (unsigned)d.T);
  const int H = d.H, W = d.W;
  const size_t plane = (size_t)H * W;
  const size_t f = (size_t)d.sfr[s];
  const int32_t* nb = d.snb[s];
  const int32_t* wf = d.swf[s];
  const bool in = y < H && x < W;
  const size_t o = (size_t)y * W + x;
  e = in ? __ldg(d.scs[s] + o) - __ldg(d.sct[s] + o) : 0;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const int y2 = y + DYk(k), x2 = x + DXk(k);
    int rk = 0;
    if (in && y2 >= 0 && y2 < H && x2 >= 0 && x2 < W) {
      const int c = __ldg(nb + k * plane + o);
      rk = c;
      if (wf) {
        const size_t oq = (size_t)y2 * W + x2;
        const int cq = __ldg(nb + (k ^ 1) * plane + oq);
        if ((k & 1) == 0) {
          const int fv = max(-cq, min(c, __ldg(wf + (k >> 1) * plane + o)));
          rk = c - fv;
          e -= fv;
        } else {
          const int fv = max(-c, min(cq, __ldg(wf + ((k ^ 1) >> 1) * plane + oq)));
          rk = c + fv;
          e += fv;
        }
      }
    }
    r[k] = rk;
  }
}

// ---- shared-memory tile state (push kernel): es[TPX], rs[K][TPX]; pixel-at-a-time so
// no register arrays stay live.
// Caller-layout pointers of the frame a slot holds.
struct FramePtrs {
  size_t fr;  // batch frame index
  const int32_t* cs;
  const int32_t* ct;
  const int32_t* nb;
  const int32_t* wf;
  int32_t* fs;
};
__device__ __forceinline__ FramePtrs frame_ptrs(const Dev& d, const IO& io, int s, int K) {
  const size_t plane = (size_t)d.H * d.W;
  const size_t fr = (size_t)d.sfr[s];  // batch frame held by this slot
  FramePtrs p;
  p.fr = fr;
  p.cs = d.scs[s];
  p.ct = d.sct[s];
  p.nb = d.snb[s];
  p.wf = d.swf[s];
  p.fs = d.sfs[s];
  return p;
}

// Init pass, cap loads: thread t owns the 4 consecutive pixels (t/8, 4(t%8)..+3) of the tile.
template <int K>
__device__ __forceinline__ void init_load(const Dev& d, const FramePtrs& P, int ty, int tx, bool vec, int (&a)[4],
                                          int (&b)[4], int (&c)[K][4]) {
  const int t = threadIdx.x, iy = t >> 3, ix0 = (t & 7) * 4;
  const int H = d.H, W = d.W;
  const size_t plane = (size_t)H * W;
  const int y = ty * TS + iy, x0 = tx * TS + ix0;
  const size_t o0 = (size_t)y * W + x0;
  if (vec && y < H && x0 + 3 < W) {
    const int4 va = __ldg(reinterpret_cast<const int4*>(P.cs + o0));
    const int4 vb = __ldg(reinterpret_cast<const int4*>(P.ct + o0));
    a[0] = va.x; a[1] = va.y; a[2] = va.z; a[3] = va.w;
    b[0] = vb.x; b[1] = vb.y; b[2] = vb.z; b[3] = vb.w;
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const int4 v = __ldg(reinterpret_cast<const int4*>(P.nb + k * plane + o0));
      c[k][0] = v.x; c[k][1] = v.y; c[k][2] = v.z; c[k][3] = v.w;
    }
  } else {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const bool in = y < H && x0 + i < W;
      a[i] = in ? __ldg(P.cs + o0 + i) : 0;
      b[i] = in ? __ldg(P.ct + o0 + i) : 0;
#pragma unroll
      for (int k = 0; k < K; ++k) c[k][i] = in ? __ldg(P.nb + k * plane + o0 + i) : 0;
    }
  }
}

// e, r of a tile into shared memory (es[TPX], rs[K][TPX]): from the materialised state, else
// recomputed from the caps (+ clamped warm flows).  16-byte accesses, thread t owning the 4
// consecutive pixels 4t..4t+3, whenever the layout allows.  Block-wide; ends with a barrier.
template <int K>
__device__ __forceinline__ void tile_load_smem(const Dev& d, const IO& io, size_t gt, int* es, int* rs, bool vec) {
  const int t = threadIdx.x;
  if (d.mat[gt]) {
    reinterpret_cast<int4*>(es)[t] = reinterpret_cast<const int4*>(d.e + gt * TPX)[t];
#pragma unroll
    for (int k = 0; k < K; ++k)
      reinterpret_cast<int4*>(rs + k * TPX)[t] = reinterpret_cast<const int4*>(Rp(d, K, gt, k))[t];
    __syncthreads();
    return;
  }
  const int s = (int)((unsigned)gt / (unsigned)d.T), tile = (int)(gt - (size_t)s * d.T);
  const int ty = tile / d.TX, tx = tile - ty * d.TX;
  const int H = d.H, W = d.W;
  const int ix = t & 31, iy0 = t >> 5;
  if (vec && !d.swf[s]) {  // cold, aligned rows: the init pass's loads (row t/8, columns 4(t%8)..+3)
    const FramePtrs P = frame_ptrs(d, io, s, K);
    int a[4], b[4], c[K][4];
    init_load<K>(d, P, ty, tx, true, a, b, c);
    const int y = ty * TS + (t >> 3), x0 = tx * TS + (t & 7) * 4;
    const bool inner = ty > 0 && tx > 0 && (ty + 1) * TS < H && (tx + 1) * TS < W;
    int ev[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int x = x0 + i;
      const bool in = y < H && x < W;
      int vm = in ? 0xff : 0;
      if (in && !inner) {
        vm = 0;
#pragma unroll
        for (int k = 0; k < K; ++k)
          vm |= ((unsigned)(y + DYk(k)) < (unsigned)H && (unsigned)(x + DXk(k)) < (unsigned)W) << k;
      }
      ev[i] = in ? a[i] - b[i] : 0;
#pragma unroll
      for (int k = 0; k < K; ++k) c[k][i] = ((vm >> k) & 1) ? c[k][i] : 0;
    }
    reinterpret_cast<int4*>(es)[t] = make_int4(ev[0], ev[1], ev[2], ev[3]);
#pragma unroll
    for (int k = 0; k < K; ++k)
      reinterpret_cast<int4*>(rs + k * TPX)[t] = make_int4(c[k][0], c[k][1], c[k][2], c[k][3]);
    __syncthreads();
    return;
  }
  const size_t plane = (size_t)H * W;
  const size_t f = (size_t)d.sfr[s];
  const int32_t* cs = d.scs[s];
  const int32_t* ct = d.sct[s];
  const int32_t* nb = d.snb[s];
  const int32_t* wf = d.swf[s];
  if (K == 4 && vec && wf && ((uintptr_t)wf & 15) == 0) {
    // warm 4-neighbour, aligned rows: thread t takes row t/8, columns 4(t%8)..+3; every value
    // the clamp needs in one batch of loads -- its own caps and flows (16-byte), the reverse
    // caps and flows of the rows above / below (16-byte, same columns) and of the pixels left /
    // right of its 4 (scalars)
    const int iy = t >> 3, ix0 = (t & 7) * 4;
    const int y = ty * TS + iy, x0 = tx * TS + ix0;
    int ev[4] = {0, 0, 0, 0}, rk[4][4] = {};
    if (y < H && x0 < W) {
      const size_t o = (size_t)y * W + x0;
      const bool up = y > 0, dn = y + 1 < H, lf = x0 > 0, rt = x0 + 4 < W;
      const int4 zero = make_int4(0, 0, 0, 0);
      const int4 a = __ldg(reinterpret_cast<const int4*>(cs + o));
      const int4 b = __ldg(reinterpret_cast<const int4*>(ct + o));
      const int4 c0 = __ldg(reinterpret_cast<const int4*>(nb + o));              // E
      const int4 c1 = __ldg(reinterpret_cast<const int4*>(nb + plane + o));      // W
      const int4 c2 = __ldg(reinterpret_cast<const int4*>(nb + 2 * plane + o));  // S
      const int4 c3 = __ldg(reinterpret_cast<const int4*>(nb + 3 * plane + o));  // N
      const int4 f0 = __ldg(reinterpret_cast<const int4*>(wf + o));              // flow E
      const int4 f1 = __ldg(reinterpret_cast<const int4*>(wf + plane + o));      // flow S
      const int4 cNdn = dn ? __ldg(reinterpret_cast<const int4*>(nb + 3 * plane + o + W)) : zero;  // c(q->p), q below
      const int4 cSup = up ? __ldg(reinterpret_cast<const int4*>(nb + 2 * plane + o - W)) : zero;  // c(q->p), q above
      const int4 f1up = up ? __ldg(reinterpret_cast<const int4*>(wf + plane + o - W)) : zero;      // flow S of q above
      const int cWr = rt ? __ldg(nb + plane + o + 4) : 0;  // c(q->p), q right of the 4th pixel
      const int cEl = lf ? __ldg(nb + o - 1) : 0;          // c(q->p), q left of the 1st
      const int f0l = lf ? __ldg(wf + o - 1) : 0;          // flow E of q left of the 1st
      const int A[4] = {a.x, a.y, a.z, a.w}, B[4] = {b.x, b.y, b.z, b.w};
      const int C0[4] = {c0.x, c0.y, c0.z, c0.w}, C1[4] = {c1.x, c1.y, c1.z, c1.w};
      const int C2[4] = {c2.x, c2.y, c2.z, c2.w}, C3[4] = {c3.x, c3.y, c3.z, c3.w};
      const int F0[4] = {f0.x, f0.y, f0.z, f0.w}, F1[4] = {f1.x, f1.y, f1.z, f1.w};
      const int CN[4] = {cNdn.x, cNdn.y, cNdn.z, cNdn.w}, CS[4] = {cSup.x, cSup.y, cSup.z, cSup.w};
      const int F1U[4] = {f1up.x, f1up.y, f1up.z, f1up.w};
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int x = x0 + i;
        int e = A[i] - B[i];
        if (x + 1 < W) {  // E: forward arc, flow stored here
          const int cq = i < 3 ? C1[i + 1] : cWr;
          const int fv = max(-cq, min(C0[i], F0[i]));
          rk[0][i] = C0[i] - fv;
          e -= fv;
        }
        if (x > 0) {  // W: the left neighbour's forward arc
          const int cq = i > 0 ? C0[i - 1] : cEl, fr = i > 0 ? F0[i - 1] : f0l;
          const int fv = max(-C1[i], min(cq, fr));
          rk[1][i] = C1[i] + fv;
          e += fv;
        }
        if (dn) {  // S: forward arc
          const int fv = max(-CN[i], min(C2[i], F1[i]));
          rk[2][i] = C2[i] - fv;
          e -= fv;
        }
        if (up) {  // N: the upper neighbour's forward arc
          const int fv = max(-C3[i], min(CS[i], F1U[i]));
          rk[3][i] = C3[i] + fv;
          e += fv;
        }
        ev[i] = e;
      }
    }
    reinterpret_cast<int4*>(es)[t] = make_int4(ev[0], ev[1], ev[2], ev[3]);
#pragma unroll
    for (int k = 0; k < 4; ++k)
      reinterpret_cast<int4*>(rs + k * TPX)[t] = make_int4(rk[k][0], rk[k][1], rk[k][2], rk[k][3]);
    __syncthreads();
    return;
  }
#pragma unroll 1
  for (int j = 0; j < 4; ++j) {
    const int y = ty * TS + iy0 + 8 * j, x = tx * TS + ix, lp = (iy0 + 8 * j) * TS + ix;
    int ev = 0;
    const bool in = y < H && x < W;
    const size_t o = (size_t)y * W + x;
    if (in) ev = __ldg(cs + o) - __ldg(ct + o);
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const int y2 = y + DYk(k), x2 = x + DXk(k);
      int rk = 0;
      if (in && y2 >= 0 && y2 < H && x2 >= 0 && x2 < W) {
        const int c = __ldg(nb + k * plane + o);
        rk = c;
        if (wf) {  // a1w: identical clamp to tile_from_caps / tile_init
          const size_t oq = (size_t)y2 * W + x2;
          const int cq = __ldg(nb + (k ^ 1) * plane + oq);
          if ((k & 1) == 0) {
            const int fv = max(-cq, min(c, __ldg(wf + (k >> 1) * plane + o)));
            rk = c - fv;
            ev -= fv;
          } else {
            const int fv = max(-c, min(cq, __ldg(wf + ((k ^ 1) >> 1) * plane + oq)));
            rk = c + fv;
            ev += fv;
          }
        }
      }
      rs[k * TPX + lp] = rk;
    }
    es[lp] = ev;
  }
  __syncthreads();
}

// Flow that arrived across the tile border since the tile last absorbed, per direction and
// receiver slot: infl[k][slot] = sent - got (wrapping uint32 arithmetic: the amount in
// flight on one arc is below 2^31), marking it absorbed.  Sender and receiver each own one
// counter, so no atomics are needed.  Coalesced: thread i < 16K handles 4
// consecutive slots of one direction with 16-byte loads.  Block-wide; ends with a barrier.
template <int K>
__device__ __forceinline__ void gather_inflow(const Dev& d, size_t gt, int* infl) {
  const int t = threadIdx.x;
  if (t < 16 * K) {
    uint4* sp = reinterpret_cast<uint4*>(d.sent + gt * K * 64) + t;
    uint4* gp = reinterpret_cast<uint4*>(d.got + gt * K * 64) + t;
    const uint4 sv = __ldcg(sp), gv = *gp;
    int4 dl;
    dl.x = (int)(sv.x - gv.x); dl.y = (int)(sv.y - gv.y); dl.z = (int)(sv.z - gv.z); dl.w = (int)(sv.w - gv.w);
    if (dl.x | dl.y | dl.z | dl.w) *gp = sv;
    reinterpret_cast<int4*>(infl)[t] = dl;
  }
  __syncthreads();
}

// Absorb inbound border flow into the shared-memory state (infl: gather_inflow's result).
template <int K>
__device__ __forceinline__ void absorb_smem(const int* infl, int* es, int* rs) {
  const int t = threadIdx.x, ix = t & 31, iy0 = t >> 5;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int iy = iy0 + 8 * j, lp = iy * TS + ix;
    if (!on_border(iy, ix)) continue;
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const int wy = iy - DYk(k), wx = ix - DXk(k);
      if ((unsigned)wy < 32u && (unsigned)wx < 32u) continue;
      const int dl = infl[k * 64 + recv_slot(k, iy, ix)];
      if (dl) {
        es[lp] += dl;
        rs[(k ^ 1) * TPX + lp] += dl;  // residual u -> w grows by the flow w -> u
      }
    }
  }
}

template <int K>
__device__ __forceinline__ void tile_store_smem(const Dev& d, size_t gt, const int* es, const int* rs) {
  const int t = threadIdx.x;  // pixels 4t..4t+3, 16-byte accesses
  const int4 ev = reinterpret_cast<const int4*>(es)[t];
  reinterpret_cast<int4*>(d.e + gt * TPX)[t] = ev;
  int f0 = (ev.x > 0 ? FL_POS : 0) | (ev.x < 0 ? FL_NEG : 0);
  int f1 = (ev.y > 0 ? FL_POS : 0) | (ev.y < 0 ? FL_NEG : 0);
  int f2 = (ev.z > 0 ? FL_POS : 0) | (ev.z < 0 ? FL_NEG : 0);
  int f3 = (ev.w > 0 ? FL_POS : 0) | (ev.w < 0 ? FL_NEG : 0);
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const int4 rk = reinterpret_cast<const int4*>(rs + k * TPX)[t];
    reinterpret_cast<int4*>(Rp(d, K, gt, k))[t] = rk;
    f0 |= (rk.x > 0) << k; f1 |= (rk.y > 0) << k; f2 |= (rk.z > 0) << k; f3 |= (rk.w > 0) << k;
  }
  ushort4 w;
  w.x = (unsigned short)f0; w.y = (unsigned short)f1; w.z = (unsigned short)f2; w.w = (unsigned short)f3;
  reinterpret_cast<ushort4*>(d.fl + gt * TPX)[t] = w;
}

// ------------------------------------------------------------------------------ a1
// Init: a streaming pass over the caps.  Computes e and r in registers (the tile stays
// un-materialised -- e, r are recomputed if a push ever touches it) and writes only the
// 2-byte fl word per pixel, the frame's sum c(v,t), the tile's sum max(0,-e) and the
// range flag.  Thread t owns 4 consecutive pixels of row t/8 (int4 loads when the caller's
// rows are 16-byte aligned).
// Init pass, per tile once the caps are in registers: computes e and r (the tile stays
// un-materialised -- e, r are recomputed if a push ever touches it) and writes only the
// 2-byte fl word per pixel, zeroes the caller's mask, flags a uniform sink tile, and adds
// the tile's sum c(v,t) and sum max(0,-e) to the frame (range flag on bad caps).
constexpr int INIT_GMAX = 32;  // tiles per init task, at most

// Per-warp partial results of one init tile (summed by the group's finalisation).
struct InitPart {
  long long sct[NTH / 32];  // sum c(v,t)
  long long neg[NTH / 32];  // sum max(0,-e)
  int fl[NTH / 32];         // bit 0: capacity out of range, bit 1: not a uniform sink tile,
                            // bit 2: not a uniform source tile
};

template <int K, bool WARM, bool EXPORT>
__device__ __forceinline__ void tile_init_regs(const Dev& d, const IO& io, size_t gt, const FramePtrs& P,
                                               const int (&a)[4], const int (&b)[4], const int (&c)[K][4],
                                               InitPart* part, bool sym = false, const int (*wq)[4] = nullptr,
                                               const int (*wfr)[4] = nullptr) {
  const int s = (int)((unsigned)gt / (unsigned)d.T), tile = (int)(gt - (size_t)s * d.T);
  const int ty = tile / d.TX, tx = tile - ty * d.TX;
  const int t = threadIdx.x, iy = t >> 3, ix0 = (t & 7) * 4;
  const int H = d.H, W = d.W;
  const size_t plane = (size_t)H * W;
  const size_t fr = P.fr;
  const int32_t* nb = P.nb;
  const int32_t* wf = P.wf;
  const int y = ty * TS + iy, x0 = tx * TS + ix0;
  const size_t o0 = (size_t)y * W + x0;
  // arcs whose far end is in the frame: all of them for tiles away from the frame border
  const bool inner = ty > 0 && tx > 0 && (ty + 1) * TS < H && (tx + 1) * TS < W;
  int acc = 0;  // OR of every in-grid capacity: one is outside [0, GC_CAP_MAX] iff acc & ~CAPMAX
  int uni = 1, src = 1;
  long long sct = 0, neg = 0;
  int fl4[4];
  int fwv[K / 2][4];  // exported forward flows of the 4 pixels (EXPORT)
  // 16-byte export stores: the 4 pixels in the frame and the rows aligned
  const bool ev4 = EXPORT && K == 4 && y < H && x0 + 3 < W && (((uintptr_t)(P.fs + o0)) & 15) == 0 && ((plane & 3) == 0);
  if (!WARM && !EXPORT && inner) {
    // cold tile away from the frame border (most tiles): every arc in the grid, no clamp
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      int f = 0, ca = a[i] | b[i];
#pragma unroll
      for (int k = 0; k < K; ++k) {
        ca |= c[k][i];
        f |= (c[k][i] > 0) << k;
      }
      acc |= ca;
      const int ev = a[i] - b[i];  // a1: pre-cancel min(cs,ct) straight s -> v -> t
      sct += b[i];
      f |= (ev > 0 ? FL_POS : 0) | (ev < 0 ? FL_NEG : 0);
      neg += ev < 0 ? -(long long)ev : 0;
      uni &= ev < 0;
      src &= ev > 0;
      fl4[i] = f;
    }
  } else
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int x = x0 + i;
    int f = 0;
    if (inner || (y < H && x < W)) {
      int vm = 0xff;  // valid-arc mask (reading c7: off-grid arcs are ignored)
      if (!inner) {
        vm = 0;
#pragma unroll
        for (int k = 0; k < K; ++k) {
          const int y2 = y + DYk(k), x2 = x + DXk(k);
          vm |= ((unsigned)y2 < (unsigned)H && (unsigned)x2 < (unsigned)W) << k;
        }
      }
      acc |= a[i] | b[i];
      int ev = a[i] - b[i];  // a1: pre-cancel min(cs,ct) straight s -> v -> t
      sct += b[i];
      int fw[K / 2];  // forward-arc flows as initialised (0 cold, the clamped warm flow)
#pragma unroll
      for (int k = 0; k < K / 2; ++k) fw[k] = 0;
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const int on = (vm >> k) & 1;
        const int ck = on ? c[k][i] : 0;
        acc |= ck;
        int rk = ck;
        if (WARM && on) {  // a1w: clamp the previous flow to the new capacities
          const int y2 = y + DYk(k), x2 = x + DXk(k);
          const size_t oq = (size_t)y2 * W + x2;
          // energy caps are symmetric (c(q -> p) = c(p -> q)): the neighbour's may not be built yet;
          // wq / wfr: the values warm4_load fetched
          const int cq = sym ? ck : (wq ? wq[k][i] : __ldg(nb + (k ^ 1) * plane + oq));
          if ((k & 1) == 0) {
            const int fraw = wfr ? wfr[k][i] : __ldg(wf + (k >> 1) * plane + o0 + i);
            const int fv = max(-cq, min(ck, fraw));
            rk = ck - fv;
            ev -= fv;
            fw[k >> 1] = fv;
          } else {
            const int fraw = wfr ? wfr[k][i] : __ldg(wf + ((k ^ 1) >> 1) * plane + oq);
            const int fv = max(-ck, min(cq, fraw));
            rk = ck + fv;
            ev += fv;
          }
        }
        f |= (rk > 0) << k;
      }
      f |= (ev > 0 ? FL_POS : 0) | (ev < 0 ? FL_NEG : 0);
      neg += ev < 0 ? -(long long)ev : 0;
      uni &= ev < 0;
      src &= ev > 0;
      if (EXPORT) {  // a5: the export of a tile no push ever touches is its initial flow
#pragma unroll
        for (int k = 0; k < K / 2; ++k) fwv[k][i] = fw[k];
        if (!ev4) {
          int32_t* fo = P.fs + o0 + i;
#pragma unroll
          for (int k = 0; k < K / 2; ++k) fo[k * plane] = fw[k];
        }
      }
    }
    fl4[i] = f;
  }
  if (ev4) {
#pragma unroll
    for (int k = 0; k < K / 2; ++k)
      *reinterpret_cast<int4*>(P.fs + k * plane + o0) = make_int4(fwv[k][0], fwv[k][1], fwv[k][2], fwv[k][3]);
  }
  int bad = (acc & ~CAPMAX) != 0;
  ushort4 w;
  w.x = (unsigned short)fl4[0]; w.y = (unsigned short)fl4[1];
  w.z = (unsigned short)fl4[2]; w.w = (unsigned short)fl4[3];
  *reinterpret_cast<ushort4*>(d.fl + gt * TPX + iy * TS + ix0) = w;
  if (y < H) {  // the caller's mask starts as the excess pixels (e > 0: always in the closure);
                 // the closure phases write the other closure pixels (and rewrite touched tiles)
    uint8_t* mk = io.mask + fr * plane + (size_t)y * W + x0;
    const uint32_t mw = ((fl4[0] >> 8) & 1u) | (((fl4[1] >> 8) & 1u) << 8) | (((fl4[2] >> 8) & 1u) << 16) |
                        (((unsigned)(fl4[3] >> 8) & 1u) << 24);
    if (x0 + 3 < W && ((uintptr_t)mk & 3) == 0) {
      *reinterpret_cast<uint32_t*>(mk) = mw;
    } else {
#pragma unroll
      for (int i = 0; i < 4; ++i)
        if (x0 + i < W) mk[i] = (uint8_t)((mw >> (8 * i)) & 1u);
    }
  }
  // warp partials (no barrier: warps run ahead to the next tile's loads); sums with REDUX on
  // 32-bit halves (per-thread sums are < 2^31, warp sums may not be)
  const unsigned long long us = (unsigned long long)sct, un = (unsigned long long)neg;
  const unsigned s_lo = __reduce_add_sync(0xffffffffu, (unsigned)(us & 0xffffu));
  const unsigned s_hi = __reduce_add_sync(0xffffffffu, (unsigned)(us >> 16));
  const unsigned n_lo = __reduce_add_sync(0xffffffffu, (unsigned)(un & 0xffffu));
  const unsigned n_hi = __reduce_add_sync(0xffffffffu, (unsigned)(un >> 16));
  const int wfl = __reduce_or_sync(0xffffffffu, bad | ((!uni) << 1) | ((!src) << 2));
  if ((t & 31) == 0) {
    part->sct[t >> 5] = (long long)s_lo + ((long long)s_hi << 16);
    part->neg[t >> 5] = (long long)n_lo + ((long long)n_hi << 16);
    part->fl[t >> 5] = wfl;
  }
}

// Per-tile results of an init group, after a barrier: tile words, frame sums, range flag,
// and the border heights of uniform sink tiles (h = 1 in frame).  uni_s[i]: bit 0 uniform
// sink, bit 1 uniform source (the fused seed of the first relabel skips both).
__device__ __forceinline__ void init_finalize(const Dev& d, size_t gt0, int n, const InitPart* part, int* uni_s) {
  const int t = threadIdx.x;
  const int s = (int)((unsigned)gt0 / (unsigned)d.T);
  if (t < n) {
    const size_t gt = gt0 + t;
    long long sa = 0, sb = 0;
    int f = 0;
#pragma unroll
    for (int w = 0; w < NTH / 32; ++w) { sa += part[t].sct[w]; sb += part[t].neg[w]; f |= part[t].fl[w]; }
    const int uni = !(f & 2), src = !(f & 4);
    if (sa) atomicAdd(&d.sumct[s], (unsigned long long)sa);
    if (sb) atomicAdd(&d.sumneg[s], (unsigned long long)sb);  // corrected by the closure seed if e changes
    d.neg0[gt] = sb;
    d.mat[gt] = 0;
    d.recv1[gt] = 0;
    d.tact[gt] = 0;
    d.tuni[gt] = uni;
    d.tsrc[gt] = src;
    d.tfix[gt] = uni;
    d.tph[gt] = -1;
    d.tmk[gt] = 0;
    d.tsk[gt] = 0;  // relabel epochs restart at 1 per frame: a stale stamp would alias
    d.tss[gt] = src ? 1 : 0;  // the first relabel (epoch 1) does not seed a uniform source tile
    if (f & 1) d.ferr[s] = 1;
    uni_s[t] = uni | (src << 1);
  }
  __syncthreads();
  for (int j = 0; j < n; ++j) {
    if (!(uni_s[j] & 1) || t >= 128) continue;
    const int tile = (int)(gt0 + j - (size_t)s * d.T);
    const int ty = tile / d.TX, tx = tile - ty * d.TX;
    const int side = t >> 5, i = t & 31;
    const int py = side == 0 ? 0 : (side == 1 ? 31 : i), px = side == 2 ? 0 : (side == 3 ? 31 : i);
    d.hedge[(gt0 + j) * 128 + t] = (ty * TS + py < d.H && tx * TS + px < d.W) ? 1 : HINF;
  }
}

// a1 / a1w: one init task = a group of d.initg consecutive tiles of a frame (more tiles per
// task on large frames: less per-task overhead; one on small frames: more parallelism).
// No barrier inside the group: each warp streams its rows of tile after tile (16-byte loads
// straight to registers) and leaves per-warp partials; one barrier and a finalisation at
// the end publish the per-tile results.

// 16-byte global -> shared copy that bypasses registers (LDGSTS); src_bytes 0 zero-fills.
__device__ __forceinline__ void cp_async16(void* dst, const void* src, int src_bytes) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(src), "r"(src_bytes) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

// Prefetch of one tile's caps into this thread's own shared slots pf[j * NTH + t]
// (j = 0: cs, 1: ct, 2 + k: c_k), the same pixels init_load reads; zero outside the frame.
template <int K>
__device__ __forceinline__ void init_prefetch(const Dev& d, const FramePtrs& P, int ty, int tx, int4* pf) {
  const int t = threadIdx.x;
  const int y = ty * TS + (t >> 3), x0 = tx * TS + (t & 7) * 4;
  const bool in = y < d.H && x0 < d.W;  // W % 4 == 0 on this path
  const size_t plane = (size_t)d.H * d.W;
  const size_t o0 = in ? (size_t)y * d.W + x0 : 0;
  const int nbytes = in ? 16 : 0;
  cp_async16(pf + t, P.cs + o0, nbytes);
  cp_async16(pf + NTH + t, P.ct + o0, nbytes);
#pragma unroll
  for (int k = 0; k < K; ++k) cp_async16(pf + (2 + k) * NTH + t, P.nb + k * plane + o0, nbytes);
  cp_async_commit();
}

template <int K>
constexpr size_t init_smem_bytes() {
  return INIT_GMAX * sizeof(InitPart) + INIT_GMAX * sizeof(int) + 128 + (2 + K) * NTH * 16;
}

// ---- NEXT-1: the energy of §4 -> capacities, in the init pass (energy mode).
// t-links: c(s,v) = psi1(A=0) + xi1(A=0) = -log p(C|A=0) - log(1 - p),
//                      c(v,t) = psi1(A=1) + xi1(A=1) = -log p(C|A=1) - log p,
// with p(C|A) a colour GMM (normalisation terms from the host) and
// p = clamp(prior / 65535, eps, 1 - eps); n-links (reading c5):
// B = lambda exp(-(dI/255)^2 / (2 sigma^2)) / dist + kappa on the integer luma
// I = (77 R + 150 G + 29 B + 128) >> 8, looked up by |dI| in nlut.  q(x) = floor(scale x + 0.5)
// clamped to [0, GC_CAP_MAX].  Evaluated in double precision (the oracle's precision).
__device__ __forceinline__ int e_quant(double x, double scale) {
  const double v = floor(scale * x + 0.5);
  return v <= 0.0 ? 0 : (v >= (double)CAPMAX ? CAPMAX : (int)v);
}
__device__ __forceinline__ double e_gmm_nll(const Gmm& g, double r, double gg, double b) {
  double v[GMM_MAX], mx = -1e300;
#pragma unroll
  for (int m = 0; m < GMM_MAX; ++m) {
    if (m >= g.M) break;
    const double dr = r - g.mean[m][0], dg = gg - g.mean[m][1], db = b - g.mean[m][2];
    const double* P = g.prec[m];
    const double q = P[0] * dr * dr + P[3] * dg * dg + P[5] * db * db +
                     2.0 * (P[1] * dr * dg + P[2] * dr * db + P[4] * dg * db);
    v[m] = g.lognorm[m] - 0.5 * q;
    mx = fmax(mx, v[m]);
  }
  double sum = 0.0;
#pragma unroll
  for (int m = 0; m < GMM_MAX; ++m) {
    if (m >= g.M) break;
    sum += exp(v[m] - mx);
  }
  return -(mx + log(sum));
}
__device__ __forceinline__ int e_luma(const uint8_t* px) { return (77 * px[0] + 150 * px[1] + 29 * px[2] + 128) >> 8; }

// Caps of this thread's 4 pixels (row t/8, columns 4(t%8)..+3 of tile (ty, tx)) from the energy,
// stored into the slot's cap buffer (the later phases read them there); off-frame: 0.
template <int K>
__device__ __forceinline__ void energy_caps(const Dev& d, const IO& io, const FramePtrs& P, int ty, int tx, int (&a)[4],
                                            int (&b)[4], int (&c)[K][4]) {
  const int t = threadIdx.x, iy = t >> 3, ix0 = (t & 7) * 4;
  const int H = d.H, W = d.W;
  const size_t plane = (size_t)H * W;
  const int y = ty * TS + iy, x0 = tx * TS + ix0;
  const uint8_t* img = io.img + P.fr * plane * 3;
  const uint16_t* pr = io.prior + P.fr * plane;
  const Gmm& g0 = io.gmm[2 * P.fr];
  const Gmm& g1 = io.gmm[2 * P.fr + 1];
  // luma of the 3 x 6 neighbourhood of the 4 pixels (rows y-1..y+1, columns x0-1..x0+4)
  int lu[3][6];
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int q = 0; q < 6; ++q) {
      const int yy = y - 1 + r, xx = x0 - 1 + q;
      lu[r][q] = ((unsigned)yy < (unsigned)H && (unsigned)xx < (unsigned)W) ? e_luma(img + ((size_t)yy * W + xx) * 3) : 0;
    }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int x = x0 + i;
    a[i] = b[i] = 0;
#pragma unroll
    for (int k = 0; k < K; ++k) c[k][i] = 0;
    if (y >= H || x >= W) continue;
    const uint8_t* pxl = img + ((size_t)y * W + x) * 3;
    const double R = pxl[0], G = pxl[1], B = pxl[2];
    double p = (double)__ldg(pr + (size_t)y * W + x) / 65535.0;
    p = fmin(fmax(p, io.eps), 1.0 - io.eps);
    a[i] = e_quant(e_gmm_nll(g0, R, G, B) - log(1.0 - p), io.scale);  // c(s,v): label 0
    b[i] = e_quant(e_gmm_nll(g1, R, G, B) - log(p), io.scale);        // c(v,t): label 1
    const int lc = lu[1][i + 1];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const int y2 = y + DYk(k), x2 = x + DXk(k);
      if ((unsigned)y2 >= (unsigned)H || (unsigned)x2 >= (unsigned)W) continue;
      const int dI = abs(lc - lu[1 + DYk(k)][i + 1 + DXk(k)]);
      c[k][i] = __ldg(io.nlut + (k >= 4 ? 256 : 0) + dI);
    }
  }
  // the slot's cap buffer, frame layout (16-byte stores when the row allows)
  if (y < H) {
    const size_t o0 = (size_t)y * W + x0;
    int32_t* cs = const_cast<int32_t*>(P.cs);
    int32_t* ct = const_cast<int32_t*>(P.ct);
    int32_t* nb = const_cast<int32_t*>(P.nb);
    if (x0 + 3 < W && (W & 3) == 0) {
      *reinterpret_cast<int4*>(cs + o0) = make_int4(a[0], a[1], a[2], a[3]);
      *reinterpret_cast<int4*>(ct + o0) = make_int4(b[0], b[1], b[2], b[3]);
#pragma unroll
      for (int k = 0; k < K; ++k)
        *reinterpret_cast<int4*>(nb + k * plane + o0) = make_int4(c[k][0], c[k][1], c[k][2], c[k][3]);
    } else {
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        if (x0 + i >= W) continue;
        cs[o0 + i] = a[i];
        ct[o0 + i] = b[i];
#pragma unroll
        for (int k = 0; k < K; ++k) nb[k * plane + o0 + i] = c[k][i];
      }
    }
  }
}

// ---- TMA (cp.async.bulk.tensor) staging of the init stream.  Tensor maps over the caller's
// cap arrays (host-built per call, gc_solver.cu): cs, ct as [n][H][W] (rank 3), nb as
// [n][K][H][W] (rank 4), boxes of 32 x 4 pixels (x 1 frame, x K planes): one box set per WARP,
// i.e. the 4 tile rows the warp owns (thread t owns row t/8, columns 4(t%8)..+3).  Each warp
// has its own mbarrier and a 512 x (2+K)-byte stage; lane 0 arms the barrier with the stage's
// byte count and issues the next tile's three loads as soon as the warp has moved the current
// one into registers, so no CTA barrier is needed (the warps stream independently) and no
// thread spends issue slots or registers on addresses.  Boxes reaching past the frame edge
// are zero-filled by the TMA unit.
struct Tmaps {
  CUtensorMap cs, ct, nb;
  int on;  // maps valid (cold frames, 16-byte aligned rows)
  int pf;  // tiles ahead of the smem load whose rows are prefetched into L2 (0: none)
  int ef;  // load the caps with an L2 evict-first policy (read once: keep the solve's working set)
};

__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                   (unsigned)__cvta_generic_to_shared(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
  unsigned done = 0;
  while (!done) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
        : "=r"(done)
        : "r"(a), "r"(parity)
        : "memory");
  }
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int c0, int c1, int c2, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
          (unsigned)__cvta_generic_to_shared(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"((unsigned)__cvta_generic_to_shared(bar))
      : "memory");
}
__device__ __forceinline__ void tma_load_3d_ef(void* dst, const CUtensorMap* map, int c0, int c1, int c2, uint64_t* bar,
                                               uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, %3, %4}], [%5], %6;" ::"r"(
          (unsigned)__cvta_generic_to_shared(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"((unsigned)__cvta_generic_to_shared(bar)),
      "l"(pol)
      : "memory");
}
__device__ __forceinline__ void tma_load_4d_ef(void* dst, const CUtensorMap* map, int c0, int c1, int c2, int c3,
                                               uint64_t* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, %3, %4, %5}], [%6], %7;" ::"r"(
          (unsigned)__cvta_generic_to_shared(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3),
      "r"((unsigned)__cvta_generic_to_shared(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ uint64_t l2_evict_first_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* map, int c0, int c1, int c2, int c3,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(
          (unsigned)__cvta_generic_to_shared(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3),
      "r"((unsigned)__cvta_generic_to_shared(bar))
      : "memory");
}

__device__ __forceinline__ void tma_prefetch_3d(const CUtensorMap* map, int c0, int c1, int c2) {
  asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global.tile [%0, {%1, %2, %3}];" ::"l"(reinterpret_cast<uint64_t>(map)),
               "r"(c0), "r"(c1), "r"(c2)
               : "memory");
}
__device__ __forceinline__ void tma_prefetch_4d(const CUtensorMap* map, int c0, int c1, int c2, int c3) {
  asm volatile("cp.async.bulk.prefetch.tensor.4d.L2.global.tile [%0, {%1, %2, %3, %4}];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(c0), "r"(c1), "r"(c2), "r"(c3)
               : "memory");
}
// Lane 0 of warp w: prefetch rows 4w..4w+3 of tile (ty, tx) into L2 (no barrier, no smem).
__device__ __forceinline__ void tma_prefetch_rows(const Tmaps& tm, int fr, int ty, int tx, int w) {
  const int x = tx * TS, y = ty * TS + 4 * w;
  tma_prefetch_3d(&tm.cs, x, y, fr);
  tma_prefetch_3d(&tm.ct, x, y, fr);
  tma_prefetch_4d(&tm.nb, x, y, 0, fr);
}

// Lane 0 of warp w: arm the warp's barrier and load rows 4w..4w+3 of tile (ty, tx) of frame fr.
template <int K>
__device__ __forceinline__ void tma_issue_rows(const Tmaps& tm, char* stage, uint64_t* bar, int fr, int ty, int tx,
                                               int w) {
  mbar_expect_tx(bar, (2 + K) * 512);
  const int x = tx * TS, y = ty * TS + 4 * w;
  if (tm.ef) {
    const uint64_t pol = l2_evict_first_policy();
    tma_load_3d_ef(stage, &tm.cs, x, y, fr, bar, pol);
    tma_load_3d_ef(stage + 512, &tm.ct, x, y, fr, bar, pol);
    tma_load_4d_ef(stage + 1024, &tm.nb, x, y, 0, fr, bar, pol);
  } else {
    tma_load_3d(stage, &tm.cs, x, y, fr, bar);
    tma_load_3d(stage + 512, &tm.ct, x, y, fr, bar);
    tma_load_4d(stage + 1024, &tm.nb, x, y, 0, fr, bar);
  }
}

// Warm 4-neighbour init loads, aligned rows (thread t: row t/8, columns 4(t%8)..+3): the
// pixel's caps, and per arc k the reverse cap c(q -> p) (wq) and the stored flow of the arc
// (wfr: the pixel's own forward flow for E / S, the neighbour's for W / N) -- one batch of
// independent loads (16-byte rows, the rows above / below, scalars left / right of the 4).
// Off-frame arcs read 0 (tile_init_regs ignores them).
__device__ __forceinline__ void warm4_load(const Dev& d, const FramePtrs& P, int ty, int tx, int (&a)[4], int (&b)[4],
                                           int (&c)[4][4], int (&wq)[4][4], int (&wfr)[4][4]) {
  const int t = threadIdx.x, iy = t >> 3, ix0 = (t & 7) * 4;
  const int H = d.H, W = d.W;
  const size_t plane = (size_t)H * W;
  const int y = ty * TS + iy, x0 = tx * TS + ix0;
  const int4 zero = make_int4(0, 0, 0, 0);
  int4 va = zero, vb = zero, c0 = zero, c1 = zero, c2 = zero, c3 = zero, f0 = zero, f1 = zero;
  int4 cNdn = zero, cSup = zero, f1up = zero;
  int cWr = 0, cEl = 0, f0l = 0;
  if (y < H && x0 < W) {
    const size_t o = (size_t)y * W + x0;
    const bool up = y > 0, dn = y + 1 < H, lf = x0 > 0, rt = x0 + 4 < W;
    va = __ldg(reinterpret_cast<const int4*>(P.cs + o));
    vb = __ldg(reinterpret_cast<const int4*>(P.ct + o));
    c0 = __ldg(reinterpret_cast<const int4*>(P.nb + o));
    c1 = __ldg(reinterpret_cast<const int4*>(P.nb + plane + o));
    c2 = __ldg(reinterpret_cast<const int4*>(P.nb + 2 * plane + o));
    c3 = __ldg(reinterpret_cast<const int4*>(P.nb + 3 * plane + o));
    f0 = __ldg(reinterpret_cast<const int4*>(P.wf + o));
    f1 = __ldg(reinterpret_cast<const int4*>(P.wf + plane + o));
    if (dn) cNdn = __ldg(reinterpret_cast<const int4*>(P.nb + 3 * plane + o + W));
    if (up) cSup = __ldg(reinterpret_cast<const int4*>(P.nb + 2 * plane + o - W));
    if (up) f1up = __ldg(reinterpret_cast<const int4*>(P.wf + plane + o - W));
    if (rt) cWr = __ldg(P.nb + plane + o + 4);
    if (lf) cEl = __ldg(P.nb + o - 1);
    if (lf) f0l = __ldg(P.wf + o - 1);
  }
  a[0] = va.x; a[1] = va.y; a[2] = va.z; a[3] = va.w;
  b[0] = vb.x; b[1] = vb.y; b[2] = vb.z; b[3] = vb.w;
  c[0][0] = c0.x; c[0][1] = c0.y; c[0][2] = c0.z; c[0][3] = c0.w;
  c[1][0] = c1.x; c[1][1] = c1.y; c[1][2] = c1.z; c[1][3] = c1.w;
  c[2][0] = c2.x; c[2][1] = c2.y; c[2][2] = c2.z; c[2][3] = c2.w;
  c[3][0] = c3.x; c[3][1] = c3.y; c[3][2] = c3.z; c[3][3] = c3.w;
  // E (k = 0): c(q -> p) = W cap of the right neighbour, flow = own E flow
  wq[0][0] = c1.y; wq[0][1] = c1.z; wq[0][2] = c1.w; wq[0][3] = cWr;
  wfr[0][0] = f0.x; wfr[0][1] = f0.y; wfr[0][2] = f0.z; wfr[0][3] = f0.w;
  // W (k = 1): c(q -> p) = E cap of the left neighbour, flow = its E flow
  wq[1][0] = cEl; wq[1][1] = c0.x; wq[1][2] = c0.y; wq[1][3] = c0.z;
  wfr[1][0] = f0l; wfr[1][1] = f0.x; wfr[1][2] = f0.y; wfr[1][3] = f0.z;
  // S (k = 2): c(q -> p) = N cap of the pixel below, flow = own S flow
  wq[2][0] = cNdn.x; wq[2][1] = cNdn.y; wq[2][2] = cNdn.z; wq[2][3] = cNdn.w;
  wfr[2][0] = f1.x; wfr[2][1] = f1.y; wfr[2][2] = f1.z; wfr[2][3] = f1.w;
  // N (k = 3): c(q -> p) = S cap of the pixel above, flow = its S flow
  wq[3][0] = cSup.x; wq[3][1] = cSup.y; wq[3][2] = cSup.z; wq[3][3] = cSup.w;
  wfr[3][0] = f1up.x; wfr[3][1] = f1up.y; wfr[3][2] = f1up.z; wfr[3][3] = f1up.w;
}

template <int K>
__device__ __forceinline__ void task_init(const Dev& d, const IO& io, size_t gt0, bool vec, int* smem,
                                          const Tmaps& tm, uint64_t* mbar, unsigned& tpar) {
  const int s = (int)((unsigned)gt0 / (unsigned)d.T), tile0 = (int)(gt0 - (size_t)s * d.T);
  const int n = min(d.initg, d.T - tile0);
  const FramePtrs P = frame_ptrs(d, io, s, K);
  InitPart* part = reinterpret_cast<InitPart*>(smem);        // [n]
  int* uni_s = reinterpret_cast<int*>(part + INIT_GMAX);     // [n]
  int a[4], b[4], c[K][4];
  if (tm.on && !P.wf) {
    // cold frames, aligned rows: TMA row boxes per warp, tile i + 1's arriving while tile i is
    // computed from registers
    const int t = threadIdx.x, w = t >> 5, lane = t & 31;
    char* stage = reinterpret_cast<char*>(((uintptr_t)(uni_s + INIT_GMAX) + 127) & ~(uintptr_t)127) + w * (2 + K) * 512;
    uint64_t* bar = mbar + w;
    const int fr = (int)P.fr;
    if (lane == 0) {
      tma_issue_rows<K>(tm, stage, bar, fr, tile0 / d.TX, tile0 % d.TX, w);
      for (int q = 1; q <= tm.pf && q < n; ++q) tma_prefetch_rows(tm, fr, (tile0 + q) / d.TX, (tile0 + q) % d.TX, w);
    }
#pragma unroll 1
    for (int i = 0; i < n; ++i) {
      mbar_wait(bar, tpar);
      tpar ^= 1u;
      {
        const int4* sv = reinterpret_cast<const int4*>(stage) + lane;
        int4 v = sv[0];
        a[0] = v.x; a[1] = v.y; a[2] = v.z; a[3] = v.w;
        v = sv[32];
        b[0] = v.x; b[1] = v.y; b[2] = v.z; b[3] = v.w;
#pragma unroll
        for (int k = 0; k < K; ++k) {
          v = sv[(2 + k) * 32];
          c[k][0] = v.x; c[k][1] = v.y; c[k][2] = v.z; c[k][3] = v.w;
        }
      }
      __syncwarp();  // the warp's stage is free for the next tile
      if (i + 1 < n && lane == 0) {
        const int tile = tile0 + i + 1;
        tma_issue_rows<K>(tm, stage, bar, fr, tile / d.TX, tile % d.TX, w);
        const int tp = tile + tm.pf;  // keep the L2 prefetch pf tiles ahead
        if (tm.pf && tp < tile0 + n) tma_prefetch_rows(tm, fr, tp / d.TX, tp % d.TX, w);
      }
      if (P.fs) tile_init_regs<K, false, true>(d, io, gt0 + i, P, a, b, c, part + i);
      else tile_init_regs<K, false, false>(d, io, gt0 + i, P, a, b, c, part + i);
    }
  } else if (vec && !P.wf) {
    // cold frames, aligned rows: tile i + 1's caps stream into shared memory (cp.async,
    // each thread its own slots, so no barrier) while tile i is computed from registers
    int4* pf = reinterpret_cast<int4*>(uni_s + INIT_GMAX);  // [(2 + K) * NTH]
    const int t = threadIdx.x;
    init_prefetch<K>(d, P, tile0 / d.TX, tile0 % d.TX, pf);
#pragma unroll 1
    for (int i = 0; i < n; ++i) {
      cp_async_wait_all();
      {
        int4 v = pf[t];
        a[0] = v.x; a[1] = v.y; a[2] = v.z; a[3] = v.w;
        v = pf[NTH + t];
        b[0] = v.x; b[1] = v.y; b[2] = v.z; b[3] = v.w;
#pragma unroll
        for (int k = 0; k < K; ++k) {
          v = pf[(2 + k) * NTH + t];
          c[k][0] = v.x; c[k][1] = v.y; c[k][2] = v.z; c[k][3] = v.w;
        }
      }
      if (i + 1 < n) {
        const int tile = tile0 + i + 1;
        init_prefetch<K>(d, P, tile / d.TX, tile % d.TX, pf);
      }
      if (P.fs) tile_init_regs<K, false, true>(d, io, gt0 + i, P, a, b, c, part + i);
      else tile_init_regs<K, false, false>(d, io, gt0 + i, P, a, b, c, part + i);
    }
  } else if (K == 4 && vec && P.wf && ((uintptr_t)P.wf & 15) == 0) {
    // warm 4-neighbour frames, aligned rows: every cap and flow the clamp needs in one batch of
    // loads per tile (warm4_load; no staging, no barrier)
#pragma unroll 1
    for (int i = 0; i < n; ++i) {
      const int tile = tile0 + i, ty = tile / d.TX, tx = tile - ty * d.TX;
      int wq[4][4], wfr[4][4];
      warm4_load(d, P, ty, tx, a, b, reinterpret_cast<int(&)[4][4]>(c), wq, wfr);
      if (P.fs) tile_init_regs<K, true, true>(d, io, gt0 + i, P, a, b, c, part + i, false, wq, wfr);
      else tile_init_regs<K, true, false>(d, io, gt0 + i, P, a, b, c, part + i, false, wq, wfr);
    }
  } else {
#pragma unroll 1
    for (int i = 0; i < n; ++i) {
      const int tile = tile0 + i, ty = tile / d.TX, tx = tile - ty * d.TX;
      init_load<K>(d, P, ty, tx, vec, a, b, c);
      if (P.wf && P.fs) tile_init_regs<K, true, true>(d, io, gt0 + i, P, a, b, c, part + i);
      else if (P.wf) tile_init_regs<K, true, false>(d, io, gt0 + i, P, a, b, c, part + i);
      else if (P.fs) tile_init_regs<K, false, true>(d, io, gt0 + i, P, a, b, c, part + i);
      else tile_init_regs<K, false, false>(d, io, gt0 + i, P, a, b, c, part + i);
    }
  }
  __syncthreads();
  init_finalize(d, gt0, n, part, uni_s);
}

// Energy-mode init pass over a group of tiles (out of line: its double-precision working set
// would otherwise share the register allocation of the streaming cap path).
template <int K>
__device__ __forceinline__ void task_init_energy(const Dev& d, const IO& io, size_t gt0, int* smem) {
  const int s = (int)((unsigned)gt0 / (unsigned)d.T), tile0 = (int)(gt0 - (size_t)s * d.T);
  const int n = min(d.initg, d.T - tile0);
  const FramePtrs P = frame_ptrs(d, io, s, K);
  InitPart* part = reinterpret_cast<InitPart*>(smem);        // [n]
  int* uni_s = reinterpret_cast<int*>(part + INIT_GMAX);     // [n]
  int a[4], b[4], c[K][4];
#pragma unroll 1
  for (int i = 0; i < n; ++i) {
    const int tile = tile0 + i, ty = tile / d.TX, tx = tile - ty * d.TX;
    energy_caps<K>(d, io, P, ty, tx, a, b, c);
    if (P.wf && P.fs) tile_init_regs<K, true, true>(d, io, gt0 + i, P, a, b, c, part + i, true);
    else if (P.wf) tile_init_regs<K, true, false>(d, io, gt0 + i, P, a, b, c, part + i, true);
    else if (P.fs) tile_init_regs<K, false, true>(d, io, gt0 + i, P, a, b, c, part + i, true);
    else tile_init_regs<K, false, false>(d, io, gt0 + i, P, a, b, c, part + i, true);
  }
  __syncthreads();
  init_finalize(d, gt0, n, part, uni_s);
}

}  // namespace gcb
