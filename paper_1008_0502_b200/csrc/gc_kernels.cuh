// gc_kernels.cuh -- sm_100a kernels of the grid min-cut hot path.
//
// Algorithm: push-relabel (Goldberg-Tarjan) on the pixel grid graph of P:331-357, run as
// tile-synchronous region discharges, with exact global relabels (BFS from the sink) as
// the termination certificate, and the canonical mask taken as the residual closure of
// the excess nodes.  The paper's GPU solver is "CUDA Cuts";
// this is a fresh B200 design, not a translation of it.
//
// State (tile-major, 32x32 tiles, frame padded to whole tiles):
//   e  [slot][tile][1024]     signed net excess: e = cs - ct + inflow - outflow.  e > 0 is
//                             excess (an "active" node), e < 0 is remaining residual
//                             capacity v -> t.  The terminal pair is pre-cancelled (a1).
//   h  [slot][tile][1024]     height / distance label (HINF = unreachable)
//   r  [slot][k][tile][1024]  residual capacity of arc v -> v + d_k
//   hedge [slot][tile][4][32] copy of the tile's boundary heights (top,bottom,left,right)
//   inbox [2][slot][tile][k][64]  flow pushed INTO the tile across its border, by arc
//                             direction and receiver edge slot; double-buffered by launch
//                             parity, written by the unique sender, zeroed by the receiver
//   reach [slot][tile][k][64] sticky min-cut reach bits arriving across the border
//   m, open [slot][tile][1024] mask bit and residual-arc bits (closure phase)
// No kernel uses global atomics on the push path; the only atomics are per-tile int64
// partial sums of the flow value.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace gcb {

constexpr int TS = 32;       // tile side
constexpr int TPX = 1024;    // pixels per tile
constexpr int NTH = 256;     // threads per CTA; thread t owns pixels (t/32 + 8j, t%32), j<4
constexpr int HINF = 0x3fffffff;
constexpr int CAPMAX = (1 << 26) - 1;
constexpr int HS = 34;       // halo'd height tile side

__host__ __device__ constexpr int DYk(int k) {
  return (k == 2 || k == 4 || k == 6) ? 1 : ((k == 3 || k == 5 || k == 7) ? -1 : 0);
}
__host__ __device__ constexpr int DXk(int k) {
  return (k == 0 || k == 4 || k == 7) ? 1 : ((k == 1 || k == 5 || k == 6) ? -1 : 0);
}

struct Dev {
  int H, W, TY, TX, T, nslot;
  int hmax;  // relabel cap: heights >= hmax are unreachable (HINF)
  int32_t* e;
  int32_t* h;
  int32_t* r;
  int32_t* hedge;
  int32_t* inbox;
  uint8_t* reach;
  uint8_t* m;
  uint8_t* open;
  int32_t* tact;   // [NS]   tile has an active node (e > 0, h < HINF)
  int32_t* bchg;   // [2][NS] tile boundary heights changed in the sweep of that parity
  int32_t* recv;   // [2][NS] tile has inbound flow in inbox of that parity
  int32_t* crecv;  // [2][NS] tile received new reach bits in the sweep of that parity
  int32_t* fdone;  // [nslot]
  int32_t* ferr;   // [nslot]
  int32_t* fstat;  // [nslot][4]
  unsigned long long* sumct;   // [nslot]
  unsigned long long* sumneg;  // [nslot]
  int32_t* ring;   // [64] per-sweep "something changed" flags
  int32_t* ctr;    // [8]
  unsigned long long* ptiles;  // [6] tiles processed per kernel class (profiling only, else NULL)
};

__device__ __forceinline__ void count_tile(const Dev& d, int cls) {
  if (d.ptiles && threadIdx.x == 0) atomicAdd(&d.ptiles[cls], 1ULL);
}

struct IO {
  const int32_t* cs;
  const int32_t* ct;
  const int32_t* nb;
  const int32_t* wf;
  int64_t* flow;
  uint8_t* mask;
  int32_t* fstate;
  int32_t* stats;
};

__device__ __forceinline__ size_t NS(const Dev& d) { return (size_t)d.nslot * d.T; }
__device__ __forceinline__ int32_t* Ep(const Dev& d, size_t gt) { return d.e + gt * TPX; }
__device__ __forceinline__ int32_t* Hp(const Dev& d, size_t gt) { return d.h + gt * TPX; }
__device__ __forceinline__ int32_t* Rp(const Dev& d, int K, int s, int k, int tile) {
  return d.r + (((size_t)s * K + k) * d.T + tile) * TPX;
}
__device__ __forceinline__ int32_t* INBp(const Dev& d, int K, int par, size_t gt, int k) {
  return d.inbox + (((size_t)par * NS(d) + gt) * K + k) * 64;
}

// Does arc (iy,ix) -> (iy,ix)+d_k leave the tile?
__device__ __forceinline__ bool crosses(int k, int iy, int ix) {
  int y2 = iy + DYk(k), x2 = ix + DXk(k);
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

// halo'd smem index of pixel (iy,ix) (which may be -1..32)
__device__ __forceinline__ int hidx(int iy, int ix) { return (iy + 1) * HS + (ix + 1); }

// Load the 34x34 halo ring of heights from the neighbours' boundary copies.
__device__ __forceinline__ void load_halo(const Dev& d, int s, int ty, int tx, int* hs, int t) {
  if (t < 128) {
    int side = t >> 5, i = t & 31;
    int nty = ty, ntx = tx, esd, pos;
    if (side == 0) { nty = ty - 1; esd = 1; pos = hidx(-1, i); }
    else if (side == 1) { nty = ty + 1; esd = 0; pos = hidx(32, i); }
    else if (side == 2) { ntx = tx - 1; esd = 3; pos = hidx(i, -1); }
    else { ntx = tx + 1; esd = 2; pos = hidx(i, 32); }
    int v = HINF;
    if (nty >= 0 && nty < d.TY && ntx >= 0 && ntx < d.TX)
      v = d.hedge[(((size_t)s * d.T + nty * d.TX + ntx) * 4 + esd) * 32 + i];
    hs[pos] = v;
  } else if (t < 132) {
    int c = t - 128;
    int dy = (c < 2) ? -1 : 1, dx = (c & 1) ? 1 : -1;
    int nty = ty + dy, ntx = tx + dx;
    int esd = dy < 0 ? 1 : 0;
    int i = dx < 0 ? 31 : 0;
    int v = HINF;
    if (nty >= 0 && nty < d.TY && ntx >= 0 && ntx < d.TX)
      v = d.hedge[(((size_t)s * d.T + nty * d.TX + ntx) * 4 + esd) * 32 + i];
    hs[hidx(dy < 0 ? -1 : 32, dx < 0 ? -1 : 32)] = v;
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

__device__ __forceinline__ bool on_border(int iy, int ix) { return iy == 0 || iy == 31 || ix == 0 || ix == 31; }

// Tile-local BFS fixpoint: h(v) = min(h(v), 1 + min{h(v+d_k) : r_k(v) > 0}) until stable.
// hs holds the halo'd heights (halo fixed); updates are written in place (monotone, so
// a racing reader sees an old or a new upper bound -- both valid).
template <int K>
__device__ __forceinline__ void bfs_fixpoint(volatile int* hs, const int (&r)[4][K], int (&h)[4], int t) {
  const int ix = t & 31, iy0 = t >> 5;
  for (;;) {
    int changed = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int iy = iy0 + 8 * j;
      if (h[j] > 1) {
        int mn = HINF;
#pragma unroll
        for (int k = 0; k < K; ++k)
          if (r[j][k] > 0) mn = min(mn, hs[hidx(iy + DYk(k), ix + DXk(k))]);
        if (mn < HINF && mn + 1 < h[j]) {
          h[j] = mn + 1;
          hs[hidx(iy, ix)] = h[j];
          changed = 1;
        }
      }
    }
    if (!__syncthreads_or(changed)) break;
  }
}

// ------------------------------------------------------------------------------ a1 / a1w
template <int K, bool WARM>
__global__ void __launch_bounds__(NTH) k_init(Dev d, IO io) {
  const int tile = blockIdx.x, s = blockIdx.y;
  const int ty = tile / d.TX, tx = tile - ty * d.TX;
  const int t = threadIdx.x, ix = t & 31, iy0 = t >> 5;
  const int H = d.H, W = d.W;
  const size_t plane = (size_t)H * W;
  const int32_t* cs = io.cs + s * plane;
  const int32_t* ct = io.ct + s * plane;
  const int32_t* nb = io.nb + s * plane * K;
  const int32_t* wf = WARM ? io.wf + s * plane * (K / 2) : nullptr;
  const size_t gt = (size_t)s * d.T + tile;
  count_tile(d, 0);
  int bad = 0;
  long long sct = 0;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int iy = iy0 + 8 * j, y = ty * TS + iy, x = tx * TS + ix, lp = iy * TS + ix;
    int ev = 0;
    int rk[K];
#pragma unroll
    for (int k = 0; k < K; ++k) rk[k] = 0;
    if (y < H && x < W) {
      const size_t o = (size_t)y * W + x;
      const int a = cs[o], b = ct[o];
      bad |= (a < 0) | (a > CAPMAX) | (b < 0) | (b > CAPMAX);
      ev = a - b;  // a1: pre-cancel min(cs,ct) straight s -> v -> t
      sct += b;
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const int y2 = y + DYk(k), x2 = x + DXk(k);
        if (y2 < 0 || y2 >= H || x2 < 0 || x2 >= W) continue;  // off-grid: ignored
        const int c = nb[k * plane + o];
        bad |= (c < 0) | (c > CAPMAX);
        if (!WARM) {
          rk[k] = c;
        } else {
          const size_t oq = (size_t)y2 * W + x2;
          if ((k & 1) == 0) {  // forward arc p -> q, flow stored at p
            const int cq = nb[(k ^ 1) * plane + oq];
            int f = wf[(k >> 1) * plane + o];
            f = max(-cq, min(c, f));  // a1w: clamp to the new capacities
            rk[k] = c - f;
            ev -= f;
          } else {  // reverse arc p -> q of the forward arc q -> p, flow stored at q
            const int cq = nb[(k ^ 1) * plane + oq];
            int f = wf[((k ^ 1) >> 1) * plane + oq];
            f = max(-c, min(cq, f));
            rk[k] = c + f;
            ev += f;
          }
        }
      }
    }
    Ep(d, gt)[lp] = ev;
#pragma unroll
    for (int k = 0; k < K; ++k) Rp(d, K, s, k, tile)[lp] = rk[k];
  }
  // clear the tile's message buffers and flags
  for (int i = t; i < 2 * K * 64; i += NTH) {
    const int par = i / (K * 64), rest = i - par * K * 64;
    INBp(d, K, par, gt, 0)[rest] = 0;
  }
  for (int i = t; i < K * 64; i += NTH) d.reach[gt * K * 64 + i] = 0;
  if (t == 0) {
    const size_t ns = NS(d);
    d.tact[gt] = 0;
    d.bchg[gt] = 0; d.bchg[ns + gt] = 0;
    d.recv[gt] = 0; d.recv[ns + gt] = 0;
    d.crecv[gt] = 0; d.crecv[ns + gt] = 0;
  }
  // frame reductions: sum of c(v,t) (for F) and the range flag
  bad = __syncthreads_or(bad);
  __shared__ long long red[NTH / 32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) sct += __shfl_xor_sync(0xffffffffu, sct, o);
  if ((t & 31) == 0) red[t >> 5] = sct;
  __syncthreads();
  if (t == 0) {
    long long tot = 0;
    for (int i = 0; i < NTH / 32; ++i) tot += red[i];
    if (tot) atomicAdd(&d.sumct[s], (unsigned long long)tot);
    if (bad) { d.ferr[s] = 1; d.fdone[s] = 1; }
  }
}

// Absorb the flow pushed into this tile in the previous launch (inbox parity `par`).
template <int K>
__device__ __forceinline__ void absorb(const Dev& d, int par, size_t gt, int (&e)[4], int (&r)[4][K], int t) {
  const int ix = t & 31, iy0 = t >> 5;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int iy = iy0 + 8 * j;
    if (!on_border(iy, ix)) continue;
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const int wy = iy - DYk(k), wx = ix - DXk(k);
      if ((unsigned)wy < 32u && (unsigned)wx < 32u) continue;
      int32_t* p = INBp(d, K, par, gt, k) + recv_slot(k, iy, ix);
      const int dl = *p;
      if (dl) {
        e[j] += dl;
        r[j][k ^ 1] += dl;  // residual u -> w grows by the flow w -> u
        *p = 0;
      }
    }
  }
}

// ------------------------------------------------------------------------------ a2 seed
// Global relabel, sweep 0: absorb in-flight flow, seed h = 1 on nodes with residual to t
// (e < 0), HINF elsewhere, and relax to the tile-local fixpoint with an INF halo.
template <int K>
__global__ void __launch_bounds__(NTH) k_bfs_seed(Dev d, int par_in, int sw) {
  const int tile = blockIdx.x, s = blockIdx.y;
  if (tile == 0 && s == 0 && threadIdx.x == 0) d.ring[(sw + 1) & 63] = 0;
  if (d.fdone[s]) return;
  count_tile(d, 1);
  const int t = threadIdx.x, ix = t & 31, iy0 = t >> 5;
  const size_t gt = (size_t)s * d.T + tile;
  const size_t ns = NS(d);
  __shared__ int hs[HS * HS];
  int e[4], r[4][K], h[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int lp = (iy0 + 8 * j) * TS + ix;
    e[j] = Ep(d, gt)[lp];
#pragma unroll
    for (int k = 0; k < K; ++k) r[j][k] = Rp(d, K, s, k, tile)[lp];
  }
  const int rcv = (par_in >= 0) ? d.recv[par_in * ns + gt] : 0;
  if (rcv) {
    absorb<K>(d, par_in, gt, e, r, t);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int lp = (iy0 + 8 * j) * TS + ix;
      Ep(d, gt)[lp] = e[j];
#pragma unroll
      for (int k = 0; k < K; ++k) Rp(d, K, s, k, tile)[lp] = r[j][k];
    }
    if (t == 0) d.recv[par_in * ns + gt] = 0;
  }
  for (int i = t; i < HS * HS; i += NTH) hs[i] = HINF;
  __syncthreads();
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    h[j] = e[j] < 0 ? 1 : HINF;
    hs[hidx(iy0 + 8 * j, ix)] = h[j];
  }
  __syncthreads();
  bfs_fixpoint<K>(hs, r, h, t);
  int act = 0;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    Hp(d, gt)[(iy0 + 8 * j) * TS + ix] = h[j];
    act |= (e[j] > 0) & (h[j] < HINF);
  }
  store_hedge(d, gt, h, t);
  act = __syncthreads_or(act);
  if (t == 0) {
    d.tact[gt] = act;
    d.bchg[(sw & 1) * ns + gt] = 1;
  }
}

// ------------------------------------------------------------------------------ a2 relax
// Global relabel, sweep sw >= 1: re-relax tiles whose neighbours' boundary heights changed
// in the previous sweep, until no boundary changes anywhere (exact BFS distances).
template <int K>
__global__ void __launch_bounds__(NTH) k_bfs_relax(Dev d, int sw) {
  const int tile = blockIdx.x, s = blockIdx.y;
  const int t = threadIdx.x, ix = t & 31, iy0 = t >> 5;
  if (tile == 0 && s == 0 && t == 0) d.ring[(sw + 1) & 63] = 0;
  if (d.fdone[s]) return;
  const int ty = tile / d.TX, tx = tile - ty * d.TX;
  const size_t gt = (size_t)s * d.T + tile;
  const size_t ns = NS(d);
  const int cur = sw & 1, prv = cur ^ 1;
  int need = 0;
  if (t < 9 && t != 4) {
    const int nty = ty + t / 3 - 1, ntx = tx + t % 3 - 1;
    if (nty >= 0 && nty < d.TY && ntx >= 0 && ntx < d.TX)
      need = d.bchg[prv * ns + (size_t)s * d.T + nty * d.TX + ntx];
  }
  need = __syncthreads_or(need);
  if (!need) {
    if (t == 0) d.bchg[cur * ns + gt] = 0;
    return;
  }
  count_tile(d, 1);
  __shared__ int hs[HS * HS];
  int e[4], r[4][K], h[4], h0[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int lp = (iy0 + 8 * j) * TS + ix;
    e[j] = Ep(d, gt)[lp];
    h[j] = h0[j] = Hp(d, gt)[lp];
#pragma unroll
    for (int k = 0; k < K; ++k) r[j][k] = Rp(d, K, s, k, tile)[lp];
    hs[hidx(iy0 + 8 * j, ix)] = h[j];
  }
  load_halo(d, s, ty, tx, hs, t);
  __syncthreads();
  bfs_fixpoint<K>(hs, r, h, t);
  int any = 0, bnd = 0, act = 0;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int iy = iy0 + 8 * j;
    const int ch = h[j] != h0[j];
    any |= ch;
    bnd |= ch & on_border(iy, ix);
    act |= (e[j] > 0) & (h[j] < HINF);
  }
  any = __syncthreads_or(any);
  if (any) {
#pragma unroll
    for (int j = 0; j < 4; ++j) Hp(d, gt)[(iy0 + 8 * j) * TS + ix] = h[j];
    store_hedge(d, gt, h, t);
  }
  bnd = __syncthreads_or(bnd);
  act = __syncthreads_or(act);
  if (t == 0) {
    if (any) d.tact[gt] = act;
    d.bchg[cur * ns + gt] = bnd;
    if (bnd) d.ring[sw & 63] = 1;
  }
}

// ------------------------------------------------------------------------------ status
// Frame is done when no tile holds an active node that can reach the sink (after an exact
// global relabel): that preflow is maximum (termination certificate).
__global__ void __launch_bounds__(NTH) k_status(Dev d, int pushes, int relabels, int sweeps) {
  const int s = blockIdx.x, t = threadIdx.x;
  if (d.fdone[s]) return;
  count_tile(d, 3);
  int any = 0;
  for (int i = t; i < d.T; i += NTH) any |= d.tact[(size_t)s * d.T + i];
  any = __syncthreads_or(any);
  if (t == 0) {
    if (!any) {
      d.fdone[s] = 1;
      d.fstat[s * 4 + 0] = pushes;
      d.fstat[s * 4 + 1] = relabels;
      d.fstat[s * 4 + 2] = sweeps;
    } else {
      atomicAdd(&d.ctr[0], 1);
    }
  }
}

// ------------------------------------------------------------------------------ a3 push
// One launch of `rounds` synchronous push / gather / relabel rounds inside each tile.
// Pushes are decided by the owner (it lowers its own e and r); receivers inside the tile
// gather them in a separate phase; pushes across the tile border go to the receiver
// tile's inbox and are absorbed at its next launch.  Border heights are those of the
// previous launch (stale); the exact global relabel restores valid labels.
template <int K>
__global__ void __launch_bounds__(NTH) k_push(Dev d, int par_in, int par_out, int rounds) {
  const int tile = blockIdx.x, s = blockIdx.y;
  if (d.fdone[s]) return;
  const int t = threadIdx.x, ix = t & 31, iy0 = t >> 5;
  const size_t gt = (size_t)s * d.T + tile;
  const size_t ns = NS(d);
  const int rcv = (par_in >= 0) ? d.recv[par_in * ns + gt] : 0;
  if (!d.tact[gt] && !rcv) return;
  count_tile(d, 2);
  const int ty = tile / d.TX, tx = tile - ty * d.TX;
  __shared__ int hs[HS * HS];
  __shared__ int ps[K][TPX];
  __shared__ int oacc[K][64];
  int e[4], r[4][K], h[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int lp = (iy0 + 8 * j) * TS + ix;
    e[j] = Ep(d, gt)[lp];
    h[j] = Hp(d, gt)[lp];
#pragma unroll
    for (int k = 0; k < K; ++k) r[j][k] = Rp(d, K, s, k, tile)[lp];
  }
  if (rcv) {
    absorb<K>(d, par_in, gt, e, r, t);
    if (t == 0) d.recv[par_in * ns + gt] = 0;
  }
#pragma unroll
  for (int j = 0; j < 4; ++j) hs[hidx(iy0 + 8 * j, ix)] = h[j];
  load_halo(d, s, ty, tx, hs, t);
  for (int i = t; i < K * 64; i += NTH) (&oacc[0][0])[i] = 0;
  __syncthreads();
  const int hmax = d.hmax;
  for (int rd = 0; rd < rounds; ++rd) {
    // push phase (owner)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int iy = iy0 + 8 * j, lp = iy * TS + ix;
      int ee = e[j];
      const int hv = h[j];
      const bool act = ee > 0 && hv < HINF;
#pragma unroll
      for (int k = 0; k < K; ++k) {
        int dl = 0;
        if (act && ee > 0 && r[j][k] > 0 && hs[hidx(iy + DYk(k), ix + DXk(k))] == hv - 1) {
          dl = min(ee, r[j][k]);
          ee -= dl;
          r[j][k] -= dl;
        }
        if (crosses(k, iy, ix)) {
          if (dl) {
            const int uy = (iy + DYk(k)) & 31, ux = (ix + DXk(k)) & 31;
            oacc[k][recv_slot(k, uy, ux)] += dl;
          }
        } else {
          ps[k][lp] = dl;
        }
      }
      e[j] = ee;
    }
    __syncthreads();
    // gather phase (receiver) + relabel decision
    int hn[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int iy = iy0 + 8 * j;
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const int wy = iy - DYk(k), wx = ix - DXk(k);
        if ((unsigned)wy < 32u && (unsigned)wx < 32u) {
          const int dl = ps[k][wy * TS + wx];
          e[j] += dl;
          r[j][k ^ 1] += dl;
        }
      }
      hn[j] = h[j];
      if (e[j] > 0 && h[j] < HINF) {
        int mn = HINF;
        bool adm = false;
#pragma unroll
        for (int k = 0; k < K; ++k) {
          if (r[j][k] > 0) {
            const int hu = hs[hidx(iy + DYk(k), ix + DXk(k))];
            adm |= (hu == h[j] - 1);
            mn = min(mn, hu);
          }
        }
        if (!adm) hn[j] = (mn >= hmax - 1) ? HINF : mn + 1;
      }
    }
    __syncthreads();
    int still = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      h[j] = hn[j];
      hs[hidx(iy0 + 8 * j, ix)] = hn[j];
      still |= (e[j] > 0) & (hn[j] < HINF);
    }
    if (!__syncthreads_or(still)) break;  // tile discharged: nothing left to push
  }
  // store state
  int act = 0;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int lp = (iy0 + 8 * j) * TS + ix;
    Ep(d, gt)[lp] = e[j];
    Hp(d, gt)[lp] = h[j];
#pragma unroll
    for (int k = 0; k < K; ++k) Rp(d, K, s, k, tile)[lp] = r[j][k];
    act |= (e[j] > 0) & (h[j] < HINF);
  }
  store_hedge(d, gt, h, t);
  // send border pushes to the neighbours' inboxes (unique writer per slot)
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int iy = iy0 + 8 * j;
    if (!on_border(iy, ix)) continue;
#pragma unroll
    for (int k = 0; k < K; ++k) {
      if (!crosses(k, iy, ix)) continue;
      const int y2 = iy + DYk(k), x2 = ix + DXk(k);
      const int uy = y2 & 31, ux = x2 & 31;
      const int sl = recv_slot(k, uy, ux);
      const int dl = oacc[k][sl];
      if (dl) {
        const int rty = ty + (y2 < 0 ? -1 : (y2 > 31 ? 1 : 0));
        const int rtx = tx + (x2 < 0 ? -1 : (x2 > 31 ? 1 : 0));
        const size_t rgt = (size_t)s * d.T + rty * d.TX + rtx;
        INBp(d, K, par_out, rgt, k)[sl] = dl;
        d.recv[par_out * ns + rgt] = 1;
      }
    }
  }
  act = __syncthreads_or(act);
  if (t == 0) d.tact[gt] = act;
}

// ------------------------------------------------------------------------------ a4 closure
// mask = closure of {v : e(v) > 0} under arcs with positive residual: the
// source side of the inclusion-minimal minimum cut.  Sweep 0 seeds every tile; later
// sweeps process tiles that received new reach bits across their border.
template <int K>
__device__ __forceinline__ void closure_fixpoint(volatile uint8_t* ms, const uint8_t* os, int (&mm)[4], int t) {
  const int ix = t & 31, iy0 = t >> 5;
  for (;;) {
    int changed = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      if (mm[j]) continue;
      const int iy = iy0 + 8 * j;
      int got = 0;
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const int wy = iy - DYk(k), wx = ix - DXk(k);
        if ((unsigned)wy < 32u && (unsigned)wx < 32u) {
          const int w = wy * TS + wx;
          got |= ms[w] & (os[w] >> k) & 1;
        }
      }
      if (got) {
        mm[j] = 1;
        ms[iy * TS + ix] = 1;
        changed = 1;
      }
    }
    if (!__syncthreads_or(changed)) break;
  }
}

template <int K>
__device__ __forceinline__ int closure_send(const Dev& d, int s, int ty, int tx, const int (&mm)[4],
                                            const int (&send)[4], const uint8_t* os, int par_out, int t) {
  const int ix = t & 31, iy0 = t >> 5;
  const size_t ns = NS(d);
  int sent = 0;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int iy = iy0 + 8 * j;
    if (!send[j] || !on_border(iy, ix)) continue;
    const int ob = os[iy * TS + ix];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      if (!crosses(k, iy, ix) || !((ob >> k) & 1)) continue;
      const int y2 = iy + DYk(k), x2 = ix + DXk(k);
      const int rty = ty + (y2 < 0 ? -1 : (y2 > 31 ? 1 : 0));
      const int rtx = tx + (x2 < 0 ? -1 : (x2 > 31 ? 1 : 0));
      if (rty < 0 || rty >= d.TY || rtx < 0 || rtx >= d.TX) continue;
      const size_t rgt = (size_t)s * d.T + rty * d.TX + rtx;
      d.reach[(rgt * K + k) * 64 + recv_slot(k, y2 & 31, x2 & 31)] = 1;
      d.crecv[par_out * ns + rgt] = 1;
      sent = 1;
    }
  }
  return sent;
}

template <int K>
__global__ void __launch_bounds__(NTH) k_closure_seed(Dev d, int sw) {
  const int tile = blockIdx.x, s = blockIdx.y;
  const int t = threadIdx.x, ix = t & 31, iy0 = t >> 5;
  if (tile == 0 && s == 0 && t == 0) d.ring[(sw + 1) & 63] = 0;
  if (d.ferr[s]) return;
  count_tile(d, 4);
  const int ty = tile / d.TX, tx = tile - ty * d.TX;
  const size_t gt = (size_t)s * d.T + tile;
  __shared__ uint8_t ms[TPX];
  __shared__ uint8_t os[TPX];
  int mm[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int lp = (iy0 + 8 * j) * TS + ix;
    const int ev = Ep(d, gt)[lp];
    int ob = 0;
#pragma unroll
    for (int k = 0; k < K; ++k) ob |= (Rp(d, K, s, k, tile)[lp] > 0) << k;
    mm[j] = ev > 0;
    ms[lp] = (uint8_t)mm[j];
    os[lp] = (uint8_t)ob;
    d.open[gt * TPX + lp] = (uint8_t)ob;
  }
  __syncthreads();
  closure_fixpoint<K>(ms, os, mm, t);
#pragma unroll
  for (int j = 0; j < 4; ++j) d.m[gt * TPX + (iy0 + 8 * j) * TS + ix] = (uint8_t)mm[j];
  int sent = closure_send<K>(d, s, ty, tx, mm, mm, os, sw & 1, t);
  sent = __syncthreads_or(sent);
  if (t == 0 && sent) d.ring[sw & 63] = 1;
}

template <int K>
__global__ void __launch_bounds__(NTH) k_closure_relax(Dev d, int sw) {
  const int tile = blockIdx.x, s = blockIdx.y;
  const int t = threadIdx.x, ix = t & 31, iy0 = t >> 5;
  if (tile == 0 && s == 0 && t == 0) d.ring[(sw + 1) & 63] = 0;
  if (d.ferr[s]) return;
  const size_t gt = (size_t)s * d.T + tile;
  const size_t ns = NS(d);
  const int cur = sw & 1, prv = cur ^ 1;
  if (!d.crecv[prv * ns + gt]) return;
  count_tile(d, 4);
  const int ty = tile / d.TX, tx = tile - ty * d.TX;
  __shared__ uint8_t ms[TPX];
  __shared__ uint8_t os[TPX];
  int mm[4], m0[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int iy = iy0 + 8 * j, lp = iy * TS + ix;
    m0[j] = d.m[gt * TPX + lp];
    os[lp] = d.open[gt * TPX + lp];
    int got = m0[j];
    if (!got && on_border(iy, ix)) {
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const int wy = iy - DYk(k), wx = ix - DXk(k);
        if ((unsigned)wy < 32u && (unsigned)wx < 32u) continue;
        got |= d.reach[(gt * K + k) * 64 + recv_slot(k, iy, ix)];
      }
    }
    mm[j] = got;
    ms[lp] = (uint8_t)got;
  }
  __syncthreads();
  if (t == 0) d.crecv[prv * ns + gt] = 0;
  closure_fixpoint<K>(ms, os, mm, t);
  int nw[4], any = 0;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    nw[j] = mm[j] & !m0[j];
    any |= nw[j];
  }
  any = __syncthreads_or(any);
  if (!any) return;
#pragma unroll
  for (int j = 0; j < 4; ++j)
    if (nw[j]) d.m[gt * TPX + (iy0 + 8 * j) * TS + ix] = 1;
  int sent = closure_send<K>(d, s, ty, tx, mm, nw, os, cur, t);
  sent = __syncthreads_or(sent);
  if (t == 0 && sent) d.ring[sw & 63] = 1;
}

// ------------------------------------------------------------------------------ a4/a5 out
template <int K>
__global__ void __launch_bounds__(NTH) k_finalize(Dev d, IO io) {
  const int tile = blockIdx.x, s = blockIdx.y;
  const int ty = tile / d.TX, tx = tile - ty * d.TX;
  const int t = threadIdx.x, ix = t & 31, iy0 = t >> 5;
  const int H = d.H, W = d.W;
  const size_t plane = (size_t)H * W;
  const size_t gt = (size_t)s * d.T + tile;
  count_tile(d, 5);
  const int err = d.ferr[s];
  long long neg = 0;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int iy = iy0 + 8 * j, y = ty * TS + iy, x = tx * TS + ix, lp = iy * TS + ix;
    if (y >= H || x >= W) continue;
    const size_t o = (size_t)y * W + x;
    io.mask[s * plane + o] = err ? 0 : d.m[gt * TPX + lp];
    const int ev = Ep(d, gt)[lp];
    neg += ev < 0 ? -(long long)ev : 0;
    if (io.fstate) {
#pragma unroll
      for (int k = 0; k < K; k += 2) {
        const int y2 = y + DYk(k), x2 = x + DXk(k);
        int f = 0;
        if (!err && y2 >= 0 && y2 < H && x2 >= 0 && x2 < W)
          f = io.nb[s * plane * K + k * plane + o] - Rp(d, K, s, k, tile)[lp];  // a5: f = c - r
        io.fstate[s * plane * (K / 2) + (k >> 1) * plane + o] = f;
      }
    }
  }
  __shared__ long long red[NTH / 32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) neg += __shfl_xor_sync(0xffffffffu, neg, o);
  if ((t & 31) == 0) red[t >> 5] = neg;
  __syncthreads();
  if (t == 0) {
    long long tot = 0;
    for (int i = 0; i < NTH / 32; ++i) tot += red[i];
    if (tot) atomicAdd(&d.sumneg[s], (unsigned long long)tot);
  }
}

// F = sum c(v,t) - sum max(0, -e): the flow that reached t.
__global__ void k_flow(Dev d, IO io) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= d.nslot) return;
  int st = 0;
  long long F = (long long)d.sumct[s] - (long long)d.sumneg[s];
  if (d.ferr[s]) { st = 2; F = -1; }
  else if (!d.fdone[s]) { st = 5; F = -1; }
  io.flow[s] = F;
  if (io.stats) {
    io.stats[s * 4 + 0] = d.fstat[s * 4 + 0];
    io.stats[s * 4 + 1] = d.fstat[s * 4 + 1];
    io.stats[s * 4 + 2] = d.fstat[s * 4 + 2];
    io.stats[s * 4 + 3] = st;
  }
  if (st) atomicAdd(&d.ctr[st == 2 ? 1 : 2], 1);
}

}  // namespace gcb
