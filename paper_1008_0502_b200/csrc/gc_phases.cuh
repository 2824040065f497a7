// gc_phases.cuh -- the per-step kernels of the device-side solve loop.
//
// The context holds `nslot` frame slots.  Every slot runs its own state machine (d.fmode),
// advanced once per step by k_control; a slot whose frame finishes is refilled with the next
// frame of the batch on the device (continuous batching), so easy and hard frames never wait
// for each other:
//   M_INIT   -- streaming pass over the caps: fl bit-planes, sum c(v,t), range check (a1/a1w)
//   M_SEED   -- global relabel, seed pass: absorb in-flight flow, h = 1 on nodes with
//               residual capacity to t, tile-local BFS fixpoint                     (a2)
//   M_BFS    -- global relabel, relax passes over tiles whose neighbours' border heights
//               changed; ends when a step changes nothing (exact BFS distances)      (a2)
//               then: no active node left -> M_CSEED, else -> M_PUSH
//   M_PUSH   -- push/relabel over active tiles (a3); ends (-> M_SEED) when the frame stops
//               delivering flow to sink-connected nodes and reaching new tiles, or when the
//               relabel budget of Goldberg's global-relabel heuristic is spent
//   M_CSEED  -- canonical mask, seed pass over every tile; writes the caller's mask    (a4)
//   M_CLOS   -- mask closure across tile borders until nothing changes               (a4)
//   M_EXPORT -- forward-arc flows for the caller's warm-start state                 (a5)
//   then the flow value is written and the slot takes the next frame (M_INIT) or idles.
// One step = k_stream (INIT/EXPORT) + k_seed (SEED/CSEED) + k_relax (BFS/CLOS) + k_push
// (PUSH) + k_control.  Each kernel walks the compact list of slots of its group that
// k_control built for this step.  Parities (dirty, inbox, reach flags) follow the global
// step counter sw.
#pragma once
#include "gc_kernels.cuh"

namespace gcb {

enum { G_STREAM = 0, G_SEED = 1, G_RELAX = 2, G_PUSH = 3, NGROUP = 4 };

__host__ __device__ __forceinline__ int mode_group(int md) {
  return (md == M_INIT || md == M_EXPORT) ? G_STREAM
         : (md == M_SEED || md == M_CSEED) ? G_SEED
         : (md == M_BFS || md == M_CLOS)   ? G_RELAX
                                           : G_PUSH;
}

// Mark the neighbour tiles that read a changed part of this tile's border.
__device__ __forceinline__ void mark_neighbours(const Dev& d, int32_t* flags, size_t gt, int bits, int K) {
  const int t = threadIdx.x;
  if (t < 8 && ((bits >> t) & 1)) {
    // bit: 0 N, 1 S, 2 W, 3 E, 4 NW, 5 NE, 6 SW, 7 SE
    const int dy = (t == 0 || t == 4 || t == 5) ? -1 : ((t == 1 || t == 6 || t == 7) ? 1 : 0);
    const int dx = (t == 2 || t == 4 || t == 6) ? -1 : ((t == 3 || t == 5 || t == 7) ? 1 : 0);
    if (t >= 4 && K == 4) return;
    const int s = (int)(gt / d.T), tile = (int)(gt - (size_t)s * d.T);
    const int ty = tile / d.TX + dy, tx = tile % d.TX + dx;
    if (ty >= 0 && ty < d.TY && tx >= 0 && tx < d.TX) flags[(size_t)s * d.T + ty * d.TX + tx] = 1;
  }
}

__device__ __forceinline__ int border_bits(int iy, int ix) {
  int b = 0;
  b |= (iy == 0) << 0;
  b |= (iy == 31) << 1;
  b |= (ix == 0) << 2;
  b |= (ix == 31) << 3;
  b |= (iy == 0 && ix == 0) << 4;
  b |= (iy == 0 && ix == 31) << 5;
  b |= (iy == 31 && ix == 0) << 6;
  b |= (iy == 31 && ix == 31) << 7;
  return b;
}

// Persistent-grid worklist over the tiles of the slots listed for group G in this step:
// each CTA takes ids blockIdx.x, +gridDim.x, ... 256 at a time, compacts those passing
// TILEPRED in shared memory and processes them one by one (block-wide body).
#define GC_LIST_BEGIN(G, TILEPRED)                                                        \
  __shared__ int wl_[NTH];                                                                \
  __shared__ int wn_;                                                                     \
  const size_t ns_ = NS(d);                                                               \
  const int lb_ = sw & 1;                                                                 \
  const int cnt_ = d.lcnt[lb_ * NGROUP + (G)];                                            \
  const int* sl_ = d.slist + ((size_t)lb_ * NGROUP + (G)) * d.nslot;                      \
  const size_t tot_ = (size_t)cnt_ * d.T;                                                 \
  for (size_t base_ = 0; base_ < tot_; base_ += (size_t)NTH * gridDim.x) {                \
    const size_t k_ = base_ + (size_t)threadIdx.x * gridDim.x + blockIdx.x;               \
    int want_ = 0;                                                                        \
    size_t id = 0;                                                                        \
    if (k_ < tot_) {                                                                      \
      const int li_ = (int)(k_ / d.T);                                                    \
      id = (size_t)sl_[li_] * d.T + (k_ - (size_t)li_ * d.T);                             \
      want_ = (TILEPRED);                                                                 \
    }                                                                                     \
    if (threadIdx.x == 0) wn_ = 0;                                                        \
    __syncthreads();                                                                      \
    if (want_) wl_[atomicAdd(&wn_, 1)] = (int)id;                                         \
    __syncthreads();                                                                      \
    const int n_ = wn_;                                                                   \
    for (int i_ = 0; i_ < n_; ++i_) {                                                     \
      const size_t gt = (size_t)wl_[i_];                                                  \
      const int md = d.fmode[gt / d.T];
#define GC_LIST_END \
  __syncthreads();  \
  }                 \
  __syncthreads();  \
  }

// ---------------------------------------------------------------- a2: seed pass (one tile)
template <int K>
__device__ __forceinline__ void tile_seed(const Dev& d, const IO& io, size_t gt, int sw, int* hs) {
  const int t = threadIdx.x, ix = t & 31, iy0 = t >> 5;
  const size_t ns = NS(d);
  const int s = (int)(gt / d.T);
  const int par_in = (sw - 1) & 1;
  int fl[4];
  if (d.recv[par_in * ns + gt]) {  // flow still in flight from the last push step
    const int tile = (int)(gt - (size_t)s * d.T);
    const int ty = tile / d.TX, tx = tile - ty * d.TX;
#pragma unroll 1
    for (int j = 0; j < 4; ++j) {  // pixel at a time: materialise, absorb, store
      const int iy = iy0 + 8 * j, lp = iy * TS + ix;
      int e, r[K];
      px_er<K>(d, io, gt, lp, ty * TS + iy, tx * TS + ix, e, r);
      if (on_border(iy, ix)) {
#pragma unroll
        for (int k = 0; k < K; ++k) {
          const int wy = iy - DYk(k), wx = ix - DXk(k);
          if ((unsigned)wy < 32u && (unsigned)wx < 32u) continue;
          int32_t* p = INBp(d, K, par_in, gt, k) + recv_slot(k, iy, ix);
          const int dl = *p;
          if (dl) { e += dl; r[k ^ 1] += dl; *p = 0; }
        }
      }
      d.e[gt * TPX + lp] = e;
#pragma unroll
      for (int k = 0; k < K; ++k) Rp(d, K, gt, k)[lp] = r[k];
      fl[j] = make_fl<K>(e, r);
      d.fl[gt * TPX + lp] = (uint16_t)fl[j];
    }
    __syncthreads();
    if (t == 0) { d.mat[gt] = 1; d.recv[par_in * ns + gt] = 0; }
  } else {
#pragma unroll
    for (int j = 0; j < 4; ++j) fl[j] = d.fl[gt * TPX + (iy0 + 8 * j) * TS + ix];
  }
  const int act = bfs_seed_tile<K>(d, gt, hs, fl);
  if (t == 0) {
    d.tact[gt] = act;
    d.dirty[(sw & 1) * ns + gt] = 1;
    d.fchg[(sw & 1) * d.nslot + s] = 1;
  }
}

// ---------------------------------------------------------------- a2: relax pass (one tile)
template <int K>
__device__ __forceinline__ void tile_relax(const Dev& d, size_t gt, int sw, int* hs, int* bits_s) {
  const int t = threadIdx.x, ix = t & 31, iy0 = t >> 5;
  const size_t ns = NS(d);
  const int cur = sw & 1, prv = cur ^ 1;
  const int s = (int)(gt / d.T), tile = (int)(gt - (size_t)s * d.T);
  const int ty = tile / d.TX, tx = tile - ty * d.TX;
  if (t == 0) { d.dirty[prv * ns + gt] = 0; *bits_s = 0; }
  int fl[4], h[4], h0[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int lp = (iy0 + 8 * j) * TS + ix;
    fl[j] = d.fl[gt * TPX + lp];
    h[j] = h0[j] = d.h[gt * TPX + lp];
    hs[hidx(iy0 + 8 * j, ix)] = h[j];
  }
  load_halo(d, s, ty, tx, hs, t);
  __syncthreads();
  bfs_fixpoint<K>(hs, fl, h);
  int any = 0, bits = 0, act = 0;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int ch = h[j] != h0[j];
    any |= ch;
    if (ch) bits |= border_bits(iy0 + 8 * j, ix);
    act |= (fl[j] & FL_POS) && h[j] < HINF;
  }
  if (bits) atomicOr(bits_s, bits);
  any = __syncthreads_or(any);
  act = __syncthreads_or(act);
  if (any) {
#pragma unroll
    for (int j = 0; j < 4; ++j) d.h[gt * TPX + (iy0 + 8 * j) * TS + ix] = h[j];
    store_hedge(d, gt, h, t);
    if (t == 0) d.tact[gt] = act;
  }
  const int b = *bits_s;
  if (b) {
    mark_neighbours(d, d.dirty + cur * ns, gt, b, K);
    if (t == 0) d.fchg[cur * d.nslot + s] = 1;
  }
}

// ---------------------------------------------------------------- a4: closure helpers
// mask = closure of {v : e(v) > 0} under arcs with positive residual: the
// source side of the inclusion-minimal minimum cut.
template <int K>
__device__ __forceinline__ void closure_fixpoint(volatile uint8_t* ms, const uint8_t* os, int (&mm)[4]) {
  const int t = threadIdx.x, ix = t & 31, iy0 = t >> 5;
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
__device__ __forceinline__ int closure_send(const Dev& d, size_t gt, const int (&send)[4], const uint8_t* os,
                                            int par_out) {
  const int t = threadIdx.x, ix = t & 31, iy0 = t >> 5;
  const size_t ns = NS(d);
  const int s = (int)(gt / d.T), tile = (int)(gt - (size_t)s * d.T);
  const int ty = tile / d.TX, tx = tile - ty * d.TX;
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

__device__ __forceinline__ void write_mask(const Dev& d, const IO& io, size_t gt, const int (&mm)[4],
                                           const int (&wr)[4]) {
  const int t = threadIdx.x, ix = t & 31, iy0 = t >> 5;
  const int s = (int)(gt / d.T), tile = (int)(gt - (size_t)s * d.T);
  const int ty = tile / d.TX, tx = tile - ty * d.TX;
  const size_t plane = (size_t)d.H * d.W;
  uint8_t* mask = io.mask + (size_t)d.sfr[s] * plane;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int y = ty * TS + iy0 + 8 * j, x = tx * TS + ix;
    if (wr[j] && y < d.H && x < d.W) mask[(size_t)y * d.W + x] = (uint8_t)mm[j];
  }
}

// ---------------------------------------------------------------- a4: closure seed (one tile)
// Every tile: m = (e > 0) closed inside the tile; writes m and the caller's mask; sends
// reach bits across the border; adds the tile's sum max(0,-e) to the flow value's sum.
template <int K>
__device__ __forceinline__ void tile_cseed(const Dev& d, const IO& io, size_t gt, int sw, uint8_t* ms, uint8_t* os,
                                           long long* red) {
  const int t = threadIdx.x, ix = t & 31, iy0 = t >> 5;
  const int s = (int)(gt / d.T);
  const int all[4] = {1, 1, 1, 1};
  if (d.ferr[s]) {  // range error: mask all 0, F = -1
    const int z[4] = {0, 0, 0, 0};
    write_mask(d, io, gt, z, all);
    return;
  }
  int mm[4];
  const int mat = d.mat[gt];
  long long neg = 0;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int lp = (iy0 + 8 * j) * TS + ix;
    const int f = d.fl[gt * TPX + lp];
    mm[j] = (f & FL_POS) ? 1 : 0;
    ms[lp] = (uint8_t)mm[j];
    os[lp] = (uint8_t)(f & 0xff);
    if (mat) {
      const int ev = d.e[gt * TPX + lp];
      neg += ev < 0 ? -(long long)ev : 0;
    }
  }
  __syncthreads();
  closure_fixpoint<K>(ms, os, mm);
#pragma unroll
  for (int j = 0; j < 4; ++j) d.m[gt * TPX + (iy0 + 8 * j) * TS + ix] = (uint8_t)mm[j];
  write_mask(d, io, gt, mm, all);
  int sent = closure_send<K>(d, gt, mm, os, sw & 1);
  sent = __syncthreads_or(sent);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) neg += __shfl_xor_sync(0xffffffffu, neg, o);
  if ((t & 31) == 0) red[t >> 5] = neg;
  __syncthreads();
  if (t == 0) {
    long long tot = 0;
    if (mat) {
      for (int i = 0; i < NTH / 32; ++i) tot += red[i];
    } else {
      tot = d.neg0[gt];
    }
    if (tot) atomicAdd(&d.sumneg[s], (unsigned long long)tot);
    if (sent) d.fchg[(sw & 1) * d.nslot + s] = 1;
  }
}

// ---------------------------------------------------------------- a4: closure relax (one tile)
template <int K>
__device__ __forceinline__ void tile_crelax(const Dev& d, const IO& io, size_t gt, int sw, uint8_t* ms, uint8_t* os) {
  const int t = threadIdx.x, ix = t & 31, iy0 = t >> 5;
  const size_t ns = NS(d);
  const int cur = sw & 1, prv = cur ^ 1;
  const int s = (int)(gt / d.T);
  int mm[4], m0[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int iy = iy0 + 8 * j, lp = iy * TS + ix;
    m0[j] = d.m[gt * TPX + lp];
    os[lp] = (uint8_t)(d.fl[gt * TPX + lp] & 0xff);
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
  closure_fixpoint<K>(ms, os, mm);
  int nw[4], any = 0;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    nw[j] = mm[j] & !m0[j];
    any |= nw[j];
  }
  any = __syncthreads_or(any);
  if (any) {
#pragma unroll
    for (int j = 0; j < 4; ++j)
      if (nw[j]) d.m[gt * TPX + (iy0 + 8 * j) * TS + ix] = 1;
    write_mask(d, io, gt, mm, nw);
    int sent = closure_send<K>(d, gt, nw, os, cur);
    sent = __syncthreads_or(sent);
    if (t == 0 && sent) d.fchg[cur * d.nslot + s] = 1;
  }
}

// ---------------------------------------------------------------- a5: export (one tile)
// Forward-arc flows f = c - r of this solve (the next frame's warm start).
template <int K>
__device__ __forceinline__ void tile_export(const Dev& d, const IO& io, size_t gt) {
  const int s = (int)(gt / d.T), tile = (int)(gt - (size_t)s * d.T);
  const int ty = tile / d.TX, tx = tile - ty * d.TX;
  const int t = threadIdx.x, ix = t & 31, iy0 = t >> 5;
  const int H = d.H, W = d.W;
  const size_t plane = (size_t)H * W;
  const size_t fr = (size_t)d.sfr[s];
#pragma unroll 1
  for (int j = 0; j < 4; ++j) {
    const int y = ty * TS + iy0 + 8 * j, x = tx * TS + ix;
    if (y >= H || x >= W) continue;
    int e, r[K];
    px_er<K>(d, io, gt, (iy0 + 8 * j) * TS + ix, y, x, e, r);
    const size_t o = (size_t)y * W + x;
#pragma unroll
    for (int k = 0; k < K; k += 2) {
      const int y2 = y + DYk(k), x2 = x + DXk(k);
      int f = 0;
      if (y2 >= 0 && y2 < H && x2 >= 0 && x2 < W) f = io.nb[fr * plane * K + k * plane + o] - r[k];
      io.fstate[fr * plane * (K / 2) + (k >> 1) * plane + o] = f;
    }
  }
}

// ---------------------------------------------------------------- step kernels
template <int K>
__global__ void __launch_bounds__(NTH, 4) k_stream(Dev d, IO io, int sw, int vec) {
  __shared__ long long red[2][NTH / 32];
  GC_LIST_BEGIN(G_STREAM, 1)
  if (md == M_INIT) {
    count_tile(d, 0);
    tile_init<K>(d, io, gt, vec != 0, red);
  } else {
    count_tile(d, 5);
    tile_export<K>(d, io, gt);
  }
  GC_LIST_END
}

template <int K>
__global__ void __launch_bounds__(NTH, 4) k_seed(Dev d, IO io, int sw) {
  __shared__ int hs[HS * HS];
  __shared__ long long red[NTH / 32];
  uint8_t* ms = reinterpret_cast<uint8_t*>(hs);  // closure tiles reuse the height buffer
  uint8_t* os = ms + TPX;
  GC_LIST_BEGIN(G_SEED, 1)
  if (md == M_SEED) {
    count_tile(d, 1);
    tile_seed<K>(d, io, gt, sw, hs);
  } else {
    count_tile(d, 4);
    tile_cseed<K>(d, io, gt, sw, ms, os, red);
  }
  GC_LIST_END
}

template <int K>
__global__ void __launch_bounds__(NTH, 4) k_relax(Dev d, IO io, int sw) {
  __shared__ int hs[HS * HS];
  __shared__ int bits_s;
  uint8_t* ms = reinterpret_cast<uint8_t*>(hs);
  uint8_t* os = ms + TPX;
  const int prv = (sw & 1) ^ 1;
  GC_LIST_BEGIN(G_RELAX, (d.fmode[id / d.T] == M_BFS ? d.dirty[prv * ns_ + id] : d.crecv[prv * ns_ + id]))
  if (md == M_BFS) {
    count_tile(d, 1);
    tile_relax<K>(d, gt, sw, hs, &bits_s);
  } else {
    count_tile(d, 4);
    tile_crelax<K>(d, io, gt, sw, ms, os);
  }
  GC_LIST_END
}

// ---------------------------------------------------------------- a3: k_push
// Up to `rounds` synchronous push / relabel rounds inside each active tile (or tile with
// inbound flow) of the slots in M_PUSH (4x the rounds once a push phase has run 8 steps:
// long-distance transport).  e, r and two height buffers live in shared memory.  Push
// phase: every active pixel v (e > 0, finite h) pushes delta = min(e, r_k) along admissible
// arcs (h(u) = h(v) - 1): it lowers its own r_k, raises r_opp(u) (unique writer: u cannot
// push back to v in the same round) and moves delta between e(v) and e(u) with shared-memory
// atomics.  Relabel phase (Jacobi): h'(v) = 1 + min h(u) over residual arcs for active
// pixels without an admissible arc.  Pushes across the tile border accumulate per receiver
// slot and go to the receiver tile's inbox at the end (absorbed at its next step).  Border
// heights are those of the previous step (stale); the exact global relabel restores valid
// labels and certifies termination.
template <int K>
constexpr size_t push_smem_bytes() { return sizeof(int) * (2 * HS * HS + TPX + K * TPX + K * 64); }

template <int K>
__global__ void __launch_bounds__(NTH, 4) k_push(Dev d, IO io, int sw, int rounds) {
  const int t = threadIdx.x, ix = t & 31, iy0 = t >> 5;
  extern __shared__ int smem_push[];  // push_smem_bytes<K>() of dynamic shared memory
  int(*hb)[HS * HS] = reinterpret_cast<int(*)[HS * HS]>(smem_push);  // heights, 2 buffers
  int* es = smem_push + 2 * HS * HS;                                  // excess
  int* rs = es + TPX;                                                 // residuals [K][TPX]
  int(*oacc)[64] = reinterpret_cast<int(*)[64]>(rs + K * TPX);        // border pushes by slot
  const int hmax = d.hmax;
  const int par_out = sw & 1, par_in = par_out ^ 1;
  GC_LIST_BEGIN(G_PUSH, (d.tact[id] || d.recv[par_in * ns_ + id]))
  (void)md;
  count_tile(d, 2);
  const int s = (int)(gt / d.T), tile = (int)(gt - (size_t)s * d.T);
  const int ty = tile / d.TX, tx = tile - ty * d.TX;
  const int rcv = d.recv[par_in * ns_ + gt];
  const int nround = d.fpush[s] >= 8 ? 4 * rounds : rounds;
  long long neg0 = 0;
  tile_load_smem<K>(d, io, gt, es, rs);
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int ev = es[(iy0 + 8 * j) * TS + ix];
    neg0 += ev < 0 ? -(long long)ev : 0;
  }
  if (rcv) absorb_smem<K>(d, par_in, gt, es, rs);
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int hv = d.h[gt * TPX + (iy0 + 8 * j) * TS + ix];
    hb[0][hidx(iy0 + 8 * j, ix)] = hv;
    hb[1][hidx(iy0 + 8 * j, ix)] = hv;
  }
  load_halo(d, s, ty, tx, hb[0], t);
  load_halo(d, s, ty, tx, hb[1], t);
  for (int i = t; i < K * 64; i += NTH) (&oacc[0][0])[i] = 0;
  __syncthreads();
  if (rcv && t == 0) d.recv[par_in * ns_ + gt] = 0;
  int nrel = 0;  // relabel operations (global-relabel heuristic, k_control)
  int cb = 0;    // current height buffer
  for (int rd = 0; rd < nround; ++rd) {
    const int* hc = hb[cb];
    // push phase (owner)
#pragma unroll 1
    for (int j = 0; j < 4; ++j) {
      const int iy = iy0 + 8 * j, lp = iy * TS + ix;
      int ee = es[lp];
      const int hv = hc[hidx(iy, ix)];
      if (ee > 0 && hv < HINF) {
        int sent = 0;
#pragma unroll
        for (int k = 0; k < K; ++k) {
          const int rk = rs[k * TPX + lp];
          if (ee > 0 && rk > 0 && hc[hidx(iy + DYk(k), ix + DXk(k))] == hv - 1) {
            const int dl = min(ee, rk);
            ee -= dl;
            sent += dl;
            rs[k * TPX + lp] = rk - dl;
            if (crosses(k, iy, ix)) {
              oacc[k][recv_slot(k, (iy + DYk(k)) & 31, (ix + DXk(k)) & 31)] += dl;
            } else {
              const int u = (iy + DYk(k)) * TS + ix + DXk(k);
              atomicAdd(&es[u], dl);
              rs[(k ^ 1) * TPX + u] += dl;  // unique writer: u cannot push back to v this round
            }
          }
        }
        if (sent) atomicSub(&es[lp], sent);
      }
    }
    __syncthreads();
    // relabel phase (Jacobi: read hc, write the other buffer)
    int* hn = hb[cb ^ 1];
    int still = 0;
#pragma unroll 1
    for (int j = 0; j < 4; ++j) {
      const int iy = iy0 + 8 * j, lp = iy * TS + ix;
      const int hv = hc[hidx(iy, ix)];
      int h2 = hv;
      if (es[lp] > 0 && hv < HINF) {
        int mn = HINF;
        bool adm = false;
#pragma unroll
        for (int k = 0; k < K; ++k) {
          if (rs[k * TPX + lp] > 0) {
            const int hu = hc[hidx(iy + DYk(k), ix + DXk(k))];
            adm |= (hu == hv - 1);
            mn = min(mn, hu);
          }
        }
        if (!adm) {
          h2 = (mn >= hmax - 1) ? HINF : mn + 1;
          ++nrel;
        }
        still |= h2 < HINF;
      }
      hn[hidx(iy, ix)] = h2;
    }
    cb ^= 1;
    if (!__syncthreads_or(still)) break;  // tile discharged: nothing left to push
  }
  // store state
  int act = 0;
  long long neg1 = 0;
  {
    int h[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int lp = (iy0 + 8 * j) * TS + ix;
      const int ev = es[lp];
      h[j] = hb[cb][hidx(iy0 + 8 * j, ix)];
      d.h[gt * TPX + lp] = h[j];
      act |= (ev > 0) & (h[j] < HINF);
      neg1 += ev < 0 ? -(long long)ev : 0;
    }
    tile_store_smem<K>(d, gt, es, rs);
    store_hedge(d, gt, h, t);
  }
  // send border pushes to the neighbours' inboxes (unique writer per slot)
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int iy = iy0 + 8 * j;
    if (!on_border(iy, ix)) continue;
#pragma unroll
    for (int k = 0; k < K; ++k) {
      if (!crosses(k, iy, ix)) continue;
      const int y2 = iy + DYk(k), x2 = ix + DXk(k);
      const int sl = recv_slot(k, y2 & 31, x2 & 31);
      const int dl = oacc[k][sl];
      if (dl) {
        const int rty = ty + (y2 < 0 ? -1 : (y2 > 31 ? 1 : 0));
        const int rtx = tx + (x2 < 0 ? -1 : (x2 > 31 ? 1 : 0));
        const size_t rgt = (size_t)s * d.T + rty * d.TX + rtx;
        INBp(d, K, par_out, rgt, k)[sl] = dl;
        d.recv[par_out * ns_ + rgt] = 1;
      }
    }
  }
  act = __syncthreads_or(act);
  // progress counters of this step (k_control): flow delivered to sink-connected nodes,
  // relabels, tiles touched for the first time in this push phase
  long long absorbed = neg0 - neg1;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    nrel += __shfl_xor_sync(0xffffffffu, nrel, o);
    absorbed += __shfl_xor_sync(0xffffffffu, absorbed, o);
  }
  if ((t & 31) == 0) {
    if (nrel) atomicAdd(&d.frel[s], (unsigned long long)nrel);
    if (absorbed > 0) atomicAdd(&d.fabs_[s], (unsigned long long)absorbed);
  }
  if (t == 0) {
    d.tact[gt] = act;
    d.mat[gt] = 1;
    const int ph = d.fph[s];
    if (d.tph[gt] != ph) {
      d.tph[gt] = ph;
      atomicAdd(&d.fnew[s], 1);
    }
  }
  GC_LIST_END
}

// ---------------------------------------------------------------- k_control
// Advances every slot's state machine after a step (one CTA per slot), finishes frames
// (flow value, stats), refills finished slots with the next frame, and builds the slot
// lists of the next step.  F = sum c(v,t) - sum max(0,-e): the flow that reached t.
__device__ __forceinline__ void finish_frame(const Dev& d, const IO& io, int s) {
  const int f = d.sfr[s];
  int st = 0;
  long long F = (long long)d.sumct[s] - (long long)d.sumneg[s];
  if (d.ferr[s]) { st = 2; F = -1; atomicAdd(&d.gctr[2], 1); }
  io.flow[f] = F;
  if (io.stats) {
    io.stats[f * 4 + 0] = d.fstat[s * 4 + 0];
    io.stats[f * 4 + 1] = d.fstat[s * 4 + 1];
    io.stats[f * 4 + 2] = d.fstat[s * 4 + 2];
    io.stats[f * 4 + 3] = st;
  }
  atomicAdd(&d.gctr[1], 1);
}

__global__ void __launch_bounds__(NTH) k_control(Dev d, IO io, int sw, long long relabel_budget, int max_push,
                                                 int nframes) {
  const int s = blockIdx.x, t = threadIdx.x;
  const int cur = sw & 1, nxt = cur ^ 1;
  if (s == 0 && t < NGROUP) d.lcnt[cur * NGROUP + t] = 0;  // this step's lists are consumed
  const int md = d.fmode[s];
  if (md == M_IDLE) return;
  const int chg = d.fchg[cur * d.nslot + s];
  int nact = 0;
  if (md == M_BFS && !chg) {  // relabel converged: any active node left that reaches t?
    for (int i = t; i < d.T; i += NTH) nact |= d.tact[(size_t)s * d.T + i];
    nact = __syncthreads_or(nact);
  }
  if (t != 0) return;
  int nm = md;
  int* st = d.fstat + s * 4;
  bool finished = false;
  if (md == M_INIT) {
    nm = d.ferr[s] ? M_CSEED : M_SEED;
  } else if (md == M_SEED) {
    nm = M_BFS;
    st[1] += 1;
  } else if (md == M_BFS) {
    st[2] += 1;
    if (!chg) {
      if (nact) {
        nm = M_PUSH;
        d.fpush[s] = 0;
        d.fstall[s] = 0;
        d.frel[s] = 0;
        d.fabs_[s] = 0;
        d.fnew[s] = 0;
        d.fph[s] += 1;
      } else {
        nm = M_CSEED;  // termination certificate: the preflow is maximum
      }
    }
  } else if (md == M_PUSH) {
    st[0] += 1;
    const int np = ++d.fpush[s];
    const bool stalled = d.fabs_[s] == 0 && d.fnew[s] == 0;
    d.fabs_[s] = 0;
    d.fnew[s] = 0;
    const int stall = stalled ? ++d.fstall[s] : (d.fstall[s] = 0);
    if (stall >= 1 + np / 4 || d.frel[s] > (unsigned long long)relabel_budget || np >= max_push) nm = M_SEED;
  } else if (md == M_CSEED || md == M_CLOS) {
    if (chg) nm = M_CLOS;
    else if (io.fstate && !d.ferr[s]) nm = M_EXPORT;
    else finished = true;
  } else if (md == M_EXPORT) {
    finished = true;
  }
  if (finished) {
    finish_frame(d, io, s);
    const int nf = atomicAdd(&d.gctr[0], 1);
    if (nf < nframes) {  // refill the slot with the next frame of the batch
      d.sfr[s] = nf;
      d.ferr[s] = 0;
      d.fph[s] = 0; d.fpush[s] = 0; d.fnew[s] = 0; d.fstall[s] = 0;
      d.fchg[cur * d.nslot + s] = 0;
      st[0] = st[1] = st[2] = st[3] = 0;
      d.fabs_[s] = 0; d.frel[s] = 0; d.sumct[s] = 0; d.sumneg[s] = 0;
      nm = M_INIT;
    } else {
      nm = M_IDLE;
    }
  }
  d.fmode[s] = nm;
  d.fchg[nxt * d.nslot + s] = 0;
  if (nm != M_IDLE) {
    const int g = mode_group(nm);
    const int pos = atomicAdd(&d.lcnt[nxt * NGROUP + g], 1);
    d.slist[((size_t)nxt * NGROUP + g) * d.nslot + pos] = s;
  }
}

// Initial slot assignment: slot s holds frame s, all slots in M_INIT (listed for step 0).
__global__ void k_setup(Dev d, int nframes) {
  for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < d.nslot; s += gridDim.x * blockDim.x) {
    d.sfr[s] = s;
    d.fmode[s] = M_INIT;
    d.slist[G_STREAM * d.nslot + s] = s;  // list buffer 0, group STREAM
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    d.lcnt[G_STREAM] = d.nslot;
    d.gctr[0] = d.nslot;
  }
}

// max_launches exceeded: frames not finished get F = -1, status GC_ERR_NOCONV.
__global__ void k_abort(Dev d, IO io, int nframes) {
  for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < d.nslot; s += gridDim.x * blockDim.x) {
    if (d.fmode[s] == M_IDLE) continue;
    const int f = d.sfr[s];
    io.flow[f] = -1;
    if (io.stats) io.stats[f * 4 + 3] = 5;
  }
  const int first = d.gctr[0];
  for (int f = first + blockIdx.x * blockDim.x + threadIdx.x; f < nframes; f += gridDim.x * blockDim.x) {
    io.flow[f] = -1;
    if (io.stats) io.stats[f * 4 + 3] = 5;
  }
}

}  // namespace gcb
