// gc_phases.cuh -- the device-side solver: one persistent kernel (k_solve) runs every phase
// of every frame of a batch as 32x32-tile tasks taken from a global work queue
// (DESIGN.md §3).
//
// The context holds `nslot` frame slots.  Each slot runs a state machine (d.fmode):
//   M_INIT   -- all tiles: streaming pass over the caps: fl bit-planes, sum c(v,t), range
//               check (a1 / a1w)
//   M_SEED   -- all tiles: global relabel, seed: absorb in-flight flow, h = 1 on nodes with
//               residual capacity to t, tile-local BFS fixpoint with an INF halo        (a2)
//   M_BFS    -- tiles whose neighbours' border heights changed: tile-local fixpoint with
//               the neighbours' border heights as halo; a changed border requests the
//               neighbour tiles (asynchronous Bellman-Ford over tiles, exact at
//               quiescence)                                                            (a2)
//               then: no active node left -> M_CSEED, else -> M_PUSH
//   M_PUSH   -- active tiles under the phase's height cap and tiles with inbound flow:
//               push/relabel rounds in shared memory (a3); a tile that stays active
//               requests itself, border flow requests the receiver; ends at quiescence or
//               when the phase's budgets are spent -> M_CSEED (certificate attempt)
//   M_CSEED  -- touched tiles: closure of the excess nodes inside the tile (the canonical
//               mask and the termination certificate), written to the caller's mask   (a4)
//   M_CLOS   -- closure across tile borders until nothing changes; reaching a node with
//               e < 0 fails the attempt (-> M_SEED), else the frame is solved          (a4)
//   (a5, the caller's warm-start state: the init pass writes every tile's initial flow to
//    flow_state_out, the closure seed of a tile a push touched its current one)
//   then the flow value is written and the slot takes the next frame (M_INIT) or idles.
//
// Scheduling.  A ring of tile ids with ticket counters (qhead, qtail).  Per frame, fout
// counts the tasks of the running phase that are queued or running; the CTA whose task
// brings it to zero runs the phase transition and enqueues the next phase's tasks (it
// holds a +1 guard on fout while it enqueues).  In the request-driven phases (BFS, PUSH,
// CLOS) treq[tile] > 0 means "queued or running": a request that finds it 0 enqueues the
// tile; a task subtracts the requests it started with when it ends and re-enqueues the
// tile if more arrived meanwhile -- so a tile is never processed by two CTAs at once and
// every change a tile must react to is seen by a later run of it.  Writers fence before
// they signal; all mutable state is read through L2.
#pragma once
#include "gc_kernels.cuh"

namespace gcb {

#ifndef GC_MINB
#define GC_MINB 4  // resident CTAs per SM the register budget is sized for
#endif
// Batches of frames of at least this many tiles that refill their slots run the 3-CTA-per-SM
// variant (80 registers, little spilling): a hard frame's long dependency chain of tile tasks
// then runs beside the streaming frames with two co-resident CTAs per SM instead of three
// (C4 ~37 -> ~32 ms per step).
constexpr int GC_MINB_LARGE = 3;
// Sequence passes (few frames in flight, each a latency-bound chain): 2 CTAs per SM, 128
// registers (C3 8 x 120 warm 20.3 -> 21.5 Gpx/s, cold 21.1 -> 23.2 against 3 per SM).
constexpr int GC_MINB_SEQ = 2;
constexpr int GC_LARGE_TILES = 1000;
constexpr uint32_t QEMPTY = 0xffffffffu;
constexpr uint32_t QEXIT = 0xfffffffeu;
constexpr uint32_t QNOP = 0xfffffffdu;  // releases a CTA waiting on the init ring (no task)

struct Ctl {
  long long relabel_budget;  // relabels per push phase (alpha x frame pixels)
  long long max_tasks;       // watchdog: tasks per launch before GC_ERR_NOCONV
  int vis_budget;            // push tasks per push phase
  int stall;                 // push tasks without progress before the phase drains
  int bndsh;                 // relabel distance bound 2 + 2^(1 + bndsh x attempts)
  int wavesh;                // push height cap: lowest active + 2^(wavesh x attempts)
  int stallx;                // the stall bound doubles with every failed certificate attempt
                             // beyond the first stallx (hard frames: long transport)
  int wave;                  // push phase starts on active tiles with min height <= lowest + wave
  int selfrun;               // 0: an active tile always runs again; 1: only after progress
  int rounds;                // push/relabel rounds per push task
  int nframes;
  int vec;                   // caller rows 16-byte aligned: int4 loads in the init pass
  int K4;                    // 4-neighbour frames (no diagonal arcs)
  int seqL;                  // sequence mode (gc_solve_sequences): frames per sequence; 0: batch
  int seqS;                  // sequence mode: number of sequences
  int seqWarm;               // sequence mode: frame t >= 1 warm-started from frame t-1's flows
};

// Slot s takes batch frame f: its frame index and where its warm-start flows come from and
// its exported flows go.  Batch mode: the caller's warm_flow / flow_state_out planes of frame
// f.  Sequence mode (f = j * L + t): frame 0 of sequence j starts from the caller's
// warm_flow[j] (or cold); frame t >= 1 from the ping-pong buffer frame t-1 exported into
// (warm) or cold; frame t exports into buffer t & 1, the last frame into flow_state_out[j].
// Distance bound of a global relabel after `ce` failed certificate attempts: 2 + 2^(1 +
// bndsh x ce) (HINF -- exact -- once that exceeds any distance in the frame).
__device__ __forceinline__ int relabel_bound(const Dev& d, const Ctl& c, int ce) {
  const int sh = min(ce * c.bndsh, 30);
  return (sh >= 24 || (2ll << sh) >= d.hmax) ? HINF : 2 + (2 << sh);
}

__device__ __forceinline__ void slot_assign(const Dev& d, const IO& io, const Ctl& c, int s, int f) {
  GC_CHECK(d, s >= 0 && s < d.nslot && f >= 0 && f < c.nframes);
  const size_t pl = (size_t)d.H * d.W * (c.K4 ? 2 : 4);
  const size_t plane = (size_t)d.H * d.W, K = c.K4 ? 4 : 8;
  d.sfr[s] = f;
  if (d.capbuf) {  // energy mode: the init pass builds the caps into the slot's buffer
    int32_t* cb = d.capbuf + (size_t)(d.capbyframe ? f : s) * (2 + K) * plane;
    d.scs[s] = cb;
    d.sct[s] = cb + plane;
    d.snb[s] = cb + 2 * plane;
  } else {
    d.scs[s] = io.cs + (size_t)f * plane;
    d.sct[s] = io.ct + (size_t)f * plane;
    d.snb[s] = io.nb + (size_t)f * plane * K;
  }
  d.fbe[s] = 1;  // the frame's first global relabel is seeded by its init tasks
  d.fbnd[s] = relabel_bound(d, c, 0);
  if (!c.seqL) {
    d.swf[s] = io.wf ? io.wf + (size_t)f * pl : nullptr;
    d.sfs[s] = io.fstate ? io.fstate + (size_t)f * pl : nullptr;
    return;
  }
  const int j = f / c.seqL, tt = f - j * c.seqL;
  int32_t* buf = d.fbuf + (size_t)s * 2 * pl;
  d.swf[s] = tt == 0 ? (io.wf ? io.wf + (size_t)j * pl : nullptr) : (c.seqWarm ? buf + ((tt - 1) & 1) * pl : nullptr);
  d.sfs[s] = tt == c.seqL - 1 ? (io.fstate ? io.fstate + (size_t)j * pl : nullptr)
                              : (c.seqWarm ? buf + (tt & 1) * pl : nullptr);
}

// ------------------------------------------------------------------ queue primitives
// Release/acquire fence at GPU scope (cheaper than __threadfence's sequentially consistent
// fence); every mutable load goes to L2 (-dlcm=cg), so it is all the ordering needed.
__device__ __forceinline__ void fence_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
__device__ __forceinline__ uint32_t ld_acquire_u32(const volatile uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ int ld_acquire_s32(const int32_t* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Band (NEXT-3 partition) owning tile gt: 0 unless the call is partitioned.
__device__ __forceinline__ int part_of(const Dev& d, size_t gt) {
  if (d.nparts <= 1) return 0;
  const int s = (int)((unsigned)gt / (unsigned)d.T), tile = (int)(gt - (size_t)s * d.T);
  return min(tile / d.TX / d.prow, d.nparts - 1);
}
__device__ __forceinline__ void q_put(const Dev& d, int r, unsigned long long p, uint32_t v) {
  volatile uint32_t* slot = d.q + (size_t)r * (d.qmask + 1) + (p & d.qmask);
  while (*slot != QEMPTY) __nanosleep(32);  // previous lap not consumed yet (capacity 2x: never in practice)
  *slot = v;
}
// A task entry to the ring of the band owning its tile.
__device__ __forceinline__ void chain_put(const Dev& d, uint32_t v) {
  const int r = part_of(d, v & 0x00ffffffu);
  q_put(d, r, atomicAdd(d.qtail + 2 * r, 1ULL), v);
}
__device__ __forceinline__ void qi_put(const Dev& d, int r, unsigned long long p, uint32_t v) {
  volatile uint32_t* slot = d.qi + (size_t)r * (d.qimask + 1) + (p & d.qimask);
  while (*slot != QEMPTY) __nanosleep(32);
  *slot = v;
}

// Queue entry: the phase a task belongs to (it cannot change while the task is queued),
// the number of consecutive tiles it covers (1..16; bulk seed / closure-seed tasks take
// groups of tiles), and the first tile (< 2^24).
__device__ __forceinline__ uint32_t qent(int md, size_t gt, int cnt = 1) {
  return ((uint32_t)md << 28) | ((uint32_t)(cnt - 1) << 24) | (uint32_t)gt;
}

// Neighbour tile of gt on side b (0 N, 1 S, 2 W, 3 E, 4 NW, 5 NE, 6 SW, 7 SE); -1 if off-frame.
__device__ __forceinline__ long long side_tile(const Dev& d, size_t gt, int b) {
  const int dy = (b == 0 || b == 4 || b == 5) ? -1 : ((b == 1 || b == 6 || b == 7) ? 1 : 0);
  const int dx = (b == 2 || b == 4 || b == 6) ? -1 : ((b == 3 || b == 5 || b == 7) ? 1 : 0);
  const int s = (int)((unsigned)gt / (unsigned)d.T), tile = (int)(gt - (size_t)s * d.T);
  const int ty = tile / d.TX + dy, tx = tile % d.TX + dx;
  if (ty < 0 || ty >= d.TY || tx < 0 || tx >= d.TX) return -1;
  return (long long)s * d.T + ty * d.TX + tx;
}

__device__ __forceinline__ int side_bit(int dy, int dx) {
  return dy < 0 ? (dx < 0 ? 4 : (dx > 0 ? 5 : 0)) : (dy > 0 ? (dx < 0 ? 6 : (dx > 0 ? 7 : 1)) : (dx < 0 ? 2 : 3));
}

// Block-wide: flag the neighbour tiles on the sides set in `bits` as part of the first task
// set of the next phase (the phase transition collects the flags).
__device__ __forceinline__ void flag_sides(const Dev& d, size_t gt, int bits, int K) {
  const int t = threadIdx.x;
  if (t < 8 && ((bits >> t) & 1) && !(t >= 4 && K == 4)) {
    const long long n = side_tile(d, gt, t);
    if (n >= 0) {
      d.flag[n] = 1;
      d.fflag[(unsigned)gt / (unsigned)d.T] = 1;  // the phase has a follow-up task set
    }
  }
}

// Sides of the tile whose halo reads pixel (iy, ix)'s height.
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

// Flow still in flight into the tile: materialise e, r pixel at a time (from the stored
// state or the caps), absorb the inbound border flow, store; returns the new fl words.
template <int K>
__device__ __forceinline__ void absorb_pixelwise(const Dev& d, const IO& io, size_t gt, int (&fl)[4], int* infl) {
  const int t = threadIdx.x, ix = t & 31, iy0 = t >> 5;
  const int s = (int)((unsigned)gt / (unsigned)d.T), tile = (int)(gt - (size_t)s * d.T);
  const int ty = tile / d.TX, tx = tile - ty * d.TX;
  gather_inflow<K>(d, gt, infl);
#pragma unroll 1
  for (int j = 0; j < 4; ++j) {
    const int iy = iy0 + 8 * j, lp = iy * TS + ix;
    int e, r[K];
    px_er<K>(d, io, gt, lp, ty * TS + iy, tx * TS + ix, e, r);
    if (on_border(iy, ix)) {
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const int wy = iy - DYk(k), wx = ix - DXk(k);
        if ((unsigned)wy < 32u && (unsigned)wx < 32u) continue;
        const int dl = infl[k * 64 + recv_slot(k, iy, ix)];
        if (dl) { e += dl; r[k ^ 1] += dl; }
      }
    }
    d.e[gt * TPX + lp] = e;
#pragma unroll
    for (int k = 0; k < K; ++k) Rp(d, K, gt, k)[lp] = r[k];
    fl[j] = make_fl<K>(e, r);
    d.fl[gt * TPX + lp] = (uint16_t)fl[j];
  }
  __syncthreads();
  if (t == 0) {
    d.mat[gt] = 1;
    d.recv1[gt] = 0;
    d.tuni[gt] = 0;  // the tile changed: no longer a known uniform sink / source tile (a seed
    d.tsrc[gt] = 0;  // recomputes)
    d.tfix[gt] = 0;
  }
}

// Halo ring entry t (t < 132: 4 sides x 32, then the corners NW NE SW SE) of tile (ty, tx):
// the neighbour's border height (HINF off-frame), its hidx position and its side bit.
__device__ __forceinline__ int halo_candidate(const Dev& d, int s, int ty, int tx, int t, int& pos, int& bit) {
  int nty = ty, ntx = tx, hi;
  if (t < 128) {
    const int side = t >> 5, i = t & 31;
    int esd;
    if (side == 0) { nty = ty - 1; esd = 1; pos = hidx(-1, i); bit = 0; }
    else if (side == 1) { nty = ty + 1; esd = 0; pos = hidx(32, i); bit = 1; }
    else if (side == 2) { ntx = tx - 1; esd = 3; pos = hidx(i, -1); bit = 2; }
    else { ntx = tx + 1; esd = 2; pos = hidx(i, 32); bit = 3; }
    hi = esd * 32 + i;
  } else {
    const int c = t - 128;
    const int dy = (c < 2) ? -1 : 1, dx = (c & 1) ? 1 : -1;
    bit = dy < 0 ? (dx < 0 ? 4 : 5) : (dx < 0 ? 6 : 7);
    nty = ty + dy;
    ntx = tx + dx;
    pos = hidx(dy < 0 ? -1 : 32, dx < 0 ? -1 : 32);
    hi = (dy < 0 ? 1 : 0) * 32 + (dx < 0 ? 31 : 0);
  }
  if (nty < 0 || nty >= d.TY || ntx < 0 || ntx >= d.TX) return HINF;
  return d.hedge[((size_t)s * d.T + nty * d.TX + ntx) * 128 + hi];
}

// ---------------------------------------------------------------- a2: seed (one tile)
// Absorbs flow still in flight from the push phase (materialising e, r pixel at a time),
// seeds h = 1 where the node has residual capacity to t, relaxes to the tile-local
// fixpoint with an INF halo, and flags the tiles that must be relaxed first: the
// neighbours that see a finite border height, and itself if a neighbour is a uniform sink
// tile (whose seed is skipped: nothing can have changed in it).
template <int K>
__device__ __forceinline__ void task_seed(const Dev& d, const IO& io, size_t gt, int* hs, int* bc) {
  const int t = threadIdx.x, ix = t & 31, iy0 = t >> 5;
  const int s = (int)((unsigned)gt / (unsigned)d.T);
  if (t == 0) {
    bc[0] = __ldcg(d.recv1 + gt);
    bc[2] = __ldcg(d.tuni + gt) | __ldcg(d.tsrc + gt);
    bc[6] = __ldcg(d.fbe + s);
    bc[7] = 0;
    bc[4] = __ldcg(d.fbnd + s);
  }
  __syncthreads();
  const int rcv = bc[0];
  // a uniform sink tile (h = 1, hedge published) or a uniform source tile (no sink: h = HINF,
  // its tss stamp says so) without inflow is not seeded (the transition stamped it)
  if (bc[2] && !rcv) return;
  // halo: the border heights of the neighbours whose seed was skipped in this relabel
  // (uniform sink tiles: final), INF elsewhere -- the BFS phase brings in the others.  The
  // candidates of every side are loaded together with the skip stamps and the fl words
  // (one round trip) and selected after the barrier.
  const int tile_ = (int)(gt - (size_t)s * d.T);
  const int ty_ = tile_ / d.TX, tx_ = tile_ - ty_ * d.TX;
  if (t < 8) {
    const long long n = side_tile(d, gt, t);
    const int ok = n >= 0 && !(t >= 4 && K == 4) && __ldcg(d.tsk + n) == bc[6];
    if (ok) atomicOr(&bc[7], 1 << t);
  }
  int hpos = 0, hbit = 0, hval = HINF;
  if (t < 132) hval = halo_candidate(d, s, ty_, tx_, t, hpos, hbit);
  int fl[4];
  if (rcv) absorb_pixelwise<K>(d, io, gt, fl, hs + 2048);
  else {
#pragma unroll
    for (int j = 0; j < 4; ++j) fl[j] = d.fl[gt * TPX + (iy0 + 8 * j) * TS + ix];
  }
  __syncthreads();
  if (t < 132) hs[hpos] = ((bc[7] >> hbit) & 1) ? hval : HINF;
  int h[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    h[j] = (fl[j] & FL_NEG) ? 1 : HINF;
    hs[hidx(iy0 + 8 * j, ix)] = h[j];
  }
  __syncthreads();
  bfs_fixpoint<K>(hs, fl, h, bc[4]);
  int act = 0, fix = 1, uni = 1, src = 1, bits = 0, mnh = HINF;
  const int tile = (int)(gt - (size_t)s * d.T);
  const int ty = tile / d.TX, tx = tile - ty * d.TX;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int iy = iy0 + 8 * j;
    d.h[gt * TPX + iy * TS + ix] = h[j];
    act |= (fl[j] & FL_POS) && h[j] < HINF;
    if (fl[j] & FL_POS) mnh = min(mnh, h[j]);
    fix &= (h[j] == 1) || !(fl[j] & 0xff);
    const bool in = ty * TS + iy < d.H && tx * TS + ix < d.W;
    uni &= !in || (fl[j] & FL_NEG);
    src &= !in || (fl[j] & FL_POS);
    if (on_border(iy, ix) && h[j] < HINF) bits |= border_bits(iy, ix);
  }
  store_hedge(d, gt, h, t);
  bits = __reduce_or_sync(0xffffffffu, bits);
  mnh = __reduce_min_sync(0xffffffffu, mnh);
  if (t == 0) { bc[1] = 0; bc[5] = HINF; }
  act = __syncthreads_or(act);
  if ((t & 31) == 0) atomicMin(&bc[5], mnh);
  fix = __syncthreads_and(fix);
  uni = __syncthreads_and(uni);
  src = __syncthreads_and(src);
  if ((t & 31) == 0 && bits) atomicOr(&bc[1], bits);
  if (t == 0) {
    d.tact[gt] = act;
    d.tminh[gt] = bc[5];
    d.tfix[gt] = fix;
    d.tuni[gt] = uni;
    d.tsrc[gt] = src;
    d.tss[gt] = 0;  // h and hedge written in this relabel
  }
  flag_sides(d, gt, bc[1], K);
}

// ---------------------------------------------------------------- a2: relax (one tile)
// Returns (in bc[1]) the sides whose tiles must be requested: their halo reads a changed
// border height.
template <int K>
__device__ __forceinline__ void task_relax(const Dev& d, size_t gt, int* hs, int* bc) {
  const int t = threadIdx.x, ix = t & 31, iy0 = t >> 5;
  const int s = (int)((unsigned)gt / (unsigned)d.T), tile = (int)(gt - (size_t)s * d.T);
  const int ty = tile / d.TX, tx = tile - ty * d.TX;
  if (t == 0) {
    bc[1] = 0;
    bc[4] = __ldcg(d.fbnd + s);
    const int ep = __ldcg(d.fbe + s);
    bc[6] = ep;
    bc[7] = __ldcg(d.tss + gt) == ep;  // seed skipped (uniform source): stored h stale, HINF
  }
  __syncthreads();
  const int ep = bc[6], stale = bc[7];
  int fl[4], h[4], h0[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int lp = (iy0 + 8 * j) * TS + ix;
    fl[j] = d.fl[gt * TPX + lp];
    h[j] = h0[j] = stale ? HINF : d.h[gt * TPX + lp];
    hs[hidx(iy0 + 8 * j, ix)] = h[j];
  }
  load_halo(d, s, ty, tx, hs, t, ep);
  __syncthreads();
  bfs_fixpoint<K>(hs, fl, h, bc[4]);
  int any = 0, bits = 0, act = 0, fix = 1, mnh = HINF;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int ch = h[j] != h0[j];
    any |= ch;
    if (ch) bits |= border_bits(iy0 + 8 * j, ix);
    act |= (fl[j] & FL_POS) && h[j] < HINF;
    if (fl[j] & FL_POS) mnh = min(mnh, h[j]);
    fix &= (h[j] == 1) || !(fl[j] & 0xff);
  }
  bits = __reduce_or_sync(0xffffffffu, bits);
  mnh = __reduce_min_sync(0xffffffffu, mnh);
  if (t == 0) bc[5] = HINF;
  __syncthreads();
  if ((t & 31) == 0 && bits) atomicOr(&bc[1], bits);
  if ((t & 31) == 0) atomicMin(&bc[5], mnh);
  any = __syncthreads_or(any);
  act = __syncthreads_or(act);
  fix = __syncthreads_and(fix);
  if (any) {
#pragma unroll
    for (int j = 0; j < 4; ++j) d.h[gt * TPX + (iy0 + 8 * j) * TS + ix] = h[j];
    store_hedge(d, gt, h, t);
    if (t == 0) { d.tact[gt] = act; d.tfix[gt] = fix; d.tminh[gt] = bc[5]; }
    if (stale) {  // h and hedge now hold this relabel's values: readers may use them
      __syncthreads();
      if (t == 0) {
        fence_gpu();
        d.tss[gt] = 0;
      }
    }
  }
}

// ---------------------------------------------------------------- a4: closure helpers
// The closure of {v : e(v) > 0} under arcs with positive residual.  If it holds no node
// with e < 0 (residual capacity to t), no excess can reach t: the preflow is maximum and
// the closure is the source side of the inclusion-minimal minimum cut --
// the certificate that ends a solve.  Otherwise the attempt fails (cfail) and the frame
// returns to a global relabel.  Border reach marks carry the attempt's epoch, so a failed
// attempt leaves nothing behind.  The caller's mask starts as the excess pixels (the init
// pass writes it; they are in every closure): a tile a push touched (mat) rewrites all its
// bytes in its closure seed, an untouched tile only writes the closure pixels beyond its
// excess pixels ("extras", flagged in tmk so that the next attempt rewrites the tile).
__device__ __forceinline__ int closure_epoch(const Dev& d, int s) { return __ldcg(d.sep + s) % 255 + 1; }

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

// Marks the border arcs leaving the pixels with send[j] set with the epoch (a mark is only
// set if the receiving pixel is not an excess node -- those are in the closure anyway -- and
// was not set before in this attempt); returns the sides (side_bit) of the neighbour tiles
// that got a NEW mark.  Each mark slot has one writer (the tile of the sending pixel), so the
// check-and-set needs no atomic; since only new marks request the receiver, the closure
// phase ends once no tile adds a pixel.
template <int K>
__device__ __forceinline__ int closure_send(const Dev& d, size_t gt, const int (&send)[4], const uint8_t* os,
                                            int ep, const uint16_t* flh) {
  const int t = threadIdx.x, ix = t & 31, iy0 = t >> 5;
  const int s = (int)((unsigned)gt / (unsigned)d.T), tile = (int)(gt - (size_t)s * d.T);
  const int ty = tile / d.TX, tx = tile - ty * d.TX;
  int sides = 0;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int iy = iy0 + 8 * j;
    if (!send[j] || !on_border(iy, ix)) continue;
    const int ob = os[iy * TS + ix];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      if (!crosses(k, iy, ix) || !((ob >> k) & 1)) continue;
      const int y2 = iy + DYk(k), x2 = ix + DXk(k);
      if (flh[hidx(y2, x2)] & FL_POS) continue;  // an excess node: in the closure anyway
      const int dy = y2 < 0 ? -1 : (y2 > 31 ? 1 : 0), dx = x2 < 0 ? -1 : (x2 > 31 ? 1 : 0);
      const int rty = ty + dy, rtx = tx + dx;
      if (rty < 0 || rty >= d.TY || rtx < 0 || rtx >= d.TX) continue;
      const size_t rgt = (size_t)s * d.T + rty * d.TX + rtx;
      uint8_t* mk = d.reach + (rgt * K + k) * 64 + recv_slot(k, y2 & 31, x2 & 31);
      if (*mk != (uint8_t)ep) {
        *mk = (uint8_t)ep;
        sides |= 1 << side_bit(dy, dx);
      }
    }
  }
  return sides;
}

// OR of per-thread side bits into bc[1] (block-wide); returns it.
__device__ __forceinline__ int block_or_bits(int bits, int* bc) {
  bits = __reduce_or_sync(0xffffffffu, bits);
  if (threadIdx.x == 0) bc[1] = 0;
  __syncthreads();
  if ((threadIdx.x & 31) == 0 && bits) atomicOr(&bc[1], bits);
  __syncthreads();
  return bc[1];
}

// The caller's mask bytes of the tile's in-frame pixels with wr[j] set: mm[j].
__device__ __forceinline__ void mask_write(const Dev& d, const IO& io, size_t gt, const int (&mm)[4],
                                           const int (&wr)[4]) {
  const int t = threadIdx.x, ix = t & 31, iy0 = t >> 5;
  const int s = (int)((unsigned)gt / (unsigned)d.T), tile = (int)(gt - (size_t)s * d.T);
  const int ty = tile / d.TX, tx = tile - ty * d.TX;
  uint8_t* mask = io.mask + (size_t)d.sfr[s] * d.H * d.W;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int y = ty * TS + iy0 + 8 * j, x = tx * TS + ix;
    if (wr[j] && y < d.H && x < d.W) mask[(size_t)y * d.W + x] = (uint8_t)mm[j];
  }
}

template <int K>
__device__ __forceinline__ void task_export(const Dev& d, const IO& io, size_t gt);

// ---------------------------------------------------------------- a4: closure seed (one tile)
// Absorbs flow still in flight, closes {e > 0} inside the tile, writes the mask bytes that
// differ from the init pass's (all of a touched tile), marks reach across the border
// (flagging the receivers for the closure phase), checks the certificate, and brings the
// tile's share of sum max(0,-e) up to date.  An untouched uniform source tile (every pixel
// e > 0: closure = the whole tile, mask already written) only marks its border arcs.  A
// frame with out-of-range caps gets an all-0 mask here (gc.h).
// The words the closure seeds of a group of tiles decide on, loaded for the whole group at once
// (thread j: tile gt0 + j; one round trip instead of one per tile): gw[j] = {mode, mat | recv1,
// every mask byte rewritten, epoch, recv1}.  mode 2: range error (mask all 0, F = -1); 1: skip --
// the attempt already failed, or (a tile of the group outside the task set) an untouched uniform
// sink tile without extra mask bytes; 3: untouched uniform source tile (border marks only);
// 0: full closure seed.  Block-wide; ends with a barrier.
__device__ __forceinline__ void cseed_group_words(const Dev& d, size_t gt0, int gcnt, int (*gw)[5]) {
  const int t = threadIdx.x;
  if (t < gcnt) {
    const size_t gt = gt0 + t;
    const int s = (int)((unsigned)gt / (unsigned)d.T);
    // every word at once (independent loads)
    const int r1 = __ldcg(d.recv1 + gt), fe = __ldcg(d.ferr + s), cf = __ldcg(d.cfail + s);
    const int tu = __ldcg(d.tuni + gt), mt = __ldcg(d.mat + gt), tm = __ldcg(d.tmk + gt);
    const int tsr = __ldcg(d.tsrc + gt);
    const int cp = __ldcg(d.sep + s);
    gw[t][0] = fe ? 2 : ((cf > 0) | ((tu != 0) & (mt == 0) & (r1 == 0) & (tm == 0))) ? 1
                                                                                     : ((tsr != 0) & (mt == 0) & (r1 == 0)) ? 3 : 0;
    gw[t][1] = mt | r1;       // e, r materialised: rewrite every mask byte, recompute the deficit
    gw[t][2] = (mt | r1) | tm;  // every mask byte of the tile is (re)written
    gw[t][3] = cp % 255 + 1;  // closure epoch (closure_epoch)
    gw[t][4] = r1;
  }
  __syncthreads();
}

template <int K>
__device__ __forceinline__ void task_cseed(const Dev& d, const IO& io, size_t gt, uint8_t* ms, uint8_t* os,
                                           long long* red, int* bc, const int* gw) {
  const int t = threadIdx.x, ix = t & 31, iy0 = t >> 5;
  const int s = (int)((unsigned)gt / (unsigned)d.T);
  if (t == 0) {
    bc[0] = gw[4];
    bc[2] = gw[0];
    bc[3] = gw[1];
    bc[5] = gw[2];
    bc[4] = gw[3];
  }
  __syncthreads();
  const int mode = bc[2];
  if (mode == 1) return;
  if (mode == 2) {  // range error: the frame's mask is all 0
    const int none[4] = {0, 0, 0, 0}, all[4] = {1, 1, 1, 1};
    mask_write(d, io, gt, none, all);
    return;
  }
  uint16_t* flh = reinterpret_cast<uint16_t*>(ms + 12288);  // the neighbours' border fl words
  {
    const int tile = (int)(gt - (size_t)s * d.T);
    load_fl_halo(d, s, tile / d.TX, tile % d.TX, flh, t);  // issued with the tile's own loads
  }
  int fl[4];
  if (bc[0]) absorb_pixelwise<K>(d, io, gt, fl, reinterpret_cast<int*>(ms) + 2048);
  else {
#pragma unroll
    for (int j = 0; j < 4; ++j) fl[j] = d.fl[gt * TPX + (iy0 + 8 * j) * TS + ix];
  }
  const int ep = bc[4];
  const int mat = bc[3], wall = bc[5];
  int mm[4], pos[4];
  long long neg = 0;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int lp = (iy0 + 8 * j) * TS + ix;
    pos[j] = (fl[j] & FL_POS) ? 1 : 0;
    mm[j] = pos[j];
    ms[lp] = (uint8_t)mm[j];
    os[lp] = (uint8_t)(fl[j] & 0xff);
    if (mat) {
      const int ev = d.e[gt * TPX + lp];
      neg += ev < 0 ? -(long long)ev : 0;
    }
  }
  __syncthreads();
  int fail = 0, extra = 0;
  if (mode == 0) {
    closure_fixpoint<K>(ms, os, mm);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      fail |= mm[j] && (fl[j] & FL_NEG);
      extra |= mm[j] & !pos[j];
    }
    fail = __syncthreads_or(fail);
    extra = __syncthreads_or(extra);
    if (wall) {
      const int all[4] = {1, 1, 1, 1};
      mask_write(d, io, gt, mm, all);
    } else if (extra) {
      int wr[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) wr[j] = mm[j] & !pos[j];
      mask_write(d, io, gt, mm, wr);
    }
  }
  const int sides = block_or_bits(closure_send<K>(d, gt, mm, os, ep, flh), bc);
  if (mat) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) neg += __shfl_xor_sync(0xffffffffu, neg, o);
    if ((t & 31) == 0) red[t >> 5] = neg;
    __syncthreads();
  }
  if (t == 0) {
    if (mat) {  // replace the tile's share of sum max(0,-e) by its current value
      long long tot = 0;
      for (int i = 0; i < NTH / 32; ++i) tot += red[i];
      const long long dl = tot - d.neg0[gt];
      if (dl) atomicAdd(&d.sumneg[s], (unsigned long long)dl);
      d.neg0[gt] = tot;
    }
    if (mode == 0 && wall) d.tmk[gt] = extra ? ep : 0;  // every byte rewritten just now
    else if (extra) d.tmk[gt] = ep;
    if (fail) atomicAdd(&d.cfail[s], 2);  // cfail: 0 / -1 (after the BFS certificate) + 2 per failure
  }
  flag_sides(d, gt, sides, K);
  // a5: a tile a push touched exports its forward-arc flows here (the init pass wrote every
  // other tile's); a failed attempt's export is rewritten by the next attempt, which
  // closure-seeds every materialised tile again
  if (mat && d.sfs[s]) task_export<K>(d, io, gt);
}

// ---------------------------------------------------------------- a4: closure relax (one tile)
// Recomputes the tile's closure from its excess pixels and the reach marks of this attempt,
// writes mask bytes of its pixels beyond the excess ones, checks the certificate and marks
// the border arcs of those pixels.  Returns the sides to request (new marks) in bc[1].
template <int K>
__device__ __forceinline__ void task_crelax(const Dev& d, const IO& io, size_t gt, uint8_t* ms, uint8_t* os,
                                            int* bc) {
  const int t = threadIdx.x, ix = t & 31, iy0 = t >> 5;
  const int s = (int)((unsigned)gt / (unsigned)d.T);
  if (t == 0) {
    bc[1] = 0;
    bc[2] = __ldcg(d.cfail + s) > 0;
    bc[4] = closure_epoch(d, s);
  }
  __syncthreads();
  if (bc[2]) return;  // the attempt already failed
  const int ep = bc[4];
  int mm[4], pos[4], fl[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int iy = iy0 + 8 * j, lp = iy * TS + ix;
    fl[j] = d.fl[gt * TPX + lp];
    pos[j] = (fl[j] & FL_POS) ? 1 : 0;
    os[lp] = (uint8_t)(fl[j] & 0xff);
    int got = pos[j];
    if (!got && on_border(iy, ix)) {
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const int wy = iy - DYk(k), wx = ix - DXk(k);
        if ((unsigned)wy < 32u && (unsigned)wx < 32u) continue;
        got |= __ldcg(d.reach + (gt * K + k) * 64 + recv_slot(k, iy, ix)) == ep;
      }
    }
    mm[j] = got;
    ms[lp] = (uint8_t)got;
  }
  __syncthreads();
  closure_fixpoint<K>(ms, os, mm);
  int nw[4], any = 0, fail = 0;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    nw[j] = mm[j] & !pos[j];  // closure pixels beyond the excess ones (their bytes may be new)
    any |= nw[j];
    fail |= nw[j] && (fl[j] & FL_NEG);
  }
  any = __syncthreads_or(any);
  fail = __syncthreads_or(fail);
  if (any) mask_write(d, io, gt, mm, nw);
  if (t == 0) {
    if (any) d.tmk[gt] = ep;
    if (fail) atomicAdd(&d.cfail[s], 2);
  }
  if (any && !fail) {
    uint16_t* flh = reinterpret_cast<uint16_t*>(ms + 12288);
    load_fl_halo(d, s, (int)(gt - (size_t)s * d.T) / d.TX, (int)(gt - (size_t)s * d.T) % d.TX, flh, t);
    __syncthreads();
    block_or_bits(closure_send<K>(d, gt, nw, os, ep, flh), bc);  // sides to request, in bc[1]
  }
}

// ---------------------------------------------------------------- a5: export (one tile)
// Forward-arc flows f = c - r of this solve (the next frame's warm start).
template <int K>
__device__ __forceinline__ void task_export(const Dev& d, const IO& io, size_t gt) {
  const int s = (int)((unsigned)gt / (unsigned)d.T), tile = (int)(gt - (size_t)s * d.T);
  const int ty = tile / d.TX, tx = tile - ty * d.TX;
  const int t = threadIdx.x, ix = t & 31, iy0 = t >> 5;
  const int H = d.H, W = d.W;
  const size_t plane = (size_t)H * W;
  const size_t fr = (size_t)d.sfr[s];
  int32_t* fsp = d.sfs[s];
  const int32_t* nbp = d.snb[s];
  if (K == 4 && (W & 3) == 0 && (((uintptr_t)fsp | (uintptr_t)nbp) & 15) == 0) {
    // aligned rows (a materialised tile, the only kind exported here): thread t takes row t/8,
    // columns 4(t%8)..+3 -- every residual and cap of its forward arcs in 16-byte loads at once
    const int iy = t >> 3, ix0 = (t & 7) * 4;
    const int y = ty * TS + iy, x0 = tx * TS + ix0;
    if (y < H && x0 < W) {
      const size_t o = (size_t)y * W + x0;
      int4 rv[K / 2], cv[K / 2];
#pragma unroll
      for (int kk = 0; kk < K / 2; ++kk) {
        rv[kk] = *reinterpret_cast<const int4*>(Rp(d, K, gt, 2 * kk) + iy * TS + ix0);
        cv[kk] = __ldg(reinterpret_cast<const int4*>(nbp + 2 * kk * plane + o));
      }
#pragma unroll
      for (int kk = 0; kk < K / 2; ++kk) {
        const int k = 2 * kk, y2 = y + DYk(k);
        const int* rr = &rv[kk].x;
        const int* cc = &cv[kk].x;
        int f[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int x2 = x0 + i + DXk(k);
          f[i] = (y2 >= 0 && y2 < H && x2 >= 0 && x2 < W) ? cc[i] - rr[i] : 0;
        }
        *reinterpret_cast<int4*>(fsp + kk * plane + o) = make_int4(f[0], f[1], f[2], f[3]);
      }
    }
    return;
  }
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
      if (y2 >= 0 && y2 < H && x2 >= 0 && x2 < W) f = d.snb[s][k * plane + o] - r[k];
      fsp[(k >> 1) * plane + o] = f;
    }
  }
}

// ---------------------------------------------------------------- a3: push (one tile)
// Up to `rounds` synchronous push / relabel rounds inside the tile.  e, r and two height
// buffers live in shared memory.  Push phase: every active pixel v (e > 0, finite h)
// pushes delta = min(e, r_k) along admissible arcs (h(u) = h(v) - 1): it lowers its own
// r_k, raises r_opp(u) (unique writer: u cannot push back to v in the same round) and
// moves delta between e(v) and e(u) with shared-memory atomics.  Relabel phase (Jacobi):
// h'(v) = 1 + min h(u) over residual arcs for active pixels without an admissible arc.
// Pushes across the tile border accumulate per receiver slot and are added to the
// receiver's cumulative `sent` counters at the end; the receiver is requested.  Border
// heights are the neighbours' last published ones (possibly stale); the exact global
// relabel restores valid labels and certifies termination.
template <int K>
constexpr size_t push_smem_bytes() { return sizeof(int) * (2 * HS * HS + TPX + K * TPX + K * 64); }
// dynamic shared memory of k_solve: the largest task layout
template <int K>
constexpr size_t solve_smem_bytes() {
  return push_smem_bytes<K>() > init_smem_bytes<K>() ? push_smem_bytes<K>() : init_smem_bytes<K>();
}
static_assert(init_smem_bytes<4>() <= push_smem_bytes<4>() && init_smem_bytes<8>() <= push_smem_bytes<8>(),
              "the init pass's prefetch buffer must fit the push tile's shared memory");

// Returns the sides whose tiles received border flow in bc[1] and "still active" in bc[3].
template <int K>
__device__ __forceinline__ void task_push(const Dev& d, const IO& io, size_t gt, const Ctl& c, int* smem, int* bc,
                                          long long* red) {
  const int t = threadIdx.x, ix = t & 31, iy0 = t >> 5;
  int(*hb)[HS * HS] = reinterpret_cast<int(*)[HS * HS]>(smem);  // heights, 2 buffers
  int* es = smem + 2 * HS * HS;                                   // excess
  int* rs = es + TPX;                                             // residuals [K][TPX]
  int(*oacc)[64] = reinterpret_cast<int(*)[64]>(rs + K * TPX);    // border pushes by slot
  const int hmax = d.hmax;
  const int s = (int)((unsigned)gt / (unsigned)d.T), tile = (int)(gt - (size_t)s * d.T);
  const int ty = tile / d.TX, tx = tile - ty * d.TX;
  if (t == 0) {
    // phase budget spent or no progress lately: the frame drains to the next global relabel
    // (every word loaded at once: independent loads, one round trip)
    const int vis = __ldcg(d.fvis + s);
    const int cep = __ldcg(d.cep + s);  // failed certificate attempts: longer phases
    const long long rel = (long long)__ldcg(d.frel + s);
    const int prg = __ldcg(d.fprog + s), drn = __ldcg(d.fdrain + s);
    const int tu = __ldcg(d.tuni + gt), cap = __ldcg(d.fcap + s);
    const int ep = __ldcg(d.fbe + s), ts = __ldcg(d.tss + gt);
    const bool cond = (rel > (c.relabel_budget << min(cep, 10))) | (vis >= c.vis_budget) |
                      (vis - prg > (c.stall << min(max(cep - c.stallx, 0), 24)));
    bc[0] = cond | (drn != 0);
    if (cond) d.fdrain[s] = 1;  // no more requests in this phase
    bc[1] = 0;
    // inbound flow: take the flag (acquire: the senders set it after their counters)
    bc[2] = bc[0] ? 0 : atomicExch(&d.recv1[gt], 0);
    fence_gpu();
    bc[3] = 0;
    bc[4] = tu;
    bc[5] = HINF;
    bc[7] = cap;  // pixels higher than this are frozen in this phase
    bc[6] = ep;
    red[0] = ts == ep;  // seed skipped (uniform source), no relax since: stored h stale, HINF
  }
  __syncthreads();
  if (bc[0]) {
    if (d.pdbg && t == 0) atomicAdd(&d.pdbg[4], 1ULL);
    return;
  }
  const int rcv = bc[2], uni = bc[4], hcap = bc[7], hep = bc[6], stale = (int)red[0];
  tile_load_smem<K>(d, io, gt, es, rs, c.vec != 0);
  long long neg0 = 0;  // deficit of the tile before the task (flow absorbed = progress)
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int ev = es[(iy0 + 8 * j) * TS + ix];
    neg0 += ev < 0 ? -(long long)ev : 0;
  }
  if (rcv) {
    gather_inflow<K>(d, gt, &oacc[0][0]);  // oacc is free until the rounds: borrow it
    absorb_smem<K>(&oacc[0][0], es, rs);
    __syncthreads();
  }
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int iy = iy0 + 8 * j;
    // a uniform sink tile's heights are not stored: h = 1 in frame
    const int hv = uni ? ((ty * TS + iy < d.H && tx * TS + ix < d.W) ? 1 : HINF)
                       : (stale ? HINF : d.h[gt * TPX + iy * TS + ix]);
    hb[0][hidx(iy, ix)] = hv;
    hb[1][hidx(iy, ix)] = hv;
  }
  load_halo(d, s, ty, tx, hb[0], t, hep);
  load_halo(d, s, ty, tx, hb[1], t, hep);
  for (int i = t; i < K * 64; i += NTH) (&oacc[0][0])[i] = 0;
  __syncthreads();
  int nrel = 0;  // relabel operations (global-relabel heuristic)
  int cb = 0;    // current height buffer
  // rounds: c.rounds, extended block by block (up to 8x) while the last block moved flow
  // out of the tile or into deficit nodes (long-distance transport)
  int blockprog = 0;
  for (int rd = 0;; ++rd) {
    if (rd >= c.rounds && (rd % c.rounds) == 0) {
      if (!blockprog || rd >= 8 * c.rounds) break;
      blockprog = 0;
    }
    const int* hc = hb[cb];
    int prog = 0;
    // push phase (owner)
#pragma unroll 1
    for (int j = 0; j < 4; ++j) {
      const int iy = iy0 + 8 * j, lp = iy * TS + ix;
      int ee = es[lp];
      const int hv = hc[hidx(iy, ix)];
      if (ee > 0 && hv <= hcap) {
        int rk[K], hu[K];  // all loads first (independent), then the sequential pushes
#pragma unroll
        for (int k = 0; k < K; ++k) {
          rk[k] = rs[k * TPX + lp];
          hu[k] = hc[hidx(iy + DYk(k), ix + DXk(k))];
        }
        int sent = 0;
#pragma unroll
        for (int k = 0; k < K; ++k) {
          if (ee > 0 && rk[k] > 0 && hu[k] == hv - 1) {
            const int dl = min(ee, rk[k]);
            ee -= dl;
            sent += dl;
            rs[k * TPX + lp] = rk[k] - dl;
            if (crosses(k, iy, ix)) {
              oacc[k][recv_slot(k, (iy + DYk(k)) & 31, (ix + DXk(k)) & 31)] += dl;
              prog = 1;
            } else {
              const int u = (iy + DYk(k)) * TS + ix + DXk(k);
              prog |= atomicAdd(&es[u], dl) < 0;  // reached a deficit node
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
      if (es[lp] > 0 && hv <= hcap) {
        int mn = HINF;
        bool adm = false;
        int rk[K], hu[K];
#pragma unroll
        for (int k = 0; k < K; ++k) {
          rk[k] = rs[k * TPX + lp];
          hu[k] = hc[hidx(iy + DYk(k), ix + DXk(k))];
        }
#pragma unroll
        for (int k = 0; k < K; ++k) {
          if (rk[k] > 0) {
            adm |= (hu[k] == hv - 1);
            mn = min(mn, hu[k]);
          }
        }
        if (!adm) {
          h2 = (mn >= hmax - 1) ? HINF : mn + 1;
          ++nrel;
        }
        still |= h2 <= hcap;
      }
      hn[hidx(iy, ix)] = h2;
    }
    cb ^= 1;
    if (d.pdbg && t == 0) atomicAdd(&d.pdbg[5], 1ULL);
    const int flags = __syncthreads_or(still | (prog << 1));
    blockprog |= flags & 2;
    if (!(flags & 1)) break;  // tile discharged: nothing left to push
  }
  // store state
  int act = 0, amin = HINF;
  long long neg1 = 0;
  {
    int h[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int lp = (iy0 + 8 * j) * TS + ix;
      const int ev = es[lp];
      h[j] = hb[cb][hidx(iy0 + 8 * j, ix)];
      d.h[gt * TPX + lp] = h[j];
      act |= (ev > 0) & (h[j] <= hcap);
      if (ev > 0) amin = min(amin, h[j]);
      neg1 += ev < 0 ? -(long long)ev : 0;
    }
    amin = __reduce_min_sync(0xffffffffu, amin);
    if ((t & 31) == 0 && amin < HINF) atomicMin(&bc[5], amin);
    tile_store_smem<K>(d, gt, es, rs);
    store_hedge(d, gt, h, t);
  }
  // border pushes: add to the receivers' cumulative counters (unique writer per slot),
  // one slot per thread (coalesced per direction).  The receiver is flagged (recv1: the flow
  // is absorbed at its next task, seed or closure seed at the latest) and requested only if
  // a receiving pixel can pass the flow on in this phase: 1 < h <= cap by our halo (a sink
  // node just absorbs it; a node above the cap is frozen).
  int sides = 0;
  for (int i = t; i < K * 64; i += NTH) {
    const int dl = (&oacc[0][0])[i];
    if (dl) {
      const int k = i >> 6, sl = i & 63;
      int dy, dx, uy, ux;
      recv_tile_offset(k, sl, dy, dx);
      recv_pixel(k, sl, uy, ux);
      const size_t rgt = (size_t)s * d.T + (ty + dy) * d.TX + (tx + dx);
      uint32_t* p = SENTp(d, K, rgt, k) + sl;
      *p = __ldcg(p) + (uint32_t)dl;
      const int b = side_bit(dy, dx);
      const int hu = hb[cb][hidx(uy + 32 * dy, ux + 32 * dx)];
      sides |= (1 << b) | ((hu > 1 && hu <= hcap) << (8 + b));
    }
  }
  fence_gpu();  // the counters are visible before the receivers' recv1 flags (release)
  act = __syncthreads_or(act);
  const int sb2 = block_or_bits(sides, bc);
  sides = sb2 & 255;
  if (t < 8 && ((sides >> t) & 1)) d.recv1[side_tile(d, gt, t)] = 1;
  __syncthreads();
  if (t == 0) bc[1] = (sb2 >> 8) & 255;  // the receivers to request (task completion)
  // progress counters: relabels of this phase, tasks, flow absorbed by deficit nodes
  long long absorbed = neg0 - neg1;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    nrel += __shfl_xor_sync(0xffffffffu, nrel, o);
    absorbed += __shfl_xor_sync(0xffffffffu, absorbed, o);
  }
  if ((t & 31) == 0) red[t >> 5] = absorbed;
  if ((t & 31) == 0 && nrel) atomicAdd(&d.frel[s], (unsigned long long)nrel);
  __syncthreads();
  if (t == 0) {
    long long ab = 0;
    for (int i = 0; i < NTH / 32; ++i) ab += red[i];
    const int ph = d.fph[s];
    const bool first = d.tph[gt] != ph;  // first visit in this phase
    d.tph[gt] = ph;
    d.tact[gt] = act;
    d.mat[gt] = 1;
    d.tuni[gt] = 0;
    d.tsrc[gt] = 0;
    d.tfix[gt] = 0;
    d.tss[gt] = 0;  // h and hedge were written (after the fence above)
    const int v = atomicAdd(&d.fvis[s], 1) + 1;
    // progress: flow absorbed by deficit nodes, or excess at a height lower than any seen
    // so far in the phase (flow moving toward the sink; excess that only sloshes and
    // climbs does not count), or -- once a certificate attempt has failed, i.e. flow has
    // far to go -- excess reaching a tile for the first time in the phase
    const bool lower = bc[5] < HINF && atomicMin(&d.fhmin[s], bc[5]) > bc[5];
    if (ab > 0 || lower || (first && d.cep[s] > 0)) atomicMax(&d.fprog[s], v);
    atomicAdd(&d.fstat[s * 4 + 0], 1);
    // run again only if this task got somewhere: flow absorbed by deficit nodes or sent
    // across the border.  A tile whose excess only sloshed and climbed waits for the
    // next certificate attempt / global relabel instead of spinning on stale labels.
    bc[3] = act && (c.selfrun == 0 || ab > 0 || sides != 0);
    if (d.pdbg) {
      atomicAdd(&d.pdbg[0], 1ULL);
      if (lower) atomicAdd(&d.pdbg[1], 1ULL);
      if (ab > 0) atomicAdd(&d.pdbg[2], 1ULL);
      if (sides) atomicAdd(&d.pdbg[3], 1ULL);
      if (act) atomicAdd(&d.pdbg[6], 1ULL);
      if (rcv) atomicAdd(&d.pdbg[7], 1ULL);
      if (!lower && ab <= 0 && !sides) atomicAdd(&d.pdbg[8], 1ULL);
    }
  }
}

// ---------------------------------------------------------------- a2 fused into a1
// The seed of the frame's first global relabel (epoch 1, bound fbnd), run by the init task
// for the tiles of its group that are neither uniform sink nor uniform source (those are
// never seeded: h = 1 published at init / h = HINF by their tss stamp): h = 1 on nodes with
// e < 0, tile-local BFS fixpoint with an INF halo (the relax phase brings the neighbours'
// heights in: the neighbours that see a finite border height are flagged here, the tiles
// next to a uniform sink tile by the INIT -> BFS transition).  fl was written by this CTA.
template <int K>
__device__ void init_seed_group(const Dev& d, size_t gt0, int* smem) {
  const int t = threadIdx.x, ix = t & 31, iy0 = t >> 5;
  const int s = (int)((unsigned)gt0 / (unsigned)d.T), tile0 = (int)(gt0 - (size_t)s * d.T);
  const int n = min(d.initg, d.T - tile0);
  const int* uni_s = reinterpret_cast<const int*>(reinterpret_cast<const InitPart*>(smem) + INIT_GMAX);
  int* hs = const_cast<int*>(uni_s) + INIT_GMAX;  // [HS * HS]
  int* sc = hs + HS * HS;                         // scratch [4]
  const int bnd = __ldcg(d.fbnd + s);
  for (int j = 0; j < n; ++j) {
    if (uni_s[j]) continue;
    const size_t gt = gt0 + j;
    __syncthreads();  // hs / sc of the previous tile consumed
    int fl[4], h[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) fl[q] = __ldcg(d.fl + gt * TPX + (iy0 + 8 * q) * TS + ix);
    for (int i = t; i < HS * HS; i += NTH) hs[i] = HINF;
    if (t == 0) { sc[0] = 0; sc[1] = HINF; }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      h[q] = (fl[q] & FL_NEG) ? 1 : HINF;
      hs[hidx(iy0 + 8 * q, ix)] = h[q];
    }
    __syncthreads();
    bfs_fixpoint<K>(hs, fl, h, bnd);
    int act = 0, fix = 1, bits = 0, mnh = HINF;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int iy = iy0 + 8 * q;
      d.h[gt * TPX + iy * TS + ix] = h[q];
      act |= (fl[q] & FL_POS) && h[q] < HINF;
      if (fl[q] & FL_POS) mnh = min(mnh, h[q]);
      fix &= (h[q] == 1) || !(fl[q] & 0xff);
      if (on_border(iy, ix) && h[q] < HINF) bits |= border_bits(iy, ix);
    }
    store_hedge(d, gt, h, t);
    bits = __reduce_or_sync(0xffffffffu, bits);
    mnh = __reduce_min_sync(0xffffffffu, mnh);
    if ((t & 31) == 0) {
      if (bits) atomicOr(&sc[0], bits);
      atomicMin(&sc[1], mnh);
    }
    act = __syncthreads_or(act);
    fix = __syncthreads_and(fix);
    if (t == 0) {
      d.tact[gt] = act;
      d.tminh[gt] = sc[1];
      d.tfix[gt] = fix;
    }
    flag_sides(d, gt, sc[0], K);
  }
}

// ---------------------------------------------------------------- transitions
// first task set of a phase: NONE = the slot idles; EMPTY = no task (the next transition
// follows at once)
enum { SET_NONE = 0, SET_ALL = 1, SET_FLAG = 2, SET_TACT = 3, SET_SEED = 4, SET_CSEED = 5, SET_EMPTY = 6,
       SET_INITG = 8 };

__device__ __forceinline__ void finish_frame(const Dev& d, const IO& io, int s, const Ctl& c, int f) {
  GC_CHECK(d, f >= 0 && f < c.nframes && d.fout[s] >= 1);
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
  if (atomicAdd(&d.gctr[1], 1) + 1 == c.nframes) {
    __threadfence();
    *(volatile int*)&d.done[0] = 1;
  }
}

// Run by one CTA when the phase of slot s has no task left (fout[s] == 0): decide the next
// phase and enqueue its tasks.  Loops while a phase turns out to have no task at all.
__device__ __forceinline__ void transition(const Dev& d, const IO& io, int s, const Ctl& c, int* bc, uint32_t* sbits,
                                        int sbits_words) {
  const int t = threadIdx.x;
  if (t == 0) atomicAdd(&d.fout[s], 1);  // guard: no other CTA can see fout == 0 while we enqueue
  __shared__ int sw[12];  // the slot's words, loaded at once (one round trip)
  uint64_t tp0 = 0, tp1 = 0;  // development section timers (profiling runs only)
  const bool tprof = d.pdbg != nullptr && t == 0;
  for (;;) {
    if (tprof) { asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tp0)); atomicAdd(&d.pdbg[9], 1ULL); }
    fence_gpu();
    if (t == 0) {
      const int a0 = __ldcg(d.fmode + s), a1 = __ldcg(d.ferr + s), a2 = __ldcg(d.cep + s), a3 = __ldcg(d.cfail + s);
      const int a4 = __ldcg(d.fbnd + s), a5 = __ldcg(d.fbe + s), a6 = __ldcg(d.fph + s), a7 = __ldcg(d.sep + s);
      const int a8 = __ldcg(d.fstat + s * 4 + 1), a9 = __ldcg(d.sfr + s), a10 = __ldcg(d.fflag + s);
      sw[0] = a0; sw[1] = a1; sw[2] = a2; sw[3] = a3; sw[4] = a4;
      sw[5] = a5; sw[6] = a6; sw[7] = a7; sw[8] = a8; sw[9] = a9; sw[10] = a10;
    }
    __syncthreads();
    const int md = sw[0];
    int nact = 0, hlo = HINF;
    if (md == M_BFS) {
      for (int b0 = 0; b0 < d.T; b0 += 8 * NTH) {  // 8 tiles per thread per round trip
        int ta[8], tm[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int i = b0 + j * NTH + t;
          const size_t gt = (size_t)s * d.T + i;
          ta[j] = i < d.T ? __ldcg(d.tact + gt) : 0;
          tm[j] = i < d.T ? __ldcg(d.tminh + gt) : HINF;
        }
#pragma unroll
        for (int j = 0; j < 8; ++j)
          if (ta[j]) { nact = 1; hlo = min(hlo, tm[j]); }
      }
      hlo = __reduce_min_sync(0xffffffffu, hlo);
      if (t == 0) bc[6] = HINF;
      __syncthreads();
      if ((t & 31) == 0) atomicMin(&bc[6], hlo);
    }
    nact = __syncthreads_or(nact);
    // push wave: the phase starts on the active tiles nearest the sink; farther ones wait
    // for the next global relabel (most are cut off by then) unless flow reaches them
    // and pixels above the cap do not take part in the phase at all (frozen): in a typical
    // frame only the excess next to the object boundary has anywhere to go, and the closure
    // certificate proves the rest trapped.  The cap doubles with every failed attempt.
    const int cepn = sw[2];
    const long long capw = cepn == 0 ? (long long)c.wave : (long long)max(c.wave, 1) << min(cepn * c.wavesh, 20);
    const int hcap = md == M_BFS ? (int)min((long long)min(HINF - 1, sw[4]), (long long)bc[6] + capw) : HINF - 1;
    if (tprof) { asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tp1)); atomicAdd(&d.pdbg[10], tp1 - tp0); tp0 = tp1; }
    if (t == 0) {
      int nm = md, kind = SET_ALL;
      int* st = d.fstat + s * 4;
      bool finished = false;
      if (md == M_INIT) {
        // the init tasks seeded the first global relabel (init_seed_group): straight to its
        // relax phase; range error: the closure seeds zero the mask
        nm = sw[1] ? M_CSEED : M_BFS;
        kind = sw[1] ? SET_ALL : SET_FLAG;
        if (!sw[1]) st[1] = sw[8] + 1;
      } else if (md == M_SEED) {
        nm = M_BFS;
        kind = SET_FLAG;
        st[1] = sw[8] + 1;
      } else if (md == M_BFS) {
        if (nact) {
          nm = M_PUSH;
          kind = SET_TACT;
          d.frel[s] = 0;
          d.fvis[s] = 0;
          d.fprog[s] = 0;
          d.fdrain[s] = 0;
          d.fhmin[s] = HINF;
          d.fcap[s] = hcap;
          d.fph[s] = sw[6] + 1;
        } else {
          nm = M_CSEED;
          kind = SET_CSEED;
          // an exact relabel without an active node is the termination certificate: the
          // closure cannot fail (marker); after a bounded one it is an ordinary attempt
          d.cfail[s] = sw[4] >= HINF ? -1 : 0;
        }
      } else if (md == M_PUSH) {
        // try to certify at once: the closure of the excess nodes; if it reaches a node with
        // e < 0 the frame returns to a global relabel (epochs are unique within a frame for
        // 250 attempts; beyond that only the BFS certificate leads to the closure)
        if (sw[2] < 250) { nm = M_CSEED; kind = SET_CSEED; }
        else { nm = M_SEED; kind = SET_SEED; }
      } else if (md == M_CSEED || md == M_CLOS) {
        const int cf = sw[3];
        if (cf > 0 && (cf & 1)) {  // a closure after the BFS certificate failed: internal error
          atomicExch(&d.gctr[3], 1);
          *(volatile int*)&d.done[1] = 1;
          nm = M_IDLE;
          kind = SET_NONE;
        } else if (cf > 0) {  // not maximum yet: next attempt after a global relabel
          d.cfail[s] = 0;
          sw[2] += 1;
          d.cep[s] = sw[2];
          nm = M_SEED;
          kind = SET_SEED;
        } else if (md == M_CSEED && sw[10]) {
          nm = M_CLOS;
          kind = SET_FLAG;
        } else {  // certified (no closure relax needed, or done): the mask is written
          d.cfail[s] = 0;
          finished = true;  // (flow_state_out is written by the init pass and the closure seeds)
        }
      }
      if (finished) {
        finish_frame(d, io, s, c, sw[9]);
        // refill the slot: the next frame of the batch, or in sequence mode the next frame of
        // the slot's sequence, then the first frame of the next sequence not started
        int nf;
        if (c.seqL) {
          const int f = sw[9];
          if ((f + 1) % c.seqL != 0) {
            nf = f + 1;
          } else {
            const int j = atomicAdd(&d.gctr[0], 1);
            nf = j < c.seqS ? j * c.seqL : c.nframes;
          }
        } else {
          nf = atomicAdd(&d.gctr[0], 1);
        }
        if (nf < c.nframes) {
          slot_assign(d, io, c, s, nf);
          d.ferr[s] = 0;
          d.fph[s] = 0; d.fvis[s] = 0; d.fprog[s] = 0;
          st[0] = st[1] = st[2] = st[3] = 0;
          d.frel[s] = 0; d.sumct[s] = 0; d.sumneg[s] = 0;
          d.cep[s] = 0; d.cfail[s] = 0; d.fdrain[s] = 0;  // (fbe, fbnd: slot_assign)
          nm = M_INIT;
          kind = SET_INITG;
        } else {
          nm = M_IDLE;
          kind = SET_NONE;
          {  // a slot goes idle: release the CTAs parked on the init ring (tickets beyond its
             // tail; in batch mode no init group will be queued any more), one no-op entry each
            for (int r = 0; r < d.nparts; ++r) {
              const unsigned long long ih = atomicAdd(d.qihead + 2 * r, 0ULL), it = atomicAdd(d.qitail + 2 * r, 0ULL);
              const unsigned parked = ih > it ? (unsigned)min(ih - it, (unsigned long long)gridDim.x) : 0u;
              if (parked) {
                const unsigned long long p0 = atomicAdd(d.qitail + 2 * r, (unsigned long long)parked);
                for (unsigned i = 0; i < parked; ++i) qi_put(d, r, p0 + i, QNOP);
              }
            }
          }
        }
      }
      int fbe = finished ? 1 : sw[5];  // (slot_assign: the next frame starts at relabel 1)
      if (nm == M_SEED) {  // a new global relabel, bounded (relabel_bound)
        fbe += 1;
        d.fbe[s] = fbe;
        d.fbnd[s] = relabel_bound(d, c, sw[2]);
      }
      bc[1] = 0;
      if (nm == M_CSEED) {  // a new closure attempt: the next reach-mark epoch of the slot
        d.fflag[s] = 0;     // (set again by a closure seed that flags a tile for closure relax)
        const int se = sw[7] + 1;
        d.sep[s] = se;
        bc[1] = (se % 255) == 0;  // wrapped: clear the slot's marks first
      }
      bc[3] = fbe;
      d.fmode[s] = nm;
      bc[4] = kind;
      bc[2] = nm;
    }
    __syncthreads();
    if (tprof) { asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tp1)); atomicAdd(&d.pdbg[11], tp1 - tp0); tp0 = tp1; }
    const int kind = bc[4];
    if (kind == SET_NONE) break;
    if (bc[1]) {  // reach-mark epoch wrapped (every 255 attempts of a slot): clear its marks
      uint32_t* rm = reinterpret_cast<uint32_t*>(d.reach + (size_t)s * d.T * (c.K4 ? 4 : 8) * 64);
      const size_t words = (size_t)d.T * (c.K4 ? 4 : 8) * 16;
      for (size_t i = t; i < words; i += NTH) rm[i] = 0u;
      fence_gpu();
      __syncthreads();
    }
    // enqueue the phase's first task set, NTH tiles at a time
    const size_t base_gt = (size_t)s * d.T;
    // closure seeds: an untouched uniform source tile whose neighbours are all uniform source
    // tiles has nothing to do (its closure is the whole tile, its mask bytes are written, and
    // no border arc reaches a pixel that is not an excess node) -- a bit per tile of tsrc
    const bool srcskip = kind == SET_CSEED && (d.T + 31) / 32 <= sbits_words;
    // the first relabel's relax phase: a tile next to a uniform sink tile is relaxed (its fused
    // seed had an INF halo) -- a bit per tile of tuni
    const bool unibits = kind == SET_FLAG && md == M_INIT;
    if (srcskip || unibits) {
      const int32_t* w = srcskip ? d.tsrc : d.tuni;
      for (int b0 = 0; b0 < d.T; b0 += 8 * NTH) {  // 8 words per thread per round trip
        int v[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int i = b0 + j * NTH + t;
          v[j] = i < d.T ? __ldcg(w + base_gt + i) : 0;
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int i = b0 + j * NTH + t;
          const unsigned bal = __ballot_sync(0xffffffffu, v[j] != 0);
          if ((t & 31) == 0 && i < d.T + 31) sbits[i >> 5] = bal;
        }
      }
      __syncthreads();
    }
    // batches of TB x NTH tiles: every tile word of the batch loaded at once (one round trip),
    // the decisions, a block-wide scan of the entries, ONE reservation of queue slots and task
    // counts for the whole batch, the entries written -- a few round trips per batch instead of
    // three per 256 tiles
    if (tprof) { asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tp1)); atomicAdd(&d.pdbg[12], tp1 - tp0); tp0 = tp1; }
    constexpr int TB = 8;
    __shared__ int wsum[NTH / 32];
    for (int bb = 0; kind != SET_EMPTY && bb < d.T; bb += TB * NTH) {
      int w0[TB], w1[TB], w2[TB], w3[TB];
#pragma unroll
      for (int c2 = 0; c2 < TB; ++c2) {  // loads only (independent)
        const int i = bb + c2 * NTH + t;
        w0[c2] = w1[c2] = w2[c2] = w3[c2] = 0;
        if (i >= d.T) continue;
        const size_t gt = base_gt + i;
        if (kind == SET_SEED) {
          w0[c2] = __ldcg(d.tuni + gt); w1[c2] = __ldcg(d.tsrc + gt); w2[c2] = __ldcg(d.recv1 + gt);
        } else if (kind == SET_CSEED) {
          w0[c2] = __ldcg(d.tuni + gt); w1[c2] = __ldcg(d.mat + gt); w2[c2] = __ldcg(d.recv1 + gt);
          w3[c2] = __ldcg(d.tmk + gt);
        } else if (kind == SET_FLAG) {
          w0[c2] = __ldcg(d.flag + gt); w1[c2] = (md == M_SEED || md == M_INIT) ? __ldcg(d.tfix + gt) : 0;
        } else if (kind == SET_TACT) {
          w0[c2] = __ldcg(d.tact + gt); w1[c2] = __ldcg(d.tminh + gt);
        }
      }
      asm volatile("" ::: "memory");  // every load above is issued before any store below
      unsigned wbits = 0;   // bit c2: this thread enqueues an entry for chunk c2
#pragma unroll
      for (int c2 = 0; c2 < TB; ++c2) {  // decisions and their side effects
        const int i = bb + c2 * NTH + t;
        int want = 0;
        if (i < d.T) {
          const size_t gt = base_gt + i;
          if (kind == SET_ALL) {
            want = 1;
            d.flag[gt] = 0;
          } else if (kind == SET_INITG) {
            want = (i % d.initg) == 0;  // one init task per tile group
          } else if (kind == SET_SEED) {  // untouched uniform sink tiles keep h = 1, uniform source
            const int tu = w0[c2], tsr = w1[c2], r1 = w2[c2];
            want = !((tu | tsr) && !r1);  // tiles have no sink pixel: h = HINF until relaxed
            if (!want && tu) d.tsk[gt] = bc[3];
            if (!want && !tu) {
              d.tss[gt] = bc[3];
              d.tact[gt] = 0;
            }
            d.flag[gt] = 0;
          } else if (kind == SET_CSEED) {  // untouched uniform sink tiles are never in the closure
            const int tu = w0[c2], mt = w1[c2], r1 = w2[c2], tm = w3[c2];
            want = !(tu && !mt && !r1) || tm != 0;  // mask bytes of a failed attempt are rewritten
            if (want && srcskip && !mt && !r1 && !tm && ((sbits[i >> 5] >> (i & 31)) & 1)) {
              const int ty = i / d.TX, tx = i - ty * d.TX;
              bool inner = true;
              for (int dy = -1; dy <= 1; ++dy)
                for (int dx = -1; dx <= 1; ++dx) {
                  const int ny = ty + dy, nx = tx + dx;
                  if ((dy == 0 && dx == 0) || ny < 0 || ny >= d.TY || nx < 0 || nx >= d.TX) continue;
                  if (dy != 0 && dx != 0 && c.K4) continue;  // no diagonal arcs
                  const int n = ny * d.TX + nx;
                  inner &= ((sbits[n >> 5] >> (n & 31)) & 1) != 0;
                }
              if (inner) want = 0;
            }
            d.flag[gt] = 0;
          } else if (kind == SET_FLAG) {
            want = w0[c2];
            if (want) d.flag[gt] = 0;
            if (unibits && !((sbits[i >> 5] >> (i & 31)) & 1)) {
              const int ty = i / d.TX, tx = i - ty * d.TX;
              for (int dy = -1; dy <= 1; ++dy)
                for (int dx = -1; dx <= 1; ++dx) {
                  const int ny = ty + dy, nx = tx + dx;
                  if ((dy == 0 && dx == 0) || ny < 0 || ny >= d.TY || nx < 0 || nx >= d.TX) continue;
                  if (dy != 0 && dx != 0 && c.K4) continue;  // no diagonal arcs
                  const int n = ny * d.TX + nx;
                  want |= (sbits[n >> 5] >> (n & 31)) & 1;
                }
            }
            if (w1[c2]) want = 0;  // (seed / init relax sets) a relax cannot change it
          } else {
            want = w0[c2] && w1[c2] <= hcap;
          }
          if (want && (kind == SET_FLAG || kind == SET_TACT)) d.treq[gt] = 1;
        }
        // seed / closure-seed tasks take groups of d.bulkg consecutive tiles (the task skips
        // the tiles of its group that are not in the set): the group leader enqueues
        if ((kind == SET_SEED || kind == SET_CSEED) && d.bulkg > 1) {
          const int bg = d.bulkg;
          const unsigned bal = __ballot_sync(0xffffffffu, want);
          const int lane = t & 31, lead = lane & ~(bg - 1);
          want = (lane == lead) && ((bal >> lead) & ((1u << bg) - 1));
        }
        wbits |= (unsigned)(want != 0) << c2;
      }
      // block-wide exclusive scan of the entry counts
      const int mine = __popc(wbits);
      int incl = mine;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, incl, o);
        if ((t & 31) >= o) incl += v;
      }
      if ((t & 31) == 31) wsum[t >> 5] = incl;
      if (tprof) { asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tp1)); atomicAdd(&d.pdbg[15], tp1 - tp0); tp0 = tp1; }
      fence_gpu();  // this thread's tile-word writes are visible before the entries
      __syncthreads();
      if (tprof) { asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tp1)); atomicAdd(&d.pdbg[16], tp1 - tp0); tp0 = tp1; }
      int wbase = 0, total = 0;
#pragma unroll
      for (int w = 0; w < NTH / 32; ++w) {
        const int v = wsum[w];
        if (w < (t >> 5)) wbase += v;
        total += v;
      }
      if (total == 0) {
        __syncthreads();
        continue;
      }
      if (t == 0) {
        atomicAdd(&d.fout[s], total);
        if (d.nparts <= 1) {
          const unsigned long long p0 = atomicAdd(kind == SET_INITG ? d.qitail : d.qtail, (unsigned long long)total);
          bc[6] = (int)(p0 & 0xffffffffu);
          bc[7] = (int)(p0 >> 32);
        }
      }
      __syncthreads();
      if (tprof) { asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tp1)); atomicAdd(&d.pdbg[17], tp1 - tp0); tp0 = tp1; }
      const unsigned long long p0 = ((unsigned long long)(uint32_t)bc[7] << 32) | (uint32_t)bc[6];
      unsigned long long pos = p0 + (unsigned long long)(wbase + incl - mine);
#pragma unroll
      for (int c2 = 0; c2 < TB; ++c2) {
        if (!((wbits >> c2) & 1)) continue;
        const int i = bb + c2 * NTH + t;
        const int gcnt = ((kind == SET_SEED || kind == SET_CSEED) && d.bulkg > 1) ? min(d.bulkg, d.T - i) : 1;
        const uint32_t ent = qent(bc[2], base_gt + i, gcnt);
        if (d.nparts > 1) {  // partitioned: each entry to its band's CHAIN ring -- init groups
          // too: the band's CTAs may all be parked on that ring (no other CTA serves the band)
          const int r = part_of(d, base_gt + i);
          if (d.pdbg && r != (int)(blockIdx.x % (unsigned)d.nparts)) atomicAdd(&d.pdbg[19], 1ULL);  // cross-band
          q_put(d, r, atomicAdd(d.qtail + 2 * r, 1ULL), ent);
        } else if (kind == SET_INITG) {
          qi_put(d, 0, pos, ent);
        } else {
          q_put(d, 0, pos, ent);
        }
        ++pos;
      }
      __syncthreads();
      if (tprof) { asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tp1)); atomicAdd(&d.pdbg[18], tp1 - tp0); tp0 = tp1; }
    }
    if (tprof) { asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tp1)); atomicAdd(&d.pdbg[13], tp1 - tp0); tp0 = tp1; }
    if (t == 0) {
      const int left = atomicSub(&d.fout[s], 1) - 1;
      GC_CHECK(d, left >= 0);
      if (left == 0) atomicAdd(&d.fout[s], 1);  // every task already done (or none): go on
      bc[4] = left;
    }
    __syncthreads();
    if (tprof) { asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tp1)); atomicAdd(&d.pdbg[14], tp1 - tp0); tp0 = tp1; }
    if (bc[4] != 0) break;
  }
  __syncthreads();
}

// ---------------------------------------------------------------- the persistent kernel
// EN: energy mode (NEXT-1, the init pass builds the caps from the energy) -- a kernel of its own
// so that the cap-streaming kernel carries none of its code or registers.
template <int K, bool EN = false, int MB = GC_MINB>
__global__ void __launch_bounds__(NTH, MB) k_solve(const __grid_constant__ Dev d, const __grid_constant__ IO io,
                                                         const __grid_constant__ Ctl c, const __grid_constant__ Tmaps tm) {
  extern __shared__ __align__(128) int smem[];
  __shared__ uint64_t mbar[NTH / 32];  // one TMA barrier per warp (init stream)
  unsigned tpar = 0;                   // the warp's barrier phase
  if ((threadIdx.x & 31) == 0) mbar_init(&mbar[threadIdx.x >> 5], 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();
  __shared__ int bc[8];
  __shared__ long long red[NTH / 32];
  __shared__ uint32_t task_s;
  __shared__ uint32_t next_s;  // continuation kept by this CTA (QEMPTY: none)
  if (threadIdx.x == 0) next_s = QEMPTY;
  const int t = threadIdx.x;
  const bool prof = d.pns != nullptr;
  const int myband = d.nparts > 1 ? (int)(blockIdx.x % (unsigned)d.nparts) : 0;
  unsigned long long t_idle = 0;
  unsigned ntask_local = 0;
  for (;;) {
    if (t == 0 && next_s != QEMPTY) {  // local continuation
      task_s = next_s;
      next_s = QEMPTY;
    } else if (t == 0) {
      uint64_t w0 = 0;
      if (prof) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(w0));
      // latency-critical tasks first, then init groups.  A ticket is taken only when the ring
      // looked non-empty; a CTA that lost the race waits for the ring's next entry (chain
      // tasks arrive every few ns; the init ring is released by QNOP entries at the end).
      // Both rings empty: wait on a ticket of q (the next chain task is picked up at once).
      uint32_t v = QEMPTY;
      int ns = 32, spins = 0;
      volatile uint32_t* slot;
      {
        unsigned long long qh, qt, qih, qit;  // one 16-byte load per ring: head, tail
        const int r = myband;                 // partitioned: this CTA's band's rings only
        asm volatile("ld.volatile.global.v2.u64 {%0, %1}, [%2];" : "=l"(qh), "=l"(qt) : "l"(d.qhead + 2 * r));
        asm volatile("ld.volatile.global.v2.u64 {%0, %1}, [%2];" : "=l"(qih), "=l"(qit) : "l"(d.qihead + 2 * r));
        if (qt <= qh && qit > qih) {
          slot = d.qi + (size_t)r * (d.qimask + 1) + (atomicAdd(d.qihead + 2 * r, 1ULL) & d.qimask);
        } else {
          slot = d.q + (size_t)r * (d.qmask + 1) + (atomicAdd(d.qhead + 2 * r, 1ULL) & d.qmask);
        }
      }
      // acquire: the task's producers wrote its state before they queued it
      while ((v = ld_acquire_u32(slot)) == QEMPTY) {
        if (*(volatile int*)&d.done[0] || *(volatile int*)&d.done[1]) { v = QEXIT; break; }
        if ((++spins & 255) == 0 && *d.hostabort) { *(volatile int*)&d.done[1] = 1; v = QEXIT; break; }
        __nanosleep(ns);
        ns = ns < 1024 ? 2 * ns : 1024;
      }
      if (v != QEXIT) *slot = QEMPTY;
      if (prof) {
        uint64_t w1;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(w1));
        t_idle += w1 - w0;
      }
      task_s = v;
    }
    if (t == 0 && (++ntask_local & 15) == 0) {  // watchdogs: task budget, host stop request, abort
      if (atomicAdd(d.ntask, 16ULL) + 16 >= (unsigned long long)c.max_tasks) *(volatile int*)&d.done[1] = 1;
      if ((ntask_local & 255) == 0 && *d.hostabort) *(volatile int*)&d.done[1] = 1;
      // the abort flag is read by thread 0 alone: every thread of the CTA then takes the
      // same decision from task_s (a per-thread read could split the CTA at a barrier)
      if (*(volatile int*)&d.done[1]) task_s = QEXIT;
    }
    __syncthreads();
    const uint32_t v = task_s;
    if (v == QEXIT) break;
    if (v == QNOP) {
      __syncthreads();  // every thread has read task_s before thread 0 takes the next one
      continue;
    }
    const size_t gt = v & 0x00ffffffu;
    const int s = (int)((unsigned)gt / (unsigned)d.T);
    GC_CHECK(d, gt < NS(d) && (v >> 28) <= M_CLOS && s < d.nslot);
    GC_CHECK(d, gt + ((v >> 24) & 15) < NS(d) && (unsigned)d.sfr[s] < (unsigned)c.nframes);
    const int md = (int)(v >> 28);
    const int gcnt = (int)((v >> 24) & 15) + 1;
    const bool reqd = md == M_BFS || md == M_PUSH || md == M_CLOS;  // request-driven phase
    int c0 = 0;
    uint64_t w0 = 0;
    __shared__ int drain_s;
    if (t == 0) {
      // the tile's pending requests at the start (acquire: read before any of its state; the
      // queue slot was read with acquire, and a continuation was queued by this CTA itself)
      if (reqd) c0 = ld_acquire_s32(d.treq + gt);
      if (prof) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(w0));
      bc[1] = 0;
      bc[3] = 0;
    }
    __syncthreads();
    int cls = 0;
    switch (md) {
      case M_INIT:
        if constexpr (EN) task_init_energy<K>(d, io, gt, smem);
        else task_init<K>(d, io, gt, c.vec != 0, smem, tm, mbar, tpar);
        init_seed_group<K>(d, gt, smem);
        cls = 0;
        break;
      case M_SEED:
        for (int j = 0; j < gcnt; ++j) {
          if (j) __syncthreads();
          task_seed<K>(d, io, gt + j, smem, bc);
        }
        cls = 1;
        break;
      case M_BFS:
        task_relax<K>(d, gt, smem, bc);
        if (t == 0) atomicAdd(&d.fstat[s * 4 + 2], 1);
        cls = 1;
        break;
      case M_PUSH: task_push<K>(d, io, gt, c, smem, bc, red); cls = 2; break;
      case M_CSEED: {
        __shared__ int gw[16][5];
        cseed_group_words(d, gt, gcnt, gw);
        bool first = true;
        for (int j = 0; j < gcnt; ++j) {
          if (gw[j][0] == 1) continue;  // skipped tile: no barrier, no round trip
          if (!first) __syncthreads();
          first = false;
          task_cseed<K>(d, io, gt + j, reinterpret_cast<uint8_t*>(smem), reinterpret_cast<uint8_t*>(smem) + TPX, red, bc,
                        gw[j]);
        }
        cls = 4;
        break;
      }
      case M_CLOS:
        task_crelax<K>(d, io, gt, reinterpret_cast<uint8_t*>(smem), reinterpret_cast<uint8_t*>(smem) + TPX, bc);
        cls = 4;
        break;
      default: break;  // (no other task kinds)
    }
    // release this task's writes, then request the neighbour tiles it changed.  One
    // continuation stays in this CTA (next_s): the tile itself if it must run again, else
    // the first newly queued neighbour -- dependency chains (a BFS wave, flow moving
    // across tiles) then advance without a trip through the queue.
    fence_gpu();
    if (t == 0) drain_s = md == M_PUSH && __ldcg(d.fdrain + s);  // one read: one decision per CTA
    __syncthreads();
    int rem = 0;
    if (reqd) {
      // concurrently: thread 0 settles the tile's own requests, threads 1..8 request the
      // neighbours; no requests while a push phase drains (inflow stays flagged in recv1
      // and is absorbed by the next closure seed / seed)
      const bool drain = drain_s != 0;
      if (t == 0) {
        if (drain) {
          atomicExch(&d.treq[gt], 0);
        } else {
          const int sub = c0 - (bc[3] ? 1 : 0);  // a push task still active keeps one request
          rem = atomicSub(&d.treq[gt], sub) - sub;
          if (rem > 0 && atomicCAS(&next_s, QEMPTY, qent(md, gt)) != QEMPTY)  // run again
            chain_put(d, qent(md, gt));
        }
      } else if (t <= 8 && !drain) {
        const int b = t - 1;
        if (((bc[1] >> b) & 1) && !(b >= 4 && K == 4)) {
          const long long n = side_tile(d, gt, b);
          GC_CHECK(d, n < (long long)NS(d) && (n < 0 || (size_t)n / d.T == (size_t)s));
          if (n >= 0 && !(md == M_BFS && __ldcg(d.tfix + n))) {
            if (atomicAdd(&d.treq[n], 1) == 0) {
              atomicAdd(&d.fout[s], 1);
              const bool own = part_of(d, (size_t)n) == myband;  // another band's tile: its ring
              if (prof && !own) atomicAdd(&d.pdbg[19], 1ULL);   // (cross-band requests)
              if (!own || atomicCAS(&next_s, QEMPTY, qent(md, n)) != QEMPTY) chain_put(d, qent(md, n));
            }
          }
        }
      }
      __syncthreads();
    }
    if (t == 0) {
      int last = 0;
      if (!reqd || rem <= 0) {
        const int before = atomicSub(&d.fout[s], 1);
        GC_CHECK(d, before >= 1);
        last = before == 1;
      }
      bc[3] = last;
      if (prof) {
        uint64_t w1;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(w1));
        atomicAdd(&d.pns[cls], (unsigned long long)(w1 - w0));
        if (d.trace) {
          const unsigned long long i = atomicAdd(d.trace_n, 1ULL);
          if (i < d.trace_cap) {
            unsigned long long* r = d.trace + 4 * i;
            r[0] = w0;
            r[1] = w1 - w0;
            r[2] = ((unsigned long long)md << 56) | ((unsigned long long)gcnt << 48) |
                   ((unsigned long long)blockIdx.x << 32) | (unsigned)d.sfr[s];
            r[3] = gt - (size_t)s * d.T;
          }
        }
        // tiles processed (an init task covers a group of tiles)
        const int tl = (int)(gt - (size_t)s * d.T);
        atomicAdd(&d.ptiles[cls], md == M_INIT ? (unsigned long long)min(d.initg, d.T - tl) : (unsigned long long)gcnt);
      }
    }
    __syncthreads();
    if (bc[3]) {
      uint64_t w0t = 0;
      if (prof && t == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(w0t));
      const int sfr0 = d.sfr[s];
      transition(d, io, s, c, bc, reinterpret_cast<uint32_t*>(smem), (int)(sizeof(int) * (2 * HS * HS + TPX + K * TPX + K * 64) / 4));
      if (prof && t == 0) {
        uint64_t w1;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(w1));
        t_idle += w1 - w0t;
        if (d.trace) {  // transition record: md 15, tile = the new mode
          const unsigned long long i = atomicAdd(d.trace_n, 1ULL);
          if (i < d.trace_cap) {
            unsigned long long* r = d.trace + 4 * i;
            r[0] = w0t;
            r[1] = w1 - w0t;
            r[2] = (15ULL << 56) | ((unsigned long long)blockIdx.x << 32) | (unsigned)sfr0;
            r[3] = (unsigned long long)(unsigned)__ldcg(d.fmode + s);
          }
        }
      }
    }
  }
  if (prof && t == 0) atomicAdd(&d.pns[3], t_idle);
}

// Initial slot assignment: slot s holds frame s in M_INIT, every init tile group of every
// slot queued -- on the chain ring: nothing else is queued yet, and a call whose frames all
// fit the slots (no refills) then never uses the init ring, whose non-blocking claim lets
// idle CTAs overshoot it (C3 sequence steps of 8 VGA frames: 4x slower with the initial
// groups on the init ring).
__global__ void k_setup(Dev d, IO io, Ctl c) {
  const int G = (d.T + d.initg - 1) / d.initg;  // init tasks per frame
  const size_t ntask = (size_t)d.nslot * G;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < ntask; i += (size_t)gridDim.x * blockDim.x) {
    const size_t s = i / G, g = i - s * G;
    if (d.nparts > 1) {  // partitioned: each init group to its band's ring
      const int r = part_of(d, s * d.T + g * d.initg);
      d.q[(size_t)r * (d.qmask + 1) + (atomicAdd(d.qtail + 2 * r, 1ULL) & d.qmask)] = qent(M_INIT, s * d.T + g * d.initg);
    } else {
      d.q[i] = qent(M_INIT, s * d.T + g * d.initg);
    }
    if (g == 0) {
      slot_assign(d, io, c, (int)s, c.seqL ? (int)s * c.seqL : (int)s);  // slot s: frame s / sequence s
      d.fmode[s] = M_INIT;
      d.fout[s] = G;
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    if (d.nparts <= 1) *d.qtail = ntask;
    d.gctr[0] = d.nslot;
  }
}

// Aborted (watchdog / host timeout): frames not finished get F = -1, status GC_ERR_NOCONV
// (flow_out was preset to -1 and stats to 0 before the launch: a frame still reading -1 with
// status 0 did not finish); the frames in progress report their counters so far.
__global__ void k_abort(Dev d, IO io, int nframes) {
  const int i0 = blockIdx.x * blockDim.x + threadIdx.x, stride = gridDim.x * blockDim.x;
  for (int s = i0; s < d.nslot; s += stride) {
    if (d.fmode[s] == M_IDLE || !io.stats) continue;
    const int f = d.sfr[s];
    for (int i = 0; i < 3; ++i) io.stats[f * 4 + i] = d.fstat[s * 4 + i];
  }
  for (int f = i0; f < nframes; f += stride) {
    if (io.flow[f] != -1) continue;
    if (io.stats && io.stats[f * 4 + 3] == 2) continue;  // range error: finished
    if (io.stats) io.stats[f * 4 + 3] = 5;
  }
}

}  // namespace gcb
