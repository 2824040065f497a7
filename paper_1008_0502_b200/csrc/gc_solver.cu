// gc_solver.cu -- host driver and C ABI (include/gc.h) of the B200 grid min-cut library.
//
// Per call: carve the scratch pool into frame slots, queue every tile of the first frames,
// and launch ONE persistent kernel (k_solve, gc_phases.cuh) that runs all phases of all
// frames of the batch from a device-side work queue, refilling slots as frames finish.
// The host only waits (with a timeout that asks the kernel to stop through a mapped host
// word) and reads three counters back.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

#include <string>
#include <vector>

#include <cudaTypedefs.h>

#include "gc.h"
#include "gc_phases.cuh"

using namespace gcb;

struct gc_ctx {
  int dev = 0, K = 4, max_h = 0, max_w = 0, max_batch = 0, rounds = 8, period = 2;
  double alpha = 0.2;        // global relabel after alpha x (frame pixels) relabel operations
  long long max_launches = 1000000;
  size_t pool_bytes = 0;
  char* pool = nullptr;
  int32_t* hpin = nullptr;  // pinned host words for polling
  int32_t* habort = nullptr;      // mapped pinned word: host -> kernel stop request
  int32_t* habort_dev = nullptr;  // its device alias
  double timeout_s = 300.0;       // wall-clock bound of one k_solve launch
  int vis_mult = 64;              // push tasks per push phase = vis_mult x frame tiles
  int stall = 64;                 // push tasks without progress before a push phase drains
  int stallx = 8;                 // ... doubled per failed certificate attempt beyond stallx
  int wave = 0;                   // push cap: heights above the lowest active one + wave freeze
                                  // (doubled from 1 per failed certificate attempt)
  int selfrun = 0;                // 1: a push tile re-runs itself only after progress
  int tma = 1;                    // TMA staging of the init stream when the layout allows
  int tmapf = 0;                  // ... with an L2 prefetch this many tiles ahead (measured: slower)
  int l2ef = 0;                   // ... with an L2 evict-first policy on the cap loads
  int nparts = 1;                 // NEXT-3 band partition of each frame (gc_set_partitions)
  int grid = 0;                   // k_solve CTAs of the last launch
  int grid_max = 0;               // persistent grid of k_solve<K> on this context's device
  int grid_max_large = 0;         // ... of the large-frame variant k_solve<K, false, GC_MINB_LARGE>
  int grid_max_seq = 0;           // ... of the sequence-pass variant k_solve<K, false, GC_MINB_SEQ>
  std::string err;
  long long last_launches = 0;
  bool prof = false;
  int prof_level = 0;                    // 2: also the per-task trace (development)
  unsigned long long* trace = nullptr;   // device trace buffer [trace_cap][4] + counter
  unsigned long long trace_cap = 0;
  long long prof_n[6] = {0, 0, 0, 0, 0, 0};
  long long prof_tiles[6] = {0, 0, 0, 0, 0, 0};
  unsigned long long* dtiles = nullptr;  // device counters [12]: tasks [6], ns [6]
  double prof_ms[6] = {0, 0, 0, 0, 0, 0};
  double kernel_ms = 0;
  unsigned long long dbg[20] = {0};  // development counters (profiling only)
  std::vector<cudaEvent_t> evpool;
  std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> pending;
  size_t evnext = 0;
  // host-API staging (device)
  char* stage = nullptr;
  size_t stage_bytes = 0;
  cudaStream_t copy_st = nullptr;                  // H2D of the next chunk, overlapped with the solve
  cudaEvent_t ev_in[2] = {nullptr, nullptr};       // staging buffer b filled
  cudaEvent_t ev_free[2] = {nullptr, nullptr};     // staging buffer b solved and read back
  size_t words_bytes = 0;
  // the border-flow counters (sent, got) of the last call's layout are balanced (every frame
  // finished, so all its border flow was absorbed: sent == got, the invariant a refilled slot
  // already relies on); a call with the same layout then skips zeroing them
  bool sg_clean = false;
  int sg_key[5] = {0, 0, 0, 0, 0};
  int32_t* fbuf = nullptr;  // sequence mode: ping-pong flow buffers of the slots
  size_t fbuf_bytes = 0;
  int32_t* capbuf = nullptr;  // energy mode: the slots' cap buffers
  size_t capbuf_bytes = 0;
  int32_t* elut = nullptr;    // energy mode: n-link LUT [2][256]
  void* scratch[2] = {nullptr, nullptr};  // gc_saliency's pyramids / reductions (grow-only)
  size_t scratch_bytes[2] = {0, 0};
};

// Grow-only device scratch of the context for the other translation units of the library
// (gc_saliency.cu); not part of gc.h.  NULL if the allocation fails.
extern "C" __attribute__((visibility("hidden"))) void* gc_ctx_scratch(gc_ctx* c, int i, size_t bytes) {
  if (bytes > c->scratch_bytes[i]) {
    if (c->scratch[i]) cudaFree(c->scratch[i]);
    c->scratch[i] = nullptr;
    c->scratch_bytes[i] = 0;
    if (cudaMalloc(&c->scratch[i], bytes) != cudaSuccess) { cudaGetLastError(); return nullptr; }
    c->scratch_bytes[i] = bytes;
  }
  return c->scratch[i];
}
extern "C" __attribute__((visibility("hidden"))) void gc_ctx_set_launches(gc_ctx* c, long long n) { c->last_launches = n; }

namespace {

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// Development tuning knobs (environment variables), compiled in only with -DGC_DEV_KNOBS
// (`make DEV=1`).  The product library reads no environment variable but GC_TIMEOUT_S.
const char* knob(const char* name) {
#ifdef GC_DEV_KNOBS
  return getenv(name);
#else
  (void)name;
  return nullptr;
#endif
}

// Bytes of scratch per frame with T tiles.
size_t frame_bytes(int K, size_t T) {
  size_t b = 0;
  b += 2 * T * TPX * 4;           // e, h
  b += (size_t)K * T * TPX * 4;   // r
  b += T * TPX * 2;               // fl
  b += T * 128 * 4;               // hedge
  b += 2 * T * K * 64 * 4;        // sent, got
  b += T * K * 64;                // reach
  b += T * 8 + 13 * T * 4;        // neg0 + tile flags
  b += 2 * T * 4 * 2;             // queues (capacity >= 2 x tiles in flight)
  b += 4 * 25 + 8 * 9;            // frame words
  return b + 16 * 256;            // alignment slack
}

int tiles_of(int H, int W) { return ((H + TS - 1) / TS) * ((W + TS - 1) / TS); }

size_t pow2_at_least(size_t x) {
  size_t p = 1;
  while (p < x) p <<= 1;
  return p;
}

// Carve the pool for nslot frames of geometry H x W.
Dev carve(gc_ctx* c, int nslot, int H, int W, size_t* sentgot_bytes, size_t* q_bytes) {
  Dev d;
  memset(&d, 0, sizeof(d));
  d.H = H; d.W = W;
  d.TY = (H + TS - 1) / TS; d.TX = (W + TS - 1) / TS; d.T = d.TY * d.TX;
  d.nslot = nslot;
  d.hmax = d.T * TPX + 2;
  d.nparts = c->nparts;
  d.prow = (d.TY + d.nparts - 1) / d.nparts;  // tile rows per band (the last band may be short)
  // Tiles per init task and per seed / closure-seed task: large groups amortise the per-task
  // cost when many frames are in flight (C4), single tiles spread a latency-bound call's few
  // frames over the CTAs (C3 sequences: 8 VGA frames in flight)
  {
    const long long inflight = (long long)nslot * d.T, ctas = c->grid_max > 0 ? c->grid_max : 592;
    long long g = d.T / 20;  // (T / 32 capped QVGA batches at 2 tiles per task: C2 47-49 -> 53 Gpx/s
                             //  at 4-8; VGA batches: 8-16 best, 20 slower)
    const long long g2 = inflight / (4 * ctas);
    if (g2 < g) g = g2;
    d.initg = (int)(g < 1 ? 1 : (g > 32 ? 32 : g));
    const long long b = inflight / (8 * ctas);
    d.bulkg = b >= 8 ? 8 : (b >= 4 ? 4 : (b >= 2 ? 2 : 1));
  }
  if (const char* ev = knob("GC_INITG")) d.initg = atoi(ev) > 0 && atoi(ev) <= INIT_GMAX ? atoi(ev) : d.initg;
  if (const char* ev = knob("GC_BULKG")) d.bulkg = atoi(ev) == 1 || atoi(ev) == 2 || atoi(ev) == 4 || atoi(ev) == 8 || atoi(ev) == 16 ? atoi(ev) : d.bulkg;
  const size_t T = d.T, ns = (size_t)nslot * T, K = c->K;
  char* p = c->pool;
  auto take = [&](size_t bytes) { char* q = p; p += align_up(bytes, 256); return q; };
  // per-frame words and the queue counters first: contiguous, so one memset clears them
  char* fw = take((size_t)nslot * (4 * 25 + 8 * 9) + 64 * 4 + 32 * GC_PARTS_MAX);  // <= 25 int + 9 u64 per slot
  int32_t* w = (int32_t*)fw;
  d.fmode = w; w += nslot;
  d.sfr = w; w += nslot;
  d.fout = w; w += nslot;
  d.ferr = w; w += nslot;
  d.fph = w; w += nslot;
  d.fvis = w; w += nslot;
  d.fprog = w; w += nslot;
  d.cep = w; w += nslot;
  d.cfail = w; w += nslot;
  d.fdrain = w; w += nslot;
  d.fhmin = w; w += nslot;
  d.fbe = w; w += nslot;
  d.fcap = w; w += nslot;
  d.fbnd = w; w += nslot;
  d.sep = w; w += nslot;
  d.fflag = w; w += nslot;
  d.fstat = w; w += 4 * nslot;
  d.gctr = w; w += 4;
  d.done = w; w += 4;
  unsigned long long* u = (unsigned long long*)align_up((size_t)w, 16);
  d.frel = u; u += nslot;
  d.sumct = u; u += nslot;
  d.sumneg = u; u += nslot;
  d.scs = (const int32_t**)u; u += nslot;  // per-slot cap / flow pointers (k_setup / refills assign)
  d.sct = (const int32_t**)u; u += nslot;
  d.snb = (const int32_t**)u; u += nslot;
  d.swf = (const int32_t**)u; u += nslot;
  d.sfs = (int32_t**)u; u += nslot;
  u = (unsigned long long*)align_up((size_t)u, 16);
  const int R = d.nparts;
  d.qhead = u;  // [R] (head, tail) pairs of the chain rings, then of the init rings
  d.qtail = u + 1;
  d.qihead = u + 2 * R;
  d.qitail = u + 2 * R + 1;
  u += 4 * R;
  d.ntask = u; u += 1;
  c->words_bytes = (char*)u - fw;
  d.treq = (int32_t*)take(ns * 4);
  d.flag = (int32_t*)take(ns * 4);  // zeroed per call with treq, sent, got (init-seeds set flags)
  d.sent = (uint32_t*)take(ns * K * 64 * 4);
  d.got = (uint32_t*)take(ns * K * 64 * 4);
  d.reach = (uint8_t*)(d.got + ns * K * 64);  // zeroed per call with treq .. got (epochs: Dev::sep)
  *sentgot_bytes = (char*)(d.reach + ns * K * 64) - (char*)d.treq;
  take(ns * K * 64);
  // per band (one ring pair when not partitioned): capacity >= 2 x the band's tiles in flight
  const size_t bt = (size_t)nslot * (R > 1 ? (size_t)d.prow * d.TX : T);
  const size_t qcap = pow2_at_least(2 * bt + 1024);
  d.q = (uint32_t*)take(qcap * 4 * R);
  d.qmask = (uint32_t)(qcap - 1);
  // init ring: every slot's init groups once, plus one release entry per CTA (k_solve)
  const size_t qicap = pow2_at_least(2 * ((size_t)nslot * ((R > 1 ? (size_t)d.prow * d.TX : T) / d.initg + 2) + 4096) + 1024);
  d.qi = (uint32_t*)take(qicap * 4 * R);
  d.qimask = (uint32_t)(qicap - 1);
  *q_bytes = (char*)(d.qi + qicap) - (char*)d.q;
  d.e = (int32_t*)take(ns * TPX * 4);
  d.h = (int32_t*)take(ns * TPX * 4);
  d.r = (int32_t*)take(ns * K * TPX * 4);
  d.fl = (uint16_t*)take(ns * TPX * 2);
  d.hedge = (int32_t*)take(ns * 128 * 4);

  d.neg0 = (long long*)take(ns * 8);
  d.mat = (int32_t*)take(ns * 4);
  d.tact = (int32_t*)take(ns * 4);
  d.recv1 = (int32_t*)take(ns * 4);
  d.tuni = (int32_t*)take(ns * 4);
  d.tfix = (int32_t*)take(ns * 4);
  d.tph = (int32_t*)take(ns * 4);
  d.tminh = (int32_t*)take(ns * 4);
  d.tsk = (int32_t*)take(ns * 4);
  d.tsrc = (int32_t*)take(ns * 4);
  d.tss = (int32_t*)take(ns * 4);
  d.tmk = (int32_t*)take(ns * 4);
  d.hostabort = c->habort_dev;
  d.ptiles = c->prof ? c->dtiles : nullptr;
  d.pns = c->prof ? c->dtiles + 6 : nullptr;
  d.pdbg = c->prof ? c->dtiles + 12 : nullptr;
  d.trace = c->prof_level >= 2 ? c->trace + 1 : nullptr;
  d.trace_n = c->prof_level >= 2 ? c->trace : nullptr;
  d.trace_cap = c->trace_cap;
  return d;
}


bool ck(gc_ctx* c, cudaError_t e, const char* what) {
  if (e == cudaSuccess) return true;
  char buf[256];
  snprintf(buf, sizeof(buf), "%s: %s", what, cudaGetErrorString(e));
  c->err = buf;
  return false;
}

struct Launcher {
  gc_ctx* c;
  cudaStream_t st;
  long long n = 0;  // kernel launches issued
};

// Device time of every k_solve launch (CUDA events on the launching stream; always on).
void resolve_timing(gc_ctx* c) {
  for (auto& p : c->pending) {
    float ms = 0;
    cudaEventElapsedTime(&ms, p.second.first, p.second.second);
    for (int i = 0; i < 6; ++i) c->prof_n[i] += 1;
    c->kernel_ms += ms;
  }
  c->pending.clear();
  c->evnext = 0;
}

// Profiling counters of the last solve (profiling builds of the run only): tasks and summed
// CTA time per class.
void resolve_profile(gc_ctx* c) {
  unsigned long long t[32];
  if (cudaMemcpy(t, c->dtiles, sizeof(t), cudaMemcpyDeviceToHost) == cudaSuccess) {
    for (int i = 0; i < 20; ++i) c->dbg[i] += t[12 + i];
    for (int i = 0; i < 6; ++i) {
      c->prof_tiles[i] += (long long)t[i];
      // CTA-time of the class averaged over the persistent grid: the classes (3 = queue
      // wait + transitions) then add up to the kernel's duration
      c->prof_ms[i] += c->grid > 0 ? (double)t[6 + i] / 1e6 / c->grid : 0.0;
    }
    cudaMemset(c->dtiles, 0, sizeof(t));
  }
}

// Persistent grid size: resident CTAs per SM x SMs.
template <typename F>
int persistent_grid(gc_ctx* c, F kernel, size_t dyn_smem = 0) {
  int sms = 0, per = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kernel, NTH, dyn_smem);
  if (per < 1) per = 1;
  if (sms < 1) sms = 148;
  return sms * per;
}

// Frame slots of a call: as many as the pool holds, but no more than needed to keep the
// GPU busy -- about 40k tiles in flight, at least 24 frames.  More slots only lengthen the
// task queue, i.e. the latency of every dependency-chain step (measured: 1080p 8-nbr runs
// fastest with 15-40 slots, QVGA / VGA level off at 8k-16k tiles in flight).
int chunk_frames(gc_ctx* c, int H, int W, bool energy = false) {
  const size_t T = tiles_of(H, W);
  const size_t fb = frame_bytes(c->K, T);
  size_t n = c->pool_bytes / fb;
  // large frames: 16 slots -- the cold-start frame's chain shares the GPU with fewer streaming
  // frames (C4 1024 x 1080p, same box: 16 slots 28.8-30.7 ms, 24 slots 29.7-33.3 ms)
  // (energy solves keep 24: their init pass is float64-heavy and wants the parallelism -- 16
  // slots measured 234 vs 175 ms per 1024 frames)
  size_t want = (T >= GC_LARGE_TILES && !energy) ? 16 : (T >= 40000 / 24 ? 24 : (40000 + T - 1) / T);
  if (const char* ev = knob("GC_SLOTS")) want = atoi(ev) > 0 ? atoi(ev) : want;  // tuning knob
  if (n > want) n = want;
  if (n < 1) n = 1;
  if (c->max_batch > 0 && n > (size_t)c->max_batch) n = c->max_batch;
  if (n * T >= (1u << 24)) n = ((1u << 24) - 1) / T;  // queue entries hold 24-bit tile ids
  const char* env = knob("GC_CHUNK");
  if (env && atoi(env) > 0 && (size_t)atoi(env) < n) n = atoi(env);
  return (int)n;
}

// TMA descriptors of the init stream (gc_kernels.cuh Tmaps): cs / ct as rank-3 [n][H][W],
// nb as rank-4 [n][K][H][W] int32 tensors, 32 x 4-pixel boxes (one warp's rows of a tile).
// Needs 16-byte aligned bases and W % 4 == 0 (strides multiple of 16 bytes): ctl.vec.
bool make_tmaps(gc_ctx* c, const IO& io, int nframes, int H, int W, int K, Tmaps* tm) {
  static PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    else
      cudaGetLastError();
  }
  if (!enc) return false;
  (void)c;
  const cuuint64_t plane = (cuuint64_t)H * W * 4;
  const cuuint64_t d3[3] = {(cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)nframes};
  const cuuint64_t s3[2] = {(cuuint64_t)W * 4, plane};
  const cuuint32_t b3[3] = {32, 4, 1};
  const cuuint64_t d4[4] = {(cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)K, (cuuint64_t)nframes};
  const cuuint64_t s4[3] = {(cuuint64_t)W * 4, plane, plane * K};
  const cuuint32_t b4[4] = {32, 4, (cuuint32_t)K, 1};
  const cuuint32_t e[4] = {1, 1, 1, 1};
  auto one = [&](CUtensorMap* m, const void* base, int rank, const cuuint64_t* dims, const cuuint64_t* str,
                 const cuuint32_t* box) {
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_INT32, rank, const_cast<void*>(base), dims, str, box, e,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
  };
  return one(&tm->cs, io.cs, 3, d3, s3, b3) && one(&tm->ct, io.ct, 3, d3, s3, b3) && one(&tm->nb, io.nb, 4, d4, s4, b4);
}

double now_s() {
  timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return ts.tv_sec + 1e-9 * ts.tv_nsec;
}

// Solve `nframes` frames of geometry H x W with the slots the pool holds: slots are refilled
// on the device as frames finish (continuous batching).
// Sequence mode (seqL > 0, gc_solve_sequences): nframes = seqS x seqL frames, frame t of a
// sequence solved after frame t-1 in the same slot (warm-started from its flows if seqWarm).
// The per-call initial state of a solve in one launch instead of one memset per region: up to
// 8 segments of 32-bit words, each filled with its value (grid-stride).
struct ClearSeg {
  uint32_t* p;
  size_t n;  // words
  uint32_t v;
};
struct ClearList {
  ClearSeg seg[8];
  int cnt;
};
__global__ void k_clear(const __grid_constant__ ClearList L) {
  const size_t i0 = blockIdx.x * (size_t)blockDim.x + threadIdx.x, stride = (size_t)gridDim.x * blockDim.x;
  for (int j = 0; j < L.cnt; ++j) {
    uint32_t* p = L.seg[j].p;
    const size_t n = L.seg[j].n;
    const uint32_t v = L.seg[j].v;
    if ((((uintptr_t)p) & 15) == 0) {  // 16-byte stores for the aligned part
      uint4* q = reinterpret_cast<uint4*>(p);
      const uint4 vv = make_uint4(v, v, v, v);
      for (size_t i = i0; i < n / 4; i += stride) q[i] = vv;
      for (size_t i = (n / 4) * 4 + i0; i < n; i += stride) p[i] = v;
    } else {
      for (size_t i = i0; i < n; i += stride) p[i] = v;
    }
  }
}

template <int K>
gc_status solve_chunk(gc_ctx* c, const IO& io, int nframes, int H, int W, cudaStream_t st, Launcher& L, int seqS = 0,
                      int seqL = 0, int seqWarm = 0, int32_t* caps_out = nullptr) {
  const int units = seqL ? seqS : nframes;  // slots serve frames, or whole sequences
  const int cf = chunk_frames(c, H, W, io.img != nullptr);
  const int nslot = cf < units ? cf : units;
  size_t sg_bytes = 0, q_bytes = 0;
  Dev d = carve(c, nslot, H, W, &sg_bytes, &q_bytes);
  if (seqL && seqWarm) {  // ping-pong flow buffers, two per slot
    const size_t need = (size_t)nslot * 2 * (K / 2) * H * W * 4;
    if (need > c->fbuf_bytes) {
      if (c->fbuf) cudaFree(c->fbuf);
      c->fbuf = nullptr;
      c->fbuf_bytes = 0;
      if (cudaMalloc(&c->fbuf, need) != cudaSuccess) { cudaGetLastError(); c->err = "flow buffers"; return GC_ERR_OOM; }
      c->fbuf_bytes = need;
    }
    d.fbuf = c->fbuf;
  }
  if (io.img) {  // energy mode: caps built into the caller's caps_out, else the slots' buffers
    if (caps_out) {
      d.capbuf = caps_out;
      d.capbyframe = 1;
    } else {
      const size_t need = (size_t)nslot * (2 + K) * H * W * 4;
      if (need > c->capbuf_bytes) {
        if (c->capbuf) cudaFree(c->capbuf);
        c->capbuf = nullptr;
        c->capbuf_bytes = 0;
        if (cudaMalloc(&c->capbuf, need) != cudaSuccess) { cudaGetLastError(); c->err = "cap buffers"; return GC_ERR_OOM; }
        c->capbuf_bytes = need;
      }
      d.capbuf = c->capbuf;
    }
    if (caps_out && !ck(c, cudaMemsetAsync(caps_out, 0, (size_t)nframes * (2 + K) * H * W * 4, st), "memset"))
      return GC_ERR_CUDA;  // off-grid entries stay 0
  }
  // the call's initial state, one k_clear launch: unfinished frames read F = -1 and status 0
  // until the kernel writes them (k_abort relies on it); slot words; requests, flags, reach
  // marks (and the border-flow counters unless balanced, below); the rings (empty = all ones)
  ClearList cl;
  memset(&cl, 0, sizeof(cl));
  auto seg = [&](void* p, size_t bytes, uint32_t v) { cl.seg[cl.cnt++] = ClearSeg{(uint32_t*)p, bytes / 4, v}; };
  seg(io.flow, (size_t)nframes * 8, 0xffffffffu);
  if (io.stats) seg(io.stats, (size_t)nframes * 16, 0u);
  const size_t smem = solve_smem_bytes<K>();
  const size_t ns = (size_t)nslot * d.T;
  // large frames streamed through refilled slots (cap solves): the 3-CTA-per-SM variant
  // (GC_LARGE_TILES, gc_phases.cuh).  Measured: C4 (1024 x 1080p) 33-40 -> 31.6-34.3 ms per
  // step (a hard frame's chain runs beside the streaming frames); calls whose frames all fit
  // the slots keep 4 CTAs per SM (C5's 8 serpentine frames, all long chains: 5.9 vs 4.9 Mpx/s)
  // Sequence passes: the 2-CTA-per-SM variant (GC_MINB_SEQ: few frames in flight, each a
  // latency-bound chain -- C3 8 x 120 warm 18.7 -> 21.5 Gpx/s, cold 21.4 -> 23.2)
  const bool seqv = !io.img && seqL > 0 && c->grid_max_seq > 0;
  bool large = !io.img && !seqv && d.T >= GC_LARGE_TILES && nframes > nslot && c->grid_max_large > 0;
  if (const char* ev = knob("GC_LARGE")) large = !io.img && c->grid_max_large > 0 && atoi(ev) != 0;  // tuning knob
  int grid = seqv ? c->grid_max_seq : (large ? c->grid_max_large : c->grid_max);  // per context (gc_create)
  if (const char* ev = knob("GC_GRID")) grid = atoi(ev) > 0 && atoi(ev) < grid ? atoi(ev) : grid;
  c->grid = grid;
  seg(d.fmode, c->words_bytes, 0u);
  {
    const int key[5] = {nslot, H, W, K, d.nparts};
    const bool reuse = c->sg_clean && memcmp(key, c->sg_key, sizeof(key)) == 0;
    c->sg_clean = false;  // until this call completes
    memcpy(c->sg_key, key, sizeof(key));
    if (!reuse) {
      seg(d.treq, sg_bytes, 0u);
    } else {  // requests and flags, and the reach marks (their epochs restart per call)
      seg(d.treq, (char*)d.sent - (char*)d.treq, 0u);
      seg(d.reach, (char*)d.treq + sg_bytes - (char*)d.reach, 0u);
    }
  }
  seg(d.q, q_bytes, 0xffffffffu);
  {
    size_t words = 0;
    for (int j = 0; j < cl.cnt; ++j) words += cl.seg[j].n;
    const size_t blocks = (words / 4 + 255) / 256;
    k_clear<<<(unsigned)(blocks < 1 ? 1 : (blocks > 1184 ? 1184 : blocks)), 256, 0, st>>>(cl);
    ++L.n;
    if (!ck(c, cudaGetLastError(), "k_clear launch")) return GC_ERR_CUDA;
  }
  Ctl ctl;
  ctl.relabel_budget = (long long)(c->alpha * (double)d.T * TPX);
  ctl.vis_budget = c->vis_mult * d.T;
  ctl.stall = c->stall;
  ctl.stallx = c->stallx;
  // growth per failed certificate attempt: relabel bound 2 + 2^(1 + 2a), push cap lowest + 4^a
  // (x2 per attempt: 28 -> 20 ms for C4's cold-start frame alone, same results)
  ctl.bndsh = 2;
  ctl.wavesh = 2;
  if (const char* ev = knob("GC_BNDSH")) ctl.bndsh = atoi(ev) > 0 ? atoi(ev) : ctl.bndsh;
  if (const char* ev = knob("GC_WAVESH")) ctl.wavesh = atoi(ev) > 0 ? atoi(ev) : ctl.wavesh;
  ctl.wave = c->wave;
  ctl.selfrun = c->selfrun;
  ctl.rounds = c->rounds;
  ctl.nframes = nframes;
  ctl.K4 = K == 4;
  ctl.seqL = seqL;
  ctl.seqS = seqS;
  ctl.seqWarm = seqWarm;
  // int4 loads in the init pass when every caller row is 16-byte aligned
  ctl.vec = (W % 4 == 0) && ((uintptr_t)io.cs % 16 == 0) && ((uintptr_t)io.ct % 16 == 0) &&
            ((uintptr_t)io.nb % 16 == 0) && (!io.wf || (uintptr_t)io.wf % 16 == 0) &&
            (!d.capbuf || (uintptr_t)d.capbuf % 16 == 0);
  // watchdog: max_launches "sweeps" of the tiles in flight
  const double mt = (double)c->max_launches * (double)ns;
  ctl.max_tasks = mt > 9e18 ? (long long)9e18 : (long long)mt;
  *c->habort = 0;
  Tmaps tm;
  memset(&tm, 0, sizeof(tm));
  tm.on = ctl.vec && c->tma && !io.img && make_tmaps(c, io, nframes, H, W, K, &tm);
  tm.pf = c->tmapf;
  tm.ef = c->l2ef;
  k_setup<<<(unsigned)((ns + NTH - 1) / NTH < 4096 ? (ns + NTH - 1) / NTH : 4096), NTH, 0, st>>>(d, io, ctl);
  ++L.n;
  // the launch's device time, always measured (gc_get_kernel_ms): two events per launch
  if (c->evnext + 2 > c->evpool.size()) {
    for (int i = 0; i < 16; ++i) {
      cudaEvent_t ev;
      if (!ck(c, cudaEventCreate(&ev), "event")) return GC_ERR_CUDA;
      c->evpool.push_back(ev);
    }
  }
  cudaEvent_t e0 = c->evpool[c->evnext++];
  cudaEvent_t e1 = c->evpool[c->evnext++];
  cudaEventRecord(e0, st);
  if (io.img) k_solve<K, true><<<grid, NTH, smem, st>>>(d, io, ctl, tm);
  else if (seqv) k_solve<K, false, GC_MINB_SEQ><<<grid, NTH, smem, st>>>(d, io, ctl, tm);
  else if (large) k_solve<K, false, GC_MINB_LARGE><<<grid, NTH, smem, st>>>(d, io, ctl, tm);
  else k_solve<K><<<grid, NTH, smem, st>>>(d, io, ctl, tm);
  ++L.n;
  cudaEventRecord(e1, st);
  c->pending.push_back({0, {e0, e1}});
  if (!ck(c, cudaGetLastError(), "k_solve launch")) return GC_ERR_CUDA;
  cudaMemcpyAsync(c->hpin, d.gctr, 32, cudaMemcpyDeviceToHost, st);  // gctr[4], done[4]
  // wait (spinning for the first 2 ms: small calls are latency-bound, a sleep costs ~60 us);
  // past the timeout ask the kernel to stop (it polls the mapped word)
  const double t0 = now_s();
  for (;;) {
    const cudaError_t q = cudaStreamQuery(st);
    if (q == cudaSuccess) break;
    if (q != cudaErrorNotReady) { ck(c, q, "k_solve"); return GC_ERR_CUDA; }
    const double el = now_s() - t0;
    if (!*c->habort && el > c->timeout_s) *(volatile int32_t*)c->habort = 1;
    if (el > 2e-3) {
      struct timespec ts = {0, 20000};
      nanosleep(&ts, nullptr);
    }
  }
  const bool aborted = c->hpin[5] != 0 || c->hpin[1] < nframes;
  if (aborted && knob("GC_DEBUG")) {  // development aid: where did each slot stop?
    std::vector<int32_t> w(c->words_bytes / 4);
    cudaMemcpy(w.data(), d.fmode, w.size() * 4, cudaMemcpyDeviceToHost);
    const int32_t* base = w.data();
    for (int i = 0; i < nslot; ++i)
      fprintf(stderr, "slot %d frame %d mode %d fout %d ferr %d fph %d fvis %d fprog %d cep %d cfail %d\n", i,
              base[(d.sfr - d.fmode) + i], base[i], base[(d.fout - d.fmode) + i], base[(d.ferr - d.fmode) + i],
              base[(d.fph - d.fmode) + i], base[(d.fvis - d.fmode) + i], base[(d.fprog - d.fmode) + i],
              base[(d.cep - d.fmode) + i], base[(d.cfail - d.fmode) + i]);
    fprintf(stderr, "gctr %d %d %d done %d %d\n", base[d.gctr - d.fmode], base[d.gctr - d.fmode + 1],
            base[d.gctr - d.fmode + 2], base[d.done - d.fmode], base[d.done - d.fmode + 1]);
  }
  if (aborted) {
    k_abort<<<(nframes + NTH - 1) / NTH < 4096 ? (nframes + NTH - 1) / NTH : 4096, NTH, 0, st>>>(d, io, nframes);
    ++L.n;
    if (!ck(c, cudaStreamSynchronize(st), "abort")) return GC_ERR_CUDA;
    if (c->hpin[3] >= 2) {
      char buf[96];
      snprintf(buf, sizeof(buf), "device check failed at gc_*.cuh line %d", c->hpin[3] - 2);
      c->err = buf;
      return GC_ERR_CUDA;
    }
    if (c->hpin[3]) {
      c->err = "internal inconsistency: a closure after the BFS certificate reached a node with e < 0";
      return GC_ERR_CUDA;
    }
    if (*c->habort) c->err = "solve timed out (host watchdog)";
    return GC_ERR_NOCONV;
  }
  c->sg_clean = true;  // every frame finished: the border-flow counters are balanced
  if (c->hpin[2]) return GC_ERR_RANGE;
  return GC_OK;
}

gc_status check_batch(gc_ctx* c, const gc_batch* b) {
  if (!c) return GC_ERR_ARG;
  if (!b) { c->err = "batch is NULL"; return GC_ERR_ARG; }
  if (b->n < 0 || b->H <= 0 || b->W <= 0 || b->H > c->max_h || b->W > c->max_w) {
    char buf[160];
    snprintf(buf, sizeof(buf), "bad dims n=%d H=%d W=%d (max %dx%d)", b->n, b->H, b->W, c->max_h, c->max_w);
    c->err = buf;
    return GC_ERR_ARG;
  }
  if (b->n > 0 && (!b->cap_s || !b->cap_t || !b->cap_nb || !b->flow_out || !b->mask_out)) {
    c->err = "NULL required pointer";
    return GC_ERR_ARG;
  }
  return GC_OK;
}

gc_status worst(gc_status a, gc_status b) {
  if (a == GC_ERR_CUDA || b == GC_ERR_CUDA) return GC_ERR_CUDA;
  if (a == GC_ERR_RANGE || b == GC_ERR_RANGE) return GC_ERR_RANGE;
  if (a == GC_ERR_NOCONV || b == GC_ERR_NOCONV) return GC_ERR_NOCONV;
  return a != GC_OK ? a : b;
}

static_assert(sizeof(gc_gmm) == sizeof(Gmm), "gc_gmm and the device Gmm share one layout");

// NEXT-1: the n-link cap by |dI| (0..255) for axial (row 0) and diagonal (row 1) arcs, in
// double precision (include/gc.h gc_energy_params).
__global__ void k_energy_lut(double lambda, double sigma, double kappa, double scale, int32_t* lut) {
  const int j = blockIdx.x, dI = threadIdx.x;
  const double x = dI / 255.0;
  const double dist = j ? sqrt(2.0) : 1.0;
  const double B = lambda * exp(-(x * x) / (2.0 * sigma * sigma)) / dist + kappa;
  const double v = floor(scale * B + 0.5);
  lut[j * 256 + dI] = v <= 0.0 ? 0 : (v >= (double)CAPMAX ? CAPMAX : (int)v);
}

// NEXT-2: prior update (include/gc.h gc_prior_update).  One CTA per 64 x 64 output block of a
// frame: the mask block and its radius halo (replicated border) in shared memory, the row
// pass into shared memory as exact integers, the column pass and the integer Kalman blend in
// registers; 16 output pixels per thread, coalesced 2-byte stores.  HBM-bound stencil.
struct PriorP {
  int radius, band;
  int taps[GC_PRIOR_RMAX + 1];
  long long G2;
};
constexpr int PB = 64;                       // output block side
constexpr int PS = PB + 2 * GC_PRIOR_RMAX;   // staged side
__global__ void __launch_bounds__(256) k_prior(int H, int W, const uint8_t* __restrict__ mask,
                                               const uint16_t* __restrict__ q, const int32_t* __restrict__ wf,
                                               const __grid_constant__ PriorP p, uint16_t* __restrict__ out) {
  __shared__ uint8_t ms[PS][PS];
  __shared__ int rs[PS][PB];
  const int f = blockIdx.z, oy = blockIdx.y * PB, ox = blockIdx.x * PB, R = p.radius, t = threadIdx.x;
  const size_t plane = (size_t)H * W;
  const uint8_t* m = mask + (size_t)f * plane;
  const int S = PB + 2 * R;
  // staged rows: a warp per row, lanes over columns (no integer division)
  for (int r = t >> 5; r < S; r += 8) {
    const int yy = min(max(oy - R + r, 0), H - 1);
    const uint8_t* row = m + (size_t)yy * W;
    for (int cc = t & 31; cc < S; cc += 32) ms[r][cc] = row[min(max(ox - R + cc, 0), W - 1)] != 0;
  }
  __syncthreads();
  for (int r = t >> 6; r < S; r += 4) {  // row pass: 64 threads per staged row, one output column each
    const int cc = t & 63;
    int acc = p.taps[0] * ms[r][cc + R];
    for (int k = 1; k <= R; ++k) acc += p.taps[k] * (ms[r][cc + R - k] + ms[r][cc + R + k]);
    rs[r][cc] = acc;
  }
  __syncthreads();
  const unsigned long long w = (unsigned long long)wf[f];
  const unsigned long long D = 4096ull * (unsigned long long)p.G2;  // < 2^43
  const double invD = 1.0 / (double)D;
  for (int i = t; i < PB * PB; i += 256) {  // column pass + blend
    const int r = i >> 6, c = i & 63, y = oy + r, x = ox + c;
    if (y >= H || x >= W) continue;
    int s = p.taps[0] * rs[r + R][c];  // S <= G^2 < 2^31 (G <= 33 x 1024)
    for (int k = 1; k <= R; ++k) s += p.taps[k] * (rs[r + R - k][c] + rs[r + R + k][c]);
    const size_t o = (size_t)f * plane + (size_t)y * W + x;
    uint16_t code = 0;
    if (y >= p.band && x >= p.band && y < H - p.band && x < W - p.band) {
      const unsigned long long num = w * (unsigned long long)s * 65535ull +
                                     (4096ull - w) * q[o] * (unsigned long long)p.G2 + 2048ull * (unsigned long long)p.G2;
      // exact floor(num / D) without a 64-bit divide: a double estimate (off by at most one:
      // the quotient is <= 65535) corrected with exact 64-bit products
      unsigned long long qt = (unsigned long long)((double)num * invD);
      if (qt * D > num) --qt;
      else if ((qt + 1) * D <= num) ++qt;
      code = (uint16_t)qt;
    }
    out[o] = code;
  }
}

// a6: per-frame digest of solved frames (gc_frame_digest): F, popcount and a 64-bit hash of
// the mask, H(m) = sum over set pixels p of splitmix64(p + 1) mod 2^64 (order-independent, so
// blocks reduce in any order).  grid (blocks per frame, n); out zeroed before the launch.
__device__ __forceinline__ unsigned long long dg_mix(unsigned long long z) {
  z += 0x9e3779b97f4a7c15ULL;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

__global__ void k_digest(size_t plane, const int64_t* flow, const uint8_t* mask, unsigned long long* out) {
  const int f = blockIdx.y;
  const uint8_t* m = mask + (size_t)f * plane;
  unsigned long long pop = 0, h = 0;
  const size_t stride = (size_t)gridDim.x * blockDim.x * 4;
  for (size_t p = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) * 4; p < plane; p += stride) {
    if (p + 3 < plane && (((uintptr_t)(m + p)) & 3) == 0) {
      const uint32_t w = *reinterpret_cast<const uint32_t*>(m + p);
      if (w) {
#pragma unroll
        for (int i = 0; i < 4; ++i)
          if ((w >> (8 * i)) & 0xffu) { ++pop; h += dg_mix(p + i + 1); }
      }
    } else {
      for (size_t i = p; i < p + 4 && i < plane; ++i)
        if (m[i]) { ++pop; h += dg_mix(i + 1); }
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    pop += __shfl_xor_sync(0xffffffffu, pop, o);
    h += __shfl_xor_sync(0xffffffffu, h, o);
  }
  if ((threadIdx.x & 31) == 0) {
    if (pop) atomicAdd(out + (size_t)f * 4 + 1, pop);
    if (h) atomicAdd(out + (size_t)f * 4 + 2, h);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) out[(size_t)f * 4] = (unsigned long long)flow[f];
}

}  // namespace

extern "C" {

gc_status gc_create(const gc_config* cfg, gc_ctx** out) {
  if (!out) return GC_ERR_ARG;
  *out = nullptr;
  gc_config z;
  memset(&z, 0, sizeof(z));
  const gc_config& g = cfg ? *cfg : z;
  gc_ctx* c = new gc_ctx();
  if (cfg && g.device >= 0) {
    c->dev = g.device;  // an explicit ordinal (0 = device 0)
  } else if (cudaGetDevice(&c->dev) != cudaSuccess) {  // device < 0 (or no config): current device
    delete c;
    return GC_ERR_CUDA;
  }
  c->K = g.neighborhood ? g.neighborhood : 4;
  if (c->K != 4 && c->K != 8) { delete c; return GC_ERR_ARG; }
  c->max_h = g.max_h > 0 ? g.max_h : 1080;
  c->max_w = g.max_w > 0 ? g.max_w : 1920;
  c->rounds = g.rounds_per_launch > 0 ? g.rounds_per_launch : 16;  // 8 -> 16: 4K serpentine 3.8 -> 3.4 s, typical frames unchanged
  c->period = g.relabel_period > 0 ? g.relabel_period : 2;
  c->max_launches = g.max_launches > 0 ? g.max_launches : 1000000;
  c->max_batch = g.max_batch > 0 ? g.max_batch : 0;
  if (const char* ev = knob("GC_ALPHA")) c->alpha = atof(ev);          // tuning knobs
  if (const char* ev = knob("GC_VIS")) c->vis_mult = atoi(ev);
  if (const char* ev = knob("GC_STALL")) c->stall = atoi(ev);
  if (const char* ev = knob("GC_STALLX")) c->stallx = atoi(ev);
  if (const char* ev = knob("GC_WAVE")) c->wave = atoi(ev);
  if (const char* ev = knob("GC_SELFRUN")) c->selfrun = atoi(ev);
  if (const char* ev = knob("GC_TMA")) c->tma = atoi(ev);
  if (const char* ev = knob("GC_TMAPF")) c->tmapf = atoi(ev);
  if (const char* ev = knob("GC_L2EF")) c->l2ef = atoi(ev);
  if (const char* ev = getenv("GC_TIMEOUT_S")) c->timeout_s = atof(ev);
  if (g.max_h < 0 || g.max_w < 0 || g.max_batch < 0) { delete c; return GC_ERR_ARG; }
  if (cudaSetDevice(c->dev) != cudaSuccess) { delete c; return GC_ERR_CUDA; }
  const size_t fb = frame_bytes(c->K, tiles_of(c->max_h, c->max_w));
  size_t nf;
  if (c->max_batch > 0) {
    nf = c->max_batch;
  } else {
    // default: enough frames per pass to fill 148 SMs with active tiles (only a small
    // fraction of a realistic frame's tiles is active after the first global relabel),
    // bounded by a scratch budget of min(8 GB, 1/16 of device memory)
    size_t fr = 0, tot = 0;
    cudaMemGetInfo(&fr, &tot);
    size_t budget = (size_t)8 << 30;
    if (tot > 0 && tot / 16 < budget) budget = tot / 16;
    if (const char* ev = knob("GC_SCRATCH_MB")) budget = (size_t)atoll(ev) << 20;  // tuning knob
    nf = budget / fb;
    if (nf < 1) nf = 1;
  }
  c->pool_bytes = nf * fb + ((size_t)GC_PARTS_MAX << 18);  // + the band rings of a partitioned call
  if (cudaMalloc(&c->pool, c->pool_bytes) != cudaSuccess) { cudaGetLastError(); delete c; return GC_ERR_OOM; }
  if (cudaMallocHost(&c->hpin, 64) != cudaSuccess) { cudaFree(c->pool); delete c; return GC_ERR_OOM; }
  if (cudaMalloc(&c->dtiles, 256) != cudaSuccess) { cudaFree(c->pool); cudaFreeHost(c->hpin); delete c; return GC_ERR_OOM; }
  cudaMemset(c->dtiles, 0, 256);
  if (cudaHostAlloc(&c->habort, 64, cudaHostAllocMapped) != cudaSuccess ||
      cudaHostGetDevicePointer((void**)&c->habort_dev, c->habort, 0) != cudaSuccess) {
    cudaGetLastError();
    cudaFree(c->pool); cudaFreeHost(c->hpin); cudaFree(c->dtiles);
    if (c->habort) cudaFreeHost(c->habort);
    delete c;
    return GC_ERR_OOM;
  }
  *c->habort = 0;
  // persistent grid (resident CTAs per SM x SMs of this device), per context
  {
    const size_t smem = c->K == 8 ? solve_smem_bytes<8>() : solve_smem_bytes<4>();
    cudaError_t e = c->K == 8 ? cudaFuncSetAttribute(k_solve<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)
                              : cudaFuncSetAttribute(k_solve<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e == cudaSuccess)
      e = c->K == 8 ? cudaFuncSetAttribute(k_solve<8, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)
                    : cudaFuncSetAttribute(k_solve<4, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e == cudaSuccess)
      e = c->K == 8 ? cudaFuncSetAttribute(k_solve<8, false, GC_MINB_LARGE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)
                    : cudaFuncSetAttribute(k_solve<4, false, GC_MINB_LARGE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    c->grid_max = c->K == 8 ? persistent_grid(c, k_solve<8>, smem) : persistent_grid(c, k_solve<4>, smem);
    c->grid_max_large = c->K == 8 ? persistent_grid(c, k_solve<8, false, GC_MINB_LARGE>, smem)
                                  : persistent_grid(c, k_solve<4, false, GC_MINB_LARGE>, smem);
    if (e == cudaSuccess)
      e = c->K == 8 ? cudaFuncSetAttribute(k_solve<8, false, GC_MINB_SEQ>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)
                    : cudaFuncSetAttribute(k_solve<4, false, GC_MINB_SEQ>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    c->grid_max_seq = c->K == 8 ? persistent_grid(c, k_solve<8, false, GC_MINB_SEQ>, smem)
                                : persistent_grid(c, k_solve<4, false, GC_MINB_SEQ>, smem);
    if (e != cudaSuccess) {
      cudaGetLastError();
      gc_destroy(c);
      return GC_ERR_CUDA;
    }
  }
  *out = c;
  return GC_OK;
}

void gc_destroy(gc_ctx* c) {
  if (!c) return;
  for (auto ev : c->evpool) cudaEventDestroy(ev);
  if (c->pool) cudaFree(c->pool);
  if (c->stage) cudaFree(c->stage);
  for (int b = 0; b < 2; ++b) {
    if (c->ev_in[b]) cudaEventDestroy(c->ev_in[b]);
    if (c->ev_free[b]) cudaEventDestroy(c->ev_free[b]);
  }
  if (c->copy_st) cudaStreamDestroy(c->copy_st);
  if (c->hpin) cudaFreeHost(c->hpin);
  if (c->habort) cudaFreeHost(c->habort);
  if (c->dtiles) cudaFree(c->dtiles);
  for (int i = 0; i < 2; ++i)
    if (c->scratch[i]) cudaFree(c->scratch[i]);
  if (c->trace) cudaFree(c->trace);
  if (c->fbuf) cudaFree(c->fbuf);
  if (c->capbuf) cudaFree(c->capbuf);
  if (c->elut) cudaFree(c->elut);
  delete c;
}

const char* gc_last_error(const gc_ctx* c) { return c ? c->err.c_str() : "NULL context"; }

long long gc_last_launches(const gc_ctx* c) { return c ? c->last_launches : 0; }

gc_status gc_set_partitions(gc_ctx* c, int parts) {
  if (!c) return GC_ERR_ARG;
  if (parts < 1 || parts > GC_PARTS_MAX || parts > c->grid_max) {
    c->err = "gc_set_partitions: parts must be in [1, GC_PARTS_MAX]";
    return GC_ERR_ARG;
  }
  c->nparts = parts;
  return GC_OK;
}

void gc_set_profiling(gc_ctx* c, int enable) {
  if (!c) return;
  c->prof = enable != 0;
  c->prof_level = enable;
  if (enable >= 2 && !c->trace) {  // development trace: 4M task records
    c->trace_cap = 4u << 20;
    if (cudaMalloc(&c->trace, (c->trace_cap * 4 + 1) * 8) != cudaSuccess) {
      cudaGetLastError();
      c->trace = nullptr;
      c->trace_cap = 0;
      c->prof_level = 1;
    } else {
      cudaMemset(c->trace, 0, 8);
    }
  }
}

// Development trace of the last solves (profiling level 2; not part of gc.h): copies up to
// `cap` records of 4 u64 (see Dev::trace) to host `out`, returns the number recorded (may
// exceed cap) and resets the trace if reset != 0.
long long gc_debug_trace(gc_ctx* c, unsigned long long* out, long long cap, int reset) {
  if (!c || !c->trace) return 0;
  unsigned long long n = 0;
  cudaMemcpy(&n, c->trace, 8, cudaMemcpyDeviceToHost);
  const unsigned long long m = n < (unsigned long long)cap ? n : (unsigned long long)cap;
  const unsigned long long mm = m < c->trace_cap ? m : c->trace_cap;
  if (out && mm) cudaMemcpy(out, c->trace + 1, mm * 32, cudaMemcpyDeviceToHost);
  if (reset) cudaMemset(c->trace, 0, 8);
  return (long long)n;
}

void gc_get_profile(gc_ctx* c, long long* launches, double* ms, long long* tiles, int reset) {
  if (!c) return;
  for (int i = 0; i < 6; ++i) {
    if (launches) launches[i] = c->prof_n[i];
    if (ms) ms[i] = c->prof_ms[i];
    if (tiles) tiles[i] = c->prof_tiles[i];
  }
  if (reset)
    for (int i = 0; i < 6; ++i) { c->prof_n[i] = 0; c->prof_ms[i] = 0; c->prof_tiles[i] = 0; }
}

// Development counters of the push phase (profiling only; not part of gc.h).
void gc_debug_counters(gc_ctx* c, unsigned long long* out16, int reset) {
  if (!c) return;
  for (int i = 0; i < 20; ++i) {
    if (out16) out16[i] = c->dbg[i];
    if (reset) c->dbg[i] = 0;
  }
}

double gc_get_kernel_ms(gc_ctx* c, int reset) {
  if (!c) return 0.0;
  const double v = c->kernel_ms;
  if (reset) c->kernel_ms = 0;
  return v;
}

gc_status gc_frame_digest(gc_ctx* c, int n, int H, int W, const int64_t* flow, const uint8_t* mask, int64_t* out,
                          void* stream) {
  if (!c) return GC_ERR_ARG;
  if (n < 0 || H <= 0 || W <= 0 || (n > 0 && (!flow || !mask || !out))) {
    c->err = "gc_frame_digest: bad arguments";
    return GC_ERR_ARG;
  }
  if (n == 0) return GC_OK;
  cudaSetDevice(c->dev);
  cudaStream_t st = (cudaStream_t)stream;
  const size_t plane = (size_t)H * W;
  if (!ck(c, cudaMemsetAsync(out, 0, (size_t)n * 32, st), "digest memset")) return GC_ERR_CUDA;
  const unsigned bx = (unsigned)((plane / 4 + 255) / 256 < 64 ? (plane / 4 + 255) / 256 + 1 : 64);
  k_digest<<<dim3(bx, (unsigned)n), 256, 0, st>>>(plane, flow, mask, reinterpret_cast<unsigned long long*>(out));
  if (!ck(c, cudaGetLastError(), "k_digest launch")) return GC_ERR_CUDA;
  if (!ck(c, cudaStreamSynchronize(st), "k_digest")) return GC_ERR_CUDA;
  c->last_launches = 1;
  return GC_OK;
}

gc_status gc_gmm_prepare(int M, const double* w, const double* mean, const double* cov, gc_gmm* out) {
  if (M < 1 || M > GC_GMM_MAX || !w || !mean || !cov || !out) return GC_ERR_ARG;
  memset(out, 0, sizeof(*out));
  out->M = M;
  for (int m = 0; m < M; ++m) {
    const double* S = cov + 9 * m;
    if (!(w[m] > 0)) return GC_ERR_ARG;
    // inverse and determinant of the symmetric 3x3 S by cofactors (double precision)
    const double a = S[0], b = S[1], cc = S[2], e = S[4], f = S[5], i = S[8];
    const double A = e * i - f * f, B = -(b * i - f * cc), C = b * f - e * cc;
    const double det = a * A + b * B + cc * C;
    if (!(det > 0) || !(a > 0) || !(a * e - b * b > 0)) return GC_ERR_ARG;  // Sylvester: positive definite
    const double E = a * i - cc * cc, F = -(a * f - b * cc), I = a * e - b * b;
    out->prec[m][0] = A / det; out->prec[m][1] = B / det; out->prec[m][2] = C / det;
    out->prec[m][3] = E / det; out->prec[m][4] = F / det; out->prec[m][5] = I / det;
    for (int j = 0; j < 3; ++j) out->mean[m][j] = mean[3 * m + j];
    out->lognorm[m] = log(w[m]) - 0.5 * (3.0 * log(2.0 * M_PI) + log(det));
  }
  return GC_OK;
}

gc_status gc_gauss_taps(double sigma, int radius, int* taps) {
  if (!(sigma > 0) || radius < 0 || radius > GC_PRIOR_RMAX || !taps) return GC_ERR_ARG;
  for (int i = 0; i <= radius; ++i) taps[i] = (int)floor(1024.0 * exp(-(double)i * i / (2.0 * sigma * sigma)) + 0.5);
  return GC_OK;
}

gc_status gc_kalman_step(double s1, double s2, double v_prev, int* wf_q12, double* v_next) {
  if (!(s1 > 0) || !(s2 >= 0) || !(v_prev >= 0) || !wf_q12) return GC_ERR_ARG;
  const double den = s1 + s2 + v_prev;
  *wf_q12 = (int)floor(4096.0 * s1 / den + 0.5);
  if (v_next) *v_next = s1 * (s2 + v_prev) / den;
  return GC_OK;
}

gc_status gc_prior_update(gc_ctx* c, int n, int H, int W, const uint8_t* mask_prev, const uint16_t* q,
                          const int32_t* wf, const gc_prior_params* pp, uint16_t* prior_out, void* stream) {
  if (!c) return GC_ERR_ARG;
  if (n < 0 || H <= 0 || W <= 0 || !pp || (n > 0 && (!mask_prev || !q || !wf || !prior_out))) {
    c->err = "gc_prior_update: bad arguments";
    return GC_ERR_ARG;
  }
  PriorP p;
  p.radius = pp->radius;
  p.band = pp->band;
  long long G = 0;
  if (p.radius < 0 || p.radius > GC_PRIOR_RMAX || p.band < 0 || pp->taps[0] <= 0) {
    c->err = "gc_prior_update: bad params";
    return GC_ERR_ARG;
  }
  for (int i = 0; i <= GC_PRIOR_RMAX; ++i) {
    p.taps[i] = i <= p.radius ? pp->taps[i] : 0;
    if (p.taps[i] < 0 || p.taps[i] > 1024) { c->err = "gc_prior_update: bad taps"; return GC_ERR_ARG; }
    G += (i == 0 ? 1 : 2) * (long long)p.taps[i];
  }
  p.G2 = G * G;
  if (n == 0) return GC_OK;
  cudaSetDevice(c->dev);
  cudaStream_t st = (cudaStream_t)stream;
  const size_t plane = (size_t)H * W;
  for (int f0 = 0; f0 < n; f0 += 65535) {  // gridDim.z <= 65535 frames per launch
    const int m = n - f0 < 65535 ? n - f0 : 65535;
    k_prior<<<dim3((W + PB - 1) / PB, (H + PB - 1) / PB, m), 256, 0, st>>>(H, W, mask_prev + f0 * plane, q + f0 * plane,
                                                                            wf + f0, p, prior_out + f0 * plane);
    if (!ck(c, cudaGetLastError(), "k_prior launch")) return GC_ERR_CUDA;
  }
  if (!ck(c, cudaStreamSynchronize(st), "k_prior")) return GC_ERR_CUDA;
  c->last_launches = 1;
  return GC_OK;
}

gc_status gc_solve_energy(gc_ctx* c, const gc_energy_batch* b, void* stream) {
  if (!c) return GC_ERR_ARG;
  if (!b) { c->err = "energy batch is NULL"; return GC_ERR_ARG; }
  const gc_energy_params& p = b->params;
  if (b->n < 0 || b->H <= 0 || b->W <= 0 || b->H > c->max_h || b->W > c->max_w) {
    c->err = "bad dims";
    return GC_ERR_ARG;
  }
  if (b->n > 0 && (!b->image || !b->prior || !b->gmm || !b->flow_out || !b->mask_out)) {
    c->err = "NULL required pointer";
    return GC_ERR_ARG;
  }
  if (!(p.sigma > 0) || !(p.eps > 0 && p.eps < 0.5) || !(p.scale > 0) || !(p.lambda >= 0) || !(p.kappa >= 0)) {
    c->err = "bad energy parameters";
    return GC_ERR_ARG;
  }
  c->err.clear();
  cudaSetDevice(c->dev);
  cudaStream_t st = (cudaStream_t)stream;
  Launcher L{c, st};
  gc_status res = GC_OK;
  if (b->n > 0) {
    if (!c->elut && !ck(c, cudaMalloc(&c->elut, 2 * 256 * 4), "lut alloc")) return GC_ERR_OOM;
    k_energy_lut<<<2, 256, 0, st>>>(p.lambda, p.sigma, p.kappa, p.scale, c->elut);
    ++L.n;
    IO io{nullptr, nullptr, nullptr, b->warm_flow, b->flow_out, b->mask_out, b->flow_state_out, b->stats_out,
          b->image, b->prior, reinterpret_cast<const Gmm*>(b->gmm), c->elut, p.eps, p.scale};
    res = (c->K == 8) ? solve_chunk<8>(c, io, b->n, b->H, b->W, st, L, 0, 0, 0, b->caps_out)
                      : solve_chunk<4>(c, io, b->n, b->H, b->W, st, L, 0, 0, 0, b->caps_out);
  }
  c->last_launches = L.n;
  resolve_timing(c);
  if (c->prof) resolve_profile(c);
  if (res == GC_ERR_NOCONV && c->err.empty()) c->err = "max_launches exceeded before convergence";
  return res;
}

gc_status gc_solve_batch(gc_ctx* c, const gc_batch* b, void* stream) {
  gc_status s0 = check_batch(c, b);
  if (s0 != GC_OK) return s0;
  c->err.clear();
  cudaSetDevice(c->dev);
  cudaStream_t st = (cudaStream_t)stream;
  const int H = b->H, W = b->W, K = c->K;
  const size_t plane = (size_t)H * W;
  Launcher L{c, st};
  gc_status res = GC_OK;
  if (b->n > 0) {
    IO io{b->cap_s, b->cap_t, b->cap_nb, b->warm_flow, b->flow_out, b->mask_out, b->flow_state_out, b->stats_out};
    res = (K == 8) ? solve_chunk<8>(c, io, b->n, H, W, st, L) : solve_chunk<4>(c, io, b->n, H, W, st, L);
  }
  (void)plane;
  c->last_launches = L.n;
  resolve_timing(c);
  if (c->prof) resolve_profile(c);
  if (res == GC_ERR_RANGE && c->err.empty()) c->err = "capacity out of range [0, GC_CAP_MAX] in some frame";
  if (res == GC_ERR_NOCONV && c->err.empty()) c->err = "max_launches exceeded before convergence";
  return res;
}

gc_status gc_solve_sequences(gc_ctx* c, const gc_seq_batch* b, void* stream) {
  if (!c) return GC_ERR_ARG;
  if (!b) { c->err = "sequence batch is NULL"; return GC_ERR_ARG; }
  const long long nf = (long long)b->S * b->L;
  if (b->S < 0 || b->L <= 0 || b->H <= 0 || b->W <= 0 || b->H > c->max_h || b->W > c->max_w || nf > (1ll << 30)) {
    char buf[160];
    snprintf(buf, sizeof(buf), "bad dims S=%d L=%d H=%d W=%d (max %dx%d)", b->S, b->L, b->H, b->W, c->max_h, c->max_w);
    c->err = buf;
    return GC_ERR_ARG;
  }
  if (nf > 0 && (!b->cap_s || !b->cap_t || !b->cap_nb || !b->flow_out || !b->mask_out)) {
    c->err = "NULL required pointer";
    return GC_ERR_ARG;
  }
  c->err.clear();
  cudaSetDevice(c->dev);
  cudaStream_t st = (cudaStream_t)stream;
  Launcher L{c, st};
  gc_status res = GC_OK;
  if (nf > 0) {
    IO io{b->cap_s, b->cap_t, b->cap_nb, b->warm_flow, b->flow_out, b->mask_out, b->flow_state_out, b->stats_out};
    const int w = b->warm != 0;
    res = (c->K == 8) ? solve_chunk<8>(c, io, (int)nf, b->H, b->W, st, L, b->S, b->L, w)
                      : solve_chunk<4>(c, io, (int)nf, b->H, b->W, st, L, b->S, b->L, w);
  }
  c->last_launches = L.n;
  resolve_timing(c);
  if (c->prof) resolve_profile(c);
  if (res == GC_ERR_RANGE && c->err.empty()) c->err = "capacity out of range [0, GC_CAP_MAX] in some frame";
  if (res == GC_ERR_NOCONV && c->err.empty()) c->err = "max_launches exceeded before convergence";
  return res;
}

gc_status gc_solve_batch_host(gc_ctx* c, const gc_batch* b, void* stream) {
  gc_status s0 = check_batch(c, b);
  if (s0 != GC_OK) return s0;
  c->err.clear();
  cudaSetDevice(c->dev);
  cudaStream_t st = (cudaStream_t)stream;
  const int H = b->H, W = b->W, K = c->K;
  const size_t plane = (size_t)H * W;
  int chunk = chunk_frames(c, H, W);
  if (chunk > b->n) chunk = b->n > 0 ? b->n : 1;
  // Two staging buffers when the batch spans several chunks: the H2D copy of chunk i+1 runs on
  // copy_st while chunk i is solved on `st` (solve_chunk blocks the host, so the copy is
  // enqueued before it); the D2H read-back of chunk i follows its solve on `st`.
  const int nchunks = (b->n + chunk - 1) / chunk;
  const int nbuf = nchunks > 1 ? 2 : 1;
  struct Stage {
    int32_t *cs, *ct, *nb, *wf, *fs, *st;
    uint8_t* mask;
    int64_t* flow;
    size_t bytes;  // extent of the layout from the buffer's start
  };
  // one staging buffer's layout for m frames: caps (2+K planes), warm (K/2), flow state (K/2),
  // mask (1 B), flow (8 B), stats (16 B); every sub-buffer 256-byte aligned.  The buffer size
  // (`half`) comes from this same layout, so no sub-buffer can reach into the next buffer.
  auto layout = [&](char* base, int m) {
    size_t off = 0;
    auto take = [&](size_t bytes) { char* q = base + off; off += align_up(bytes, 256); return q; };
    Stage s;
    s.cs = (int32_t*)take(m * plane * 4);
    s.ct = (int32_t*)take(m * plane * 4);
    s.nb = (int32_t*)take(m * plane * 4 * K);
    s.wf = b->warm_flow ? (int32_t*)take(m * plane * 4 * (K / 2)) : nullptr;
    s.fs = b->flow_state_out ? (int32_t*)take(m * plane * 4 * (K / 2)) : nullptr;
    s.mask = (uint8_t*)take(m * plane);
    s.flow = (int64_t*)take(m * 8);
    s.st = (int32_t*)take(m * 16);
    s.bytes = off;
    return s;
  };
  const size_t half = layout(nullptr, chunk).bytes;
  const size_t need = half * nbuf;
  if (need > c->stage_bytes) {
    if (c->stage) cudaFree(c->stage);
    c->stage = nullptr;
    c->stage_bytes = 0;
    if (cudaMalloc(&c->stage, need) != cudaSuccess) { cudaGetLastError(); c->err = "staging alloc"; return GC_ERR_OOM; }
    c->stage_bytes = need;
  }
  if (!c->copy_st) {
    if (!ck(c, cudaStreamCreateWithFlags(&c->copy_st, cudaStreamNonBlocking), "copy stream")) return GC_ERR_CUDA;
    for (int k = 0; k < 2; ++k) {
      if (!ck(c, cudaEventCreateWithFlags(&c->ev_in[k], cudaEventDisableTiming), "event") ||
          !ck(c, cudaEventCreateWithFlags(&c->ev_free[k], cudaEventDisableTiming), "event"))
        return GC_ERR_CUDA;
    }
  }
  auto stage_of = [&](int i) {
    const int f0 = i * chunk, m = b->n - f0 < chunk ? b->n - f0 : chunk;
    return layout(c->stage + (size_t)(i % nbuf) * half, m);
  };
  auto upload = [&](int i) {  // H2D of chunk i on copy_st, once its buffer's previous chunk is read back
    const int f0 = i * chunk, m = b->n - f0 < chunk ? b->n - f0 : chunk, k = i % nbuf;
    const Stage s = stage_of(i);
    cudaStream_t cs = c->copy_st;
    if (i >= nbuf) cudaStreamWaitEvent(cs, c->ev_free[k], 0);
    cudaMemcpyAsync(s.cs, b->cap_s + f0 * plane, m * plane * 4, cudaMemcpyHostToDevice, cs);
    cudaMemcpyAsync(s.ct, b->cap_t + f0 * plane, m * plane * 4, cudaMemcpyHostToDevice, cs);
    cudaMemcpyAsync(s.nb, b->cap_nb + f0 * plane * K, m * plane * 4 * K, cudaMemcpyHostToDevice, cs);
    if (s.wf)
      cudaMemcpyAsync(s.wf, b->warm_flow + f0 * plane * (K / 2), m * plane * 4 * (K / 2), cudaMemcpyHostToDevice, cs);
    cudaEventRecord(c->ev_in[k], cs);
  };
  gc_status res = GC_OK;
  Launcher L{c, st};
  // copy_st starts after the work already on the caller's stream (a previous call's staging use)
  cudaEventRecord(c->ev_free[0], st);
  cudaStreamWaitEvent(c->copy_st, c->ev_free[0], 0);
  if (nchunks > 0) upload(0);
  for (int i = 0; i < nchunks; ++i) {
    const int f0 = i * chunk, m = b->n - f0 < chunk ? b->n - f0 : chunk, k = i % nbuf;
    if (i + 1 < nchunks) upload(i + 1);
    const Stage s = stage_of(i);
    cudaStreamWaitEvent(st, c->ev_in[k], 0);
    IO io{s.cs, s.ct, s.nb, s.wf, s.flow, s.mask, s.fs, s.st};
    gc_status r = (K == 8) ? solve_chunk<8>(c, io, m, H, W, st, L) : solve_chunk<4>(c, io, m, H, W, st, L);
    res = worst(res, r);
    if (r == GC_ERR_CUDA) break;
    cudaMemcpyAsync(b->mask_out + f0 * plane, s.mask, m * plane, cudaMemcpyDeviceToHost, st);
    cudaMemcpyAsync(b->flow_out + f0, s.flow, m * 8, cudaMemcpyDeviceToHost, st);
    if (b->stats_out) cudaMemcpyAsync(b->stats_out + f0 * 4, s.st, m * 16, cudaMemcpyDeviceToHost, st);
    if (s.fs)
      cudaMemcpyAsync(b->flow_state_out + f0 * plane * (K / 2), s.fs, m * plane * 4 * (K / 2), cudaMemcpyDeviceToHost,
                      st);
    cudaEventRecord(c->ev_free[k], st);
  }
  if (!ck(c, cudaStreamSynchronize(c->copy_st), "host solve copies")) res = GC_ERR_CUDA;
  if (!ck(c, cudaStreamSynchronize(st), "host solve")) res = GC_ERR_CUDA;
  c->last_launches = L.n;
  resolve_timing(c);
  if (c->prof) resolve_profile(c);
  if (res == GC_ERR_RANGE && c->err.empty()) c->err = "capacity out of range [0, GC_CAP_MAX] in some frame";
  if (res == GC_ERR_NOCONV && c->err.empty()) c->err = "max_launches exceeded before convergence";
  return res;
}

}  // extern "C"
