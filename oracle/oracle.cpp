// oracle.cpp -- CPU ORACLE for the per-frame grid min-cut.  TEST INFRASTRUCTURE ONLY.
//
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
// may load this library.  It shares no code with the CUDA path (paper_1008_0502_b200/):
// no headers, no helpers, no tables.  It is plain and slow on purpose.
//
// What it computes (§4 "Segmentation with graph cuts"):
//   The graph of P:331-357: one vertex per pixel plus s and t; "a pair of mutually
//   connected directed edges" per neighbouring pixel pair (footnote P:336-338) with
//   capacity c(v_x, v_y) = cap_nb[k][y][x] for the arc x -> x + d_k; t-links
//   c(s, v_x) = cap_s (cost of label 0) and c(v_x, t) = cap_t (cost of label 1)
//   (reading c1: source side = label 1 = object).  Arcs pointing off the
//   grid are dropped (reading c7).  "The minimum cut of the graph separating the
//   source and the sink provides the MAP configuration".
//   Outputs: F* = max-flow value = min-cut capacity (int64, exact), and the canonical
//   mask = the set of pixels reachable from s in the residual graph of the maximum
//   flow (reading c2: the inclusion-minimal minimum cut; ties go to label 0).
//
// Two independent max-flow algorithms compute F* and a maximum flow:
//   - Dinic (level graph by BFS from s, blocking flow by DFS with current-arc
//     pointers; iterative, because augmenting paths reach ~10^6 pixels);
//   - Boykov-Kolmogorov (search trees S and T grown from s and t, augmentation along
//     the found path, orphan adoption), the algorithm family the paper cites for graph
//     cuts (SPEC S:485 names it for the CPU program).
// After either, the mask is recomputed by a plain BFS from s over arcs with positive
// residual capacity -- never read off BK's trees (SURVEY.md §7 "hard parts" 2).
//
// Also: brute force over all 2^N labelings (N <= 24) of the cut capacity
//   cut(S) = sum_{v notin S} c(s,v) + sum_{v in S} c(v,t) + sum_{p in S, q notin S} c(p->q)
// (SURVEY.md §8(c) "plain definition"), with mask* = intersection of all minimisers; and
// an evaluator of that same cut(S) for a given mask (duality check).
#include <stdint.h>
#include <string.h>

#include <algorithm>
#include <atomic>
#include <thread>
#include <vector>

namespace {

const int DY[8] = {0, 0, 1, -1, 1, -1, 1, -1};
const int DX[8] = {1, -1, 0, 0, 1, -1, -1, 1};

// Residual graph with paired arcs: arc a and a^1 are mutual reverses.
struct Graph {
  int n = 0;  // vertices: pixels 0..N-1, s = N, t = N+1
  int s = 0, t = 0;
  std::vector<int> first;   // first arc out of a vertex (-1 = none)
  std::vector<int> next;    // next arc out of the same tail
  std::vector<int> head;    // head vertex of the arc
  std::vector<int64_t> res; // residual capacity

  void init(int nv) {
    n = nv;
    first.assign(nv, -1);
    next.clear(); head.clear(); res.clear();
  }
  // adds arc u->v with capacity cuv and its partner v->u with capacity cvu
  void add_pair(int u, int v, int64_t cuv, int64_t cvu) {
    int a = (int)head.size();
    head.push_back(v); res.push_back(cuv); next.push_back(first[u]); first[u] = a;
    head.push_back(u); res.push_back(cvu); next.push_back(first[v]); first[v] = a + 1;
  }
  int tail(int a) const { return head[a ^ 1]; }
};

// Build the graph of P:331-357 for one frame.  cap_nb is [K][H][W].
void build(Graph& g, int H, int W, int K, const int32_t* cs, const int32_t* ct, const int32_t* nb) {
  int N = H * W;
  g.init(N + 2);
  g.s = N; g.t = N + 1;
  for (int v = 0; v < N; ++v) {
    // t-links: s -> v with c(s,v) (reverse 0), v -> t with c(v,t) (reverse 0)
    g.add_pair(g.s, v, cs[v], 0);
    g.add_pair(v, g.t, ct[v], 0);
  }
  // n-links: the pair (p -> q, q -> p) for each unordered neighbour pair, taken once
  // through the "forward" directions k = 0 (E), 2 (S), 4 (SE), 6 (SW); the reverse
  // direction of k is k^1, whose capacity is stored at q.
  for (int y = 0; y < H; ++y)
    for (int x = 0; x < W; ++x)
      for (int k = 0; k < K; k += 2) {
        int y2 = y + DY[k], x2 = x + DX[k];
        if (y2 < 0 || y2 >= H || x2 < 0 || x2 >= W) continue;  // off-grid: ignored (c7)
        int p = y * W + x, q = y2 * W + x2;
        int64_t cpq = nb[(int64_t)k * N + p];
        int64_t cqp = nb[(int64_t)(k ^ 1) * N + q];
        g.add_pair(p, q, cpq, cqp);
      }
}

// ---------------------------------------------------------------- Dinic
int64_t dinic(Graph& g) {
  const int n = g.n;
  std::vector<int> level(n), it(n), queue(n);
  std::vector<int> path;  // arc stack of the current DFS path
  int64_t flow = 0;
  for (;;) {
    // BFS levels from s over arcs with residual > 0
    std::fill(level.begin(), level.end(), -1);
    int qh = 0, qt = 0;
    level[g.s] = 0; queue[qt++] = g.s;
    while (qh < qt) {
      int u = queue[qh++];
      for (int a = g.first[u]; a != -1; a = g.next[a])
        if (g.res[a] > 0 && level[g.head[a]] < 0) {
          level[g.head[a]] = level[u] + 1;
          queue[qt++] = g.head[a];
        }
    }
    if (level[g.t] < 0) break;
    for (int v = 0; v < n; ++v) it[v] = g.first[v];
    // blocking flow: repeated DFS s -> t along level-increasing arcs (iterative)
    for (;;) {
      path.clear();
      int u = g.s;
      bool found = false;
      while (true) {
        if (u == g.t) { found = true; break; }
        int& a = it[u];
        while (a != -1 && !(g.res[a] > 0 && level[g.head[a]] == level[u] + 1)) a = g.next[a];
        if (a == -1) {  // dead end: retreat
          if (u == g.s) break;
          level[u] = -1;  // prune
          int back = path.back(); path.pop_back();
          u = g.tail(back);
          it[u] = g.next[it[u]];
          continue;
        }
        path.push_back(a);
        u = g.head[a];
      }
      if (!found) break;
      int64_t d = INT64_MAX;
      for (int a : path) d = std::min(d, g.res[a]);
      for (int a : path) { g.res[a] -= d; g.res[a ^ 1] += d; }
      flow += d;
    }
  }
  return flow;
}

// ---------------------------------------------------------------- Boykov-Kolmogorov
// As published (Boykov & Kolmogorov, PAMI 2004): terminal arcs are not scanned as
// adjacency -- every pixel starts as a child of s or t through its t-link (after pushing
// min(c(s,v), c(v,t)) straight s -> v -> t), then search trees S and T grow along
// n-links, an S-T meeting arc gives an augmenting path, saturated tree arcs create
// orphans, and orphans are re-adopted (timestamp/distance validity test) or freed.
// tree[v]: 0 free, 1 S, 2 T.  parent[v]: TERM (child of its terminal), NONE, or the
// n-link arc from the parent to v (S) / from v to the parent (T).
// Build order of build(): arcs 4v, 4v+1 = (s->v, v->s); 4v+2, 4v+3 = (v->t, t->v).
int64_t boykov_kolmogorov(Graph& g) {
  const int N = g.n - 2;
  const int NONE = -1, TERM = -2;
  std::vector<int> tree(N, 0), parent(N, NONE), ts(N, 0), dist(N, 0);
  std::vector<char> in_active(N, 0);
  std::vector<int> active;  // FIFO with head index
  size_t ahead = 0;
  std::vector<int> orphans;
  int64_t flow = 0;
  int TIME = 0;
  auto aS = [](int v) { return 4 * v; };      // s -> v
  auto aT = [](int v) { return 4 * v + 2; };  // v -> t
  auto push_arc = [&](int a, int64_t d) { g.res[a] -= d; g.res[a ^ 1] += d; };

  for (int v = 0; v < N; ++v) {
    int64_t d = std::min(g.res[aS(v)], g.res[aT(v)]);
    if (d > 0) { push_arc(aS(v), d); push_arc(aT(v), d); flow += d; }
    if (g.res[aS(v)] > 0) tree[v] = 1;
    else if (g.res[aT(v)] > 0) tree[v] = 2;
    if (tree[v]) { parent[v] = TERM; dist[v] = 1; active.push_back(v); in_active[v] = 1; }
  }
  auto pnode = [&](int v) -> int {  // parent pixel of a non-root tree pixel
    int a = parent[v];
    return tree[v] == 1 ? g.tail(a) : g.head[a];
  };
  auto is_term = [&](int v) { return v >= N; };

  for (;;) {
    // ---- growth
    int meet = -1;  // n-link arc p -> q with p in S, q in T, residual > 0
    while (ahead < active.size() && meet < 0) {
      int p = active[ahead];
      if (tree[p] == 0) { ++ahead; in_active[p] = 0; continue; }
      int tr = tree[p];
      for (int a = g.first[p]; a != -1; a = g.next[a]) {
        int q = g.head[a];
        if (is_term(q)) continue;
        int64_t c = (tr == 1) ? g.res[a] : g.res[a ^ 1];
        if (c <= 0) continue;
        if (tree[q] == 0) {
          tree[q] = tr;
          parent[q] = (tr == 1) ? a : (a ^ 1);
          ts[q] = ts[p];
          dist[q] = dist[p] + 1;
          if (!in_active[q]) { active.push_back(q); in_active[q] = 1; }
        } else if (tree[q] != tr) {
          meet = (tr == 1) ? a : (a ^ 1);
          break;
        }
      }
      if (meet < 0) { ++ahead; in_active[p] = 0; }
    }
    if (meet < 0) break;

    // ---- augmentation along s -> ... -> p -> q -> ... -> t
    ++TIME;
    int p = g.tail(meet), q = g.head[meet];
    int64_t d = g.res[meet];
    int u;
    for (u = p; parent[u] != TERM; u = g.tail(parent[u])) d = std::min(d, g.res[parent[u]]);
    d = std::min(d, g.res[aS(u)]);
    for (u = q; parent[u] != TERM; u = g.head[parent[u]]) d = std::min(d, g.res[parent[u]]);
    d = std::min(d, g.res[aT(u)]);
    push_arc(meet, d);
    for (u = p; parent[u] != TERM;) {
      int a = parent[u];
      push_arc(a, d);
      int pu = g.tail(a);
      if (g.res[a] == 0) { parent[u] = NONE; orphans.push_back(u); }
      u = pu;
    }
    push_arc(aS(u), d);
    if (g.res[aS(u)] == 0) { parent[u] = NONE; orphans.push_back(u); }
    for (u = q; parent[u] != TERM;) {
      int a = parent[u];
      push_arc(a, d);
      int pu = g.head[a];
      if (g.res[a] == 0) { parent[u] = NONE; orphans.push_back(u); }
      u = pu;
    }
    push_arc(aT(u), d);
    if (g.res[aT(u)] == 0) { parent[u] = NONE; orphans.push_back(u); }
    flow += d;

    // ---- adoption
    while (!orphans.empty()) {
      int o = orphans.back(); orphans.pop_back();
      int tr = tree[o];
      if ((tr == 1 && g.res[aS(o)] > 0) || (tr == 2 && g.res[aT(o)] > 0)) {
        parent[o] = TERM; ts[o] = TIME; dist[o] = 1;
        continue;
      }
      int best = NONE, dmin = INT32_MAX;
      for (int a = g.first[o]; a != -1; a = g.next[a]) {
        int v = g.head[a];
        if (is_term(v) || tree[v] != tr) continue;
        int pa = (tr == 1) ? (a ^ 1) : a;  // S: arc v -> o ; T: arc o -> v
        if (g.res[pa] <= 0) continue;
        int dd = 0, j = v;
        bool ok;
        for (;;) {
          if (ts[j] == TIME) { dd += dist[j]; ok = true; break; }
          if (parent[j] == NONE) { ok = false; break; }
          ++dd;
          if (parent[j] == TERM) { ts[j] = TIME; dist[j] = 1; ok = true; break; }
          j = pnode(j);
        }
        if (!ok) continue;
        if (dd < dmin) { dmin = dd; best = pa; }
        for (j = v; ts[j] != TIME; j = pnode(j)) { ts[j] = TIME; dist[j] = dd--; }
      }
      if (best != NONE) {
        parent[o] = best; ts[o] = TIME; dist[o] = dmin + 1;
        continue;
      }
      for (int a = g.first[o]; a != -1; a = g.next[a]) {
        int v = g.head[a];
        if (is_term(v) || tree[v] != tr) continue;
        int pa = (tr == 1) ? (a ^ 1) : a;
        if (g.res[pa] > 0 && !in_active[v]) { active.push_back(v); in_active[v] = 1; }
        int child_arc = (tr == 1) ? a : (a ^ 1);  // S: o -> v ; T: v -> o
        if (parent[v] == child_arc) { parent[v] = NONE; orphans.push_back(v); }
      }
      tree[o] = 0;
      parent[o] = NONE;
    }
    if (ahead > 4096 && ahead >= active.size() / 2) {
      active.erase(active.begin(), active.begin() + ahead);
      ahead = 0;
    }
  }
  return flow;
}

// mask = pixels reachable from s over residual arcs (reading c2)
void residual_mask(const Graph& g, uint8_t* mask, int N) {
  std::vector<char> seen(g.n, 0);
  std::vector<int> q;
  q.push_back(g.s); seen[g.s] = 1;
  for (size_t i = 0; i < q.size(); ++i) {
    int u = q[i];
    for (int a = g.first[u]; a != -1; a = g.next[a])
      if (g.res[a] > 0 && !seen[g.head[a]]) { seen[g.head[a]] = 1; q.push_back(g.head[a]); }
  }
  for (int v = 0; v < N; ++v) mask[v] = seen[v] ? 1 : 0;
}

}  // namespace

extern "C" {

// Solves one frame.  algo 0 = Dinic, 1 = Boykov-Kolmogorov.  Returns F*; writes mask [H][W].
// If flow_fwd != NULL, writes the net n-link flow on the forward directions
// [K/2][H][W] (plane j = direction 2j), for warm-start tests.
int64_t oracle_solve(int algo, int H, int W, int K, const int32_t* cs, const int32_t* ct, const int32_t* nb,
                     uint8_t* mask, int32_t* flow_fwd) {
  Graph g;
  build(g, H, W, K, cs, ct, nb);
  std::vector<int64_t> cap0 = g.res;
  int64_t F = (algo == 1) ? boykov_kolmogorov(g) : dinic(g);
  residual_mask(g, mask, H * W);
  if (flow_fwd) {
    int N = H * W;
    memset(flow_fwd, 0, sizeof(int32_t) * (size_t)(K / 2) * N);
    // arcs were added in build() order: 2 t-link pairs per pixel, then n-link pairs
    int a = 4 * N;
    for (int y = 0; y < H; ++y)
      for (int x = 0; x < W; ++x)
        for (int k = 0; k < K; k += 2) {
          int y2 = y + DY[k], x2 = x + DX[k];
          if (y2 < 0 || y2 >= H || x2 < 0 || x2 >= W) continue;
          flow_fwd[(int64_t)(k / 2) * N + y * W + x] = (int32_t)(cap0[a] - g.res[a]);
          a += 2;
        }
  }
  return F;
}

// cut(S) of SURVEY.md §8(c) for S = {v : mask[v] = 1}; off-grid arcs ignored.
int64_t oracle_cut_value(int H, int W, int K, const int32_t* cs, const int32_t* ct, const int32_t* nb,
                         const uint8_t* mask) {
  int N = H * W;
  int64_t c = 0;
  for (int v = 0; v < N; ++v) c += mask[v] ? (int64_t)ct[v] : (int64_t)cs[v];
  for (int y = 0; y < H; ++y)
    for (int x = 0; x < W; ++x)
      for (int k = 0; k < K; ++k) {
        int y2 = y + DY[k], x2 = x + DX[k];
        if (y2 < 0 || y2 >= H || x2 < 0 || x2 >= W) continue;
        if (mask[y * W + x] && !mask[y2 * W + x2]) c += nb[(int64_t)k * N + y * W + x];
      }
  return c;
}

// Brute force over all 2^N labelings (N <= 24): F* = min cut(S), mask* = intersection
// of all minimisers.  Returns F*; -1 if N too large.
int64_t oracle_brute(int H, int W, int K, const int32_t* cs, const int32_t* ct, const int32_t* nb,
                     uint8_t* mask) {
  int N = H * W;
  if (N > 24) return -1;
  std::vector<uint8_t> m(N);
  int64_t best = INT64_MAX;
  uint32_t inter = 0;
  for (uint32_t S = 0; S < (1u << N); ++S) {
    for (int v = 0; v < N; ++v) m[v] = (S >> v) & 1u;
    int64_t c = oracle_cut_value(H, W, K, cs, ct, nb, m.data());
    if (c < best) { best = c; inter = S; }
    else if (c == best) inter &= S;
  }
  for (int v = 0; v < N; ++v) mask[v] = (inter >> v) & 1u;
  return best;
}

// Batch of n frames on `threads` host threads (one frame per task), for the CPU baseline.
void oracle_solve_batch(int algo, int n, int H, int W, int K, const int32_t* cs, const int32_t* ct,
                        const int32_t* nb, uint8_t* mask, int64_t* F, int threads) {
  if (threads < 1) threads = 1;
  std::atomic<int> next(0);
  int64_t px = (int64_t)H * W;
  auto work = [&]() {
    for (;;) {
      int i = next.fetch_add(1);
      if (i >= n) break;
      F[i] = oracle_solve(algo, H, W, K, cs + i * px, ct + i * px, nb + i * px * K, mask + i * px, nullptr);
    }
  };
  std::vector<std::thread> pool;
  for (int i = 0; i < threads; ++i) pool.emplace_back(work);
  for (auto& th : pool) th.join();
}

}  // extern "C"
