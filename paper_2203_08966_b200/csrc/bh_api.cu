// bh_api.cu -- the handle and the extern "C" entry points of libbh.so.
//
// The handle owns only workspace (sort scratch, the tree, the resident body
// state); callers own every buffer they pass.  Nothing here synchronises the
// stream except bh_check, the cell-count read inside a build (one 8-byte D2H
// per build) and the explicit query calls (bh_tree_size, bh_stats_get).
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <utility>
#include <vector>

#include "bh_internal.cuh"

using namespace bh;

namespace {
thread_local std::string g_err;

int fail(int code, const std::string &msg) {
  g_err = msg;
  return code;
}

#define BH_CUDA(expr)                                                              \
  do {                                                                             \
    cudaError_t e_ = (expr);                                                       \
    if (e_ != cudaSuccess)                                                         \
      return fail(e_ == cudaErrorMemoryAllocation ? BH_OUT_OF_MEMORY : BH_CUDA_ERROR, \
                  std::string(#expr) + ": " + cudaGetErrorString(e_));             \
  } while (0)

#define BH_LAUNCHED()                                                              \
  do {                                                                             \
    cudaError_t e_ = cudaGetLastError();                                           \
    if (e_ != cudaSuccess)                                                         \
      return fail(BH_CUDA_ERROR, std::string("kernel launch: ") + cudaGetErrorString(e_)); \
  } while (0)

#define BH_TRY(expr)          \
  do {                        \
    int r_ = (expr);          \
    if (r_ != BH_OK) return r_; \
  } while (0)

inline cudaStream_t S(void *s) { return static_cast<cudaStream_t>(s); }
}  // namespace

struct bh_handle {
  int device = 0;
  int precision = BH_FP32;
  // replicated ranks: peers' resident acc / work (bh_sim_set_peers)
  int npeers = 0;
  void *peer_acc[kMaxPeers] = {}, *peer_work[kMaxPeers] = {};
  bool peer_ipc = false;
  void *peer_own_acc = nullptr, *peer_own_work = nullptr;  // our buffers when the peers mapped them
  DeviceFlags *flags = nullptr;   // device
  DeviceFlags *hflags = nullptr;  // pinned host mirror
  uint32_t *hC = nullptr;         // pinned: off[n-1], newc[n-1]
  double *dR = nullptr;           // device scratch R (sim path)
  double *hR = nullptr;           // pinned
  // sort / build scratch
  Buf keys, keys2, vals, vals2, sort_tmp, scan_tmp, lcp, newc, off;
  // tree
  int64_t tree_n = -1, C = 0, max_level = 0;
  // sync-free build (fp32 resident path): capacity, device count, snapshot
  bool async_tree = false;
  int64_t cap = 0, C_true = 0;
  int cur_step = 0;       // step index inside a bh_sim_step call (recorded on overflow)
  int mom_leaf = 0;       // > 0: the moments cover only what a walk with leaf size >= mom_leaf reads
  int *dCtrue = nullptr;
  int *hstat = nullptr;  // pinned: [0] = C, [1..22] = internal cells per level
  int grid_lvl[kMaxLevel + 1] = {0};
  Buf bk_pos, bk_vel, bk_acc, bk_id, bk_work;
  // distributed build (decomposition.py): boundary lcps, shared cells, branches
  int bnd_prev = -1, bnd_next = -1;
  Buf shared, branch, rec_of_cell, wparent;
  int64_t nbranch = 0;
  // locally essential trees of the last build_local
  Buf let_present, let_expand, let_bodies, let_isbranch, let_rflag, let_bcount, let_rpos,
      let_bpos, let_scan_tmp, let_brec, let_tail, let_boxkey, let_lvl, let_list;
  uint32_t *hlet = nullptr;  // pinned: LET sizes per receiver
  // work of the last walk is in work_sorted; its scatter to the caller's order
  // (work_orig) is deferred until someone reads it (a random 4-byte scatter:
  // ~3.8 ms per step at 1e8 bodies), and dropped inside a multi-step call
  bool work_dirty = false;
  bool drop_work = false;
  // bh_sim_step_host: staging and the side stream for the early position copy
  Buf hs_a, hs_b, hs_pos;
  float *host_pos4 = nullptr;  // the caller's pos4 of the running bh_sim_step_host call
  cudaStream_t side = nullptr;
  cudaStream_t cp[2] = {nullptr, nullptr};  // concurrent host copies (H2D reads overlap on PCIe)
  cudaEvent_t ev_cp[3] = {nullptr, nullptr, nullptr};
  cudaEvent_t ev_pos = nullptr, ev_side = nullptr;
  int let_nrank = 0;
  int64_t let_nrec = 0;
  double R = 1.0;
  Buf link, parent, child8, lvl, lvl_list, cm64, q64, tbod, mclass, hperm;
  int *hlvl = nullptr;  // pinned: internal cells per level of the last build
  int sms = 148;
  int allow_dup = 0;       // bh_set_allow_duplicates; the sim path uses leaf_size > 1
  const float4 *tbod32 = nullptr;   // bodies of the current tree (sorted)
  const double4 *tbod64 = nullptr;
  // fp32 walk tree (compacted per (theta, leaf size))
  Buf smask, nck, wbase, wnodes, wscan_tmp;
  int *dCp = nullptr;
  double walk_theta = -1.0;
  int walk_leaf = -1;
  bool walk_valid = false;
  // resident simulation state (Morton order)
  int64_t sim_n = 0;
  Buf pos, pos2, vel, vel2, acc, id, id2, work_sorted, work_orig;
  // instrumentation
  struct Mark { int phase; cudaEvent_t a, b; };
  bool timing = false;
  std::vector<Mark> marks;
  std::vector<cudaEvent_t> pool;
  Mark open{0, nullptr, nullptr};
  double phase_ms[BH_NPHASES] = {0};
  int64_t launches = 0;

  cudaEvent_t get_event() {
    if (!pool.empty()) { cudaEvent_t e = pool.back(); pool.pop_back(); return e; }
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    return e;
  }
  void fold_marks() {
    for (Mark &m : marks) {
      cudaEventSynchronize(m.b);
      float ms = 0.f;
      cudaEventElapsedTime(&ms, m.a, m.b);
      phase_ms[m.phase] += ms;
      pool.push_back(m.a);
      pool.push_back(m.b);
    }
    marks.clear();
  }
  void tbegin(int phase, cudaStream_t s) {
    if (!timing) return;
    if (open.a) {  // a phase left open by an error return: recycle its events, drop the mark
      pool.push_back(open.a);
      pool.push_back(open.b);
    }
    open.phase = phase;
    open.a = get_event();
    open.b = get_event();
    cudaEventRecord(open.a, s);
  }
  void tend(cudaStream_t s) {
    if (!timing || !open.a) return;
    cudaEventRecord(open.b, s);
    marks.push_back(open);
    open.a = open.b = nullptr;
    if (marks.size() > 4096) fold_marks();
  }

  TreeView view() {
    TreeView t;
    t.n = tree_n;
    t.C = C;
    t.dC = async_tree ? dCtrue : nullptr;
    t.bnd_prev = bnd_prev;
    t.bnd_next = bnd_next;
    t.keys = keys2.as<uint64_t>();
    t.lcp = lcp.as<int8_t>();
    t.off = off.as<uint32_t>();
    t.newc = newc.as<uint32_t>();
    t.link = link.as<int4>();
    t.parent = parent.as<int>();
    t.child8 = child8.as<int>();
    t.bod32 = tbod32;
    t.bod64 = tbod64;
    t.cm64 = cm64.as<double4>();
    t.q64 = q64.as<double>();
    if (mom_leaf > 1) {  // a walk-only tree: its class bytes (emit) and the moments'
      t.mclass = mclass.as<uint8_t>();  // lists of opened cells drive the compaction
      t.mleaf = mom_leaf;
      t.mlvl = lvl.as<int>();
      t.mlist = lvl_list.as<int>();
    }
    return t;
  }
};

static void close_peers(bh_handle *h) {
  if (h->peer_ipc)
    for (int r = 0; r < h->npeers; ++r) {
      if (h->peer_acc[r]) cudaIpcCloseMemHandle(h->peer_acc[r]);
      if (h->peer_work[r]) cudaIpcCloseMemHandle(h->peer_work[r]);
    }
  for (int r = 0; r < kMaxPeers; ++r) h->peer_acc[r] = h->peer_work[r] = nullptr;
  h->npeers = 0;
  h->peer_ipc = false;
}

namespace {

int read_flags(bh_handle *h, cudaStream_t s) {
  BH_CUDA(cudaMemcpyAsync(h->hflags, h->flags, sizeof(DeviceFlags), cudaMemcpyDeviceToHost, s));
  BH_CUDA(cudaStreamSynchronize(s));
  return BH_OK;
}

// consume latched device error bits (report once)
int take_flag_error(bh_handle *h, cudaStream_t s) {
  int bits = h->hflags->bits;
  if (!bits) return BH_OK;
  long long bad = h->hflags->first_bad;
  // clear
  int zero = 0;
  long long big = 0x7fffffffffffffffll;
  cudaMemcpyAsync(&h->flags->bits, &zero, sizeof(int), cudaMemcpyHostToDevice, s);
  cudaMemcpyAsync(&h->flags->first_bad, &big, sizeof(long long), cudaMemcpyHostToDevice, s);
  cudaStreamSynchronize(s);
  h->hflags->bits = 0;
  if (bits & FLAG_OUT_OF_DOMAIN)
    return fail(BH_OUT_OF_DOMAIN, "position of body " + std::to_string(bad) +
                                      " outside domain [-R, R)");
  if (bits & FLAG_UNSORTED)
    return fail(BH_UNSORTED, "bodies must be sorted by spatial key for a hashed build");
  if (bits & FLAG_DUPLICATE)
    return fail(BH_DUPLICATE_KEY,
                "two bodies share the level-21 cell; positions are closer than the tree "
                "resolution");
  if (bits & FLAG_DEPTH) return fail(BH_DEPTH_OVERFLOW, "tree depth cap 21 exceeded");
  if (bits & FLAG_WALK_BOUNDS) return fail(BH_STACK_OVERFLOW, "walk frontier or list bound exceeded");
  return fail(BH_CUDA_ERROR, "unknown device flag");
}

int ensure_sort(bh_handle *h, int64_t n) {
  BH_CUDA(h->keys.ensure(sizeof(uint64_t) * (n + 1)));
  BH_CUDA(h->keys2.ensure(sizeof(uint64_t) * (n + 1)));
  BH_CUDA(h->vals.ensure(sizeof(uint32_t) * (n + 1)));
  BH_CUDA(h->vals2.ensure(sizeof(uint32_t) * (n + 1)));
  BH_CUDA(h->sort_tmp.ensure(sort_temp_bytes(n) + 16));
  return BH_OK;
}

int sort_keys(bh_handle *h, int64_t n, cudaStream_t s, bool iota_vals = false) {
  // keys/vals -> keys2/vals2 (iota_vals: the values are the input positions, not read)
  if (n <= 0) return BH_OK;
  BH_CUDA(sort_pairs(h->sort_tmp.p, h->sort_tmp.bytes, h->keys.as<uint64_t>(),
                     h->keys2.as<uint64_t>(), iota_vals ? nullptr : h->vals.as<uint32_t>(),
                     h->vals2.as<uint32_t>(), n, s));
  h->launches += sort_launches();
  return BH_OK;
}

// Build over Morton-sorted bodies whose keys are already in keys2
// (hashed.py:448-515).  Exactly one of bod32 / bod64 is non-null.
int build_sorted(bh_handle *h, int64_t n, const float4 *bod32, const double4 *bod64,
                 cudaStream_t s, int allow_dup = -1) {
  if (allow_dup < 0) allow_dup = h->allow_dup;
  BH_CUDA(h->lcp.ensure(n + 16));
  BH_CUDA(h->newc.ensure(sizeof(uint32_t) * (n + 1)));
  BH_CUDA(h->off.ensure(sizeof(uint32_t) * (n + 1)));
  BH_CUDA(h->scan_tmp.ensure(scan_temp_bytes(n) + 16));
  if (n > 0) {
    BH_CUDA(h->lvl.ensure(sizeof(int) * 4 * (kMaxLevel + 2)));
    launch_lcp_new(h->keys2.as<uint64_t>(), n, h->lcp.as<int8_t>(), h->newc.as<uint32_t>(),
                   h->flags, h->lvl.as<int>(), allow_dup, s, h->bnd_prev, h->bnd_next);
    BH_CUDA(exclusive_scan_u32(h->scan_tmp.p, h->scan_tmp.bytes, h->newc.as<uint32_t>(),
                               h->off.as<uint32_t>(), n, s));
    BH_LAUNCHED();
    BH_CUDA(cudaMemcpyAsync(h->hC, h->off.as<uint32_t>() + (n - 1), 4, cudaMemcpyDeviceToHost, s));
    BH_CUDA(cudaMemcpyAsync(h->hC + 1, h->newc.as<uint32_t>() + (n - 1), 4,
                            cudaMemcpyDeviceToHost, s));
    BH_CUDA(cudaMemcpyAsync(h->hlvl, h->lvl.p, sizeof(int) * (kMaxLevel + 1),
                            cudaMemcpyDeviceToHost, s));
  }
  BH_CUDA(cudaMemcpyAsync(h->hR, h->dR, sizeof(double), cudaMemcpyDeviceToHost, s));
  BH_TRY(read_flags(h, s));
  BH_TRY(take_flag_error(h, s));
  const int64_t C = n > 0 ? 1 + (int64_t)h->hC[0] + (int64_t)h->hC[1] : 1;
  if (C > 0x7fffffffll) return fail(BH_OUT_OF_MEMORY, "more than 2^31-1 cells");
  h->C = C;
  h->C_true = C;
  h->async_tree = false;
  h->mom_leaf = 0;
  h->tree_n = n;
  h->R = *h->hR;
  BH_CUDA(h->link.ensure(sizeof(int4) * C));
  BH_CUDA(h->parent.ensure(sizeof(int) * C));
  BH_CUDA(h->lvl_list.ensure(sizeof(int) * C));
  BH_CUDA(h->lvl.ensure(sizeof(int) * 4 * (kMaxLevel + 2)));
  BH_CUDA(h->child8.ensure(sizeof(int) * 8 * C));
  BH_CUDA(cudaMemsetAsync(h->child8.p, 0xFF, sizeof(int) * 8 * C, s));
  BH_CUDA(h->cm64.ensure(sizeof(double4) * C));
  BH_CUDA(h->q64.ensure(sizeof(double) * kQStride * C));
  h->walk_valid = false;
  if (n == 0) {  // hashed.py:459-462: an empty root
    int4 root = make_int4(1, 0, 0, 0);
    BH_CUDA(cudaMemcpyAsync(h->link.p, &root, sizeof(int4), cudaMemcpyHostToDevice, s));
    BH_CUDA(cudaMemsetAsync(h->cm64.p, 0, sizeof(double4), s));
    BH_CUDA(cudaMemsetAsync(h->q64.p, 0, sizeof(double) * 6, s));
    int m1 = -1;
    BH_CUDA(cudaMemcpyAsync(h->parent.p, &m1, sizeof(int), cudaMemcpyHostToDevice, s));
    BH_CUDA(cudaStreamSynchronize(s));
    h->max_level = 0;
    return BH_OK;
  }
  TreeView t = h->view();
  t.bod32 = bod32;
  t.bod64 = bod64;
  h->tbod32 = bod32;
  h->tbod64 = bod64;
  launch_emit(t, bod32, bod64, s);
  h->max_level = 0;
  for (int l = 0; l <= kMaxLevel; ++l)
    if (h->hlvl[l] > 0) h->max_level = l + 1;
  // one cooperative sweep over the device level counts (no launch per level)
  BH_CUDA((cudaError_t)launch_moments_coop(t, h->lvl.as<int>(), h->lvl_list.as<int>(), h->sms, s));
  BH_LAUNCHED();
  return BH_OK;
}

// Sync-free variant of build_sorted for the fp32 resident path: the cell
// count and the per-level counts stay on the device; buffers are sized to a
// capacity (2n, grown from the largest tree seen) and an overflow is flagged,
// detected at the end of the bh_sim_step call and repaired by re-running it.
int build_sorted_async(bh_handle *h, int64_t n, const float4 *bod32, cudaStream_t s,
                       int allow_dup, int leaf) {
  if (n <= 1) return build_sorted(h, n, bod32, nullptr, s, allow_dup);
  int64_t cap = std::max<int64_t>(h->cap, 2 * n + 1024);
  if (cap > 0x7fffffffll) cap = 0x7fffffffll;
  h->cap = cap;
  BH_CUDA(h->lcp.ensure(n + 16));
  BH_CUDA(h->newc.ensure(sizeof(uint32_t) * (n + 1)));
  BH_CUDA(h->off.ensure(sizeof(uint32_t) * (n + 1)));
  BH_CUDA(h->scan_tmp.ensure(scan_temp_bytes(n) + 16));
  BH_CUDA(h->lvl.ensure(sizeof(int) * 4 * (kMaxLevel + 2)));
  launch_lcp_new(h->keys2.as<uint64_t>(), n, h->lcp.as<int8_t>(), h->newc.as<uint32_t>(),
                 h->flags, h->lvl.as<int>(), allow_dup, s);
  BH_CUDA(exclusive_scan_u32(h->scan_tmp.p, h->scan_tmp.bytes, h->newc.as<uint32_t>(),
                             h->off.as<uint32_t>(), n, s));
  launch_set_count(h->off.as<uint32_t>(), h->newc.as<uint32_t>(), n, cap, h->dCtrue, h->flags, s, h->cur_step);
  BH_CUDA(h->link.ensure(sizeof(int4) * cap));
  BH_CUDA(h->parent.ensure(sizeof(int) * cap));
  BH_CUDA(h->lvl_list.ensure(sizeof(int) * cap));
  BH_CUDA(h->child8.ensure(sizeof(int) * 8 * cap));
  BH_CUDA(h->cm64.ensure(sizeof(double4) * cap));
  BH_CUDA(h->q64.ensure(sizeof(double) * kQStride * cap));
  // walk-only trees (leaf > 1): the two-pass emit sets the rows of the opened
  // cells itself; the other rows are never read
  // (not for a rank's local tree of the distributed build: k_mark_shared follows
  // child rows down the boundary paths, through buckets)
  const bool two_pass = leaf > 1 && leaf <= 64 && h->bnd_prev < 0 && h->bnd_next < 0;
  if (!two_pass) BH_CUDA(cudaMemsetAsync(h->child8.p, 0xFF, sizeof(int) * 8 * cap, s));
  h->C = cap;
  h->tree_n = n;
  h->async_tree = true;
  h->walk_valid = false;
  h->tbod32 = bod32;
  h->tbod64 = nullptr;
  h->mom_leaf = 0;  // (the class bytes of an earlier tree are stale)
  TreeView t = h->view();
  if (leaf > 1) {  // a walk-only tree: the emit kernel classifies the cells for the moments
    BH_CUDA(h->mclass.ensure(cap + 16));
    BH_CUDA(cudaMemsetAsync(h->mclass.p, 0, cap + 16, s));  // cells the emit skips: class 0
    t.mclass = h->mclass.as<uint8_t>();
    t.mleaf = leaf;
  }
  // (the creator list lives in lvl_list, which the moments kernels fill afterwards)
  if (!(two_pass && launch_emit_walk(t, bod32, h->lvl_list.as<int>(), h->lvl.as<int>() + 4 * (kMaxLevel + 1),
                                     h->sms, s))) {
    if (two_pass) BH_CUDA(cudaMemsetAsync(h->child8.p, 0xFF, sizeof(int) * 8 * cap, s));
    launch_emit(t, bod32, nullptr, s);
  }
  // a walk-only tree: moments of the cells a leaf-size-`leaf` walk reads
  BH_CUDA((cudaError_t)launch_moments_coop(t, h->lvl.as<int>(), h->lvl_list.as<int>(), h->sms, s, leaf));
  h->mom_leaf = leaf > 1 ? leaf : 0;
  h->launches += leaf > 1 ? 7 : 4;  // walk-only trees: two emit passes + the list and bucket-moment kernels
  BH_LAUNCHED();
  return BH_OK;
}

// Read back (one sync) what the sync-free builds of this call left on the
// device: the true cell count (stats, capacity growth), per-level counts
// (next call's grid sizes) and the flags.  Returns 1 on a capacity overflow.
int async_readback(bh_handle *h, cudaStream_t s, int *overflow) {
  *overflow = 0;
  if (!h->async_tree) return BH_OK;
  BH_CUDA(cudaMemcpyAsync(h->hstat, h->dCtrue, sizeof(int), cudaMemcpyDeviceToHost, s));
  BH_CUDA(cudaMemcpyAsync(h->hstat + 1, h->lvl.p, sizeof(int) * (kMaxLevel + 1),
                          cudaMemcpyDeviceToHost, s));
  BH_TRY(read_flags(h, s));
  if (h->hflags->bits & FLAG_OVERFLOW) {
    *overflow = 1;
    int keep = h->hflags->bits & ~FLAG_OVERFLOW;
    BH_CUDA(cudaMemcpyAsync(&h->flags->bits, &keep, sizeof(int), cudaMemcpyHostToDevice, s));
    BH_CUDA(cudaStreamSynchronize(s));
    h->hflags->bits = keep;
    h->cap = std::min<int64_t>(0x7fffffffll, h->hstat[0] + h->hstat[0] / 4 + 1024);
    return BH_OK;
  }
  BH_TRY(take_flag_error(h, s));
  h->C_true = h->hstat[0];
  h->max_level = 0;
  for (int l = 0; l <= kMaxLevel; ++l) {
    const int cnt = h->hstat[1 + l];
    h->grid_lvl[l] = cnt > 0 ? grid_for(cnt + cnt / 4 + 64, 128) : 1;
    if (cnt > 0) h->max_level = l + 1;
  }
  return BH_OK;
}

void fill_walk_params(bh_handle *h, WalkParams &P, int64_t nt, double theta, double eps,
                      int leaf) {
  P.C = (int)h->C;
  P.nt = (int)nt;
  P.e2 = eps * eps;
  P.e2f = (float)(eps * eps);
  P.theta = theta;
  P.leaf = leaf;
  for (int l = 0; l <= kMaxLevel; ++l) {
    double side = std::ldexp(2.0 * h->R, -l);
    P.side64[l] = side;
    double r = side / theta;  // theta == 0 -> inf: never accept
    P.mac2f[l] = (float)(r * r);
  }
}

// (Re)build the compact fp32 walk tree for (theta, leaf) -- bh_walk.cu
int ensure_walk_tree(bh_handle *h, double theta, int leaf, cudaStream_t s) {
  if (leaf < 1) leaf = 1;
  if (h->mom_leaf > 0 && h->mom_leaf != leaf)  // a walk-only tree holds what one leaf size reads
    return fail(BH_BAD_ARG, "the resident tree was built for walks with leaf size " +
                                std::to_string(h->mom_leaf) + "; prepare again for leaf size " +
                                std::to_string(leaf));
  if (h->walk_valid && h->walk_theta == theta && h->walk_leaf == leaf) return BH_OK;
  const int64_t C = h->C;
  BH_CUDA(h->smask.ensure(sizeof(uint32_t) * C));
  BH_CUDA(h->nck.ensure(sizeof(uint32_t) * C));
  BH_CUDA(h->wbase.ensure(sizeof(uint32_t) * C));
  BH_CUDA(h->wnodes.ensure(sizeof(WalkNode) * C));
  BH_CUDA(h->wscan_tmp.ensure(scan_temp_bytes(C) + 16));
  TreeView t = h->view();
  launch_walk_tree(t, h->dR, theta, leaf, h->smask.as<uint32_t>(), h->nck.as<uint32_t>(),
                   h->wbase.as<uint32_t>(), h->wscan_tmp.p, h->wscan_tmp.bytes,
                   h->wnodes.as<WalkNode>(), h->dCp, s);
  h->launches += h->mom_leaf > 1 && h->mom_leaf == leaf ? 6 : 5;  // walk-only: list count, 3 scan, bases, records
  BH_LAUNCHED();
  h->walk_valid = true;
  h->walk_theta = theta;
  h->walk_leaf = leaf;
  return BH_OK;
}

// An upper bound on the walk records of the current tree (the walk's record
// indices must fit the v9 frontier word's 28 bits): the records are a subset
// of the cells; a sync-free build knows its cell count only from the last
// readback, so the bound then takes the last count with growth slack.
int64_t walk_records_bound(bh_handle *h) {
  const int64_t alloc = (int64_t)(h->wnodes.bytes / sizeof(WalkNode));
  if (!h->async_tree) return std::min<int64_t>(alloc, h->C);
  return h->C_true > 0 ? std::min<int64_t>(alloc, h->C_true + h->C_true / 4 + 1024) : alloc;
}

int reset_counters(bh_handle *h, cudaStream_t s) {
  BH_CUDA(cudaMemsetAsync(&h->flags->pp, 0, 2 * sizeof(unsigned long long), s));
  return BH_OK;
}

__global__ void k_scatter_work(const int *ws, const uint32_t *id, int64_t n, int *wo) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) wo[id[i]] = ws[i];
}

template <class T4>
__global__ void k_store4(const T4 *src, const uint32_t *id, int64_t n, T4 *dst) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) dst[id[i]] = src[i];
}
__global__ void k_store3(const double4 *src, const uint32_t *id, int64_t n, double *dst) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double4 v = src[i];
  int64_t j = id[i];
  dst[3 * j] = v.x; dst[3 * j + 1] = v.y; dst[3 * j + 2] = v.z;
}
__global__ void k_work64(const int *w, int64_t n, int64_t *out) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = w[i];
}
__global__ void k_iota32(uint32_t *v, int64_t n) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) v[i] = (uint32_t)i;
}
__global__ void k_fill_int(int *v, int64_t n, int x) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) v[i] = x;
}

// simulation.py:370-396 (algorithm 1, one rank) on resident state, split into
// phases so a multi-GPU driver can exchange between them:
//   prepare: bounds -> keys -> stable sort -> permute bodies -> build -> walk tree
//   walk   : targets [begin, end) of the Morton-sorted bodies
int flush_work(bh_handle *h, cudaStream_t s);
int sim_prepare(bh_handle *h, double theta, double eps, int leaf, bool bounds_ready,
                cudaStream_t s) {
  BH_TRY(flush_work(h, s));
  const int64_t n = h->sim_n;
  const bool f32 = h->precision == BH_FP32;
  if (!(theta >= 0.0) || !(eps >= 0.0)) return fail(BH_BAD_ARG, "theta and eps must be >= 0");
  if (!bounds_ready) {
    h->tbegin(BH_PHASE_INTEGRATE, s);
    launch_reset_flags_bounds(h->flags, s);
    if (f32) launch_maxabs_f32(h->pos.as<float4>(), n, h->flags, s);
    else launch_kick_drift_max_f64(h->pos.as<double4>(), h->vel.as<double4>(), nullptr, n, 0.0,
                                   0.0, h->flags, s);
    h->tend(s);
    h->launches += 2;
  }
  BH_TRY(ensure_sort(h, n));
  h->tbegin(BH_PHASE_KEYS, s);
  launch_finish_R(h->flags, f32 ? 0 : 1, h->dR, s);
  if (f32)
    launch_keys_f32(h->pos.as<float4>(), n, h->dR, h->keys.as<uint64_t>(), nullptr, h->flags, s);
  else
    launch_keys_f64(h->pos.as<double>(), 4, n, h->dR, h->keys.as<uint64_t>(), nullptr, h->flags, s);
  h->tend(s);
  h->tbegin(BH_PHASE_SORT, s);
  BH_TRY(sort_keys(h, n, s, true));
  h->tend(s);
  h->tbegin(BH_PHASE_PERMUTE, s);
  if (f32)
    launch_gather_f32(h->vals2.as<uint32_t>(), n, h->pos.as<float4>(), h->pos2.as<float4>(),
                      h->vel.as<float4>(), h->vel2.as<float4>(), h->id.as<uint32_t>(),
                      h->id2.as<uint32_t>(), s);
  else
    launch_gather_f64(h->vals2.as<uint32_t>(), n, h->pos.as<double4>(), h->pos2.as<double4>(),
                      h->vel.as<double4>(), h->vel2.as<double4>(), h->id.as<uint32_t>(),
                      h->id2.as<uint32_t>(), s);
  std::swap(h->pos, h->pos2);
  std::swap(h->vel, h->vel2);
  std::swap(h->id, h->id2);
  h->tend(s);
  BH_LAUNCHED();
  h->tbegin(BH_PHASE_BUILD, s);
  if (f32)
    BH_TRY(build_sorted_async(h, n, h->pos.as<float4>(), s, h->allow_dup || leaf > 1, leaf));
  else
    BH_TRY(build_sorted(h, n, nullptr, h->pos.as<double4>(), s, h->allow_dup || leaf > 1));
  h->tend(s);
  if (f32) {  // the walk records are part of the build (the walk phase is the traversal alone)
    h->tbegin(BH_PHASE_BUILD, s);
    BH_TRY(ensure_walk_tree(h, theta, leaf, s));
    h->tend(s);
  }
  h->launches += 6;  // finish_R, keys, gather, lcp_new, emit, level scatter (+ per-level)
  return BH_OK;
}

// keys (with the R already in dR), stable sort, permutation -- no build
int sim_sort(bh_handle *h, cudaStream_t s) {
  BH_TRY(flush_work(h, s));
  const int64_t n = h->sim_n;
  const bool f32 = h->precision == BH_FP32;
  BH_TRY(ensure_sort(h, n));
  if (n == 0) return BH_OK;
  h->tbegin(BH_PHASE_KEYS, s);
  if (f32)
    launch_keys_f32(h->pos.as<float4>(), n, h->dR, h->keys.as<uint64_t>(), nullptr, h->flags, s);
  else
    launch_keys_f64(h->pos.as<double>(), 4, n, h->dR, h->keys.as<uint64_t>(), nullptr, h->flags, s);
  h->tend(s);
  h->tbegin(BH_PHASE_SORT, s);
  BH_TRY(sort_keys(h, n, s, true));
  h->tend(s);
  h->tbegin(BH_PHASE_PERMUTE, s);
  if (f32)
    launch_gather_f32(h->vals2.as<uint32_t>(), n, h->pos.as<float4>(), h->pos2.as<float4>(),
                      h->vel.as<float4>(), h->vel2.as<float4>(), h->id.as<uint32_t>(),
                      h->id2.as<uint32_t>(), s);
  else
    launch_gather_f64(h->vals2.as<uint32_t>(), n, h->pos.as<double4>(), h->pos2.as<double4>(),
                      h->vel.as<double4>(), h->vel2.as<double4>(), h->id.as<uint32_t>(),
                      h->id2.as<uint32_t>(), s);
  std::swap(h->pos, h->pos2);
  std::swap(h->vel, h->vel2);
  std::swap(h->id, h->id2);
  // acc follows its body too (a migrated state's kick needs it)
  if (f32) {
    launch_gather_f32(h->vals2.as<uint32_t>(), n, h->acc.as<float4>(), h->pos2.as<float4>(),
                      nullptr, nullptr, nullptr, nullptr, s);
    BH_CUDA(cudaMemcpyAsync(h->acc.p, h->pos2.p, sizeof(float4) * n, cudaMemcpyDeviceToDevice, s));
  } else {
    launch_gather_f64(h->vals2.as<uint32_t>(), n, h->acc.as<double4>(), h->pos2.as<double4>(),
                      nullptr, nullptr, nullptr, nullptr, s);
    BH_CUDA(cudaMemcpyAsync(h->acc.p, h->pos2.p, sizeof(double4) * n, cudaMemcpyDeviceToDevice, s));
  }
  h->launches += 4;
  BH_LAUNCHED();
  h->tend(s);
  return BH_OK;
}

int sim_walk(bh_handle *h, double theta, double eps, int leaf, int64_t begin, int64_t end,
             int record_work, cudaStream_t s) {
  const int64_t n = h->sim_n;
  const bool f32 = h->precision == BH_FP32;
  if (begin < 0 || end > n || begin > end) return fail(BH_BAD_ARG, "walk range outside [0, n]");
  const int64_t nt = end - begin;
  if (h->npeers && (h->acc.p != h->peer_own_acc || h->work_sorted.p != h->peer_own_work))
    return fail(BH_BAD_ARG, "result buffers reallocated since the peers mapped them: set peers again");
  BH_TRY(reset_counters(h, s));
  if (f32) {  // (normally already built by sim_prepare)
    h->tbegin(BH_PHASE_BUILD, s);
    BH_TRY(ensure_walk_tree(h, theta, leaf, s));
    h->tend(s);
  }
  h->tbegin(BH_PHASE_WALK, s);
  int *w32 = record_work ? h->work_sorted.as<int>() + begin : nullptr;
  W9Peers peers;  // the same rows of every peer's buffers (replicated ranks)
  peers.n = h->npeers;
  const size_t row = f32 ? sizeof(float4) : sizeof(double4);
  for (int r = 0; r < h->npeers; ++r) {
    peers.acc[r] = reinterpret_cast<float *>(static_cast<char *>(h->peer_acc[r]) + row * begin);
    peers.work[r] = static_cast<int *>(h->peer_work[r]) + begin;
  }
  // warps of Hilbert-ordered targets (bh_walk.cu): tighter target groups, same
  // per-target interaction sets and (fp64) the same per-target summation order
  const uint32_t *perm = nullptr;
  if (walk_hilbert_enabled() && nt > 64) {
    BH_CUDA(h->hperm.ensure(sizeof(uint32_t) * (nt + 1)));
    launch_hilbert_chunks(h->keys2.as<uint64_t>() + begin, nt, h->hperm.as<uint32_t>(), s);  // the tree's keys
    perm = h->hperm.as<uint32_t>();
    h->launches += 1;
  }
  if (f32) {
    launch_walk_f32(h->wnodes.as<WalkNode>(), walk_records_bound(h), h->pos.as<float4>(),
                    h->pos.as<float>() + 4 * begin, 4, perm, (int)nt, (float)(eps * eps), leaf,
                    h->acc.as<float>() + 4 * begin, 4, nullptr, w32, h->flags, s, h->npeers ? &peers : nullptr);
  } else {
    WalkParams P;
    fill_walk_params(h, P, nt, theta, eps, leaf);
    launch_walk_f64(P, h->cm64.as<double4>(), h->q64.as<double>(), h->link.as<int4>(),
                    h->pos.as<double4>(), h->pos.as<double>() + 4 * begin, 4, perm,
                    h->acc.as<double>() + 4 * begin, 4, nullptr, w32, h->flags, s);
    if (h->npeers) launch_peer_scatter(h->acc.as<double>() + 4 * begin, row, w32, nt, peers, s);
  }
  h->tend(s);
  h->launches += 1;
  BH_LAUNCHED();
  return BH_OK;
}

int sim_scatter_work(bh_handle *h, cudaStream_t s) {
  const int64_t n = h->sim_n;
  h->work_dirty = false;
  if (n <= 0) return BH_OK;
  k_scatter_work<<<grid_for(n, 256), 256, 0, s>>>(h->work_sorted.as<int>(), h->id.as<uint32_t>(), n,
                                                  h->work_orig.as<int>());
  h->launches += 1;
  BH_LAUNCHED();
  return BH_OK;
}

int sim_forces_impl(bh_handle *h, double theta, double eps, int leaf, int record_work,
                    bool bounds_ready, cudaStream_t s) {
  BH_TRY(sim_prepare(h, theta, eps, leaf, bounds_ready, s));
  BH_TRY(sim_walk(h, theta, eps, leaf, 0, h->sim_n, record_work, s));
  if (record_work) h->work_dirty = true;  // scattered when read (flush_work)
  return BH_OK;
}

// the pending work scatter must run before the permutation changes or a read
int flush_work(bh_handle *h, cudaStream_t s) {
  if (!h->work_dirty) return BH_OK;
  if (h->drop_work) {  // a multi-step call: the next walk records work again
    h->work_dirty = false;
    return BH_OK;
  }
  return sim_scatter_work(h, s);
}

int sim_begin_step(bh_handle *h, double dt, cudaStream_t s) {
  const int64_t n = h->sim_n;
  const double half = 0.5 * dt;  // simulation.py:494: kick(0.5*dt), drift(dt)
  h->tbegin(BH_PHASE_INTEGRATE, s);
  launch_reset_flags_bounds(h->flags, s);
  if (h->precision == BH_FP32)
    launch_kick_drift_max_f32(h->pos.as<float4>(), h->vel.as<float4>(), h->acc.as<float4>(), n,
                              (float)half, (float)dt, h->flags, s);
  else
    launch_kick_drift_max_f64(h->pos.as<double4>(), h->vel.as<double4>(), h->acc.as<double4>(),
                              n, half, dt, h->flags, s);
  h->tend(s);
  h->launches += 2;
  BH_LAUNCHED();
  return BH_OK;
}

int sim_end_step(bh_handle *h, double dt, cudaStream_t s) {
  const int64_t n = h->sim_n;
  const double half = 0.5 * dt;  // simulation.py:500: kick(0.5*dt)
  h->tbegin(BH_PHASE_INTEGRATE, s);
  if (h->precision == BH_FP32)  // skipped on the device if this call's build overflowed
    launch_kick_f32(h->vel.as<float4>(), h->acc.as<float4>(), n, (float)half, s, h->flags);
  else launch_kick4_f64(h->vel.as<double4>(), h->acc.as<double4>(), n, half, s);
  h->tend(s);
  h->launches += 1;
  BH_LAUNCHED();
  return BH_OK;
}

}  // namespace

// ============================================================== C-ABI
extern "C" {

const char *bh_last_error(void) { return g_err.c_str(); }
int bh_version(void) { return 1; }

int bh_create(bh_handle **out, int device, int precision) {
  if (!out) return fail(BH_BAD_ARG, "out is NULL");
  if (precision != BH_FP32 && precision != BH_FP64) return fail(BH_BAD_ARG, "bad precision");
  BH_CUDA(cudaSetDevice(device));
  bh_handle *h = new bh_handle();
  h->device = device;
  h->precision = precision;
  cudaDeviceGetAttribute(&h->sms, cudaDevAttrMultiProcessorCount, device);
  BH_CUDA(cudaMalloc(&h->flags, sizeof(DeviceFlags)));
  BH_CUDA(cudaMallocHost(&h->hflags, sizeof(DeviceFlags)));
  BH_CUDA(cudaMallocHost(&h->hC, 4 * sizeof(uint32_t)));
  BH_CUDA(cudaMalloc(&h->dR, sizeof(double)));
  BH_CUDA(cudaMalloc(&h->dCp, sizeof(int)));
  BH_CUDA(cudaMalloc(&h->dCtrue, sizeof(int)));
  BH_CUDA(cudaMallocHost(&h->hstat, sizeof(int) * (kMaxLevel + 4)));
  BH_CUDA(cudaMallocHost(&h->hR, sizeof(double)));
  BH_CUDA(cudaMallocHost(&h->hlvl, sizeof(int) * (kMaxLevel + 2)));
  BH_CUDA(cudaMallocHost(&h->hlet, sizeof(uint32_t) * 4 * 32));
  DeviceFlags init;
  memset(&init, 0, sizeof(init));
  init.first_bad = 0x7fffffffffffffffll;
  BH_CUDA(cudaMemcpy(h->flags, &init, sizeof(init), cudaMemcpyHostToDevice));
  *h->hflags = init;
  *out = h;
  return BH_OK;
}

int bh_destroy(bh_handle *h) {
  if (!h) return BH_OK;
  cudaSetDevice(h->device);
  close_peers(h);
  Buf *bufs[] = {&h->keys, &h->keys2, &h->vals, &h->vals2, &h->sort_tmp, &h->scan_tmp,
                 &h->lcp, &h->newc, &h->off, &h->link, &h->parent, &h->child8, &h->lvl, &h->lvl_list, &h->hperm,
                 &h->cm64, &h->q64, &h->mclass, &h->smask, &h->nck, &h->wbase, &h->wnodes, &h->wscan_tmp, &h->tbod, &h->pos, &h->pos2,
                 &h->vel, &h->vel2, &h->acc, &h->id, &h->id2, &h->work_sorted, &h->work_orig,
                 &h->bk_pos, &h->bk_vel, &h->bk_acc, &h->bk_id, &h->bk_work,
                 &h->shared, &h->branch, &h->rec_of_cell, &h->wparent, &h->let_present,
                 &h->let_expand, &h->let_bodies, &h->let_isbranch, &h->let_rflag, &h->let_bcount,
                 &h->let_rpos, &h->let_bpos, &h->let_scan_tmp, &h->let_brec, &h->let_tail, &h->let_boxkey, &h->let_lvl, &h->let_list, &h->hs_a, &h->hs_b, &h->hs_pos};
  for (Buf *b : bufs) b->release();
  cudaFree(h->flags);
  cudaFreeHost(h->hflags);
  cudaFreeHost(h->hC);
  cudaFree(h->dR);
  cudaFree(h->dCp);
  cudaFree(h->dCtrue);
  cudaFreeHost(h->hstat);
  cudaFreeHost(h->hR);
  cudaFreeHost(h->hlvl);
  cudaFreeHost(h->hlet);
  if (h->ev_pos) cudaEventDestroy(h->ev_pos);
  if (h->ev_side) cudaEventDestroy(h->ev_side);
  if (h->side) cudaStreamDestroy(h->side);
  for (cudaStream_t c : h->cp)
    if (c) cudaStreamDestroy(c);
  for (cudaEvent_t e : h->ev_cp)
    if (e) cudaEventDestroy(e);
  h->fold_marks();
  for (cudaEvent_t e : h->pool) cudaEventDestroy(e);
  delete h;
  return BH_OK;
}

int bh_check(bh_handle *h, void *stream) {
  if (!h) return fail(BH_BAD_ARG, "handle is NULL");
  BH_CUDA(cudaGetLastError());
  int overflow = 0;
  BH_TRY(async_readback(h, S(stream), &overflow));
  if (overflow)
    return fail(BH_OUT_OF_MEMORY,
                "tree cell capacity exceeded during a phased step; capacity grown, redo the step");
  BH_TRY(read_flags(h, S(stream)));
  return take_flag_error(h, S(stream));
}

int bh_bounds_f32(bh_handle *h, const float *d_pos4, int64_t n, double *d_R, void *stream) {
  if (!h || n < 0 || (n && !d_pos4) || !d_R) return fail(BH_BAD_ARG, "bh_bounds_f32: bad args");
  launch_reset_flags_bounds(h->flags, S(stream));
  launch_maxabs_f32(reinterpret_cast<const float4 *>(d_pos4), n, h->flags, S(stream));
  launch_finish_R(h->flags, 0, d_R, S(stream));
  BH_LAUNCHED();
  return BH_OK;
}

int bh_bounds_f64(bh_handle *h, const double *d_pos3, int64_t n, double *d_R, void *stream) {
  if (!h || n < 0 || (n && !d_pos3) || !d_R) return fail(BH_BAD_ARG, "bh_bounds_f64: bad args");
  launch_reset_flags_bounds(h->flags, S(stream));
  launch_maxabs_f64(d_pos3, n, h->flags, S(stream));
  launch_finish_R(h->flags, 1, d_R, S(stream));
  BH_LAUNCHED();
  return BH_OK;
}

int bh_morton_f32(bh_handle *h, const float *d_pos4, int64_t n, const double *d_R,
                  uint64_t *d_keys, void *stream) {
  if (!h || n < 0 || !d_R || (n && (!d_pos4 || !d_keys))) return fail(BH_BAD_ARG, "bh_morton_f32: bad args");
  launch_keys_f32(reinterpret_cast<const float4 *>(d_pos4), n, d_R, d_keys, nullptr, h->flags,
                  S(stream));
  BH_LAUNCHED();
  return BH_OK;
}

int bh_morton_f64(bh_handle *h, const double *d_pos3, int64_t n, const double *d_R,
                  uint64_t *d_keys, void *stream) {
  if (!h || n < 0 || !d_R || (n && (!d_pos3 || !d_keys))) return fail(BH_BAD_ARG, "bh_morton_f64: bad args");
  launch_keys_f64(d_pos3, 3, n, d_R, d_keys, nullptr, h->flags, S(stream));
  BH_LAUNCHED();
  return BH_OK;
}

int bh_sort(bh_handle *h, const uint64_t *d_keys, int64_t n, uint64_t *d_keys_sorted,
            int64_t *d_perm, void *stream) {
  if (!h || n < 0 || (n && (!d_keys || !d_perm))) return fail(BH_BAD_ARG, "bh_sort: bad args");
  if (n == 0) return BH_OK;
  cudaStream_t s = S(stream);
  BH_TRY(ensure_sort(h, n));
  BH_CUDA(cudaMemcpyAsync(h->keys.p, d_keys, sizeof(uint64_t) * n, cudaMemcpyDeviceToDevice, s));
  k_iota32<<<grid_for(n, 256), 256, 0, s>>>(h->vals.as<uint32_t>(), n);
  BH_TRY(sort_keys(h, n, s));
  if (d_keys_sorted)
    BH_CUDA(cudaMemcpyAsync(d_keys_sorted, h->keys2.p, sizeof(uint64_t) * n,
                            cudaMemcpyDeviceToDevice, s));
  launch_iota64(d_perm, h->vals2.as<uint32_t>(), n, s);
  BH_LAUNCHED();
  return BH_OK;
}

int bh_scan_u32(bh_handle *h, const uint32_t *d_in, int64_t n, uint32_t *d_out, int inclusive, void *stream) {
  if (!h || n < 0 || (n && (!d_in || !d_out))) return fail(BH_BAD_ARG, "bh_scan_u32: bad args");
  if (n == 0) return BH_OK;
  BH_CUDA(h->scan_tmp.ensure(scan_temp_bytes(n) + 16));
  if (inclusive) BH_CUDA(inclusive_scan_u32(h->scan_tmp.p, h->scan_tmp.bytes, d_in, d_out, n, S(stream)));
  else BH_CUDA(exclusive_scan_u32(h->scan_tmp.p, h->scan_tmp.bytes, d_in, d_out, n, S(stream)));
  h->launches += 1;
  return BH_OK;
}

int bh_build_f32(bh_handle *h, const float *d_pos4_sorted, int64_t n, const double *d_R,
                 void *stream) {
  if (!h || n < 0 || !d_R || (n && !d_pos4_sorted)) return fail(BH_BAD_ARG, "bh_build_f32: bad args");
  if (h->precision != BH_FP32) return fail(BH_BAD_ARG, "handle is fp64; use bh_build_f64");
  cudaStream_t s = S(stream);
  BH_TRY(ensure_sort(h, n));
  BH_CUDA(h->tbod.ensure(sizeof(float4) * (n + 1)));
  if (n) BH_CUDA(cudaMemcpyAsync(h->tbod.p, d_pos4_sorted, sizeof(float4) * n,
                                 cudaMemcpyDeviceToDevice, s));
  BH_CUDA(cudaMemcpyAsync(h->dR, d_R, sizeof(double), cudaMemcpyDeviceToDevice, s));
  // hashed.py:463: keys recomputed from the (sorted) positions
  launch_keys_f32(h->tbod.as<float4>(), n, h->dR, h->keys2.as<uint64_t>(), nullptr, h->flags, s);
  return build_sorted(h, n, h->tbod.as<float4>(), nullptr, s);
}

int bh_build_f64(bh_handle *h, const double *d_pos3_sorted, const double *d_mass_sorted,
                 int64_t n, const double *d_R, void *stream) {
  if (!h || n < 0 || !d_R || (n && (!d_pos3_sorted || !d_mass_sorted)))
    return fail(BH_BAD_ARG, "bh_build_f64: bad args");
  if (h->precision != BH_FP64) return fail(BH_BAD_ARG, "handle is fp32; use bh_build_f32");
  cudaStream_t s = S(stream);
  BH_TRY(ensure_sort(h, n));
  BH_CUDA(h->tbod.ensure(sizeof(double4) * (n + 1)));
  launch_pack_bodies_f64(d_pos3_sorted, d_mass_sorted, n, h->tbod.as<double4>(), s);
  BH_CUDA(cudaMemcpyAsync(h->dR, d_R, sizeof(double), cudaMemcpyDeviceToDevice, s));
  launch_keys_f64(d_pos3_sorted, 3, n, h->dR, h->keys2.as<uint64_t>(), nullptr, h->flags, s);
  return build_sorted(h, n, nullptr, h->tbod.as<double4>(), s);
}

int bh_set_allow_duplicates(bh_handle *h, int allow) {
  if (!h) return fail(BH_BAD_ARG, "bh_set_allow_duplicates: bad args");
  h->allow_dup = allow != 0;
  return BH_OK;
}

int bh_tree_size(bh_handle *h, int64_t *n_cells) {
  if (!h || !n_cells) return fail(BH_BAD_ARG, "bh_tree_size: bad args");
  if (h->tree_n < 0) return fail(BH_NO_TREE, "no tree has been built");
  if (h->async_tree) {
    int overflow = 0;
    BH_TRY(async_readback(h, nullptr, &overflow));
    if (overflow) return fail(BH_OUT_OF_MEMORY, "tree cell capacity exceeded");
  }
  *n_cells = h->async_tree ? h->C_true : h->C;
  return BH_OK;
}

__global__ void k_tree_fits(const int *dC, int64_t cap, int32_t *out) { out[0] = *dC <= cap ? 1 : 0; }

int bh_sim_tree_fits_dev(bh_handle *h, int32_t *d_out, void *stream) {
  if (!h || !d_out) return fail(BH_BAD_ARG, "bh_sim_tree_fits_dev: bad args");
  if (h->tree_n < 0) return fail(BH_NO_TREE, "no tree has been built");
  cudaStream_t s = S(stream);
  if (!h->async_tree) {
    const int32_t one = 1;
    BH_CUDA(cudaMemcpyAsync(d_out, &one, sizeof(one), cudaMemcpyHostToDevice, s));
    BH_CUDA(cudaStreamSynchronize(s));  // (the host source is on the stack)
    return BH_OK;
  }
  k_tree_fits<<<1, 1, 0, s>>>(h->dCtrue, h->C, d_out);
  h->launches += 1;
  BH_LAUNCHED();
  return BH_OK;
}

int bh_export_tree(bh_handle *h, uint64_t *d_key, int8_t *d_level, double *d_centre,
                   double *d_side, double *d_mass, double *d_com, double *d_quad,
                   int64_t *d_count, int32_t *d_children, void *stream) {
  if (!h) return fail(BH_BAD_ARG, "bh_export_tree: bad args");
  if (h->tree_n < 0) return fail(BH_NO_TREE, "no tree has been built");
  if (h->mom_leaf > 0)
    return fail(BH_BAD_ARG, "the resident tree is a walk-only tree (cells inside buckets have no moments); "
                            "build it with bh_build_* to export");
  launch_export(h->view(), h->R, d_key, d_level, d_centre, d_side, d_mass, d_com, d_quad, d_count,
                d_children, S(stream));
  BH_LAUNCHED();
  return BH_OK;
}

static int traverse_common(bh_handle *h, const void *targets, int64_t n, double theta,
                           double eps, int leaf, void *acc, int64_t *work, bool f32,
                           cudaStream_t s) {
  if (h->tree_n < 0) return fail(BH_NO_TREE, "no tree has been built");
  if (!(theta >= 0.0) || !(eps >= 0.0)) return fail(BH_BAD_ARG, "theta and eps must be >= 0");
  if (n > 0x7fffffffll) return fail(BH_BAD_ARG, "too many targets");
  if (n == 0) return BH_OK;
  const int comps = f32 ? 4 : 3;
  const size_t esz = f32 ? sizeof(float) : sizeof(double);
  BH_TRY(reset_counters(h, s));
  if (h->tree_n == 0) {  // flattree.py:152: empty tree -> zero acc, zero work
    BH_CUDA(cudaMemsetAsync(acc, 0, esz * comps * n, s));
    if (work) BH_CUDA(cudaMemsetAsync(work, 0, sizeof(int64_t) * n, s));
    return BH_OK;
  }
  // order the targets along the Morton curve so warps walk coherent lists
  BH_TRY(ensure_sort(h, n));
  if (f32)
    launch_keys_clamped_f32(static_cast<const float *>(targets), 4, n, h->dR,
                            h->keys.as<uint64_t>(), h->vals.as<uint32_t>(), s);
  else
    launch_keys_clamped_f64(static_cast<const double *>(targets), 3, n, h->dR,
                            h->keys.as<uint64_t>(), h->vals.as<uint32_t>(), s);
  // keys2 holds the tree's keys (needed by export): sort into keys (tmp) instead
  BH_CUDA(h->work_sorted.ensure(sizeof(uint64_t) * (n + 1)));
  BH_CUDA(sort_pairs(h->sort_tmp.p, h->sort_tmp.bytes, h->keys.as<uint64_t>(),
                     h->work_sorted.as<uint64_t>(), h->vals.as<uint32_t>(),
                     h->vals2.as<uint32_t>(), n, s));
  WalkParams P;
  fill_walk_params(h, P, n, theta, eps, leaf);
  if (f32) {
    BH_TRY(ensure_walk_tree(h, theta, leaf, s));
    launch_walk_f32(h->wnodes.as<WalkNode>(), walk_records_bound(h), h->tbod.as<float4>(),
                    static_cast<const float *>(targets), 4, h->vals2.as<uint32_t>(), (int)n,
                    (float)(eps * eps), leaf, static_cast<float *>(acc), 4, work, nullptr,
                    h->flags, s);
  } else
    launch_walk_f64(P, h->cm64.as<double4>(), h->q64.as<double>(), h->link.as<int4>(),
                    h->tbod.as<double4>(), static_cast<const double *>(targets), 3,
                    h->vals2.as<uint32_t>(), static_cast<double *>(acc), 3, work, nullptr,
                    h->flags, s);
  BH_LAUNCHED();
  return BH_OK;
}

int bh_traverse_f32(bh_handle *h, const float *d_targets4, int64_t n, double theta, double eps,
                    int leaf_size, float *d_acc4, int64_t *d_work, void *stream) {
  if (!h || n < 0 || (n && (!d_targets4 || !d_acc4))) return fail(BH_BAD_ARG, "bh_traverse_f32: bad args");
  if (h->precision != BH_FP32) return fail(BH_BAD_ARG, "handle is fp64; use bh_traverse_f64");
  return traverse_common(h, d_targets4, n, theta, eps, leaf_size, d_acc4, d_work, true, S(stream));
}

int bh_traverse_f64(bh_handle *h, const double *d_targets3, int64_t n, double theta,
                    double eps, int leaf_size, double *d_acc3, int64_t *d_work, void *stream) {
  if (!h || n < 0 || (n && (!d_targets3 || !d_acc3))) return fail(BH_BAD_ARG, "bh_traverse_f64: bad args");
  if (h->precision != BH_FP64) return fail(BH_BAD_ARG, "handle is fp32; use bh_traverse_f32");
  return traverse_common(h, d_targets3, n, theta, eps, leaf_size, d_acc3, d_work, false, S(stream));
}

int bh_kick_f32(bh_handle *h, float *d_vel4, const float *d_acc4, int64_t n, double dt, void *stream) {
  if (!h || n < 0) return fail(BH_BAD_ARG, "bh_kick_f32: bad args");
  launch_kick_f32(reinterpret_cast<float4 *>(d_vel4), reinterpret_cast<const float4 *>(d_acc4), n,
                  (float)dt, S(stream));
  BH_LAUNCHED();
  return BH_OK;
}
int bh_drift_f32(bh_handle *h, float *d_pos4, const float *d_vel4, int64_t n, double dt, void *stream) {
  if (!h || n < 0) return fail(BH_BAD_ARG, "bh_drift_f32: bad args");
  launch_drift_f32(reinterpret_cast<float4 *>(d_pos4), reinterpret_cast<const float4 *>(d_vel4), n,
                   (float)dt, S(stream));
  BH_LAUNCHED();
  return BH_OK;
}
int bh_kick_f64(bh_handle *h, double *d_vel3, const double *d_acc3, int64_t n, double dt, void *stream) {
  if (!h || n < 0) return fail(BH_BAD_ARG, "bh_kick_f64: bad args");
  launch_kick_f64(d_vel3, d_acc3, n, dt, S(stream));
  BH_LAUNCHED();
  return BH_OK;
}
int bh_drift_f64(bh_handle *h, double *d_pos3, const double *d_vel3, int64_t n, double dt, void *stream) {
  if (!h || n < 0) return fail(BH_BAD_ARG, "bh_drift_f64: bad args");
  launch_drift_f64(d_pos3, d_vel3, n, dt, S(stream));
  BH_LAUNCHED();
  return BH_OK;
}

int bh_direct_f64(bh_handle *h, const double *d_pos3, const double *d_mass, int64_t n, double eps,
                  double *d_acc3, void *stream) {
  if (!h || n < 0) return fail(BH_BAD_ARG, "bh_direct_f64: bad args");
  launch_direct_f64(d_pos3, d_mass, n, eps, d_acc3, S(stream));
  BH_LAUNCHED();
  return BH_OK;
}
int bh_potential_f64(bh_handle *h, const double *d_pos3, const double *d_mass, int64_t n,
                     double eps, double *d_partial, void *stream) {
  if (!h || n < 0) return fail(BH_BAD_ARG, "bh_potential_f64: bad args");
  launch_potential_f64(d_pos3, d_mass, n, eps, d_partial, S(stream));
  BH_LAUNCHED();
  return BH_OK;
}

__global__ void k_pack_vel_f64(const double *v3, int64_t n, double4 *out) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = make_double4(v3[3 * i], v3[3 * i + 1], v3[3 * i + 2], 0.0);
}

int bh_sim_load(bh_handle *h, const void *d_pos, const void *d_vel, const double *d_mass,
                const void *d_acc, int64_t n, void *stream) {
  if (!h || n < 0 || (n && (!d_pos || !d_vel))) return fail(BH_BAD_ARG, "bh_sim_load: bad args");
  if (n > 0x7fffffffll) return fail(BH_BAD_ARG, "too many bodies");
  const bool f32 = h->precision == BH_FP32;
  if (!f32 && n && !d_mass) return fail(BH_BAD_ARG, "fp64 bh_sim_load needs masses");
  cudaStream_t s = S(stream);
  const size_t e4 = f32 ? sizeof(float4) : sizeof(double4);
  Buf *b4[] = {&h->pos, &h->pos2, &h->vel, &h->vel2, &h->acc};
  for (Buf *b : b4) BH_CUDA(b->ensure(e4 * (n + 1)));
  BH_CUDA(h->id.ensure(sizeof(uint32_t) * (n + 1)));
  BH_CUDA(h->id2.ensure(sizeof(uint32_t) * (n + 1)));
  BH_CUDA(h->work_sorted.ensure(sizeof(int64_t) * (n + 1)));
  BH_CUDA(h->work_orig.ensure(sizeof(int) * (n + 1)));
  h->sim_n = n;
  h->work_dirty = false;
  if (n == 0) return BH_OK;
  if (f32) {
    BH_CUDA(cudaMemcpyAsync(h->pos.p, d_pos, e4 * n, cudaMemcpyDeviceToDevice, s));
    BH_CUDA(cudaMemcpyAsync(h->vel.p, d_vel, e4 * n, cudaMemcpyDeviceToDevice, s));
  } else {
    launch_pack_bodies_f64(static_cast<const double *>(d_pos), d_mass, n, h->pos.as<double4>(), s);
    k_pack_vel_f64<<<grid_for(n, 256), 256, 0, s>>>(static_cast<const double *>(d_vel), n,
                                                    h->vel.as<double4>());
  }
  if (!d_acc) {
    BH_CUDA(cudaMemsetAsync(h->acc.p, 0, e4 * n, s));
  } else if (f32) {
    BH_CUDA(cudaMemcpyAsync(h->acc.p, d_acc, e4 * n, cudaMemcpyDeviceToDevice, s));
  } else {
    k_pack_vel_f64<<<grid_for(n, 256), 256, 0, s>>>(static_cast<const double *>(d_acc), n,
                                                    h->acc.as<double4>());
  }
  k_iota32<<<grid_for(n, 256), 256, 0, s>>>(h->id.as<uint32_t>(), n);
  k_fill_int<<<grid_for(n, 256), 256, 0, s>>>(h->work_orig.as<int>(), n, 1);  // simulation.py:482
  BH_LAUNCHED();
  return BH_OK;
}

int bh_sim_forces(bh_handle *h, double theta, double eps, int leaf_size, int record_work,
                  void *stream) {
  if (!h) return fail(BH_BAD_ARG, "bh_sim_forces: bad args");
  if (h->sim_n == 0) return BH_OK;
  for (int attempt = 0; attempt < 3; ++attempt) {  // forces only permute: safe to redo
    BH_TRY(sim_forces_impl(h, theta, eps, leaf_size, record_work, false, S(stream)));
    int overflow = 0;
    BH_TRY(async_readback(h, S(stream), &overflow));
    if (!overflow) return BH_OK;
  }
  return fail(BH_OUT_OF_MEMORY, "tree cell capacity kept overflowing");
}

// `steps` KDK steps (simulation.py:492-502) with no state snapshot.  A
// sync-free build that overflows its capacity flags the device; every later
// kernel of the call that reads the tree or moves the state skips (the walk
// sees an empty tree, the kicks return), so the state is exactly what the
// failed step's kick+drift left.  The call then grows the capacity and resumes
// at that step's force evaluation.
static int sim_steps(bh_handle *h, double dt, double theta, double eps, int leaf_size, int steps,
                     cudaStream_t s, bool *pos_hook_done, void (*pos_hook)(bh_handle *, cudaStream_t)) {
  int k = 0;
  bool resume = false;
  for (int attempt = 0; attempt < 4; ++attempt) {
    for (; k < steps; ++k) {
      h->cur_step = k;
      if (!resume) {
        BH_TRY(sim_begin_step(h, dt, s));
        if (pos_hook && !*pos_hook_done) {
          pos_hook(h, s);
          *pos_hook_done = true;
        }
      }
      BH_TRY(sim_forces_impl(h, theta, eps, leaf_size, 1, !resume, s));
      resume = false;
      BH_TRY(sim_end_step(h, dt, s));
    }
    int overflow = 0;
    BH_TRY(async_readback(h, s, &overflow));
    if (!overflow) return BH_OK;
    k = std::max(0, std::min(steps - 1, h->hflags->ovf_step));  // capacity grown: redo that step's forces
    resume = true;
  }
  return fail(BH_OUT_OF_MEMORY, "tree cell capacity kept overflowing");
}

int bh_sim_step(bh_handle *h, double dt, double theta, double eps, int leaf_size, int steps,
                void *stream) {
  if (!h || !(dt > 0.0) || steps < 0) return fail(BH_BAD_ARG, "bh_sim_step: bad args");
  if (h->sim_n == 0 || steps == 0) return BH_OK;
  cudaStream_t s = S(stream);
  struct DropWork {  // inside the call every walk records work: only the last one is kept
    bh_handle *h;
    explicit DropWork(bh_handle *hh) : h(hh) { h->drop_work = true; }
    ~DropWork() { h->drop_work = false; }
  } drop(h);
  bool unused = false;
  return sim_steps(h, dt, theta, eps, leaf_size, steps, s, &unused, nullptr);
}

__global__ void k_expand3(const float *__restrict__ v3, int64_t n, float4 *__restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = make_float4(v3[3 * i], v3[3 * i + 1], v3[3 * i + 2], 0.f);
}
__global__ void k_store3f(const float4 *__restrict__ src, const uint32_t *__restrict__ id, int64_t n,
                          float *__restrict__ dst3) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const float4 v = src[i];
  float *o = dst3 + 3 * (int64_t)id[i];
  o[0] = v.x; o[1] = v.y; o[2] = v.z;
}

// One call from host arrays (the reference's numpy Bodies, fp32): load
// pos4 (x, y, z, m) / vel3 / acc3, run `steps` KDK steps, write the state back
// in the caller's order, and (work != NULL) the last walk's per-body work
// pp + 2 pc (simulation.py:394-395).  For one step the positions are final
// after the drift, so their device->host copy runs on a side stream under the
// tree build and walk; velocities, accelerations and work follow the final
// kick.  Host arrays should be pinned for the copies to be asynchronous.
static void early_pos_copy(bh_handle *h, cudaStream_t s) {
  const int64_t n = h->sim_n;
  cudaMemcpyAsync(h->hs_pos.p, h->pos.p, sizeof(float4) * n, cudaMemcpyDeviceToDevice, s);
  cudaEventRecord(h->ev_pos, s);
  cudaStreamWaitEvent(h->side, h->ev_pos, 0);
  cudaMemcpyAsync(h->host_pos4, h->hs_pos.p, sizeof(float4) * n, cudaMemcpyDeviceToHost, h->side);
  cudaEventRecord(h->ev_side, h->side);
}

int bh_sim_step_host(bh_handle *h, float *pos4, float *vel3, float *acc3, int32_t *work, int64_t n, double dt,
                     double theta, double eps, int leaf_size, int steps, void *stream) {
  if (!h || n < 1 || !pos4 || !vel3 || !acc3 || !(dt > 0.0) || steps < 1)
    return fail(BH_BAD_ARG, "bh_sim_step_host: bad args");
  if (h->precision != BH_FP32) return fail(BH_BAD_ARG, "bh_sim_step_host: fp32 handles");
  cudaStream_t s = S(stream);
  if (!h->side) BH_CUDA(cudaStreamCreateWithFlags(&h->side, cudaStreamNonBlocking));
  if (!h->ev_pos) BH_CUDA(cudaEventCreateWithFlags(&h->ev_pos, cudaEventDisableTiming));
  if (!h->ev_side) BH_CUDA(cudaEventCreateWithFlags(&h->ev_side, cudaEventDisableTiming));
  for (cudaStream_t &c : h->cp)
    if (!c) BH_CUDA(cudaStreamCreateWithFlags(&c, cudaStreamNonBlocking));
  for (cudaEvent_t &e : h->ev_cp)
    if (!e) BH_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  BH_CUDA(h->hs_a.ensure(sizeof(float) * 3 * n));
  BH_CUDA(h->hs_b.ensure(sizeof(float) * 3 * n));
  BH_CUDA(h->hs_pos.ensure(sizeof(float4) * n));
  // load: positions straight into the resident buffer, 3-vectors through staging
  {
    Buf *b4[] = {&h->pos, &h->pos2, &h->vel, &h->vel2, &h->acc};
    for (Buf *b : b4) BH_CUDA(b->ensure(sizeof(float4) * (n + 1)));
    BH_CUDA(h->id.ensure(sizeof(uint32_t) * (n + 1)));
    BH_CUDA(h->id2.ensure(sizeof(uint32_t) * (n + 1)));
    BH_CUDA(h->work_sorted.ensure(sizeof(int64_t) * (n + 1)));
    BH_CUDA(h->work_orig.ensure(sizeof(int) * (n + 1)));
  }
  h->sim_n = n;
  // the three input copies run concurrently (PCIe reads overlap: 48 -> 53 GB/s)
  BH_CUDA(cudaEventRecord(h->ev_cp[0], s));
  BH_CUDA(cudaStreamWaitEvent(h->cp[0], h->ev_cp[0], 0));
  BH_CUDA(cudaStreamWaitEvent(h->cp[1], h->ev_cp[0], 0));
  BH_CUDA(cudaMemcpyAsync(h->pos.p, pos4, sizeof(float4) * n, cudaMemcpyHostToDevice, s));
  BH_CUDA(cudaMemcpyAsync(h->hs_a.p, vel3, sizeof(float) * 3 * n, cudaMemcpyHostToDevice, h->cp[0]));
  BH_CUDA(cudaMemcpyAsync(h->hs_b.p, acc3, sizeof(float) * 3 * n, cudaMemcpyHostToDevice, h->cp[1]));
  BH_CUDA(cudaEventRecord(h->ev_cp[1], h->cp[0]));
  BH_CUDA(cudaEventRecord(h->ev_cp[2], h->cp[1]));
  BH_CUDA(cudaStreamWaitEvent(s, h->ev_cp[1], 0));
  BH_CUDA(cudaStreamWaitEvent(s, h->ev_cp[2], 0));
  const int g = grid_for(n, 256);
  k_expand3<<<g, 256, 0, s>>>(h->hs_a.as<float>(), n, h->vel.as<float4>());
  k_expand3<<<g, 256, 0, s>>>(h->hs_b.as<float>(), n, h->acc.as<float4>());
  k_iota32<<<g, 256, 0, s>>>(h->id.as<uint32_t>(), n);
  k_fill_int<<<g, 256, 0, s>>>(h->work_orig.as<int>(), n, 1);  // simulation.py:482
  h->launches += 4;
  h->work_dirty = false;  // freshly loaded: work_orig = 1
  bool pos_sent = false;
  h->host_pos4 = pos4;
  {
    struct DropWork {
      bh_handle *h;
      explicit DropWork(bh_handle *hh) : h(hh) { h->drop_work = true; }
      ~DropWork() { h->drop_work = false; }
    } drop(h);
    BH_TRY(sim_steps(h, dt, theta, eps, leaf_size, steps, s, &pos_sent, steps == 1 ? early_pos_copy : nullptr));
  }
  const uint32_t *id = h->id.as<uint32_t>();
  if (!pos_sent) {
    k_store4<float4><<<g, 256, 0, s>>>(h->pos.as<float4>(), id, n, h->hs_pos.as<float4>());
    BH_CUDA(cudaMemcpyAsync(pos4, h->hs_pos.p, sizeof(float4) * n, cudaMemcpyDeviceToHost, s));
  }
  k_store3f<<<g, 256, 0, s>>>(h->vel.as<float4>(), id, n, h->hs_a.as<float>());
  BH_CUDA(cudaEventRecord(h->ev_cp[1], s));
  k_store3f<<<g, 256, 0, s>>>(h->acc.as<float4>(), id, n, h->hs_b.as<float>());
  // vel goes back while acc is being gathered; the two copies overlap
  BH_CUDA(cudaStreamWaitEvent(h->cp[0], h->ev_cp[1], 0));
  BH_CUDA(cudaMemcpyAsync(vel3, h->hs_a.p, sizeof(float) * 3 * n, cudaMemcpyDeviceToHost, h->cp[0]));
  BH_CUDA(cudaEventRecord(h->ev_cp[2], h->cp[0]));
  BH_CUDA(cudaMemcpyAsync(acc3, h->hs_b.p, sizeof(float) * 3 * n, cudaMemcpyDeviceToHost, s));
  if (work) {  // the last walk's work, scattered to the caller's order (int32)
    BH_TRY(sim_scatter_work(h, s));
    BH_CUDA(cudaMemcpyAsync(work, h->work_orig.p, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, s));
  }
  BH_CUDA(cudaStreamWaitEvent(s, h->ev_cp[2], 0));
  if (pos_sent) BH_CUDA(cudaStreamWaitEvent(s, h->ev_side, 0));
  h->launches += 2 + (pos_sent ? 0 : 1);
  BH_LAUNCHED();
  return BH_OK;
}

int bh_sim_begin_step(bh_handle *h, double dt, void *stream) {
  if (!h || !(dt > 0.0)) return fail(BH_BAD_ARG, "bh_sim_begin_step: bad args");
  if (h->sim_n == 0) return BH_OK;
  return sim_begin_step(h, dt, S(stream));
}

int bh_sim_prepare(bh_handle *h, double theta, double eps, int leaf_size, int bounds_ready,
                   void *stream) {
  if (!h) return fail(BH_BAD_ARG, "bh_sim_prepare: bad args");
  if (h->sim_n == 0) return BH_OK;
  return sim_prepare(h, theta, eps, leaf_size, bounds_ready != 0, S(stream));
}

int bh_sim_walk_range(bh_handle *h, double theta, double eps, int leaf_size, int64_t begin,
                      int64_t end, int record_work, void *stream) {
  if (!h) return fail(BH_BAD_ARG, "bh_sim_walk_range: bad args");
  if (h->sim_n == 0) return BH_OK;
  return sim_walk(h, theta, eps, leaf_size, begin, end, record_work, S(stream));
}

int bh_sim_ipc_handles(bh_handle *h, void *out128) {
  if (!h || !out128 || !h->acc.p || !h->work_sorted.p) return fail(BH_BAD_ARG, "bh_sim_ipc_handles: no state");
  cudaIpcMemHandle_t a, w;
  BH_CUDA(cudaIpcGetMemHandle(&a, h->acc.p));
  BH_CUDA(cudaIpcGetMemHandle(&w, h->work_sorted.p));
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "ipc handle size");
  memcpy(out128, &a, 64);
  memcpy(static_cast<char *>(out128) + 64, &w, 64);
  return BH_OK;
}

int bh_sim_set_peers(bh_handle *h, int npeers, const void *handles) {
  if (!h || npeers < 0 || npeers > kMaxPeers || (npeers && !handles))
    return fail(BH_BAD_ARG, "bh_sim_set_peers: bad args (at most 7 peers)");
  BH_CUDA(cudaSetDevice(h->device));
  close_peers(h);
  for (int r = 0; r < npeers; ++r) {
    cudaIpcMemHandle_t a, w;
    memcpy(&a, static_cast<const char *>(handles) + 128 * r, 64);
    memcpy(&w, static_cast<const char *>(handles) + 128 * r + 64, 64);
    void *pa = nullptr, *pw = nullptr;
    cudaError_t e = cudaIpcOpenMemHandle(&pa, a, cudaIpcMemLazyEnablePeerAccess);
    if (e == cudaSuccess) e = cudaIpcOpenMemHandle(&pw, w, cudaIpcMemLazyEnablePeerAccess);
    h->peer_acc[r] = pa;
    h->peer_work[r] = pw;
    h->npeers = r + 1;
    h->peer_ipc = true;
    h->peer_own_acc = h->acc.p;
    h->peer_own_work = h->work_sorted.p;
    if (e != cudaSuccess) {
      close_peers(h);
      return fail(BH_CUDA_ERROR, std::string("bh_sim_set_peers: ") + cudaGetErrorString(e));
    }
  }
  return BH_OK;
}

int bh_sim_set_peer_ptrs(bh_handle *h, int npeers, void *const *acc, void *const *work) {
  if (!h || npeers < 0 || npeers > kMaxPeers || (npeers && (!acc || !work)))
    return fail(BH_BAD_ARG, "bh_sim_set_peer_ptrs: bad args (at most 7 peers)");
  close_peers(h);
  for (int r = 0; r < npeers; ++r) {
    h->peer_acc[r] = acc[r];
    h->peer_work[r] = work[r];
  }
  h->npeers = npeers;
  h->peer_own_acc = h->acc.p;
  h->peer_own_work = h->work_sorted.p;
  return BH_OK;
}

int bh_sim_result_ptrs(bh_handle *h, void **acc, void **work) {
  if (!h || !acc || !work) return fail(BH_BAD_ARG, "bh_sim_result_ptrs: bad args");
  *acc = h->acc.p;
  *work = h->work_sorted.p;
  return BH_OK;
}

int bh_sim_scatter_work(bh_handle *h, void *stream) {
  if (!h) return fail(BH_BAD_ARG, "bh_sim_scatter_work: bad args");
  return sim_scatter_work(h, S(stream));
}

int bh_sim_end_step(bh_handle *h, double dt, void *stream) {
  if (!h || !(dt > 0.0)) return fail(BH_BAD_ARG, "bh_sim_end_step: bad args");
  if (h->sim_n == 0) return BH_OK;
  return sim_end_step(h, dt, S(stream));
}

__global__ void k_gather_work(const int *wo, const uint32_t *id, int64_t b, int64_t e, int *dst) {
  int64_t i = b + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < e) dst[i - b] = wo[id[i]];
}

// ------------------------------------------------ distributed build entry points
int bh_sim_local_maxabs(bh_handle *h, double *out, void *stream) {
  if (!h || !out) return fail(BH_BAD_ARG, "bh_sim_local_maxabs: bad args");
  BH_TRY(read_flags(h, S(stream)));
  union { unsigned u; float f; } v;
  v.u = h->hflags->maxabs_bits;
  *out = h->precision == BH_FP32 ? (double)v.f : h->hflags->maxabs64;
  return BH_OK;
}

int bh_sim_set_R(bh_handle *h, double R, void *stream) {
  if (!h || !(R > 0.0)) return fail(BH_BAD_ARG, "bh_sim_set_R: bad args");
  *h->hR = R;
  BH_CUDA(cudaMemcpyAsync(h->dR, h->hR, sizeof(double), cudaMemcpyHostToDevice, S(stream)));
  BH_CUDA(cudaStreamSynchronize(S(stream)));
  return BH_OK;
}

int bh_sim_sort(bh_handle *h, void *stream) {
  if (!h) return fail(BH_BAD_ARG, "bh_sim_sort: bad args");
  return sim_sort(h, S(stream));
}

// Morton keys of the current bodies in their current order (no sort) with the
// R already set -- the routing keys of the distributed step's migration.
int bh_sim_keys(bh_handle *h, uint64_t *d_keys, void *stream) {
  if (!h || (!d_keys && h->sim_n)) return fail(BH_BAD_ARG, "bh_sim_keys: bad args");
  const int64_t n = h->sim_n;
  if (n == 0) return BH_OK;
  cudaStream_t s = S(stream);
  BH_TRY(ensure_sort(h, n));
  h->tbegin(BH_PHASE_KEYS, s);
  if (h->precision == BH_FP32)
    launch_keys_f32(h->pos.as<float4>(), n, h->dR, h->keys.as<uint64_t>(), h->vals.as<uint32_t>(),
                    h->flags, s);
  else
    launch_keys_f64(h->pos.as<double>(), 4, n, h->dR, h->keys.as<uint64_t>(),
                    h->vals.as<uint32_t>(), h->flags, s);
  h->tend(s);
  BH_CUDA(cudaMemcpyAsync(d_keys, h->keys.p, sizeof(uint64_t) * n, cudaMemcpyDeviceToDevice, s));
  h->launches += 1;
  BH_LAUNCHED();
  return BH_OK;
}

int bh_sim_load_state(bh_handle *h, const void *d_pos, const void *d_vel, const void *d_acc,
                      const int32_t *d_work, int64_t n, void *stream) {
  BH_TRY(bh_sim_load(h, d_pos, d_vel, nullptr, d_acc, n, stream));
  if (n > 0 && d_work)
    BH_CUDA(cudaMemcpyAsync(h->work_orig.p, d_work, sizeof(int) * n, cudaMemcpyDeviceToDevice,
                            S(stream)));
  return BH_OK;
}

// Build this rank's tree over its (sorted) key range, with leaf depths made
// global by the neighbour ranks' boundary keys; mark the shared cells; build the
// walk tree (shared cells always expanded, so every branch node has a record);
// return the number of branch nodes.  fp32 handles.  Synchronises.
int bh_sim_build_local(bh_handle *h, double theta, int leaf_size, int has_prev, uint64_t prev_key,
                       int has_next, uint64_t next_key, int64_t *nbranch, void *stream) {
  if (!h || !nbranch) return fail(BH_BAD_ARG, "bh_sim_build_local: bad args");
  if (h->precision != BH_FP32) return fail(BH_BAD_ARG, "distributed build is fp32");
  cudaStream_t s = S(stream);
  const int64_t n = h->sim_n;
  if (n == 0) { *nbranch = 0; return BH_OK; }
  uint64_t kfirst = 0, klast = 0;
  BH_CUDA(cudaMemcpyAsync(&kfirst, h->keys2.p, 8, cudaMemcpyDeviceToHost, s));
  BH_CUDA(cudaMemcpyAsync(&klast, h->keys2.as<uint64_t>() + (n - 1), 8, cudaMemcpyDeviceToHost, s));
  BH_CUDA(cudaStreamSynchronize(s));
  auto lcp_host = [](uint64_t a, uint64_t b) {
    uint64_t x = a ^ b;
    int bits = x ? 64 - __builtin_clzll(x) : 0;
    return kMortonBits - (bits + 2) / 3;
  };
  h->bnd_prev = has_prev ? lcp_host(prev_key, kfirst) : -1;
  h->bnd_next = has_next ? lcp_host(klast, next_key) : -1;
  const int allow_dup = h->allow_dup || leaf_size > 1;
  h->tbegin(BH_PHASE_BUILD, s);
  int rc = build_sorted(h, n, h->pos.as<float4>(), nullptr, s, allow_dup);
  if (rc != BH_OK) { h->bnd_prev = h->bnd_next = -1; return rc; }
  const int64_t C = h->C;
  BH_CUDA(h->shared.ensure(C + 16));
  BH_CUDA(h->branch.ensure(sizeof(int) * (8 * (2 * kMaxLevel + 2) + 8)));
  BH_CUDA(h->rec_of_cell.ensure(sizeof(int) * C));
  BH_CUDA(h->wparent.ensure(sizeof(int) * C));
  TreeView t = h->view();
  launch_mark_shared(t, h->shared.as<uint8_t>(), h->branch.as<int>() + 1, h->branch.as<int>(), s);
  BH_CUDA(h->smask.ensure(sizeof(uint32_t) * C));
  BH_CUDA(h->nck.ensure(sizeof(uint32_t) * C));
  BH_CUDA(h->wbase.ensure(sizeof(uint32_t) * C));
  BH_CUDA(h->wnodes.ensure(sizeof(WalkNode) * C));
  BH_CUDA(h->wscan_tmp.ensure(scan_temp_bytes(C) + 16));
  launch_walk_tree(t, h->dR, theta, leaf_size, h->smask.as<uint32_t>(), h->nck.as<uint32_t>(),
                   h->wbase.as<uint32_t>(), h->wscan_tmp.p, h->wscan_tmp.bytes,
                   h->wnodes.as<WalkNode>(), h->dCp, s, h->shared.as<uint8_t>(),
                   h->rec_of_cell.as<int>(), h->wparent.as<int>());
  h->walk_valid = false;  // a forced-shared walk tree is not the local-walk tree
  int nb = 0;
  BH_CUDA(cudaMemcpyAsync(&nb, h->branch.p, sizeof(int), cudaMemcpyDeviceToHost, s));
  h->tend(s);
  BH_CUDA(cudaStreamSynchronize(s));
  BH_LAUNCHED();
  h->nbranch = nb;
  *nbranch = nb;
  h->bnd_prev = h->bnd_next = -1;
  return BH_OK;
}

int bh_sim_branch_export(bh_handle *h, uint64_t *d_key, int32_t *d_level, int64_t *d_count,
                         double *d_mom10, int32_t *d_rec, int32_t *d_lo, void *stream) {
  if (!h) return fail(BH_BAD_ARG, "bh_sim_branch_export: bad args");
  TreeView t = h->view();
  launch_branch_export(t, h->branch.as<int>() + 1, (int)h->nbranch, h->rec_of_cell.as<int>(), d_key,
                       d_level, d_count, d_mom10, d_rec, d_lo, S(stream));
  BH_LAUNCHED();
  return BH_OK;
}

__global__ void k_mark_branch_recs(const int *branch, int nb, const int *rec_of_cell,
                                   uint8_t *isbranch, int *brec) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= nb) return;
  const int j = rec_of_cell[branch[k]];
  isbranch[j] = 1;
  brec[k] = j;
}

// Locally essential trees of this rank's last bh_sim_build_local for every
// other rank: d_boxes = [nrank][nbox][6] (min xyz, max xyz)
// covering each rank's bodies (empty boxes: min > max).  Fills rec_counts / body_counts (host, [nrank]) with the LET
// sizes for each receiver (0 for self).  Synchronises.
int bh_sim_let(bh_handle *h, const double *d_boxes, int nbox, int nrank, int self,
               int64_t *rec_counts, int64_t *body_counts, void *stream) {
  if (!h || !d_boxes || nbox < 1 || nrank < 1 || nrank > 32 || self < 0 || self >= nrank ||
      !rec_counts || !body_counts)
    return fail(BH_BAD_ARG, "bh_sim_let: bad args");
  cudaStream_t s = S(stream);
  int cp = 0;
  BH_CUDA(cudaMemcpyAsync(&cp, h->dCp, sizeof(int), cudaMemcpyDeviceToHost, s));
  BH_CUDA(cudaStreamSynchronize(s));
  const int64_t n = cp;
  h->let_nrank = nrank;
  h->let_nrec = n;
  for (int q = 0; q < nrank; ++q) rec_counts[q] = body_counts[q] = 0;
  if (n == 0 || h->sim_n == 0) return BH_OK;
  Buf *u32s[] = {&h->let_present, &h->let_expand, &h->let_bodies};
  for (Buf *b : u32s) BH_CUDA(b->ensure(sizeof(uint32_t) * (n + 1)));
  const int64_t nn = n * nrank;  // [receiver][record]
  BH_CUDA(h->let_rflag.ensure(sizeof(uint32_t) * (nn + 1)));
  BH_CUDA(h->let_bcount.ensure(sizeof(uint32_t) * (nn + 1)));
  BH_CUDA(h->let_rpos.ensure(sizeof(uint32_t) * (nn + 1)));  // inclusive scans
  BH_CUDA(h->let_bpos.ensure(sizeof(uint32_t) * (nn + 1)));
  BH_CUDA(h->let_isbranch.ensure(n + 16));
  BH_CUDA(h->let_brec.ensure(sizeof(int) * (h->nbranch + 1)));
  BH_CUDA(h->let_scan_tmp.ensure(inclusive_scan_temp_bytes(nn) + 16));
  BH_CUDA(h->let_tail.ensure(sizeof(uint32_t) * 2 * nrank));
  h->tbegin(BH_PHASE_LET, s);
  BH_CUDA(cudaMemsetAsync(h->let_isbranch.p, 0, n, s));
  if (h->nbranch > 0)
    k_mark_branch_recs<<<grid_for(h->nbranch, 128), 128, 0, s>>>(
        h->branch.as<int>() + 1, (int)h->nbranch, h->rec_of_cell.as<int>(), h->let_isbranch.as<uint8_t>(),
        h->let_brec.as<int>());
  const WalkNode *W = h->wnodes.as<WalkNode>();
  BH_CUDA(h->let_lvl.ensure(sizeof(int) * 3 * (kMaxLevel + 1)));
  BH_CUDA(h->let_list.ensure(sizeof(int) * (n + 1)));
  launch_let_mark(W, (int)n, h->wparent.as<int>(), h->let_isbranch.as<uint8_t>(), d_boxes, nbox, nrank, self,
                  h->let_lvl.as<int>(), h->let_list.as<int>(), h->sms, h->let_present.as<uint32_t>(),
                  h->let_expand.as<uint32_t>(), h->let_bodies.as<uint32_t>(), s);
  BH_CUDA(cudaGetLastError());
  launch_let_flags_all(W, (int)n, h->let_isbranch.as<uint8_t>(), h->let_present.as<uint32_t>(),
                       h->let_bodies.as<uint32_t>(), nrank, self, h->let_rflag.as<uint32_t>(),
                       h->let_bcount.as<uint32_t>(), s);
  BH_CUDA(inclusive_scan_u32(h->let_scan_tmp.p, h->let_scan_tmp.bytes, h->let_rflag.as<uint32_t>(),
                             h->let_rpos.as<uint32_t>(), nn, s));
  BH_CUDA(inclusive_scan_u32(h->let_scan_tmp.p, h->let_scan_tmp.bytes, h->let_bcount.as<uint32_t>(),
                             h->let_bpos.as<uint32_t>(), nn, s));
  launch_let_tails(h->let_rpos.as<uint32_t>(), h->let_bpos.as<uint32_t>(), (int)n, nrank,
                   h->let_tail.as<uint32_t>(), s);
  h->tend(s);
  BH_CUDA(cudaMemcpyAsync(h->hlet, h->let_tail.p, sizeof(uint32_t) * 2 * nrank, cudaMemcpyDeviceToHost, s));
  BH_CUDA(cudaStreamSynchronize(s));
  for (int q = 0; q < nrank; ++q) {
    if (q == self) continue;
    rec_counts[q] = h->hlet[2 * q];
    body_counts[q] = h->hlet[2 * q + 1];
  }
  h->launches += 8;
  BH_LAUNCHED();
  return BH_OK;
}

// Pack the LET for receiver q (sizes from bh_sim_let): records [rec_counts[q]]
// (WalkNode), bodies [body_counts[q]] (float4) and, per branch node of this
// rank, (first child in the LET | -1, first body in the LET | -1).
int bh_sim_let_pack(bh_handle *h, int q, void *d_rec_out, float *d_bodies_out, int32_t *d_bmap_out,
                    void *stream) {
  if (!h || q < 0 || q >= h->let_nrank) return fail(BH_BAD_ARG, "bh_sim_let_pack: bad args");
  cudaStream_t s = S(stream);
  const int64_t n = h->let_nrec;
  if (n == 0) return BH_OK;
  const WalkNode *W = h->wnodes.as<WalkNode>();
  h->tbegin(BH_PHASE_LET, s);
  launch_let_pack(W, (int)n, h->let_expand.as<uint32_t>(), h->let_bodies.as<uint32_t>(), q,
                  h->let_rflag.as<uint32_t>(), h->let_rpos.as<uint32_t>(), h->let_bcount.as<uint32_t>(),
                  h->let_bpos.as<uint32_t>(), h->pos.as<float4>(), static_cast<WalkNode *>(d_rec_out),
                  reinterpret_cast<float4 *>(d_bodies_out), s);
  launch_let_branchmap(W, h->let_brec.as<int>(), (int)h->nbranch, (int)n, h->let_expand.as<uint32_t>(),
                       h->let_bodies.as<uint32_t>(), q, h->let_rflag.as<uint32_t>(), h->let_rpos.as<uint32_t>(),
                       h->let_bcount.as<uint32_t>(), h->let_bpos.as<uint32_t>(),
                       reinterpret_cast<int2 *>(d_bmap_out), s);
  h->tend(s);
  h->launches += 2;
  BH_LAUNCHED();
  return BH_OK;
}

// Bounding box of each contiguous range of the sorted bodies: out[1 + g] for
// bodies [start[g], start[g+1]) (empty range: min = +inf, max = -inf), and
// out[0] = their union.  Float min/max through order-preserving int keys so a
// range of any length is reduced by the whole grid: one warp reduction and 6
// atomics per warp when the warp's bodies share a range (the common case).
__device__ __forceinline__ int ord_key(float f) {
  const int i = __float_as_int(f);
  return i >= 0 ? i : i ^ 0x7fffffff;
}
__device__ __forceinline__ float ord_val(int k) { return __int_as_float(k >= 0 ? k : k ^ 0x7fffffff); }

__global__ void k_box_init(int *__restrict__ key, int ngroup) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < 6 * ngroup) key[t] = (t % 6) < 3 ? INT_MAX : INT_MIN;
}

// Each warp reduces a contiguous chunk of bodies; per-lane running min/max are
// flushed (warp reduction, then shared-memory atomics) whenever the warp's
// range changes, and each block flushes its shared boxes to global at the end.
__device__ __forceinline__ void box_flush(int g, float (&mn)[3], float (&mx)[3], int *sk) {
  for (int a = 0; a < 3; ++a)
    for (int o = 16; o > 0; o >>= 1) {
      mn[a] = fminf(mn[a], __shfl_xor_sync(0xffffffffu, mn[a], o));
      mx[a] = fmaxf(mx[a], __shfl_xor_sync(0xffffffffu, mx[a], o));
    }
  if ((threadIdx.x & 31) == 0 && g >= 0)
    for (int a = 0; a < 3; ++a) {
      atomicMin(&sk[6 * g + a], ord_key(mn[a]));
      atomicMax(&sk[6 * g + 3 + a], ord_key(mx[a]));
    }
  for (int a = 0; a < 3; ++a) { mn[a] = INFINITY; mx[a] = -INFINITY; }
}

__global__ void k_range_boxes(const float4 *__restrict__ pos, int64_t n, const int64_t *__restrict__ start,
                              int ngroup, int64_t chunk, int *__restrict__ key) {
  __shared__ int64_t st[257];
  __shared__ int sk[6 * 256];
  for (int g = threadIdx.x; g <= ngroup; g += blockDim.x) st[g] = start[g];
  for (int t = threadIdx.x; t < 6 * ngroup; t += blockDim.x) sk[t] = (t % 6) < 3 ? INT_MAX : INT_MIN;
  __syncthreads();
  const unsigned lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t b = warp * chunk, e = b + chunk < n ? b + chunk : n;
  float mn[3] = {INFINITY, INFINITY, INFINITY}, mx[3] = {-INFINITY, -INFINITY, -INFINITY};
  int gcur = -1;
  for (int64_t base = b; base < e; base += 32) {
    const int64_t i = base + lane;
    const bool v = i < e;
    // range of the warp's first body; the whole warp handles one range per pass
    int g0 = 0;
    {
      int lo = 0, hi = ngroup - 1;  // last g with st[g] <= base
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (st[mid] <= base) lo = mid; else hi = mid - 1;
      }
      g0 = lo;
    }
    if (g0 != gcur) {
      box_flush(gcur, mn, mx, sk);
      gcur = g0;
    }
    if (v) {
      const float4 p = pos[i];
      if (i < st[g0 + 1]) {
        mn[0] = fminf(mn[0], p.x); mn[1] = fminf(mn[1], p.y); mn[2] = fminf(mn[2], p.z);
        mx[0] = fmaxf(mx[0], p.x); mx[1] = fmaxf(mx[1], p.y); mx[2] = fmaxf(mx[2], p.z);
      } else {  // the warp straddles a range boundary: later ranges go straight to shared
        int lo = g0, hi = ngroup - 1;
        while (lo < hi) {
          const int mid = (lo + hi + 1) >> 1;
          if (st[mid] <= i) lo = mid; else hi = mid - 1;
        }
        atomicMin(&sk[6 * lo + 0], ord_key(p.x)); atomicMin(&sk[6 * lo + 1], ord_key(p.y));
        atomicMin(&sk[6 * lo + 2], ord_key(p.z)); atomicMax(&sk[6 * lo + 3], ord_key(p.x));
        atomicMax(&sk[6 * lo + 4], ord_key(p.y)); atomicMax(&sk[6 * lo + 5], ord_key(p.z));
      }
    }
  }
  box_flush(gcur, mn, mx, sk);
  __syncthreads();
  for (int t = threadIdx.x; t < 6 * ngroup; t += blockDim.x) {
    const int k = sk[t];
    if ((t % 6) < 3) { if (k != INT_MAX) atomicMin(&key[t], k); }
    else if (k != INT_MIN) atomicMax(&key[t], k);
  }
}

__global__ void k_box_finish(const int *__restrict__ key, int ngroup, double *__restrict__ out) {
  const int a = threadIdx.x;
  if (a >= 6) return;
  double u = a < 3 ? INFINITY : -INFINITY;
  for (int g = 0; g < ngroup; ++g) {
    const int k = key[6 * g + a];
    const bool empty = a < 3 ? k == INT_MAX : k == INT_MIN;
    const double v = empty ? (a < 3 ? INFINITY : -INFINITY) : (double)ord_val(k);
    out[6 * (1 + g) + a] = v;
    u = a < 3 ? fmin(u, v) : fmax(u, v);
  }
  out[a] = u;
}

// Target boxes of this rank for the LET (fp32 handles, after bh_sim_sort):
// d_start[ngroup + 1] body offsets; d_out[(1 + ngroup) * 6].
int bh_sim_target_boxes(bh_handle *h, const int64_t *d_start, int ngroup, double *d_out, void *stream) {
  if (!h || !d_start || !d_out || ngroup < 1 || ngroup > 256)
    return fail(BH_BAD_ARG, "bh_sim_target_boxes: bad args");
  if (h->precision != BH_FP32) return fail(BH_BAD_ARG, "bh_sim_target_boxes: fp32 handles");
  cudaStream_t s = S(stream);
  BH_CUDA(h->let_boxkey.ensure(sizeof(int) * 6 * ngroup));
  k_box_init<<<grid_for(6 * ngroup, 256), 256, 0, s>>>(h->let_boxkey.as<int>(), ngroup);
  const int64_t n = h->sim_n;
  if (n > 0) {
    const int64_t warps = std::min<int64_t>((n + 255) / 256, 4 * 8 * (int64_t)h->sms);
    const int64_t chunk = ((n + warps - 1) / warps + 31) / 32 * 32;
    const int blocks = (int)((((n + chunk - 1) / chunk) + 7) / 8);
    k_range_boxes<<<blocks, 256, 0, s>>>(h->pos.as<float4>(), n, d_start, ngroup, chunk,
                                          h->let_boxkey.as<int>());
  }
  k_box_finish<<<1, 32, 0, s>>>(h->let_boxkey.as<int>(), ngroup, d_out);
  h->launches += 3;
  BH_LAUNCHED();
  return BH_OK;
}

// Copy the walk records of the last bh_sim_build_local (d_out may be NULL to
// query the count).  Synchronises.
int bh_sim_walk_records(bh_handle *h, void *d_out, int64_t *n_out, void *stream) {
  if (!h || !n_out) return fail(BH_BAD_ARG, "bh_sim_walk_records: bad args");
  cudaStream_t s = S(stream);
  int cp = 0;
  BH_CUDA(cudaMemcpyAsync(&cp, h->dCp, sizeof(int), cudaMemcpyDeviceToHost, s));
  BH_CUDA(cudaStreamSynchronize(s));
  *n_out = cp;
  if (d_out && cp > 0)
    BH_CUDA(cudaMemcpyAsync(d_out, h->wnodes.p, sizeof(WalkNode) * cp, cudaMemcpyDeviceToDevice, s));
  return BH_OK;
}

// The walk's Hilbert target order for caller target arrays (the distributed
// walk): the same deterministic permutation for pass A and pass B
static const uint32_t *caller_target_order(bh_handle *h, const float *d_targets4, int64_t nt, cudaStream_t s) {
  if (!walk_hilbert_enabled() || nt <= 64) return nullptr;
  if (h->hperm.ensure(sizeof(uint32_t) * (nt + 1)) != cudaSuccess) return nullptr;
  launch_hilbert_chunks_pos(reinterpret_cast<const float4 *>(d_targets4), nt, h->dR, h->hperm.as<uint32_t>(), s);
  h->launches += 1;
  return h->hperm.as<uint32_t>();
}

// The fp32 walk over a caller-assembled record array (layout of WalkNode in
// bh_walk.cu; record 0 is the root) and a caller body array (bucket bodies).
int bh_walk_records_f32(bh_handle *h, const void *d_records, int64_t nrec, const float *d_bodies4,
                        const float *d_targets4, int64_t nt, double eps, int leaf_size,
                        float *d_acc4, int32_t *d_work, void *stream) {
  if (!h || nrec <= 0 || !d_records || nt < 0 || (nt && (!d_targets4 || !d_acc4)))
    return fail(BH_BAD_ARG, "bh_walk_records_f32: bad args");
  cudaStream_t s = S(stream);
  BH_TRY(reset_counters(h, s));
  h->tbegin(BH_PHASE_WALK, s);
  const uint32_t *perm = caller_target_order(h, d_targets4, nt, s);
  launch_walk_f32(static_cast<const WalkNode *>(d_records), nrec, reinterpret_cast<const float4 *>(d_bodies4),
                  d_targets4, 4, perm, (int)nt, (float)(eps * eps), leaf_size, d_acc4, 4, nullptr,
                  d_work, h->flags, s);
  h->tend(s);
  h->launches += 1;
  BH_LAUNCHED();
  return BH_OK;
}

// The LET overlap, pass A: walk over the local part of the
// assembled tree; remote branch records flagged (d.w | 1<<30) are not opened
// and each warp's (target chunk, record, masks) goes to d_defer[cap] (count in
// *d_count; entries past cap are dropped and the count says so).
int bh_walk_records_defer_f32(bh_handle *h, const void *d_records, int64_t nrec, const float *d_bodies4,
                              const float *d_targets4, int64_t nt, double eps, int leaf_size, float *d_acc4,
                              int32_t *d_work, int32_t *d_defer, uint32_t *d_count, int64_t cap, void *stream) {
  if (!h || nrec <= 0 || !d_records || nt < 0 || (nt && (!d_targets4 || !d_acc4)) || !d_defer || !d_count)
    return fail(BH_BAD_ARG, "bh_walk_records_defer_f32: bad args");
  cudaStream_t s = S(stream);
  BH_TRY(reset_counters(h, s));
  BH_CUDA(cudaMemsetAsync(d_count, 0, sizeof(uint32_t), s));
  DeferArgs dfr;
  dfr.out = reinterpret_cast<int4 *>(d_defer);
  dfr.count = d_count;
  dfr.cap = (int)std::min<int64_t>(cap, 0x7fffffff);
  h->tbegin(BH_PHASE_WALK, s);
  const uint32_t *perm = caller_target_order(h, d_targets4, nt, s);
  launch_walk_defer_f32(static_cast<const WalkNode *>(d_records), nrec, reinterpret_cast<const float4 *>(d_bodies4),
                        d_targets4, (int)nt, (float)(eps * eps), leaf_size, d_acc4, d_work, h->flags, dfr, false, s,
                        perm);
  h->tend(s);
  h->launches += 1;
  BH_LAUNCHED();
  return BH_OK;
}

// Pass B: resume the deferred entries d_entries[n_entries] (target chunk,
// record, m0, m1) over the full tree, d_fcnc[record] = (first child, nchild);
// results are added into d_acc4 / d_work.
int bh_walk_records_resume_f32(bh_handle *h, const void *d_records, int64_t nrec, const float *d_bodies4,
                               const float *d_targets4, int64_t nt, double eps, int leaf_size, float *d_acc4,
                               int32_t *d_work, const int32_t *d_entries, int64_t n_entries,
                               const int32_t *d_fcnc, void *stream) {
  if (!h || nrec <= 0 || !d_records || nt < 0 || n_entries < 0 || (n_entries && (!d_entries || !d_fcnc)))
    return fail(BH_BAD_ARG, "bh_walk_records_resume_f32: bad args");
  if (n_entries == 0 || nt == 0) return BH_OK;
  cudaStream_t s = S(stream);
  DeferArgs dfr;
  dfr.in = reinterpret_cast<const int4 *>(d_entries);
  dfr.nin = (int)n_entries;
  dfr.fcnc = reinterpret_cast<const int2 *>(d_fcnc);
  h->tbegin(BH_PHASE_WALK, s);
  const uint32_t *perm = caller_target_order(h, d_targets4, nt, s);  // pass A's order (deterministic)
  launch_walk_defer_f32(static_cast<const WalkNode *>(d_records), nrec, reinterpret_cast<const float4 *>(d_bodies4),
                        d_targets4, (int)nt, (float)(eps * eps), leaf_size, d_acc4, d_work, h->flags, dfr, true, s,
                        perm);
  h->tend(s);
  h->launches += 1;
  BH_LAUNCHED();
  return BH_OK;
}

int bh_sim_export(bh_handle *h, int what, int64_t begin, int64_t end, void *dst, void *stream) {
  if (!h || !dst || begin < 0 || end > h->sim_n || begin > end)
    return fail(BH_BAD_ARG, "bh_sim_export: bad args");
  const int64_t k = end - begin;
  if (k == 0) return BH_OK;
  cudaStream_t s = S(stream);
  const size_t e4 = h->precision == BH_FP32 ? sizeof(float4) : sizeof(double4);
  switch (what) {
    case BH_SIM_ACC:
      BH_CUDA(cudaMemcpyAsync(dst, h->acc.as<char>() + e4 * begin, e4 * k, cudaMemcpyDeviceToDevice, s));
      break;
    case BH_SIM_POS:
      BH_CUDA(cudaMemcpyAsync(dst, h->pos.as<char>() + e4 * begin, e4 * k, cudaMemcpyDeviceToDevice, s));
      break;
    case BH_SIM_WORK:
      BH_CUDA(cudaMemcpyAsync(dst, h->work_sorted.as<int>() + begin, sizeof(int) * k,
                              cudaMemcpyDeviceToDevice, s));
      break;
    case BH_SIM_PREV_WORK:
      BH_TRY(flush_work(h, s));
      k_gather_work<<<grid_for(k, 256), 256, 0, s>>>(h->work_orig.as<int>(), h->id.as<uint32_t>(),
                                                     begin, end, static_cast<int *>(dst));
      BH_LAUNCHED();
      break;
    case BH_SIM_VEL:
      BH_CUDA(cudaMemcpyAsync(dst, h->vel.as<char>() + e4 * begin, e4 * k, cudaMemcpyDeviceToDevice, s));
      break;
    case BH_SIM_ID:
      BH_CUDA(cudaMemcpyAsync(dst, h->id.as<uint32_t>() + begin, sizeof(uint32_t) * k,
                              cudaMemcpyDeviceToDevice, s));
      break;
    case BH_SIM_KEYS:
      BH_CUDA(cudaMemcpyAsync(dst, h->keys2.as<uint64_t>() + begin, sizeof(uint64_t) * k,
                              cudaMemcpyDeviceToDevice, s));
      break;
    default:
      return fail(BH_BAD_ARG, "bh_sim_export: unknown array");
  }
  return BH_OK;
}

int bh_sim_import(bh_handle *h, int what, int64_t begin, int64_t end, const void *src, void *stream) {
  if (!h || !src || begin < 0 || end > h->sim_n || begin > end)
    return fail(BH_BAD_ARG, "bh_sim_import: bad args");
  const int64_t k = end - begin;
  if (k == 0) return BH_OK;
  cudaStream_t s = S(stream);
  const size_t e4 = h->precision == BH_FP32 ? sizeof(float4) : sizeof(double4);
  switch (what) {
    case BH_SIM_ACC:
      BH_CUDA(cudaMemcpyAsync(h->acc.as<char>() + e4 * begin, src, e4 * k, cudaMemcpyDeviceToDevice, s));
      break;
    case BH_SIM_WORK:
      BH_CUDA(cudaMemcpyAsync(h->work_sorted.as<int>() + begin, src, sizeof(int) * k,
                              cudaMemcpyDeviceToDevice, s));
      break;
    default:
      return fail(BH_BAD_ARG, "bh_sim_import: acc and work only");
  }
  return BH_OK;
}

int bh_sim_store(bh_handle *h, void *d_pos, void *d_vel, void *d_acc, int64_t *d_work,
                 void *stream) {
  if (!h) return fail(BH_BAD_ARG, "bh_sim_store: bad args");
  const int64_t n = h->sim_n;
  if (n == 0) return BH_OK;
  cudaStream_t s = S(stream);
  const int g = grid_for(n, 256);
  const uint32_t *id = h->id.as<uint32_t>();
  if (h->precision == BH_FP32) {
    if (d_pos) k_store4<float4><<<g, 256, 0, s>>>(h->pos.as<float4>(), id, n, (float4 *)d_pos);
    if (d_vel) k_store4<float4><<<g, 256, 0, s>>>(h->vel.as<float4>(), id, n, (float4 *)d_vel);
    if (d_acc) k_store4<float4><<<g, 256, 0, s>>>(h->acc.as<float4>(), id, n, (float4 *)d_acc);
  } else {
    if (d_pos) k_store3<<<g, 256, 0, s>>>(h->pos.as<double4>(), id, n, (double *)d_pos);
    if (d_vel) k_store3<<<g, 256, 0, s>>>(h->vel.as<double4>(), id, n, (double *)d_vel);
    if (d_acc) k_store3<<<g, 256, 0, s>>>(h->acc.as<double4>(), id, n, (double *)d_acc);
  }
  if (d_work) {
    BH_TRY(flush_work(h, s));
    k_work64<<<g, 256, 0, s>>>(h->work_orig.as<int>(), n, d_work);
  }
  BH_LAUNCHED();
  return BH_OK;
}

int bh_stats_get(bh_handle *h, bh_stats *out, void *stream) {
  if (!h || !out) return fail(BH_BAD_ARG, "bh_stats_get: bad args");
  BH_TRY(read_flags(h, S(stream)));
  out->n_bodies = h->tree_n < 0 ? 0 : h->tree_n;
  if (h->async_tree) {
    int overflow = 0;
    BH_TRY(async_readback(h, S(stream), &overflow));
  }
  out->n_cells = h->async_tree ? h->C_true : h->C;
  out->max_level = h->max_level;
  out->pp = (int64_t)h->hflags->pp;
  out->pc = (int64_t)h->hflags->pc;
  out->work = out->pp + 2 * out->pc;
  out->launches = h->launches;
  out->n_records = 0;
  if (h->walk_valid) {  // the walk tree's record count (device), one more 4-byte read
    int nr = 0;
    BH_CUDA(cudaMemcpyAsync(h->hstat + kMaxLevel + 2, h->dCp, sizeof(int), cudaMemcpyDeviceToHost, S(stream)));
    BH_CUDA(cudaStreamSynchronize(S(stream)));
    nr = h->hstat[kMaxLevel + 2];
    out->n_records = nr;
  }
  return BH_OK;
}

int bh_timing_enable(bh_handle *h, int on) {
  if (!h) return fail(BH_BAD_ARG, "bh_timing_enable: bad args");
  h->timing = on != 0;
  return BH_OK;
}

int bh_timing_reset(bh_handle *h) {
  if (!h) return fail(BH_BAD_ARG, "bh_timing_reset: bad args");
  h->fold_marks();
  for (double &x : h->phase_ms) x = 0.0;
  h->launches = 0;
  return BH_OK;
}

int bh_timing_get(bh_handle *h, double *ms_out, int nphases) {
  if (!h || !ms_out || nphases < 0) return fail(BH_BAD_ARG, "bh_timing_get: bad args");
  h->fold_marks();
  for (int i = 0; i < nphases && i < BH_NPHASES; ++i) ms_out[i] = h->phase_ms[i];
  return BH_OK;
}

static int fma_peak(bh_handle *h, bool fp64, double *tflops_out, void *stream) {
  cudaStream_t s = S(stream);
  int sms = 0;
  BH_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, h->device));
  Buf out;
  BH_CUDA(out.ensure(64));
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  double flops = 0.0;
  const int iters = fp64 ? 1 << 12 : 1 << 14;
  for (int k = 0; k < 2; ++k) {  // warm-up, then timed
    if (k) cudaEventRecord(a, s);
    if (fp64) run_dfma(out.as<double>(), sms, iters, &flops, s);
    else run_ffma(out.as<float>(), sms, iters, &flops, s);
  }
  cudaEventRecord(b, s);
  BH_LAUNCHED();
  BH_CUDA(cudaEventSynchronize(b));
  float ms = 0.f;
  cudaEventElapsedTime(&ms, a, b);
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  out.release();
  *tflops_out = flops / (ms * 1e-3) / 1e12;
  return BH_OK;
}
int bh_host_register(void *p, int64_t bytes) {
  if (!p || bytes <= 0) return fail(BH_BAD_ARG, "bh_host_register: bad args");
  BH_CUDA(cudaHostRegister(p, (size_t)bytes, cudaHostRegisterDefault));
  return BH_OK;
}
int bh_host_unregister(void *p) {
  if (!p) return fail(BH_BAD_ARG, "bh_host_unregister: bad args");
  BH_CUDA(cudaHostUnregister(p));
  return BH_OK;
}

int bh_ffma_peak(bh_handle *h, double *tflops_out, void *stream) {
  if (!h || !tflops_out) return fail(BH_BAD_ARG, "bh_ffma_peak: bad args");
  return fma_peak(h, false, tflops_out, stream);
}
int bh_dfma_peak(bh_handle *h, double *tflops_out, void *stream) {
  if (!h || !tflops_out) return fail(BH_BAD_ARG, "bh_dfma_peak: bad args");
  return fma_peak(h, true, tflops_out, stream);
}

}  // extern "C"
