// bh_walk.cu -- the fp32 force traversal (flattree.py:258-317) and the walk
// tree it runs on.  Compiled with -ftz=true (no denormal fix-up around
// MUFU.RSQ; distances here are never denormal).
//
// Walk tree.  The reference tree keeps one body per leaf; with leaf size L a
// cell of count <= L is never opened, so its subtree is dead
// weight for the walk.  k_slots / k_nchild / k_compact copy the cells a walk
// can reach -- the root and every child of a cell with count > L -- into 64-byte
// records laid out with each cell's children contiguous (in slot order), the
// MAC threshold (side/theta)^2 baked in:
//
//   a = {-com.x, -com.y, -com.z, mac2}   MAC test (d = p + a)
//   b = {qxx, qxy, qxy, qyy}             quadrupole, paired for FFMA2
//   c = {qxz, qyz, mass, qzz}
//   d = {first_child | lo, count, nchild, level}
//        internal (count > L): children at [first_child, first_child+nchild)
//        bucket / leaf (count <= L, or a level-21 duplicate-key cell):
//        nchild = 0, its bodies are the sorted bodies [lo, lo+count)
//
// Walk.  fp32 mode must reproduce each target's reference interaction *set*
// (which cells pass the MAC, which are opened); the summation order only moves
// fp32 rounding.  So instead of the reference's per-target DFS, a warp walks a
// masked stack: an entry (first_child, nchild, mask0, mask1) says "these
// children must be examined for the targets in the masks" (the targets that
// opened their parent).  Popping an entry runs one warp-uniform loop over the
// siblings: per child each target applies the reference MAC itself -- accept
// (quadrupole pc), leaf (softened pp), bucket (pp over its bodies) or open
// (ballot -> push the child's own entry).  A cell is examined for a target
// exactly when the target opened its parent, as in the reference recursion.
//
// Two targets per lane (64 per warp): lane l of warp w owns the Morton-adjacent
// targets 64w+2l, 64w+2l+1 as float2 pairs, so the MAC / pc / pp math runs in
// FFMA2/FMUL2/FADD2 (the kernel is issue-bound; a packed instruction does two
// FMAs per issue slot).  The union of 64 Morton-consecutive interaction lists
// is only ~1.11x that of 32 (cfg2: 1803 vs 1628 cells), so each 64-byte cell
// record loaded serves ~1.8x more target interactions than with one target
// per lane.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <climits>
#include <cstddef>
#include <cstdlib>
#include <cooperative_groups.h>

#include "bh_internal.cuh"

namespace bh {

__device__ __forceinline__ int64_t tree_count(const TreeView &t) { return t.dC ? *t.dC : t.C; }
// a sync-free build that overflowed its capacity built nothing (k_emit and
// k_moments_coop returned early): the walk tree is then one empty root record,
// so nothing below reads the unbuilt cells (the call is redone, bh_api.cu)
__device__ __forceinline__ bool tree_overflowed(const TreeView &t) { return t.dC && *t.dC > t.C; }

__device__ __forceinline__ int child_slot(const TreeView &t, int64_t c) {
  const int4 L = t.link[c];
  return (int)((t.keys[L.z] >> (3 * (kMortonBits - L.w))) & 7);
}

// A cell's children are reachable when it can be opened: count > L, or it is
// the root (the walk always starts at the root's children, flattree.py:271-279)
__device__ __forceinline__ bool expandable(const TreeView &t, int64_t c, int leaf,
                                           const uint8_t *force) {
  if (force && force[c]) return true;  // a rank's shared cell (distributed build)
  const int4 L = t.link[c];
  // level-21 cells of duplicate keys have no children: always buckets
  return (L.y > leaf || (c == 0 && L.y > 1)) && L.w < kMaxLevel;
}

// slot masks of the expandable cells
__global__ void k_slots(TreeView t, int leaf, const uint8_t *force, uint32_t *__restrict__ smask) {
  int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c <= 0 || c >= tree_count(t) || c >= t.C || tree_overflowed(t)) return;
  const int P = t.parent[c];
  if (expandable(t, P, leaf, force)) atomicOr(&smask[P], 1u << child_slot(t, c));
}

// children per reachable internal cell (0 for buckets, leaves, pruned cells)
__global__ void k_nchild(TreeView t, int leaf, const uint8_t *force,
                         const uint32_t *__restrict__ smask, uint32_t *__restrict__ nck) {
  int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= t.C) return;
  if (c >= tree_count(t) || tree_overflowed(t)) {  // capacity tail (sync-free build): scans as zero
    nck[c] = 0u;
    return;
  }
  const bool kept = c == 0 || expandable(t, t.parent[c], leaf, force);
  nck[c] = (kept && expandable(t, c, leaf, force)) ? (uint32_t)__popc(smask[c]) : 0u;
}

// children per reachable internal cell from the child8 rows (leaf children are
// stored as -(c + 2), absent as -1).  Without shared-cell flags a cell that can
// be opened has a parent that can be opened (counts grow up the tree), so no
// reachability test is needed.
__global__ void k_nchild_rows(TreeView t, int leaf, uint32_t *__restrict__ nck) {
  int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= t.C) return;
  uint32_t k = 0u;
  // walk-only builds for this leaf size: the emit kernel's class byte says which
  // cells the walk opens (no link read for the cells inside buckets)
  const bool opens = t.mclass && t.mleaf == leaf
                         ? (t.mclass[c] >= 2 && t.mclass[c] != kClassLeafRecord)
                         : (c < tree_count(t) && expandable(t, c, leaf, nullptr));
  if (c < tree_count(t) && !tree_overflowed(t) && opens) {
    const int4 *row = reinterpret_cast<const int4 *>(t.child8 + 8 * c);
    const int4 r0 = row[0], r1 = row[1];
    k = (r0.x != -1) + (r0.y != -1) + (r0.z != -1) + (r0.w != -1) + (r1.x != -1) + (r1.y != -1) +
        (r1.z != -1) + (r1.w != -1);
  }
  nck[c] = k;
}

// The 64-byte walk record of cell c (MAC threshold from R, negated com,
// paired quadrupole words, first child or first body)
__device__ __forceinline__ WalkNode walk_record(const TreeView &t, int64_t c, const double *__restrict__ dR,
                                                double theta, bool internal, const uint32_t *__restrict__ nck,
                                                const uint32_t *__restrict__ base) {
  const int4 L = t.link[c];
  const double4 cm = t.cm64[c];
  WalkNode nd;
  // negated com: the walk forms d = p - com as p + a (one FADD2 per axis)
  const double r = ldexp(2.0 * dR[0], -L.w) / theta;  // theta == 0 -> inf: never accept
  nd.a = make_float4(-(float)cm.x, -(float)cm.y, -(float)cm.z, (float)(r * r));
  float q0 = 0.f, q1 = 0.f, q2 = 0.f, q3 = 0.f, q4 = 0.f, q5 = 0.f;
  if (L.y > 1) {
    const double *q = t.q64 + kQStride * c;
    q0 = (float)q[0]; q1 = (float)q[1]; q2 = (float)q[2];
    q3 = (float)q[3]; q4 = (float)q[4]; q5 = (float)q[5];
  }
  nd.b = make_float4(q0, q1, q1, q3);
  nd.c = make_float4(q2, q4, (float)cm.w, q5);
  nd.d = make_int4(internal ? 1 + (int)base[c] : L.z, L.y, internal ? (int)nck[c] : 0, L.w);
  return nd;
}

__global__ void k_compact(TreeView t, const double *__restrict__ dR, double theta, int leaf,
                          const uint8_t *force, const uint32_t *__restrict__ smask,
                          const uint32_t *__restrict__ nck, const uint32_t *__restrict__ base,
                          WalkNode *__restrict__ out, int *__restrict__ dCp,
                          int *__restrict__ rec_of_cell, int *__restrict__ wparent) {
  int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t C = tree_count(t);
  if (tree_overflowed(t)) {  // one empty root record (count 0: the walk interacts with nothing)
    if (c == 0) {
      WalkNode nd;
      nd.a = make_float4(0.f, 0.f, 0.f, 0.f);
      nd.b = nd.a;
      nd.c = nd.a;
      nd.d = make_int4(0, 0, 0, 0);
      out[0] = nd;
      *dCp = 1;
      if (rec_of_cell) rec_of_cell[0] = 0;
      if (wparent) wparent[0] = -1;
    }
    return;
  }
  if (c >= C || c >= t.C) return;
  if (c == C - 1) *dCp = (int)(1 + base[C - 1] + nck[C - 1]);
  int j = 0;
  if (c > 0) {
    if (t.mclass && t.mleaf == leaf && !force && t.mclass[c] == 0) {  // inside a bucket (class byte)
      if (rec_of_cell) rec_of_cell[c] = -1;
      return;
    }
    const int P = t.parent[c];
    if (!expandable(t, P, leaf, force)) {  // pruned (inside a bucket)
      if (rec_of_cell) rec_of_cell[c] = -1;
      return;
    }
    if (smask) {
      const int slot = child_slot(t, c);
      j = 1 + (int)base[P] + __popc(smask[P] & ((1u << slot) - 1u));
    } else {  // rank among the parent's present children, from its child8 row
      const int4 *row = reinterpret_cast<const int4 *>(t.child8 + 8 * (int64_t)P);
      const int4 r0 = row[0], r1 = row[1];
      const int v[8] = {r0.x, r0.y, r0.z, r0.w, r1.x, r1.y, r1.z, r1.w};
      const int cl = -(int)c - 2;  // a leaf child is stored as -(c + 2)
      int rank = 0;
#pragma unroll
      for (int s = 0; s < 8; ++s) {
        if (v[s] == (int)c || v[s] == cl) break;
        rank += v[s] != -1;
      }
      j = 1 + (int)base[P] + rank;
    }
  }
  const bool internal = expandable(t, c, leaf, force);
  if (rec_of_cell) rec_of_cell[c] = j;
  if (wparent) {  // record parent links (LET selection walks them top-down)
    if (c == 0) wparent[0] = -1;
    if (internal)
      for (int k = 0; k < (int)nck[c]; ++k) wparent[1 + (int)base[c] + k] = j;
  }
  out[j] = walk_record(t, c, dR, theta, internal, nck, base);
}

// Walk-only trees: the same records written from the parents' side.  The
// moments kernel listed every cell the walk opens (by level, in `mlist`);
// 8 lanes take one such cell, one child slot each, rank the present children
// by ballot and write their records -- no per-cell parent lookups, and the
// cells inside buckets are never touched.
__global__ void k_compact_parents(TreeView t, const double *__restrict__ dR, double theta, int leaf,
                                  const uint32_t *__restrict__ nck, const uint32_t *__restrict__ base,
                                  WalkNode *__restrict__ out, int *__restrict__ dCp) {
  const int64_t C = tree_count(t);
  const int64_t gt = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (tree_overflowed(t)) {
    if (gt == 0) {
      WalkNode nd;
      nd.a = make_float4(0.f, 0.f, 0.f, 0.f);
      nd.b = nd.a;
      nd.c = nd.a;
      nd.d = make_int4(0, 0, 0, 0);
      out[0] = nd;
      *dCp = 1;
    }
    return;
  }
  if (gt == 0) {  // the root's record (and the record count, unless the list scan set it)
    if (dCp) *dCp = (int)(1 + base[C - 1] + nck[C - 1]);
    out[0] = walk_record(t, 0, dR, theta, expandable(t, 0, leaf, nullptr), nck, base);
  }
  const int *cnt = t.mlvl + 2 * (kMaxLevel + 1);  // cursors = cells listed per level
  const int *offs = t.mlvl + (kMaxLevel + 1);
  int total = 0;
#pragma unroll 1
  for (int l = 0; l <= kMaxLevel; ++l) total += cnt[l];
  const int s = threadIdx.x & 7, sub = (threadIdx.x & 31) >> 3;
  const int64_t warp = gt >> 5, nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t wb = warp * 4; wb < total; wb += nwarps * 4) {  // warp-uniform: 4 cells per pass
    const int64_t g = wb + sub;
    int P = -1;
    if (g < total) {
      int r = (int)g;
      for (int l = 0; l <= kMaxLevel; ++l) {
        if (r < cnt[l]) {
          P = t.mlist[offs[l] + r];
          break;
        }
        r -= cnt[l];
      }
    }
    int c = -1;
    if (P >= 0) {
      c = t.child8[8 * (int64_t)P + s];
      if (c < -1) c = -c - 2;  // a leaf child, stored as -(c + 2)
    }
    const unsigned grp = 0xffu << (threadIdx.x & 24);
    const unsigned have = __ballot_sync(0xffffffffu, c >= 0) & grp;
    if (c >= 0) {
      const int rank = __popc(have & ((1u << (threadIdx.x & 31)) - 1u));
      const int j = 1 + (int)base[P] + rank;
      const uint8_t cl = t.mclass[c];
      out[j] = walk_record(t, c, dR, theta, cl >= 2 && cl != kClassLeafRecord, nck, base);
    }
  }
}

// Walk-only trees: children are counted and the record bases scanned over the
// list of opened cells only (~1% of the cells), not over every cell.
//   k_nchild_list   nck[P] and ncl[g] for the g-th listed cell P (level order)
//   k_scan_list_*   exclusive scan of ncl[0, total) in place (total on device)
//   k_base_list     base[P] = scanned ncl[g]; the record count
__device__ __forceinline__ int listed_cell(const int *cnt, const int *offs, const int *list, int64_t g) {
  int r = (int)g;
  for (int l = 0; l <= kMaxLevel; ++l) {
    if (r < cnt[l]) return list[offs[l] + r];
    r -= cnt[l];
  }
  return -1;
}
__global__ void k_nchild_list(TreeView t, uint32_t *__restrict__ nck, uint32_t *__restrict__ ncl) {
  if (tree_overflowed(t)) return;
  __shared__ int cnt[kMaxLevel + 1], offs[kMaxLevel + 1], total;
  if (threadIdx.x == 0) {
    int tot = 0;
    for (int l = 0; l <= kMaxLevel; ++l) {
      cnt[l] = t.mlvl[2 * (kMaxLevel + 1) + l];  // cells listed per level
      offs[l] = t.mlvl[(kMaxLevel + 1) + l];
      tot += cnt[l];
    }
    total = tot;
  }
  __syncthreads();
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < total; g += (int64_t)gridDim.x * blockDim.x) {
    const int P = listed_cell(cnt, offs, t.mlist, g);
    const int4 *row = reinterpret_cast<const int4 *>(t.child8 + 8 * (int64_t)P);
    const int4 r0 = row[0], r1 = row[1];
    const uint32_t k = (r0.x != -1) + (r0.y != -1) + (r0.z != -1) + (r0.w != -1) + (r1.x != -1) +
                       (r1.y != -1) + (r1.z != -1) + (r1.w != -1);
    nck[P] = k;
    ncl[g] = k;
  }
}
// exclusive scan of v[0, total) in place, total = the listed cells (on device):
// tile sums, one block scans them (and sets the record count), tiles add their prefix
constexpr int kLTile = 4096;  // 256 threads x 16 (the tile sums fit the C-sized scan temp)
__device__ __forceinline__ int listed_total(const TreeView &t) {
  int tot = 0;
  for (int l = 0; l <= kMaxLevel; ++l) tot += t.mlvl[2 * (kMaxLevel + 1) + l];
  return tot;
}
__device__ __forceinline__ unsigned block_excl_256(unsigned v, unsigned *wsum, unsigned *all) {
  const unsigned lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  unsigned incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned x = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= (unsigned)o) incl += x;
  }
  if (lane == 31) wsum[w] = incl;
  __syncthreads();
  unsigned woff = 0, tot = 0;
  for (int i = 0; i < (int)(blockDim.x >> 5); ++i) {
    woff += i < (int)w ? wsum[i] : 0u;
    tot += wsum[i];
  }
  if (all) *all = tot;
  __syncthreads();
  return woff + incl - v;
}
__global__ void __launch_bounds__(256) k_scan_list_tiles(const TreeView t, const uint32_t *__restrict__ v,
                                                         uint32_t *__restrict__ tsum) {
  if (tree_overflowed(t)) return;
  __shared__ unsigned wsum[8];
  const int64_t total = listed_total(t), ntiles = (total + kLTile - 1) / kLTile;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    unsigned sum = 0;
    for (int k = 0; k < kLTile / 256; ++k) {
      const int64_t i = tile * kLTile + k * 256 + threadIdx.x;
      if (i < total) sum += v[i];
    }
    unsigned all;
    block_excl_256(sum, wsum, &all);
    if (threadIdx.x == 0) tsum[tile] = all;
  }
}
__global__ void __launch_bounds__(1024) k_scan_list_top(const TreeView t, uint32_t *__restrict__ tsum,
                                                        int *__restrict__ dCp) {
  if (tree_overflowed(t)) {  // the build overflowed (redone): one empty root record
    if (threadIdx.x == 0) *dCp = 1;
    return;
  }
  __shared__ unsigned wsum[32];
  const int64_t total = listed_total(t), ntiles = (total + kLTile - 1) / kLTile;
  const int64_t per = (ntiles + 1023) / 1024;
  const int64_t b = per * threadIdx.x, e = b + per < ntiles ? b + per : ntiles;
  unsigned run = 0;
  for (int64_t i = b; i < e; ++i) run += tsum[i];
  const unsigned lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  unsigned incl = run;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned x = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= (unsigned)o) incl += x;
  }
  if (lane == 31) wsum[w] = incl;
  __syncthreads();
  unsigned woff = 0, all = 0;
  for (int i = 0; i < 32; ++i) {
    woff += i < (int)w ? wsum[i] : 0u;
    all += wsum[i];
  }
  unsigned ex = woff + incl - run;
  for (int64_t i = b; i < e; ++i) {
    const unsigned x = tsum[i];
    tsum[i] = ex;
    ex += x;
  }
  if (threadIdx.x == 0) *dCp = 1 + (int)all;  // the root and every listed cell's children
}
__global__ void __launch_bounds__(256) k_scan_list_down(const TreeView t, uint32_t *__restrict__ v,
                                                        const uint32_t *__restrict__ tsum) {
  if (tree_overflowed(t)) return;
  __shared__ unsigned wsum[8];
  const int64_t total = listed_total(t), ntiles = (total + kLTile - 1) / kLTile;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t i0 = tile * kLTile + (int64_t)threadIdx.x * (kLTile / 256);
    unsigned x[kLTile / 256], sum = 0;
#pragma unroll
    for (int k = 0; k < kLTile / 256; ++k) {
      x[k] = i0 + k < total ? v[i0 + k] : 0u;
      sum += x[k];
    }
    unsigned run = tsum[tile] + block_excl_256(sum, wsum, nullptr);
#pragma unroll
    for (int k = 0; k < kLTile / 256; ++k) {
      if (i0 + k < total) v[i0 + k] = run;
      run += x[k];
    }
  }
}
__global__ void k_base_list(TreeView t, const uint32_t *__restrict__ ncl, uint32_t *__restrict__ base) {
  if (tree_overflowed(t)) return;
  __shared__ int cnt[kMaxLevel + 1], offs[kMaxLevel + 1], total;
  if (threadIdx.x == 0) {
    int tot = 0;
    for (int l = 0; l <= kMaxLevel; ++l) {
      cnt[l] = t.mlvl[2 * (kMaxLevel + 1) + l];
      offs[l] = t.mlvl[(kMaxLevel + 1) + l];
      tot += cnt[l];
    }
    total = tot;
  }
  __syncthreads();
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < total; g += (int64_t)gridDim.x * blockDim.x)
    base[listed_cell(cnt, offs, t.mlist, g)] = ncl[g];
}

void launch_walk_tree(const TreeView &t, const double *dR, double theta, int leaf,
                      uint32_t *smask, uint32_t *nck, uint32_t *base, void *scan_tmp,
                      size_t scan_bytes, WalkNode *out, int *dCp, cudaStream_t s,
                      const uint8_t *force, int *rec_of_cell, int *wparent) {
  const int g = grid_for(t.C, 256);
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  if (!force && t.mclass && t.mleaf == leaf && t.mlvl && !rec_of_cell && !wparent) {  // walk-only tree
    uint32_t *ncl = smask;  // scratch (>= C entries), unused on this path
    uint32_t *tsum = static_cast<uint32_t *>(scan_tmp);  // (>= C / 4096 tile sums)
    k_nchild_list<<<sms * 4, 256, 0, s>>>(t, nck, ncl);
    k_scan_list_tiles<<<sms * 4, 256, 0, s>>>(t, ncl, tsum);
    k_scan_list_top<<<1, 1024, 0, s>>>(t, tsum, dCp);
    k_scan_list_down<<<sms * 4, 256, 0, s>>>(t, ncl, tsum);
    k_base_list<<<sms * 4, 256, 0, s>>>(t, ncl, base);
    k_compact_parents<<<sms * 8, 256, 0, s>>>(t, dR, theta, leaf, nck, base, out, nullptr);
    return;
  }
  if (!force) {  // children counted and ranked from the child8 rows: no slot-mask pass
    k_nchild_rows<<<g, 256, 0, s>>>(t, leaf, nck);
    exclusive_scan_u32(scan_tmp, scan_bytes, nck, base, t.C, s);
    k_compact<<<g, 256, 0, s>>>(t, dR, theta, leaf, force, nullptr, nck, base, out, dCp, rec_of_cell, wparent);
    return;
  }
  cudaMemsetAsync(smask, 0, sizeof(uint32_t) * t.C, s);
  k_slots<<<g, 256, 0, s>>>(t, leaf, force, smask);
  k_nchild<<<g, 256, 0, s>>>(t, leaf, force, smask, nck);
  exclusive_scan_u32(scan_tmp, scan_bytes, nck, base, t.C, s);
  k_compact<<<g, 256, 0, s>>>(t, dR, theta, leaf, force, smask, nck, base, out, dCp, rec_of_cell,
                              wparent);
}

// ------------------------------------------------ locally essential trees
// Conservative box-MAC: a record is taken (pc) by every target
// of a receiver if, for each of the receiver's target boxes, even the box point
// nearest its com passes the MAC with a relative margin that covers the fp32
// rounding of d2 on the receiving side.  Empty boxes (lo > hi) never object.
__device__ __forceinline__ double box_d2(const double c[3], const double *box) {
  double d2 = 0.0;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const double lo = box[a], hi = box[3 + a];
    const double g = c[a] < lo ? lo - c[a] : (c[a] > hi ? c[a] - hi : 0.0);
    d2 += g * g;
  }
  return d2;
}

// One record, one warp: the receivers' member boxes are tested lane-parallel
// A record is taken by every target of receiver q if it is clear of q's union
// box (box 0: passing it passes them all) or of every member box.
__device__ __forceinline__ void let_mark_warp(const WalkNode *__restrict__ W, int j, const int *__restrict__ wparent,
                                              const uint8_t *__restrict__ isbranch, const double *__restrict__ boxes,
                                              int nbox, int nrank, int self, uint32_t *__restrict__ present,
                                              uint32_t *__restrict__ expand, uint32_t *__restrict__ bodies) {
  const unsigned lane = threadIdx.x & 31;
  const WalkNode r = W[j];
  const uint32_t all = ((nrank >= 32 ? 0xffffffffu : (1u << nrank) - 1u)) & ~(1u << self);
  const uint32_t p = isbranch[j] ? all : (wparent[j] >= 0 ? expand[wparent[j]] : 0u);
  uint32_t fail = 0;
  if (p && r.d.y > 1) {
    const double c[3] = {-(double)r.a.x, -(double)r.a.y, -(double)r.a.z};
    const double lim = (double)r.a.w * (1.0 + 1e-5) + 1e-30;
    for (int q = 0; q < nrank; ++q) {
      if (!((p >> q) & 1u)) continue;
      const double *bq = boxes + (size_t)6 * nbox * q;
      if (box_d2(c, bq) > lim) continue;  // clear of the union: taken by every target of q
      bool f = nbox == 1;
      for (int k = 1 + (int)lane; k < nbox; k += 32) f = f || !(box_d2(c, bq + 6 * k) > lim);
      if (__any_sync(0xffffffffu, f)) fail |= 1u << q;
    }
  }
  if (lane == 0) {
    present[j] = p;
    expand[j] = r.d.z > 0 ? (p & fail) : 0u;
    bodies[j] = (r.d.z > 0 || r.d.y <= 1) ? 0u : (p & fail);
  }
}

// One cooperative launch: bucket the records by level, then sweep the levels
// top-down with a grid barrier between them (a record's parent is one level up).
namespace cg = cooperative_groups;
__global__ void __launch_bounds__(256) k_let_mark_coop(const WalkNode *__restrict__ W, int nrec,
                                                       const int *__restrict__ wparent,
                                                       const uint8_t *__restrict__ isbranch,
                                                       const double *__restrict__ boxes, int nbox, int nrank,
                                                       int self, int *__restrict__ lvl, int *__restrict__ list,
                                                       uint32_t *__restrict__ present, uint32_t *__restrict__ expand,
                                                       uint32_t *__restrict__ bodies) {
  cg::grid_group grid = cg::this_grid();
  int *cnt = lvl, *offs = lvl + (kMaxLevel + 1), *cur = lvl + 2 * (kMaxLevel + 1);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (tid <= kMaxLevel) { cnt[tid] = 0; cur[tid] = 0; }
  grid.sync();
  __shared__ int h[kMaxLevel + 1], base[kMaxLevel + 1];
  for (int64_t c0 = (int64_t)blockIdx.x * blockDim.x; c0 < nrec; c0 += stride) {  // level histogram
    if (threadIdx.x <= kMaxLevel) h[threadIdx.x] = 0;
    __syncthreads();
    const int64_t j = c0 + threadIdx.x;
    if (j < nrec) atomicAdd(&h[W[j].d.w], 1);
    __syncthreads();
    if (threadIdx.x <= kMaxLevel && h[threadIdx.x]) atomicAdd(&cnt[threadIdx.x], h[threadIdx.x]);
    __syncthreads();
  }
  grid.sync();
  if (tid == 0) {
    int acc = 0;
    for (int l = 0; l <= kMaxLevel; ++l) { offs[l] = acc; acc += cnt[l]; }
  }
  grid.sync();
  for (int64_t c0 = (int64_t)blockIdx.x * blockDim.x; c0 < nrec; c0 += stride) {  // bucket by level
    if (threadIdx.x <= kMaxLevel) h[threadIdx.x] = 0;
    __syncthreads();
    const int64_t j = c0 + threadIdx.x;
    int l = -1, rank = 0;
    if (j < nrec) { l = W[j].d.w; rank = atomicAdd(&h[l], 1); }
    __syncthreads();
    if (threadIdx.x <= kMaxLevel && h[threadIdx.x])
      base[threadIdx.x] = offs[threadIdx.x] + atomicAdd(&cur[threadIdx.x], h[threadIdx.x]);
    __syncthreads();
    if (l >= 0) list[base[l] + rank] = (int)j;
    __syncthreads();
  }
  grid.sync();
  const int64_t warp = tid >> 5, nwarps = stride >> 5;
  for (int l = 0; l <= kMaxLevel; ++l) {
    const int n_l = cnt[l];
    if (n_l == 0) continue;
    for (int64_t k = warp; k < n_l; k += nwarps)
      let_mark_warp(W, list[offs[l] + k], wparent, isbranch, boxes, nbox, nrank, self, present, expand, bodies);
    grid.sync();
  }
}

// all receivers at once (grid.y = receiver): rflag = the record goes to q
// (present and not a branch node -- those travel with the branch allgather);
// bcount = bodies shipped with it
__global__ void k_let_flags_all(const WalkNode *__restrict__ W, int nrec, const uint8_t *__restrict__ isbranch,
                                const uint32_t *__restrict__ present, const uint32_t *__restrict__ bodies,
                                int self, uint32_t *__restrict__ rflag, uint32_t *__restrict__ bcount) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  const int q = blockIdx.y;
  if (j >= nrec) return;
  const size_t o = (size_t)q * nrec + j;
  const bool me = q == self;
  rflag[o] = (!me && !isbranch[j] && ((present[j] >> q) & 1u)) ? 1u : 0u;
  bcount[o] = (!me && ((bodies[j] >> q) & 1u)) ? (uint32_t)W[j].d.y : 0u;
}

// receiver q's LET sizes from the inclusive scans over [nrank][nrec]
__global__ void k_let_tails(const uint32_t *__restrict__ rinc, const uint32_t *__restrict__ binc, int nrec,
                            int nrank, uint32_t *__restrict__ tails) {
  const int q = threadIdx.x;
  if (q >= nrank) return;
  const size_t e = (size_t)(q + 1) * nrec - 1, b = (size_t)q * nrec;
  tails[2 * q] = rinc[e] - (q ? rinc[b - 1] : 0u);
  tails[2 * q + 1] = binc[e] - (q ? binc[b - 1] : 0u);
}

// exclusive position of record j in receiver q's LET / body list
__device__ __forceinline__ uint32_t let_pos(const uint32_t *flag, const uint32_t *inc, int nrec, int q, int j) {
  const size_t o = (size_t)q * nrec + j;
  return inc[o] - flag[o] - (q ? inc[(size_t)q * nrec - 1] : 0u);
}

// Pack the LET for receiver q: its records in W order (children blocks stay
// contiguous), child links remapped into the LET, bucket body ranges into the
// LET's body list; records the receiver never opens get nchild = 0.
__global__ void k_let_pack(const WalkNode *__restrict__ W, int nrec, const uint32_t *__restrict__ expand,
                           const uint32_t *__restrict__ bodies, int q, const uint32_t *__restrict__ rflag,
                           const uint32_t *__restrict__ rinc, const uint32_t *__restrict__ bcount,
                           const uint32_t *__restrict__ binc, const float4 *__restrict__ src_bodies,
                           WalkNode *__restrict__ out, float4 *__restrict__ out_bodies) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= nrec) return;
  const bool body_need = (bodies[j] >> q) & 1u;
  if (body_need) {
    const uint32_t bp = let_pos(bcount, binc, nrec, q, j);
    for (int k = 0; k < W[j].d.y; ++k) out_bodies[bp + k] = src_bodies[W[j].d.x + k];
  }
  if (!rflag[(size_t)q * nrec + j]) return;
  WalkNode r = W[j];
  if ((expand[j] >> q) & 1u) r.d.x = (int)let_pos(rflag, rinc, nrec, q, r.d.x);
  else if (body_need) r.d.x = (int)let_pos(bcount, binc, nrec, q, j);
  else { r.d.z = 0; if (r.d.y > 1) r.d.x = -1; }  // never opened by the receiver
  out[let_pos(rflag, rinc, nrec, q, j)] = r;
}

// Branch roots for receiver q: (first child in the LET | -1, first body in
// the LET's body list | -1).
__global__ void k_let_branchmap(const WalkNode *__restrict__ W, const int *__restrict__ brec, int nb, int nrec,
                                const uint32_t *__restrict__ expand, const uint32_t *__restrict__ bodies, int q,
                                const uint32_t *__restrict__ rflag, const uint32_t *__restrict__ rinc,
                                const uint32_t *__restrict__ bcount, const uint32_t *__restrict__ binc,
                                int2 *__restrict__ map) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= nb) return;
  const int j = brec[k];
  const WalkNode r = W[j];
  map[k] = make_int2(((expand[j] >> q) & 1u) ? (int)let_pos(rflag, rinc, nrec, q, r.d.x) : -1,
                     ((bodies[j] >> q) & 1u) ? (int)let_pos(bcount, binc, nrec, q, j) : -1);
}

void launch_let_mark(const WalkNode *W, int nrec, const int *wparent, const uint8_t *isbranch,
                     const double *boxes, int nbox, int nrank, int self, int *lvl, int *list, int sms,
                     uint32_t *present, uint32_t *expand, uint32_t *bodies, cudaStream_t s) {
  if (nrec <= 0) return;
  static int per_sm = 0;
  if (per_sm == 0) {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_let_mark_coop, 256, 0);
    if (per_sm < 1) per_sm = 1;
  }
  const int blocks = (int)std::min<int64_t>((int64_t)sms * per_sm, ((int64_t)nrec + 255) / 256);
  void *args[] = {(void *)&W, &nrec, (void *)&wparent, (void *)&isbranch, (void *)&boxes, &nbox, &nrank, &self,
                  &lvl, &list, &present, &expand, &bodies};
  cudaLaunchCooperativeKernel((void *)k_let_mark_coop, dim3(blocks < 1 ? 1 : blocks), dim3(256), args, 0, s);
}
void launch_let_flags_all(const WalkNode *W, int nrec, const uint8_t *isbranch, const uint32_t *present,
                          const uint32_t *bodies, int nrank, int self, uint32_t *rflag, uint32_t *bcount,
                          cudaStream_t s) {
  if (nrec <= 0) return;
  dim3 g(grid_for(nrec, 256), nrank);
  k_let_flags_all<<<g, 256, 0, s>>>(W, nrec, isbranch, present, bodies, self, rflag, bcount);
}
void launch_let_tails(const uint32_t *rinc, const uint32_t *binc, int nrec, int nrank, uint32_t *tails,
                      cudaStream_t s) {
  k_let_tails<<<1, 32, 0, s>>>(rinc, binc, nrec, nrank, tails);
}
void launch_let_pack(const WalkNode *W, int nrec, const uint32_t *expand, const uint32_t *bodies, int q,
                     const uint32_t *rflag, const uint32_t *rinc, const uint32_t *bcount, const uint32_t *binc,
                     const float4 *src_bodies, WalkNode *out, float4 *out_bodies, cudaStream_t s) {
  if (nrec <= 0) return;
  k_let_pack<<<grid_for(nrec, 256), 256, 0, s>>>(W, nrec, expand, bodies, q, rflag, rinc, bcount, binc,
                                                 src_bodies, out, out_bodies);
}
void launch_let_branchmap(const WalkNode *W, const int *brec, int nb, int nrec, const uint32_t *expand,
                          const uint32_t *bodies, int q, const uint32_t *rflag, const uint32_t *rinc,
                          const uint32_t *bcount, const uint32_t *binc, int2 *map, cudaStream_t s) {
  if (nb <= 0) return;
  k_let_branchmap<<<grid_for(nb, 128), 128, 0, s>>>(W, brec, nb, nrec, expand, bodies, q, rflag, rinc, bcount,
                                                    binc, map);
}

__device__ __forceinline__ float2 f2(float x, float y) { return make_float2(x, y); }
// a v9 frontier word: first child | nchild << 28, built unsigned (nchild = 8
// would shift into the sign bit of an int)
__device__ __forceinline__ int fc_word(int first, int nchild) {
  return (int)((unsigned)first | ((unsigned)nchild << 28));
}
__device__ __forceinline__ float2 f2(float x) { return make_float2(x, x); }

#ifndef BH_WALK_BLOCK
#define BH_WALK_BLOCK 128  // 4 warps; 8 blocks/SM at <= 64 registers
#endif
constexpr int kWalkBlock = BH_WALK_BLOCK;
#ifndef BH_WALK_MINB
#define BH_WALK_MINB (1152 / BH_WALK_BLOCK)  // 9 blocks of 128 (<= 56 registers): +12% warps, -1%
#endif
constexpr int kStack = 8 * (kMaxLevel + 1) + 8;  // <= 8 pending siblings per level

#ifdef BH_WALK_HIST
// diagnostics: [0, 65) targets accepting each non-leaf visit; [65, 130) targets examining it
__device__ unsigned long long g_walk_hist[130];
extern "C" int bh_debug_walk_hist(unsigned long long *out) {
  return (int)cudaMemcpyFromSymbol(out, g_walk_hist, sizeof(g_walk_hist));
}
#endif

// Walk modes (the LET overlap of the distributed step):
//   kWalkFull   -- the whole tree;
//   kWalkDefer  -- pass A: records flagged kDeferBit in d.w (remote branch nodes
//                  whose subtrees are still in flight) are not opened; the
//                  warp's (record, masks) is appended to a list instead;
//   kWalkResume -- pass B: one warp per deferred (target chunk, record, masks),
//                  walking the record's subtree (first child, nchild from
//                  fcnc[record]) and adding into acc/work atomically.
enum { kWalkFull = 0, kWalkDefer = 1, kWalkResume = 2 };
#ifndef BH_BUCKET_UNROLL
#define BH_BUCKET_UNROLL 2
#endif
constexpr int kBucketUnroll = BH_BUCKET_UNROLL;  // bucket pp loop unroll

constexpr int kDeferBit = 1 << 30;

template <bool BUCKET, int MODE>
__global__ void __launch_bounds__(kWalkBlock, BH_WALK_MINB) k_walk(
    const WalkNode *__restrict__ T, const float4 *__restrict__ bodies,
    const float *__restrict__ targets, int tstride, const uint32_t *__restrict__ tperm, int nt,
    float e2, int leaf, float *__restrict__ acc, int astride, int64_t *__restrict__ work64,
    int *__restrict__ work32, DeviceFlags *f, DeferArgs dfr) {
  __shared__ int4 stack_all[kWalkBlock / 32][kStack];
  int4 *stk = stack_all[threadIdx.x >> 5];
  const unsigned lane = threadIdx.x & 31;
  const int64_t gwarp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int4 entry = make_int4(0, 0, 0, 0);
  if (MODE == kWalkResume) {
    if (gwarp >= dfr.nin) return;  // warp-uniform
    entry = dfr.in[gwarp];
  }
  const int64_t warp = MODE == kWalkResume ? (int64_t)entry.x : gwarp;
  const int64_t t0 = warp * 64 + 2 * lane, t1 = t0 + 1;
  const bool v0 = t0 < nt, v1 = t1 < nt;
  const int64_t s0 = v0 ? (tperm ? (int64_t)tperm[t0] : t0) : 0;
  const int64_t s1 = v1 ? (tperm ? (int64_t)tperm[t1] : t1) : 0;
  float2 X = f2(0.f), Y = f2(0.f), Z = f2(0.f);
  if (v0) { const float *q = targets + s0 * tstride; X.x = q[0]; Y.x = q[1]; Z.x = q[2]; }
  if (v1) { const float *q = targets + s1 * tstride; X.y = q[0]; Y.y = q[1]; Z.y = q[2]; }
  float2 AX = f2(0.f), AY = f2(0.f), AZ = f2(0.f);
  int pp0 = 0, pp1 = 0, pc0 = 0, pc1 = 0;
  const float2 E2 = f2(e2);
  const unsigned bit = 1u << lane;

  // current entry: examine children [fc, fc+nc) for the targets in (m0, m1)
  int4 e = make_int4(0, 1, (int)__ballot_sync(0xffffffffu, v0), (int)__ballot_sync(0xffffffffu, v1));
  if (MODE == kWalkResume) {
    const int2 fc = dfr.fcnc[entry.y];
    e = make_int4(fc.x, fc.y, entry.z, entry.w);
  } else if (T[0].d.y > 1) {  // root internal: the walk starts at its children (flattree.py:271-279)
    const int4 rd = T[0].d;
    e.x = rd.x;
    e.y = rd.z;
  }
  int sp = 0;
  for (;;) {
    const bool in0 = (unsigned)e.z & bit, in1 = (unsigned)e.w & bit;
    for (int c = e.x; c < e.x + e.y; ++c) {
      const WalkNode *nd = T + c;
      const float4 a = nd->a;
      const int4 d = nd->d;
      const float4 b = nd->b;  // quadrupole words loaded with the MAC word (latency overlap)
      const float4 q = nd->c;
      const int cnt = __reduce_max_sync(0xffffffffu, d.y);  // warp-uniform
      const float2 DX = __fadd2_rn(X, f2(a.x));
      const float2 DY = __fadd2_rn(Y, f2(a.y));
      const float2 DZ = __fadd2_rn(Z, f2(a.z));
      const float2 D2 = __ffma2_rn(DZ, DZ, __ffma2_rn(DY, DY, __fmul2_rn(DX, DX)));
      if (cnt == 1) {  // leaf: softened pp, the body itself skipped (flattree.py:287-294)
        const bool m0 = in0 && D2.x > 0.f, m1 = in1 && D2.y > 0.f;
        const float2 W = __fadd2_rn(D2, E2);
        const float2 R = f2(m0 ? rsqrtf(W.x) : 0.f, m1 ? rsqrtf(W.y) : 0.f);
        const float2 S = __fmul2_rn(__fmul2_rn(R, R), __fmul2_rn(R, f2(-nd->c.z)));
        AX = __ffma2_rn(S, DX, AX);
        AY = __ffma2_rn(S, DY, AY);
        AZ = __ffma2_rn(S, DZ, AZ);
        pp0 += m0; pp1 += m1;
        continue;
      }
      const bool c0 = in0 && D2.x > a.w, c1 = in1 && D2.y > a.w;  // MAC (flattree.py:295)
#ifdef BH_WALK_HIST
      {
        const int na = __popc(__ballot_sync(0xffffffffu, c0)) + __popc(__ballot_sync(0xffffffffu, c1));
        const int ni = __popc((unsigned)e.z) + __popc((unsigned)e.w);
        if (lane == 0) { atomicAdd(&g_walk_hist[na], 1ull); atomicAdd(&g_walk_hist[65 + ni], 1ull); }
      }
#endif
      if (__any_sync(0xffffffffu, c0 || c1)) {

        const float2 R = f2(c0 ? rsqrtf(D2.x) : 0.f, c1 ? rsqrtf(D2.y) : 0.f);
        const float2 R2 = __fmul2_rn(R, R);
        const float2 R3 = __fmul2_rn(R2, R);
        const float2 R5 = __fmul2_rn(R3, R2);
        const float2 QX = __ffma2_rn(f2(q.x), DZ, __ffma2_rn(f2(b.y), DY, __fmul2_rn(f2(b.x), DX)));
        const float2 QY = __ffma2_rn(f2(q.y), DZ, __ffma2_rn(f2(b.w), DY, __fmul2_rn(f2(b.y), DX)));
        const float2 QZ = __ffma2_rn(f2(q.w), DZ, __ffma2_rn(f2(q.y), DY, __fmul2_rn(f2(q.x), DX)));
        const float2 RQR = __ffma2_rn(DZ, QZ, __ffma2_rn(DY, QY, __fmul2_rn(DX, QX)));
        // a = (-M - 2.5 (d.Q.d)/r^4) d/r^3 + (Q.d)/r^5      (physics.py:195-213)
        const float2 S =
            __fmul2_rn(__ffma2_rn(__fmul2_rn(RQR, __fmul2_rn(R2, R2)), f2(-2.5f), f2(-q.z)), R3);
        AX = __ffma2_rn(R5, QX, __ffma2_rn(S, DX, AX));
        AY = __ffma2_rn(R5, QY, __ffma2_rn(S, DY, AY));
        AZ = __ffma2_rn(R5, QZ, __ffma2_rn(S, DZ, AZ));
        pc0 += c0; pc1 += c1;
      }
      const bool o0 = in0 && !c0, o1 = in1 && !c1;  // opened (or bucket-resolved)
      const unsigned b0 = __ballot_sync(0xffffffffu, o0), b1 = __ballot_sync(0xffffffffu, o1);
      if ((b0 | b1) == 0u) continue;
      if (d.z > 0) {  // open: its children become an entry
        if (lane == 0) stk[sp] = make_int4(d.x, d.z, (int)b0, (int)b1);
        ++sp;
      } else if (MODE == kWalkDefer && (d.w & kDeferBit)) {  // subtree not here yet: defer
        if (lane == 0) {
          const unsigned slot = atomicAdd(dfr.count, 1u);
          if (slot < (unsigned)dfr.cap) dfr.out[slot] = make_int4((int)warp, c, (int)b0, (int)b1);
        }
      } else if (BUCKET) {  // bucket rule: pp over its bodies
        // unrolled so the body loads of several iterations are in flight at once
        // (the loop was bound by their latency): walk -4% at cfg2, -6% at cfg3
#pragma unroll(kBucketUnroll)
        for (int j = d.x; j < d.x + cnt; ++j) {
          const float4 bb = bodies[j];
          const float2 EX = __ffma2_rn(f2(bb.x), f2(-1.f), X);
          const float2 EY = __ffma2_rn(f2(bb.y), f2(-1.f), Y);
          const float2 EZ = __ffma2_rn(f2(bb.z), f2(-1.f), Z);
          const float2 Q2 = __ffma2_rn(EZ, EZ, __ffma2_rn(EY, EY, __fmul2_rn(EX, EX)));
          const bool m0 = o0 && Q2.x > 0.f, m1 = o1 && Q2.y > 0.f;
          const float2 W = __fadd2_rn(Q2, E2);
          const float2 R = f2(m0 ? rsqrtf(W.x) : 0.f, m1 ? rsqrtf(W.y) : 0.f);
          const float2 S = __fmul2_rn(__fmul2_rn(R, R), __fmul2_rn(R, f2(-bb.w)));
          AX = __ffma2_rn(S, EX, AX);
          AY = __ffma2_rn(S, EY, AY);
          AZ = __ffma2_rn(S, EZ, AZ);
          pp0 += m0; pp1 += m1;
        }
      }
    }
    if (sp == 0) break;
    __syncwarp();
    e = stk[--sp];
  }
  if (MODE == kWalkResume) {  // add to pass A's results (several entries may share a target)
    const bool u0 = v0 && ((unsigned)entry.z >> lane & 1u), u1 = v1 && ((unsigned)entry.w >> lane & 1u);
    if (u0) {
      float *o = acc + s0 * astride;
      atomicAdd(o, AX.x); atomicAdd(o + 1, AY.x); atomicAdd(o + 2, AZ.x);
      if (work32) atomicAdd(work32 + s0, pp0 + 2 * pc0);
      if (work64) atomicAdd((unsigned long long *)(work64 + s0), (unsigned long long)(pp0 + 2 * pc0));
    }
    if (u1) {
      float *o = acc + s1 * astride;
      atomicAdd(o, AX.y); atomicAdd(o + 1, AY.y); atomicAdd(o + 2, AZ.y);
      if (work32) atomicAdd(work32 + s1, pp1 + 2 * pc1);
      if (work64) atomicAdd((unsigned long long *)(work64 + s1), (unsigned long long)(pp1 + 2 * pc1));
    }
  } else {
    if (v0) {
      float *o = acc + s0 * astride;
      o[0] = AX.x; o[1] = AY.x; o[2] = AZ.x;
      const int w = pp0 + 2 * pc0;  // WORK_PP, WORK_PC (octree.py:23-25)
      if (work64) work64[s0] = w;
      if (work32) work32[s0] = w;
    }
    if (v1) {
      float *o = acc + s1 * astride;
      o[0] = AX.y; o[1] = AY.y; o[2] = AZ.y;
      const int w = pp1 + 2 * pc1;
      if (work64) work64[s1] = w;
      if (work32) work32[s1] = w;
    }
  }
  const unsigned spp = __reduce_add_sync(0xffffffffu, (unsigned)(pp0 + pp1));
  const unsigned spc = __reduce_add_sync(0xffffffffu, (unsigned)(pc0 + pc1));
  if (lane == 0) {
    atomicAdd(&f->pp, (unsigned long long)spp);
    atomicAdd(&f->pc, (unsigned long long)spc);
  }
}

// ------------------------------------------------ group-classified walk (v9)
// Same per-target interaction sets as k_walk, different schedule.  The warp's
// 64 targets have a bounding box [lo, hi].  Because fp32 rounding is monotone,
// evaluating the per-target MAC expression d2 = fma(dz,dz, fma(dy,dy, dx*dx)),
// d = p + a, on the box's nearest / farthest corner bounds every target's d2
// from below / above exactly.  So a cell whose nearest-corner d2 passes the MAC
// is accepted by every target (certain-accept), one whose farthest-corner d2
// fails it is opened by every target (certain-open); only the rest (mixed)
// need the per-target test.  Cells are classified 32 at a time, one per lane,
// taken from a frontier of (first_child, nchild, mask0, mask1) entries:
//   certain-accept -> pc list (the record, masks)      evaluated densely; cells that
//            every target of the warp reached (about half) are listed apart and
//            drained with no masks, predicates or per-entry counters
//   leaf / certain-open bucket -> pp list (lo, count | cell, 0 for a leaf, masks)
//   certain-open internal -> frontier entry (its children, same masks)
//   mixed -> per-target MAC, warp-uniform (as k_walk): pc for the accepting
//            targets now, open / bucket for the others
// The lists are drained (flushed) in tight loops with no tree control, which is
// where the FP32 pipe does its work.  A cell is examined for a target exactly
// when the target opened its parent, as in the reference recursion.
#ifndef BH_W9_FULLMAX
#define BH_W9_FULLMAX 64
#endif
constexpr int kW9Full = BH_W9_FULLMAX;  // full 32-cell batches while sp <= this
// after a full batch sp <= kW9Full + 32; single-entry (DFS) batches above it add
// at most 8 entries per level
constexpr int kW9Frontier = kW9Full + 32 + 8 * (kMaxLevel + 1) + 8;
// Only the top kW9Fcap entries live in shared memory.  Measured peaks are < 100
// entries (cfg2-cfg4: 0 warps above 99), so the proven bound kW9Frontier is
// served by a per-warp spill area in global memory: when a batch could push the
// shared part past kW9Fcap, its bottom kW9Spill entries move out (LIFO order is
// kept), and they move back when the shared part empties.  A warp takes a spill
// slot from a device-wide bitmap on its first spill (<= 64 resident warps per SM,
// so a slot is always free) and returns it at exit.
#ifndef BH_W9_FCAP
#define BH_W9_FCAP 128
#endif
constexpr int kW9Fcap = BH_W9_FCAP;
constexpr int kW9Spill = 64;
static_assert(kW9Fcap >= kW9Spill + 32 && kW9Fcap - kW9Spill <= kW9Spill, "spill layout");
struct W9Spill {
  unsigned *bits = nullptr;  // one bit per slot
  int *fc = nullptr;         // [slot][kW9Frontier]
  uint2 *fm = nullptr;
  int nwords = 0;
};
#ifndef BH_W9_CHECK
#define BH_W9_CHECK 0  // 1: latch FLAG_WALK_BOUNDS instead of overrunning (costs 1.7%; the bounds are proven)
#endif
#ifndef BH_W9_FLUSH
#define BH_W9_FLUSH 20
#endif
#ifndef BH_W9_PPFLUSH
#define BH_W9_PPFLUSH 128
#endif
constexpr int kW9Flush = BH_W9_FLUSH;      // the pc list is drained at >= kW9Flush entries
constexpr int kW9List = kW9Flush + 32;     // a batch adds <= 32
constexpr int kW9PpFlush = BH_W9_PPFLUSH;  // the pp list at >= kW9PpFlush (more buckets to pack)
constexpr int kW9PpList = kW9PpFlush + 32;
#ifndef BH_W9_BLOCK
#define BH_W9_BLOCK 128
#endif
#ifndef BH_W9_MINB
#define BH_W9_MINB 6
#endif
constexpr int kW9Block = BH_W9_BLOCK;
#ifndef BH_W9_PCUNROLL
#define BH_W9_PCUNROLL 4
#endif
constexpr int kW9PcUnroll = BH_W9_PCUNROLL;
#ifndef BH_W9_HALVES
#define BH_W9_HALVES 0  // 1: lane l holds targets (l, l + 32) instead of (2l, 2l + 1); see k_walk9 (measured 1% slower)
#endif
#ifndef BH_W9_PPSTAGE
#define BH_W9_PPSTAGE 0  // 1: pp drain with each pass's bucket bodies staged in shared memory by cp.async.bulk (measured 1% slower)
#endif
#ifndef BH_W9_PPUNROLL
#define BH_W9_PPUNROLL 4  // staged pp passes: body loop unroll (the bodies are LDS reads)
#endif
constexpr int kW9PpUnroll = BH_W9_PPUNROLL;
constexpr int kW9StageF4 = 128;  // BH_W9_PPSTAGE: bodies per staging buffer (2 KB)
constexpr int kW9NcShift = 28;  // frontier entry: first_child | nchild << 28, unsigned (records < 2^28)

#ifndef BH_W9_PPPACK
#define BH_W9_PPPACK 1  // pp drain: buckets with disjoint lane sets share a pass (see flush_pp)
#endif
#ifndef BH_W9_PPPIPE
#define BH_W9_PPPIPE 0  // 1, 2: pp passes load the next (two) pair(s) of bodies first (measured 3-4% slower)
#endif
#ifndef BH_W9_PPPREF
#define BH_W9_PPPREF 0  // 1: pp drain prefetches the next pass's body lines to L1 at the start of a pass (measured neutral)
#endif
#ifndef BH_W9_PPSORT
#define BH_W9_PPSORT 0  // pp drain: pack the buckets longest first (CPU model: 0.64 -> 0.55 of the broadcast iterations)
#endif
#ifdef BH_W9_STATS
// diagnostics (-DBH_W9_STATS): per-warp schedule counters summed over the launch
//  0 batches  1 cells classified  2 mixed  3 mixed with an accepting target
//  4 pc entries flushed  5 their mask bits  6 pp leaf entries  7 their mask bits
//  8 pp bucket entries  9 pp passes  10 pass body iterations  11 bucket (target, body) slots used
//  12 frontier pushes (certain-open)  13 pc flushes  14 pp flushes  15 mixed opened (pushed / bucket)
//  16 mixed accepting target bits  17 bucket entries' mask bits
//  18 pc entries with full masks (unmasked drain)  19 mixed cells accepted by one half only
//  20 pp passes of one half  21 their body iterations
__device__ unsigned long long g_w9_stats[64];  // [32, 64): histogram of the warp's peak frontier depth / 10
extern "C" int bh_debug_w9_stats(unsigned long long *out, int reset) {
  int e = (int)cudaMemcpyFromSymbol(out, g_w9_stats, sizeof(g_w9_stats));
  if (reset) {
    static const unsigned long long z[64] = {};
    cudaMemcpyToSymbol(g_w9_stats, z, sizeof(z));
  }
  return e;
}
#define W9S(i, v) (st[i] += (v))
#else
#define W9S(i, v) ((void)0)
#endif

// cp.async.bulk (the bulk-copy / TMA engine) into shared memory, completing on
// a per-warp mbarrier (BH_W9_PPSTAGE).
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
// one bulk copy (the TMA engine; SASS UBLKCP) of `bytes` (a multiple of 16, both
// addresses 16-byte aligned) into shared memory, completing bytes on `bar`
__device__ __forceinline__ void bulk_copy(void *dst, const void *src, unsigned bytes, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// the phase's one arrival, announcing the bytes its copies will complete
__device__ __forceinline__ void mbar_arrive_expect(uint64_t *bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, unsigned parity) {
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  }
}

// c += (bits != 0) as one predicated add (the compiler's select form is two instructions)
#ifndef BH_W9_CNTASM
#define BH_W9_CNTASM 1
#endif
__device__ __forceinline__ void w9_count(int &c, unsigned bits) {
#if BH_W9_CNTASM
  asm("{ .reg .pred p; setp.ne.u32 p, %1, 0; @p add.s32 %0, %0, 1; }" : "+r"(c) : "r"(bits));
#else
  c += bits != 0u;
#endif
}

// Per-warp shared memory (~7.4 KB).  Masks ride in record words the drains do
// not read: a.w (mac2) and b.z (the duplicate qxy) of a staged pc record, b.z
// and d.w (level) of a staged mixed record.  The pc list has two ends: entries
// that every target of the warp reached (both masks full) fill it from the
// bottom, masked entries from the top (see flush_pc).
struct W9Warp {
  int fc[kW9Fcap];         // frontier (top): first_child | nchild << kW9NcShift
  uint2 fm[kW9Fcap];       //                 (mask0, mask1)
  float4 pcr[kW9List][3];  // accepted cells: a (mask0 in .w), b (mask1 in .z), c with -M in .z
  int4 pp[kW9PpList];      // pp: (lo, count, mask0, mask1) or a leaf record (cell, 0, ...)
#if BH_W9_PPSORT
  uint8_t pord[kW9PpList]; // pp drain: the entries longest bucket first
#endif
  union {
    struct {
      float4 mxr[32][3];   // mixed cells of the batch: a, b (mask0 in .z), c with -M in .z
      int4 mxd[32];        //                           d (mask1 in .w)
    };
    uint8_t psel[32][32];  // pp drain (after the batch): entry + 1 of each lane in each pass
  };
#if BH_W9_PPSTAGE
  // pp drain: two staging buffers of kW9StageF4 bodies, one pass each.  Buffer 0
  // is the (drained) pc list; buffer 1 the second half of the union above plus
  // stg1 (which must follow it directly).
  float4 stg1[kW9StageF4 - 64];
  uint64_t sbar[2];        // one mbarrier per buffer
#endif
};
#if BH_W9_PPSTAGE
static_assert(sizeof(float4) * 3 * kW9List >= sizeof(float4) * kW9StageF4, "staging buffer 0 is the pc list");
static_assert(offsetof(W9Warp, stg1) == offsetof(W9Warp, psel) + 2048, "staging buffer 1 spans the union's tail and stg1");
#endif

__device__ __forceinline__ float w9_shfl_min(float v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v = fminf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ float w9_shfl_max(float v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
// |d| over the box's range of d = p + a (d in [gl, gh]): nearest and farthest
__device__ __forceinline__ void w9_range(float lo, float hi, float a, float &mn, float &mx) {
  const float gl = __fadd_rn(lo, a), gh = __fadd_rn(hi, a);
  mn = gl > 0.f ? gl : (gh < 0.f ? -gh : 0.f);
  mx = fmaxf(fabsf(gl), fabsf(gh));
}

template <bool BUCKET, int MODE>
__global__ void __launch_bounds__(kW9Block, BH_W9_MINB) k_walk9(
    const WalkNode *__restrict__ T, const float4 *__restrict__ bodies,
    const float *__restrict__ targets, int tstride, const uint32_t *__restrict__ tperm, int nt,
    float e2, float *__restrict__ acc, int astride, int64_t *__restrict__ work64,
    int *__restrict__ work32, DeviceFlags *f, int fullmax, DeferArgs dfr, W9Peers peers, W9Spill spl) {
  extern __shared__ int4 w9_smem[];
  W9Warp &S = reinterpret_cast<W9Warp *>(w9_smem)[threadIdx.x >> 5];
  const unsigned lane = threadIdx.x & 31;
  const unsigned FULL = 0xffffffffu;
  const int64_t gwarp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int4 entry = make_int4(0, 0, 0, 0);  // kWalkResume: (target chunk, record, mask0, mask1)
  if (MODE == kWalkResume) {
    if (gwarp >= dfr.nin) return;  // warp-uniform
    entry = dfr.in[gwarp];
  }
  const int64_t warp = MODE == kWalkResume ? (int64_t)entry.x : gwarp;
#if BH_W9_HALVES
  // lane l holds targets l and l + 32 of the warp's 64: the .x and .y halves of
  // the packed math are then the two spatial halves of the group (targets are
  // in curve order), and 17% of the pc entries (6% with the interleaved
  // mapping) are reached by targets of one half only and run as scalar FFMA.
  // But sets of neighbouring targets then occupy twice the lanes, so the pp
  // drain packs fewer buckets per pass (+20% body iterations at cfg3): 1% slower
  // overall, off.
  const int64_t t0 = warp * 64 + lane, t1 = t0 + 32;
#else
  const int64_t t0 = warp * 64 + 2 * lane, t1 = t0 + 1;
#endif
  const bool v0 = t0 < nt, v1 = t1 < nt;
  const int64_t s0 = v0 ? (tperm ? (int64_t)tperm[t0] : t0) : 0;
  const int64_t s1 = v1 ? (tperm ? (int64_t)tperm[t1] : t1) : 0;
  float2 X = f2(0.f), Y = f2(0.f), Z = f2(0.f);
  if (v0) { const float *q = targets + s0 * tstride; X.x = q[0]; Y.x = q[1]; Z.x = q[2]; }
  if (v1) { const float *q = targets + s1 * tstride; X.y = q[0]; Y.y = q[1]; Z.y = q[2]; }
  // the box of the warp's valid targets (lane 0 always has a valid target)
  const float INF = __int_as_float(0x7f800000);
  const float lox = w9_shfl_min(fminf(v0 ? X.x : INF, v1 ? X.y : INF));
  const float loy = w9_shfl_min(fminf(v0 ? Y.x : INF, v1 ? Y.y : INF));
  const float loz = w9_shfl_min(fminf(v0 ? Z.x : INF, v1 ? Z.y : INF));
  const float hix = w9_shfl_max(fmaxf(v0 ? X.x : -INF, v1 ? X.y : -INF));
  const float hiy = w9_shfl_max(fmaxf(v0 ? Y.x : -INF, v1 ? Y.y : -INF));
  const float hiz = w9_shfl_max(fmaxf(v0 ? Z.x : -INF, v1 ? Z.y : -INF));
  float2 AX = f2(0.f), AY = f2(0.f), AZ = f2(0.f);
  int pp0 = 0, pp1 = 0, pc0 = 0, pc1 = 0;
  const float2 E2 = f2(e2);
  const unsigned bit = 1u << lane;
  const unsigned lt = bit - 1u;

  int sp = 1, npf = 0, nph = 0, npp = 0;  // pc entries (every target / masked), pp entries
  int gsp = 0, slot = -1;  // spilled entries, spill slot (warp-uniform)
#ifdef BH_W9_STATS
  unsigned long long st[24] = {};
  int spmax = 0;
#endif
  if (MODE == kWalkResume) {  // the deferred record's subtree, for the targets that opened it
    const int2 fc = dfr.fcnc[entry.y];
    if (fc.y <= 0) sp = 0;
    else if (lane == 0) {
      S.fc[0] = fc_word(fc.x, fc.y);
      S.fm[0] = make_uint2((unsigned)entry.z, (unsigned)entry.w);
    }
  } else {
    const unsigned m0 = __ballot_sync(FULL, v0), m1 = __ballot_sync(FULL, v1);
    if (lane == 0) {  // root internal: start at its children (flattree.py:271-279)
      const int4 rd = T[0].d;
      S.fc[0] = rd.y > 1 ? fc_word(rd.x, rd.z) : fc_word(0, 1);
      S.fm[0] = make_uint2(m0, m1);
    }
  }
#if BH_W9_PPSTAGE
  unsigned sphase = 0;  // bit b: the parity buffer b's barrier completes next
  if (BUCKET && lane == 0) {
    mbar_init(&S.sbar[0], 1);
    mbar_init(&S.sbar[1], 1);
  }
#endif
  __syncwarp();

  // one target's share of a pc entry: the scalar twin of the packed evaluation below
  auto pc_tail = [&](const float4 b, const float4 q, float nm, unsigned ub, float dx, float dy, float dz, float d2,
                     float &ax, float &ay, float &az, int &cnt) {  // nm = -M, ub != 0: the lane's target takes part
    const float r = ub ? rsqrtf(d2) : 0.f;
    const float r2 = __fmul_rn(r, r);
    const float qx = __fmaf_rn(q.x, dz, __fmaf_rn(b.y, dy, __fmul_rn(b.x, dx)));
    const float qy = __fmaf_rn(q.y, dz, __fmaf_rn(b.w, dy, __fmul_rn(b.y, dx)));
    const float qz = __fmaf_rn(q.w, dz, __fmaf_rn(q.y, dy, __fmul_rn(q.x, dx)));
    const float rqr = __fmaf_rn(dz, qz, __fmaf_rn(dy, qy, __fmul_rn(dx, qx)));
    const float r5 = __fmul_rn(__fmul_rn(r2, r2), r);
    const float v = __fmaf_rn(__fmul_rn(rqr, r2), -2.5f, __fmul_rn(nm, d2));
    ax = __fmaf_rn(r5, __fmaf_rn(dx, v, qx), ax);
    ay = __fmaf_rn(r5, __fmaf_rn(dy, v, qy), ay);
    az = __fmaf_rn(r5, __fmaf_rn(dz, v, qz), az);
    w9_count(cnt, ub);
  };
  // dense pc over the list (the FP32-pipe work), two targets per lane: the nf
  // entries at the bottom are reached by every target of the warp (no masks,
  // counted once per flush), the nm entries at the list's top carry masks
  auto pc_eval = [&](const float4 a, const float4 b, const float4 q, const float2 R, const float2 DX, const float2 DY,
                     const float2 DZ, const float2 D2) {
    const float2 R2 = __fmul2_rn(R, R);
    const float2 QX = __ffma2_rn(f2(q.x), DZ, __ffma2_rn(f2(b.y), DY, __fmul2_rn(f2(b.x), DX)));
    const float2 QY = __ffma2_rn(f2(q.y), DZ, __ffma2_rn(f2(b.w), DY, __fmul2_rn(f2(b.y), DX)));
    const float2 QZ = __ffma2_rn(f2(q.w), DZ, __ffma2_rn(f2(q.y), DY, __fmul2_rn(f2(q.x), DX)));
    const float2 RQR = __ffma2_rn(DZ, QZ, __ffma2_rn(DY, QY, __fmul2_rn(DX, QX)));
    // -M d/r^3 + Qd/r^5 - 2.5 (dQd) d/r^7 = r^-5 (Qd + d (-M d2 - 2.5 dQd r^-2)): 30 packed ops (q.z = -M)
    const float2 R5 = __fmul2_rn(__fmul2_rn(R2, R2), R);
    const float2 V = __ffma2_rn(__fmul2_rn(RQR, R2), f2(-2.5f), __fmul2_rn(f2(q.z), D2));
    AX = __ffma2_rn(R5, __ffma2_rn(DX, V, QX), AX);
    AY = __ffma2_rn(R5, __ffma2_rn(DY, V, QY), AY);
    AZ = __ffma2_rn(R5, __ffma2_rn(DZ, V, QZ), AZ);
  };
  auto flush_pc = [&](int nf, int nm) {
    W9S(13, nf + nm > 0); W9S(4, nf + nm); W9S(18, nf);
#ifdef BH_W9_STATS
    W9S(5, 64ull * nf);
    for (int k = kW9List - nm; k < kW9List; ++k)
      W9S(5, __popc((unsigned)__float_as_int(S.pcr[k][0].w)) + __popc((unsigned)__float_as_int(S.pcr[k][1].z)));
#endif
#pragma unroll(kW9PcUnroll)
    for (int k = 0; k < nf; ++k) {
      const float4 a = S.pcr[k][0];
      const float4 b = S.pcr[k][1];
      const float4 q = S.pcr[k][2];
      const float2 DX = __fadd2_rn(X, f2(a.x));
      const float2 DY = __fadd2_rn(Y, f2(a.y));
      const float2 DZ = __fadd2_rn(Z, f2(a.z));
      const float2 D2 = __ffma2_rn(DZ, DZ, __ffma2_rn(DY, DY, __fmul2_rn(DX, DX)));
      pc_eval(a, b, q, f2(rsqrtf(D2.x), rsqrtf(D2.y)), DX, DY, DZ, D2);
    }
    pc0 += nf;
    pc1 += nf;
#pragma unroll(kW9PcUnroll)
    for (int k = kW9List - nm; k < kW9List; ++k) {
      const float4 a = S.pcr[k][0];
      const float4 b = S.pcr[k][1];
      const float4 q = S.pcr[k][2];
      const unsigned ub0 = (unsigned)__float_as_int(a.w) & bit, ub1 = (unsigned)__float_as_int(b.z) & bit;
      const float2 DX = __fadd2_rn(X, f2(a.x));
      const float2 DY = __fadd2_rn(Y, f2(a.y));
      const float2 DZ = __fadd2_rn(Z, f2(a.z));
      const float2 D2 = __ffma2_rn(DZ, DZ, __ffma2_rn(DY, DY, __fmul2_rn(DX, DX)));
      pc_eval(a, b, q, f2(ub0 ? rsqrtf(D2.x) : 0.f, ub1 ? rsqrtf(D2.y) : 0.f), DX, DY, DZ, D2);
      w9_count(pc0, ub0);
      w9_count(pc1, ub1);
    }
  };
  // dense pp over the bodies of the listed leaves / buckets (self skipped by r2 > 0)
  // (E = body - target and +m: the same bits as (target - body) and -m, one negation fewer)
  auto pp_body = [&](const float4 bb, bool u0, bool u1) {
    const float2 EX = __ffma2_rn(X, f2(-1.f), f2(bb.x));
    const float2 EY = __ffma2_rn(Y, f2(-1.f), f2(bb.y));
    const float2 EZ = __ffma2_rn(Z, f2(-1.f), f2(bb.z));
    const float2 Q2 = __ffma2_rn(EZ, EZ, __ffma2_rn(EY, EY, __fmul2_rn(EX, EX)));
    const bool m0 = u0 && Q2.x > 0.f, m1 = u1 && Q2.y > 0.f;
    const float2 W = __fadd2_rn(Q2, E2);
    const float2 R = f2(m0 ? rsqrtf(W.x) : 0.f, m1 ? rsqrtf(W.y) : 0.f);
    const float2 Sc = __fmul2_rn(__fmul2_rn(R, R), __fmul2_rn(R, f2(bb.w)));
    AX = __ffma2_rn(Sc, EX, AX);
    AY = __ffma2_rn(Sc, EY, AY);
    AZ = __ffma2_rn(Sc, EZ, AZ);
    if (m0) ++pp0;
    if (m1) ++pp1;
  };
  auto pp_one = [&](const float4 bb, bool u, float x, float y, float z, float &ax, float &ay, float &az, int &cnt) {
    const float ex = __fsub_rn(bb.x, x), ey = __fsub_rn(bb.y, y), ez = __fsub_rn(bb.z, z);
    const float q2 = __fmaf_rn(ez, ez, __fmaf_rn(ey, ey, __fmul_rn(ex, ex)));
    const bool m = u && q2 > 0.f;
    const float r = m ? rsqrtf(__fadd_rn(q2, e2)) : 0.f;
    const float sc = __fmul_rn(__fmul_rn(r, r), __fmul_rn(r, bb.w));
    ax = __fmaf_rn(sc, ex, ax);
    ay = __fmaf_rn(sc, ey, ay);
    az = __fmaf_rn(sc, ez, az);
    if (m) ++cnt;
  };
  auto flush_pp = [&](int n) {
#if BH_W9_PPSTAGE
    // As the packed drain below (buckets with disjoint lane sets share a pass),
    // and the bodies of a pass reach shared memory by bulk copies (the TMA
    // engine), one per bucket, issued a pass ahead into the other of two
    // staging buffers: the body loop reads shared memory instead of waiting on
    // a global load per cache line.  A pass holds at most kW9StageF4 bodies.
    // The pc list is empty here (buffer 0 is its storage).  Lane p keeps pass
    // p's used lanes, length and staged bodies; a packed entry's .y becomes
    // count | buffer offset << 8.
    W9S(14, n > 0);
    int k0 = 0;
    while (k0 < n) {
      unsigned used = 0u;
      int plen = 0, pf4 = 0, npass = 0, k = k0;
      for (; k < n; ++k) {
        const int4 en = S.pp[k];
        const bool u0 = (unsigned)en.z & bit, u1 = (unsigned)en.w & bit;
        if (en.y == 0) {  // leaf record: its com and mass are the body (a LET leaf has no body index here)
          W9S(6, 1); W9S(7, __popc((unsigned)en.z) + __popc((unsigned)en.w));
          const WalkNode *nd = T + en.x;
          const float4 a = nd->a;
          pp_body(make_float4(-a.x, -a.y, -a.z, nd->c.z), u0, u1);
          continue;
        }
        if (!BUCKET) continue;
        if (en.y > kW9StageF4) {  // a run of equal keys longer than a buffer: straight from global memory
#pragma unroll(kBucketUnroll)
          for (int j = en.x; j < en.x + en.y; ++j) pp_body(bodies[j], u0, u1);
          continue;
        }
        W9S(8, 1); W9S(17, __popc((unsigned)en.z) + __popc((unsigned)en.w));
        W9S(11, (unsigned long long)en.y * (__popc((unsigned)en.z) + __popc((unsigned)en.w)));
        const unsigned lm = (unsigned)en.z | (unsigned)en.w;
        // (a bucket every lane reads shares a pass with nothing: no search)
        const unsigned fit = lm == FULL ? 0u :
            __ballot_sync(FULL, (int)lane < npass && (used & lm) == 0u && pf4 + en.y <= kW9StageF4);
        int p;
        if (fit) {
          p = __ffs(fit) - 1;
        } else {
          if (npass == 32) break;  // run these passes, then pack the rest
          p = npass++;
          S.psel[p][lane] = 0;
        }
        const int off = __shfl_sync(FULL, pf4, p);
        if ((int)lane == p) {
          used |= lm;
          plen = max(plen, en.y);
          pf4 += en.y;
        }
        if (lane == 0) S.pp[k].y = en.y | off << 8;
        if ((lm >> lane) & 1u) S.psel[p][lane] = (uint8_t)(k + 1);
      }
      W9S(9, npass);
      if (BUCKET && npass > 0) {
        auto stage = [&](int b) { return b ? reinterpret_cast<float4 *>(&S.psel[0][0]) + 64 : &S.pcr[0][0]; };
        // the bulk copies of pass p: the first lane of each bucket copies it
        auto issue = [&](int p) {
          __syncwarp();
          fence_proxy_async();  // the buffer's earlier reads and writes precede the copies
          const int e = (int)S.psel[p][lane] - 1;
          uint64_t *bar = &S.sbar[p & 1];
          if (e >= 0) {
            const int4 en = S.pp[e];
            if ((((unsigned)en.z | (unsigned)en.w) & lt) == 0u)
              bulk_copy(stage(p & 1) + (en.y >> 8), bodies + en.x, (unsigned)(en.y & 255) * 16u, bar);
          }
          const int tot = __shfl_sync(FULL, pf4, p);
          if (lane == 0) mbar_arrive_expect(bar, (unsigned)tot * 16u);
        };
        issue(0);
        for (int p = 0; p < npass; ++p) {
          if (p + 1 < npass) issue(p + 1);
          const int len = __shfl_sync(FULL, plen, p);
          W9S(10, len);
          const int e = (int)S.psel[p][lane] - 1;
          const float4 *sb = stage(p & 1);
          int cnt = 0;
          bool u0 = false, u1 = false;
          if (e >= 0) {
            const int4 en = S.pp[e];
            sb += en.y >> 8;
            cnt = en.y & 255;
            u0 = (unsigned)en.z & bit;
            u1 = (unsigned)en.w & bit;
          }
          mbar_wait(&S.sbar[p & 1], sphase >> (p & 1) & 1u);
          sphase ^= 1u << (p & 1);
#pragma unroll(kW9PpUnroll)
          for (int j = 0; j < len; ++j) {
            const bool v = j < cnt;
            pp_body(sb[v ? j : 0], u0 && v, u1 && v);
          }
        }
      }
      __syncwarp();
      k0 = k;
    }
#elif BH_W9_PPPACK
    // Leaf records one at a time (their body is the record); buckets packed:
    // greedy first-fit of the listed buckets into passes whose lane sets
    // (targets 2l, 2l+1 <-> lane l) do not overlap, so one pass over the
    // longest of its buckets serves them all -- each lane follows the one
    // bucket holding its targets (a pass's body loads have one address per
    // bucket).  The interaction sets are unchanged; only the fp32 summation
    // order per target moves.  Lane p keeps pass p's used lanes and length.
    W9S(14, n > 0);
#if BH_W9_PPSORT
    {  // stable rank by bucket length, longest first (leaf records, length 0, last)
      int r0 = 0, r1 = 0, r2 = 0;
      const int c0 = lane < (unsigned)n ? S.pp[lane].y : 0;
      const int c1 = lane + 32 < (unsigned)n ? S.pp[lane + 32].y : 0;
      const int c2 = lane + 64 < (unsigned)n ? S.pp[lane + 64].y : 0;
      for (int f = 0; f < n; ++f) {
        const int cf = S.pp[f].y;
        r0 += cf > c0 || (cf == c0 && f < (int)lane);
        r1 += cf > c1 || (cf == c1 && f < (int)lane + 32);
        r2 += cf > c2 || (cf == c2 && f < (int)lane + 64);
      }
      __syncwarp();
      if (lane < (unsigned)n) S.pord[r0] = (uint8_t)lane;
      if (lane + 32 < (unsigned)n) S.pord[r1] = (uint8_t)(lane + 32);
      if (lane + 64 < (unsigned)n) S.pord[r2] = (uint8_t)(lane + 64);
      __syncwarp();
    }
#endif
    int k0 = 0;
    while (k0 < n) {
      unsigned used = 0u;
      int plen = 0, npass = 0, k = k0;
      for (; k < n; ++k) {
#if BH_W9_PPSORT
        const int ek = S.pord[k];
#else
        const int ek = k;
#endif
        const int4 en = S.pp[ek];
        const bool u0 = (unsigned)en.z & bit, u1 = (unsigned)en.w & bit;
        if (en.y == 0) {  // leaf record: its com and mass are the body (a LET leaf has no body index here)
          W9S(6, 1); W9S(7, __popc((unsigned)en.z) + __popc((unsigned)en.w));
          const WalkNode *nd = T + en.x;
          const float4 a = nd->a;
          pp_body(make_float4(-a.x, -a.y, -a.z, nd->c.z), u0, u1);
          continue;
        }
        W9S(8, 1); W9S(17, __popc((unsigned)en.z) + __popc((unsigned)en.w));
        W9S(11, (unsigned long long)en.y * (__popc((unsigned)en.z) + __popc((unsigned)en.w)));
        const unsigned lm = (unsigned)en.z | (unsigned)en.w;
        const unsigned fit = lm == FULL ? 0u : __ballot_sync(FULL, (int)lane < npass && (used & lm) == 0u);
        int p;
        if (fit) {
          p = __ffs(fit) - 1;
        } else {
          if (npass == 32) break;  // run these passes, then pack the rest
          p = npass++;
          S.psel[p][lane] = 0;
        }
        if ((int)lane == p) {
          used |= lm;
          plen = max(plen, en.y);
        }
        if ((lm >> lane) & 1u) S.psel[p][lane] = (uint8_t)(ek + 1);
      }
      __syncwarp();
      W9S(9, npass);
      for (int p = 0; p < npass; ++p) {
        const int len = __shfl_sync(FULL, plen, p);
        W9S(10, len);
        const int e = (int)S.psel[p][lane] - 1;
        int lo = 0, cnt = 0;
        bool u0 = false, u1 = false;
        if (e >= 0) {
          const int4 en = S.pp[e];
          lo = en.x;
          cnt = en.y;
          u0 = (unsigned)en.z & bit;
          u1 = (unsigned)en.w & bit;
        }
#if BH_W9_PPPIPE == 2
        const float4 *bp = bodies + lo;  // two pairs ahead
        float4 c0 = bp[0], c1 = bp[1 < cnt ? 1 : 0], n0 = bp[2 < cnt ? 2 : 0], n1 = bp[3 < cnt ? 3 : 0];
        for (int j = 0; j < len; j += 2) {
          const float4 m0 = bp[j + 4 < cnt ? j + 4 : 0], m1 = bp[j + 5 < cnt ? j + 5 : 0];
          pp_body(c0, u0 && j < cnt, u1 && j < cnt);
          pp_body(c1, u0 && j + 1 < cnt && j + 1 < len, u1 && j + 1 < cnt && j + 1 < len);
          c0 = n0; c1 = n1; n0 = m0; n1 = m1;
        }
#elif BH_W9_PPPIPE
        // software-pipelined: the next pair of bodies is loaded before the
        // current pair is evaluated (the loop was bound by the load latency)
        const float4 *bp = bodies + lo;
        float4 c0 = bp[0 < cnt ? 0 : 0], c1 = bp[1 < cnt ? 1 : 0];
        for (int j = 0; j < len; j += 2) {
          const float4 n0 = bp[j + 2 < cnt ? j + 2 : 0], n1 = bp[j + 3 < cnt ? j + 3 : 0];
          pp_body(c0, u0 && j < cnt, u1 && j < cnt);
          pp_body(c1, u0 && j + 1 < cnt && j + 1 < len, u1 && j + 1 < cnt && j + 1 < len);
          c0 = n0;
          c1 = n1;
        }
#else
#if BH_W9_PPPREF
        // the next pass's body lines are requested now (prefetch to L1: no
        // register, no wait); the lanes of a bucket take its 128-byte lines in turn
        if (p + 1 < npass) {
          const int e2n = (int)S.psel[p + 1][lane] - 1;
          if (e2n >= 0) {
            const int4 nn = S.pp[e2n];
            const int rk = __popc(((unsigned)nn.z | (unsigned)nn.w) & lt);  // this lane's rank in the bucket's lane set
            if (rk * 8 < nn.y) asm volatile("prefetch.global.L1 [%0];" ::"l"(bodies + nn.x + rk * 8));
          }
        }
#endif
        // a pass whose buckets are read by targets of one half only: scalar
        const bool hx = __any_sync(FULL, u0), hy = __any_sync(FULL, u1);
        // (a lane past its bucket's end re-reads the last body, masked: c0 = c1 = 0 without a bucket)
        const int ilast = lo + max(cnt - 1, 0), c0 = u0 ? cnt : 0, c1 = u1 ? cnt : 0;
        int ib = lo;
        if (hx && hy) {
#pragma unroll(kBucketUnroll)
          for (int j = 0; j < len; ++j) {
            pp_body(bodies[ib], j < c0, j < c1);
            ib = min(ib + 1, ilast);
          }
        } else if (hx) {
          W9S(20, 1); W9S(21, len);
#pragma unroll(kBucketUnroll)
          for (int j = 0; j < len; ++j) {
            pp_one(bodies[ib], j < c0, X.x, Y.x, Z.x, AX.x, AY.x, AZ.x, pp0);
            ib = min(ib + 1, ilast);
          }
        } else {
          W9S(20, 1); W9S(21, len);
#pragma unroll(kBucketUnroll)
          for (int j = 0; j < len; ++j) {
            pp_one(bodies[ib], j < c1, X.y, Y.y, Z.y, AX.y, AY.y, AZ.y, pp1);
            ib = min(ib + 1, ilast);
          }
        }
#endif
      }
      __syncwarp();
      k0 = k;
    }
#else
    for (int k = 0; k < n; ++k) {
      const int4 en = S.pp[k];
      const bool u0 = (unsigned)en.z & bit, u1 = (unsigned)en.w & bit;
      if (en.y == 0) {  // leaf record: its com and mass are the body (a LET leaf has no body index here)
        const WalkNode *nd = T + en.x;
        const float4 a = nd->a;
        pp_body(make_float4(-a.x, -a.y, -a.z, nd->c.z), u0, u1);
        continue;
      }
#pragma unroll(kBucketUnroll)
      for (int j = en.x; j < en.x + en.y; ++j) pp_body(bodies[j], u0, u1);
    }
#endif
  };

  while (sp > 0 || gsp > 0) {
    if (sp > kW9Fcap - 32) {  // a batch pushes <= 32 entries: move the bottom kW9Spill out
      if (slot < 0) {
        if (lane == 0) {
          int w = (int)(gwarp % spl.nwords);
          for (;;) {
            const unsigned v = *((volatile unsigned *)spl.bits + w);
            if (v != FULL) {
              const unsigned b = 1u << (__ffs(~v) - 1);
              if (!(atomicOr(spl.bits + w, b) & b)) {
                slot = w * 32 + __ffs(b) - 1;
                break;
              }
            } else if (++w == spl.nwords) w = 0;
          }
        }
        slot = __shfl_sync(FULL, slot, 0);
      }
      int *gfc = spl.fc + (int64_t)slot * kW9Frontier + gsp;
      uint2 *gfm = spl.fm + (int64_t)slot * kW9Frontier + gsp;
      for (int i = lane; i < kW9Spill; i += 32) { gfc[i] = S.fc[i]; gfm[i] = S.fm[i]; }
      int rfc = 0, rfc2 = 0;
      uint2 rfm = make_uint2(0, 0), rfm2 = make_uint2(0, 0);
      const int rest = sp - kW9Spill;  // <= kW9Spill
      if ((int)lane < rest) { rfc = S.fc[kW9Spill + lane]; rfm = S.fm[kW9Spill + lane]; }
      if ((int)lane + 32 < rest) { rfc2 = S.fc[kW9Spill + 32 + lane]; rfm2 = S.fm[kW9Spill + 32 + lane]; }
      __syncwarp();
      if ((int)lane < rest) { S.fc[lane] = rfc; S.fm[lane] = rfm; }
      if ((int)lane + 32 < rest) { S.fc[32 + lane] = rfc2; S.fm[32 + lane] = rfm2; }
      __syncwarp();
      gsp += kW9Spill;
      sp = rest;
    } else if (sp == 0) {  // shared part empty: the top kW9Spill spilled entries come back
      gsp -= kW9Spill;
      const int *gfc = spl.fc + (int64_t)slot * kW9Frontier + gsp;
      const uint2 *gfm = spl.fm + (int64_t)slot * kW9Frontier + gsp;
      for (int i = lane; i < kW9Spill; i += 32) { S.fc[i] = gfc[i]; S.fm[i] = gfm[i]; }
      __syncwarp();
      sp = kW9Spill;
    }
    // ---- gather up to 32 cells from the top entries (one entry above kW9Full)
    const int ne = sp + gsp <= fullmax ? min(sp, 32) : 1;
    int4 E = make_int4(0, 0, 0, 0);
    if ((int)lane < ne) {
      const int fcnc = S.fc[sp - 1 - lane];
      const uint2 fm = S.fm[sp - 1 - lane];
      E = make_int4(fcnc & ((1 << kW9NcShift) - 1), (int)((unsigned)fcnc >> kW9NcShift), (int)fm.x, (int)fm.y);
    }
    const int nc = (int)lane < ne ? E.y : 0;
    int incl = nc;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(FULL, incl, o);
      if ((int)lane >= o) incl += v;
    }
    const int excl = incl - nc;
    const int take = nc > 0 ? max(0, min(nc, 32 - excl)) : 0;
    const int kfull = __popc(__ballot_sync(FULL, nc > 0 && incl <= 32));  // entries used up
    const int ncell = min(32, __shfl_sync(FULL, incl, ne - 1));
    const unsigned starts = __reduce_or_sync(FULL, take > 0 ? 1u << excl : 0u);
    __syncwarp();
    if ((int)lane == kfull && lane < (unsigned)ne && take > 0)  // partly used: keep the rest
      S.fc[sp - 1 - lane] = fc_word(E.x + take, E.y - take);
    sp -= kfull;
    const int src = __popc(starts & (FULL >> (31 - lane))) - 1;
    const int cfc = __shfl_sync(FULL, E.x, src), cex = __shfl_sync(FULL, excl, src);
    const unsigned m0 = (unsigned)__shfl_sync(FULL, E.z, src), m1 = (unsigned)__shfl_sync(FULL, E.w, src);
    const bool valid = (int)lane < ncell;
    const int cell = cfc + ((int)lane - cex);

    // ---- classify one cell per lane
    bool to_pp = false, to_pc = false, to_fr = false, to_mx = false;
    int4 d = make_int4(0, 0, 0, 0);
    float4 a = make_float4(0.f, 0.f, 0.f, 0.f);
    if (valid) {
      const WalkNode *nd = T + cell;
      a = nd->a;
      d = nd->d;
      if (d.y == 0) {
        // empty tree (no bodies): nothing to interact with
      } else if (d.y == 1) {
        to_pp = true;  // leaf: pp, no MAC (flattree.py:287-294)
      } else {
        float nx, ny, nz, xx, xy, xz;
        w9_range(lox, hix, a.x, nx, xx);
        w9_range(loy, hiy, a.y, ny, xy);
        w9_range(loz, hiz, a.z, nz, xz);
        const float dmin2 = __fmaf_rn(nz, nz, __fmaf_rn(ny, ny, __fmul_rn(nx, nx)));
        const float dmax2 = __fmaf_rn(xz, xz, __fmaf_rn(xy, xy, __fmul_rn(xx, xx)));
        if (dmin2 > a.w) to_pc = true;                      // every target accepts
        else if (!(dmax2 > a.w)) {                          // every target opens
          if (d.z > 0) to_fr = true;
          else if (MODE == kWalkDefer && (d.w & kDeferBit)) {  // subtree not here yet: defer
            const unsigned slot = atomicAdd(dfr.count, 1u);
            if (slot < (unsigned)dfr.cap) dfr.out[slot] = make_int4((int)warp, cell, (int)m0, (int)m1);
          } else to_pp = BUCKET;
        } else to_mx = true;
      }
    }
    const unsigned bpp = __ballot_sync(FULL, to_pp), bpc = __ballot_sync(FULL, to_pc);
    const unsigned bfr = __ballot_sync(FULL, to_fr), bmx = __ballot_sync(FULL, to_mx);
    // the bounds (frontier: §3 of DESIGN.md; lists: < kW9Flush + 32) hold by
    // construction; checked anyway (warp-uniform) so a violation is loud, not a
    // shared-memory overrun
    if (BH_W9_CHECK && (sp + __popc(bfr) + __popc(bmx) > kW9Fcap ||
        gsp + sp + __popc(bfr) + __popc(bmx) > kW9Frontier || npf + nph + __popc(bpc) > kW9List ||
        npp + __popc(bpp) + __popc(bmx) > kW9PpList)) {
      if (lane == 0) {
        atomicOr(&f->bits, FLAG_WALK_BOUNDS);
        if (slot >= 0) atomicAnd(spl.bits + (slot >> 5), ~(1u << (slot & 31)));  // never leak a spill slot
      }
      return;
    }
    if (to_pp) S.pp[npp + __popc(bpp & lt)] = d.y == 1 ? make_int4(cell, 0, (int)m0, (int)m1)
                                                   : make_int4(d.x, d.y, (int)m0, (int)m1);
    // accepted cells that only some of the warp's targets reached: the list's top end (masked drain)
    const unsigned bph = __ballot_sync(FULL, to_pc && (m0 & m1) != FULL);
    if (to_pc) {
      const bool hf = (m0 & m1) != FULL;
      const int slot = hf ? kW9List - 1 - nph - __popc(bph & lt) : npf + __popc(bpc & ~bph & lt);
      float4 b = T[cell].b;
      b.z = __int_as_float((int)m1);
      S.pcr[slot][0] = make_float4(a.x, a.y, a.z, __int_as_float((int)m0));
      S.pcr[slot][1] = b;
      float4 cq = T[cell].c;
      cq.z = -cq.z;  // the drains use -M
      S.pcr[slot][2] = cq;
    }
    if (to_fr) {
      const int slot = sp + __popc(bfr & lt);
      S.fc[slot] = fc_word(d.x, d.z);
      S.fm[slot] = make_uint2(m0, m1);
    }
    if (to_mx) {
      const int slot = __popc(bmx & lt);
      float4 b = T[cell].b;
      b.z = __int_as_float((int)m0);
      S.mxr[slot][0] = a;
      S.mxr[slot][1] = b;
      float4 cq = T[cell].c;
      cq.z = -cq.z;  // -M, as in the pc list
      S.mxr[slot][2] = cq;
      // a deferrable record (pass A) keeps its index, flagged by nchild = -1
      const bool dfr_rec = MODE == kWalkDefer && d.z == 0 && (d.w & kDeferBit);
      S.mxd[slot] = make_int4(dfr_rec ? cell : d.x, d.y, dfr_rec ? -1 : d.z, (int)m1);
    }
    npp += __popc(bpp);
    npf += __popc(bpc & ~bph);
    nph += __popc(bph);
    sp += __popc(bfr);
    const int nmx = __popc(bmx);
    W9S(0, 1); W9S(1, ncell); W9S(2, nmx); W9S(12, __popc(bfr));
#ifdef BH_W9_STATS
    spmax = max(spmax, gsp + sp + nmx);
#endif
    __syncwarp();

    // ---- mixed cells: the per-target MAC (warp-uniform, as k_walk)
    for (int k = 0; k < nmx; ++k) {
      const float4 a = S.mxr[k][0];
      const float4 b = S.mxr[k][1];
      const float4 q = S.mxr[k][2];
      const int4 dd = S.mxd[k];
      const unsigned mb0 = (unsigned)__float_as_int(b.z), mb1 = (unsigned)dd.w;  // the targets that reached the cell
      const float2 DX = __fadd2_rn(X, f2(a.x));
      const float2 DY = __fadd2_rn(Y, f2(a.y));
      const float2 DZ = __fadd2_rn(Z, f2(a.z));
      const float2 D2 = __ffma2_rn(DZ, DZ, __ffma2_rn(DY, DY, __fmul2_rn(DX, DX)));
      const bool c0 = (mb0 & bit) && D2.x > a.w, c1 = (mb1 & bit) && D2.y > a.w;  // MAC (flattree.py:295)
      const unsigned A0 = __ballot_sync(FULL, c0), A1 = __ballot_sync(FULL, c1);  // the accepting targets
      if (A0 && A1) {
        W9S(3, 1); W9S(16, __popc(A0) + __popc(A1));
        const float2 R = f2(c0 ? rsqrtf(D2.x) : 0.f, c1 ? rsqrtf(D2.y) : 0.f);
        const float2 R2 = __fmul2_rn(R, R);
        const float2 QX = __ffma2_rn(f2(q.x), DZ, __ffma2_rn(f2(b.y), DY, __fmul2_rn(f2(b.x), DX)));
        const float2 QY = __ffma2_rn(f2(q.y), DZ, __ffma2_rn(f2(b.w), DY, __fmul2_rn(f2(b.y), DX)));
        const float2 QZ = __ffma2_rn(f2(q.w), DZ, __ffma2_rn(f2(q.y), DY, __fmul2_rn(f2(q.x), DX)));
        const float2 RQR = __ffma2_rn(DZ, QZ, __ffma2_rn(DY, QY, __fmul2_rn(DX, QX)));
        const float2 R5 = __fmul2_rn(__fmul2_rn(R2, R2), R);  // the 30-op form of flush_pc
        const float2 V = __ffma2_rn(__fmul2_rn(RQR, R2), f2(-2.5f), __fmul2_rn(f2(q.z), D2));
        AX = __ffma2_rn(R5, __ffma2_rn(DX, V, QX), AX);
        AY = __ffma2_rn(R5, __ffma2_rn(DY, V, QY), AY);
        AZ = __ffma2_rn(R5, __ffma2_rn(DZ, V, QZ), AZ);
        w9_count(pc0, A0 & bit);
        w9_count(pc1, A1 & bit);
      } else if (A0) {  // accepted by targets of one half only: scalar
        W9S(3, 1); W9S(19, 1); W9S(16, __popc(A0));
        pc_tail(b, q, q.z, A0 & bit, DX.x, DY.x, DZ.x, D2.x, AX.x, AY.x, AZ.x, pc0);
      } else if (A1) {
        W9S(3, 1); W9S(19, 1); W9S(16, __popc(A1));
        pc_tail(b, q, q.z, A1 & bit, DX.y, DY.y, DZ.y, D2.y, AX.y, AY.y, AZ.y, pc1);
      }
      const unsigned o0 = mb0 & ~A0, o1 = mb1 & ~A1;  // the targets that open it
      if ((o0 | o1) == 0u) continue;
      W9S(15, 1);
      if (dd.z > 0) {
        if (lane == 0) {
          S.fc[sp] = fc_word(dd.x, dd.z);
          S.fm[sp] = make_uint2(o0, o1);
        }
        ++sp;
      } else if (MODE == kWalkDefer && dd.z < 0) {
        if (lane == 0) {
          const unsigned slot = atomicAdd(dfr.count, 1u);
          if (slot < (unsigned)dfr.cap) dfr.out[slot] = make_int4((int)warp, dd.x, (int)o0, (int)o1);
        }
      } else if (BUCKET) {
        if (lane == 0) S.pp[npp] = make_int4(dd.x, dd.y, (int)o0, (int)o1);
        ++npp;
      }
    }
    __syncwarp();
#if BH_W9_PPSTAGE
    // the staged pp drain borrows the pc list's storage: drain that first
    if (npf + nph >= kW9Flush || npp >= kW9PpFlush) { flush_pc(npf, nph); npf = nph = 0; }
#else
    if (npf + nph >= kW9Flush) { flush_pc(npf, nph); npf = nph = 0; }
#endif
    if (npp >= kW9PpFlush) { flush_pp(npp); npp = 0; }
    __syncwarp();
  }
  flush_pc(npf, nph);
  flush_pp(npp);

  if (MODE == kWalkResume) {  // add to pass A's results (several entries may share a target)
    const bool u0 = v0 && ((unsigned)entry.z >> lane & 1u), u1 = v1 && ((unsigned)entry.w >> lane & 1u);
    if (u0) {
      float *o = acc + s0 * astride;
      atomicAdd(o, AX.x); atomicAdd(o + 1, AY.x); atomicAdd(o + 2, AZ.x);
      if (work32) atomicAdd(work32 + s0, pp0 + 2 * pc0);
      if (work64) atomicAdd((unsigned long long *)(work64 + s0), (unsigned long long)(pp0 + 2 * pc0));
    }
    if (u1) {
      float *o = acc + s1 * astride;
      atomicAdd(o, AX.y); atomicAdd(o + 1, AY.y); atomicAdd(o + 2, AZ.y);
      if (work32) atomicAdd(work32 + s1, pp1 + 2 * pc1);
      if (work64) atomicAdd((unsigned long long *)(work64 + s1), (unsigned long long)(pp1 + 2 * pc1));
    }
  } else {
    // rows of 4 floats (the resident layout): one 16-byte store per row, so a
    // peer's row travels as one NVLink write (w = 0; nothing reads it)
    const bool row4 = astride == 4;
    const float4 r0 = make_float4(AX.x, AY.x, AZ.x, 0.f), r1 = make_float4(AX.y, AY.y, AZ.y, 0.f);
    if (v0) {
      float *o = acc + s0 * astride;
      if (row4) *reinterpret_cast<float4 *>(o) = r0;
      else { o[0] = AX.x; o[1] = AY.x; o[2] = AZ.x; }
      const int w = pp0 + 2 * pc0;  // WORK_PP, WORK_PC (octree.py:23-25)
      if (work64) work64[s0] = w;
      if (work32) work32[s0] = w;
    }
    if (v1) {
      float *o = acc + s1 * astride;
      if (row4) *reinterpret_cast<float4 *>(o) = r1;
      else { o[0] = AX.y; o[1] = AY.y; o[2] = AZ.y; }
      const int w = pp1 + 2 * pc1;
      if (work64) work64[s1] = w;
      if (work32) work32[s1] = w;
    }
    // replicated ranks: the same rows of every peer's buffers, over NVLink
    // (static indices: the parameter struct is not copied to local memory)
#pragma unroll
    for (int r = 0; r < kMaxPeers; ++r) {
      if (r >= peers.n) break;
      if (v0) {
        float *o = peers.acc[r] + s0 * astride;
        if (row4) *reinterpret_cast<float4 *>(o) = r0;
        else { o[0] = AX.x; o[1] = AY.x; o[2] = AZ.x; }
        if (work32 && peers.work[r]) peers.work[r][s0] = pp0 + 2 * pc0;
      }
      if (v1) {
        float *o = peers.acc[r] + s1 * astride;
        if (row4) *reinterpret_cast<float4 *>(o) = r1;
        else { o[0] = AX.y; o[1] = AY.y; o[2] = AZ.y; }
        if (work32 && peers.work[r]) peers.work[r][s1] = pp1 + 2 * pc1;
      }
    }
    // the peers read these rows after the stream barrier that follows this
    // kernel: make the remote stores visible system-wide first
    if (peers.n > 0) __threadfence_system();
  }
  if (slot >= 0 && lane == 0) atomicAnd(spl.bits + (slot >> 5), ~(1u << (slot & 31)));
  const unsigned spp = __reduce_add_sync(FULL, (unsigned)(pp0 + pp1));
  const unsigned spc = __reduce_add_sync(FULL, (unsigned)(pc0 + pc1));
  if (lane == 0) {
    atomicAdd(&f->pp, (unsigned long long)spp);
    atomicAdd(&f->pc, (unsigned long long)spc);
#ifdef BH_W9_STATS
    for (int i = 0; i < 24; ++i) atomicAdd(&g_w9_stats[i], st[i]);
    atomicAdd(&g_w9_stats[32 + min(31, spmax / 10)], 1ull);
#endif
  }
}

static bool walk9_enabled() {  // BH_WALK_V4=1: the masked-stack walk (k_walk) instead
  static int on = -1;
  if (on < 0) {
    const char *e = getenv("BH_WALK_V4");
    on = (e && *e && *e != '0') ? 0 : 1;
  }
  return on == 1;
}
// full-batch threshold (<= kW9Full, which sizes the frontier); BH_W9_FULL=0 runs
// every batch as one sibling set (the DFS mode the frontier bound rests on)
static int walk9_fullmax() {
  static int v = -1;
  if (v < 0) {
    const char *e = getenv("BH_W9_FULL");
    v = e && *e ? std::max(0, std::min(kW9Full, atoi(e))) : kW9Full;
  }
  return v;
}

__global__ void k_latch_flag(DeviceFlags *f, unsigned bit) { atomicOr(&f->bits, bit); }

// the frontier spill area of the current device (allocated once per device, never freed)
static W9Spill walk9_spill() {
  static W9Spill per_dev[64];
  int dev = 0;
  cudaGetDevice(&dev);
  W9Spill &w = per_dev[dev & 63];
  if (!w.bits) {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int nslot = sms * 64;  // >= resident warps (2048 threads per SM)
    W9Spill t;
    t.nwords = (nslot + 31) / 32;
    if (cudaMalloc(&t.bits, sizeof(unsigned) * t.nwords) != cudaSuccess ||
        cudaMemset(t.bits, 0, sizeof(unsigned) * t.nwords) != cudaSuccess ||
        cudaMalloc(&t.fc, sizeof(int) * (size_t)t.nwords * 32 * kW9Frontier) != cudaSuccess ||
        cudaMalloc(&t.fm, sizeof(uint2) * (size_t)t.nwords * 32 * kW9Frontier) != cudaSuccess)
      return W9Spill{};
    w = t;
  }
  return w;
}

template <bool BUCKET, int MODE>
static void launch_walk9(const WalkNode *T, const float4 *bodies, const float *targets, int tstride,
                         const uint32_t *tperm, int nt, float e2, float *acc, int astride, int64_t *work64,
                         int *work32, DeviceFlags *f, const DeferArgs &dfr, cudaStream_t s,
                         const W9Peers &peers) {
  const size_t smem = sizeof(W9Warp) * (kW9Block / 32);
  static bool init = false;
  if (!init) {
    cudaFuncSetAttribute(k_walk9<BUCKET, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    init = true;
  }
  const int64_t warps = MODE == kWalkResume ? (int64_t)dfr.nin : ((int64_t)nt + 63) / 64;
  if (warps <= 0) return;
  const W9Spill spl = walk9_spill();
  if (!spl.bits) {  // no memory for the spill area: fail loudly at the next check
    k_latch_flag<<<1, 1, 0, s>>>(f, FLAG_WALK_BOUNDS);
    return;
  }
  k_walk9<BUCKET, MODE><<<grid_for(warps * 32, kW9Block), kW9Block, smem, s>>>(
      T, bodies, targets, tstride, tperm, nt, e2, acc, astride, work64, work32, f, walk9_fullmax(), dfr, peers,
      spl);
}
template <int MODE>
static void launch_walk9_mode(const WalkNode *T, const float4 *bodies, const float *targets, int tstride,
                              const uint32_t *tperm, int nt, float e2, int leaf, float *acc, int astride,
                              int64_t *work64, int *work32, DeviceFlags *f, const DeferArgs &dfr, cudaStream_t s,
                              const W9Peers &peers = W9Peers{}) {
  if (leaf > 1)
    launch_walk9<true, MODE>(T, bodies, targets, tstride, tperm, nt, e2, acc, astride, work64, work32, f, dfr, s,
                             peers);
  else
    launch_walk9<false, MODE>(T, bodies, targets, tstride, tperm, nt, e2, acc, astride, work64, work32, f, dfr, s,
                              peers);
}

template <int MODE>
static void launch_walk_mode(const WalkNode *T, const float4 *bodies, const float *targets, int tstride,
                             const uint32_t *tperm, int nt, float e2, int leaf, float *acc, int astride,
                             int64_t *work64, int *work32, DeviceFlags *f, const DeferArgs &dfr, cudaStream_t s) {
  const int64_t warps = MODE == kWalkResume ? (int64_t)dfr.nin : ((int64_t)nt + 63) / 64;
  if (warps <= 0) return;
  const int g = grid_for(warps * 32, kWalkBlock);
  if (leaf > 1)
    k_walk<true, MODE><<<g, kWalkBlock, 0, s>>>(T, bodies, targets, tstride, tperm, nt, e2, leaf, acc, astride,
                                                work64, work32, f, dfr);
  else
    k_walk<false, MODE><<<g, kWalkBlock, 0, s>>>(T, bodies, targets, tstride, tperm, nt, e2, leaf, acc, astride,
                                                 work64, work32, f, dfr);
}

void launch_walk_f32(const WalkNode *T, int64_t nrec_max, const float4 *bodies, const float *targets,
                     int tstride, const uint32_t *tperm, int nt, float e2, int leaf, float *acc, int astride,
                     int64_t *work64, int *work32, DeviceFlags *f, cudaStream_t s, const W9Peers *peers) {
  if (nt <= 0) return;
  if (walk9_enabled() && nrec_max < (int64_t(1) << kW9NcShift)) {  // peers stored by the epilogue
    launch_walk9_mode<kWalkFull>(T, bodies, targets, tstride, tperm, nt, e2, leaf, acc, astride, work64, work32,
                                 f, DeferArgs{}, s, peers ? *peers : W9Peers{});
    return;
  }
  launch_walk_mode<kWalkFull>(T, bodies, targets, tstride, tperm, nt, e2, leaf, acc, astride, work64, work32, f,
                              DeferArgs{}, s);
  if (peers && peers->n > 0) launch_peer_scatter(acc, sizeof(float) * astride, work32, nt, *peers, s);
}

// ------------------------------------------------ target order of the walk
// A warp walks 64 consecutive targets; 64 Morton-consecutive bodies can
// straddle a coarse cell boundary (a jump of the Z curve), which widens the
// group's box: more mixed cells, sparser pc/pp lists.  Inside each chunk of
// 4096 sorted targets (a union of whole sub-cells plus two partial ends) the
// targets are reordered along the Hilbert curve, which has no such jumps
// (CPU model, tools/order_sim.py: -3.5% pc evaluations, -11% mixed cells).
// The interaction sets are unchanged; only the grouping of targets into warps
// (and so the fp32 summation order) moves.
// The curve as a 24-state machine over the Morton digits (octant -> Hilbert
// digit, next state), derived from Skilling's transpose and checked against it
// by tools/hilbert_table.py; one combined byte per (state, octant).
__constant__ uint8_t kHilDigit[24][8] = {{0, 1, 3, 2, 7, 6, 4, 5}, {0, 7, 1, 6, 3, 4, 2, 5}, {0, 3, 7, 4, 1, 2, 6, 5}, {0, 1, 7, 6, 3, 2, 4, 5}, {6, 5, 7, 4, 1, 2, 0, 3}, {6, 1, 7, 0, 5, 2, 4, 3}, {4, 7, 3, 0, 5, 6, 2, 1}, {2, 1, 3, 0, 5, 6, 4, 7}, {6, 7, 5, 4, 1, 0, 2, 3}, {6, 7, 1, 0, 5, 4, 2, 3}, {0, 7, 3, 4, 1, 6, 2, 5}, {0, 3, 1, 2, 7, 4, 6, 5}, {6, 5, 1, 2, 7, 4, 0, 3}, {4, 7, 5, 6, 3, 0, 2, 1}, {2, 1, 5, 6, 3, 0, 4, 7}, {6, 1, 5, 2, 7, 0, 4, 3}, {4, 3, 7, 0, 5, 2, 6, 1}, {4, 5, 7, 6, 3, 2, 0, 1}, {2, 5, 1, 6, 3, 4, 0, 7}, {2, 3, 1, 0, 5, 4, 6, 7}, {4, 3, 5, 2, 7, 0, 6, 1}, {4, 5, 3, 2, 7, 6, 0, 1}, {2, 5, 3, 4, 1, 6, 0, 7}, {2, 3, 5, 4, 1, 0, 6, 7}};
__constant__ uint8_t kHilNext[24][8] = {{1, 3, 15, 0, 20, 21, 10, 0}, {2, 6, 11, 13, 9, 3, 1, 1}, {0, 4, 17, 11, 10, 2, 16, 2}, {10, 0, 16, 17, 5, 3, 1, 3}, {5, 4, 3, 12, 22, 4, 21, 2}, {4, 7, 2, 6, 5, 5, 9, 3}, {7, 8, 13, 19, 6, 10, 6, 16}, {7, 5, 14, 9, 7, 22, 6, 23}, {9, 1, 8, 15, 23, 20, 8, 10}, {8, 10, 19, 16, 9, 5, 9, 1}, {11, 13, 8, 0, 2, 6, 10, 10}, {3, 12, 1, 11, 21, 2, 20, 11}, {15, 12, 18, 12, 0, 4, 17, 11}, {14, 9, 13, 1, 6, 23, 13, 20}, {14, 15, 14, 18, 7, 8, 13, 19}, {12, 14, 15, 15, 11, 13, 8, 0}, {19, 17, 4, 7, 16, 16, 2, 6}, {18, 17, 5, 3, 16, 17, 22, 21}, {18, 18, 12, 14, 19, 17, 4, 7}, {19, 18, 9, 5, 19, 16, 23, 22}, {23, 21, 20, 20, 12, 14, 11, 13}, {22, 21, 20, 21, 15, 0, 18, 17}, {22, 22, 23, 21, 4, 7, 12, 14}, {23, 22, 23, 20, 8, 15, 19, 18}};

// One block of 1024 threads per chunk of 4096 targets, four per thread: the
// Hilbert index from the tree's Morton key (21 table steps), 20 bits of it
// below the chunk's common prefix and the 12-bit chunk position packed in one
// word, sorted by a bitonic network (in-thread for strides >= 1024, shared
// memory for 32..512, shuffles below).  The order only has to preserve
// locality, so the truncated keys are enough.
#ifndef BH_HIL_RADIX
#define BH_HIL_RADIX 1  // 1: 4-pass stable radix, 2: one counting pass on 12 bits (cheaper, loses order: slower walk), 0: bitonic
#endif
constexpr int kHilChunk = 4096;
constexpr int kHilThreads = 1024;
constexpr int kHilPer = kHilChunk / kHilThreads;
#ifndef BH_HIL_MINB
#define BH_HIL_MINB 2
#endif
__device__ __forceinline__ uint64_t hil_spread(uint64_t v) {  // 21 bits -> every third bit
  v &= 0x1fffffull;
  v = (v | v << 32) & 0x1f00000000ffffull;
  v = (v | v << 16) & 0x1f0000ff0000ffull;
  v = (v | v << 8) & 0x100f00f00f00f00full;
  v = (v | v << 4) & 0x10c30c30c30c30c3ull;
  v = (v | v << 2) & 0x1249249249249249ull;
  return v;
}
// Morton key of a target from its position (targets without tree keys: the
// distributed walk's caller arrays); only the order matters, fp32 quantisation
__device__ __forceinline__ uint64_t morton_of_pos(const float4 p, const double *dR) {
  const double R = *dR;
  const float inv = (float)((double)(1 << 21) / (2.0 * R)), fR = (float)R;
  const auto q = [&](float v) { return (uint64_t)fminf(fmaxf(floorf((v + fR) * inv), 0.f), 2097151.f); };
  return hil_spread(q(p.x)) << 2 | hil_spread(q(p.y)) << 1 | hil_spread(q(p.z));
}
__global__ void __launch_bounds__(kHilThreads, BH_HIL_MINB) k_hilbert_chunks(const uint64_t *__restrict__ mkeys, int nt,
                                                                uint32_t *__restrict__ perm,
                                                                const float4 *__restrict__ pos = nullptr,
                                                                const double *__restrict__ dR = nullptr) {
  __shared__ uint32_t sv[kHilChunk];
  __shared__ uint8_t tab[24 * 8];
  __shared__ uint64_t smin[32], smax[32];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  if (tid < 24 * 8) tab[tid] = (uint8_t)(kHilDigit[tid >> 3][tid & 7] << 5 | kHilNext[tid >> 3][tid & 7]);
  __syncthreads();
  const int64_t c0 = (int64_t)blockIdx.x * kHilChunk;
  uint64_t h[kHilPer];
  uint64_t mn = ~0ull, mx = 0ull;
#pragma unroll
  for (int r = 0; r < kHilPer; ++r) {
    const int e = BH_HIL_RADIX ? w * 128 + 32 * r + lane : tid + kHilThreads * r;  // element of item r
    h[r] = 0;
    if (c0 + e < nt) {
      const uint64_t m = mkeys ? mkeys[c0 + e] : morton_of_pos(pos[c0 + e], dR);
      uint64_t k = 0;
      int st = 0;
#pragma unroll
      for (int l = 0; l < kMortonBits; ++l) {
        const uint8_t v = tab[st * 8 + (int)((m >> (3 * (kMortonBits - 1 - l))) & 7)];
        k = k << 3 | (v >> 5);
        st = v & 31;
      }
      h[r] = k;
      mn = k < mn ? k : mn;
      mx = k > mx ? k : mx;
    }
  }
  // the chunk's key range: the bits below its common prefix order it
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const uint64_t a = __shfl_xor_sync(0xffffffffu, mn, o), b = __shfl_xor_sync(0xffffffffu, mx, o);
    mn = a < mn ? a : mn;
    mx = b > mx ? b : mx;
  }
  if (lane == 0) { smin[w] = mn; smax[w] = mx; }
  __syncthreads();
  mn = smin[0];
  mx = smax[0];
  for (int i = 1; i < kHilThreads / 32; ++i) {
    mn = smin[i] < mn ? smin[i] : mn;
    mx = smax[i] > mx ? smax[i] : mx;
  }
  const uint64_t span = mx - mn;  // (every chunk holds a target: mx >= mn)
  const int top = span ? 63 - __clzll((long long)span) : 0;
  const int shift = top > 19 ? top - 19 : 0;
  uint32_t v[kHilPer];
#if BH_HIL_RADIX == 2
  // one counting pass on the top 12 bits below the common prefix (4096 buckets
  // for 4096 targets: a bucket is a tiny region, its internal order is free)
  {
    const int sh12 = top > 11 ? top - 11 : 0;
    for (int b = tid; b < kHilChunk; b += kHilThreads) sv[b] = 0u;
    __syncthreads();
    unsigned bk[kHilPer], rk[kHilPer];
#pragma unroll
    for (int r = 0; r < kHilPer; ++r) {
      const int e = w * 128 + 32 * r + lane;
      bk[r] = c0 + e < nt ? (unsigned)((h[r] - mn) >> sh12) : 0xffffffffu;
      rk[r] = bk[r] != 0xffffffffu ? atomicAdd(&sv[bk[r]], 1u) : 0u;
    }
    __syncthreads();
    // exclusive scan of the 4096 bucket counts: 4 consecutive per thread
    unsigned c[kHilPer], run = 0;
#pragma unroll
    for (int q = 0; q < kHilPer; ++q) { c[q] = sv[tid * kHilPer + q]; run += c[q]; }
    unsigned incl = run;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned x = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= (unsigned)o) incl += x;
    }
    __shared__ unsigned wsum2[32];
    if (lane == 31) wsum2[w] = incl;
    __syncthreads();
    unsigned woff = 0;
    if (lane < (unsigned)w) woff = wsum2[lane];
#pragma unroll
    for (int o = 16; o; o >>= 1) woff += __shfl_xor_sync(0xffffffffu, woff, o);
    unsigned ex = woff + incl - run;
#pragma unroll
    for (int q = 0; q < kHilPer; ++q) { sv[tid * kHilPer + q] = ex; ex += c[q]; }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < kHilPer; ++r) {
      const int e = w * 128 + 32 * r + lane;
      if (c0 + e < nt) perm[c0 + sv[bk[r]] + rk[r]] = (uint32_t)(c0 + e);
    }
    return;
  }
#elif BH_HIL_RADIX
  // stable LSD radix sort of the 20 key bits, 4 passes of 5 bits; element
  // w*128 + 32 r + lane is item r of lane `lane` in warp w (ranks from ballots)
  __shared__ unsigned wh[32][33];  // per warp: digit counts, then offsets
  __shared__ unsigned wtot[32];
#pragma unroll
  for (int r = 0; r < kHilPer; ++r) {
    const int e = w * 128 + 32 * r + lane;
    v[r] = c0 + e < nt ? ((uint32_t)((h[r] - mn) >> shift) << 12) | (uint32_t)e : 0xffffffffu;
  }
  const unsigned lt = (1u << lane) - 1u;
  for (int pass = 0; pass < 4; ++pass) {
    const int sh = 12 + 5 * pass;
    wh[w][lane] = 0u;
    __syncwarp();
    unsigned rk[kHilPer];
#pragma unroll
    for (int r = 0; r < kHilPer; ++r) {
      const unsigned d = (v[r] >> sh) & 31u;
      unsigned peers = 0xffffffffu;
#pragma unroll
      for (int b = 0; b < 5; ++b) match_bit(peers, d, 1u << b);
      const unsigned base = wh[w][d];
      __syncwarp();
      if (lane == 31u - __clz(peers)) wh[w][d] = base + __popc(peers);
      __syncwarp();
      rk[r] = base + __popc(peers & lt);
    }
    __syncthreads();
    // exclusive offsets in (digit, warp) order: thread (d = tid / 32, w' = tid % 32)
    {
      const int d = tid >> 5, ww = tid & 31;
      const unsigned c = wh[ww][d];
      unsigned incl = c;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned x = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= (unsigned)o) incl += x;
      }
      if (lane == 31) wtot[d] = incl;
      __syncthreads();
      unsigned before = 0;
      for (int q = 0; q < d; ++q) before += wtot[q];
      wh[ww][d] = before + incl - c;
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < kHilPer; ++r) sv[wh[w][(v[r] >> sh) & 31u] + rk[r]] = v[r];
    __syncthreads();
#pragma unroll
    for (int r = 0; r < kHilPer; ++r) v[r] = sv[w * 128 + 32 * r + lane];
    __syncthreads();
  }
#pragma unroll
  for (int r = 0; r < kHilPer; ++r) {
    const int e = w * 128 + 32 * r + lane;
    if (c0 + e < nt) perm[c0 + e] = (uint32_t)c0 + (v[r] & (kHilChunk - 1));
  }
  return;
#endif
#pragma unroll
  for (int r = 0; r < kHilPer; ++r) {
    const int e = tid + kHilThreads * r;
    v[r] = c0 + e < nt ? ((uint32_t)((h[r] - mn) >> shift) << 12) | (uint32_t)e : 0xffffffffu;
  }
  for (int k = 2; k <= kHilChunk; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      if (j >= kHilThreads) {  // partners in this thread's registers
        const int rj = j / kHilThreads;
#pragma unroll
        for (int r = 0; r < kHilPer; ++r) {
          if (r & rj) continue;
          const int e = tid + kHilThreads * r;
          const bool up = (e & k) == 0;
          const uint32_t a = v[r], b = v[r | rj];
          v[r] = up ? min(a, b) : max(a, b);
          v[r | rj] = up ? max(a, b) : min(a, b);
        }
        continue;
      }
      uint32_t p[kHilPer];
      if (j >= 32) {
#pragma unroll
        for (int r = 0; r < kHilPer; ++r) sv[tid + kHilThreads * r] = v[r];
        __syncthreads();
#pragma unroll
        for (int r = 0; r < kHilPer; ++r) p[r] = sv[(tid ^ j) + kHilThreads * r];
        __syncthreads();
      } else {
#pragma unroll
        for (int r = 0; r < kHilPer; ++r) p[r] = __shfl_xor_sync(0xffffffffu, v[r], j);
      }
#pragma unroll
      for (int r = 0; r < kHilPer; ++r) {
        const int e = tid + kHilThreads * r;
        const bool up = (e & k) == 0, lower = (e & j) == 0;
        v[r] = (lower == up) ? min(v[r], p[r]) : max(v[r], p[r]);
      }
    }
  }
#pragma unroll
  for (int r = 0; r < kHilPer; ++r) {
    const int e = tid + kHilThreads * r;
    if (c0 + e < nt) perm[c0 + e] = (uint32_t)c0 + (v[r] & (kHilChunk - 1));
  }
}

void launch_hilbert_chunks(const uint64_t *mkeys, int64_t nt, uint32_t *perm, cudaStream_t s) {
  if (nt <= 0) return;
  k_hilbert_chunks<<<(unsigned)((nt + kHilChunk - 1) / kHilChunk), kHilThreads, 0, s>>>(mkeys, (int)nt, perm);
}
void launch_hilbert_chunks_pos(const float4 *pos, int64_t nt, const double *dR, uint32_t *perm, cudaStream_t s) {
  if (nt <= 0) return;
  k_hilbert_chunks<<<(unsigned)((nt + kHilChunk - 1) / kHilChunk), kHilThreads, 0, s>>>(nullptr, (int)nt, perm,
                                                                                       pos, dR);
}

bool walk_hilbert_enabled() {  // BH_WALK_HILBERT=0: Morton-consecutive warps
  static int on = -1;
  if (on < 0) {
    const char *e = getenv("BH_WALK_HILBERT");
    on = (e && *e == '0') ? 0 : 1;
  }
  return on == 1;
}

// rows of the walked range to every peer (the fp64 walk and the v4 fallback):
// 16-byte vector copies, one grid per peer
__global__ void k_peer_scatter(const int4 *__restrict__ src, int64_t n16, int4 *__restrict__ dst) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
  __threadfence_system();  // visible to the peer before the barrier that follows
}
__global__ void k_peer_scatter_i32(const int *__restrict__ src, int64_t n, int *__restrict__ dst) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
  __threadfence_system();
}
void launch_peer_scatter(const void *acc, size_t row_bytes, const int *work, int64_t nt, const W9Peers &p,
                         cudaStream_t s) {
  if (nt <= 0) return;
  const int64_t n16 = nt * (int64_t)row_bytes / 16;
  for (int r = 0; r < p.n; ++r) {
    k_peer_scatter<<<std::min<int64_t>(1184, (n16 + 255) / 256), 256, 0, s>>>(static_cast<const int4 *>(acc), n16,
                                                                            reinterpret_cast<int4 *>(p.acc[r]));
    if (work && p.work[r])
      k_peer_scatter_i32<<<std::min<int64_t>(1184, (nt + 255) / 256), 256, 0, s>>>(work, nt, p.work[r]);
  }
}

void launch_walk_defer_f32(const WalkNode *T, int64_t nrec_max, const float4 *bodies, const float *targets, int nt,
                           float e2, int leaf, float *acc, int *work32, DeviceFlags *f, const DeferArgs &dfr,
                           bool resume, cudaStream_t s, const uint32_t *tperm) {
  if (nt <= 0) return;
  if (walk9_enabled() && nrec_max < (int64_t(1) << kW9NcShift)) {
    if (resume)
      launch_walk9_mode<kWalkResume>(T, bodies, targets, 4, tperm, nt, e2, leaf, acc, 4, nullptr, work32, f, dfr,
                                     s);
    else
      launch_walk9_mode<kWalkDefer>(T, bodies, targets, 4, tperm, nt, e2, leaf, acc, 4, nullptr, work32, f, dfr, s);
    return;
  }
  if (resume)
    launch_walk_mode<kWalkResume>(T, bodies, targets, 4, tperm, nt, e2, leaf, acc, 4, nullptr, work32, f, dfr, s);
  else
    launch_walk_mode<kWalkDefer>(T, bodies, targets, 4, tperm, nt, e2, leaf, acc, 4, nullptr, work32, f, dfr, s);
}

}  // namespace bh
