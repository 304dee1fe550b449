// bh_internal.cuh -- shared declarations of libbh.so (not part of the C-ABI).
//
// Data layout in HBM (all arrays indexed by pre-order cell index c or by
// Morton-sorted body index i):
//
//   bodies  (fp32) float4 {x,y,z,m}          (fp64) double4 {x,y,z,m}
//   keys    u64[n]   sorted 63-bit Morton keys
//   lcp     i8[n]    shared octant levels of (i, i+1)          hashed.py:376-388
//   off     u32[n]   exclusive scan of cells created per body
//   link    int4[C]  {skip, count, lo, level}: skip = index after the subtree
//                    (pre-order), count = bodies below, lo = first sorted body
//   parent  i32[C], child8 i32[C][8] (slot order), level-bucketed cell list
//   cm64    double4[C] {com, mass}, q64 double[C][kQStride] (6 used) fp64 moments
//   wnodes  WalkNode[C'] 64-byte fp32 walk records of the cells a walk with
//                    leaf size L can reach, children contiguous (bh_walk.cu)
//
// The pre-order layout makes the reference's depth-first walk stackless: the
// first child of c is c+1, and "do not descend" is "jump to skip[c]".
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/bh.h"

namespace bh {

constexpr int kMortonBits = 21;
constexpr int kMaxLevel = 21;
constexpr int kWarp = 32;
// quadrupole row stride in doubles: 8 (64-byte aligned rows: whole-sector reads
// and writes; 6 are used)
constexpr int kQStride = 8;

// device error flag bits (latched, reported by bh_check / build)
enum : int {
  FLAG_OUT_OF_DOMAIN = 1,
  FLAG_DUPLICATE = 2,
  FLAG_UNSORTED = 4,
  FLAG_DEPTH = 8,
  FLAG_OVERFLOW = 16,  // sync-free build: more cells than the preallocated capacity
  FLAG_WALK_BOUNDS = 32,  // a walk's per-warp frontier or list would overflow (never, by construction)
};

struct DeviceFlags {
  int bits;
  int pad;
  long long first_bad;  // body index of the first out-of-domain body
  unsigned long long pp;
  unsigned long long pc;
  unsigned int maxabs_bits;  // float bits of max |x| (fp32 bounds)
  int pad2;
  double maxabs64;           // fp64 bounds scratch (as ull bits for atomicMax)
  int ovf_step;              // sync-free build: the step of a bh_sim_step call that overflowed first
  int pad3;
};
// true once a sync-free build of this call has overflowed its capacity: every
// later kernel of the call that reads the tree or moves the state skips, so the
// state is left as the failed step's kick+drift made it (bh_api.cu redoes it)
__device__ __forceinline__ bool overflowed(const DeviceFlags *f) {
  return f && (*reinterpret_cast<const volatile int *>(&f->bits) & FLAG_OVERFLOW);
}

// ---------------------------------------------------------------- buffers
struct Buf {
  void *p = nullptr;
  size_t bytes = 0;
  cudaError_t ensure(size_t want) {
    if (want <= bytes) return cudaSuccess;
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
    size_t grow = want + want / 8 + 256;
    cudaError_t e = cudaMalloc(&p, grow);
    if (e != cudaSuccess) return e;
    bytes = grow;
    // zero once at allocation: the sort / scan look-back words must never hold a
    // stale epoch by accident (bh_sort.cu); everything else overwrites
    return cudaMemset(p, 0, grow);
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
  }
  template <class T>
  T *as() const { return static_cast<T *>(p); }
};

// ---------------------------------------------------------------- kernels
// All launchers enqueue on `s` and never synchronise.

// bounds (morton.py:33-42)
void launch_reset_flags_bounds(DeviceFlags *f, cudaStream_t s);
void launch_maxabs_f32(const float4 *pos, int64_t n, DeviceFlags *f, cudaStream_t s);
void launch_maxabs_f64(const double *pos3, int64_t n, DeviceFlags *f, cudaStream_t s);
void launch_finish_R(const DeviceFlags *f, int fp64, double *d_R, cudaStream_t s);

// keys (morton.py:109-125); vals (if non-null) = iota
void launch_keys_f32(const float4 *pos, int64_t n, const double *d_R, uint64_t *keys,
                     uint32_t *vals, DeviceFlags *f, cudaStream_t s);
void launch_keys_f64(const double *pos, int stride, int64_t n, const double *d_R,
                     uint64_t *keys, uint32_t *vals, DeviceFlags *f, cudaStream_t s);
// keys of arbitrary targets for coherence ordering only (clamped, never flags)
void launch_keys_clamped_f32(const float *pos, int stride, int64_t n, const double *d_R,
                             uint64_t *keys, uint32_t *vals, cudaStream_t s);
void launch_keys_clamped_f64(const double *pos, int stride, int64_t n, const double *d_R,
                             uint64_t *keys, uint32_t *vals, cudaStream_t s);

// tree build (hashed.py:376-515)
void launch_lcp_new(const uint64_t *keys, int64_t n, int8_t *lcp, uint32_t *newc,
                    DeviceFlags *f, int *lvl_cnt, int allow_dup, cudaStream_t s,
                    int bnd_prev = -1, int bnd_next = -1);
struct TreeView {
  int64_t n = 0;       // bodies
  int64_t C = 0;       // cells; with dC set: the allocated capacity (grid bound)
  const int *dC = nullptr;  // sync-free build: the true cell count, on device
  int bnd_prev = -1, bnd_next = -1;  // distributed build: lcp with neighbour ranks
  const uint64_t *keys = nullptr;
  const int8_t *lcp = nullptr;
  const uint32_t *off = nullptr;   // exclusive scan of newc
  const uint32_t *newc = nullptr;
  int4 *link = nullptr;
  int *parent = nullptr;
  int *child8 = nullptr;   // [C][8] child indices in slot order (-1 = absent)
  const float4 *bod32 = nullptr;   // sorted bodies the tree was built from
  const double4 *bod64 = nullptr;
  double4 *cm64 = nullptr;
  double *q64 = nullptr;   // [C][6]
  // fp32 walk-only builds (leaf size mleaf > 1): per-cell class written by the
  // emit kernel -- 0: not a walk record (inside a bucket), 1: a bucket (moments
  // from its bodies), 2 + level: a cell the walk opens, kClassLeafRecord: a
  // one-body walk record (its body is its moments)
  uint8_t *mclass = nullptr;
  int mleaf = 0;
  // and the moments kernel's lists of the opened cells: level counts / offsets /
  // listed counts (3 x 22 ints) and the cell list
  const int *mlvl = nullptr;
  const int *mlist = nullptr;
};
constexpr uint8_t kClassLeafRecord = 255;
void launch_emit(const TreeView &t, const float4 *bod32, const double4 *bod64, cudaStream_t s);
// walk-only trees (t.mclass, 1 < t.mleaf <= 64, fp32 bodies): the two-pass emit
// (scratch: int[n] creator list, counter: one int); no memset of child8 needed.
// Returns false (nothing launched) when the tree is not of that kind.
bool launch_emit_walk(const TreeView &t, const float4 *bod32, int *scratch, int *counter, int sms, cudaStream_t s);
// cursor: int[kMaxLevel+1] scratch; list: int[C]
// Moments: C on device (launch_set_count) or host, per-level counts on device
// (lvl: counts[22] from k_lcp_new | offsets[22] | cursors[22]); one cooperative
// launch sweeps the levels deepest-first with grid-wide barriers between them.
void launch_set_count(const uint32_t *off, const uint32_t *newc, int64_t n, int64_t cap,
                      int *dC, DeviceFlags *f, cudaStream_t s, int step = 0);
// leaf > 1: the fp32 walk tree only (moments of opened cells and buckets; the
// cells inside buckets are skipped), leaf <= 1: every cell (the reference tree)
int launch_moments_coop(const TreeView &t, int *lvl, int *list, int sms, cudaStream_t s, int leaf = 0);
void launch_export(const TreeView &t, double R, uint64_t *key, int8_t *level, double *centre,
                   double *side, double *mass, double *com, double *quad, int64_t *count,
                   int32_t *children, cudaStream_t s);

// traversal (flattree.py:258-317)
struct WalkParams {
  int C;
  int nt;
  float e2f;
  double e2;
  double theta;
  int leaf;            // leaf_size (<=1: reference walk)
  float mac2f[kMaxLevel + 1];   // fp32: (side_l/theta)^2, +inf for theta == 0
  double side64[kMaxLevel + 1]; // fp64: exact side of level l
};
// fp32 walk tree (bh_walk.cu): 64-byte records of the cells a walk with leaf
// size L can reach, each cell's children contiguous, MAC threshold baked in
struct __align__(16) WalkNode {
  float4 a;  // -com.x, -com.y, -com.z, mac2 = (side/theta)^2
  float4 b;  // qxx, qxy, qxy, qyy
  float4 c;  // qxz, qyz, mass, qzz
  int4 d;    // first_child (internal) | lo (bucket/leaf), count, nchild, level
};
// MAC threshold (side_l/theta)^2 per level is formed on device from R
// force (optional): cells always treated as expandable (a rank's shared
// cells); rec_of_cell (optional): walk record index of every kept cell
void launch_walk_tree(const TreeView &t, const double *dR, double theta, int leaf,
                      uint32_t *smask, uint32_t *nck, uint32_t *base, void *scan_tmp,
                      size_t scan_bytes, WalkNode *out, int *dCp, cudaStream_t s,
                      const uint8_t *force = nullptr, int *rec_of_cell = nullptr,
                      int *wparent = nullptr);
// locally essential trees (bh_walk.cu)
void launch_let_mark(const WalkNode *W, int nrec, const int *wparent, const uint8_t *isbranch,
                     const double *boxes, int nbox, int nrank, int self, int *lvl /* 3 x 22 ints */,
                     int *list /* nrec */, int sms, uint32_t *present, uint32_t *expand, uint32_t *bodies,
                     cudaStream_t s);
// all receivers at once: rflag/bcount [nrank][nrec]; after inclusive scans of
// both (rinc/binc), tails[2q..] = receiver q's record and body counts
void launch_let_flags_all(const WalkNode *W, int nrec, const uint8_t *isbranch, const uint32_t *present,
                          const uint32_t *bodies, int nrank, int self, uint32_t *rflag, uint32_t *bcount,
                          cudaStream_t s);
void launch_let_tails(const uint32_t *rinc, const uint32_t *binc, int nrec, int nrank, uint32_t *tails,
                      cudaStream_t s);
void launch_let_pack(const WalkNode *W, int nrec, const uint32_t *expand, const uint32_t *bodies, int q,
                     const uint32_t *rflag, const uint32_t *rinc, const uint32_t *bcount, const uint32_t *binc,
                     const float4 *src_bodies, WalkNode *out, float4 *out_bodies, cudaStream_t s);
void launch_let_branchmap(const WalkNode *W, const int *brec, int nb, int nrec, const uint32_t *expand,
                          const uint32_t *bodies, int q, const uint32_t *rflag, const uint32_t *rinc,
                          const uint32_t *bcount, const uint32_t *binc, int2 *map, cudaStream_t s);
// distributed build
void launch_mark_shared(const TreeView &t, uint8_t *shared, int *branch, int *nbranch,
                        cudaStream_t s);
void launch_branch_export(const TreeView &t, const int *branch, int nb, const int *rec_of_cell,
                          uint64_t *key, int *level, int64_t *count, double *mom, int *rec,
                          int *lo, cudaStream_t s);
// Replicated-tree ranks (SURVEY §8e stage 1): peer ranks' result buffers,
// opened over NVLink (cudaIpcOpenMemHandle), already offset to the walked
// range.  The walk's epilogue stores each target's acceleration and work into
// every peer as well as locally, so no all-reduce follows the walk.
constexpr int kMaxPeers = 7;
// peers &= lanes whose bit `bitmask` of d equals this lane's (one step of a
// ballot match): one bit test feeds the vote and the mask -- 3-4 instructions,
// where `p ? bb : ~bb` in C++ made the compiler derive the predicate twice (~8)
__device__ __forceinline__ void match_bit(unsigned &peers, unsigned d, unsigned bitmask) {
  asm("{ .reg .pred p; .reg .b32 t, m;\n"
      "  and.b32 t, %1, %2; setp.ne.u32 p, t, 0;\n"
      "  vote.sync.ballot.b32 t, p, 0xffffffff;\n"
      "  selp.b32 m, 0xffffffff, 0, p;\n"
      "  xor.b32 t, t, m; not.b32 t, t; and.b32 %0, %0, t; }"
      : "+r"(peers)
      : "r"(d), "r"(bitmask));
}

struct W9Peers {
  int n = 0;
  float *acc[kMaxPeers] = {};
  int *work[kMaxPeers] = {};
};
// copy rows [0, nt) of acc (row_bytes each) and work (int) into every peer
void launch_peer_scatter(const void *acc, size_t row_bytes, const int *work, int64_t nt, const W9Peers &p,
                         cudaStream_t s);
// nrec_max: an upper bound on the records in T (the group-classified walk packs
// record indices in 28 bits; larger trees take the masked-stack walk)
void launch_walk_f32(const WalkNode *T, int64_t nrec_max, const float4 *bodies, const float *targets,
                     int tstride, const uint32_t *tperm, int nt, float e2, int leaf, float *acc, int astride,
                     int64_t *work64, int *work32, DeviceFlags *f, cudaStream_t s,
                     const W9Peers *peers = nullptr);
// Hilbert order of the targets inside each chunk of 4096, from their sorted
// Morton keys (perm: chunk-local permutation of [0, nt), for the walk's
// tperm); BH_WALK_HILBERT=0 disables
void launch_hilbert_chunks(const uint64_t *mkeys, int64_t nt, uint32_t *perm, cudaStream_t s);
// the same from target positions (fp32 quantisation with the handle's R)
void launch_hilbert_chunks_pos(const float4 *pos, int64_t nt, const double *dR, uint32_t *perm, cudaStream_t s);
bool walk_hilbert_enabled();
// deferred walk (LET overlap): pass A appends (target chunk, record, m0, m1) to
// out[cap] for records flagged in d.w; pass B (resume) walks in[nin] with
// fcnc[record] = (first child, nchild) and adds into acc/work atomically
struct DeferArgs {
  int4 *out = nullptr;
  unsigned *count = nullptr;
  int cap = 0;
  const int4 *in = nullptr;
  int nin = 0;
  const int2 *fcnc = nullptr;
};
void launch_walk_defer_f32(const WalkNode *T, int64_t nrec_max, const float4 *bodies, const float *targets, int nt,
                           float e2, int leaf, float *acc, int *work32, DeviceFlags *f, const DeferArgs &dfr,
                           bool resume, cudaStream_t s,
                           const uint32_t *tperm = nullptr);
void launch_walk_f64(const WalkParams &p, const double4 *cm64, const double *q64,
                     const int4 *link, const double4 *bodies, const double *targets,
                     int tstride, const uint32_t *tperm, double *acc, int astride,
                     int64_t *work64, int *work32, DeviceFlags *f, cudaStream_t s);

// integrator (integrator.py:37-44) and body permutation
void launch_kick_f32(float4 *vel, const float4 *acc, int64_t n, float h, cudaStream_t s,
                     const DeviceFlags *skip_on_overflow = nullptr);
void launch_drift_f32(float4 *pos, const float4 *vel, int64_t n, float dt, cudaStream_t s);
void launch_kick_f64(double *vel3, const double *acc3, int64_t n, double h, cudaStream_t s);
void launch_drift_f64(double *pos3, const double *vel3, int64_t n, double dt, cudaStream_t s);
// fused: v += a*h (if kick), x += v*dt, max|x| -> flags (sim path)
void launch_kick_drift_max_f32(float4 *pos, float4 *vel, const float4 *acc, int64_t n,
                               float h, float dt, DeviceFlags *f, cudaStream_t s);
void launch_kick_drift_max_f64(double4 *pos, double4 *vel, const double4 *acc, int64_t n,
                               double h, double dt, DeviceFlags *f, cudaStream_t s);
void launch_kick4_f64(double4 *vel, const double4 *acc, int64_t n, double h, cudaStream_t s);
void launch_gather_f32(const uint32_t *idx, int64_t n, const float4 *a, float4 *a2,
                       const float4 *b, float4 *b2, const uint32_t *id, uint32_t *id2,
                       cudaStream_t s);
void launch_gather_f64(const uint32_t *idx, int64_t n, const double4 *a, double4 *a2,
                       const double4 *b, double4 *b2, const uint32_t *id, uint32_t *id2,
                       cudaStream_t s);
void launch_pack_bodies_f64(const double *pos3, const double *mass, int64_t n, double4 *out,
                            cudaStream_t s);
void launch_iota64(int64_t *out, const uint32_t *vals, int64_t n, cudaStream_t s);

// validation kernels (physics.py:216-285)
void launch_direct_f64(const double *pos3, const double *mass, int64_t n, double eps,
                       double *acc3, cudaStream_t s);
void launch_potential_f64(const double *pos3, const double *mass, int64_t n, double eps,
                          double *partial, cudaStream_t s);

// FFMA throughput microbenchmark (fills *flops with the FP32 flops issued)
void run_ffma(float *out, int sms, int iters, double *flops, cudaStream_t s);
void run_dfma(double *out, int sms, int iters, double *flops, cudaStream_t s);

// radix sort of (key, u32 value) pairs over bits [0, 63) -- stable (bh_sort.cu);
// vin == nullptr sorts (key, input index) pairs without reading values
size_t sort_temp_bytes(int64_t n);
cudaError_t sort_pairs(void *temp, size_t temp_bytes, const uint64_t *kin, uint64_t *kout,
                       const uint32_t *vin, uint32_t *vout, int64_t n, cudaStream_t s);
size_t scan_temp_bytes(int64_t n);
size_t inclusive_scan_temp_bytes(int64_t n);
cudaError_t inclusive_scan_u32(void *temp, size_t temp_bytes, const uint32_t *in, uint32_t *out,
                               int64_t n, cudaStream_t s);
cudaError_t exclusive_scan_u32(void *temp, size_t temp_bytes, const uint32_t *in, uint32_t *out,
                               int64_t n, cudaStream_t s);
int sort_launches();

inline int grid_for(int64_t n, int block) {
  int64_t g = (n + block - 1) / block;
  if (g < 1) g = 1;
  if (g > 0x7fffffff) g = 0x7fffffff;
  return (int)g;
}

}  // namespace bh
