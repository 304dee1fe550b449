// bh_exact.cu -- kernels whose fp64 arithmetic must match the reference bit for
// bit.  This translation unit is compiled with -fmad=false: the reference
// (numpy / numba without fast-math) never contracts a*b+c into an FMA, and one
// contracted d2 flips a MAC decision (SURVEY.md §7 "fp64 bit-exactness").
// Explicit fma() calls below are deliberate (error-free transforms).
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <climits>
#include <cooperative_groups.h>

#include "bh_internal.cuh"

namespace bh {

// ------------------------------------------------------------------ keys
// morton.py:60-68 _spread
__device__ __forceinline__ uint64_t spread21(uint64_t v) {
  v &= 0x1FFFFFull;
  v = (v | (v << 32)) & 0x1F00000000FFFFull;
  v = (v | (v << 16)) & 0x1F0000FF0000FFull;
  v = (v | (v << 8)) & 0x100F00F00F00F00Full;
  v = (v | (v << 4)) & 0x10C30C30C30C30C3ull;
  v = (v | (v << 2)) & 0x1249249249249249ull;
  return v;
}

// morton.py:119-125: floor(((x + R) / (2R)) * 2^21), clipped to [0, 2^21 - 1]
__device__ __forceinline__ uint64_t quantize(double x, double R, double twoR) {
  double s = floor((x + R) / twoR * 2097152.0);
  s = s < 0.0 ? 0.0 : s;
  s = s > 2097151.0 ? 2097151.0 : s;
  return (uint64_t)s;
}

__device__ __forceinline__ uint64_t morton3(double x, double y, double z, double R,
                                            double twoR) {
  return (spread21(quantize(x, R, twoR)) << 2) | (spread21(quantize(y, R, twoR)) << 1) |
         spread21(quantize(z, R, twoR));
}

__device__ __forceinline__ bool in_domain(double x, double R) {
  return (x >= -R) && (x < R);  // morton.py:116: min < -R or max >= R raises
}

template <class Loader>
__global__ void k_keys(Loader ld, int64_t n, const double *__restrict__ d_R,
                       uint64_t *__restrict__ keys, uint32_t *__restrict__ vals,
                       DeviceFlags *f, int check) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double R = *d_R;
  const double twoR = 2.0 * R;
  double x, y, z;
  ld(i, x, y, z);
  if (check && !(in_domain(x, R) && in_domain(y, R) && in_domain(z, R))) {
    atomicOr(&f->bits, FLAG_OUT_OF_DOMAIN);
    atomicMin(&f->first_bad, (long long)i);
  }
  keys[i] = morton3(x, y, z, R, twoR);
  if (vals) vals[i] = (uint32_t)i;
}

struct LoadF4 {
  const float4 *p;
  __device__ void operator()(int64_t i, double &x, double &y, double &z) const {
    float4 v = p[i];
    x = v.x; y = v.y; z = v.z;
  }
};
struct LoadF {
  const float *p; int stride;
  __device__ void operator()(int64_t i, double &x, double &y, double &z) const {
    const float *q = p + i * stride;
    x = q[0]; y = q[1]; z = q[2];
  }
};
struct LoadD {
  const double *p; int stride;
  __device__ void operator()(int64_t i, double &x, double &y, double &z) const {
    const double *q = p + i * stride;
    x = q[0]; y = q[1]; z = q[2];
  }
};

void launch_keys_f32(const float4 *pos, int64_t n, const double *d_R, uint64_t *keys,
                     uint32_t *vals, DeviceFlags *f, cudaStream_t s) {
  if (n <= 0) return;
  k_keys<<<grid_for(n, 256), 256, 0, s>>>(LoadF4{pos}, n, d_R, keys, vals, f, 1);
}
void launch_keys_f64(const double *pos, int stride, int64_t n, const double *d_R,
                     uint64_t *keys, uint32_t *vals, DeviceFlags *f, cudaStream_t s) {
  if (n <= 0) return;
  k_keys<<<grid_for(n, 256), 256, 0, s>>>(LoadD{pos, stride}, n, d_R, keys, vals, f, 1);
}

template <class Loader>
__global__ void k_keys_clamped(Loader ld, int64_t n, const double *__restrict__ d_R,
                               uint64_t *__restrict__ keys, uint32_t *__restrict__ vals) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double R = *d_R;
  double x, y, z;
  ld(i, x, y, z);
  // ordering key only: NaN/out-of-domain targets clamp (quantize clips)
  x = x != x ? 0.0 : x; y = y != y ? 0.0 : y; z = z != z ? 0.0 : z;
  keys[i] = morton3(x, y, z, R, 2.0 * R);
  vals[i] = (uint32_t)i;
}
void launch_keys_clamped_f32(const float *pos, int stride, int64_t n, const double *d_R,
                             uint64_t *keys, uint32_t *vals, cudaStream_t s) {
  if (n <= 0) return;
  k_keys_clamped<<<grid_for(n, 256), 256, 0, s>>>(LoadF{pos, stride}, n, d_R, keys, vals);
}
void launch_keys_clamped_f64(const double *pos, int stride, int64_t n, const double *d_R,
                             uint64_t *keys, uint32_t *vals, cudaStream_t s) {
  if (n <= 0) return;
  k_keys_clamped<<<grid_for(n, 256), 256, 0, s>>>(LoadD{pos, stride}, n, d_R, keys, vals);
}

// ------------------------------------------------------------- tree build
__device__ __forceinline__ int64_t tree_count(const TreeView &t) { return t.dC ? *t.dC : t.C; }

__device__ __forceinline__ double4 ldcg4(const double4 *p) {
  const double2 *q = reinterpret_cast<const double2 *>(p);
  double2 a = __ldcg(q), b = __ldcg(q + 1);
  return make_double4(a.x, a.y, b.x, b.y);
}

// hashed.py:376-388 _lcp_levels: 21 - ceil(bitlen(a ^ b) / 3)
__device__ __forceinline__ int lcp_of(uint64_t a, uint64_t b) {
  // kMortonBits - ceil(bits / 3) with bits = the position of the highest
  // differing bit + 1, written on 32-bit halves (the 64-bit clz and the
  // division compiled to twice the instructions): for x != 0 it is
  // 20 - p / 3 with p the highest set bit, and p / 3 = (43 p) >> 7 for p < 64
  const uint64_t x = a ^ b;
  const uint32_t hi = (uint32_t)(x >> 32), lo = (uint32_t)x;
  if (x == 0) return kMortonBits;
  const int p = hi ? 63 - __clz((int)hi) : 31 - __clz((int)lo);
  return kMortonBits - 1 - ((p * 43) >> 7);
}
static_assert(kMortonBits == 21, "lcp_of: 21 levels of 3 bits");

// hashed.py:475-489: sortedness / duplicate checks, lcp, depth, cells per body.
// newc[i] = depth[i] - start[i] with start = lcp[i-1] (0 for i = 0).
// Also counts the internal cells each level will hold (levels start+1 ..
// depth-1 of every body; the last created cell is the body's leaf) so that the
// level-synchronous moments launches can be sized on the host.
// allow_dup (bucket mode, SURVEY.md §7 "Duplicate keys"): bodies with equal
// keys cannot be separated; they share one level-21 cell (count = run length)
// that is never opened and is resolved body by body.  The reference raises
// instead (hashed.py:477-482), which is what allow_dup = 0 reproduces.
// bnd_prev / bnd_next (>= 0 on a rank of a distributed build): shared octant
// levels of the first / last local key with the neighbouring rank's last / first
// key, so leaves sit at their global depth (the reference inserts the
// neighbour bodies for the same purpose, hashed.py:539-602).
__global__ void k_lcp_new(const uint64_t *__restrict__ keys, int64_t n,
                          int8_t *__restrict__ lcp, uint32_t *__restrict__ newc,
                          DeviceFlags *f, int *__restrict__ lvl_cnt, int allow_dup,
                          int bnd_prev, int bnd_next) {
  __shared__ int h[kMaxLevel + 2];
  if (threadIdx.x <= kMaxLevel + 1) h[threadIdx.x] = 0;
  __syncthreads();
  // grid-stride: the per-level counts leave each block once (global atomics on
  // 22 addresses from every block of a one-body-per-thread grid serialise in L2)
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
  uint64_t k = keys[i];
  int lp = -1, ln = -1;
  if (i > 0) lp = lcp_of(keys[i - 1], k);
  if (i + 1 < n) {
    uint64_t kn = keys[i + 1];
    if (kn < k) atomicOr(&f->bits, FLAG_UNSORTED);
    if (kn == k && !allow_dup) atomicOr(&f->bits, FLAG_DUPLICATE);
    ln = lcp_of(k, kn);
    lcp[i] = (int8_t)ln;
  }
  int depth = (lp > ln ? lp : ln) + 1;
  if (depth > kMaxLevel) {
    if (allow_dup) depth = kMaxLevel;
    else atomicOr(&f->bits, FLAG_DEPTH);
  }
  const int depth_local = depth;  // cells above it hold >= 2 local bodies
  if (i == 0 && bnd_prev >= 0) depth = max(depth, min(bnd_prev + 1, kMaxLevel));
  if (i == n - 1 && bnd_next >= 0) depth = max(depth, min(bnd_next + 1, kMaxLevel));
  int start = i > 0 ? lp : 0;
  newc[i] = (uint32_t)(depth - start);
  for (int l = start + 1; l < depth_local && l <= kMaxLevel; ++l) atomicAdd(&h[l], 1);
  if (ln == kMaxLevel && lp < kMaxLevel) atomicAdd(&h[kMaxLevel], 1);  // duplicate-run cell
  }
  __syncthreads();
  if (threadIdx.x == 0 && blockIdx.x == 0) atomicAdd(&h[0], n > 1 ? 1 : 0);  // the root
  __syncthreads();
  if (threadIdx.x <= kMaxLevel && h[threadIdx.x]) atomicAdd(&lvl_cnt[threadIdx.x], h[threadIdx.x]);
}

void launch_lcp_new(const uint64_t *keys, int64_t n, int8_t *lcp, uint32_t *newc,
                    DeviceFlags *f, int *lvl_cnt, int allow_dup, cudaStream_t s, int bnd_prev,
                    int bnd_next) {
  if (n <= 0) return;
  cudaMemsetAsync(lvl_cnt, 0, sizeof(int) * (kMaxLevel + 1), s);
  static int g = 0;
  if (g == 0) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    g = sms * 8;
  }
  const int blocks = (int)std::min<int64_t>(g, (n + 255) / 256);
  k_lcp_new<<<blocks, 256, 0, s>>>(keys, n, lcp, newc, f, lvl_cnt, allow_dup, bnd_prev, bnd_next);
}

// first b > i whose level-l prefix differs from body i's (n if none):
// galloping then bisection over the sorted keys.
__device__ __forceinline__ int64_t run_end(const uint64_t *__restrict__ keys, int64_t n,
                                           int64_t i, uint64_t pref, int shift) {
  int64_t lo = i, step = 1;
  while (lo + step < n && (keys[lo + step] >> shift) == pref) {
    lo += step;
    step <<= 1;
  }
  int64_t hi = lo + step < n ? lo + step : n;
  while (hi - lo > 1) {
    int64_t mid = lo + ((hi - lo) >> 1);
    if ((keys[mid] >> shift) == pref) lo = mid; else hi = mid;
  }
  return hi;
}

// first b <= i whose level-l prefix equals body i's
__device__ __forceinline__ int64_t run_begin(const uint64_t *__restrict__ keys, int64_t i,
                                             uint64_t pref, int shift) {
  int64_t hi = i, step = 1;
  while (hi - step >= 0 && (keys[hi - step] >> shift) == pref) {
    hi -= step;
    step <<= 1;
  }
  int64_t lo = hi - step >= 0 ? hi - step : -1;  // lo differs (or -1)
  while (hi - lo > 1) {
    int64_t mid = lo + ((hi - lo) >> 1);
    if ((keys[mid] >> shift) == pref) hi = mid; else lo = mid;
  }
  return hi;
}

// hashed.py:391-441 _build_kernel, in parallel: body i creates the cells of
// levels start+1..depth[i]; their pre-order indices are 1 + off[i] + k.  The
// parent of the first of them is the level-`start` cell holding body i, created
// by the first body j of that run.
__global__ void k_emit(TreeView t, const float4 *__restrict__ bod32,
                       const double4 *__restrict__ bod64) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t n = t.n;
  if (i >= n) return;
  const int C = (int)tree_count(t);
  if (C > t.C) return;  // sync-free build overflowed its capacity (flagged; redone)
  const int L = t.mleaf;
  if (i == 0) {
    t.link[0] = make_int4(C, (int)n, 0, 0);
    t.parent[0] = -1;
    if (t.mclass) t.mclass[0] = n > 1 ? 2 : 0;  // the walk opens a root holding > 1 body
    if (n == 1 && t.bnd_prev < 0 && t.bnd_next < 0) {  // hashed.py:464-474: root = leaf
      double4 b;
      if (bod64) {
        b = bod64[0];
      } else {
        float4 v = bod32[0];
        b = make_double4(v.x, v.y, v.z, v.w);
      }
      t.cm64[0] = b;
      return;
    }
  }
  const uint64_t k = t.keys[i];
  const int lp = i > 0 ? t.lcp[i - 1] : -1;
  const int ln = i + 1 < n ? t.lcp[i] : -1;
  int depth = min((lp > ln ? lp : ln) + 1, kMaxLevel);  // clamp: duplicate keys
  if (i == 0 && t.bnd_prev >= 0) depth = max(depth, min(t.bnd_prev + 1, kMaxLevel));
  if (i == n - 1 && t.bnd_next >= 0) depth = max(depth, min(t.bnd_next + 1, kMaxLevel));
  const int start = i > 0 ? lp : 0;
  const int base = 1 + (int)t.off[i];
  int par = 0;
  bool par_open = n > 1;  // walk-only builds: does the walk open the parent of the next cell?
  if (start > 0) {
    const int shift = 3 * (kMortonBits - start);
    const int64_t j = run_begin(t.keys, i, k >> shift, shift);
    const int startj = j > 0 ? t.lcp[j - 1] : 0;
    par = 1 + (int)t.off[j] + (start - startj - 1);
    // the level-`start` parent holds the run from body j: more than L bodies iff
    // body j + L still shares its prefix
    if (t.mclass) par_open = j + L < n && (t.keys[j + L] >> shift) == (k >> shift);
  }
  if (t.mclass) {
    // Walk-only tree (fp32 sim path, leaf size L > 1): only what the walk reads
    // is written -- the cells the walk opens, its buckets and one-body records.
    // A cell below a bucket is never read: the body stops at its first such
    // cell (its class byte stays 0 from the memset), so the deep part of the
    // tree costs no stores and no run-end searches.  parent[] is not needed.
    for (int l = start + 1; l <= depth; ++l) {
      if (!par_open) break;  // inside a bucket
      const int c = base + (l - start - 1);
      const bool leafc = l == depth && ln != kMaxLevel;
      t.child8[8 * (int64_t)par + (int)((k >> (3 * (kMortonBits - l))) & 7)] = leafc ? -(c + 2) : c;
      if (l == depth && ln == kMaxLevel) {  // first body of a duplicate-key run: a bucket
        const int64_t end = run_end(t.keys, n, i, k, 0);
        const int skip = end < n ? 1 + (int)t.off[end] : C;
        t.link[c] = make_int4(skip, (int)(end - i), (int)i, l);
        t.mclass[c] = 1;
        break;
      }
      if (leafc) {  // a one-body record: its body is its moments
        t.link[c] = make_int4(c + 1, 1, (int)i, l);
        t.mclass[c] = kClassLeafRecord;
        const float4 v = bod32[i];
        t.cm64[c] = make_double4(v.x, v.y, v.z, v.w);
        break;
      }
      const int shift = 3 * (kMortonBits - l);
      const int64_t end = run_end(t.keys, n, i, k >> shift, shift);
      const int skip = end < n ? 1 + (int)t.off[end] : C;
      t.link[c] = make_int4(skip, (int)(end - i), (int)i, l);
      const bool opens = end - i > L;  // l < 21 here
      t.mclass[c] = opens ? (uint8_t)(2 + l) : 1;
      par_open = opens;
      par = c;
    }
    return;
  }
  for (int l = start + 1; l <= depth; ++l) {
    const int c = base + (l - start - 1);
    t.parent[c] = par;
    // a leaf child is stored as -(c + 2): the moments read no link word for it
    const bool leafc = l == depth && ln != kMaxLevel;
    t.child8[8 * (int64_t)par + (int)((k >> (3 * (kMortonBits - l))) & 7)] = leafc ? -(c + 2) : c;
    if (l == depth && ln == kMaxLevel) {  // first body of a duplicate-key run
      const int64_t end = run_end(t.keys, n, i, k, 0);
      const int skip = end < n ? 1 + (int)t.off[end] : C;
      t.link[c] = make_int4(skip, (int)(end - i), (int)i, l);
    } else if (l == depth) {
      t.link[c] = make_int4(c + 1, 1, (int)i, l);
      double4 b;
      if (bod64) {
        b = bod64[i];
      } else {
        float4 v = bod32[i];
        b = make_double4(v.x, v.y, v.z, v.w);
      }
      t.cm64[c] = b;
    } else {
      const int shift = 3 * (kMortonBits - l);
      const int64_t end = run_end(t.keys, n, i, k >> shift, shift);
      const int skip = end < n ? 1 + (int)t.off[end] : C;
      t.link[c] = make_int4(skip, (int)(end - i), (int)i, l);
    }
    par = c;
  }
}

void launch_emit(const TreeView &t, const float4 *bod32, const double4 *bod64,
                 cudaStream_t s) {
  if (t.n <= 0) return;
  k_emit<<<grid_for(t.n, 128), 128, 0, s>>>(t, bod32, bod64);
}

// ---- walk-only emit in two passes (fp32 sim path, leaf size 1 < L <= 64)
// Only ~15% of the bodies create a cell the walk reads (the first body of each
// walk record), and each of them searches the sorted keys for run ends -- long
// chains of dependent loads.  Pass 1 finds them without a search and lists
// them densely; pass 2 runs the searches for the listed bodies only.
//   The level-l cell holding body i has more than L bodies iff some window of
// L + 1 consecutive sorted bodies containing i shares its level-l prefix, i.e.
// iff l <= maxW(i) = max over a in [i - L, i] of lcp(keys[a], keys[a + L]).
// So body i creates walk records iff its first new cell's parent (level
// start = lcp[i-1]) is opened -- start <= maxW(i), or the root (n > 1) -- and
// its new cell at level l is opened iff l <= maxW(i).  Pass 1 also sets the
// child rows of the opened cells it will create to -1 (absent), so the tree
// needs no memset of the full child8 array (32 B per cell).
constexpr int kEmitThreads = 256;
constexpr int kEmitHalo = 64;  // >= L
__global__ void __launch_bounds__(kEmitThreads) k_emit_mark(TreeView t, const float4 *__restrict__ bod32,
                                                            int *__restrict__ creators, int *__restrict__ ncreators) {
  __shared__ uint64_t ks[kEmitThreads + 2 * kEmitHalo];
  // W as 16-bit values, read two at a time: the window maximum below is packed
  // (VIMNMX3.S16x2); byte reads with their sign extensions were 4 instructions
  // per element, 132 per body at L = 32
  __shared__ __align__(8) int16_t ws[kEmitThreads + kEmitHalo + 2];
  const int64_t n = t.n;
  const int C = (int)tree_count(t);
  if (C > t.C) return;  // sync-free build overflowed its capacity (flagged; redone)
  const int L = t.mleaf;
  const int64_t b0 = (int64_t)blockIdx.x * kEmitThreads;
  for (int k = threadIdx.x; k < kEmitThreads + 2 * kEmitHalo; k += kEmitThreads) {
    const int64_t g = b0 - kEmitHalo + k;  // ks[k] = keys[b0 - H + k]
    ks[k] = g >= 0 && g < n ? t.keys[g] : 0ull;
  }
  __syncthreads();
  for (int k = threadIdx.x; k < kEmitThreads + kEmitHalo; k += kEmitThreads) {
    const int64_t a = b0 - kEmitHalo + k;  // ws[k] = W(a), -1 without a full window
    ws[k] = (int16_t)(a >= 0 && a + L < n ? lcp_of(ks[k], ks[k + L]) : -1);
  }
  __syncthreads();
  const int64_t i = b0 + threadIdx.x;
  bool creator = false;
  if (i < n) {
    const int li = threadIdx.x + kEmitHalo;
    if (i == 0) {
      t.link[0] = make_int4(C, (int)n, 0, 0);
      if (t.parent) t.parent[0] = -1;
      t.mclass[0] = n > 1 ? 2 : 0;  // the walk opens a root holding > 1 body
      if (n > 1) {
        int4 *row = reinterpret_cast<int4 *>(t.child8);
        row[0] = row[1] = make_int4(-1, -1, -1, -1);
      }
      if (n == 1 && t.bnd_prev < 0 && t.bnd_next < 0) {  // hashed.py:464-474: root = leaf
        const float4 v = bod32[0];
        t.cm64[0] = make_double4(v.x, v.y, v.z, v.w);
      }
    }
    // lcp with the neighbours from the staged keys (= t.lcp, hashed.py:376-388)
    const int lp = i > 0 ? lcp_of(ks[li - 1], ks[li]) : -1;
    const int ln = i + 1 < n ? lcp_of(ks[li], ks[li + 1]) : -1;
    int depth = min((lp > ln ? lp : ln) + 1, kMaxLevel);
    if (i == 0 && t.bnd_prev >= 0) depth = max(depth, min(t.bnd_prev + 1, kMaxLevel));
    if (i == n - 1 && t.bnd_next >= 0) depth = max(depth, min(t.bnd_next + 1, kMaxLevel));
    const int start = i > 0 ? lp : 0;
    // max of W over the elements [li - L, li]; -1 (0xffff) is the identity
    const unsigned *w32 = reinterpret_cast<const unsigned *>(ws);
    const int wlo = li - L, wa = wlo >> 1, wb = li >> 1;
    unsigned acc = w32[wa];
    if (wlo & 1) acc |= 0x0000ffffu;                   // element wlo - 1 is outside
    unsigned last = w32[wb];
    if (!(li & 1)) last |= 0xffff0000u;                // element li + 1 is outside
    acc = wa == wb ? (acc | (last & 0xffff0000u)) : __vmaxs2(acc, last);
    for (int q = wa + 1; q < wb; q += 2)
      acc = __vimax3_s16x2(acc, w32[q], q + 1 < wb ? w32[q + 1] : 0xffffffffu);
    const int maxw = max((int)(short)(acc & 0xffffu), (int)(short)(acc >> 16));
    creator = n > 1 && (start == 0 || start <= maxw);
    if (creator) {  // the rows of the opened cells this body creates: all slots absent
      const int base = 1 + (int)t.off[i];
      int4 *row = reinterpret_cast<int4 *>(t.child8);
      for (int l = start + 1; l <= depth && l <= maxw && l < kMaxLevel; ++l) {
        if (l == depth) break;  // the body's last cell is a leaf or a duplicate-key bucket
        const int64_t c = base + (l - start - 1);
        row[2 * c] = row[2 * c + 1] = make_int4(-1, -1, -1, -1);
      }
    }
  }
  // densely list the creators: one global atomic per block (one per warp was
  // ~300K same-address atomics at 1e7 bodies, serialised in L2)
  __shared__ int wcnt[kEmitThreads / 32];
  __shared__ int bbase;
  const unsigned m = __ballot_sync(0xffffffffu, creator);
  const unsigned lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) wcnt[w] = __popc(m);
  __syncthreads();
  if (threadIdx.x == 0) {
    int tot = 0;
    for (int q = 0; q < kEmitThreads / 32; ++q) {
      const int c = wcnt[q];
      wcnt[q] = tot;
      tot += c;
    }
    bbase = tot ? atomicAdd(ncreators, tot) : 0;
  }
  __syncthreads();
  if (creator) creators[bbase + wcnt[w] + __popc(m & ((1u << lane) - 1u))] = (int)i;
}

__global__ void __launch_bounds__(128) k_emit_create(TreeView t, const float4 *__restrict__ bod32,
                                                     const int *__restrict__ creators,
                                                     const int *__restrict__ ncreators) {
  const int64_t n = t.n;
  const int C = (int)tree_count(t);
  if (C > t.C) return;
  const int L = t.mleaf;
  const int nc = *ncreators;
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < nc; q += gridDim.x * blockDim.x) {
    const int64_t i = creators[q];
    const uint64_t k = t.keys[i];
    const int lp = i > 0 ? t.lcp[i - 1] : -1;
    const int ln = i + 1 < n ? t.lcp[i] : -1;
    int depth = min((lp > ln ? lp : ln) + 1, kMaxLevel);
    if (i == 0 && t.bnd_prev >= 0) depth = max(depth, min(t.bnd_prev + 1, kMaxLevel));
    if (i == n - 1 && t.bnd_next >= 0) depth = max(depth, min(t.bnd_next + 1, kMaxLevel));
    const int start = i > 0 ? lp : 0;
    const int base = 1 + (int)t.off[i];
    int par = 0;
    if (start > 0) {
      const int shift = 3 * (kMortonBits - start);
      const int64_t j = run_begin(t.keys, i, k >> shift, shift);
      const int startj = j > 0 ? t.lcp[j - 1] : 0;
      par = 1 + (int)t.off[j] + (start - startj - 1);
    }
    for (int l = start + 1; l <= depth; ++l) {
      const int c = base + (l - start - 1);
      const bool leafc = l == depth && ln != kMaxLevel;
      t.child8[8 * (int64_t)par + (int)((k >> (3 * (kMortonBits - l))) & 7)] = leafc ? -(c + 2) : c;
      if (l == depth && ln == kMaxLevel) {  // first body of a duplicate-key run: a bucket
        const int64_t end = run_end(t.keys, n, i, k, 0);
        const int skip = end < n ? 1 + (int)t.off[end] : C;
        t.link[c] = make_int4(skip, (int)(end - i), (int)i, l);
        t.mclass[c] = 1;
        break;
      }
      if (leafc) {  // a one-body record: its body is its moments
        t.link[c] = make_int4(c + 1, 1, (int)i, l);
        t.mclass[c] = kClassLeafRecord;
        const float4 v = bod32[i];
        t.cm64[c] = make_double4(v.x, v.y, v.z, v.w);
        break;
      }
      const int shift = 3 * (kMortonBits - l);
      // more than L bodies iff body i + L still shares the prefix (l < 21 here)
      const bool opens = i + L < n && (t.keys[i + L] >> shift) == (k >> shift);
      int64_t end;
      if (opens) {
        end = run_end(t.keys, n, i + L, k >> shift, shift);
      } else {  // <= L bodies: a short forward probe
        int64_t e = i + 1;
        while (e < n && e <= i + L && (t.keys[e] >> shift) == (k >> shift)) ++e;
        end = e;
      }
      const int skip = end < n ? 1 + (int)t.off[end] : C;
      t.link[c] = make_int4(skip, (int)(end - i), (int)i, l);
      t.mclass[c] = opens ? (uint8_t)(2 + l) : 1;
      if (!opens) break;
      par = c;
    }
  }
}

bool launch_emit_walk(const TreeView &t, const float4 *bod32, int *scratch, int *counter, int sms, cudaStream_t s) {
  if (t.n <= 0 || !t.mclass || !bod32 || t.mleaf <= 1 || t.mleaf > kEmitHalo) return false;
  cudaMemsetAsync(counter, 0, sizeof(int), s);
  k_emit_mark<<<(unsigned)((t.n + kEmitThreads - 1) / kEmitThreads), kEmitThreads, 0, s>>>(t, bod32, scratch, counter);
  // one thread per creator for up to n / 4 of them (measured ~15%: the searches
  // are latency chains, so they want many threads, not a few long loops)
  const int64_t g = std::max<int64_t>(sms * 16, (t.n / 4 + 127) / 128);
  k_emit_create<<<(unsigned)g, 128, 0, s>>>(t, bod32, scratch, counter);
  return true;
}

// a sorted body as (x, y, z, m) in double
__device__ __forceinline__ double4 body64(const TreeView &t, int64_t j) {
  if (t.bod64) return t.bod64[j];
  const float4 v = t.bod32[j];
  return make_double4(v.x, v.y, v.z, v.w);
}

// Moments of a level-21 cell holding bodies with identical keys (bucket mode
// only): the same combine as _moments_kernel with the bodies, in sorted order,
// as leaf children.  Mirrored by the extended oracle (oracle/bh_oracle.c).
__device__ void dup_cell_moments(const TreeView &t, int p) {
  const int4 L = t.link[p];
  double total = 0.0, cx = 0.0, cy = 0.0, cz = 0.0;
  for (int j = L.z; j < L.z + L.y; ++j) {
    const double4 b = body64(t, j);
    if (b.w == 0.0) continue;
    total += b.w;
    cx += b.w * b.x;
    cy += b.w * b.y;
    cz += b.w * b.z;
  }
  double2 *q2o = reinterpret_cast<double2 *>(t.q64 + kQStride * (int64_t)p);
  if (total == 0.0) {
    t.cm64[p] = make_double4(0.0, 0.0, 0.0, 0.0);
    q2o[0] = q2o[1] = q2o[2] = make_double2(0.0, 0.0);
    return;
  }
  cx /= total;
  cy /= total;
  cz /= total;
  double qxx = 0.0, qxy = 0.0, qxz = 0.0, qyy = 0.0, qyz = 0.0, qzz = 0.0;
  for (int j = L.z; j < L.z + L.y; ++j) {
    const double4 b = body64(t, j);
    const double m = b.w;
    if (m == 0.0) continue;
    double dx = b.x - cx, dy = b.y - cy, dz = b.z - cz;
    double d2 = dx * dx + dy * dy + dz * dz;
    qxx += 0.0 + m * (3.0 * (dx * dx) - d2);
    qxy += 0.0 + m * (3.0 * (dx * dy) - 0.0);
    qxz += 0.0 + m * (3.0 * (dx * dz) - 0.0);
    qyy += 0.0 + m * (3.0 * (dy * dy) - d2);
    qyz += 0.0 + m * (3.0 * (dy * dz) - 0.0);
    qzz += 0.0 + m * (3.0 * (dz * dz) - d2);
  }
  t.cm64[p] = make_double4(cx, cy, cz, total);
  q2o[0] = make_double2(qxx, qxy);
  q2o[1] = make_double2(qxz, qyy);
  q2o[2] = make_double2(qyz, qzz);
}

// flattree.py:201-252 _moments_kernel for one cell, with one lane per child
// slot (8 lanes per cell, 4 cells per warp): the child loads of a cell go out
// in parallel from 8 lanes, and the slot-ordered sums -- the reference's exact
// expression order -- are formed from a per-warp shared-memory exchange.  Each
// lane forms its child's products (m*x, and q_c + m*(3 dx dx - d2)); the sums
// are sequential in slot order, skipping absent and massless children.
// Every lane of the warp must call it (p < 0: no cell).  xs: the warp's [32][11].
__device__ void cell_moments8(const TreeView &t, int p, double (*xs)[11]) {
  const int lane = threadIdx.x & 31, s = lane & 7, g0 = lane & ~7;
  int c = -1;
  bool leafc = false;
  if (p >= 0) {
    c = t.child8[8 * (int64_t)p + s];
    leafc = c < -1;  // leaf child, stored as -(c + 2)
    if (leafc) c = -c - 2;
  }
  const unsigned have = (__ballot_sync(0xffffffffu, c >= 0) >> g0) & 0xffu;
  const bool cell = p >= 0 && have != 0u;
  if (p >= 0 && have == 0u && s == 0) dup_cell_moments(t, p);  // duplicate-key cell
  double4 cm = make_double4(0.0, 0.0, 0.0, 0.0);
  bool hasq = false;
  if (c >= 0) {
    cm = t.cm64[c];
    hasq = !leafc;  // leaves keep quad = 0 (flattree.py:207-208); other cells hold > 1 body
  }
  const double m = cm.w;
  const bool use = c >= 0 && m != 0.0;
  double *mine = xs[lane];
  mine[0] = use ? 1.0 : 0.0;
  mine[1] = m;
  mine[2] = m * cm.x;
  mine[3] = m * cm.y;
  mine[4] = m * cm.z;
  __syncwarp();
  double total = 0.0, cx = 0.0, cy = 0.0, cz = 0.0;
  for (int j = 0; j < 8; ++j) {
    const double *o = xs[g0 + j];
    if (o[0] == 0.0) continue;
    total += o[1];
    cx += o[2];
    cy += o[3];
    cz += o[4];
  }
  double t0 = 0.0, t1 = 0.0, t2 = 0.0, t3 = 0.0, t4 = 0.0, t5 = 0.0;
  if (cell && total != 0.0) {
    cx /= total;
    cy /= total;
    cz /= total;
    if (use) {
      double q0 = 0.0, q1 = 0.0, q2 = 0.0, q3 = 0.0, q4 = 0.0, q5 = 0.0;
      if (hasq) {
        const double2 *qc = reinterpret_cast<const double2 *>(t.q64 + kQStride * (int64_t)c);
        const double2 a = qc[0], b = qc[1], d = qc[2];
        q0 = a.x; q1 = a.y; q2 = b.x; q3 = b.y; q4 = d.x; q5 = d.y;
      }
      const double dx = cm.x - cx, dy = cm.y - cy, dz = cm.z - cz;
      const double d2 = dx * dx + dy * dy + dz * dz;
      t0 = q0 + m * (3.0 * (dx * dx) - d2);
      t1 = q1 + m * (3.0 * (dx * dy) - 0.0);
      t2 = q2 + m * (3.0 * (dx * dz) - 0.0);
      t3 = q3 + m * (3.0 * (dy * dy) - d2);
      t4 = q4 + m * (3.0 * (dy * dz) - 0.0);
      t5 = q5 + m * (3.0 * (dz * dz) - d2);
    }
  }
  __syncwarp();
  mine[5] = t0; mine[6] = t1; mine[7] = t2; mine[8] = t3; mine[9] = t4; mine[10] = t5;
  __syncwarp();
  if (cell && s == 0) {
    double *qo = t.q64 + kQStride * (int64_t)p;
    if (total == 0.0) {
      t.cm64[p] = make_double4(0.0, 0.0, 0.0, 0.0);
      for (int k = 0; k < 6; ++k) qo[k] = 0.0;
    } else {
      double qxx = 0.0, qxy = 0.0, qxz = 0.0, qyy = 0.0, qyz = 0.0, qzz = 0.0;
      for (int j = 0; j < 8; ++j) {
        const double *o = xs[g0 + j];
        if (o[0] == 0.0) continue;
        qxx += o[5]; qxy += o[6]; qxz += o[7]; qyy += o[8]; qyz += o[9]; qzz += o[10];
      }
      t.cm64[p] = make_double4(cx, cy, cz, total);
      double2 *q2o = reinterpret_cast<double2 *>(qo);
      q2o[0] = make_double2(qxx, qxy);
      q2o[1] = make_double2(qxz, qyy);
      q2o[2] = make_double2(qyz, qzz);
      q2o[3] = make_double2(0.0, 0.0);  // pad: whole-sector write
    }
  }
  __syncwarp();
}

// fp32 walk trees only (leaf size L > 1): the moments of a bucket -- a cell the
// walk never opens (count <= L, or a level-21 duplicate-key cell) whose parent
// it does open -- straight from its <= L contiguous sorted bodies, 8 lanes per
// cell (strided bodies, fixed-order butterfly sums).  The cells inside buckets
// are never read by the walk, so their moments are not formed at all.  Equal
// to the recursive combine up to fp64 rounding (the records are rounded to
// fp32).  Every lane of the warp must call it (p < 0: no cell).
#ifdef BH_MOM_TIMERS
// diagnostics (-DBH_MOM_TIMERS): %globaltimer at each phase boundary of the last
// k_moments_coop launch ([0] start, [1] lists, [2] buckets, [3 + i] after level run i)
__device__ unsigned long long g_mom_t[64];
__device__ int g_mom_nt;
extern "C" int bh_debug_mom_timers(unsigned long long *out, int *n) {
  cudaMemcpyFromSymbol(n, g_mom_nt, sizeof(int));
  return (int)cudaMemcpyFromSymbol(out, g_mom_t, sizeof(g_mom_t));
}
__device__ __forceinline__ void mom_mark(int i) {
  if (blockIdx.x == 0 && threadIdx.x == 0 && i < 64) {
    unsigned long long v;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(v));
    g_mom_t[i] = v;
    g_mom_nt = i + 1;
  }
}
#define MOM_MARK(i) mom_mark(i)
#else
#define MOM_MARK(i) ((void)0)
#endif

#ifndef BH_BUCKET_ONEPASS
#define BH_BUCKET_ONEPASS 1
#endif
__device__ void bucket_moments8(const TreeView &t, int p) {
  const int s = threadIdx.x & 7;
  int lo = 0, cnt = 0;
  if (p >= 0) {
    const int4 L = t.link[p];
    lo = L.z;
    cnt = L.y;
  }
#if BH_BUCKET_ONEPASS
  // One read of the bodies: mass, first and second moments about the bucket's
  // first body x0 (offsets are bucket-sized, so the shift to the centre of mass
  // below cancels nothing large), then the central quadrupole
  // Q_ab = 3 S_ab - delta_ab tr S with S = sum m r r^T - M c c^T, c = com - x0.
  // every body load of the cell is issued before any arithmetic (one memory
  // round trip, not one per strided step); cells of more than 32 bodies
  // (duplicate-key cells) finish in a loop
  double4 x0 = make_double4(0.0, 0.0, 0.0, 0.0);
  double tm = 0.0, sx = 0.0, sy = 0.0, sz = 0.0;
  double sxx = 0.0, syy = 0.0, szz = 0.0, sxy = 0.0, sxz = 0.0, syz = 0.0;
  auto add = [&](const double4 b) {
    const double dx = b.x - x0.x, dy = b.y - x0.y, dz = b.z - x0.z;
    const double mx = b.w * dx, my = b.w * dy, mz = b.w * dz;
    tm += b.w;
    sx += mx; sy += my; sz += mz;
    sxx += mx * dx; syy += my * dy; szz += mz * dz;
    sxy += mx * dy; sxz += mx * dz; syz += my * dz;
  };
#ifdef BH_MOM_TIMERS
  if (p >= 0 && s == 0) {
    atomicAdd(&g_mom_t[60], (unsigned long long)cnt);
    atomicMax(&g_mom_t[61], (unsigned long long)cnt);
  }
#endif
#if defined(BH_BUCKET_DIAG) && BH_BUCKET_DIAG == 1  // timing only: skip the bucket entirely
  return;
#endif
  if (t.bod64) {
    if (cnt > 0) x0 = t.bod64[lo];
    for (int j = s; j < cnt; j += 8) add(t.bod64[lo + j]);
  } else {
    float4 v[4];
    const float4 v0 = cnt > 0 ? t.bod32[lo] : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int q = 0; q < 4; ++q) v[q] = s + 8 * q < cnt ? t.bod32[lo + s + 8 * q] : make_float4(0.f, 0.f, 0.f, 0.f);
    x0 = make_double4(v0.x, v0.y, v0.z, v0.w);
    // absent slots have zero mass: they add exactly 0
#pragma unroll
    for (int q = 0; q < 4; ++q) add(make_double4(v[q].x, v[q].y, v[q].z, v[q].w));
    for (int j = s + 32; j < cnt; j += 8) {
      const float4 f = t.bod32[lo + j];
      add(make_double4(f.x, f.y, f.z, f.w));
    }
  }
#if defined(BH_BUCKET_DIAG) && BH_BUCKET_DIAG == 2  // timing only: no reduction
  if (0)
#endif
#pragma unroll
  for (int o = 1; o < 8; o <<= 1) {
    tm += __shfl_xor_sync(0xffffffffu, tm, o);
    sx += __shfl_xor_sync(0xffffffffu, sx, o);
    sy += __shfl_xor_sync(0xffffffffu, sy, o);
    sz += __shfl_xor_sync(0xffffffffu, sz, o);
    sxx += __shfl_xor_sync(0xffffffffu, sxx, o);
    syy += __shfl_xor_sync(0xffffffffu, syy, o);
    szz += __shfl_xor_sync(0xffffffffu, szz, o);
    sxy += __shfl_xor_sync(0xffffffffu, sxy, o);
    sxz += __shfl_xor_sync(0xffffffffu, sxz, o);
    syz += __shfl_xor_sync(0xffffffffu, syz, o);
  }
  if (p >= 0 && s == 0) {
    double cx = 0.0, cy = 0.0, cz = 0.0;
    double q0 = 0.0, q1 = 0.0, q2 = 0.0, q3 = 0.0, q4 = 0.0, q5 = 0.0;
    if (tm != 0.0) {
      cx = sx / tm; cy = sy / tm; cz = sz / tm;
      const double Sxx = sxx - tm * cx * cx, Syy = syy - tm * cy * cy, Szz = szz - tm * cz * cz;
      const double tr = Sxx + Syy + Szz;
      q0 = 3.0 * Sxx - tr;
      q1 = 3.0 * (sxy - tm * cx * cy);
      q2 = 3.0 * (sxz - tm * cx * cz);
      q3 = 3.0 * Syy - tr;
      q4 = 3.0 * (syz - tm * cy * cz);
      q5 = 3.0 * Szz - tr;
      cx += x0.x; cy += x0.y; cz += x0.z;
    }
    t.cm64[p] = make_double4(cx, cy, cz, tm);
    double2 *q2o = reinterpret_cast<double2 *>(t.q64 + kQStride * (int64_t)p);
    q2o[0] = make_double2(q0, q1);
    q2o[1] = make_double2(q2, q3);
    q2o[2] = make_double2(q4, q5);
    q2o[3] = make_double2(0.0, 0.0);
  }
#else
  double tm = 0.0, sx = 0.0, sy = 0.0, sz = 0.0;
  for (int j = s; j < cnt; j += 8) {
    const double4 b = body64(t, lo + j);
    tm += b.w;
    sx += b.w * b.x;
    sy += b.w * b.y;
    sz += b.w * b.z;
  }
#pragma unroll
  for (int o = 1; o < 8; o <<= 1) {
    tm += __shfl_xor_sync(0xffffffffu, tm, o);
    sx += __shfl_xor_sync(0xffffffffu, sx, o);
    sy += __shfl_xor_sync(0xffffffffu, sy, o);
    sz += __shfl_xor_sync(0xffffffffu, sz, o);
  }
  double cx = 0.0, cy = 0.0, cz = 0.0;
  if (tm != 0.0) {
    cx = sx / tm;
    cy = sy / tm;
    cz = sz / tm;
  }
  double q0 = 0.0, q1 = 0.0, q2 = 0.0, q3 = 0.0, q4 = 0.0, q5 = 0.0;
  for (int j = s; j < cnt && tm != 0.0; j += 8) {
    const double4 b = body64(t, lo + j);
    const double dx = b.x - cx, dy = b.y - cy, dz = b.z - cz;
    const double d2 = dx * dx + dy * dy + dz * dz;
    q0 += b.w * (3.0 * (dx * dx) - d2);
    q1 += b.w * (3.0 * (dx * dy));
    q2 += b.w * (3.0 * (dx * dz));
    q3 += b.w * (3.0 * (dy * dy) - d2);
    q4 += b.w * (3.0 * (dy * dz));
    q5 += b.w * (3.0 * (dz * dz) - d2);
  }
#pragma unroll
  for (int o = 1; o < 8; o <<= 1) {
    q0 += __shfl_xor_sync(0xffffffffu, q0, o);
    q1 += __shfl_xor_sync(0xffffffffu, q1, o);
    q2 += __shfl_xor_sync(0xffffffffu, q2, o);
    q3 += __shfl_xor_sync(0xffffffffu, q3, o);
    q4 += __shfl_xor_sync(0xffffffffu, q4, o);
    q5 += __shfl_xor_sync(0xffffffffu, q5, o);
  }
  if (p >= 0 && s == 0) {
    t.cm64[p] = make_double4(cx, cy, cz, tm);
    double2 *q2o = reinterpret_cast<double2 *>(t.q64 + kQStride * (int64_t)p);
    q2o[0] = make_double2(q0, q1);
    q2o[1] = make_double2(q2, q3);
    q2o[2] = make_double2(q4, q5);
    q2o[3] = make_double2(0.0, 0.0);
  }
#endif
}

// the fp32 walk opens a cell iff count > L (the root: count > 1) below level 21
__device__ __forceinline__ bool walk_opens(int64_t c, int4 L, int leaf) {
  return (L.y > leaf || (c == 0 && L.y > 1)) && L.w < kMaxLevel;
}

// C = 1 + off[n-1] + newc[n-1] on device; flag an overflow of the capacity
__global__ void k_set_count(const uint32_t *off, const uint32_t *newc, int64_t n, int64_t cap,
                            int *dC, DeviceFlags *f, int step) {
  int64_t C = n > 0 ? 1 + (int64_t)off[n - 1] + newc[n - 1] : 1;
  if (C > cap && !(f->bits & FLAG_OVERFLOW)) {  // the first overflow of the call: remember its step
    f->ovf_step = step;
    __threadfence();
    atomicOr(&f->bits, FLAG_OVERFLOW);
  }
  dC[0] = (int)C;
}
void launch_set_count(const uint32_t *off, const uint32_t *newc, int64_t n, int64_t cap,
                      int *dC, DeviceFlags *f, cudaStream_t s, int step) {
  k_set_count<<<1, 1, 0, s>>>(off, newc, n, cap, dC, f, step);
}

// Walk-only trees (fp32 sim path, L > 1): list the opened cells by level and
// the buckets (from the end of `list`) from the emit kernel's class bytes, then
// form the bucket moments -- two plain launches ahead of the level sweep.
__global__ void __launch_bounds__(256) k_mom_lists(TreeView t, int *__restrict__ lvl, int *__restrict__ list) {
  const int64_t C = tree_count(t);
  if (C > t.C) return;
  int *cnt = lvl, *offsg = lvl + (kMaxLevel + 1), *cur = lvl + 2 * (kMaxLevel + 1);
  int *nbuck = lvl + 3 * (kMaxLevel + 1);
  __shared__ int offs[kMaxLevel + 1];
  __shared__ int h[kMaxLevel + 1], base[kMaxLevel + 1];
  __shared__ int hb, bbase;
  if (threadIdx.x == 0) {
    int acc = 0;
    for (int l = 0; l <= kMaxLevel; ++l) {
      offs[l] = acc;
      if (blockIdx.x == 0) offsg[l] = acc;
      acc += cnt[l];
    }
  }
  __syncthreads();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    // walk-only tree: the emit kernel classified every cell (one byte each);
    // 16 cells per thread and pass (one 16-byte read; 4 per pass spent its time
    // in the three block barriers of a pass)
    constexpr int kPer = 16;
    for (int64_t c0 = (int64_t)blockIdx.x * blockDim.x * kPer; c0 < C; c0 += stride * kPer) {
      if (threadIdx.x <= kMaxLevel) h[threadIdx.x] = 0;
      if (threadIdx.x == 0) hb = 0;
      __syncthreads();
      const int64_t cb = c0 + kPer * (int64_t)threadIdx.x;
      uint32_t w[kPer / 4] = {};
      if (cb + kPer <= C) {
        const uint4 v = *reinterpret_cast<const uint4 *>(t.mclass + cb);
        w[0] = v.x; w[1] = v.y; w[2] = v.z; w[3] = v.w;
      } else {
        for (int q = 0; q < kPer; ++q)
          if (cb + q < C) w[q >> 2] |= (uint32_t)t.mclass[cb + q] << (8 * (q & 3));
      }
      int rank[kPer];
#pragma unroll
      for (int q = 0; q < kPer; ++q) {
        const unsigned cl = (w[q >> 2] >> (8 * (q & 3))) & 255u;
        rank[q] = -1;  // opened cell: rank in its level's list; bucket: -2 - rank
        if (cl >= 2 && cl != kClassLeafRecord) rank[q] = atomicAdd(&h[cl - 2], 1);
        else if (cl == 1) rank[q] = -2 - atomicAdd(&hb, 1);
      }
      __syncthreads();
      if (threadIdx.x <= kMaxLevel && h[threadIdx.x])
        base[threadIdx.x] = offs[threadIdx.x] + atomicAdd(&cur[threadIdx.x], h[threadIdx.x]);
      if (threadIdx.x == 0 && hb) bbase = atomicAdd(nbuck, hb);
      __syncthreads();
#pragma unroll
      for (int q = 0; q < kPer; ++q) {
        const unsigned cl = (w[q >> 2] >> (8 * (q & 3))) & 255u;
        if (rank[q] >= 0) list[base[cl - 2] + rank[q]] = (int)(cb + q);
        else if (rank[q] <= -2) list[C - 1 - (bbase + (-2 - rank[q]))] = (int)(cb + q);
      }
      __syncthreads();
    }
}

__global__ void __launch_bounds__(256) k_bucket_moments(TreeView t, const int *__restrict__ lvl,
                                                        const int *__restrict__ list) {
  const int64_t C = tree_count(t);
  if (C > t.C) return;
  const int nb = lvl[3 * (kMaxLevel + 1)];
  const int sub = (threadIdx.x & 31) >> 3;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t b0 = warp * 4; b0 < nb; b0 += nwarps * 4) {
    const int64_t k = b0 + sub;
    bucket_moments8(t, k < nb ? list[C - 1 - k] : -1);
  }
}

// One cooperative launch (all blocks co-resident): offsets from the device
// level counts, bucket the internal cells by level, then sweep the levels
// deepest-first with a grid-wide barrier between levels (a cell's children are
// one level deeper, hence final when its level runs).
namespace cg = cooperative_groups;
#ifndef BH_MOM_MINB
#define BH_MOM_MINB 4
#endif
__global__ void __launch_bounds__(256, BH_MOM_MINB) k_moments_coop(TreeView t, int *__restrict__ lvl,
                                                     int *__restrict__ list, int leaf) {
  cg::grid_group grid = cg::this_grid();
  const int64_t C = tree_count(t);
  if (C > t.C) return;  // overflowed build (uniform across the grid): nothing valid
  int *cnt = lvl, *offs = lvl + (kMaxLevel + 1), *cur = lvl + 2 * (kMaxLevel + 1);
  int *nbuck = lvl + 3 * (kMaxLevel + 1);  // pruned mode: buckets listed from the end of `list`
  MOM_MARK(0);
  const bool prelisted = leaf > 1 && t.mclass;
  if (blockIdx.x == 0 && threadIdx.x == 0 && !prelisted) {
    int acc = 0;
    for (int l = 0; l <= kMaxLevel; ++l) {
      offs[l] = acc;
      cur[l] = 0;
      acc += cnt[l];
    }
    *nbuck = 0;
  }
  grid.sync();
  __shared__ int h[kMaxLevel + 1], base[kMaxLevel + 1];
  __shared__ int hb, bbase;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  if (leaf > 1 && t.mclass) {
    // walk-only tree: listed by k_mom_lists, bucket moments formed by k_bucket_moments
  } else {
  for (int64_t c0 = (int64_t)blockIdx.x * blockDim.x; c0 < C; c0 += stride) {
    if (threadIdx.x <= kMaxLevel) h[threadIdx.x] = 0;
    if (threadIdx.x == 0) hb = 0;
    __syncthreads();
    const int64_t c = c0 + threadIdx.x;
    int l = -1, rank = 0, brank = -1;
    if (c < C) {
      const int4 L = t.link[c];
      if (L.y > 1) {
        if (leaf <= 1 || walk_opens(c, L, leaf)) {
          l = L.w;
          rank = atomicAdd(&h[l], 1);
        } else if (walk_opens(t.parent[c], t.link[t.parent[c]], leaf)) {
          brank = atomicAdd(&hb, 1);  // a bucket: moments from its bodies
        }  // else inside a bucket: never read by the walk
      }
    }
    __syncthreads();
    if (threadIdx.x <= kMaxLevel && h[threadIdx.x])
      base[threadIdx.x] = offs[threadIdx.x] + atomicAdd(&cur[threadIdx.x], h[threadIdx.x]);
    if (threadIdx.x == 0 && hb) bbase = atomicAdd(nbuck, hb);
    __syncthreads();
    if (l >= 0) list[base[l] + rank] = (int)c;
    if (brank >= 0) list[C - 1 - (bbase + brank)] = (int)c;
    __syncthreads();
  }
  }
  grid.sync();
  MOM_MARK(1);
  const int sub = (threadIdx.x & 31) >> 3;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = stride >> 5;
  if (leaf > 1 && !prelisted) {  // the buckets first (no level order among them), then only the opened cells
    const int nb = *nbuck;
#ifdef BH_MOM_TIMERS
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      g_mom_t[62] = (unsigned long long)nb;
      int no = 0;
      for (int l = 0; l <= kMaxLevel; ++l) no += cur[l];
      g_mom_t[63] = (unsigned long long)no;
    }
#endif
    for (int64_t b0 = warp * 4; b0 < nb; b0 += nwarps * 4) {
      const int64_t k = b0 + sub;
      bucket_moments8(t, k < nb ? list[C - 1 - k] : -1);
    }
    grid.sync();
  }
  MOM_MARK(2);
#ifdef BH_MOM_TIMERS
  int nmark = 3;
#endif
  // Runs of consecutive small levels (few cells: the top of the tree and the
  // deepest levels) are swept by block 0 alone with block barriers; the rest
  // of the grid waits at one grid barrier after the run.
  // 8 lanes per cell (cell_moments8): a warp takes 4 cells per pass.
  int *lc = leaf > 1 ? cur : cnt;  // cells listed per level (pruned mode: the opened ones)
  __shared__ double xs[256 / 32][32][11];
  double(*wx)[11] = xs[threadIdx.x >> 5];
  const int small = 2 * (int)(blockDim.x >> 3);
  int l = kMaxLevel;
  while (l >= 0) {
    const int n_l = lc[l];
    if (n_l == 0) { --l; continue; }
    if (n_l <= small) {
      int l2 = l;
      while (l2 >= 0 && lc[l2] <= small) --l2;  // run = levels (l2, l]
      if (blockIdx.x == 0) {
        for (int ll = l; ll > l2; --ll) {
          const int nll = lc[ll], bll = offs[ll];
          for (int base = (int)(threadIdx.x >> 5) * 4; base < nll; base += (int)(blockDim.x >> 5) * 4) {
            const int k = base + sub;
            cell_moments8(t, k < nll ? list[bll + k] : -1, wx);
          }
          __syncthreads();
        }
      }
      l = l2;
      grid.sync();
      MOM_MARK(nmark++);
      continue;
    }
    const int b_l = offs[l];
    for (int64_t base = warp * 4; base < n_l; base += nwarps * 4) {
      const int64_t k = base + sub;
      cell_moments8(t, k < n_l ? list[b_l + k] : -1, wx);
    }
    grid.sync();
    MOM_MARK(nmark++);
    --l;
  }
}

int launch_moments_coop(const TreeView &t, int *lvl, int *list, int sms, cudaStream_t s, int leaf) {
  if (t.n <= 1) return 0;
  if (leaf > 1 && t.mclass) {
    cudaMemsetAsync(lvl + 2 * (kMaxLevel + 1), 0, sizeof(int) * (kMaxLevel + 2), s);  // cur, nbuck
    const int64_t cells = t.C + 16;
    const int gl = (int)std::min<int64_t>((cells + 4095) / 4096, (int64_t)sms * 8);
    k_mom_lists<<<gl, 256, 0, s>>>(t, lvl, list);
    k_bucket_moments<<<sms * 8, 256, 0, s>>>(t, lvl, list);
  }
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_moments_coop, 256, 0);
  if (per_sm < 1) per_sm = 1;
  dim3 grid(sms * per_sm), block(256);
  TreeView tv = t;
  void *args[] = {&tv, &lvl, &list, &leaf};
  return (int)cudaLaunchCooperativeKernel((void *)k_moments_coop, grid, block, args, 0, s);
}


// FlatTree export (flattree.py:34-52; hashed.py:111-129 cell_geometry for the
// centre, same child-offset arithmetic as _build_kernel).
__global__ void k_export(TreeView t, double R, uint64_t *key, int8_t *level, double *centre,
                         double *side, double *mass, double *com, double *quad,
                         int64_t *count, int32_t *children) {
  int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= t.C || c >= tree_count(t)) return;
  int4 L = t.link[c];
  int l = L.w;
  uint64_t pref = 0;
  if (c > 0) pref = t.keys[L.z] >> (3 * (kMortonBits - l));
  if (key) key[c] = c == 0 ? 1ull : (pref | (1ull << (3 * l)));
  if (level) level[c] = (int8_t)l;
  if (centre || side) {
    double cen0 = 0.0, cen1 = 0.0, cen2 = 0.0, sd = 2.0 * R;
    for (int lv = l - 1; lv >= 0; --lv) {
      int slot = (int)((pref >> (3 * lv)) & 7);
      double half = 0.25 * sd;
      cen0 += (slot & 4) ? half : -half;
      cen1 += (slot & 2) ? half : -half;
      cen2 += (slot & 1) ? half : -half;
      sd = 0.5 * sd;
    }
    if (centre) { centre[3 * c] = cen0; centre[3 * c + 1] = cen1; centre[3 * c + 2] = cen2; }
    if (side) side[c] = sd;
  }
  double4 cm = t.cm64[c];
  if (mass) mass[c] = cm.w;
  if (com) { com[3 * c] = cm.x; com[3 * c + 1] = cm.y; com[3 * c + 2] = cm.z; }
  if (quad) {
    for (int k = 0; k < 6; ++k) quad[6 * c + k] = L.y > 1 ? t.q64[kQStride * c + k] : 0.0;
  }
  if (count) count[c] = t.n == 0 ? 0 : L.y;
  if (children) {
    const int4 *row = reinterpret_cast<const int4 *>(t.child8 + 8 * c);
    int4 r0 = row[0], r1 = row[1];
    auto dec = [](int v) { return v < -1 ? -v - 2 : v; };  // leaf children are stored as -(c + 2)
    r0 = make_int4(dec(r0.x), dec(r0.y), dec(r0.z), dec(r0.w));
    r1 = make_int4(dec(r1.x), dec(r1.y), dec(r1.z), dec(r1.w));
    int32_t *o = children + 8 * c;
    o[0] = r0.x; o[1] = r0.y; o[2] = r0.z; o[3] = r0.w;
    o[4] = r1.x; o[5] = r1.y; o[6] = r1.z; o[7] = r1.w;
  }
}

void launch_export(const TreeView &t, double R, uint64_t *key, int8_t *level, double *centre,
                   double *side, double *mass, double *com, double *quad, int64_t *count,
                   int32_t *children, cudaStream_t s) {
  if (t.C <= 0) return;
  k_export<<<grid_for(t.C, 256), 256, 0, s>>>(t, R, key, level, centre, side, mass, com, quad,
                                              count, children);
}

// ------------------------------------------- distributed build (one rank)
// Shared cells of a rank's local tree: the root and the cells on the first /
// last local body's path down to the levels it shares with the neighbouring
// rank's boundary key.  Their counts and moments are partial (the neighbour
// holds bodies in them); every other cell holds only this rank's bodies and is
// exactly the global tree's cell.  Branch nodes (hashed.py:609-630) are the
// unshared children of shared cells -- or the root when there is no neighbour.
__global__ void k_mark_shared(TreeView t, uint8_t *__restrict__ shared, int *__restrict__ branch,
                              int *__restrict__ nbranch) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  int nb = 0;
  if (t.bnd_prev < 0 && t.bnd_next < 0) {  // no neighbour: the root is the branch
    branch[nb++] = 0;
    *nbranch = nb;
    return;
  }
  int list[2 * kMaxLevel + 2];
  int ns = 0;
  shared[0] = 1;
  list[ns++] = 0;
  for (int side = 0; side < 2; ++side) {
    const int bnd = side == 0 ? t.bnd_prev : t.bnd_next;
    if (bnd < 0) continue;
    const uint64_t k = t.keys[side == 0 ? 0 : t.n - 1];
    int cur = 0;
    for (int l = 1; l <= bnd && l <= kMaxLevel; ++l) {
      int c = t.child8[8 * (int64_t)cur + (int)((k >> (3 * (kMortonBits - l))) & 7)];
      if (c == -1) break;
      if (c < -1) c = -c - 2;  // a leaf child
      if (!shared[c]) {
        shared[c] = 1;
        list[ns++] = c;
      }
      cur = c;
    }
  }
  // branch nodes: unshared children of shared cells (shared cells in pre-order)
  for (int a = 1; a < ns; ++a)  // insertion sort of the <= 43 shared cells
    for (int b = a; b > 0 && list[b - 1] > list[b]; --b) {
      int tmp = list[b]; list[b] = list[b - 1]; list[b - 1] = tmp;
    }
  for (int q = 0; q < ns; ++q) {
    const int c = list[q];
    for (int s = 0; s < 8; ++s) {
      int ch = t.child8[8 * (int64_t)c + s];
      if (ch < -1) ch = -ch - 2;  // a leaf child
      if (ch >= 0 && !shared[ch]) branch[nb++] = ch;
    }
  }
  *nbranch = nb;
}

void launch_mark_shared(const TreeView &t, uint8_t *shared, int *branch, int *nbranch,
                        cudaStream_t s) {
  cudaMemsetAsync(shared, 0, t.C, s);
  k_mark_shared<<<1, 32, 0, s>>>(t, shared, branch, nbranch);
}

// One row per branch node: cell key, level, count, exact fp64 moments, and its
// walk record index (rec_of_cell) -- the payload of the branch-node allgather
// (hashed.py:633-639).
__global__ void k_branch_export(TreeView t, const int *__restrict__ branch, int nb,
                                const int *__restrict__ rec_of_cell, uint64_t *key, int *level,
                                int64_t *count, double *mom /* [nb][10] */, int *rec, int *lo) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= nb) return;
  const int c = branch[k];
  const int4 L = t.link[c];
  const uint64_t pref = t.keys[L.z] >> (3 * (kMortonBits - L.w));
  key[k] = c == 0 ? 1ull : (pref | (1ull << (3 * L.w)));
  level[k] = L.w;
  count[k] = L.y;
  const double4 cm = t.cm64[c];
  double *m = mom + 10 * (int64_t)k;
  m[0] = cm.w; m[1] = cm.x; m[2] = cm.y; m[3] = cm.z;
  for (int q = 0; q < 6; ++q) m[4 + q] = L.y > 1 ? t.q64[kQStride * (int64_t)c + q] : 0.0;
  rec[k] = rec_of_cell ? rec_of_cell[c] : -1;
  if (lo) lo[k] = L.z;
}

void launch_branch_export(const TreeView &t, const int *branch, int nb, const int *rec_of_cell,
                          uint64_t *key, int *level, int64_t *count, double *mom, int *rec,
                          int *lo, cudaStream_t s) {
  if (nb <= 0) return;
  k_branch_export<<<grid_for(nb, 128), 128, 0, s>>>(t, branch, nb, rec_of_cell, key, level, count,
                                                    mom, rec, lo);
}

// ------------------------------------------------------------- fp64 walk
// Correctly rounded x^1.5 (the reference computes (d2+e2)**1.5 with libm pow,
// which is correctly rounded in practice): x*sqrt(x) evaluated in double-double
// and rounded once.
__device__ __forceinline__ double pow15(double x) {
  double s = __dsqrt_rn(x);
  double e = fma(-s, s, x);          // exact residual x - s^2
  double t = e / (2.0 * s);          // sqrt(x) = s + t + O(t^2)
  double p = x * s;
  double pl = fma(x, s, -p);         // exact low part of x*s
  return p + (pl + x * t);
}

__device__ __forceinline__ void pp64(double px, double py, double pz, double4 b, double e2,
                                     double &ax, double &ay, double &az, int &npp) {
  double dx = px - b.x, dy = py - b.y, dz = pz - b.z;
  double d2 = dx * dx + dy * dy + dz * dz;
  if (d2 == 0.0) return;
  double denom = pow15(d2 + e2);
  ax += (-b.w * dx) / denom;
  ay += (-b.w * dy) / denom;
  az += (-b.w * dz) / denom;
  ++npp;
}

// flattree.py:258-317 _traverse_kernel.  One warp walks the union of its 32
// targets' interaction lists in pre-order: each lane keeps its own "next" cell
// (its private DFS position); the warp visits the minimum, lanes positioned
// there evaluate it.  Every lane therefore sees exactly the reference's list,
// in the reference's order, so its fp64 sums are the reference's sums.
__global__ void __launch_bounds__(128) k_walk_f64(
    WalkParams P, const double4 *__restrict__ cm, const double *__restrict__ q64,
    const int4 *__restrict__ link, const double4 *__restrict__ bodies,
    const double *__restrict__ targets, int tstride, const uint32_t *__restrict__ tperm,
    double *__restrict__ acc, int astride, int64_t *__restrict__ work64,
    int *__restrict__ work32, DeviceFlags *f) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool valid = t < P.nt;
  const int64_t src = valid ? (tperm ? (int64_t)tperm[t] : t) : 0;
  double px = 0.0, py = 0.0, pz = 0.0;
  if (valid) {
    const double *q = targets + src * tstride;
    px = q[0]; py = q[1]; pz = q[2];
  }
  double ax = 0.0, ay = 0.0, az = 0.0;
  int npp = 0, npc = 0;
  int next = valid ? (P.C == 1 ? 0 : 1) : INT_MAX;
  while (true) {
    const int i = __reduce_min_sync(0xffffffffu, next);
    if (i >= P.C) break;
    if (next != i) continue;
    const double4 c = cm[i];
    const int4 L = link[i];
    const double dx = px - c.x, dy = py - c.y, dz = pz - c.z;
    const double d2 = dx * dx + dy * dy + dz * dz;
    if (L.y == 1) {
      if (d2 != 0.0) {
        double denom = pow15(d2 + P.e2);
        ax += (-c.w * dx) / denom;
        ay += (-c.w * dy) / denom;
        az += (-c.w * dz) / denom;
        ++npp;
      }
      next = i + 1;
    } else if (d2 > 0.0 && P.side64[L.w] < P.theta * sqrt(d2)) {
      const double *q = q64 + kQStride * (int64_t)i;
      const double r1 = sqrt(d2);
      const double qrx = q[0] * dx + q[1] * dy + q[2] * dz;
      const double qry = q[1] * dx + q[3] * dy + q[4] * dz;
      const double qrz = q[2] * dx + q[4] * dy + q[5] * dz;
      const double rqr = dx * qrx + dy * qry + dz * qrz;
      const double mono = -c.w / (d2 * r1);
      const double c5 = d2 * d2 * r1;
      const double c7 = 2.5 * rqr / (d2 * d2 * d2 * r1);
      ax += mono * dx + qrx / c5 - c7 * dx;
      ay += mono * dy + qry / c5 - c7 * dy;
      az += mono * dz + qrz / c5 - c7 * dz;
      ++npc;
      next = L.x;
    } else if (P.leaf > 1 && (L.y <= P.leaf || L.w == kMaxLevel)) {  // bucket / dup cell
      for (int j = L.z; j < L.z + L.y; ++j) pp64(px, py, pz, bodies[j], P.e2, ax, ay, az, npp);
      next = L.x;
    } else {
      next = i + 1;
    }
  }
  if (valid) {
    double *o = acc + src * astride;
    o[0] = ax; o[1] = ay; o[2] = az;
    const int w = npp * 1 + npc * 2;  // WORK_PP, WORK_PC (octree.py:23-25)
    if (work64) work64[src] = w;
    if (work32) work32[src] = w;
  }
  unsigned long long spp = npp, spc = npc;
  for (int o = 16; o > 0; o >>= 1) {
    spp += __shfl_xor_sync(0xffffffffu, spp, o);
    spc += __shfl_xor_sync(0xffffffffu, spc, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(&f->pp, spp);
    atomicAdd(&f->pc, spc);
  }
}

void launch_walk_f64(const WalkParams &p, const double4 *cm64, const double *q64,
                     const int4 *link, const double4 *bodies, const double *targets,
                     int tstride, const uint32_t *tperm, double *acc, int astride,
                     int64_t *work64, int *work32, DeviceFlags *f, cudaStream_t s) {
  if (p.nt <= 0) return;
  k_walk_f64<<<grid_for(p.nt, 128), 128, 0, s>>>(p, cm64, q64, link, bodies, targets, tstride,
                                                 tperm, acc, astride, work64, work32, f);
}

// ------------------------------------------------------ fp64 integrator
// integrator.py:37-44: v += a*h; x += v*dt (two roundings each, as numpy)
__global__ void k_kick_f64(double *v, const double *a, int64_t n3, double h) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n3) v[i] = v[i] + a[i] * h;
}
void launch_kick_f64(double *vel3, const double *acc3, int64_t n, double h, cudaStream_t s) {
  if (n <= 0) return;
  k_kick_f64<<<grid_for(3 * n, 256), 256, 0, s>>>(vel3, acc3, 3 * n, h);
}
void launch_drift_f64(double *pos3, const double *vel3, int64_t n, double dt, cudaStream_t s) {
  if (n <= 0) return;
  k_kick_f64<<<grid_for(3 * n, 256), 256, 0, s>>>(pos3, vel3, 3 * n, dt);
}

__device__ __forceinline__ unsigned long long dmax_bits(double a) {
  return (unsigned long long)__double_as_longlong(fabs(a));
}

// resident fp64 state {x,y,z,m} / {vx,vy,vz,0}: optional half kick, drift,
// and the max|x| of the drifted positions (next step's bounds)
__global__ void k_kick_drift_max_f64(double4 *pos, double4 *vel, const double4 *acc, int64_t n,
                                     double h, double dt, DeviceFlags *f) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  unsigned long long m = 0;
  if (i < n) {
    double4 x = pos[i];
    if (dt != 0.0) {
      double4 v = vel[i];
      if (acc) {
        double4 a = acc[i];
        v.x = v.x + a.x * h; v.y = v.y + a.y * h; v.z = v.z + a.z * h;
        vel[i] = v;
      }
      x.x = x.x + v.x * dt; x.y = x.y + v.y * dt; x.z = x.z + v.z * dt;
      pos[i] = x;
    }
    unsigned long long a = dmax_bits(x.x), b = dmax_bits(x.y), c = dmax_bits(x.z);
    m = a > b ? a : b;
    m = m > c ? m : c;
  }
  for (int o = 16; o > 0; o >>= 1) {
    unsigned long long r = __shfl_xor_sync(0xffffffffu, m, o);
    m = r > m ? r : m;
  }
  if ((threadIdx.x & 31) == 0 && m) atomicMax((unsigned long long *)&f->maxabs64, m);
}
void launch_kick_drift_max_f64(double4 *pos, double4 *vel, const double4 *acc, int64_t n,
                               double h, double dt, DeviceFlags *f, cudaStream_t s) {
  if (n <= 0) return;
  k_kick_drift_max_f64<<<grid_for(n, 256), 256, 0, s>>>(pos, vel, acc, n, h, dt, f);
}

__global__ void k_kick4_f64(double4 *vel, const double4 *acc, int64_t n, double h) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double4 v = vel[i], a = acc[i];
  v.x = v.x + a.x * h; v.y = v.y + a.y * h; v.z = v.z + a.z * h;
  vel[i] = v;
}
void launch_kick4_f64(double4 *vel, const double4 *acc, int64_t n, double h, cudaStream_t s) {
  if (n <= 0) return;
  k_kick4_f64<<<grid_for(n, 256), 256, 0, s>>>(vel, acc, n, h);
}

__global__ void k_maxabs_f64(const double *p, int64_t n3, DeviceFlags *f) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  unsigned long long m = i < n3 ? dmax_bits(p[i]) : 0ull;
  for (int o = 16; o > 0; o >>= 1) {
    unsigned long long r = __shfl_xor_sync(0xffffffffu, m, o);
    m = r > m ? r : m;
  }
  if ((threadIdx.x & 31) == 0 && m) atomicMax((unsigned long long *)&f->maxabs64, m);
}
void launch_maxabs_f64(const double *pos3, int64_t n, DeviceFlags *f, cudaStream_t s) {
  if (n <= 0) return;
  k_maxabs_f64<<<grid_for(3 * n, 256), 256, 0, s>>>(pos3, 3 * n, f);
}

// morton.py:41-42: R = 1.001 * extreme, or 1.0 for an all-zero cloud
__global__ void k_finish_R(const DeviceFlags *f, int fp64, double *d_R) {
  // maxabs64 holds the bits of a non-negative double (atomicMax on its bits)
  double extreme = fp64 ? f->maxabs64 : (double)__uint_as_float(f->maxabs_bits);
  *d_R = extreme > 0.0 ? 1.001 * extreme : 1.0;
}
void launch_finish_R(const DeviceFlags *f, int fp64, double *d_R, cudaStream_t s) {
  k_finish_R<<<1, 1, 0, s>>>(f, fp64, d_R);
}

// ----------------------------------------------------- validation kernels
// physics.py:216-242 _accel_all_pairs: per target, sources in index order
// (same summation order as the reference, so the result is bit-identical).
__global__ void __launch_bounds__(256) k_direct_f64(const double *__restrict__ pos,
                                                    const double *__restrict__ mass,
                                                    int64_t n, double e2, double *acc) {
  __shared__ double4 tile[256];
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  double xi = 0, yi = 0, zi = 0;
  if (i < n) { xi = pos[3 * i]; yi = pos[3 * i + 1]; zi = pos[3 * i + 2]; }
  double ax = 0.0, ay = 0.0, az = 0.0;
  for (int64_t j0 = 0; j0 < n; j0 += 256) {
    int64_t j = j0 + threadIdx.x;
    __syncthreads();
    if (j < n) tile[threadIdx.x] = make_double4(pos[3 * j], pos[3 * j + 1], pos[3 * j + 2], mass[j]);
    __syncthreads();
    int lim = (int)(n - j0 < 256 ? n - j0 : 256);
    for (int k = 0; k < lim; ++k) {
      if (j0 + k == i) continue;
      double4 s = tile[k];
      double dx = xi - s.x, dy = yi - s.y, dz = zi - s.z;
      double r2 = dx * dx + dy * dy + dz * dz;
      if (r2 == 0.0) continue;
      double w = s.w / ((r2 + e2) * sqrt(r2 + e2));
      ax -= w * dx;
      ay -= w * dy;
      az -= w * dz;
    }
  }
  if (i < n) { acc[3 * i] = ax; acc[3 * i + 1] = ay; acc[3 * i + 2] = az; }
}
void launch_direct_f64(const double *pos3, const double *mass, int64_t n, double eps,
                       double *acc3, cudaStream_t s) {
  if (n <= 0) return;
  k_direct_f64<<<grid_for(n, 256), 256, 0, s>>>(pos3, mass, n, eps * eps, acc3);
}

// physics.py:273-285 _potential_pairs: partial[i] = sum_{j>i} -m_i m_j / r_soft
__global__ void __launch_bounds__(256) k_potential_f64(const double *__restrict__ pos,
                                                       const double *__restrict__ mass,
                                                       int64_t n, double e2, double *partial) {
  __shared__ double4 tile[256];
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  double xi = 0, yi = 0, zi = 0, mi = 0;
  if (i < n) { xi = pos[3 * i]; yi = pos[3 * i + 1]; zi = pos[3 * i + 2]; mi = mass[i]; }
  double pot = 0.0;
  int64_t jstart = (int64_t)blockIdx.x * blockDim.x;  // j > i only
  for (int64_t j0 = jstart; j0 < n; j0 += 256) {
    int64_t j = j0 + threadIdx.x;
    __syncthreads();
    if (j < n) tile[threadIdx.x] = make_double4(pos[3 * j], pos[3 * j + 1], pos[3 * j + 2], mass[j]);
    __syncthreads();
    int lim = (int)(n - j0 < 256 ? n - j0 : 256);
    for (int k = 0; k < lim; ++k) {
      if (j0 + k <= i) continue;
      double4 s = tile[k];
      double dx = xi - s.x, dy = yi - s.y, dz = zi - s.z;
      double r2 = dx * dx + dy * dy + dz * dz;
      pot -= mi * s.w / sqrt(r2 + e2);
    }
  }
  if (i < n) partial[i] = pot;
}
void launch_potential_f64(const double *pos3, const double *mass, int64_t n, double eps,
                          double *partial, cudaStream_t s) {
  if (n <= 0) return;
  k_potential_f64<<<grid_for(n, 256), 256, 0, s>>>(pos3, mass, n, eps * eps, partial);
}

}  // namespace bh
