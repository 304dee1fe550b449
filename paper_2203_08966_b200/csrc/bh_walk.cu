// bh_walk.cu -- the fp32 force traversal (flattree.py:258-317) and the walk
// tree it runs on.  Compiled with -ftz=true (no denormal fix-up around
// MUFU.RSQ; distances here are never denormal).
//
// Walk tree.  The reference tree keeps one body per leaf; with leaf size L a
// cell of count <= L is never opened, so its subtree is dead
// weight for the walk.  k_keep/k_compact copy the cells the walk can reach --
// the root and every child of a cell with count > L -- in pre-order into a
// compact array of 64-byte records, with the MAC threshold (side/theta)^2 baked
// in and the skip links remapped.  At L = 1 every cell is kept.
//
//   a = {com.x, com.y, com.z, mac2}      MAC test   (with d)
//   b = {qxx, qxy, qxy, qyy}             quadrupole, paired for FFMA2
//   c = {qxz, qyz, mass, qzz}
//   d = {skip, count, lo, level}         skip = index after the subtree (i+1
//                                        for pruned buckets), lo = first body
//
// Walk.  One warp walks the union of its 32 targets' interaction lists in
// pre-order; every lane keeps its own DFS position `next` and evaluates exactly
// its reference list (per-lane MAC).  The node loads have a warp-uniform
// address (one wavefront each).  The quadrupole evaluation pairs the x/y
// components in FFMA2/FMUL2 instructions: the kernel is issue-bound, and a
// packed instruction does two FMAs per issue slot (measured: FFMA2 runs at the
// same 74 TFLOP/s pipe rate as FFMA but frees issue slots).
#include <cuda_runtime.h>
#include <stdint.h>

#include <climits>

#include "bh_internal.cuh"

namespace bh {

__global__ void k_keep(TreeView t, int leaf, uint32_t *__restrict__ keep) {
  int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= t.C) return;
  uint32_t k = 1;
  if (c > 0) k = t.link[t.parent[c]].y > leaf ? 1u : 0u;
  keep[c] = k;
}

void launch_keep(const TreeView &t, int leaf, uint32_t *keep, cudaStream_t s) {
  k_keep<<<grid_for(t.C, 256), 256, 0, s>>>(t, leaf, keep);
}

__global__ void k_compact(TreeView t, WalkTable tab, int leaf, const uint32_t *__restrict__ keep,
                          const uint32_t *__restrict__ widx, WalkNode *__restrict__ out,
                          int *__restrict__ dCp) {
  int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t C = t.C;
  if (c >= C) return;
  const int Cp = (int)(widx[C - 1] + keep[C - 1]);
  if (c == C - 1) *dCp = Cp;
  if (!keep[c]) return;
  const int j = (int)widx[c];
  const int4 L = t.link[c];
  const double4 cm = t.cm64[c];
  WalkNode nd;
  nd.a = make_float4((float)cm.x, (float)cm.y, (float)cm.z, tab.mac2[L.w]);
  float q0 = 0.f, q1 = 0.f, q2 = 0.f, q3 = 0.f, q4 = 0.f, q5 = 0.f;
  if (L.y > 1) {
    const double *q = t.q64 + 6 * c;
    q0 = (float)q[0]; q1 = (float)q[1]; q2 = (float)q[2];
    q3 = (float)q[3]; q4 = (float)q[4]; q5 = (float)q[5];
  }
  nd.b = make_float4(q0, q1, q1, q3);
  nd.c = make_float4(q2, q4, (float)cm.w, q5);
  int nxt;
  if (L.y <= leaf) nxt = j + 1;  // bucket / leaf: subtree pruned
  else nxt = L.x < C ? (int)widx[L.x] : Cp;
  nd.d = make_int4(nxt, L.y, L.z, L.w);
  out[j] = nd;
}

void launch_compact(const TreeView &t, const WalkTable &tab, int leaf, const uint32_t *keep,
                    const uint32_t *widx, WalkNode *out, int *dCp, cudaStream_t s) {
  k_compact<<<grid_for(t.C, 256), 256, 0, s>>>(t, tab, leaf, keep, widx, out, dCp);
}

__device__ __forceinline__ float2 f2(float x, float y) { return make_float2(x, y); }
__device__ __forceinline__ float2 f2(float x) { return make_float2(x, x); }

template <bool BUCKET>
__global__ void __launch_bounds__(256) k_walk2(
    const WalkNode *__restrict__ T, const int *__restrict__ dCp,
    const float4 *__restrict__ bodies, const float *__restrict__ targets, int tstride,
    const uint32_t *__restrict__ tperm, int nt, float e2, int leaf, float *__restrict__ acc,
    int astride, int64_t *__restrict__ work64, int *__restrict__ work32, DeviceFlags *f) {
  const int Cp = *dCp;
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool valid = t < nt;
  const int64_t src = valid ? (tperm ? (int64_t)tperm[t] : t) : 0;
  float px = 0.f, py = 0.f, pz = 0.f;
  if (valid) {
    const float *q = targets + src * tstride;
    px = q[0]; py = q[1]; pz = q[2];
  }
  float2 axy = f2(0.f);
  float az = 0.f;
  int npp = 0, npc = 0;
  int next = valid ? (Cp == 1 ? 0 : 1) : INT_MAX;
  for (;;) {
    const int i = __reduce_min_sync(0xffffffffu, next);
    if (i >= Cp) break;
    const WalkNode *nd = T + i;
    const float4 a = nd->a;
    const int4 d = nd->d;
    const bool active = next == i;
    const float2 dxy = f2(px - a.x, py - a.y);
    const float dz = pz - a.z;
    const float2 sq = __fmul2_rn(dxy, dxy);
    const float d2 = fmaf(dz, dz, sq.x + sq.y);
    if (d.y == 1) {  // leaf: softened pp with its body (flattree.py:287-294)
      if (active) {
        if (d2 > 0.f) {
          const float m = nd->c.z;
          const float r = rsqrtf(d2 + e2);
          const float s = -m * r * r * r;
          axy = __ffma2_rn(f2(s), dxy, axy);
          az = fmaf(s, dz, az);
          ++npp;
        }
        next = i + 1;
      }
    } else if (active && d2 > a.w) {  // MAC: side < theta*|d| (flattree.py:295)
      const float4 b = nd->b;
      const float4 c = nd->c;
      const float r = rsqrtf(d2);
      const float r2 = r * r;
      const float r3 = r * r2;
      const float r5 = r3 * r2;
      float2 qxy = __fmul2_rn(f2(b.x, b.y), f2(dxy.x));
      qxy = __ffma2_rn(f2(b.z, b.w), f2(dxy.y), qxy);
      qxy = __ffma2_rn(f2(c.x, c.y), f2(dz), qxy);
      const float qz = fmaf(c.w, dz, fmaf(c.y, dxy.y, c.x * dxy.x));
      const float2 tq = __fmul2_rn(dxy, qxy);
      const float rqr = fmaf(dz, qz, tq.x + tq.y);
      // a = (-M - 2.5 (d.Q.d)/r^4) d/r^3 + (Q.d)/r^5      (physics.py:195-213)
      const float s = fmaf(rqr * (r2 * r2), -2.5f, -c.z) * r3;
      axy = __ffma2_rn(f2(s), dxy, axy);
      axy = __ffma2_rn(f2(r5), qxy, axy);
      az = fmaf(s, dz, fmaf(r5, qz, az));
      ++npc;
      next = d.x;
    } else if (active) {
      if (BUCKET && d.y <= leaf) {  // bucket rule
        const int j1 = d.z + d.y;
        for (int j = d.z; j < j1; ++j) {
          const float4 bb = bodies[j];
          const float2 exy = f2(px - bb.x, py - bb.y);
          const float ez = pz - bb.z;
          const float2 s2 = __fmul2_rn(exy, exy);
          const float r2 = fmaf(ez, ez, s2.x + s2.y);
          if (r2 > 0.f) {
            const float r = rsqrtf(r2 + e2);
            const float s = -bb.w * r * r * r;
            axy = __ffma2_rn(f2(s), exy, axy);
            az = fmaf(s, ez, az);
            ++npp;
          }
        }
      }
      next = i + 1;
    }
  }
  if (valid) {
    float *o = acc + src * astride;
    o[0] = axy.x; o[1] = axy.y; o[2] = az;
    const int w = npp + 2 * npc;  // WORK_PP, WORK_PC (octree.py:23-25)
    if (work64) work64[src] = w;
    if (work32) work32[src] = w;
  }
  const unsigned spp = __reduce_add_sync(0xffffffffu, (unsigned)npp);
  const unsigned spc = __reduce_add_sync(0xffffffffu, (unsigned)npc);
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(&f->pp, (unsigned long long)spp);
    atomicAdd(&f->pc, (unsigned long long)spc);
  }
}

void launch_walk2_f32(const WalkNode *T, const int *dCp, const float4 *bodies,
                      const float *targets, int tstride, const uint32_t *tperm, int nt, float e2,
                      int leaf, float *acc, int astride, int64_t *work64, int *work32,
                      DeviceFlags *f, cudaStream_t s) {
  if (nt <= 0) return;
  if (leaf > 1)
    k_walk2<true><<<grid_for(nt, 256), 256, 0, s>>>(T, dCp, bodies, targets, tstride, tperm, nt,
                                                    e2, leaf, acc, astride, work64, work32, f);
  else
    k_walk2<false><<<grid_for(nt, 256), 256, 0, s>>>(T, dCp, bodies, targets, tstride, tperm, nt,
                                                     e2, leaf, acc, astride, work64, work32, f);
}

}  // namespace bh
