// bh_fast.cu -- fp32 kernels (FMA contraction allowed): bounds reduction,
// the fused integrator and body gathers (radix sort and scans: bh_sort.cu).
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <climits>

#include "bh_internal.cuh"

namespace bh {

// ---------------------------------------------------------------- bounds
__device__ __forceinline__ unsigned fabs_bits(float a) { return __float_as_uint(fabsf(a)); }

// one atomic per block (a per-warp atomic on one address serialises in L2:
// 3e6 of them at 1e8 bodies)
__device__ __forceinline__ void block_max_to(unsigned m, unsigned *dst) {
  __shared__ unsigned wm[32];
  m = __reduce_max_sync(0xffffffffu, m);
  if ((threadIdx.x & 31) == 0) wm[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x < 32) {
    unsigned v = threadIdx.x < (blockDim.x >> 5) ? wm[threadIdx.x] : 0u;
    v = __reduce_max_sync(0xffffffffu, v);
    if (threadIdx.x == 0 && v) atomicMax(dst, v);
  }
}
// grid for the streaming kernels: a few resident waves, grid-stride inside
static inline int stream_grid(int64_t n) {
  static int g = 0;
  if (g == 0) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    g = sms * 8;
  }
  const int64_t need = (n + 255) / 256;
  return (int)std::max<int64_t>(1, std::min<int64_t>(need, g));
}

// morton.py:39-42: max |x| over all bodies and axes (float bits are
// order-preserving for non-negative floats; NaN sorts above +inf and makes R
// NaN, which the key kernel then reports as out of domain)
__global__ void k_maxabs_f32(const float4 *__restrict__ p, int64_t n, DeviceFlags *f) {
  unsigned m = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const float4 v = p[i];
    m = max(m, max(fabs_bits(v.x), max(fabs_bits(v.y), fabs_bits(v.z))));
  }
  block_max_to(m, &f->maxabs_bits);
}

__global__ void k_reset_bounds(DeviceFlags *f) {
  f->maxabs_bits = 0;
  f->maxabs64 = 0.0;
}
void launch_reset_flags_bounds(DeviceFlags *f, cudaStream_t s) { k_reset_bounds<<<1, 1, 0, s>>>(f); }

void launch_maxabs_f32(const float4 *pos, int64_t n, DeviceFlags *f, cudaStream_t s) {
  if (n <= 0) return;
  k_maxabs_f32<<<stream_grid(n), 256, 0, s>>>(pos, n, f);
}

// ------------------------------------------------------------ integrator
__global__ void k_kick_f32(float4 *v, const float4 *a, int64_t n, float h, const DeviceFlags *f) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n || overflowed(f)) return;
  float4 x = v[i], y = a[i];
  x.x += y.x * h; x.y += y.y * h; x.z += y.z * h;
  v[i] = x;
}
void launch_kick_f32(float4 *vel, const float4 *acc, int64_t n, float h, cudaStream_t s,
                     const DeviceFlags *skip_on_overflow) {
  if (n <= 0) return;
  k_kick_f32<<<grid_for(n, 256), 256, 0, s>>>(vel, acc, n, h, skip_on_overflow);
}
// drift keeps the mass in .w untouched
__global__ void k_drift_f32(float4 *x, const float4 *v, int64_t n, float dt) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  float4 p = x[i], u = v[i];
  p.x += u.x * dt; p.y += u.y * dt; p.z += u.z * dt;
  x[i] = p;
}
void launch_drift_f32(float4 *pos, const float4 *vel, int64_t n, float dt, cudaStream_t s) {
  if (n <= 0) return;
  k_drift_f32<<<grid_for(n, 256), 256, 0, s>>>(pos, vel, n, dt);
}

// integrator.py:37-44 in the _drive order (simulation.py:492-495):
// v += a*h; x += v*dt; plus max|x| of the new positions for the next bounds
__global__ void k_kick_drift_max_f32(float4 *__restrict__ pos, float4 *__restrict__ vel,
                                     const float4 *__restrict__ acc, int64_t n, float h,
                                     float dt, DeviceFlags *f) {
  if (overflowed(f)) return;  // a failed build earlier in this call: the state waits for the redo
  unsigned m = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    float4 x = pos[i];
    if (dt != 0.f) {
      float4 v = vel[i];
      if (acc) {
        float4 a = acc[i];
        v.x += a.x * h; v.y += a.y * h; v.z += a.z * h;
        vel[i] = v;
      }
      x.x += v.x * dt; x.y += v.y * dt; x.z += v.z * dt;
      pos[i] = x;
    }
    m = max(m, max(fabs_bits(x.x), max(fabs_bits(x.y), fabs_bits(x.z))));
  }
  block_max_to(m, &f->maxabs_bits);
}
void launch_kick_drift_max_f32(float4 *pos, float4 *vel, const float4 *acc, int64_t n,
                               float h, float dt, DeviceFlags *f, cudaStream_t s) {
  if (n <= 0) return;
  k_kick_drift_max_f32<<<stream_grid(n), 256, 0, s>>>(pos, vel, acc, n, h, dt, f);
}

// ---------------------------------------------------------------- gathers
template <class T>
__global__ void k_gather(const uint32_t *__restrict__ idx, int64_t n, const T *__restrict__ a,
                         T *__restrict__ a2, const T *__restrict__ b, T *__restrict__ b2,
                         const uint32_t *__restrict__ id, uint32_t *__restrict__ id2) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint32_t j = idx[i];
  a2[i] = a[j];
  if (b) b2[i] = b[j];
  if (id) id2[i] = id[j];
}
void launch_gather_f32(const uint32_t *idx, int64_t n, const float4 *a, float4 *a2,
                       const float4 *b, float4 *b2, const uint32_t *id, uint32_t *id2,
                       cudaStream_t s) {
  if (n <= 0) return;
  k_gather<float4><<<grid_for(n, 256), 256, 0, s>>>(idx, n, a, a2, b, b2, id, id2);
}
void launch_gather_f64(const uint32_t *idx, int64_t n, const double4 *a, double4 *a2,
                       const double4 *b, double4 *b2, const uint32_t *id, uint32_t *id2,
                       cudaStream_t s) {
  if (n <= 0) return;
  k_gather<double4><<<grid_for(n, 256), 256, 0, s>>>(idx, n, a, a2, b, b2, id, id2);
}

__global__ void k_pack_f64(const double *pos3, const double *mass, int64_t n, double4 *out) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  out[i] = make_double4(pos3[3 * i], pos3[3 * i + 1], pos3[3 * i + 2], mass ? mass[i] : 0.0);
}
void launch_pack_bodies_f64(const double *pos3, const double *mass, int64_t n, double4 *out,
                            cudaStream_t s) {
  if (n <= 0) return;
  k_pack_f64<<<grid_for(n, 256), 256, 0, s>>>(pos3, mass, n, out);
}

__global__ void k_iota64(int64_t *out, const uint32_t *vals, int64_t n) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = vals[i];
}
void launch_iota64(int64_t *out, const uint32_t *vals, int64_t n, cudaStream_t s) {
  if (n <= 0) return;
  k_iota64<<<grid_for(n, 256), 256, 0, s>>>(out, vals, n);
}

// --------------------------------------------------- FFMA peak microbench
// 8 independent FFMA chains per thread, 8 warps x 4 blocks per SM: the FP32
// pipe's sustained issue rate at the current clock (walk roofline denominator)
__device__ __forceinline__ float fma_t(float x, float a, float b) { return fmaf(x, a, b); }
__device__ __forceinline__ double fma_t(double x, double a, double b) { return fma(x, a, b); }
template <class T>
__global__ void __launch_bounds__(256) k_ffma(T *out, int iters, T a, T b) {
  T x[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) x[k] = threadIdx.x * 1e-3f + k;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int r = 0; r < 8; ++r) {
#pragma unroll
      for (int k = 0; k < 8; ++k) x[k] = fma_t(x[k], a, b);
    }
  }
  T sum = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) sum += x[k];
  if (sum == (T)1234.5) out[0] = sum;
}
void run_ffma(float *out, int sms, int iters, double *flops, cudaStream_t s) {
  const int blocks = sms * 4, threads = 256;
  k_ffma<float><<<blocks, threads, 0, s>>>(out, iters, 0.999999f, 1e-7f);
  *flops = 2.0 * 64.0 * (double)iters * blocks * threads;
}
// the same loop in fp64 (DFMA): the roofline denominator of the fp64 walk
void run_dfma(double *out, int sms, int iters, double *flops, cudaStream_t s) {
  const int blocks = sms * 4, threads = 256;
  k_ffma<double><<<blocks, threads, 0, s>>>(out, iters, 0.999999, 1e-7);
  *flops = 2.0 * 64.0 * (double)iters * blocks * threads;
}

}  // namespace bh
