// pc_probe.cu -- throughput of the walk's pc drain loop in isolation: the
// k_walk9 flush_pc body over a list of 20 staged records in shared memory,
// all mask bits set, 24-32 warps per SM.  Reports SMSP cycles per list entry
// per warp (the formula is 30 packed FP ops = 60 FMA-pipe cycles at 2 per op).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -ftz=true -o tools/pc_probe tools/pc_probe.cu
#include <cstdio>
#include <cuda_runtime.h>
#include <cstring>
static float bits_f(int v) { float f; memcpy(&f, &v, 4); return f; }

__device__ __forceinline__ float2 f2(float x) { return make_float2(x, x); }

template <int FORM>
__global__ void __launch_bounds__(128, 6) k_pc(const float4 *__restrict__ rec, int nrec, int reps, float *out) {
  __shared__ float4 pcr[4][20][3];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = lane; i < 60; i += 32) pcr[w][i / 3][i % 3] = rec[(blockIdx.x * 7 + i) % nrec];
  __syncwarp();
  const unsigned bit = 1u << lane;
  const float4 t0 = rec[(blockIdx.x * 131 + threadIdx.x) % nrec];
  float2 X = make_float2(0.1f + t0.x * 1e-3f, 0.2f + t0.y * 1e-3f), Y = make_float2(0.3f + t0.z * 1e-3f, 0.31f - lane * 1e-3f),
         Z = make_float2(-0.2f - t0.x * 1e-4f, -0.21f);
  float2 AX = f2(0.f), AY = f2(0.f), AZ = f2(0.f);
  int pc0 = 0, pc1 = 0;
  for (int r = 0; r < reps; ++r) {
#pragma unroll 4
    for (int k = 0; k < 20; ++k) {
      const float4 a = pcr[w][k][0];
      const float4 b = pcr[w][k][1];
      const float4 q = pcr[w][k][2];
      const bool u0 = (unsigned)__float_as_int(a.w) & bit, u1 = (unsigned)__float_as_int(b.z) & bit;
      const float2 DX = __fadd2_rn(X, f2(a.x));
      const float2 DY = __fadd2_rn(Y, f2(a.y));
      const float2 DZ = __fadd2_rn(Z, f2(a.z));
      const float2 D2 = __ffma2_rn(DZ, DZ, __ffma2_rn(DY, DY, __fmul2_rn(DX, DX)));
      float2 R;
      if (FORM == 3) R = make_float2(rsqrtf(D2.x), rsqrtf(D2.y));  // no masking
      else if (FORM == 4) R = __fmul2_rn(D2, f2(0.37f));         // no MUFU
      else R = make_float2(u0 ? rsqrtf(D2.x) : 0.f, u1 ? rsqrtf(D2.y) : 0.f);
      const float2 R2 = __fmul2_rn(R, R);
      const float2 QX = __ffma2_rn(f2(q.x), DZ, __ffma2_rn(f2(b.y), DY, __fmul2_rn(f2(b.x), DX)));
      const float2 QY = __ffma2_rn(f2(q.y), DZ, __ffma2_rn(f2(b.w), DY, __fmul2_rn(f2(b.y), DX)));
      const float2 QZ = __ffma2_rn(f2(q.w), DZ, __ffma2_rn(f2(q.y), DY, __fmul2_rn(f2(q.x), DX)));
      if (FORM == 0 || FORM == 3 || FORM == 4) {  // k_walk9 (BH_W9_PC30)
        const float2 RQR = __ffma2_rn(DZ, QZ, __ffma2_rn(DY, QY, __fmul2_rn(DX, QX)));
        const float2 R5 = __fmul2_rn(__fmul2_rn(R2, R2), R);
        const float2 V = __ffma2_rn(__fmul2_rn(RQR, R2), f2(-2.5f), __fmul2_rn(f2(-q.z), D2));
        AX = __ffma2_rn(R5, __ffma2_rn(DX, V, QX), AX);
        AY = __ffma2_rn(R5, __ffma2_rn(DY, V, QY), AY);
        AZ = __ffma2_rn(R5, __ffma2_rn(DZ, V, QZ), AZ);
      } else if (FORM == 1) {  // scaled: T = R5*d, U = R5*Q d (3 + 3 FMUL2), A += T V + U
        const float2 RQR = __ffma2_rn(DZ, QZ, __ffma2_rn(DY, QY, __fmul2_rn(DX, QX)));
        const float2 R5 = __fmul2_rn(__fmul2_rn(R2, R2), R);
        const float2 V = __ffma2_rn(__fmul2_rn(RQR, R2), f2(-2.5f), __fmul2_rn(f2(-q.z), D2));
        const float2 W = __fmul2_rn(R5, V);
        AX = __ffma2_rn(W, DX, __ffma2_rn(R5, QX, AX));
        AY = __ffma2_rn(W, DY, __ffma2_rn(R5, QY, AY));
        AZ = __ffma2_rn(W, DZ, __ffma2_rn(R5, QZ, AZ));
      } else if (FORM == 6) {  // the 3-packed ops as scalar FFMAs per target
        const float2 RQ1 = __fmul2_rn(DX, QX);
        const float2 RQR = make_float2(fmaf(DZ.x, QZ.x, fmaf(DY.x, QY.x, RQ1.x)), fmaf(DZ.y, QZ.y, fmaf(DY.y, QY.y, RQ1.y)));
        const float2 R5 = __fmul2_rn(__fmul2_rn(R2, R2), R);
        const float2 V = __ffma2_rn(__fmul2_rn(RQR, R2), f2(-2.5f), __fmul2_rn(f2(-q.z), D2));
        AX = make_float2(fmaf(R5.x, fmaf(DX.x, V.x, QX.x), AX.x), fmaf(R5.y, fmaf(DX.y, V.y, QX.y), AX.y));
        AY = make_float2(fmaf(R5.x, fmaf(DY.x, V.x, QY.x), AY.x), fmaf(R5.y, fmaf(DY.y, V.y, QY.y), AY.y));
        AZ = make_float2(fmaf(R5.x, fmaf(DZ.x, V.x, QZ.x), AZ.x), fmaf(R5.y, fmaf(DZ.y, V.y, QZ.y), AZ.y));
      } else if (FORM == 7) {  // the 3-packed ops as FMUL2 + FADD2
        const float2 RQR = __fadd2_rn(__fmul2_rn(DZ, QZ), __fadd2_rn(__fmul2_rn(DY, QY), __fmul2_rn(DX, QX)));
        const float2 R5 = __fmul2_rn(__fmul2_rn(R2, R2), R);
        const float2 V = __ffma2_rn(__fmul2_rn(RQR, R2), f2(-2.5f), __fmul2_rn(f2(-q.z), D2));
        AX = __fadd2_rn(__fmul2_rn(R5, __fadd2_rn(__fmul2_rn(DX, V), QX)), AX);
        AY = __fadd2_rn(__fmul2_rn(R5, __fadd2_rn(__fmul2_rn(DY, V), QY)), AY);
        AZ = __fadd2_rn(__fmul2_rn(R5, __fadd2_rn(__fmul2_rn(DZ, V), QZ)), AZ);
      } else if (FORM >= 8 && FORM <= 10) {  // timing: one group of 3-packed ops given a broadcast operand
        const float2 RQR = FORM == 10 ? __ffma2_rn(DZ, f2(q.x), __ffma2_rn(DY, f2(b.x), __fmul2_rn(DX, QX)))
                                      : __ffma2_rn(DZ, QZ, __ffma2_rn(DY, QY, __fmul2_rn(DX, QX)));
        const float2 R5 = __fmul2_rn(__fmul2_rn(R2, R2), R);
        const float2 V = __ffma2_rn(__fmul2_rn(RQR, R2), f2(-2.5f), __fmul2_rn(f2(-q.z), D2));
        if (FORM == 8) {  // outer cheap
          AX = __ffma2_rn(R5, f2(b.w), __ffma2_rn(DX, V, QX));
          AY = __ffma2_rn(R5, f2(b.x), __ffma2_rn(DY, V, QY));
          AZ = __ffma2_rn(R5, f2(a.z), __ffma2_rn(DZ, V, QZ));
          AX = __fadd2_rn(AX, AY);
        } else if (FORM == 9) {  // inner cheap
          AX = __ffma2_rn(R5, __ffma2_rn(DX, f2(a.x), QX), AX);
          AY = __ffma2_rn(V, __ffma2_rn(DY, f2(a.y), QY), AY);
          AZ = __ffma2_rn(R5, __ffma2_rn(DZ, f2(a.z), QZ), AZ);
        } else {
          AX = __ffma2_rn(R5, __ffma2_rn(DX, V, QX), AX);
          AY = __ffma2_rn(R5, __ffma2_rn(DY, V, QY), AY);
          AZ = __ffma2_rn(R5, __ffma2_rn(DZ, V, QZ), AZ);
        }
      } else if (FORM == 5) {  // timing only: the 3-packed-operand ops given a broadcast operand
        const float2 RQR = __ffma2_rn(DZ, f2(q.x), __ffma2_rn(DY, f2(b.x), __fmul2_rn(DX, QX)));
        const float2 R5 = __fmul2_rn(__fmul2_rn(R2, R2), R);
        const float2 V = __ffma2_rn(__fmul2_rn(RQR, R2), f2(-2.5f), __fmul2_rn(f2(-q.z), D2));
        AX = __ffma2_rn(R5, f2(b.w), __ffma2_rn(DX, f2(a.x), QX));
        AY = __ffma2_rn(V, f2(b.w), __ffma2_rn(DY, f2(a.y), AY));
        AZ = __ffma2_rn(R5, f2(a.z), __ffma2_rn(DZ, f2(a.z), AZ));
      } else {  // FORM 2: scalar FFMA per target (no packing)
        float ax[2], ay[2], az[2];
        const float dxs[2] = {DX.x, DX.y}, dys[2] = {DY.x, DY.y}, dzs[2] = {DZ.x, DZ.y};
        const float d2s[2] = {D2.x, D2.y}, rs[2] = {R.x, R.y};
#pragma unroll
        for (int t = 0; t < 2; ++t) {
          const float dx = dxs[t], dy = dys[t], dz = dzs[t], r = rs[t], r2 = r * r;
          const float qx = fmaf(q.x, dz, fmaf(b.y, dy, b.x * dx));
          const float qy = fmaf(q.y, dz, fmaf(b.w, dy, b.y * dx));
          const float qz = fmaf(q.w, dz, fmaf(q.y, dy, q.x * dx));
          const float rqr = fmaf(dz, qz, fmaf(dy, qy, dx * qx));
          const float r5 = r2 * r2 * r;
          const float v = fmaf(rqr * r2, -2.5f, -q.z * d2s[t]);
          ax[t] = r5 * fmaf(dx, v, qx);
          ay[t] = r5 * fmaf(dy, v, qy);
          az[t] = r5 * fmaf(dz, v, qz);
        }
        AX = __fadd2_rn(AX, make_float2(ax[0], ax[1]));
        AY = __fadd2_rn(AY, make_float2(ay[0], ay[1]));
        AZ = __fadd2_rn(AZ, make_float2(az[0], az[1]));
      }
      pc0 += u0; pc1 += u1;
    }
  }
  const float s = AX.x + AX.y + AY.x + AY.y + AZ.x + AZ.y + pc0 + pc1;
  if (s == 1234.5f) out[0] = s;
}

template <int FORM>
static void run(const char *name, const float4 *rec, int sms, int blocks_per_sm) {
  float *out;
  cudaMalloc(&out, 4);
  const int reps = 400, blocks = sms * blocks_per_sm;
  k_pc<FORM><<<blocks, 128>>>(rec, 600, 2, out);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k_pc<FORM><<<blocks, 128>>>(rec, 600, reps, out);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  int khz;
  cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, 0);
  const double entries_per_smsp = (double)blocks * 4 * reps * 20 / (sms * 4);
  const double cyc = ms * 1e-3 * khz * 1e3;
  printf("%-28s %d blocks/SM: %.2f ms, %.1f SMSP cycles per warp-entry\n", name, blocks_per_sm, ms,
         cyc / entries_per_smsp);
  cudaFree(out);
}


// FORM 11-14: the pc30 body under different loop shapes
template <int UNR, bool REGREC, bool TWOACC>
__global__ void __launch_bounds__(128, 6) k_pc2(const float4 *__restrict__ rec, int nrec, int reps, float *out) {
  __shared__ float4 pcr[4][20][3];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = lane; i < 60; i += 32) pcr[w][i / 3][i % 3] = rec[(blockIdx.x * 7 + i) % nrec];
  __syncwarp();
  const unsigned bit = 1u << lane;
  const float4 t0 = rec[(blockIdx.x * 131 + threadIdx.x) % nrec];
  float2 X = make_float2(0.1f + t0.x * 1e-3f, 0.2f + t0.y * 1e-3f), Y = make_float2(0.3f + t0.z * 1e-3f, 0.31f - lane * 1e-3f),
         Z = make_float2(-0.2f - t0.x * 1e-4f, -0.21f);
  float2 AX[2] = {f2(0.f), f2(0.f)}, AY[2] = {f2(0.f), f2(0.f)}, AZ[2] = {f2(0.f), f2(0.f)};
  int pc0 = 0, pc1 = 0;
  float4 ra = pcr[w][0][0], rb = pcr[w][0][1], rq = pcr[w][0][2];
  for (int r = 0; r < reps; ++r) {
#pragma unroll UNR
    for (int k = 0; k < 20; ++k) {
      float4 a, b, q;
      if (REGREC) { a = ra; b = rb; q = rq; ra.x += 1e-7f; rb.y += 1e-9f; }
      else { a = pcr[w][k][0]; b = pcr[w][k][1]; q = pcr[w][k][2]; }
      const int s = TWOACC ? (k & 1) : 0;
      const bool u0 = (unsigned)__float_as_int(a.w) & bit, u1 = (unsigned)__float_as_int(b.z) & bit;
      const float2 DX = __fadd2_rn(X, f2(a.x));
      const float2 DY = __fadd2_rn(Y, f2(a.y));
      const float2 DZ = __fadd2_rn(Z, f2(a.z));
      const float2 D2 = __ffma2_rn(DZ, DZ, __ffma2_rn(DY, DY, __fmul2_rn(DX, DX)));
      const float2 R = make_float2(u0 ? rsqrtf(D2.x) : 0.f, u1 ? rsqrtf(D2.y) : 0.f);
      const float2 R2 = __fmul2_rn(R, R);
      const float2 QX = __ffma2_rn(f2(q.x), DZ, __ffma2_rn(f2(b.y), DY, __fmul2_rn(f2(b.x), DX)));
      const float2 QY = __ffma2_rn(f2(q.y), DZ, __ffma2_rn(f2(b.w), DY, __fmul2_rn(f2(b.y), DX)));
      const float2 QZ = __ffma2_rn(f2(q.w), DZ, __ffma2_rn(f2(q.y), DY, __fmul2_rn(f2(q.x), DX)));
      const float2 RQR = __ffma2_rn(DZ, QZ, __ffma2_rn(DY, QY, __fmul2_rn(DX, QX)));
      const float2 R5 = __fmul2_rn(__fmul2_rn(R2, R2), R);
      const float2 V = __ffma2_rn(__fmul2_rn(RQR, R2), f2(-2.5f), __fmul2_rn(f2(-q.z), D2));
      AX[s] = __ffma2_rn(R5, __ffma2_rn(DX, V, QX), AX[s]);
      AY[s] = __ffma2_rn(R5, __ffma2_rn(DY, V, QY), AY[s]);
      AZ[s] = __ffma2_rn(R5, __ffma2_rn(DZ, V, QZ), AZ[s]);
      pc0 += u0; pc1 += u1;
    }
  }
  const float s = AX[0].x + AX[0].y + AY[0].x + AY[0].y + AZ[0].x + AZ[0].y + AX[1].x + AY[1].y + AZ[1].x + pc0 + pc1;
  if (s == 1234.5f) out[0] = s;
}

template <int UNR, bool REGREC, bool TWOACC>
static void run2(const char *name, const float4 *rec, int sms, int blocks_per_sm) {
  float *out;
  cudaMalloc(&out, 4);
  const int reps = 400, blocks = sms * blocks_per_sm;
  k_pc2<UNR, REGREC, TWOACC><<<blocks, 128>>>(rec, 600, 2, out);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k_pc2<UNR, REGREC, TWOACC><<<blocks, 128>>>(rec, 600, reps, out);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  int khz;
  cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, 0);
  const double entries_per_smsp = (double)blocks * 4 * reps * 20 / (sms * 4);
  printf("%-28s %d blocks/SM: %.2f ms, %.1f SMSP cycles per warp-entry\n", name, blocks_per_sm, ms,
         ms * 1e-3 * khz * 1e3 / entries_per_smsp);
  cudaFree(out);
}


// 4 targets per lane: two float2 sets share each staged record
__global__ void __launch_bounds__(128, 6) k_pc4(const float4 *__restrict__ rec, int nrec, int reps, float *out) {
  __shared__ float4 pcr[4][20][3];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = lane; i < 60; i += 32) pcr[w][i / 3][i % 3] = rec[(blockIdx.x * 7 + i) % nrec];
  __syncwarp();
  const unsigned bit = 1u << lane;
  const float4 t0 = rec[(blockIdx.x * 131 + threadIdx.x) % nrec];
  float2 X[2], Y[2], Z[2], AX[2], AY[2], AZ[2];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    X[h] = make_float2(0.1f + t0.x * 1e-3f + h * 1e-3f, 0.2f + t0.y * 1e-3f);
    Y[h] = make_float2(0.3f + t0.z * 1e-3f, 0.31f - lane * 1e-3f + h * 1e-3f);
    Z[h] = make_float2(-0.2f - t0.x * 1e-4f, -0.21f - h * 1e-3f);
    AX[h] = AY[h] = AZ[h] = f2(0.f);
  }
  int pc0 = 0, pc1 = 0;
  for (int r = 0; r < reps; ++r) {
#pragma unroll 2
    for (int k = 0; k < 20; ++k) {
      const float4 a = pcr[w][k][0];
      const float4 b = pcr[w][k][1];
      const float4 q = pcr[w][k][2];
      const bool u0 = (unsigned)__float_as_int(a.w) & bit, u1 = (unsigned)__float_as_int(b.z) & bit;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const float2 DX = __fadd2_rn(X[h], f2(a.x));
        const float2 DY = __fadd2_rn(Y[h], f2(a.y));
        const float2 DZ = __fadd2_rn(Z[h], f2(a.z));
        const float2 D2 = __ffma2_rn(DZ, DZ, __ffma2_rn(DY, DY, __fmul2_rn(DX, DX)));
        const float2 R = make_float2(u0 ? rsqrtf(D2.x) : 0.f, u1 ? rsqrtf(D2.y) : 0.f);
        const float2 R2 = __fmul2_rn(R, R);
        const float2 QX = __ffma2_rn(f2(q.x), DZ, __ffma2_rn(f2(b.y), DY, __fmul2_rn(f2(b.x), DX)));
        const float2 QY = __ffma2_rn(f2(q.y), DZ, __ffma2_rn(f2(b.w), DY, __fmul2_rn(f2(b.y), DX)));
        const float2 QZ = __ffma2_rn(f2(q.w), DZ, __ffma2_rn(f2(q.y), DY, __fmul2_rn(f2(q.x), DX)));
        const float2 RQR = __ffma2_rn(DZ, QZ, __ffma2_rn(DY, QY, __fmul2_rn(DX, QX)));
        const float2 R5 = __fmul2_rn(__fmul2_rn(R2, R2), R);
        const float2 V = __ffma2_rn(__fmul2_rn(RQR, R2), f2(-2.5f), __fmul2_rn(f2(-q.z), D2));
        AX[h] = __ffma2_rn(R5, __ffma2_rn(DX, V, QX), AX[h]);
        AY[h] = __ffma2_rn(R5, __ffma2_rn(DY, V, QY), AY[h]);
        AZ[h] = __ffma2_rn(R5, __ffma2_rn(DZ, V, QZ), AZ[h]);
      }
      pc0 += u0; pc1 += u1;
    }
  }
  const float s = AX[0].x + AX[0].y + AY[0].x + AY[0].y + AZ[0].x + AZ[0].y + AX[1].x + AX[1].y + AY[1].x + AY[1].y + AZ[1].x + AZ[1].y + pc0 + pc1;
  if (s == 1234.5f) out[0] = s;
}
static void run4(const float4 *rec, int sms, int blocks_per_sm) {
  float *out;
  cudaMalloc(&out, 4);
  const int reps = 400, blocks = sms * blocks_per_sm;
  k_pc4<<<blocks, 128>>>(rec, 600, 2, out);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k_pc4<<<blocks, 128>>>(rec, 600, reps, out);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  int khz;
  cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, 0);
  const double entries_per_smsp = (double)blocks * 4 * reps * 20 / (sms * 4);
  printf("%-28s %d blocks/SM: %.2f ms, %.1f SMSP cycles per warp-entry (128 targets)\n", "4 targets per lane", blocks_per_sm, ms,
         ms * 1e-3 * khz * 1e3 / entries_per_smsp);
  cudaFree(out);
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float4 h[600];
  for (int i = 0; i < 600; ++i) {
    const float t = 0.37f * i;
    h[i] = make_float4(-1.5f - 0.1f * __builtin_sinf(t), 0.8f + 0.05f * __builtin_cosf(t), 0.4f, bits_f(-1));
    if (i % 3 == 1) h[i] = make_float4(1e-3f, 2e-4f, bits_f(-1), 3e-4f);
    if (i % 3 == 2) h[i] = make_float4(-1e-4f, 5e-4f, 0.01f, -7e-4f);
  }
  float4 *rec;
  cudaMalloc(&rec, sizeof(h));
  cudaMemcpy(rec, h, sizeof(h), cudaMemcpyHostToDevice);
  for (int bps : {6}) {
    run<0>("pc30 (k_walk9)", rec, sms, bps);
    run<1>("pc31 split accumulate", rec, sms, bps);
    run<2>("scalar per target", rec, sms, bps);
    run<3>("pc30 unmasked", rec, sms, bps);
    run<4>("pc30 no MUFU", rec, sms, bps);
    run<5>("pc30 no 3-packed ops (timing)", rec, sms, bps);
    run<6>("3-packed ops as scalar FFMA", rec, sms, bps);
    run<7>("3-packed ops as FMUL2+FADD2", rec, sms, bps);
    run2<1, false, false>("unroll 1", rec, sms, bps);
    run2<2, false, false>("unroll 2", rec, sms, bps);
    run2<4, false, false>("unroll 4", rec, sms, bps);
    run2<8, false, false>("unroll 8", rec, sms, bps);
    run2<4, true, false>("unroll 4, records in regs", rec, sms, bps);
    run2<4, false, true>("unroll 4, two accumulators", rec, sms, bps);
    run4(rec, sms, bps);
    run4(rec, sms, 4);
  }
  return 0;
}
