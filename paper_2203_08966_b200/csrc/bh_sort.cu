// bh_sort.cu -- hand-written stable LSD radix sort of (u64 key, u32 value)
// pairs over bits [0, 63) and single-pass u32 scans, for sm_100a.
//
// Replaces np.argsort(keys, kind="stable") (morton.py:128-130): the sorted
// order is the stable one (ties keep their input order), bit for bit.
//
// Sort = one histogram pass + 8 digit passes of 8 bits ("onesweep"):
//   k_sort_hist   one read of the keys: the 8 digit histograms (run-length
//                 aggregated shared-memory atomics, one global add per bin and
//                 block)
//   k_sort_pass   per 4096-key tile: load (coalesced, warp-striped), rank every
//                 key inside its warp with __match_any_sync (stable: lanes and
//                 items in input order), warp offsets per digit, publish the
//                 tile's digit counts, decoupled look-back over the previous
//                 tiles for each digit's global offset, local reorder through
//                 shared memory, and a run-coalesced scatter of keys and values
// Tiles take their index from an atomic counter in launch order, so every
// tile's predecessors are running or done (the look-back always terminates).
// Look-back words carry a flag, a per-pass epoch and the count in one 64-bit
// store, so the status array is never cleared between passes or calls.
//
// Algorithmic traffic: 8 passes x (8 + 4) B x (read + write)
// = 192 B/body, plus 8 B/body for the histogram read.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <atomic>

#include "bh_internal.cuh"

namespace bh {

namespace {

constexpr int kDigitBits = 8;
constexpr int kBins = 1 << kDigitBits;
constexpr int kPasses = 8;  // 64 bits; the top pass sees bits 56..62 (bit 63 is 0)
constexpr int kSortThreads = 256;
constexpr int kSortItems = 16;
constexpr int kTile = kSortThreads * kSortItems;  // 4096 keys
constexpr int kSortWarps = kSortThreads / 32;
static_assert(kSortThreads == kBins, "one thread per digit");
constexpr int kHistThreads = 256;
constexpr int kHistItems = 16;

// look-back / status word: flag (2 bits) | epoch (30 bits) | value (32 bits)
constexpr unsigned long long kFlagAgg = 1ull << 62;
constexpr unsigned long long kFlagInc = 2ull << 62;
constexpr unsigned long long kValMask = 0xffffffffull;
constexpr unsigned long long kEpochMask = 0x3fffffffull;

std::atomic<unsigned long long> g_epoch{0};
// a fresh, process-wide unique epoch (1 .. 2^30-1): status words written by an
// earlier pass or call never match it, so no clearing is needed
inline unsigned next_epoch() {
  const unsigned long long e = g_epoch.fetch_add(1) % kEpochMask;
  return (unsigned)e + 1u;
}

__device__ __forceinline__ unsigned long long ld_status(const unsigned long long *p) {
  return *reinterpret_cast<const volatile unsigned long long *>(p);
}
__device__ __forceinline__ void st_status(unsigned long long *p, unsigned long long v) {
  *reinterpret_cast<volatile unsigned long long *>(p) = v;
}
__device__ __forceinline__ unsigned long long pack(unsigned long long flag, unsigned epoch, unsigned v) {
  return flag | ((unsigned long long)epoch << 32) | v;
}

// temp layout (all offsets 256-byte aligned)
struct SortTemp {
  uint64_t *k;             // [n] ping-pong keys
  uint32_t *v;             // [n] ping-pong values
  unsigned *hist;          // [kPasses][kBins] global digit histograms
  unsigned *counters;      // [kPasses] tile counters (self-resetting)
  unsigned long long *st;  // [tiles][kBins] look-back status
};
inline size_t al(size_t x) { return (x + 255) & ~size_t(255); }
inline int64_t sort_tiles(int64_t n) { return (n + kTile - 1) / kTile; }
inline SortTemp carve_sort(void *temp, int64_t n) {
  char *p = static_cast<char *>(temp);
  SortTemp t;
  t.k = reinterpret_cast<uint64_t *>(p); p += al(sizeof(uint64_t) * n);
  t.v = reinterpret_cast<uint32_t *>(p); p += al(sizeof(uint32_t) * n);
  t.hist = reinterpret_cast<unsigned *>(p); p += al(sizeof(unsigned) * kPasses * kBins);
  t.counters = reinterpret_cast<unsigned *>(p); p += al(sizeof(unsigned) * kPasses);
  t.st = reinterpret_cast<unsigned long long *>(p);
  return t;
}

// ------------------------------------------------------------ histograms
// Each thread reads kHistItems consecutive keys (16-byte loads) and adds run
// lengths: along the Morton-sorted resident order the high digits rarely
// change, so most of the 8 x 16 digit updates fold into one add.
__global__ void __launch_bounds__(kHistThreads) k_sort_hist(const uint64_t *__restrict__ keys, int64_t n,
                                                            unsigned *__restrict__ hist) {
  __shared__ unsigned sh[kPasses][kBins];
  for (int i = threadIdx.x; i < kPasses * kBins; i += kHistThreads) (&sh[0][0])[i] = 0u;
  __syncthreads();
  const int64_t chunk = (int64_t)kHistThreads * kHistItems;
  for (int64_t base = (int64_t)blockIdx.x * chunk; base < n; base += (int64_t)gridDim.x * chunk) {
    const int64_t i0 = base + (int64_t)threadIdx.x * kHistItems;
    uint64_t k[kHistItems];
    if (i0 + kHistItems <= n) {
      const ulonglong2 *src = reinterpret_cast<const ulonglong2 *>(keys + i0);
#pragma unroll
      for (int j = 0; j < kHistItems / 2; ++j) {
        const ulonglong2 v = __ldcs(src + j);
        k[2 * j] = v.x;
        k[2 * j + 1] = v.y;
      }
    } else {
#pragma unroll
      for (int j = 0; j < kHistItems; ++j) k[j] = i0 + j < n ? keys[i0 + j] : ~0ull;
    }
    const int64_t left = n - i0;
    const int cnt = left >= kHistItems ? kHistItems : (left > 0 ? (int)left : 0);
    if (cnt == 0) continue;
#pragma unroll
    for (int p = 0; p < kPasses; ++p) {
      unsigned d = (unsigned)(k[0] >> (kDigitBits * p)) & (kBins - 1);
      unsigned run = 1;
#pragma unroll
      for (int j = 1; j < kHistItems; ++j) {
        if (j >= cnt) break;
        const unsigned e = (unsigned)(k[j] >> (kDigitBits * p)) & (kBins - 1);
        if (e == d) {
          ++run;
        } else {
          atomicAdd(&sh[p][d], run);
          d = e;
          run = 1;
        }
      }
      atomicAdd(&sh[p][d], run);
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < kPasses * kBins; i += kHistThreads) {
    const unsigned v = (&sh[0][0])[i];
    if (v) atomicAdd(hist + i, v);
  }
}

__global__ void k_sort_zero(unsigned *hist, unsigned *counters) {
  for (int i = threadIdx.x; i < kPasses * kBins; i += blockDim.x) hist[i] = 0u;
  if (threadIdx.x < kPasses) counters[threadIdx.x] = 0u;
}

// ------------------------------------------------------------ one digit pass
struct PassSmem {
  uint64_t keys[kTile];
  uint32_t vals[kTile];
  unsigned whist[kSortWarps][kBins];  // per warp: running counts, then exclusive offsets
  unsigned start[kBins];              // exclusive digit offsets inside the tile
  long long gdelta[kBins];            // global position - tile position, per digit
  unsigned bin_start[kBins];          // exclusive scan of the global histogram
  unsigned wsum[kSortWarps];
  unsigned tile;
};

// exclusive scan of v over the block's 256 threads (one value per thread)
__device__ __forceinline__ unsigned block_excl_scan(unsigned v, unsigned *wsum, unsigned *total) {
  const unsigned lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  unsigned incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= (unsigned)o) incl += t;
  }
  if (lane == 31) wsum[w] = incl;
  __syncthreads();
  unsigned woff = 0, tot = 0;
#pragma unroll
  for (int i = 0; i < kSortWarps; ++i) {
    const unsigned s = wsum[i];
    woff += i < (int)w ? s : 0u;
    tot += s;
  }
  if (total) *total = tot;
  __syncthreads();  // wsum reusable
  return woff + incl - v;
}

__global__ void __launch_bounds__(kSortThreads) k_sort_pass(
    const uint64_t *__restrict__ kin, const uint32_t *__restrict__ vin, uint64_t *__restrict__ kout,
    uint32_t *__restrict__ vout, int64_t n, int shift, const unsigned *__restrict__ hist,
    unsigned *__restrict__ counter, unsigned long long *__restrict__ st, unsigned epoch, unsigned ntiles) {
  extern __shared__ __align__(16) unsigned char sort_smem[];
  PassSmem &S = *reinterpret_cast<PassSmem *>(sort_smem);
  const unsigned lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const unsigned FULL = 0xffffffffu;
  if (threadIdx.x == 0) {
    const unsigned t = atomicAdd(counter, 1u);
    if (t == ntiles - 1) *counter = 0u;  // every block has taken its tile: reset for the next launch
    S.tile = t;
  }
  // global digit offsets (the 256 bins of this pass), zeroed warp counts
  const unsigned hv = hist[threadIdx.x];
  for (int i = threadIdx.x; i < kSortWarps * kBins; i += kSortThreads) (&S.whist[0][0])[i] = 0u;
  {
    unsigned tot;
    S.bin_start[threadIdx.x] = block_excl_scan(hv, S.wsum, &tot);
  }
  const unsigned tile = S.tile;  // ordered by the barriers inside the scan
  const int64_t tbase = (int64_t)tile * kTile;
  const int64_t wbase = tbase + (int64_t)w * 32 * kSortItems;

  // ---- load (warp-striped: item j of lane l is key wbase + 32 j + l)
  uint64_t k[kSortItems];
  uint32_t v[kSortItems];
#pragma unroll
  for (int j = 0; j < kSortItems; ++j) {
    const int64_t i = wbase + 32 * j + lane;
    if (i < n) {
      k[j] = __ldcs(kin + i);
      v[j] = __ldcs(vin + i);
    } else {
      k[j] = ~0ull;  // pads sort after every real key of the last tile and are never stored
      v[j] = 0u;
    }
  }

  // ---- stable rank inside the warp (items in order, lanes in order)
  unsigned rank[kSortItems];
  unsigned *wh = S.whist[w];
  const unsigned lt = (1u << lane) - 1u;
#pragma unroll
  for (int j = 0; j < kSortItems; ++j) {
    const unsigned d = (unsigned)(k[j] >> shift) & (kBins - 1);
    const unsigned peers = __match_any_sync(FULL, d);
    const unsigned base = wh[d];
    __syncwarp();
    const unsigned leader = 31u - __clz(peers);
    if (lane == leader) wh[d] = base + __popc(peers);
    __syncwarp();
    rank[j] = base + __popc(peers & lt);
  }
  __syncthreads();

  // ---- per digit: warp offsets, tile count, tile offsets; publish the count
  const unsigned d = threadIdx.x;  // kSortThreads == kBins
  unsigned cnt = 0;
#pragma unroll
  for (int i = 0; i < kSortWarps; ++i) {
    const unsigned c = S.whist[i][d];
    S.whist[i][d] = cnt;
    cnt += c;
  }
  unsigned long long *my = st + (size_t)tile * kBins + d;
  if (tile == 0) st_status(my, pack(kFlagInc, epoch, cnt));
  else st_status(my, pack(kFlagAgg, epoch, cnt));
  S.start[d] = block_excl_scan(cnt, S.wsum, nullptr);  // (its barriers publish the whist offsets)
  __syncthreads();

  // ---- local reorder into shared memory
#pragma unroll
  for (int j = 0; j < kSortItems; ++j) {
    const unsigned dj = (unsigned)(k[j] >> shift) & (kBins - 1);
    const unsigned lp = S.start[dj] + S.whist[w][dj] + rank[j];
    S.keys[lp] = k[j];
    S.vals[lp] = v[j];
  }

  // ---- decoupled look-back for digit d
  unsigned excl = 0;
  if (tile > 0) {
    int64_t j = (int64_t)tile - 1;
    for (;;) {
      const unsigned long long s = ld_status(st + (size_t)j * kBins + d);
      if ((unsigned)((s >> 32) & kEpochMask) != epoch || (s >> 62) == 0) continue;  // not yet published
      excl += (unsigned)(s & kValMask);
      if ((s >> 62) == 2ull) break;
      --j;
    }
    st_status(my, pack(kFlagInc, epoch, excl + cnt));
  }
  S.gdelta[d] = (long long)S.bin_start[d] + excl - (long long)S.start[d];
  __syncthreads();

  // ---- scatter: consecutive tile slots of one digit go to consecutive addresses
#pragma unroll 4
  for (int i = threadIdx.x; i < kTile; i += kSortThreads) {
    const uint64_t key = S.keys[i];
    const unsigned di = (unsigned)(key >> shift) & (kBins - 1);
    const long long g = S.gdelta[di] + i;
    if (g < n) {
      kout[g] = key;
      vout[g] = S.vals[i];
    }
  }
}

// ------------------------------------------------------------------ scan
constexpr int kScanThreads = 256;
constexpr int kScanItems = 16;
constexpr int kScanTile = kScanThreads * kScanItems;

struct ScanTemp {
  unsigned *counter;
  unsigned long long *st;  // [tiles]
};
inline ScanTemp carve_scan(void *temp) {
  char *p = static_cast<char *>(temp);
  ScanTemp t;
  t.counter = reinterpret_cast<unsigned *>(p);
  t.st = reinterpret_cast<unsigned long long *>(p + 256);
  return t;
}

template <bool INCLUSIVE>
__global__ void __launch_bounds__(kScanThreads) k_scan_u32(const uint32_t *__restrict__ in, uint32_t *__restrict__ out,
                                                           int64_t n, unsigned *counter, unsigned long long *st,
                                                           unsigned epoch, unsigned ntiles) {
  __shared__ unsigned s_wsum[kScanThreads / 32];
  __shared__ unsigned s_tile, s_prefix;
  const unsigned lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    const unsigned t = atomicAdd(counter, 1u);
    if (t == ntiles - 1) *counter = 0u;
    s_tile = t;
  }
  __syncthreads();
  const unsigned tile = s_tile;
  const int64_t i0 = (int64_t)tile * kScanTile + (int64_t)threadIdx.x * kScanItems;
  unsigned x[kScanItems];
  if (i0 + kScanItems <= n && ((reinterpret_cast<uintptr_t>(in) & 15) == 0)) {
    const uint4 *src = reinterpret_cast<const uint4 *>(in + i0);
#pragma unroll
    for (int j = 0; j < kScanItems / 4; ++j) {
      const uint4 q = src[j];
      x[4 * j] = q.x; x[4 * j + 1] = q.y; x[4 * j + 2] = q.z; x[4 * j + 3] = q.w;
    }
  } else {
#pragma unroll
    for (int j = 0; j < kScanItems; ++j) x[j] = i0 + j < n ? in[i0 + j] : 0u;
  }
  unsigned sum = 0;
#pragma unroll
  for (int j = 0; j < kScanItems; ++j) sum += x[j];
  // block scan of the thread sums
  unsigned incl = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= (unsigned)o) incl += t;
  }
  if (lane == 31) s_wsum[w] = incl;
  __syncthreads();
  unsigned woff = 0, tot = 0;
#pragma unroll
  for (int i = 0; i < kScanThreads / 32; ++i) {
    const unsigned s = s_wsum[i];
    woff += i < (int)w ? s : 0u;
    tot += s;
  }
  // look-back by warp 0: 32 predecessors per step
  if (w == 0) {
    unsigned prefix = 0;
    if (tile == 0) {
      if (lane == 0) st_status(st, pack(kFlagInc, epoch, tot));
    } else {
      if (lane == 0) st_status(st + tile, pack(kFlagAgg, epoch, tot));
      int64_t j = (int64_t)tile - 1 - lane;  // this lane's predecessor
      for (;;) {
        unsigned long long s = 0;
        bool ready = true;
        if (j >= 0) {
          s = ld_status(st + j);
          ready = (unsigned)((s >> 32) & kEpochMask) == epoch && (s >> 62) != 0;
        }
        if (!__all_sync(0xffffffffu, ready)) continue;
        // lanes past tile 0 contribute nothing; the nearest inclusive entry ends the walk
        const bool inc = j >= 0 && (s >> 62) == 2ull;
        const unsigned incmask = __ballot_sync(0xffffffffu, inc || j < 0);
        const unsigned first = incmask ? __ffs(incmask) - 1 : 32u;  // nearest inclusive
        unsigned val = (j >= 0 && lane <= first) ? (unsigned)(s & kValMask) : 0u;
#pragma unroll
        for (int o = 16; o; o >>= 1) val += __shfl_xor_sync(0xffffffffu, val, o);
        prefix += val;
        if (incmask) break;
        j -= 32;
      }
      if (lane == 0) st_status(st + tile, pack(kFlagInc, epoch, prefix + tot));
    }
    if (lane == 0) s_prefix = prefix;
  }
  __syncthreads();
  unsigned run = s_prefix + woff + incl - sum;
#pragma unroll
  for (int j = 0; j < kScanItems; ++j) {
    if (INCLUSIVE) run += x[j];
    if (i0 + j < n) out[i0 + j] = run;
    if (!INCLUSIVE) run += x[j];
  }
}

inline size_t scan_bytes(int64_t n) {
  const int64_t tiles = std::max<int64_t>(1, (n + kScanTile - 1) / kScanTile);
  return 256 + sizeof(unsigned long long) * (size_t)tiles;
}

template <bool INCLUSIVE>
cudaError_t scan_u32(void *temp, size_t temp_bytes, const uint32_t *in, uint32_t *out, int64_t n, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  if (temp_bytes < scan_bytes(n)) return cudaErrorInvalidValue;
  const int64_t tiles = (n + kScanTile - 1) / kScanTile;
  if (tiles > 0x7fffffff) return cudaErrorInvalidValue;
  ScanTemp t = carve_scan(temp);
  k_scan_u32<INCLUSIVE><<<(unsigned)tiles, kScanThreads, 0, s>>>(in, out, n, t.counter, t.st, next_epoch(),
                                                                  (unsigned)tiles);
  return cudaGetLastError();
}

}  // namespace

size_t sort_temp_bytes(int64_t n) {
  const int64_t tiles = std::max<int64_t>(1, sort_tiles(n));
  return al(sizeof(uint64_t) * n) + al(sizeof(uint32_t) * n) + al(sizeof(unsigned) * kPasses * kBins) +
         al(sizeof(unsigned) * kPasses) + sizeof(unsigned long long) * kBins * (size_t)tiles;
}

cudaError_t sort_pairs(void *temp, size_t temp_bytes, const uint64_t *kin, uint64_t *kout, const uint32_t *vin,
                       uint32_t *vout, int64_t n, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  if (temp_bytes < sort_temp_bytes(n) || n > 0x7fffffffll) return cudaErrorInvalidValue;
  SortTemp t = carve_sort(temp, n);
  const unsigned tiles = (unsigned)sort_tiles(n);
  static bool init = false;
  if (!init) {
    cudaFuncSetAttribute(k_sort_pass, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(PassSmem));
    init = true;
  }
  k_sort_zero<<<1, 256, 0, s>>>(t.hist, t.counters);
  {
    static int sms = 0;
    if (!sms) {
      int dev = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    }
    const int64_t need = (n + kHistThreads * kHistItems - 1) / (kHistThreads * kHistItems);
    const int g = (int)std::max<int64_t>(1, std::min<int64_t>(need, 2 * sms));
    k_sort_hist<<<g, kHistThreads, 0, s>>>(kin, n, t.hist);
  }
  // 8 passes ping-pong between the temp pair and the output (even count: ends in kout)
  const uint64_t *ka = kin;
  const uint32_t *va = vin;
  for (int p = 0; p < kPasses; ++p) {
    uint64_t *kb = (p & 1) ? kout : t.k;
    uint32_t *vb = (p & 1) ? vout : t.v;
    k_sort_pass<<<tiles, kSortThreads, sizeof(PassSmem), s>>>(ka, va, kb, vb, n, kDigitBits * p, t.hist + p * kBins,
                                                               t.counters + p, t.st, next_epoch(), tiles);
    ka = kb;
    va = vb;
  }
  return cudaGetLastError();
}

size_t scan_temp_bytes(int64_t n) { return scan_bytes(n); }
size_t inclusive_scan_temp_bytes(int64_t n) { return scan_bytes(n); }
cudaError_t exclusive_scan_u32(void *temp, size_t temp_bytes, const uint32_t *in, uint32_t *out, int64_t n,
                               cudaStream_t s) {
  return scan_u32<false>(temp, temp_bytes, in, out, n, s);
}
cudaError_t inclusive_scan_u32(void *temp, size_t temp_bytes, const uint32_t *in, uint32_t *out, int64_t n,
                               cudaStream_t s) {
  return scan_u32<true>(temp, temp_bytes, in, out, n, s);
}

// number of kernels one sort_pairs / scan call launches (instrumentation)
int sort_launches() { return 2 + kPasses; }

}  // namespace bh
