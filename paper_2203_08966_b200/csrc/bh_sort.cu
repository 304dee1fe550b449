// bh_sort.cu -- hand-written stable LSD radix sort of (u64 key, u32 value)
// pairs over bits [0, 63) and u32 prefix sums, for sm_100a.
//
// Replaces np.argsort(keys, kind="stable") (morton.py:128-130): the sorted
// order is the stable one (ties keep their input order), bit for bit.
//
// Sort = one histogram pass + 8 digit passes of 8 bits ("onesweep"):
//   k_sort_hist   one read of the keys: the 8 digit histograms (run-length
//                 aggregated shared-memory atomics, one global add per bin and
//                 block)
//   k_sort_pass   per 4096-key tile: load (coalesced, warp-striped), rank every
//                 key inside its warp (peer lanes from 8 ballots, one per digit
//                 bit: stable, lanes and items in input order; MATCH.ANY was
//                 38% of the stall samples), warp offsets per digit, publish the
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
#include <cstdlib>

#include "bh_internal.cuh"

namespace bh {

namespace {

constexpr int kDigitBits = 8;
constexpr int kBins = 1 << kDigitBits;
constexpr int kPasses = 8;  // 64 bits; the top pass sees bits 56..62 (bit 63 is 0)
#ifndef BH_SORT_ITEMS
#define BH_SORT_ITEMS 16
#endif
#ifndef BH_SORT_VIDX
#define BH_SORT_VIDX 0  // 1: the tile keeps each key's position (u16), values are read at the scatter
#endif
#ifndef BH_SORT_MATCH_TOP
#define BH_SORT_MATCH_TOP 1  // the top passes whose peer masks come from MATCH.ANY (few digit values per warp)
#endif
#ifndef BH_SORT_UNIFORM
#define BH_SORT_UNIFORM 0  // 1: a warp whose 32 keys share the digit skips the ballots
#endif
#ifndef BH_SORT_BLOCKS
#define BH_SORT_BLOCKS 3  // pass-kernel blocks per SM the register budget is set for
#endif
constexpr int kSortThreads = 256;
constexpr int kSortItems = BH_SORT_ITEMS;
constexpr int kTile = kSortThreads * kSortItems;  // 4096 keys
constexpr int kSortWarps = kSortThreads / 32;
static_assert(kSortThreads == kBins, "one thread per digit");
constexpr int kHistThreads = 256;

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
  unsigned *bin_start;     // [kPasses][kBins] their exclusive scans
  unsigned *counters;      // [kPasses] tile counters (self-resetting); [kPasses]: histogram blocks done
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
  t.bin_start = reinterpret_cast<unsigned *>(p); p += al(sizeof(unsigned) * kPasses * kBins);
  t.counters = reinterpret_cast<unsigned *>(p); p += al(sizeof(unsigned) * (kPasses + 1));
  t.st = reinterpret_cast<unsigned long long *>(p);
  return t;
}

// ------------------------------------------------------------ histograms
// One read of the keys for all 8 digit histograms: a shared-memory add per key
// and digit, except that a warp whose 32 consecutive keys share a digit adds
// 32 once (along the Morton-sorted resident order the high digits are
// warp-uniform; same-address atomics from 32 lanes would serialise).  The last
// block to finish turns the histograms into exclusive bin offsets.
constexpr int kHistUnroll = 4;
constexpr int kHistParts = 4;  // interleaved copies: fewer bank conflicts between lanes
static_assert(kDigitBits == 8 && kPasses == 8, "byte digits: 4 from each 32-bit half of the key");
__global__ void __launch_bounds__(kHistThreads) k_sort_hist(const uint64_t *__restrict__ keys, int64_t n,
                                                            unsigned *__restrict__ hist,
                                                            unsigned *__restrict__ bin_start,
                                                            unsigned *__restrict__ done) {
  extern __shared__ unsigned hist_smem[];  // [kPasses][kBins][kHistParts]
  __shared__ bool last;
  for (int i = threadIdx.x; i < kPasses * kBins * kHistParts; i += kHistThreads) hist_smem[i] = 0u;
  __syncthreads();
  const unsigned lane = threadIdx.x & 31, FULL = 0xffffffffu, part = lane % kHistParts;
  const int64_t wglobal = ((int64_t)blockIdx.x * kHistThreads + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * kHistThreads) >> 5;
  for (int64_t base = wglobal * 32 * kHistUnroll; base < n; base += nwarps * 32 * kHistUnroll) {
    uint64_t k[kHistUnroll];
#pragma unroll
    for (int u = 0; u < kHistUnroll; ++u) {
      const int64_t i = base + 32 * u + lane;
      k[u] = i < n ? __ldcs(keys + i) : 0ull;
    }
#pragma unroll
    for (int u = 0; u < kHistUnroll; ++u) {
      const bool valid = base + 32 * u + lane < n;
      const unsigned lo = (unsigned)k[u], hi = (unsigned)(k[u] >> 32);
      if (valid) {  // the low bytes vary from key to key
#pragma unroll
        for (int p = 0; p < 4; ++p)
          atomicAdd(&hist_smem[(p * kBins + ((lo >> (8 * p)) & 0xffu)) * kHistParts + part], 1u);
      }
      // the high bytes are mostly shared by a warp's 32 consecutive keys
      const unsigned hi0 = __shfl_sync(FULL, hi, 0);
      const unsigned vm = __ballot_sync(FULL, valid);
      if (__all_sync(FULL, !valid || hi == hi0)) {
        if (lane < 4) atomicAdd(&hist_smem[((4 + lane) * kBins + ((hi0 >> (8 * lane)) & 0xffu)) * kHistParts],
                                (unsigned)__popc(vm));
      } else if (valid) {
#pragma unroll
        for (int p = 0; p < 4; ++p)
          atomicAdd(&hist_smem[((4 + p) * kBins + ((hi >> (8 * p)) & 0xffu)) * kHistParts + part], 1u);
      }
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < kPasses * kBins; i += kHistThreads) {
    unsigned v = 0;
#pragma unroll
    for (int q = 0; q < kHistParts; ++q) v += hist_smem[i * kHistParts + q];
    if (v) atomicAdd(hist + i, v);
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned t = atomicAdd(done, 1u);
    last = t == gridDim.x - 1;
    if (last) *done = 0u;  // every block has counted: reset for the next call
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  // exclusive scans of the 8 histograms (warp p handles pass p; 8 bins per lane)
  const int w = threadIdx.x >> 5;
  if (w < kPasses) {
    const volatile unsigned *hp = hist + w * kBins;
    unsigned v[kBins / 32], run = 0;
#pragma unroll
    for (int q = 0; q < kBins / 32; ++q) {
      v[q] = hp[lane * (kBins / 32) + q];
      run += v[q];
    }
    unsigned incl = run;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned t = __shfl_up_sync(FULL, incl, o);
      if (lane >= (unsigned)o) incl += t;
    }
    unsigned ex = incl - run;
#pragma unroll
    for (int q = 0; q < kBins / 32; ++q) {
      bin_start[w * kBins + lane * (kBins / 32) + q] = ex;
      ex += v[q];
    }
  }
}

__global__ void k_sort_zero(unsigned *hist, unsigned *counters) {
  for (int i = threadIdx.x; i < kPasses * kBins; i += blockDim.x) hist[i] = 0u;
  if (threadIdx.x <= kPasses) counters[threadIdx.x] = 0u;
}

// ------------------------------------------------------------ one digit pass
struct PassSmem {
  uint64_t keys[kTile];
#if BH_SORT_VIDX
  uint16_t vidx[kTile];  // tile position of the key in each sorted slot (values read at the scatter)
#else
  uint32_t vals[kTile];
#endif
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

#ifndef BH_SORT_FULL_LOAD
#define BH_SORT_FULL_LOAD 0  // 1: full tiles load without bounds tests (cfg3 -1.9%, cfg4 +1.7%)
#endif
#ifndef BH_SORT_FULL_SCATTER
#define BH_SORT_FULL_SCATTER 1
#endif
#ifndef BH_SORT_RANKASM
#define BH_SORT_RANKASM 1
#endif
template <int MINB, bool MATCH>
__global__ void __launch_bounds__(kSortThreads, MINB) k_sort_pass(
    const uint64_t *__restrict__ kin, const uint32_t *vin, uint64_t *__restrict__ kout,
    uint32_t *__restrict__ vout, int64_t n, int shift, const unsigned *__restrict__ bin_start,
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
  S.bin_start[threadIdx.x] = bin_start[threadIdx.x];
  for (int i = threadIdx.x; i < kSortWarps * kBins; i += kSortThreads) (&S.whist[0][0])[i] = 0u;
  __syncthreads();
  const unsigned tile = S.tile;
  const int64_t tbase = (int64_t)tile * kTile;
  const int64_t wbase = tbase + (int64_t)w * 32 * kSortItems;

  // ---- load (warp-striped: item j of lane l is key wbase + 32 j + l)
  uint64_t k[kSortItems];
#if !BH_SORT_VIDX
  uint32_t v[kSortItems];
#endif
  const bool full_tile = tbase + kTile <= n;  // (block-uniform) every tile but the last: no bounds tests
  if (BH_SORT_FULL_LOAD && full_tile) {
#pragma unroll
    for (int j = 0; j < kSortItems; ++j) {
      const int64_t i = wbase + 32 * j + lane;
      k[j] = __ldcs(kin + i);
#if !BH_SORT_VIDX
      v[j] = vin ? __ldcs(vin + i) : (uint32_t)i;
#endif
    }
  } else
#pragma unroll
  for (int j = 0; j < kSortItems; ++j) {
    const int64_t i = wbase + 32 * j + lane;
    if (i < n) {
      k[j] = __ldcs(kin + i);
#if !BH_SORT_VIDX
      v[j] = vin ? __ldcs(vin + i) : (uint32_t)i;  // no input values: the identity permutation
#endif
    } else {
      k[j] = ~0ull;  // pads sort after every real key of the last tile and are never stored
#if !BH_SORT_VIDX
      v[j] = 0u;
#endif
    }
  }

  // ---- stable rank inside the warp (items in order, lanes in order): the
  // peer masks first (independent ballots), then the sequential counter walk
  unsigned rank[kSortItems];
  unsigned *wh = S.whist[w];
  const unsigned lt = (1u << lane) - 1u;
#pragma unroll
  for (int j = 0; j < kSortItems; ++j) {
    const unsigned d = (unsigned)(k[j] >> shift) & (kBins - 1);
    unsigned peers = FULL;  // lanes whose digit equals this lane's
    if (MATCH) {
      peers = __match_any_sync(FULL, d);
    } else if (BH_SORT_UNIFORM && __all_sync(FULL, d == __shfl_sync(FULL, d, 0))) {
      peers = FULL;
    } else {
#pragma unroll
      for (int b = 0; b < kDigitBits; ++b) {
#if BH_SORT_RANKASM
        match_bit(peers, d, 1u << b);  // (bh_internal.cuh)
#else
        const unsigned bb = __ballot_sync(FULL, (d >> b) & 1u);
        peers &= ((d >> b) & 1u) ? bb : ~bb;
#endif
      }
    }
    rank[j] = peers;
  }
#pragma unroll
  for (int j = 0; j < kSortItems; ++j) {
    const unsigned d = (unsigned)(k[j] >> shift) & (kBins - 1);
    const unsigned peers = rank[j];
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
#if BH_SORT_VIDX
    S.vidx[lp] = (uint16_t)(w * 32 * kSortItems + 32 * j + lane);
#else
    S.vals[lp] = v[j];
#endif
  }

  // ---- decoupled look-back for digit d: four predecessors per round trip
  unsigned excl = 0;
  if (tile > 0) {
    int64_t j = (int64_t)tile - 1;
    for (;;) {
      unsigned long long sv[4];
#pragma unroll
      for (int q = 0; q < 4; ++q)
        sv[q] = j - q >= 0 ? ld_status(st + (size_t)(j - q) * kBins + d) : pack(kFlagInc, epoch, 0u);
      int used = 0;
      bool done = false;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const unsigned long long x = sv[q];
        if (used != q || (unsigned)((x >> 32) & kEpochMask) != epoch || (x >> 62) == 0) break;  // not yet published
        excl += (unsigned)(x & kValMask);
        ++used;
        if ((x >> 62) == 2ull) { done = true; break; }
      }
      if (done) break;
      j -= used;
    }
    st_status(my, pack(kFlagInc, epoch, excl + cnt));
  }
  S.gdelta[d] = (long long)S.bin_start[d] + excl - (long long)S.start[d];
  __syncthreads();

  // ---- scatter: consecutive tile slots of one digit go to consecutive addresses
#if !BH_SORT_VIDX
  if (BH_SORT_FULL_SCATTER && full_tile) {
#pragma unroll 4
    for (int i = threadIdx.x; i < kTile; i += kSortThreads) {
      const uint64_t key = S.keys[i];
      const unsigned di = (unsigned)(key >> shift) & (kBins - 1);
      const long long g = S.gdelta[di] + i;
      kout[g] = key;
      vout[g] = S.vals[i];
    }
    return;
  }
#endif
#pragma unroll 4
  for (int i = threadIdx.x; i < kTile; i += kSortThreads) {
    const uint64_t key = S.keys[i];
    const unsigned di = (unsigned)(key >> shift) & (kBins - 1);
    const long long g = S.gdelta[di] + i;
    if (g < n) {
      kout[g] = key;
#if BH_SORT_VIDX
      const int64_t src = tbase + S.vidx[i];
      vout[g] = vin ? vin[src] : (uint32_t)src;
#else
      vout[g] = S.vals[i];
#endif
    }
  }
}

// ------------------------------------------------------------------ scan
// Reduce-then-scan in three bandwidth-bound launches (12 B per element): the
// single-pass look-back version spent most of its time in the serial chain of
// 4096-element tiles (67 us for 1e7 elements at 8 blocks per SM).
//   k_scan_reduce  tile sums          (read 4 B)
//   k_scan_tiles   one block scans the tile sums
//   k_scan_down    tile scan + prefix (read 4 B, write 4 B)
constexpr int kScanThreads = 256;
constexpr int kScanItems = 16;
constexpr int kScanTile = kScanThreads * kScanItems;
constexpr int kScanTopThreads = 1024;

__device__ __forceinline__ void scan_load(const uint32_t *__restrict__ in, int64_t i0, int64_t n,
                                          unsigned (&x)[kScanItems]) {
  if (i0 + kScanItems <= n && ((reinterpret_cast<uintptr_t>(in + i0) & 15) == 0)) {
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
}

// exclusive scan over a block of T threads, one value each; *total = block sum
template <int T>
__device__ __forceinline__ unsigned block_scan_t(unsigned v, unsigned *wsum, unsigned *total) {
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
  for (int i = 0; i < T / 32; ++i) {
    const unsigned s = wsum[i];
    woff += i < (int)w ? s : 0u;
    tot += s;
  }
  *total = tot;
  __syncthreads();
  return woff + incl - v;
}

__global__ void __launch_bounds__(kScanThreads) k_scan_reduce(const uint32_t *__restrict__ in, int64_t n,
                                                              unsigned *__restrict__ tsum) {
  __shared__ unsigned wsum[kScanThreads / 32];
  unsigned x[kScanItems];
  scan_load(in, (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanItems, n, x);
  unsigned s = 0;
#pragma unroll
  for (int j = 0; j < kScanItems; ++j) s += x[j];
  s = __reduce_add_sync(0xffffffffu, s);
  if ((threadIdx.x & 31) == 0) wsum[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned t = 0;
#pragma unroll
    for (int i = 0; i < kScanThreads / 32; ++i) t += wsum[i];
    tsum[blockIdx.x] = t;
  }
}

// exclusive scan of the tile sums in place, one block: each thread sums a
// contiguous run of tiles, one block scan of the run totals, then each thread
// writes its run (one barrier round instead of one per 1024 tiles)
__global__ void __launch_bounds__(kScanTopThreads) k_scan_tiles(unsigned *__restrict__ tsum, int64_t ntiles) {
  __shared__ unsigned wsum[kScanTopThreads / 32];
  const int64_t per = (ntiles + kScanTopThreads - 1) / kScanTopThreads;
  const int64_t b = per * threadIdx.x, e = b + per < ntiles ? b + per : ntiles;
  unsigned run = 0;
  for (int64_t i = b; i < e; ++i) run += tsum[i];
  unsigned tot;
  unsigned ex = block_scan_t<kScanTopThreads>(run, wsum, &tot);
  for (int64_t i = b; i < e; ++i) {
    const unsigned v = tsum[i];
    tsum[i] = ex;
    ex += v;
  }
}

template <bool INCLUSIVE>
__global__ void __launch_bounds__(kScanThreads) k_scan_down(const uint32_t *__restrict__ in, uint32_t *__restrict__ out,
                                                            int64_t n, const unsigned *__restrict__ tprefix) {
  __shared__ unsigned wsum[kScanThreads / 32];
  const int64_t i0 = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanItems;
  unsigned x[kScanItems];
  scan_load(in, i0, n, x);
  unsigned sum = 0;
#pragma unroll
  for (int j = 0; j < kScanItems; ++j) sum += x[j];
  unsigned tot;
  unsigned run = tprefix[blockIdx.x] + block_scan_t<kScanThreads>(sum, wsum, &tot);
  unsigned y[kScanItems];
#pragma unroll
  for (int j = 0; j < kScanItems; ++j) {
    if (INCLUSIVE) run += x[j];
    y[j] = run;
    if (!INCLUSIVE) run += x[j];
  }
  if (i0 + kScanItems <= n && ((reinterpret_cast<uintptr_t>(out + i0) & 15) == 0)) {
    uint4 *dst = reinterpret_cast<uint4 *>(out + i0);
#pragma unroll
    for (int j = 0; j < kScanItems / 4; ++j) dst[j] = make_uint4(y[4 * j], y[4 * j + 1], y[4 * j + 2], y[4 * j + 3]);
  } else {
#pragma unroll
    for (int j = 0; j < kScanItems; ++j)
      if (i0 + j < n) out[i0 + j] = y[j];
  }
}

inline size_t scan_bytes(int64_t n) {
  const int64_t tiles = std::max<int64_t>(1, (n + kScanTile - 1) / kScanTile);
  return sizeof(unsigned) * (size_t)tiles + 256;
}

template <bool INCLUSIVE>
cudaError_t scan_u32(void *temp, size_t temp_bytes, const uint32_t *in, uint32_t *out, int64_t n, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  if (temp_bytes < scan_bytes(n)) return cudaErrorInvalidValue;
  const int64_t tiles = (n + kScanTile - 1) / kScanTile;
  if (tiles > 0x7fffffff) return cudaErrorInvalidValue;
  unsigned *tsum = static_cast<unsigned *>(temp);
  k_scan_reduce<<<(unsigned)tiles, kScanThreads, 0, s>>>(in, n, tsum);
  k_scan_tiles<<<1, kScanTopThreads, 0, s>>>(tsum, tiles);
  k_scan_down<INCLUSIVE><<<(unsigned)tiles, kScanThreads, 0, s>>>(in, out, n, tsum);
  return cudaGetLastError();
}

}  // namespace

size_t sort_temp_bytes(int64_t n) {
  const int64_t tiles = std::max<int64_t>(1, sort_tiles(n));
  return al(sizeof(uint64_t) * n) + al(sizeof(uint32_t) * n) + 2 * al(sizeof(unsigned) * kPasses * kBins) +
         al(sizeof(unsigned) * (kPasses + 1)) + sizeof(unsigned long long) * kBins * (size_t)tiles;
}

cudaError_t sort_pairs(void *temp, size_t temp_bytes, const uint64_t *kin, uint64_t *kout, const uint32_t *vin,
                       uint32_t *vout, int64_t n, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  if (temp_bytes < sort_temp_bytes(n) || n > 0x7fffffffll) return cudaErrorInvalidValue;
  SortTemp t = carve_sort(temp, n);
  const unsigned tiles = (unsigned)sort_tiles(n);
  // variants for measurement: BH_SORT_MINB=2 (no register cap), BH_SORT_MATCH=1
  // (peer masks from MATCH.ANY instead of 8 ballots)
  static int variant = -1;
  if (variant < 0) {
    const char *e = getenv("BH_SORT_MINB");
    const char *m = getenv("BH_SORT_MATCH");
    variant = ((e && atoi(e) == 2) ? 1 : 0) | ((m && atoi(m) == 1) ? 2 : 0);
    const int sm = (int)sizeof(PassSmem);
    cudaFuncSetAttribute(k_sort_pass<BH_SORT_BLOCKS, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    cudaFuncSetAttribute(k_sort_pass<2, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    cudaFuncSetAttribute(k_sort_pass<BH_SORT_BLOCKS, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    cudaFuncSetAttribute(k_sort_pass<2, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
  }
  auto pass = variant == 0 ? k_sort_pass<BH_SORT_BLOCKS, false> : variant == 1 ? k_sort_pass<2, false>
            : variant == 2 ? k_sort_pass<BH_SORT_BLOCKS, true> : k_sort_pass<2, true>;
  k_sort_zero<<<1, 256, 0, s>>>(t.hist, t.counters);
  {
    static int sms = 0;
    if (!sms) {
      int dev = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    }
    const int64_t need = (n + kHistThreads * kHistUnroll - 1) / (kHistThreads * kHistUnroll);
    const int g = (int)std::max<int64_t>(1, std::min<int64_t>(need, 3 * sms));
    const int hsm = (int)(sizeof(unsigned) * kPasses * kBins * kHistParts);
    static bool hinit = false;
    if (!hinit) {
      cudaFuncSetAttribute(k_sort_hist, cudaFuncAttributeMaxDynamicSharedMemorySize, hsm);
      hinit = true;
    }
    k_sort_hist<<<g, kHistThreads, hsm, s>>>(kin, n, t.hist, t.bin_start, t.counters + kPasses);
  }
  // 8 passes ping-pong between the temp pair and the output (even count: ends in kout)
  const uint64_t *ka = kin;
  const uint32_t *va = vin;
  for (int p = 0; p < kPasses; ++p) {
    uint64_t *kb = (p & 1) ? kout : t.k;
    uint32_t *vb = (p & 1) ? vout : t.v;
    // the top digit (octree levels 1-3) takes few values per tile: there MATCH.ANY
    // ranks faster than the 8 ballots (measured at cfg3: 65 vs 84 us)
    auto kern = (p >= kPasses - BH_SORT_MATCH_TOP && variant == 0) ? k_sort_pass<BH_SORT_BLOCKS, true> : pass;
    kern<<<tiles, kSortThreads, sizeof(PassSmem), s>>>(ka, va, kb, vb, n, kDigitBits * p, t.bin_start + p * kBins,
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
