// K4: hand-written onesweep LSD radix sort (Adinets & Merrill 2022 scheme)
//     over 64-bit entry words ((tile | truncated depth key) << id_bits | id):
//     the passes cover the key bits only and the Gaussian id rides in the
//     low bits; replaces np.lexsort((rank, key, tile_id)) (rasterizer.py:353-357).
//     8-bit digits, ceil((32 + tile_bits) / 8) passes, one global-histogram
//     pass up front, per-partition decoupled look-back with epoch-tagged
//     status words (no per-frame clearing).  Stable: partitions are ranked in
//     input order with warp-striped items and match.any peer ranking.
// K5: tile ranges (rasterizer.py:358-372) and the float64 tie fix-up: runs of
//     equal (truncated) keys inside a tile are re-ordered by the float64 depth
//     and then rank, so the final order equals the reference's float64
//     lexsort (one kernel: a run's first entry sorts the run).
#include "stp_common.cuh"

namespace stp {

constexpr int kSortThreads = 256;
constexpr int kSortWarps = kSortThreads / 32;
constexpr int kSortItems = STP_SORT_ITEMS;
constexpr int kSortTile = kSortPartition;  // kSortThreads * kSortItems items per partition
constexpr int kRadix = 256;
#ifndef STP_SORT_WARPSCAN
#define STP_SORT_WARPSCAN 1  // digit scans by warp shuffles, global prefix once per block
#endif
#ifndef STP_HIST_BALLOT
#define STP_HIST_BALLOT 0  // digit histogram with warp-aggregated (ballot) updates
#endif
#ifndef STP_SORT_SPIN_NS
#define STP_SORT_SPIN_NS 0  // back-off of the look-back spin (0: none)
#endif
#ifndef STP_SORT_LATE_LB
#define STP_SORT_LATE_LB 1  // publish the aggregate, scatter locally, then look back
#endif
#ifndef STP_SORT_LB_VEC
#define STP_SORT_LB_VEC 4  // predecessors read per look-back step
#endif
#ifndef STP_TIE_PACK
#define STP_TIE_PACK 1  // K5: a step's short tie runs packed into one round
#endif
#ifndef STP_SORT_MINB
#define STP_SORT_MINB 2  // k_onesweep min blocks per SM (1: 147 registers, K4 0.44 ms; 3: 80 registers with spills, K4 0.32 ms but the step 4.32 vs 4.22 ms, profiles/r3j)
#endif
#ifndef STP_SORT_BALLOT
#define STP_SORT_BALLOT 1  // warp ranking by ballots instead of match.any (K4 0.410 -> 0.382 ms)
#endif

// look-back word: [epoch:32 | flag:2 | count:30]
constexpr unsigned long long kFlagAgg = 1ull << 30;
constexpr unsigned long long kFlagPre = 2ull << 30;
constexpr unsigned long long kCountMask = (1ull << 30) - 1;

__device__ __forceinline__ int64_t n_entries(const unsigned long long* counters, int64_t ecap) {
  const int64_t e = (int64_t)counters[C_ENTRIES];
  return e < ecap ? e : ecap;
}

__global__ void __launch_bounds__(kSortThreads) k_sort_hist(const uint64_t* __restrict__ keys,
                                                            const unsigned long long* counters,
                                                            int64_t ecap, int passes, int shift0,
                                                            uint32_t* __restrict__ hist) {
  __shared__ uint32_t s_hist[8][kRadix];
  for (int i = threadIdx.x; i < 8 * kRadix; i += kSortThreads) (&s_hist[0][0])[i] = 0;
  __syncthreads();
  const int64_t E = n_entries(counters, ecap);
#if STP_HIST_BALLOT
  // warp-aggregated: the lanes holding the same digit (8 ballots) add once
  const int lane = threadIdx.x & 31;
  const int64_t stride = (int64_t)gridDim.x * kSortThreads;
  for (int64_t i0 = (int64_t)blockIdx.x * kSortThreads + (threadIdx.x & ~31); i0 < E;
       i0 += stride) {
    const int64_t i = i0 + lane;
    const bool in = i < E;
    const uint64_t k = in ? keys[i] : 0ull;
    for (int p = 0; p < passes; ++p) {
      const uint32_t d = (uint32_t)(k >> (shift0 + 8 * p)) & 0xffu;
      unsigned peers = __ballot_sync(kFull, in);
#pragma unroll
      for (int bit = 0; bit < 8; ++bit) {
        const unsigned bb = __ballot_sync(kFull, (d >> bit) & 1u);
        peers &= ((d >> bit) & 1u) ? bb : ~bb;
      }
      if (in && lane == __ffs(peers) - 1) atomicAdd(&s_hist[p][d], (unsigned)__popc(peers));
    }
  }
#else
  // four independent key loads in flight per thread
#ifndef STP_HIST_UNROLL
#define STP_HIST_UNROLL 4
#endif
  constexpr int U = STP_HIST_UNROLL;
  for (int64_t i0 = (int64_t)blockIdx.x * kSortThreads * U + threadIdx.x; i0 < E;
       i0 += (int64_t)gridDim.x * kSortThreads * U) {
    uint64_t k[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = i0 + (int64_t)u * kSortThreads;
      k[u] = i < E ? keys[i] : 0ull;
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (i0 + (int64_t)u * kSortThreads < E)
        for (int p = 0; p < passes; ++p)
          atomicAdd(&s_hist[p][(k[u] >> (shift0 + 8 * p)) & 0xff], 1u);
  }
#endif
  __syncthreads();
  for (int i = threadIdx.x; i < passes * kRadix; i += kSortThreads) {
    const uint32_t v = (&s_hist[0][0])[i];
    if (v) atomicAdd(hist + i, v);
  }
}

struct SortSmem {
  uint32_t warp_hist[kSortWarps][kRadix];  // per-warp digit counts -> warp offsets
  uint32_t local_off[kRadix];              // block-local exclusive digit offsets
  uint32_t global_off[kRadix];             // this partition's first output slot per digit
  uint32_t scan_tmp[kRadix];
  uint32_t gex[kRadix];                    // exclusive prefix of the pass's global histogram
  uint32_t wtot[kSortWarps];               // per-warp totals of a 256-digit block scan
  uint32_t part;
  uint64_t keys[kSortTile];
};

// exclusive prefix over the 256 digits (thread = digit): warp shuffles + the
// 8 warp totals (two barriers instead of a 16-barrier Hillis-Steele scan)
__device__ __forceinline__ uint32_t block_excl_scan256(uint32_t v, uint32_t* wtot, int lane,
                                                       int w) {
  uint32_t inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(kFull, inc, o);
    if (lane >= o) inc += y;
  }
  if (lane == 31) wtot[w] = inc;
  __syncthreads();
  uint32_t off = 0;
#pragma unroll
  for (int ww = 0; ww < kSortWarps; ++ww) off += (ww < w) ? wtot[ww] : 0u;
  __syncthreads();  // wtot is reused by the next scan
  return off + inc - v;
}

// Decoupled look-back for digit d of partition part (> 0): sums the
// predecessors' aggregates back to the first inclusive prefix.  LB_VEC
// predecessors are read per step with independent loads (one round trip
// instead of LB_VEC); an unpublished one is re-read until it is published.
__device__ __forceinline__ unsigned long long look_back(const unsigned long long* lookback,
                                                        int64_t part, int d, uint32_t epoch) {
  unsigned long long excl = 0;
  int64_t p = part - 1;
  for (;;) {
    unsigned long long v[STP_SORT_LB_VEC];
#pragma unroll
    for (int k = 0; k < STP_SORT_LB_VEC; ++k) {
      const int64_t q = p - k >= 0 ? p - k : 0;
      v[k] = *reinterpret_cast<volatile const unsigned long long*>(lookback + (size_t)q * kRadix + d);
    }
    bool done = false;
    int used = 0;
#pragma unroll
    for (int k = 0; k < STP_SORT_LB_VEC; ++k) {
      if (done || used < k) continue;  // stopped at an earlier word
      if ((v[k] >> 32) != epoch || ((v[k] >> 30) & 3ull) == 0) continue;  // not yet published
      excl += v[k] & kCountMask;
      ++used;
      if (((v[k] >> 30) & 3ull) == 2) done = true;  // inclusive prefix (partition 0 always is)
    }
    if (done) return excl;
    p -= used;
#if STP_SORT_SPIN_NS > 0
    if (!used) __nanosleep(STP_SORT_SPIN_NS);
#endif
  }
}

__global__ void __launch_bounds__(kSortThreads, STP_SORT_MINB) k_onesweep(
    const uint64_t* __restrict__ kin, uint64_t* __restrict__ kout,
    const unsigned long long* counters, int64_t ecap, int shift,
    const uint32_t* __restrict__ hist, unsigned long long* lookback,
    unsigned long long* part_counter) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  SortSmem& sm = *reinterpret_cast<SortSmem*>(smem_raw);
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int64_t E = n_entries(counters, ecap);
  const uint32_t epoch = (uint32_t)counters[C_EPOCH];
#if STP_SORT_WARPSCAN
  // the pass's global digit offsets: the same for every partition, so once
  // per persistent block
  sm.gex[tid] = block_excl_scan256(hist[tid], sm.wtot, lane, w);
#endif
  // persistent: partitions are claimed in increasing order (so the look-back
  // predecessor is always held by a running block) until the entries run out
  for (;;) {
  if (tid == 0) sm.part = (uint32_t)atomicAdd(part_counter, 1ull);
  for (int i = tid; i < kSortWarps * kRadix; i += kSortThreads) (&sm.warp_hist[0][0])[i] = 0;
  __syncthreads();
  const uint32_t part = sm.part;
  const int64_t base = (int64_t)part * kSortTile;
  if (base >= E) return;
  const int n_valid = (int)min((int64_t)kSortTile, E - base);

  // warp-striped load: warp w owns [base + w*512, +512), item k of lane l at k*32 + l
  uint64_t key[kSortItems];
  uint32_t dig[kSortItems];
  uint32_t rank[kSortItems];
#pragma unroll
  for (int k = 0; k < kSortItems; ++k) {
    const int li = w * (kSortItems * 32) + k * 32 + lane;
    if (li < n_valid) {
      key[k] = kin[base + li];
      dig[k] = (uint32_t)(key[k] >> shift) & 0xff;
    } else {
      key[k] = ~0ull;
      dig[k] = 0xff;
    }
  }
  // stable warp-level ranking
  const unsigned lt_mask = (1u << lane) - 1;
#pragma unroll
  for (int k = 0; k < kSortItems; ++k) {
#if STP_SORT_BALLOT
    // peers with the same 8-bit digit from 8 ballots (VOTE is an ALU op;
    // MATCH.ANY waits on the short scoreboard)
    unsigned peers = kFull;
#pragma unroll
    for (int bit = 0; bit < 8; ++bit) {
      const unsigned bb = __ballot_sync(kFull, (dig[k] >> bit) & 1u);
      peers &= ((dig[k] >> bit) & 1u) ? bb : ~bb;
    }
#else
    const unsigned peers = __match_any_sync(kFull, dig[k]);
#endif
    const int leader = 31 - __clz(peers);
    const uint32_t before = sm.warp_hist[w][dig[k]];
    __syncwarp();
    rank[k] = before + __popc(peers & lt_mask);
    if (lane == leader) sm.warp_hist[w][dig[k]] = before + __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  // per digit: exclusive scan across warps, block total
  uint32_t block_cnt;
#if STP_SORT_LATE_LB && STP_SORT_WARPSCAN
  // publish the aggregate, build the block-local order in shared memory, and
  // only then look back: the predecessors publish while this block scatters
  {
    const int d = tid;
    uint32_t sum = 0;
#pragma unroll
    for (int ww = 0; ww < kSortWarps; ++ww) {
      const uint32_t c = sm.warp_hist[ww][d];
      sm.warp_hist[ww][d] = sum;
      sum += c;
    }
    block_cnt = sum;
    const unsigned long long tag = (unsigned long long)epoch << 32;
    atomicExch(lookback + (size_t)part * kRadix + d,
               tag | (part == 0 ? kFlagPre : kFlagAgg) | (unsigned long long)block_cnt);
  }
  sm.local_off[tid] = block_excl_scan256(block_cnt, sm.wtot, lane, w);
  __syncthreads();
#pragma unroll
  for (int k = 0; k < kSortItems; ++k) {
    const uint32_t pos = sm.local_off[dig[k]] + sm.warp_hist[w][dig[k]] + rank[k];
    if (pos < (uint32_t)kSortTile) sm.keys[pos] = key[k];
  }
  {
    const int d = tid;
    unsigned long long excl = 0;
    if (part > 0) {
      excl = look_back(lookback, part, d, epoch);
      atomicExch(lookback + (size_t)part * kRadix + d,
                 ((unsigned long long)epoch << 32) | kFlagPre | ((excl + block_cnt) & kCountMask));
    }
    sm.global_off[d] = (uint32_t)excl + sm.gex[d];
  }
  __syncthreads();
#else
  {
    const int d = tid;  // kSortThreads == kRadix
    uint32_t sum = 0;
#pragma unroll
    for (int ww = 0; ww < kSortWarps; ++ww) {
      const uint32_t c = sm.warp_hist[ww][d];
      sm.warp_hist[ww][d] = sum;
      sum += c;
    }
    block_cnt = sum;
    // publish aggregate / inclusive prefix, then look back
    unsigned long long* my = lookback + (size_t)part * kRadix + d;
    const unsigned long long tag = (unsigned long long)epoch << 32;
    unsigned long long excl = 0;
    if (part == 0) {
      atomicExch(my, tag | kFlagPre | (unsigned long long)block_cnt);
    } else {
      atomicExch(my, tag | kFlagAgg | (unsigned long long)block_cnt);
      int64_t p = (int64_t)part - 1;
      while (true) {
        const unsigned long long v =
            *reinterpret_cast<volatile unsigned long long*>(lookback + (size_t)p * kRadix + d);
        if ((v >> 32) != epoch || ((v >> 30) & 3ull) == 0) {  // not yet published
#if STP_SORT_SPIN_NS > 0
          __nanosleep(STP_SORT_SPIN_NS);
#endif
          continue;
        }
        excl += v & kCountMask;
        if (((v >> 30) & 3ull) == 2) break;
        --p;
      }
      atomicExch(my, tag | kFlagPre | ((excl + block_cnt) & kCountMask));
    }
#if STP_SORT_WARPSCAN
    sm.global_off[d] = (uint32_t)excl + sm.gex[d];
  }
  // block-local exclusive digit offsets
  sm.local_off[tid] = block_excl_scan256(block_cnt, sm.wtot, lane, w);
  __syncthreads();
#else
    sm.global_off[d] = (uint32_t)excl;
    sm.scan_tmp[d] = hist[d];
  }
  __syncthreads();
  // exclusive scans over the 256 digits: global histogram and block counts
  {
    const int d = tid;
    uint32_t g = sm.scan_tmp[d], b = block_cnt;
    // Hillis-Steele in shared memory (256 entries)
    __shared__ uint32_t s_a[kRadix], s_b[kRadix];
    s_a[d] = g;
    s_b[d] = b;
    __syncthreads();
    for (int o = 1; o < kRadix; o <<= 1) {
      const uint32_t ya = (d >= o) ? s_a[d - o] : 0, yb = (d >= o) ? s_b[d - o] : 0;
      __syncthreads();
      s_a[d] += ya;
      s_b[d] += yb;
      __syncthreads();
    }
    sm.global_off[d] += s_a[d] - g;
    sm.local_off[d] = s_b[d] - b;
  }
  __syncthreads();
#endif
  // scatter into shared memory in block-local sorted order
#pragma unroll
  for (int k = 0; k < kSortItems; ++k) {
    const uint32_t pos = sm.local_off[dig[k]] + sm.warp_hist[w][dig[k]] + rank[k];
    if (pos < (uint32_t)kSortTile) sm.keys[pos] = key[k];
  }
  __syncthreads();
#endif
  for (int i = tid; i < n_valid; i += kSortThreads) {
    const uint64_t k = sm.keys[i];
    const uint32_t d = (uint32_t)(k >> shift) & 0xff;
    const uint32_t o = sm.global_off[d] + (uint32_t)i - sm.local_off[d];
    kout[o] = k;
  }
  __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// K5 tile ranges + float64 tie fix-up.

__device__ __forceinline__ double entry_depth64(const SplatRec* __restrict__ recs, const DevCam& cam,
                                                uint32_t id, int tile, int gw,
                                                const double2* __restrict__ aux) {
  if (aux) return aux[id].x;  // GlobalZ: view z
  const SplatRec& r = recs[id];
  const int tx = tile % gw, ty = tile / gw;
  double ptx, pty;
  max_point(r.mx, r.my, r.ca, r.cb, r.cc, r.inv_a, r.inv_c, (double)(tx * kTile),
            (double)(ty * kTile), 16.0, 0.0625, ptx, pty);
  return key_rec_at(cam, r, ptx, pty);
}

constexpr int kTieLocal = 32;

// sum over a 256-thread block (all threads call it)
__device__ __forceinline__ int block_sum(int v) {
  __shared__ int s_part[8];
  v += __shfl_xor_sync(kFull, v, 16);
  v += __shfl_xor_sync(kFull, v, 8);
  v += __shfl_xor_sync(kFull, v, 4);
  v += __shfl_xor_sync(kFull, v, 2);
  v += __shfl_xor_sync(kFull, v, 1);
  if ((threadIdx.x & 31) == 0) s_part[threadIdx.x >> 5] = v;
  __syncthreads();
  int t = 0;
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += s_part[w];
  __syncthreads();
  return t;
}

// Grid-stride over the sorted entries; per-block counts are reduced in
// registers / shared memory and added with one atomic per block (a per-entry
// or per-warp atomic on one counter serialises tens of thousands of updates).
// Each entry writes its Gaussian id and the tile bounds it starts / ends.  A
// run of equal sort keys (same tile, same truncated depth) is re-ordered by
// (float64 depth, rank) -- np.lexsort's order -- by the thread of its first
// member: it computes the members' depths, insertion-sorts them (runs are
// short; the stable LSD sort delivered them in rank order) and writes their
// ids; the other members write nothing.  Runs over kTieLocal go through the
// free ping-pong buffer d64.
__global__ void __launch_bounds__(256) k_ranges(const uint64_t* __restrict__ keys,
                                                uint32_t* __restrict__ vals,
                                                unsigned long long* counters, int64_t ecap,
                                                uint2* __restrict__ ranges,
                                                const SplatRec* __restrict__ recs, DevCam cam,
                                                int gw, int depth_bits, int id_bits,
                                                const double2* __restrict__ aux,
                                                double* __restrict__ d64,
                                                int64_t* __restrict__ status) {
  const int64_t E = n_entries(counters, ecap);
  if (status && blockIdx.x == 0 && threadIdx.x == 0) {
    // the frame status word of the asynchronous paths (stp.h StpOutputs.status)
    const int64_t total = (int64_t)counters[C_ENTRIES];
    status[0] = total > ecap ? STP_ERR_WORKSPACE_TOO_SMALL : STP_OK;
    status[1] = total;
  }
  const uint64_t id_mask = (1ull << id_bits) - 1ull;
  int heads = 0, runs = 0;
  const int lane = threadIdx.x & 31;
  // warp-uniform loop: each warp takes 32 consecutive entries per step, so
  // the runs found in a step are re-ordered by the whole warp (one lane per
  // member) instead of serially by their first member's thread
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31); i0 < E;
       i0 += stride) {
    const int64_t i = i0 + lane;
    bool short_head = false;
    int L = 1;
    uint32_t tile = 0;
    if (i < E) {
      const uint64_t w = keys[i];
      const uint64_t k = w >> id_bits;                      // tile | truncated depth
      tile = (uint32_t)(k >> depth_bits);
      const uint64_t kp = (i > 0) ? keys[i - 1] >> id_bits : ~k;
      const uint64_t kn = (i + 1 < E) ? keys[i + 1] >> id_bits : ~k;
      const uint32_t id = (uint32_t)(w & id_mask);
      if (i == 0 || (uint32_t)(kp >> depth_bits) != tile) {
        ranges[tile].x = (uint32_t)i;
        ++heads;
      }
      if (i + 1 == E || (uint32_t)(kn >> depth_bits) != tile) ranges[tile].y = (uint32_t)(i + 1);
      const bool first = i == 0 || kp != k;
      if (kn != k) {
        if (first) vals[i] = id;  // not in a run
      } else if (first) {
        ++runs;
        L = 2;
        while (i + L < E && (keys[i + L] >> id_bits) == k) ++L;
        if (L <= kTieLocal) {
          short_head = true;
        } else {
          // long runs (coincident splats): insertion sort through memory
          for (int64_t m = 0; m < L; ++m) {
            const uint32_t iv = (uint32_t)(keys[i + m] & id_mask);
            const double dv = entry_depth64(recs, cam, iv, (int)tile, gw, aux);
            int64_t p = m - 1;
            while (p >= 0) {
              const double dp = d64[i + p];
              if (!(dp > dv)) break;
              vals[i + p + 1] = vals[i + p];
              d64[i + p + 1] = dp;
              --p;
            }
            vals[i + p + 1] = iv;
            d64[i + p + 1] = dv;
          }
        }
      }
    }
    // the step's short runs, one at a time, all lanes: lane m < L computes
    // member m's float64 depth, its rank by (depth, Gaussian id) -- the
    // stable LSD sort delivered members in rank order, ids are ranks -- and
    // writes its id to the run's slot of that rank
    unsigned hb = __ballot_sync(kFull, short_head);
#if STP_TIE_PACK
    // the step's short runs packed whole into rounds of <= 32 lanes: every
    // lane of a round computes one member's float64 depth (the record
    // fetches of all packed runs overlap) and ranks it inside its run
    while (hb) {
      int64_t my_hi = 0;
      int my_m = -1, my_L = 0, my_off = 0, my_t = 0, fill = 0;
      while (hb) {
        const int src = __ffs(hb) - 1;
        const int hl = __shfl_sync(kFull, L, src);
        if (fill + hl > 32) break;  // the next run starts the next round
        hb &= hb - 1;
        const int64_t hi = __shfl_sync(kFull, i, src);
        const int ht = (int)__shfl_sync(kFull, tile, src);
        if (lane >= fill && lane < fill + hl) {
          my_hi = hi;
          my_m = lane - fill;
          my_L = hl;
          my_off = fill;
          my_t = ht;
        }
        fill += hl;
      }
      double d = INFINITY;
      uint32_t im = 0xffffffffu;
      if (my_m >= 0) {
        im = (uint32_t)(keys[my_hi + my_m] & id_mask);
        d = entry_depth64(recs, cam, im, my_t, gw, aux);
      }
      int rank = 0;
      for (int m = 0; m < 32; ++m) {
        const bool in_run = m < my_L;
        const double od = __shfl_sync(kFull, d, (my_off + (in_run ? m : 0)) & 31);
        const uint32_t oi = __shfl_sync(kFull, im, (my_off + (in_run ? m : 0)) & 31);
        rank += in_run & ((od < d) | ((od == d) & (oi < im)));
        if (!__any_sync(kFull, m + 1 < my_L)) break;
      }
      if (my_m >= 0) vals[my_hi + rank] = im;
    }
#else
    while (hb) {
      const int src = __ffs(hb) - 1;
      hb &= hb - 1;
      const int64_t hi = __shfl_sync(kFull, i, src);
      const int hl = __shfl_sync(kFull, L, src);
      const int ht = (int)__shfl_sync(kFull, tile, src);
      double d = INFINITY;
      uint32_t im = 0xffffffffu;
      if (lane < hl) {
        im = (uint32_t)(keys[hi + lane] & id_mask);
        d = entry_depth64(recs, cam, im, ht, gw, aux);
      }
      int rank = 0;
      for (int m = 0; m < hl; ++m) {
        const double od = __shfl_sync(kFull, d, m);
        const uint32_t oi = __shfl_sync(kFull, im, m);
        rank += (od < d) | ((od == d) & (oi < im));
      }
      if (lane < hl) vals[hi + rank] = im;
    }
#endif
  }
  const int nh = __syncthreads_count(heads > 0) ? block_sum(heads) : 0;
  if (threadIdx.x == 0 && nh) atomicAdd(counters + C_TILES, (unsigned long long)nh);
  const int nr = __syncthreads_count(runs > 0) ? block_sum(runs) : 0;
  if (threadIdx.x == 0 && nr) atomicAdd(counters + C_TIES, (unsigned long long)nr);
}

// ---------------------------------------------------------------------------

int launch_sort(const Frame& f, cudaStream_t s) {
  static bool attr_set = false;
  static int sweep_grid = 0;
  if (!attr_set) {
    cudaFuncSetAttribute(k_onesweep, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)sizeof(SortSmem));
    int per_sm = 0, dev = 0, n_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_onesweep, kSortThreads,
                                                  sizeof(SortSmem));
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
    sweep_grid = max(1, per_sm) * n_sm;
    attr_set = true;
  }
  // one resident wave of persistent blocks (the entry count is only known
  // on the device; a grid sized by the capacity would launch mostly idle blocks)
  const int sweep_blocks = min(f.partitions, sweep_grid);
  const int hist_blocks = device_sm_count() * 4;
  k_sort_hist<<<hist_blocks, kSortThreads, 0, s>>>(f.keys[0], f.counters, f.ecap, f.passes,
                                                    f.id_bits, f.hist);
  int cur = 0;
  for (int p = 0; p < f.passes; ++p) {
    k_onesweep<<<sweep_blocks, kSortThreads, sizeof(SortSmem), s>>>(
        f.keys[cur], f.keys[cur ^ 1], f.counters, f.ecap, f.id_bits + 8 * p,
        f.hist + p * kRadix, f.lookback + (size_t)p * f.partitions * kRadix,
        f.counters + C_PART + p);
    cur ^= 1;
  }
  return cur;
}

void launch_ranges(const Frame& f, int buf, cudaStream_t s) {
  if (f.ecap == 0 && !f.status) return;
  const int64_t blocks =
      max((int64_t)1, min((int64_t)device_sm_count() * 8, (f.ecap + 255) / 256));
  // the other ping-pong key buffer (E x 8 B) is free: float64 depths of tie runs
  double* d64 = reinterpret_cast<double*>(f.keys[buf ^ 1]);
  k_ranges<<<(unsigned)blocks, 256, 0, s>>>(f.keys[buf], f.vals, f.counters, f.ecap, f.ranges,
                                            f.recs, f.cam, f.gw, f.depth_bits, f.id_bits,
                                            f.globalz ? f.aux : nullptr, d64, f.status);
}

}  // namespace stp
