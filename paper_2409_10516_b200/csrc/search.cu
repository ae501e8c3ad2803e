// K6 graph_search: exact B200 restatement of OODGraph::search
// (/root/reference/proj/src/index_oodgraph.cpp:357-411).
//
// One warp per (head, query). The reference's unbounded frontier heap plus
// TopKCollector(ef) pool are replaced by ONE list L kept sorted best-first
// by (score desc, id asc) with per-entry {expanded, masked} flags:
//   * frontier top   = first unexpanded entry of L (cursor);
//   * pool           = first ef unmasked entries of L, worst = the ef-th;
//   * stop rule      = pool full && top.score < worst.score   (:390);
//   * dead entries   (score < worst once the pool is full) can never be popped
//     nor enter the pool, so they are dropped: L stays ~ef + #masked-live long.
// The result depends only on the SET of expanded nodes, which this loop
// reproduces exactly, so ids, f32 scores, scanned and truncated are
// bit-identical to the reference. Scores are exact: one lane per neighbour
// runs the reference's in-order f64 accumulation (products of f32 are exact
// in f64, so fma == mul+add; dot_f64, :40-44).
//
// Storage: L and the visited bitset live in shared memory; a query whose L
// outgrows it migrates L to an HBM spill slot sized for every key, and the
// bitset sits in HBM when n is too large for shared memory. No capacity
// limit is ever exposed to the caller.
#include <cfloat>
#include <cstdlib>
#include <string>

#include "common.cuh"
#include "tma.cuh"

namespace ra {
namespace {

constexpr uint8_t kExpanded = 1, kMasked = 2;

__device__ __forceinline__ bool better(double sa, uint32_t ia, double sb, uint32_t ib) {
  return sa > sb || (sa == sb && ia < ib);
}

// exact in-order f64 dot of q (pre-widened in smem) and an f32 key row
template <int D>
__device__ __forceinline__ double exact_dot(const double* __restrict__ qd,
                                            const float* __restrict__ krow, uint32_t d) {
  double acc = 0.0;
  if constexpr (D > 0) {
    const float4* k4 = reinterpret_cast<const float4*>(krow);
    float4 buf[D / 4];
#pragma unroll
    for (int c = 0; c < D / 4; ++c) buf[c] = __ldg(k4 + c);
#pragma unroll
    for (int c = 0; c < D / 4; ++c) {
      acc = fma(qd[4 * c + 0], (double)buf[c].x, acc);
      acc = fma(qd[4 * c + 1], (double)buf[c].y, acc);
      acc = fma(qd[4 * c + 2], (double)buf[c].z, acc);
      acc = fma(qd[4 * c + 3], (double)buf[c].w, acc);
    }
  } else {
    for (uint32_t i = 0; i < d; ++i) acc = fma(qd[i], (double)__ldg(krow + i), acc);
  }
  return acc;
}

// 32-lane bitonic sort, best-first under (score desc, id asc); carries a flag
__device__ __forceinline__ void warp_sort32(double& s, uint32_t& id, uint32_t& fl, int lane) {
#pragma unroll
  for (int k = 2; k <= 32; k <<= 1) {
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
      const double so = __shfl_xor_sync(kFull, s, j);
      const uint32_t io = __shfl_xor_sync(kFull, id, j);
      const uint32_t fo = __shfl_xor_sync(kFull, fl, j);
      const bool lower = (lane & j) == 0;
      const bool desc = (lane & k) == 0;  // this segment sorts best-first
      const bool other_better = better(so, io, s, id);
      const bool mine_better = better(s, id, so, io);
      const bool take = (lower == desc) ? other_better : mine_better;
      if (take) {
        s = so;
        id = io;
        fl = fo;
      }
    }
  }
}

struct ListRef {
  double* s;
  uint32_t* id;
  uint8_t* fl;
};

// in-order f64 dot of q (f64, smem) and a key row staged in shared memory
template <int D>
__device__ __forceinline__ double smem_dot(const double* __restrict__ qd,
                                           const float* __restrict__ row) {
  double acc = 0.0;
  const float4* r4 = reinterpret_cast<const float4*>(row);
#pragma unroll 8
  for (int c = 0; c < D / 4; ++c) {
    const float4 k = r4[c];
    acc = fma(qd[4 * c + 0], (double)k.x, acc);
    acc = fma(qd[4 * c + 1], (double)k.y, acc);
    acc = fma(qd[4 * c + 2], (double)k.z, acc);
    acc = fma(qd[4 * c + 3], (double)k.w, acc);
  }
  return acc;
}

// Per-warp shared-memory layout (16-B aligned pieces):
//   mbarrier | q as f64 [d_pad] | key-row tile [32][d+4] f32 (TMA target,
//   D > 0 only) | list L: s f64[cap], id u32[cap], flags u8[cap] | visited bitset
template <int D>
struct WarpLayout {
  uint32_t d_pad, cap, vis_words, vis_smem, row_stride;
  __host__ __device__ size_t rows_bytes() const {
    return D > 0 ? size_t(32) * row_stride * 4 : 0;
  }
  __host__ __device__ size_t list_off() const { return 16 + size_t(d_pad) * 8 + rows_bytes(); }
  __host__ __device__ size_t vis_off() const {
    return list_off() + ((size_t(cap) * 13 + 15) & ~size_t(15));
  }
  __host__ __device__ size_t bytes() const {
    return vis_off() + (vis_smem ? ((size_t(vis_words) * 4 + 15) & ~size_t(15)) : 0);
  }
};

template <int D>
__global__ void __launch_bounds__(128, 1) k_graph_search(SearchArgs a, uint32_t wpb,
                                                      WarpLayout<D> lay, uint32_t spill_cap) {
  extern __shared__ __align__(16) uint8_t smem[];
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t b = blockIdx.x * wpb + warp;
  if (b >= a.B) return;  // warp-uniform

  const GraphDesc g = a.desc[b];
  const uint32_t d = a.d, M = g.M, ef = g.ef, k = a.k;
  const float* __restrict__ keys = g.keys;
  const uint32_t* __restrict__ adj = g.adj;
  const uint32_t cap = lay.cap, vis_words = lay.vis_words;

  uint8_t* base = smem + size_t(warp) * lay.bytes();
  uint64_t* bar = reinterpret_cast<uint64_t*>(base);
  double* qd = reinterpret_cast<double*>(base + 16);
  float* rows = reinterpret_cast<float*>(base + 16 + size_t(lay.d_pad) * 8);
  ListRef L{reinterpret_cast<double*>(base + lay.list_off()), nullptr, nullptr};
  L.id = reinterpret_cast<uint32_t*>(L.s + cap);
  L.fl = reinterpret_cast<uint8_t*>(L.id + cap);
  uint32_t* vis = lay.vis_smem ? reinterpret_cast<uint32_t*>(base + lay.vis_off())
                               : a.vis_global + size_t(b) * vis_words;
  uint32_t lcap = cap;
  bool spilled = false;
  uint32_t phase = 0;

  if (lane == 0) mbar_init(bar);
  for (uint32_t w = lane; w < vis_words; w += 32) vis[w] = 0;
  for (uint32_t i = lane; i < d; i += 32) qd[i] = (double)a.q[size_t(b) * d + i];
  __syncwarp();

  auto masked_id = [&](uint32_t v) -> bool {
    return a.mask_bits != nullptr && ((__ldg(a.mask_bits + (v >> 5)) >> (v & 31)) & 1u);
  };
  // exact scores of the lanes in `m` (lane j scores node v): key rows land in
  // the shared tile through TMA bulk copies (one round trip for all rows),
  // then each lane runs its in-order f64 chain from shared memory
  auto score_lanes = [&](uint32_t m, bool mine, uint32_t v) -> double {
    if constexpr (D > 0) {
      const uint32_t slot = __popc(m & ((1u << lane) - 1u));
      float* row = rows + size_t(slot) * lay.row_stride;
      fence_proxy_async();
      if (lane == 0) mbar_arrive_expect_tx(bar, __popc(m) * uint32_t(D) * 4u);
      __syncwarp();
      if (mine) bulk_g2s(row, keys + size_t(v) * D, uint32_t(D) * 4u, bar);
      mbar_wait(bar, phase);
      phase ^= 1u;
      return mine ? smem_dot<D>(qd, row) : -DBL_MAX;
    } else {
      return mine ? exact_dot<0>(qd, keys + size_t(v) * d, d) : -DBL_MAX;
    }
  };

  // ---- entry (:379-384) ----
  const uint32_t entry = (uint32_t)g.entry;
  double s0 = score_lanes(1u, lane == 0, entry);
  s0 = __shfl_sync(kFull, s0, 0);
  const bool m0 = masked_id(entry);
  if (lane == 0) {
    vis[entry >> 5] |= 1u << (entry & 31);
    L.s[0] = s0;
    L.id[0] = entry;
    L.fl[0] = m0 ? kMasked : 0;
  }
  __syncwarp();
  uint32_t len = 1, cursor = 0, n_unmasked = m0 ? 0 : 1;
  uint64_t scanned = 1;
  uint32_t expanded = 0;
  bool pool_full = false;
  double worst_s = -DBL_MAX;
  // speculation: adjacency row of the likely next top, held in registers
  uint32_t pre_u = kSentinel, pre_v = kSentinel;
  const bool spec = M <= 32;

  // position of the ef-th unmasked entry; then drop dead tail entries
  auto refresh_pool = [&]() {
    if (n_unmasked < ef) {
      pool_full = false;
      return;
    }
    uint32_t need = ef, pos = 0;
    for (uint32_t c = 0; c < len; c += 32) {
      const uint32_t i = c + lane;
      const bool um = i < len && !(L.fl[i] & kMasked);
      const uint32_t bm = __ballot_sync(kFull, um);
      const uint32_t cnt = __popc(bm);
      if (need <= cnt) {
        const bool hit = um && (uint32_t)__popc(bm & ((1u << lane) - 1u)) == need - 1;
        pos = c + __ffs(__ballot_sync(kFull, hit)) - 1;
        break;
      }
      need -= cnt;
    }
    pool_full = true;
    worst_s = L.s[pos];
    // first index > pos with score < worst (scores non-increasing)
    uint32_t lo = pos + 1, hi = len;
    while (lo < hi) {
      const uint32_t mid = (lo + hi) >> 1;
      if (L.s[mid] < worst_s)
        hi = mid;
      else
        lo = mid + 1;
    }
    if (lo < len) {
      uint32_t dropped_um = 0;
      for (uint32_t c = lo; c < len; c += 32) {
        const uint32_t i = c + lane;
        dropped_um += __popc(__ballot_sync(kFull, i < len && !(L.fl[i] & kMasked)));
      }
      n_unmasked -= dropped_um;
      len = lo;
    }
  };
  refresh_pool();

  for (;;) {
    // frontier top = first unexpanded entry at or after cursor
    uint32_t top = len, ubm = 0, ubase = 0;
    for (uint32_t c = cursor; c < len; c += 32) {
      const uint32_t i = c + lane;
      const uint32_t bm = __ballot_sync(kFull, i < len && !(L.fl[i] & kExpanded));
      if (bm) {
        top = c + __ffs(bm) - 1;
        ubm = bm & (bm - 1);  // further unexpanded entries of this chunk
        ubase = c;
        break;
      }
    }
    cursor = top;
    if (top >= len) break;                       // frontier exhausted
    if (pool_full && L.s[top] < worst_s) break;  // :390
    const uint32_t u = L.id[top];
    __syncwarp();
    if (lane == 0) L.fl[top] |= kExpanded;
    ++expanded;

    // adjacency of u: from the speculation registers when it guessed right
    uint32_t vrow;
    if (spec && pre_u == u) {
      vrow = pre_v;
    } else {
      vrow = lane < M ? __ldg(adj + size_t(u) * M + lane) : kSentinel;
    }
    // speculate: the next unexpanded entry is the likely next top; start
    // loading its adjacency now and prefetch the two after it into L2
    uint32_t nxt = kSentinel;
    if (spec && ubm) {
      const uint32_t i1 = ubase + __ffs(ubm) - 1;
      nxt = L.id[i1];
      pre_v = lane < M ? __ldg(adj + size_t(nxt) * M + lane) : kSentinel;
      const uint32_t rest = ubm & (ubm - 1);
      if (lane < 2 && rest) {
        uint32_t r = rest;
        if (lane == 1) r &= r - 1;
        if (r) {
          const uint32_t cand = L.id[ubase + __ffs(r) - 1];
          if ((M * 4) % 16 == 0)
            bulk_prefetch_l2(adj + size_t(cand) * M, M * 4);
          else
            asm volatile("prefetch.global.L2 [%0];" ::"l"(adj + size_t(cand) * M));
        }
      }
    }
    pre_u = nxt;

    for (uint32_t c0 = 0; c0 < M; c0 += 32) {
      const uint32_t v = c0 == 0 ? vrow
                                 : (c0 + lane < M ? __ldg(adj + size_t(u) * M + c0 + lane)
                                                  : kSentinel);
      const bool valid = v != kSentinel;
      const uint32_t grp = __match_any_sync(kFull, v);
      const bool first = (uint32_t)(__ffs(grp) - 1) == lane;
      __syncwarp();
      const bool isnew = valid && first && !((vis[v >> 5] >> (v & 31)) & 1u);
      __syncwarp();
      if (isnew) atomicOr(&vis[v >> 5], 1u << (v & 31));
      const uint32_t newmask = __ballot_sync(kFull, isnew);
      if (!newmask) continue;
      scanned += __popc(newmask);
      const double s = score_lanes(newmask, isnew, v);
      // second speculation level: the likely next top's unvisited neighbours'
      // key rows go to L2 while this expansion's list work runs
      if (c0 == 0 && pre_u != kSentinel && pre_v != kSentinel &&
          !((vis[pre_v >> 5] >> (pre_v & 31)) & 1u))
        bulk_prefetch_l2(keys + size_t(pre_v) * d, d * 4);
      const bool msk = isnew && masked_id(v);
      const bool live = isnew && !(pool_full && s < worst_s);
      const uint32_t livemask = __ballot_sync(kFull, live);
      if (!livemask) continue;
      const uint32_t nnew = __popc(livemask);

      double ks = live ? s : -DBL_MAX;
      uint32_t kid = live ? v : kSentinel;
      uint32_t kfl = msk ? kMasked : 0;
      warp_sort32(ks, kid, kfl, lane);

      // capacity: migrate L to its HBM spill slot (sized for every key)
      if (len + nnew > lcap) {
        if (spilled || a.spill == nullptr) __trap();  // unreachable: spill_cap >= n
        uint8_t* sb = a.spill + size_t(b) * ((size_t(spill_cap) * 13 + 15) & ~size_t(15));
        ListRef G{reinterpret_cast<double*>(sb), nullptr, nullptr};
        G.id = reinterpret_cast<uint32_t*>(G.s + spill_cap);
        G.fl = reinterpret_cast<uint8_t*>(G.id + spill_cap);
        for (uint32_t i = lane; i < len; i += 32) {
          G.s[i] = L.s[i];
          G.id[i] = L.id[i];
          G.fl[i] = L.fl[i];
        }
        __syncwarp();
        L = G;
        lcap = spill_cap;
        spilled = true;
      }

      // insertion points: #entries of L better than each new entry
      uint32_t p = 0;
      if (lane < nnew) {
        uint32_t lo = 0, hi = len;
        while (lo < hi) {
          const uint32_t mid = (lo + hi) >> 1;
          if (better(L.s[mid], L.id[mid], ks, kid))
            lo = mid + 1;
          else
            hi = mid;
        }
        p = lo;
      }
      const uint32_t pmin = __shfl_sync(kFull, p, 0);
      // shift L[pmin..len) up by #new entries inserted at or before them
      for (int topi = (int)len; topi > (int)pmin; topi -= 32) {
        const int i = topi - 32 + (int)lane;
        const bool act = i >= (int)pmin;
        double si = 0.0;
        uint32_t idi = 0;
        uint8_t fi = 0;
        if (act) {
          si = L.s[i];
          idi = L.id[i];
          fi = L.fl[i];
        }
        uint32_t cnt = 0;
#pragma unroll
        for (uint32_t step = 32; step >= 1; step >>= 1) {
          const uint32_t mid = cnt + step - 1;
          const uint32_t pm = __shfl_sync(kFull, p, mid & 31);
          if (mid < nnew && (int)pm <= i) cnt += step;
        }
        __syncwarp();
        if (act) {
          L.s[i + cnt] = si;
          L.id[i + cnt] = idi;
          L.fl[i + cnt] = fi;
        }
        __syncwarp();
      }
      if (lane < nnew) {
        L.s[p + lane] = ks;
        L.id[p + lane] = kid;
        L.fl[p + lane] = (uint8_t)kfl;
      }
      __syncwarp();
      len += nnew;
      n_unmasked += __popc(__ballot_sync(kFull, lane < nnew && !(kfl & kMasked)));
      if (pmin < cursor) cursor = pmin;
      refresh_pool();
      __syncwarp();
    }
  }

  // ---- result (:402-410): first min(k, pool) unmasked entries ----
  uint32_t taken = 0;
  for (uint32_t c = 0; c < len && taken < k; c += 32) {
    const uint32_t i = c + lane;
    const bool um = i < len && !(L.fl[i] & kMasked);
    const uint32_t bm = __ballot_sync(kFull, um);
    const uint32_t r = taken + __popc(bm & ((1u << lane) - 1u));
    if (um && r < k) {
      a.ids[size_t(b) * k + r] = L.id[i];
      a.scores[size_t(b) * k + r] = (float)L.s[i];
      if (a.scores64) a.scores64[size_t(b) * k + r] = L.s[i];
    }
    taken += __popc(bm);
  }
  const uint32_t take = taken < k ? taken : k;
  for (uint32_t r = take + lane; r < k; r += 32) {
    a.ids[size_t(b) * k + r] = kSentinel;
    a.scores[size_t(b) * k + r] = __int_as_float(0x7fc00000);
    if (a.scores64) a.scores64[size_t(b) * k + r] = __longlong_as_double(0x7ff8000000000000ll);
  }
  if (lane == 0) {
    a.n_out[b] = take;
    a.scanned[b] = scanned;
    if (a.scanned_own) a.scanned_own[b] = scanned;
    a.truncated[b] = take < k;
    if (a.expanded) a.expanded[b] = expanded;
  }
}

__global__ void k_mask_bitset(const uint32_t* mask, uint64_t mask_n, uint32_t* bits,
                              uint64_t words) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < mask_n;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const uint32_t v = mask[i];
    if ((v >> 5) < words) atomicOr(bits + (v >> 5), 1u << (v & 31));
  }
}

// order-preserving 64-bit key of a double (larger double -> larger key)
__device__ __forceinline__ uint64_t okey64(double x) {
  const uint64_t u = __double_as_longlong(x);
  return (u >> 63) ? ~u : (u | (1ull << 63));
}
__device__ __forceinline__ double okey64_inv(uint64_t k) {
  return __longlong_as_double((k >> 63) ? (k & ~(1ull << 63)) : ~k);
}
// k-th largest value of s[0, n) (k >= 1, n >= k): warp radix select, 8 bits
// per pass, histogram in shared memory (256 words)
__device__ double warp_kth_largest(const double* s, uint32_t n, uint32_t k, uint32_t* hist,
                                   uint32_t lane) {
  uint64_t prefix = 0, pmask = 0;
  uint32_t need = k;
  for (int shift = 56; shift >= 0; shift -= 8) {
    for (uint32_t b = lane; b < 256; b += 32) hist[b] = 0;
    __syncwarp();
    for (uint32_t i = lane; i < n; i += 32) {
      const uint64_t key = okey64(s[i]);
      if ((key & pmask) == prefix) atomicAdd(&hist[(key >> shift) & 255u], 1u);
    }
    __syncwarp();
    uint32_t local = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) local += hist[255 - (lane * 8 + j)];
    uint32_t incl = local;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(kFull, incl, o);
      if (lane >= uint32_t(o)) incl += t;
    }
    const uint32_t excl = incl - local;
    const uint32_t owner = __ffs(__ballot_sync(kFull, excl < need && incl >= need)) - 1;
    uint32_t digit = 0, before = 0;
    if (lane == owner) {
      uint32_t acc = excl;
      for (int j = 0; j < 8; ++j) {
        const uint32_t bkt = 255 - (lane * 8 + j);
        if (acc + hist[bkt] >= need) {
          digit = bkt;
          before = acc;
          break;
        }
        acc += hist[bkt];
      }
    }
    digit = __shfl_sync(kFull, digit, owner);
    before = __shfl_sync(kFull, before, owner);
    need -= before;
    prefix |= uint64_t(digit) << shift;
    pmask |= uint64_t(255) << shift;
    __syncwarp();
  }
  return okey64_inv(prefix);
}

// ---------------------------------------------------------------------------
// K6 v4: one CTA (4 warps) per query, speculative parallel pre-expansion.
//
// Round r: (A) every warp pre-expands frontier candidates chosen by warp 0 —
// adjacency row, visited filter, TMA row copies, exact in-order chains — into
// a "packet" {neighbour ids, exact scores, masked bits}; (B) warp 0 commits
// packets strictly in the reference's pop order. The round ends at the
// first top without a packet; it is pre-expanded next round. Packets are
// pure functions of (query, node), so only the committed expansion SET
// matters and the result is bit-identical to the reference.
//
// Commit-side state needs no sorting (the v2/v3 sorted list cost ~800
// dependent instructions per pop):
//   F = unexpanded visited nodes with score >= thr (unsorted); the reference's
//       frontier top (:387) is argmax_(score desc, id asc) F;
//   U = unmasked visited nodes with score >= thr (unsorted) = the pool's
//       candidates; pool full <=> #unmasked visited >= ef, and
//       top.score < pool.worst (:390)  <=>  #{u in U : u.score > top.score} >= ef,
//       a count (independent ballots), exact as long as thr <= pool worst;
//   thr = the exact pool worst at the last compaction (U sorted, cut to ef
//       + ties) — monotone, so dropping nodes below it never changes a pop
//       or the pool.
// Arrays live in shared memory and migrate to the query's HBM spill slot if
// they outgrow it, so no input can exceed capacity.
constexpr uint32_t kCW = 4;   // warps per CTA
constexpr uint32_t kCB = 6;   // candidates pre-expanded per round
constexpr uint32_t kCP = 16;  // packet slots
constexpr uint32_t kUSlack = 64;  // U grows to ef + slack before compaction

template <int D>
struct CtaLayout {
  uint32_t d_pad, cap, vis_words, vis_smem;  // cap = capacity of F and of U
  static constexpr uint32_t kRow = D + 4;     // padded TMA row stride (floats)
  __host__ __device__ static size_t tiles_off() { return 64 + size_t(D) * 8; }
  __host__ __device__ static size_t pk_off() {
    return tiles_off() + size_t(kCW) * 32 * kRow * 4;
  }
  // packets: tag u32[P], cnt u32[P], cand u32[B], slotof u32[B], ctrl u32[8],
  // masked u8[P][32] | ids u32[P][32] | scores f64[P][32]
  __host__ __device__ static size_t pk_hdr() {
    return (size_t(kCP) * 8 + kCB * 8 + 32 + size_t(kCP) * 32 + 15) & ~size_t(15);
  }
  __host__ __device__ static size_t pk_bytes() { return pk_hdr() + size_t(kCP) * 32 * 12; }
  __host__ __device__ size_t list_off() const { return pk_off() + pk_bytes(); }
  // F: s f64[cap], id u32[cap], m u8[cap] | U: s f64[cap], id u32[cap]
  __host__ __device__ static size_t list_bytes(uint32_t c) {
    return ((size_t(c) * 13 + 15) & ~size_t(15)) + ((size_t(c) * 12 + 15) & ~size_t(15));
  }
  __host__ __device__ size_t vis_off() const { return list_off() + list_bytes(cap); }
  __host__ __device__ size_t bytes() const {
    return vis_off() + (vis_smem ? ((size_t(vis_words) * 4 + 15) & ~size_t(15)) : 0);
  }
};

struct FArr {
  double* s;
  uint32_t* id;
  uint8_t* m;
};
struct UArr {
  double* s;
  uint32_t* id;
};

template <int D>
__global__ void __launch_bounds__(kCW * 32, 1)
    k_graph_search_cta(SearchArgs a, CtaLayout<D> lay, uint32_t spill_cap) {
  extern __shared__ __align__(16) uint8_t smem[];
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t b = blockIdx.x;
  const GraphDesc g = a.desc[b];
  const uint32_t M = g.M, ef = g.ef, k = a.k;
  const float* __restrict__ keys = g.keys;
  const uint32_t* __restrict__ adj = g.adj;
  const uint32_t vis_words = lay.vis_words;
  constexpr uint32_t RS = CtaLayout<D>::kRow;

  uint64_t* bar = reinterpret_cast<uint64_t*>(smem) + warp;
  double* qd = reinterpret_cast<double*>(smem + 64);
  float* tile = reinterpret_cast<float*>(smem + CtaLayout<D>::tiles_off()) + size_t(warp) * 32 * RS;
  uint8_t* pk = smem + CtaLayout<D>::pk_off();
  uint32_t* pk_tag = reinterpret_cast<uint32_t*>(pk);
  uint32_t* pk_cnt = pk_tag + kCP;
  uint32_t* cand = pk_cnt + kCP;
  uint32_t* slotof = cand + kCB;
  uint32_t* ctrl = slotof + kCB;  // [0] = #candidates, [1] = done
  uint8_t* pk_m = reinterpret_cast<uint8_t*>(ctrl + 8);  // [kCP][32]
  uint32_t* pk_id = reinterpret_cast<uint32_t*>(pk + CtaLayout<D>::pk_hdr());
  double* pk_s = reinterpret_cast<double*>(pk_id + kCP * 32);
  uint8_t* lists = smem + lay.list_off();
  const uint32_t cap = lay.cap;
  FArr F{reinterpret_cast<double*>(lists), nullptr, nullptr};
  F.id = reinterpret_cast<uint32_t*>(F.s + cap);
  F.m = reinterpret_cast<uint8_t*>(F.id + cap);
  UArr U{reinterpret_cast<double*>(lists + ((size_t(cap) * 13 + 15) & ~size_t(15))), nullptr};
  U.id = reinterpret_cast<uint32_t*>(U.s + cap);
  uint32_t* vis = lay.vis_smem ? reinterpret_cast<uint32_t*>(smem + lay.vis_off())
                               : a.vis_global + size_t(b) * vis_words;
  uint32_t phase = 0;

  if (lane == 0) mbar_init(bar);
  for (uint32_t w = threadIdx.x; w < vis_words; w += blockDim.x) vis[w] = 0;
  for (uint32_t i = threadIdx.x; i < D; i += blockDim.x) qd[i] = (double)a.q[size_t(b) * D + i];
  if (threadIdx.x < kCP) pk_tag[threadIdx.x] = kSentinel;
  __syncthreads();

  auto masked_id = [&](uint32_t v) -> bool {
    return a.mask_bits != nullptr && ((__ldg(a.mask_bits + (v >> 5)) >> (v & 31)) & 1u);
  };
  auto visited = [&](uint32_t v) -> bool { return (vis[v >> 5] >> (v & 31)) & 1u; };
  // TMA rows of the lanes in m into this warp's tile, then in-order chains
  auto score_lanes = [&](uint32_t m, bool mine, uint32_t v) -> double {
    const uint32_t slot = __popc(m & ((1u << lane) - 1u));
    float* row = tile + size_t(slot) * RS;
    fence_proxy_async();
    if (lane == 0) mbar_arrive_expect_tx(bar, __popc(m) * uint32_t(D) * 4u);
    __syncwarp();
    if (mine) bulk_g2s(row, keys + size_t(v) * D, uint32_t(D) * 4u, bar);
    mbar_wait(bar, phase);
    phase ^= 1u;
    return mine ? smem_dot<D>(qd, row) : -DBL_MAX;
  };

  // ---- commit-warp state ----
  uint32_t nF = 0, nU = 0, capF = cap, capU = cap, expanded = 0;
  uint64_t scanned = 0, u_total = 0;
  double thr = -DBL_MAX;  // exact pool worst at the last compaction
  bool spilledF = false, spilledU = false;
  uint8_t* spill_slot = a.spill ? a.spill + size_t(b) * CtaLayout<D>::list_bytes(spill_cap) : nullptr;

  auto spill_F = [&]() {
    if (spilledF || !spill_slot) __trap();  // unreachable: spill_cap >= n
    FArr G{reinterpret_cast<double*>(spill_slot), nullptr, nullptr};
    G.id = reinterpret_cast<uint32_t*>(G.s + spill_cap);
    G.m = reinterpret_cast<uint8_t*>(G.id + spill_cap);
    for (uint32_t i = lane; i < nF; i += 32) G.s[i] = F.s[i], G.id[i] = F.id[i], G.m[i] = F.m[i];
    __syncwarp();
    F = G;
    capF = spill_cap;
    spilledF = true;
  };
  auto spill_U = [&]() {
    if (spilledU || !spill_slot) __trap();
    UArr G{reinterpret_cast<double*>(spill_slot + ((size_t(spill_cap) * 13 + 15) & ~size_t(15))),
           nullptr};
    G.id = reinterpret_cast<uint32_t*>(G.s + spill_cap);
    for (uint32_t i = lane; i < nU; i += 32) G.s[i] = U.s[i], G.id[i] = U.id[i];
    __syncwarp();
    U = G;
    capU = spill_cap;
    spilledU = true;
  };

  // sort U[0, nU) best-first (bitonic over the next power of two)
  auto sort_U = [&]() {
    uint32_t p2 = 32;
    while (p2 < nU) p2 <<= 1;
    if (p2 > capU) spill_U();
    for (uint32_t i = nU + lane; i < p2; i += 32) U.s[i] = -DBL_MAX, U.id[i] = kSentinel;
    __syncwarp();
    for (uint32_t kk = 2; kk <= p2; kk <<= 1) {
      for (uint32_t j = kk >> 1; j > 0; j >>= 1) {
        for (uint32_t i = lane; i < p2; i += 32) {
          const uint32_t pj = i ^ j;
          if (pj > i) {
            const bool desc = (i & kk) == 0;
            const double si = U.s[i], sp = U.s[pj];
            const uint32_t ii = U.id[i], ip = U.id[pj];
            if (desc ? better(sp, ip, si, ii) : better(si, ii, sp, ip)) {
              U.s[i] = sp, U.s[pj] = si;
              U.id[i] = ip, U.id[pj] = ii;
            }
          }
        }
        __syncwarp();
      }
    }
  };

  // raise thr to the exact pool worst; keep U = pool + worst ties, drop dead F
  auto compact = [&]() {
    // exact ef-th best score by radix select (warp 0's TMA tile is idle here)
    thr = warp_kth_largest(U.s, nU, ef, reinterpret_cast<uint32_t*>(tile), lane);
    uint32_t keep = 0;  // U keeps everything >= thr (the pool plus worst-score ties)
    for (uint32_t c = 0; c < nU; c += 32) {
      const uint32_t i = c + lane;
      const bool in = i < nU;
      const double sv = in ? U.s[i] : 0.0;
      const uint32_t iv = in ? U.id[i] : 0;
      const bool kp = in && sv >= thr;
      const uint32_t bm = __ballot_sync(kFull, kp);
      __syncwarp();
      if (kp) {
        const uint32_t o = keep + __popc(bm & ((1u << lane) - 1u));
        U.s[o] = sv, U.id[o] = iv;
      }
      keep += __popc(bm);
      __syncwarp();
    }
    nU = keep;
    uint32_t w = 0;
    for (uint32_t c = 0; c < nF; c += 32) {
      const uint32_t i = c + lane;
      const bool in = i < nF;
      const double s = in ? F.s[i] : 0.0;
      const uint32_t id = in ? F.id[i] : 0;
      const uint8_t m = in ? F.m[i] : 0;
      const bool kp = in && s >= thr;
      const uint32_t bm = __ballot_sync(kFull, kp);
      __syncwarp();
      if (kp) {
        const uint32_t o = w + __popc(bm & ((1u << lane) - 1u));
        F.s[o] = s, F.id[o] = id, F.m[o] = m;
      }
      w += __popc(bm);
      __syncwarp();
    }
    nF = w;
  };

  // frontier top: argmax (score desc, id asc) over F; the lane-local bests
  // are kept for select()
  double lane_bs = -DBL_MAX;
  uint32_t lane_bid = kSentinel;
  auto argmax_F = [&](double& bs, uint32_t& bid, uint32_t& bidx) {
    bs = -DBL_MAX, bid = kSentinel, bidx = kSentinel;
#pragma unroll 4
    for (uint32_t i = lane; i < nF; i += 32) {
      const double s = F.s[i];
      const uint32_t id = F.id[i];
      if (better(s, id, bs, bid)) bs = s, bid = id, bidx = i;
    }
    lane_bs = bs, lane_bid = bid;
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      const double os = __shfl_xor_sync(kFull, bs, o);
      const uint32_t oid = __shfl_xor_sync(kFull, bid, o);
      const uint32_t oix = __shfl_xor_sync(kFull, bidx, o);
      if (better(os, oid, bs, bid)) bs = os, bid = oid, bidx = oix;
    }
  };

  // add new visited nodes (lane-held) to F and, if unmasked, to U
  auto add_nodes = [&](bool isnew, double s, uint32_t v, bool msk) {
    u_total += __popc(__ballot_sync(kFull, isnew && !msk));
    const bool inF = isnew && s >= thr;
    const bool inU = inF && !msk;
    const uint32_t mf = __ballot_sync(kFull, inF), mu = __ballot_sync(kFull, inU);
    if (nF + __popc(mf) > capF) spill_F();
    if (nU + __popc(mu) > capU) spill_U();
    if (inF) {
      const uint32_t o = nF + __popc(mf & ((1u << lane) - 1u));
      F.s[o] = s, F.id[o] = v, F.m[o] = msk ? 1 : 0;
    }
    if (inU) {
      const uint32_t o = nU + __popc(mu & ((1u << lane) - 1u));
      U.s[o] = s, U.id[o] = v;
    }
    nF += __popc(mf);
    nU += __popc(mu);
    __syncwarp();
    if (u_total >= ef && nU >= ef + kUSlack) compact();
  };

  // next round's candidates: each lane's best frontier node, warp-sorted,
  // first kCB taken (approximate top-kCB; the true top is always in it);
  // packets of other nodes are dropped
  auto select = [&](bool fresh) {
    double bs = lane_bs;
    uint32_t bid = lane_bid, dummy = 0;
    if (!fresh) {
      bs = -DBL_MAX, bid = kSentinel;
      for (uint32_t i = lane; i < nF; i += 32) {
        const double s = F.s[i];
        const uint32_t id = F.id[i];
        if (better(s, id, bs, bid)) bs = s, bid = id;
      }
    }
    warp_sort32(bs, bid, dummy, lane);
    const uint32_t ntop = min(kCB, (uint32_t)__popc(__ballot_sync(kFull, bid != kSentinel)));
    // slot bookkeeping in one match: candidate ids in lanes [0, ntop), packet
    // tags in lanes [16, 16 + kCP); other lanes hold unique dummies
    static_assert(kCB <= 16 && kCP <= 16, "slot match layout");
    const uint32_t tag = lane >= 16 ? pk_tag[lane - 16] : kSentinel;
    uint32_t val = 0xFFFFFF00u + lane;  // unique dummy (never a node id < n)
    if (lane < ntop) val = bid;
    else if (lane >= 16 && tag != kSentinel) val = tag;
    const uint32_t grp = __match_any_sync(kFull, val);
    const bool is_top = lane < ntop, is_tag = lane >= 16 && tag != kSentinel;
    const bool keep = is_tag && (grp & 0xFFFFu & ((1u << ntop) - 1u));  // tag is a top
    const bool has = is_top && (grp >> 16);                               // top has a packet
    if (lane >= 16 && !keep) pk_tag[lane - 16] = kSentinel;
    const uint32_t freemask = __ballot_sync(kFull, lane >= 16 && !keep) >> 16;
    const uint32_t needmask = __ballot_sync(kFull, is_top && !has);
    if (is_top && !has) {
      const uint32_t r = __popc(needmask & ((1u << lane) - 1u));
      uint32_t fm = freemask;  // r-th free slot
      for (uint32_t j = 0; j < r; ++j) fm &= fm - 1;
      const uint32_t sl = __ffs(fm) - 1;
      pk_tag[sl] = bid;
      cand[r] = bid;
      slotof[r] = sl;
    }
    __syncwarp();
    const uint32_t nc = __popc(needmask);
    if (lane == 0) ctrl[0] = nc;
  };

  uint64_t cyc_a = 0, cyc_b = 0, t_mark = clock64();
  uint64_t cy[5] = {0, 0, 0, 0, 0};  // argmax, stop test, packet apply, add/compact, select
  uint32_t rounds = 0;
  if (warp == 0) {
    // entry (:379-384)
    const uint32_t entry = (uint32_t)g.entry;
    double s0 = score_lanes(1u, lane == 0, entry);
    s0 = __shfl_sync(kFull, s0, 0);
    const bool m0 = masked_id(entry);
    if (lane == 0) {
      vis[entry >> 5] |= 1u << (entry & 31);
      ctrl[1] = 0;
    }
    scanned = 1;
    add_nodes(lane == 0, s0, entry, m0);
    select(false);
  }
  __syncthreads();

  for (;;) {
    // ---- (A) pre-expand candidates into packets, all warps ----
    const uint32_t nc = ctrl[0];
    ++rounds;
    if (threadIdx.x == 0) ctrl[2] = 0;
    for (uint32_t ci = warp; ci < nc; ci += kCW) {
      const uint32_t c = cand[ci], sl = slotof[ci];
      const uint32_t v = lane < M ? __ldg(adj + size_t(c) * M + lane) : kSentinel;
      const bool valid = v != kSentinel;
      const uint32_t grp = __match_any_sync(kFull, v);
      const bool first = (uint32_t)(__ffs(grp) - 1) == lane;
      const bool isnew = valid && first && !visited(v);
      const uint32_t newmask = __ballot_sync(kFull, isnew);
      double s = -DBL_MAX;
      if (newmask) s = score_lanes(newmask, isnew, v);
      const uint32_t o = __popc(newmask & ((1u << lane) - 1u));
      if (isnew) {
        pk_id[sl * 32 + o] = v;
        pk_s[sl * 32 + o] = s;
        pk_m[sl * 32 + o] = masked_id(v) ? 1 : 0;
        // likely future frontier tops: their adjacency rows go to L2 now
        if ((M * 4) % 16 == 0) bulk_prefetch_l2(adj + size_t(v) * M, M * 4);
      }
      if (lane == 0) pk_cnt[sl] = __popc(newmask);
    }
    __syncthreads();
    {
      const uint64_t t = clock64();
      cyc_a += t - t_mark;
      t_mark = t;
    }
    // ---- (B) commit in reference order, warp 0 ----
    if (warp == 0) {
      bool done = false;
      for (;;) {
        double ts;
        uint32_t tid, tix;
        uint64_t tc0 = clock64();
        argmax_F(ts, tid, tix);
        uint64_t tc1 = clock64();
        cy[0] += tc1 - tc0;
        if (tid == kSentinel) {  // frontier exhausted
          done = true;
          break;
        }
        if (u_total >= ef) {  // :390 — pool full and top below its worst
          uint32_t above = 0;
#pragma unroll 4
          for (uint32_t c = 0; c < nU; c += 32)
            above += __popc(__ballot_sync(kFull, c + lane < nU && U.s[c + lane] > ts));
          if (above >= ef) {
            done = true;
            break;
          }
        }
        {
          const uint64_t t = clock64();
          cy[1] += t - tc1;
          tc1 = t;
        }
        const uint32_t hit = __ballot_sync(kFull, lane < kCP && pk_tag[lane] == tid);
        if (!hit) break;  // next round pre-expands it
        const uint32_t sl = __ffs(hit) - 1;
        // pop: swap-remove from F
        if (lane == 0) {
          --nF;
          F.s[tix] = F.s[nF], F.id[tix] = F.id[nF], F.m[tix] = F.m[nF];
          pk_tag[sl] = kSentinel;
        }
        nF = __shfl_sync(kFull, nF, 0);
        __syncwarp();
        ++expanded;
        const uint32_t cnt = pk_cnt[sl];
        const uint32_t v = lane < cnt ? pk_id[sl * 32 + lane] : kSentinel;
        const double s = lane < cnt ? pk_s[sl * 32 + lane] : -DBL_MAX;
        const bool isnew = lane < cnt && !visited(v);
        __syncwarp();
        if (isnew) atomicOr(&vis[v >> 5], 1u << (v & 31));
        scanned += __popc(__ballot_sync(kFull, isnew));
        const bool msk = isnew && pk_m[sl * 32 + lane];
        {
          const uint64_t t = clock64();
          cy[2] += t - tc1;
          tc1 = t;
        }
        add_nodes(isnew, s, v, msk);
        cy[3] += clock64() - tc1;
      }
      const uint64_t tsel = clock64();
      if (done) {
        if (lane == 0) ctrl[1] = 1;
      } else {
        select(true);  // F unchanged since the argmax that ended the loop
      }
      cy[4] += clock64() - tsel;
      __threadfence_block();
      if (lane == 0) *reinterpret_cast<volatile uint32_t*>(&ctrl[2]) = 1;
    } else {
      // helpers: 2-hop L2 prefetch for the likely next tops — neighbours that
      // beat their parent in this round's packets — while warp 0 commits
      for (uint32_t ci = warp - 1; ci < nc; ci += kCW - 1) {
        const uint32_t sl = slotof[ci];
        const uint32_t cnt = pk_cnt[sl];
        const double ps = -DBL_MAX;  // parent score unknown here: use all entries
        (void)ps;
        const uint32_t want = __ballot_sync(kFull, lane < cnt);
        uint32_t done_n = 0;
        for (uint32_t q = want; q && done_n < 4; q &= q - 1, ++done_n) {
          if (*reinterpret_cast<volatile uint32_t*>(&ctrl[2])) break;
          const uint32_t x = pk_id[sl * 32 + (__ffs(q) - 1)];
          const uint32_t nb = lane < M ? __ldg(adj + size_t(x) * M + lane) : kSentinel;
          if (nb != kSentinel && !visited(nb)) bulk_prefetch_l2(keys + size_t(nb) * D, D * 4u);
        }
      }
    }
    __syncthreads();
    {
      const uint64_t t = clock64();
      cyc_b += t - t_mark;
      t_mark = t;
    }
    if (ctrl[1]) break;
  }

  if (warp != 0) return;
  if (a.dbg && lane == 0) {
    a.dbg[size_t(b) * 12 + 0] = rounds;
    a.dbg[size_t(b) * 12 + 1] = cyc_a;
    a.dbg[size_t(b) * 12 + 2] = cyc_b;
    a.dbg[size_t(b) * 12 + 3] = expanded;
    for (int j = 0; j < 5; ++j) a.dbg[size_t(b) * 12 + 4 + j] = cy[j];
  }
  // ---- result (:402-410): the pool's top min(k, |pool|), best-first ----
  sort_U();
  const uint32_t take = nU < k ? nU : k;
  for (uint32_t r = lane; r < k; r += 32) {
    const bool have = r < take;
    a.ids[size_t(b) * k + r] = have ? U.id[r] : kSentinel;
    a.scores[size_t(b) * k + r] = have ? (float)U.s[r] : __int_as_float(0x7fc00000);
    if (a.scores64)
      a.scores64[size_t(b) * k + r] = have ? U.s[r] : __longlong_as_double(0x7ff8000000000000ll);
  }
  if (lane == 0) {
    a.n_out[b] = take;
    a.scanned[b] = scanned;
    if (a.scanned_own) a.scanned_own[b] = scanned;
    a.truncated[b] = take < k;
    if (a.expanded) a.expanded[b] = expanded;
  }
}

bool tiled_dim(uint32_t d) { return d == 128 || d == 64 || d == 32 || d == 16 || d == 8; }

struct Plan {
  uint32_t wpb, cap, vis_smem, vis_words, d_pad, row_stride;
  size_t per_warp, smem;
};

// Shared-memory plan: one query per CTA while the batch cannot fill the SMs
// (each search then owns an SM's L1 and DFMA pipe), else 4 per CTA; the
// list capacity takes what is left after q, the TMA row tile and (if it
// fits) the visited bitset.
Plan plan(const ra_ctx* ctx, uint32_t B, uint32_t max_n, uint32_t d) {
  Plan p{};
  p.d_pad = (d + 1) & ~1u;
  p.vis_words = (max_n + 31) / 32;
  p.row_stride = d + 4;
  const size_t rows = tiled_dim(d) ? size_t(32) * p.row_stride * 4 : 0;
  const size_t budget = ctx->smem_optin ? ctx->smem_optin : 227 * 1024;
  p.wpb = B <= uint32_t(ctx->num_sms) ? 1 : 4;
  for (;;) {
    const size_t per_warp_budget = budget / p.wpb;
    const size_t fixed = 16 + size_t(p.d_pad) * 8 + rows + 32;
    const size_t vis_bytes = (size_t(p.vis_words) * 4 + 15) & ~size_t(15);
    p.vis_smem = fixed + vis_bytes + 13 * 512 <= per_warp_budget;
    const size_t rest = per_warp_budget - fixed - (p.vis_smem ? vis_bytes : 0);
    uint32_t cap = uint32_t(std::min<size_t>(rest / 13, 8192));
    cap = std::min<uint32_t>(cap, std::max<uint32_t>(max_n, 64));
    cap &= ~31u;
    if (cap >= 64 || p.wpb == 1) {
      p.cap = std::max<uint32_t>(cap, 32);
      break;
    }
    p.wpb /= 2;
  }
  p.per_warp = 16 + size_t(p.d_pad) * 8 + rows + ((size_t(p.cap) * 13 + 15) & ~size_t(15)) +
               (p.vis_smem ? ((size_t(p.vis_words) * 4 + 15) & ~size_t(15)) : 0);
  p.smem = p.per_warp * p.wpb;
  return p;
}

template <int D>
void launch_d(ra_ctx* ctx, const SearchArgs& a, const Plan& p, uint32_t spill_cap) {
  auto kern = k_graph_search<D>;
  WarpLayout<D> lay{p.d_pad, p.cap, p.vis_words, p.vis_smem, p.row_stride};
  if (lay.bytes() != p.per_warp) throw Error(RA_ERR_RUNTIME, "search smem layout mismatch");
  RA_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.smem));
  const uint32_t grid = (a.B + p.wpb - 1) / p.wpb;
  kern<<<grid, 32 * p.wpb, p.smem, ctx->stream>>>(a, p.wpb, lay, spill_cap);
  RA_LAUNCH_CHECK();
}

}  // namespace

size_t search_scratch_bytes(const ra_ctx* ctx, uint32_t B, uint32_t max_n, uint32_t d) {
  (void)ctx;
  (void)d;
  // covers both kernels: v4's F+U spill slots (pow2 capacity) dominate v2's list
  uint32_t p2 = 32;
  while (p2 < max_n) p2 <<= 1;
  size_t bytes = size_t(B) * (((size_t(p2) * 13 + 15) & ~size_t(15)) +
                              ((size_t(p2) * 12 + 15) & ~size_t(15))) + 256;
  bytes += size_t(B) * ((max_n + 31) / 32) * 4 + 256;  // HBM visited bitsets
  return std::max(bytes, search_pipe_scratch_bytes(B, max_n));
}

struct CtaPlan {
  bool ok;
  uint32_t cap, vis_smem, vis_words;
  size_t bytes;
};

uint32_t pow2_at_least(uint32_t x) {
  uint32_t p = 32;
  while (p < x) p <<= 1;
  return p;
}

template <int D>
CtaPlan cta_plan(const ra_ctx* ctx, uint32_t max_n) {
  CtaPlan p{};
  const size_t budget = ctx->smem_optin ? ctx->smem_optin : 227 * 1024;
  p.vis_words = (max_n + 31) / 32;
  CtaLayout<D> lay{0, 0, p.vis_words, 0};
  const size_t fixed = lay.list_off();
  const size_t vis_bytes = (size_t(p.vis_words) * 4 + 15) & ~size_t(15);
  if (fixed + CtaLayout<D>::list_bytes(256) > budget) return p;
  p.vis_smem = fixed + vis_bytes + CtaLayout<D>::list_bytes(512) <= budget;
  const size_t rest = budget - fixed - (p.vis_smem ? vis_bytes : 0) - 32;
  uint32_t cap = uint32_t(std::min<size_t>(rest / 25, 8192));
  cap = std::min<uint32_t>(cap, pow2_at_least(std::max<uint32_t>(max_n, 64)));
  p.cap = std::max<uint32_t>(cap & ~31u, 32);
  lay.cap = p.cap;
  lay.vis_smem = p.vis_smem;
  p.bytes = lay.bytes();
  p.ok = p.bytes <= budget;
  return p;
}

template <int D>
bool try_launch_cta(ra_ctx* ctx, const SearchArgs& a, uint32_t max_n, uint8_t* scratch) {
  const CtaPlan p = cta_plan<D>(ctx, max_n);
  if (!p.ok) return false;
  SearchArgs s = a;
  const uint32_t spill_cap = pow2_at_least(max_n);
  uint8_t* cur = scratch;
  s.spill = cur;
  cur += (size_t(a.B) * CtaLayout<D>::list_bytes(spill_cap) + 255) & ~size_t(255);
  s.vis_global = p.vis_smem ? nullptr : reinterpret_cast<uint32_t*>(cur);
  CtaLayout<D> lay{uint32_t(D), p.cap, p.vis_words, p.vis_smem};
  auto kern = k_graph_search_cta<D>;
  RA_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.bytes));
  kern<<<a.B, kCW * 32, p.bytes, ctx->stream>>>(s, lay, spill_cap);
  RA_LAUNCH_CHECK();
  return true;
}

// RA_SEARCH_KERNEL = pipe (default: latency or throughput mode by batch) |
// tp | lat | tpr (throughput, register rows only) | tps (throughput, shared
// visited bits + TMA tile) | duo (tps + an expansion warp per query) | cta |
// warp selects the K6 variant
int search_variant_of(const char* e) {
  if (!e) return 0;
  const std::string s(e);
  return s == "cta" ? 1 : s == "warp" ? 2 : s == "tp" ? 3 : s == "lat" ? 4 : s == "tpr" ? 5
         : s == "tps" ? 6 : s == "duo" ? 7 : s == "pipe" || s == "auto" ? 0 : -1;
}

int search_variant(const ra_ctx* ctx) {
  static const int v = [] {
    const int x = search_variant_of(std::getenv("RA_SEARCH_KERNEL"));
    return x < 0 ? 0 : x;
  }();
  return ctx && ctx->search_kernel >= 0 ? ctx->search_kernel : v;
}

bool search_fuses_attention(const ra_ctx* ctx, const SearchArgs& a, uint32_t max_n) {
  const int v = search_variant(ctx);
  if (!(v == 0 || v == 4) || a.B == 0) return false;
  if (v == 0 && a.B > 2u * uint32_t(ctx->num_sms)) return false;  // throughput mode
  return pipe_latency_supported(ctx, a.d, a.max_M, max_n);
}

void launch_graph_search(ra_ctx* ctx, SearchArgs a, uint32_t max_n, uint8_t* scratch) {
  if (a.B == 0) return;
  const int variant = search_variant(ctx);
  if ((variant == 0 || variant >= 3 || a.bf16) &&
      launch_graph_search_pipe(ctx, a, max_n, scratch,
                               variant == 3 ? 1 : variant == 4 ? 2 : variant == 5 ? 3
                               : variant == 6 ? 4 : variant == 7 ? 5 : 0))
    return;
  // the older kernels read f32 rows; the f32 copy of a bf16 group holds the
  // same rounded values, so they stay exact for shapes the pipe kernel skips
  // v3 (CTA per query, speculative pre-expansion) for the common shapes
  if (a.max_M <= 32 && variant <= 1) {
    bool done = false;
    switch (a.d) {
      case 128: done = try_launch_cta<128>(ctx, a, max_n, scratch); break;
      case 64: done = try_launch_cta<64>(ctx, a, max_n, scratch); break;
      case 32: done = try_launch_cta<32>(ctx, a, max_n, scratch); break;
      case 16: done = try_launch_cta<16>(ctx, a, max_n, scratch); break;
      case 8: done = try_launch_cta<8>(ctx, a, max_n, scratch); break;
      default: break;
    }
    if (done) return;
  }
  const Plan p = plan(ctx, a.B, max_n, a.d);
  uint8_t* cur = scratch;
  a.spill = nullptr;
  a.vis_global = nullptr;
  if (p.cap < max_n) {
    a.spill = cur;
    cur += (size_t(a.B) * ((size_t(max_n) * 13 + 15) & ~size_t(15)) + 255) & ~size_t(255);
  }
  if (!p.vis_smem) a.vis_global = reinterpret_cast<uint32_t*>(cur);
  switch (a.d) {
    case 128: launch_d<128>(ctx, a, p, max_n); break;
    case 64: launch_d<64>(ctx, a, p, max_n); break;
    case 32: launch_d<32>(ctx, a, p, max_n); break;
    case 16: launch_d<16>(ctx, a, p, max_n); break;
    case 8: launch_d<8>(ctx, a, p, max_n); break;
    default: launch_d<0>(ctx, a, p, max_n); break;
  }
}

void launch_mask_bitset(cudaStream_t s, const uint32_t* mask, uint64_t mask_n, uint32_t* bits,
                        uint64_t words) {
  RA_CUDA(cudaMemsetAsync(bits, 0, words * 4, s));
  if (!mask_n) return;
  const uint32_t grid = (uint32_t)std::min<uint64_t>((mask_n + 255) / 256, 1024);
  k_mask_bitset<<<grid, 256, 0, s>>>(mask, mask_n, bits, words);
  RA_LAUNCH_CHECK();
}

}  // namespace ra
