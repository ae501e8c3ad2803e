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

#include "common.cuh"

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

template <int D>
__global__ void __launch_bounds__(256) k_graph_search(SearchArgs a, uint32_t wpb, uint32_t cap,
                                                      uint32_t spill_cap, int vis_smem,
                                                      uint32_t vis_words, uint32_t d_pad) {
  extern __shared__ __align__(16) uint8_t smem[];
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t b = blockIdx.x * wpb + warp;
  if (b >= a.B) return;  // warp-uniform

  const GraphDesc g = a.desc[b];
  const uint32_t d = a.d, M = g.M, ef = g.ef, k = a.k;
  const float* __restrict__ keys = g.keys;
  const uint32_t* __restrict__ adj = g.adj;

  // ---- per-warp shared memory carve-up ----
  const size_t per_warp = size_t(d_pad) * 8 + size_t(cap) * 13 + (vis_smem ? vis_words * 4 : 0);
  const size_t per_warp_al = (per_warp + 15) & ~size_t(15);
  uint8_t* base = smem + warp * per_warp_al;
  double* qd = reinterpret_cast<double*>(base);
  ListRef L{reinterpret_cast<double*>(base + size_t(d_pad) * 8), nullptr, nullptr};
  L.id = reinterpret_cast<uint32_t*>(L.s + cap);
  L.fl = reinterpret_cast<uint8_t*>(L.id + cap);
  uint32_t* vis = vis_smem ? reinterpret_cast<uint32_t*>(base + size_t(d_pad) * 8 +
                                                         ((size_t(cap) * 13 + 3) & ~size_t(3)))
                           : a.vis_global + size_t(b) * vis_words;
  uint32_t lcap = cap;
  bool spilled = false;

  for (uint32_t w = lane; w < vis_words; w += 32) vis[w] = 0;
  for (uint32_t i = lane; i < d; i += 32) qd[i] = (double)a.q[size_t(b) * d + i];
  __syncwarp();

  auto masked_id = [&](uint32_t v) -> bool {
    return a.mask_bits != nullptr && ((__ldg(a.mask_bits + (v >> 5)) >> (v & 31)) & 1u);
  };

  // ---- entry (:379-384) ----
  const uint32_t entry = (uint32_t)g.entry;
  double s0 = 0.0;
  if (lane == 0) s0 = exact_dot<D>(qd, keys + size_t(entry) * d, d);
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
    uint32_t top = len;
    for (uint32_t c = cursor; c < len; c += 32) {
      const uint32_t i = c + lane;
      const uint32_t bm = __ballot_sync(kFull, i < len && !(L.fl[i] & kExpanded));
      if (bm) {
        top = c + __ffs(bm) - 1;
        break;
      }
    }
    cursor = top;
    if (top >= len) break;                             // frontier exhausted
    if (pool_full && L.s[top] < worst_s) break;        // :390
    const uint32_t u = L.id[top];
    __syncwarp();
    if (lane == 0) L.fl[top] |= kExpanded;
    ++expanded;

    for (uint32_t c0 = 0; c0 < M; c0 += 32) {
      const uint32_t j = c0 + lane;
      const uint32_t v = j < M ? __ldg(adj + size_t(u) * M + j) : kSentinel;
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
      double s = -DBL_MAX;
      if (isnew) s = exact_dot<D>(qd, keys + size_t(v) * d, d);
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

struct Plan {
  uint32_t wpb, cap, vis_smem, vis_words, d_pad;
  size_t smem;
};

Plan plan(const ra_ctx* ctx, uint32_t B, uint32_t max_n, uint32_t d) {
  Plan p{};
  p.d_pad = (d + 1) & ~1u;
  p.vis_words = (max_n + 31) / 32;
  const size_t budget = ctx->smem_optin ? ctx->smem_optin : 227 * 1024;
  // one query per CTA while the batch cannot fill the SMs; else 4 per CTA
  p.wpb = B <= uint32_t(ctx->num_sms) ? 1 : 4;
  for (;;) {
    const size_t per_warp_budget = budget / p.wpb;
    const size_t fixed = size_t(p.d_pad) * 8 + 16;
    const size_t vis_bytes = size_t(p.vis_words) * 4;
    p.vis_smem = fixed + vis_bytes + 13 * 512 <= per_warp_budget;
    size_t rest = per_warp_budget - fixed - (p.vis_smem ? vis_bytes : 0);
    uint32_t cap = uint32_t(std::min<size_t>(rest / 13, 8192));
    cap = std::min<uint32_t>(cap, std::max<uint32_t>(max_n, 64));
    cap &= ~31u;
    if (cap >= 64 || p.wpb == 1) {
      p.cap = std::max<uint32_t>(cap, 32);
      break;
    }
    p.wpb /= 2;
  }
  const size_t per_warp = size_t(p.d_pad) * 8 + size_t(p.cap) * 13 + 4 +
                          (p.vis_smem ? size_t(p.vis_words) * 4 : 0);
  p.smem = ((per_warp + 15) & ~size_t(15)) * p.wpb;
  return p;
}

template <int D>
void launch_d(ra_ctx* ctx, const SearchArgs& a, const Plan& p, uint32_t spill_cap) {
  auto kern = k_graph_search<D>;
  RA_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.smem));
  const uint32_t grid = (a.B + p.wpb - 1) / p.wpb;
  kern<<<grid, 32 * p.wpb, p.smem, ctx->stream>>>(a, p.wpb, p.cap, spill_cap, p.vis_smem,
                                                  p.vis_words, p.d_pad);
  RA_LAUNCH_CHECK();
}

}  // namespace

size_t search_scratch_bytes(const ra_ctx* ctx, uint32_t B, uint32_t max_n, uint32_t d) {
  const Plan p = plan(ctx, B, max_n, d);
  size_t bytes = 0;
  if (p.cap < max_n) bytes += size_t(B) * ((size_t(max_n) * 13 + 15) & ~size_t(15)) + 256;
  if (!p.vis_smem) bytes += size_t(B) * p.vis_words * 4 + 256;
  return bytes;
}

void launch_graph_search(ra_ctx* ctx, SearchArgs a, uint32_t max_n, uint8_t* scratch) {
  if (a.B == 0) return;
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
