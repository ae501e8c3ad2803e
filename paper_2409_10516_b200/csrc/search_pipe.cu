// K6 v5 ("pipe"): exact OODGraph::search
// (/root/reference/proj/src/index_oodgraph.cpp:357-411) as a producer /
// consumer pipeline inside one CTA per query.
//
// Warp 0 (the commit warp) replays the reference loop exactly: frontier top
// (:387), stop rule (:390), pop, visit the top's neighbours in commit order
// (:393-399). On a hit it never touches HBM: the neighbours' ids and exact
// in-order f64 scores come from a "packet" computed ahead of time by one of
// the helper warps 1..kPW-1. Packets are pure functions of (query, node), so
// only the committed expansion SET matters and ids / f32 scores / scanned /
// truncated are bit-identical to the reference (the commit warp re-filters a
// packet against the visited set at commit time; helpers filter only as a
// hint, and a stale filter can only add entries).
//
// Scores travel as order-preserving u64 keys (-0.0 folded into +0.0, so key
// equality is double equality); (key desc, id asc) is the reference order.
//
// Commit-side state, every operation a few independent instructions:
//   F (frontier): unexpanded visited nodes with key >= thr, kept as per-lane
//     UNSORTED lists in shared memory (kFR entries per lane, column layout;
//     helpers read them directly), each lane's best entry (its head) cached
//     in registers. Insert = one store plus one head compare; a full lane
//     hands new entries to the shared overflow FO, whose best entry is
//     tracked exactly. Frontier top = 3-REDUX argmax of the lane heads vs
//     FO's best; after a pop the owner lane's new head is rescanned.
//   U (pool candidates): unmasked visited nodes with key >= thr, kUR per
//     lane (unsorted, free mask) + overflow UO. pool.full() <=> #unmasked
//     visited >= ef, and top < pool.worst (:390) <=> #{u in U : u > top} >=
//     ef: 8 compares per lane and one REDUX.
//   thr: a key with >= ef U entries at or above it, i.e. thr <= pool worst
//     (key bisection, raised when U outgrows ef + slack). Nodes below the
//     pool worst can never be popped (the stop rule fires first) nor enter
//     the pool (its worst only rises), so dropping them is exact.
// Helpers: read the frontier lists and the hint ring (likely next tops),
// claim a way of a 2-way set-associative packet table with one 64-bit CAS,
// gather the
// adjacency row, TMA the unvisited neighbours' key rows into their tile,
// run the exact chains, publish the packet; then chain greedily into the
// best new neighbour (the likely next top) while it ranks among the heads.
//
// Throughput modes reuse the commit code with one query per warp (TP / TPS:
// inline expansions) or per warp PAIR (DUO): the commit warp learns the next
// top right after reading a packet (the best of the packet's new children
// >= thr and the frontier after the pop - the visit only inserts those
// children, a compaction can only end the search), starts that expansion
// (adjacency row, filter, L2 prefetch of the new rows) and posts it, then
// visits; the expansion warp runs the exact chains and returns the packet.
#include <cfloat>
#include <cstdlib>

#include "common.cuh"
#include "tma.cuh"

#ifdef RA_PIPE_PROFILE
constexpr bool kPipeProfile = true;
#define PIPE_TICK(slot)                \
  {                                    \
    const uint64_t t_ = clock64();     \
    cy[slot] += t_ - tq;               \
    tq = t_;                           \
  }
#else
constexpr bool kPipeProfile = false;
#define PIPE_TICK(slot)
#endif

namespace ra {
namespace {

#ifndef RA_PIPE_WARPS
#define RA_PIPE_WARPS 8
#endif
constexpr uint32_t kPW = RA_PIPE_WARPS;  // warps per CTA: 0 commits, 1.. pre-expand
#ifndef RA_TP_WARPS
#define RA_TP_WARPS 8
#endif
constexpr uint32_t kTW = RA_TP_WARPS;  // TP mode: queries (warps) per CTA
#ifndef RA_TP_MINB
#define RA_TP_MINB 2  // <= 128 registers: 16 query warps per SM
#endif
constexpr int kFR = 8;             // frontier entries per lane (sorted)
#ifndef RA_HINTS
#define RA_HINTS 64
#endif
constexpr uint32_t kHintN = RA_HINTS;  // hint ring entries (a power of two >= 32)
static_assert((kHintN & (kHintN - 1)) == 0 && kHintN >= 32,
              "the hint ring index is masked with kHintN - 1");
constexpr int kUR = 8;             // pool-candidate entries per lane
#ifndef RA_PIPE_SLOT_BITS
#define RA_PIPE_SLOT_BITS 7
#endif
constexpr uint32_t kSlotBits = RA_PIPE_SLOT_BITS;
constexpr uint32_t kSlots = 1u << kSlotBits;  // packet table, 2-way set-associative by node id
constexpr uint32_t kPick = 12;     // helpers consider the best kPick heads
constexpr uint32_t kChain = 3;     // greedy chain depth after a pre-expansion
#ifndef RA_PIPE_SLACK
#define RA_PIPE_SLACK 64
#endif
constexpr uint32_t kSlackU = RA_PIPE_SLACK;  // U grows to ef + slack before thr is raised
constexpr uint32_t sFREE = 0, sBUSY = 1, sREADY = 2, sTAKEN = 3;

// order-preserving key of a double; -0.0 and +0.0 share a key
__device__ __forceinline__ uint64_t okey(double x) {
  const uint64_t u = __double_as_longlong(x + 0.0);
  return (u >> 63) ? ~u : (u | (1ull << 63));
}
__device__ __forceinline__ double okey_inv(uint64_t k) {
  return __longlong_as_double((k >> 63) ? (k & ~(1ull << 63)) : ~k);
}
// a split point strictly inside (lo, hi) for the key bisections: the midpoint
// of the two SCORES (scores cluster: a key-space midpoint of keys whose
// scores differ in sign or exponent barely moves in 8 steps), else the
// key-space midpoint. Any split keeps the bisection exact.
__device__ __forceinline__ uint64_t key_mid(uint64_t lo, uint64_t hi) {
  const uint64_t km = lo + ((hi - lo) >> 1);
  if (hi - lo < 4) return km;
  const uint64_t vm = okey(0.5 * okey_inv(lo) + 0.5 * okey_inv(hi));
  return (vm > lo && vm < hi) ? vm : km;
}
// (key desc, id asc); the empty entry (0, kSentinel) is worse than any node
__device__ __forceinline__ bool better(uint64_t ka, uint32_t ia, uint64_t kb, uint32_t ib) {
  return ka > kb || (ka == kb && ia < ib);
}
__device__ __forceinline__ uint64_t slotword(uint32_t key, uint32_t st) {
  return (uint64_t(st) << 32) | key;
}
// first slot of id's set (a node's packet lives in slot_of(id) or slot_of(id) + 1)
__device__ __forceinline__ uint32_t slot_of(uint32_t id) {
  return ((id * 2654435761u) >> (33 - kSlotBits)) << 1;
}
__device__ __forceinline__ uint32_t lanemask_lt(uint32_t lane) { return (1u << lane) - 1u; }
// release store to a shared word (the reads before it complete first)
__device__ __forceinline__ void st_release_cta(unsigned long long* p, uint64_t v) {
  asm volatile("st.release.cta.shared::cta.u64 [%0], %1;" ::"r"(
                   static_cast<uint32_t>(__cvta_generic_to_shared(p))),
               "l"(v)
               : "memory");
}

// Best-first bitonic sort of 256 (key, id) entries held by one warp, entry
// lane * 8 + i in register i: distances < 8 inside a lane, the rest by
// shuffles (15 of the 36 stages).
__device__ __forceinline__ void warp_sort256(uint64_t (&k)[8], uint32_t (&id)[8], uint32_t lane) {
#pragma unroll
  for (uint32_t kk = 2; kk <= 256; kk <<= 1) {
#pragma unroll
    for (uint32_t j = kk >> 1; j > 0; j >>= 1) {
      if (j >= 8) {
        const uint32_t lj = j >> 3;
        const bool lower = (lane & lj) == 0;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const uint32_t e = lane * 8 + i;
          const bool desc = (e & kk) == 0;
          const uint64_t pk = __shfl_xor_sync(0xffffffffu, k[i], lj);
          const uint32_t pi = __shfl_xor_sync(0xffffffffu, id[i], lj);
          // the lower index keeps the better entry in a descending block
          const bool pb = better(pk, pi, k[i], id[i]);
          if (pb == (lower == desc)) k[i] = pk, id[i] = pi;
        }
      } else {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int pj = i ^ int(j);
          if (pj > i) {
            const uint32_t e = lane * 8 + i;
            const bool desc = (e & kk) == 0;
            const bool sw = desc ? better(k[pj], id[pj], k[i], id[i])
                                 : better(k[i], id[i], k[pj], id[pj]);
            if (sw) {
              const uint64_t tk = k[i];
              const uint32_t ti = id[i];
              k[i] = k[pj], id[i] = id[pj];
              k[pj] = tk, id[pj] = ti;
            }
          }
        }
      }
    }
  }
}

// in-order f64 dot of q (f64, smem) and a key row staged in shared memory
// (dot_f64, index_oodgraph.cpp:40-44; f32 x f32 products are exact in f64).
// The chain of D dependent DFMAs is the floor; the operands of chunk c + 1
// (4 LDS.128 of q, 2 of the row) are requested during chunk c's 8 DFMAs so
// no DFMA waits on a shared-memory load.
template <int D>
__device__ __forceinline__ double row_dot(const double* __restrict__ qd,
                                          const float* __restrict__ row) {
  static_assert(D % 8 == 0, "row_dot takes d in multiples of 8");
  const double2* q2 = reinterpret_cast<const double2*>(qd);
  const float4* r4 = reinterpret_cast<const float4*>(row);
  constexpr int NC = D / 8;
  double2 qa[4], qb[4];
  float4 ra[2], rb[2];
  auto load = [&](int c, double2 (&q)[4], float4 (&r)[2]) {
#pragma unroll
    for (int j = 0; j < 4; ++j) q[j] = q2[4 * c + j];
    r[0] = r4[2 * c];
    r[1] = r4[2 * c + 1];
  };
  double acc = 0.0;
  auto fma8 = [&](const double2 (&q)[4], const float4 (&r)[2]) {
    acc = fma(q[0].x, (double)r[0].x, acc);
    acc = fma(q[0].y, (double)r[0].y, acc);
    acc = fma(q[1].x, (double)r[0].z, acc);
    acc = fma(q[1].y, (double)r[0].w, acc);
    acc = fma(q[2].x, (double)r[1].x, acc);
    acc = fma(q[2].y, (double)r[1].y, acc);
    acc = fma(q[3].x, (double)r[1].z, acc);
    acc = fma(q[3].y, (double)r[1].w, acc);
  };
  load(0, qa, ra);
#pragma unroll
  for (int c = 0; c < NC; c += 2) {
    if (c + 1 < NC) load(c + 1, qb, rb);
    fma8(qa, ra);
    if (c + 2 < NC) load(c + 2, qa, ra);
    if (c + 1 < NC) fma8(qb, rb);
  }
  return acc;
}

// the plain loop form of the same chain (the compiler interleaves the
// operand loads with the DFMAs)
template <int D>
__device__ __forceinline__ double row_dot_seq(const double* __restrict__ qd,
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

__device__ __forceinline__ double bf_lo(uint32_t w) { return (double)__uint_as_float(w << 16); }
__device__ __forceinline__ double bf_hi(uint32_t w) { return (double)__uint_as_float(w & 0xFFFF0000u); }

// in-order f64 dot of q and a bf16 row (8 elements per 16-B word; bf16 ->
// f32 -> f64 is exact, so this is dot_f64 on the rounded key)
template <int D>
__device__ __forceinline__ double row_dot_bf(const double* __restrict__ qd,
                                             const uint4* __restrict__ r4, bool global) {
  double acc = 0.0;
#pragma unroll 4
  for (int c = 0; c < D / 8; ++c) {
    const uint4 w = global ? __ldg(r4 + c) : r4[c];
    const double* q8 = qd + 8 * c;
    acc = fma(q8[0], bf_lo(w.x), acc);
    acc = fma(q8[1], bf_hi(w.x), acc);
    acc = fma(q8[2], bf_lo(w.y), acc);
    acc = fma(q8[3], bf_hi(w.y), acc);
    acc = fma(q8[4], bf_lo(w.z), acc);
    acc = fma(q8[5], bf_hi(w.z), acc);
    acc = fma(q8[6], bf_lo(w.w), acc);
    acc = fma(q8[7], bf_hi(w.w), acc);
  }
  return acc;
}

// 32-lane bitonic sort, best-first
__device__ __forceinline__ void sort32(uint64_t& k, uint32_t& id, uint32_t lane) {
#pragma unroll
  for (int kk = 2; kk <= 32; kk <<= 1) {
#pragma unroll
    for (int j = kk >> 1; j > 0; j >>= 1) {
      const uint64_t ko = __shfl_xor_sync(kFull, k, j);
      const uint32_t io = __shfl_xor_sync(kFull, id, j);
      const bool lower = (lane & j) == 0;
      const bool desc = (lane & kk) == 0;
      const bool take = (lower == desc) ? better(ko, io, k, id) : better(k, id, ko, io);
      if (take) k = ko, id = io;
    }
  }
}

// warp argmax under (key desc, id asc) with three REDUX; all lanes get it
__device__ __forceinline__ void warp_best(uint64_t& k, uint32_t& id) {
  const uint32_t hi = __reduce_max_sync(kFull, uint32_t(k >> 32));
  const bool m1 = uint32_t(k >> 32) == hi;
  const uint32_t lo = __reduce_max_sync(kFull, m1 ? uint32_t(k) : 0u);
  const bool m2 = m1 && uint32_t(k) == lo;
  id = __reduce_min_sync(kFull, m2 ? id : kSentinel);
  k = (uint64_t(hi) << 32) | lo;
}

struct PipeLayout {
  uint32_t D, MT, vis_words, vis_smem, capO;
  uint32_t duo = 0;  // TP "duo" variant: a commit warp + an expansion warp per query
  static constexpr size_t kBars = 0, kCtrl = (size_t(kPW) * 8 + 63) / 64 * 64,  // one mbarrier per warp
                          kPubK = kCtrl + 64, kPubId = kPubK + 256, kSlotW = kPubId + 128,
                          kCnt = kSlotW + size_t(kSlots) * 8, kMb = kCnt + size_t(kSlots) * 4,
                          kNk = kMb + size_t(kSlots) * 4, kPkId = kNk + size_t(kSlots) * 8,
                          kPkK = kPkId + size_t(kSlots) * 32 * 4,
                          kPubF = kPkK + size_t(kSlots) * 32 * 8,  // F: k u64[kFR][32], id u32[kFR][32]
                          kHint = kPubF + size_t(kFR) * 32 * 12,   // hints: k u64[N], id u32[N]
                          kQd = kHint + size_t(kHintN) * 12;
  __host__ __device__ size_t row_floats() const { return D + 4; }
  __host__ __device__ size_t tiles_off() const { return kQd + size_t(D) * 8; }
  __host__ __device__ size_t tile_bytes() const { return size_t(MT) * row_floats() * 4; }
  __host__ __device__ size_t vis_off() const { return tiles_off() + kPW * tile_bytes(); }
  __host__ __device__ size_t vis_bytes() const {
    return vis_smem ? ((size_t(vis_words) * 8 + 15) & ~size_t(15)) : 0;  // visited + expanded
  }
  __host__ __device__ size_t fo_off() const { return vis_off() + vis_bytes(); }
  __host__ __device__ static size_t arr_bytes(uint32_t c) {
    return (size_t(c) * 12 + 15) & ~size_t(15);
  }
  __host__ __device__ size_t uo_off() const { return fo_off() + arr_bytes(capO); }
  __host__ __device__ size_t bytes() const { return uo_off() + arr_bytes(capO); }
  // TP mode: per warp q (f64) | FO | UO | F lists; with vis_smem (the
  // "TPS" variant) also a TMA row tile and the visited bitset, behind a
  // 128-B block of per-warp mbarriers
  __host__ __device__ size_t tp_base() const { return vis_smem ? 128 : 0; }
  __host__ __device__ size_t tp_flist_off() const { return size_t(D) * 8 + 2 * arr_bytes(capO); }
  __host__ __device__ size_t tp_tile_off() const { return tp_flist_off() + size_t(kFR) * 32 * 12; }
  __host__ __device__ size_t tp_vis_off() const {
    return tp_tile_off() + (vis_smem ? tile_bytes() : 0);
  }
  __host__ __device__ size_t tp_duo_off() const {
    return tp_vis_off() + (vis_smem ? ((size_t(vis_words) * 4 + 15) & ~size_t(15)) : 0);
  }
  // duo mailbox: request u64 (seq << 32 | node), ready u32, packet flags
  // u32[2], thr u64, packet key u64[32] / id u32[32], request ids u32[32] +
  // request flags u32[2] (see k_graph_search_pipe)
  static constexpr size_t kDuoBytes = 32 + 32 * 12 + 32 * 4 + 16;
  __host__ __device__ size_t tp_warp_bytes() const { return tp_duo_off() + (duo ? kDuoBytes : 0); }
};

struct Arr {  // (key, id) array: k u64[cap] then id u32[cap]
  uint64_t* k;
  uint32_t* id;
  __device__ static Arr at(uint8_t* base, uint32_t cap) {
    Arr a{reinterpret_cast<uint64_t*>(base), nullptr};
    a.id = reinterpret_cast<uint32_t*>(a.k + cap);
    return a;
  }
};

// TP (throughput mode): every warp is a commit warp running its own query
// with inline expansions (key rows straight into registers), kTW queries
// per CTA, visited set in HBM/L2; for batches that fill the GPU many times.
// BF: key rows are read from the group's bf16 copy (half the bytes)
// Omega partial over the sorted pool's top `m` (exact search scores, rank
// order) + the W chunks folded in chunk order + merge (attention.cpp:102-157,
// the same arithmetic as k_omega_merge). All threads of the CTA; the V rows
// are staged in the (free) tile area behind the sorted array.
template <int D>
__device__ void fused_attention_tail(const SearchArgs& a, const PipeLayout& lay, uint32_t b,
                                     const Arr& A, uint32_t p2, bool fin_smem, uint32_t m,
                                     uint8_t* smem) {
  const uint32_t tid = threadIdx.x, nth = blockDim.x;
  const auto& fa = a.fa;
  constexpr uint32_t CB = 32;  // W chunk partials staged per round
  // a fresh mbarrier in ctrl[14..15] (unused words; the warps' own are left alone)
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + PipeLayout::kCtrl + 14 * 4);
  const size_t a_bytes = fin_smem ? ((PipeLayout::arr_bytes(p2) + 15) & ~size_t(15)) : 0;
  uint8_t* base = smem + lay.tiles_off() + a_bytes;
  double* red = reinterpret_cast<double*>(base);         // [8] block max
  double* wx = red + 8;                                  // [CB] chunk weights
  double* chs = wx + CB;                                 // [CB][D + 2] staged partials
  double* e = chs + size_t(CB) * (D + 2);                // [R]
  const size_t head = size_t(8 + CB + size_t(CB) * (D + 2)) * 8;
  const size_t avail = size_t(kPW) * lay.tile_bytes() - a_bytes - head;
  // rows per pass (>= 8, see fin_smem); even, so Vt stays 16-B aligned
  const uint32_t R = uint32_t(avail / (size_t(D) * 4 + 8)) & ~1u;
  if (R == 0) __trap();  // unreachable: launch_pipe_d sizes the tiles for >= 8 rows
  float* Vt = reinterpret_cast<float*>(e + R);  // [R][D]
  const float* V = fa.values[b];
  const double* ch = fa.chunk + size_t(b) * fa.nchunk * (D + 2);
  const double zo = m ? okey_inv(A.k[0]) * fa.inv_sqrt_d : -DBL_MAX;  // sorted: the max
  if (tid == 0) mbar_init(bar);
  __syncthreads();
  uint32_t rows = min(R, m), phase = 0;
  // the first pass's V rows are requested first; the W fold runs under them
  // (every issuing thread orders the area's earlier generic accesses first)
  fence_proxy_async();
  if (tid == 0) mbar_arrive_expect_tx(bar, rows * uint32_t(D) * 4u);
  __syncthreads();
  for (uint32_t i = tid; i < rows; i += nth) {
    bulk_g2s(Vt + size_t(i) * D, V + size_t(A.id[i]) * D, D * 4u, bar);
    e[i] = exp(okey_inv(A.k[i]) * fa.inv_sqrt_d - zo);
  }
  // W: the chunk partials (one staging round when they fit), their max, then
  // the chunks in order
  const bool one = fa.nchunk <= CB;
  double zw = -DBL_MAX;
  if (one) {
    for (uint32_t x = tid; x < fa.nchunk * (D + 2); x += nth) chs[x] = ch[x];
    __syncthreads();
    for (uint32_t c = 0; c < fa.nchunk; ++c) zw = fmax(zw, chs[size_t(c) * (D + 2) + D]);
  } else {
    for (uint32_t c = tid; c < fa.nchunk; c += nth) zw = fmax(zw, ch[size_t(c) * (D + 2) + D]);
#pragma unroll
    for (int o = 16; o; o >>= 1) zw = fmax(zw, __shfl_xor_sync(kFull, zw, o));
    if ((tid & 31) == 0) red[tid >> 5] = zw;
    __syncthreads();
    zw = red[0];
    for (uint32_t w = 1; w < nth / 32; ++w) zw = fmax(zw, red[w]);
  }
  double sw = 0.0, ow = 0.0;
  const uint32_t j = tid;  // this thread's output dimension (j < D)
  for (uint32_t c0 = 0; c0 < fa.nchunk; c0 += CB) {
    const uint32_t cn = min(CB, fa.nchunk - c0);
    if (!one) {
      for (uint32_t x = tid; x < cn * (D + 2); x += nth) chs[x] = ch[size_t(c0) * (D + 2) + x];
      __syncthreads();
    }
    if (tid < cn) wx[tid] = exp(chs[size_t(tid) * (D + 2) + D] - zw);
    __syncthreads();
    for (uint32_t c = 0; c < cn; ++c) {  // chunk order
      sw += wx[c] * chs[size_t(c) * (D + 2) + D + 1];
      if (j < uint32_t(D)) ow += wx[c] * chs[size_t(c) * (D + 2) + j];
    }
    __syncthreads();  // chs reused
  }
  // Omega: sum e_i v_i in rank order, pass by pass
  double acc = 0.0, so = 0.0;
  for (uint32_t t0 = 0; t0 < m; t0 += R) {
    if (t0) {
      rows = min(R, m - t0);
      __syncthreads();  // previous pass consumed
      fence_proxy_async();
      if (tid == 0) mbar_arrive_expect_tx(bar, rows * uint32_t(D) * 4u);
      __syncthreads();
      for (uint32_t i = tid; i < rows; i += nth) {
        bulk_g2s(Vt + size_t(i) * D, V + size_t(A.id[t0 + i]) * D, D * 4u, bar);
        e[i] = exp(okey_inv(A.k[t0 + i]) * fa.inv_sqrt_d - zo);
      }
    }
    mbar_wait(bar, phase);
    phase ^= 1u;
    __syncthreads();  // e[] visible
    for (uint32_t i = 0; i < rows; ++i) {
      const double ei = e[i];
      so += ei;
      if (j < uint32_t(D)) acc = fma(ei, (double)Vt[size_t(i) * D + j], acc);
    }
  }
  if (j >= uint32_t(D)) return;
  const bool we = fa.nW == 0, oe = m == 0;
  double gw = 1.0, go = 0.0;
  if (we) {
    gw = 0.0, go = 1.0;
  } else if (!oe) {
    const double zref = fmax(zw, zo);
    const double ew = exp(zw - zref) * sw, eo = exp(zo - zref) * so;
    gw = ew / (ew + eo);
    go = eo / (ew + eo);
  }
  if (!we) ow /= sw;
  const double oo = oe ? 0.0 : acc / so;
  fa.out[size_t(b) * D + j] = we ? oo : (oe ? ow : gw * ow + go * oo);
}

// the two warps of a DUO query (named barrier 1 + pair)
__device__ __forceinline__ void pair_sync(uint32_t pair) {
  asm volatile("bar.sync %0, 64;" ::"r"(pair + 1u) : "memory");
}

// DUO: pairs of warps per query in throughput mode (<= kDuoPairs per CTA:
// 14 warps at <= 144 registers fill the register file)
constexpr uint32_t kDuoPairs = 7;

template <int D, bool VS, bool TP, bool BF, bool DUO = false>
__global__ void __launch_bounds__(TP ? (DUO ? kDuoPairs * 64 : kTW * 32) : kPW * 32,
                                  TP ? (VS ? 1 : RA_TP_MINB) : 1)
    k_graph_search_pipe(SearchArgs a, PipeLayout lay, uint32_t spill_cap) {
  extern __shared__ __align__(16) uint8_t smem[];
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // DUO: with P queries per CTA, warp j < P commits query j and warp P + j
  // expands for it, so the expansion warps (the DFMA / F2F work) spread over
  // all four SMSPs (warp % 4) instead of the odd two
  const uint32_t duo_p = blockDim.x >> 6;
  const bool duo_x = DUO && warp >= duo_p;  // this warp is an expansion warp
  const uint32_t qslot = DUO ? (duo_x ? warp - duo_p : warp) : warp;
  const uint32_t b = TP ? blockIdx.x * (blockDim.x >> (DUO ? 6 : 5)) + qslot : blockIdx.x;
  if (TP && b >= a.B) return;  // warp-uniform; TP never uses CTA barriers
  const GraphDesc g = a.desc[b];
  const uint32_t M = g.M, ef = g.ef, k = a.k, n = g.n;
  const float* __restrict__ keys = g.keys;
  const uint16_t* __restrict__ keys16 = g.keys16;
  constexpr uint32_t kRowBytes = uint32_t(D) * (BF ? 2u : 4u);
  const uint32_t* __restrict__ adj = g.adj;
  constexpr uint32_t RS = D + 4;

  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + PipeLayout::kBars) + warp;
  volatile uint32_t* ctrl = reinterpret_cast<volatile uint32_t*>(smem + PipeLayout::kCtrl);
  volatile uint64_t* pub_k = reinterpret_cast<volatile uint64_t*>(smem + PipeLayout::kPubK);
  volatile uint32_t* pub_id = reinterpret_cast<volatile uint32_t*>(smem + PipeLayout::kPubId);
  volatile uint64_t* pubf_k = reinterpret_cast<volatile uint64_t*>(smem + PipeLayout::kPubF);
  volatile uint32_t* pubf_id = reinterpret_cast<volatile uint32_t*>(pubf_k + kFR * 32);
  // hint ring: the runner-up children of recent pre-expansions (likely tops
  // right after their parent commits), written by helpers, read by helpers
  volatile uint64_t* hint_k = reinterpret_cast<volatile uint64_t*>(smem + PipeLayout::kHint);
  volatile uint32_t* hint_id = reinterpret_cast<volatile uint32_t*>(hint_k + kHintN);
  // one entry into the 32-slot hint ring (any warp, one lane)
  auto push_hint = [&](uint64_t k, uint32_t id) {
    const uint32_t h = atomicAdd(const_cast<uint32_t*>(ctrl) + 12, 1u) & (kHintN - 1u);
    hint_id[h] = kSentinel;
    hint_k[h] = k;
    hint_id[h] = id;
  };
  unsigned long long* slotw = reinterpret_cast<unsigned long long*>(smem + PipeLayout::kSlotW);
  uint32_t* pk_cnt = reinterpret_cast<uint32_t*>(smem + PipeLayout::kCnt);
  uint32_t* pk_mb = reinterpret_cast<uint32_t*>(smem + PipeLayout::kMb);
  volatile uint64_t* pk_nk = reinterpret_cast<volatile uint64_t*>(smem + PipeLayout::kNk);
  uint32_t* pk_id = reinterpret_cast<uint32_t*>(smem + PipeLayout::kPkId);
  uint64_t* pk_k = reinterpret_cast<uint64_t*>(smem + PipeLayout::kPkK);
  uint8_t* const wbase = smem + lay.tp_base() + qslot * lay.tp_warp_bytes();  // TP: this query's
  double* qd = TP ? reinterpret_cast<double*>(wbase)
                  : reinterpret_cast<double*>(smem + PipeLayout::kQd);
  float* tile = reinterpret_cast<float*>(TP ? wbase + lay.tp_tile_off()
                                            : smem + lay.tiles_off() + warp * lay.tile_bytes());
  const uint32_t vw = lay.vis_words;
  uint32_t* vis = VS ? reinterpret_cast<uint32_t*>(TP ? wbase + lay.tp_vis_off()
                                                       : smem + lay.vis_off())
                     : a.vis_global + size_t(b) * 2 * vw;
  uint32_t* expd = vis + vw;
  uint8_t* spill_slot = a.spill + size_t(b) * 2 * PipeLayout::arr_bytes(spill_cap);
  // DUO mailbox (PipeLayout::kDuoBytes): the commit warp posts the next top
  // (seq << 32 | node; node = kSentinel stops the expansion warp), which
  // returns that node's packet (per-lane key / id, new / masked ballots)
  uint8_t* const duo = wbase + lay.tp_duo_off();
  volatile unsigned long long* duo_req = reinterpret_cast<volatile unsigned long long*>(duo);
  volatile uint32_t* duo_rdy = reinterpret_cast<volatile uint32_t*>(duo + 8);
  volatile uint32_t* duo_flags = reinterpret_cast<volatile uint32_t*>(duo + 12);  // [2]
  volatile uint64_t* duo_thr = reinterpret_cast<volatile uint64_t*>(duo + 24);
  volatile uint64_t* duo_pk = reinterpret_cast<volatile uint64_t*>(duo + 32);
  volatile uint32_t* duo_pi = reinterpret_cast<volatile uint32_t*>(duo + 32 + 32 * 8);
  volatile uint32_t* duo_rv = reinterpret_cast<volatile uint32_t*>(duo + 32 + 32 * 12);  // [32]
  volatile uint32_t* duo_rf = reinterpret_cast<volatile uint32_t*>(duo + 32 + 32 * 16);  // [2]

  if constexpr (TP) {
    if constexpr (DUO) {
      if (!duo_x) {
        for (uint32_t w = lane; w < vw; w += 32) vis[w] = 0;
        for (uint32_t i = lane; i < D; i += 32) qd[i] = (double)a.q[size_t(b) * D + i];
      } else if (lane == 0) {
        mbar_init(bar);
        *duo_req = 0, *duo_rdy = 0, *duo_thr = 0;
      }
      pair_sync(qslot);
    } else {
      if (VS && lane == 0) mbar_init(bar);
      for (uint32_t w = lane; w < vw; w += 32) vis[w] = 0;
      for (uint32_t i = lane; i < D; i += 32) qd[i] = (double)a.q[size_t(b) * D + i];
      __syncwarp();
    }
  } else {
    if (lane == 0) mbar_init(bar);
    // the query element is requested first (it may live in page-locked host
    // memory: a bus round trip), the bitset zeroing runs under it
    const float qe = threadIdx.x < uint32_t(D) ? a.q[size_t(b) * D + threadIdx.x] : 0.f;
    for (uint32_t w = threadIdx.x; w < 2 * vw; w += blockDim.x) vis[w] = 0;
    if (threadIdx.x < uint32_t(D)) qd[threadIdx.x] = (double)qe;
    for (uint32_t i = threadIdx.x + blockDim.x; i < D; i += blockDim.x)
      qd[i] = (double)a.q[size_t(b) * D + i];
    for (uint32_t i = threadIdx.x; i < kSlots; i += blockDim.x)
      slotw[i] = slotword(kSentinel, sFREE);
    if (threadIdx.x < 32) pub_k[threadIdx.x] = 0, pub_id[threadIdx.x] = kSentinel;
    for (uint32_t i = threadIdx.x; i < kFR * 32; i += blockDim.x) pubf_k[i] = 0, pubf_id[i] = kSentinel;
    for (uint32_t i = threadIdx.x; i < kHintN; i += blockDim.x) hint_k[i] = 0, hint_id[i] = kSentinel;
    if (threadIdx.x < 16) ctrl[threadIdx.x] = 0;
    __syncthreads();
  }

  auto masked_id = [&](uint32_t v) -> bool {
    return a.mask_bits != nullptr && ((__ldg(a.mask_bits + (v >> 5)) >> (v & 31)) & 1u);
  };
  auto vbit = [&](const uint32_t* bits, uint32_t v) -> bool {
    return (reinterpret_cast<const volatile uint32_t*>(bits)[v >> 5] >> (v & 31)) & 1u;
  };
  uint32_t phase = 0;
  uint64_t cy_adj = 0, cy_tma = 0, cy_dot = 0;  // adjacency-load / TMA-wait / dot cycles
  // Expansion of node c by this warp: lane l holds adjacency slot l; `isnew`
  // lanes hold an unvisited (at read time), first-occurrence neighbour v and
  // its exact score key. Key rows come through this warp's TMA tile.
  // The mask bit is fetched here too, so its load overlaps the row loads.
  // (adjacency / TMA wait cycles: RA_PIPE_PROFILE builds and the DUO expansion warp)
  constexpr bool kExpCy = kPipeProfile || DUO;
  auto expand = [&](uint32_t c, uint32_t& v, uint64_t& sk, bool& isnew, bool& msk) {
    const uint64_t te0 = kExpCy ? clock64() : 0;
    v = lane < M ? __ldg(adj + size_t(c) * M + lane) : kSentinel;
    const bool valid = v != kSentinel;
    const uint32_t grp = __match_any_sync(kFull, v);
    if (kExpCy) cy_adj += clock64() - te0;
    const bool first = uint32_t(__ffs(grp) - 1) == lane;
    isnew = valid && first && !vbit(vis, v);
    msk = isnew && masked_id(v);
    const uint32_t newmask = __ballot_sync(kFull, isnew);
    sk = 0;
    if constexpr (TP && !VS) {
      // every new row's lines in flight at once (the dot's loads then merge
      // with these misses instead of paying one L2 round trip per few lines)
      if (isnew && !(a.flags & 8192u)) {
        const char* r = BF ? reinterpret_cast<const char*>(keys16 + size_t(v) * D)
                           : reinterpret_cast<const char*>(keys + size_t(v) * D);
#pragma unroll
        for (int l = 0; l < D * (BF ? 2 : 4) / 128; ++l) prefetch_l1(r + 128 * l);
      }
      if (isnew) {
        double acc = 0.0;
        if constexpr (BF) {
          acc = row_dot_bf<D>(qd, reinterpret_cast<const uint4*>(keys16 + size_t(v) * D), true);
        } else {
          const float4* r4 = reinterpret_cast<const float4*>(keys + size_t(v) * D);
#pragma unroll
          for (int c = 0; c < D / 4; ++c) {
            const float4 kk = __ldg(r4 + c);
            acc = fma(qd[4 * c + 0], (double)kk.x, acc);
            acc = fma(qd[4 * c + 1], (double)kk.y, acc);
            acc = fma(qd[4 * c + 2], (double)kk.z, acc);
            acc = fma(qd[4 * c + 3], (double)kk.w, acc);
          }
        }
        sk = okey(acc);
      }
    } else if (newmask) {
      // rows through this warp's tile, lay.MT at a time (one round unless
      // the tile is shorter than the degree: TPS)
      const uint32_t o = __popc(newmask & lanemask_lt(lane)), nn = __popc(newmask);
      if (TP && !BF && nn > lay.MT) {
        // more new rows than tile slots: the tile's rows by TMA and the rest
        // L1-prefetched, all in flight at once, then ONE dot chain for every
        // lane through a generic pointer (tile or global row)
        const bool intile = o < lay.MT;
        float* row = tile + size_t(intile ? o : 0) * RS;
        fence_proxy_async();
        if (lane == 0) mbar_arrive_expect_tx(bar, lay.MT * kRowBytes);
        __syncwarp();
        const float* grow = keys + size_t(v) * D;
        if (isnew && intile) bulk_g2s(row, grow, kRowBytes, bar);
        if (isnew && !intile) {
#pragma unroll
          for (int l = 0; l < D * 4 / 128; ++l) prefetch_l1(reinterpret_cast<const char*>(grow) + 128 * l);
        }
        const uint64_t tw0 = kExpCy ? clock64() : 0;
        mbar_wait(bar, phase);
        if (kExpCy) cy_tma += clock64() - tw0;
        phase ^= 1u;
        const uint64_t td0 = kExpCy ? clock64() : 0;
        if (isnew) sk = okey(row_dot<D>(qd, intile ? static_cast<const float*>(row) : grow));
        __syncwarp();
        if (kExpCy) cy_dot += clock64() - td0;
        return;
      }
      for (uint32_t c0 = 0; c0 < nn; c0 += lay.MT) {
        const uint32_t cnt = nn - c0 < lay.MT ? nn - c0 : lay.MT;
        const bool mine = isnew && o >= c0 && o < c0 + cnt;
        float* row = tile + size_t(o - c0) * RS;
        fence_proxy_async();
        if (lane == 0) mbar_arrive_expect_tx(bar, cnt * kRowBytes);
        __syncwarp();
        if (mine) {
          if constexpr (BF) bulk_g2s(row, keys16 + size_t(v) * D, kRowBytes, bar);
          else bulk_g2s(row, keys + size_t(v) * D, kRowBytes, bar);
        }
        const uint64_t tw0 = kExpCy ? clock64() : 0;
        mbar_wait(bar, phase);
        if (kExpCy) cy_tma += clock64() - tw0;
        phase ^= 1u;
        const uint64_t td0 = kExpCy ? clock64() : 0;
        if (mine) {
          if constexpr (BF) sk = okey(row_dot_bf<D>(qd, reinterpret_cast<const uint4*>(row), false));
          else sk = okey((!TP && (a.flags & 4u)) ? row_dot_seq<D>(qd, row) : row_dot<D>(qd, row));
        }
        __syncwarp();
        if (kExpCy) cy_dot += clock64() - td0;
      }
    }
  };

  if (TP ? !duo_x : warp == 0) {
    // =================== commit warp ===================
    // F: per-lane unsorted lists in shared memory (column layout, entry i of
    // lane l at [i * 32 + l]; empty = (0, kSentinel)); the lane head (its
    // best entry and slot) in registers. Helpers read these lists directly.
    volatile uint64_t* Fl_k = TP ? reinterpret_cast<volatile uint64_t*>(wbase + lay.tp_flist_off())
                                 : pubf_k;
    volatile uint32_t* Fl_i = reinterpret_cast<volatile uint32_t*>(Fl_k + kFR * 32);
    if constexpr (TP) {
#pragma unroll
      for (int i = 0; i < kFR; ++i) Fl_k[i * 32 + lane] = 0, Fl_i[i * 32 + lane] = kSentinel;
    }
    uint64_t hk = 0, uk[kUR];
    uint32_t hi = kSentinel, hpos = 0, uid[kUR];
#pragma unroll
    for (int i = 0; i < kUR; ++i) uk[i] = 0, uid[i] = kSentinel;
    uint32_t fcnt = 0, ufree = (1u << kUR) - 1u;
    uint32_t capFO = lay.capO, capUO = lay.capO, nFO = 0, nUO = 0, pk_fo = 0, pk_uo = 0;
    uint8_t* fo_base = TP ? wbase + size_t(D) * 8 : smem + lay.fo_off();
    Arr FO = Arr::at(fo_base, lay.capO),
        UO = Arr::at(fo_base + PipeLayout::arr_bytes(lay.capO), lay.capO);
    bool fo_g = false, uo_g = false;
    uint64_t fo_k = 0;  // best FO entry (exact)
    uint32_t fo_id = kSentinel, fo_ix = 0;
    uint64_t thr = 0;
    // stop-test pivot: cH = #{u in U : key >= H} < ef means no top >= H can
    // stop the search, so the count is skipped (H = max: no pivot yet)
    uint64_t H = ~0ull;
    uint32_t cH = 0;
    uint64_t u_total = 0, scanned = 0;
    uint32_t nU = 0, expanded = 0, rot = 0;
    uint64_t c_wait = 0, c_hit = 0, c_miss = 0, c_comp = 0, c_fopop = 0, c_fsp = 0, c_usp = 0;
    const uint64_t t_begin = clock64();
    uint64_t cyc_comp = 0;
    const int bis_it = (a.flags >> 28) ? int(a.flags >> 28) * 4 : 8;  // thr bisection steps

    auto fo_rescan = [&]() {
      uint64_t bk = 0;
      uint32_t bi = kSentinel, bx = 0;
#pragma unroll 1
      for (uint32_t i = lane; i < nFO; i += 32)
        if (better(FO.k[i], FO.id[i], bk, bi)) bk = FO.k[i], bi = FO.id[i], bx = i;
      uint64_t wk = bk;
      uint32_t wi = bi;
      warp_best(wk, wi);
      fo_k = wk, fo_id = wi;
      fo_ix = __shfl_sync(kFull, bx, __ffs(__ballot_sync(kFull, bi == wi && bk == wk)) - 1);
    };
    // move an overflow array to its HBM spill region (capacity spill_cap >= n)
    auto to_global = [&](Arr& A, uint32_t cnt, uint8_t* dst) {
      Arr G = Arr::at(dst, spill_cap);
#pragma unroll 1
      for (uint32_t i = lane; i < cnt; i += 32) G.k[i] = A.k[i], G.id[i] = A.id[i];
      __syncwarp();
      A = G;
    };
    auto lane_head = [&]() {  // best entry of this lane's list
      hk = 0, hi = kSentinel, hpos = 0;
#pragma unroll
      for (int i = 0; i < kFR; ++i) {
        if (uint32_t(i) < fcnt) {
          const uint64_t x = Fl_k[i * 32 + lane];
          const uint32_t v = Fl_i[i * 32 + lane];
          if (better(x, v, hk, hi)) hk = x, hi = v, hpos = i;
        }
      }
    };
    // (x, v) into this lane's list (one store, one head compare); a full
    // lane hands the entry to FO, whose best competes with the lane heads
    auto insert_F = [&](bool ok, uint64_t x, uint32_t v) {
      const bool sp = ok && fcnt == uint32_t(kFR);
      const uint64_t sk = x;
      const uint32_t si = v;
      if (ok && !sp) {
        Fl_k[fcnt * 32 + lane] = x;
        Fl_i[fcnt * 32 + lane] = v;
        if (better(x, v, hk, hi)) hk = x, hi = v, hpos = fcnt;
        ++fcnt;
      }
      const uint32_t sm = __ballot_sync(kFull, sp);
      if (sm) {
        ++c_fsp;
        if (nFO + __popc(sm) > capFO) {
          if (fo_g) __trap();  // unreachable: spill_cap >= n
          to_global(FO, nFO, spill_slot);
          capFO = spill_cap, fo_g = true;
        }
        const uint32_t o = nFO + __popc(sm & lanemask_lt(lane));
        if (sp) FO.k[o] = sk, FO.id[o] = si;
        uint64_t bk = sp ? sk : 0;
        uint32_t bi = sp ? si : kSentinel;
        warp_best(bk, bi);
        if (better(bk, bi, fo_k, fo_id)) {
          fo_k = bk, fo_id = bi;
          fo_ix = nFO + __popc(sm & lanemask_lt(__ffs(__ballot_sync(kFull, sp && si == bi)) - 1));
        }
        nFO += __popc(sm);
        if (nFO > pk_fo) pk_fo = nFO;
        __syncwarp();
      }
    };
    auto insert_U = [&](bool ok, uint64_t x, uint32_t v) {
      const bool sp = ok && !ufree;
      if (ok && ufree) {
        const int fi = __ffs(ufree) - 1;
#pragma unroll
        for (int i = 0; i < kUR; ++i)
          if (i == fi) uk[i] = x, uid[i] = v;
        ufree &= ufree - 1;
      }
      nU += __popc(__ballot_sync(kFull, ok));
      cH += __popc(__ballot_sync(kFull, ok && x >= H));
      const uint32_t sm = __ballot_sync(kFull, sp);
      if (sm) {
        ++c_usp;
        if (nUO + __popc(sm) > capUO) {
          if (uo_g) __trap();
          to_global(UO, nUO, spill_slot + PipeLayout::arr_bytes(spill_cap));
          capUO = spill_cap, uo_g = true;
        }
        const uint32_t o = nUO + __popc(sm & lanemask_lt(lane));
        if (sp) UO.k[o] = x, UO.id[o] = v;
        nUO += __popc(sm);
        if (nUO > pk_uo) pk_uo = nUO;
        __syncwarp();
      }
    };
    auto count_gt = [&](uint64_t x) -> uint32_t {  // #{u in U : key > x}
      uint32_t c = 0;
#pragma unroll
      for (int i = 0; i < kUR; ++i) c += uk[i] > x;
#pragma unroll 1
      for (uint32_t i = lane; i < nUO; i += 32) c += UO.k[i] > x;
      return __reduce_add_sync(kFull, c);
    };
    // raise thr toward the pool worst (the ef-th best key of U) by key
    // bisection, then drop F / U entries below it
    auto compact = [&]() {
      ++c_comp;
      uint64_t lo = ~0ull, hi = 0;
#pragma unroll
      for (int i = 0; i < kUR; ++i)
        if (uid[i] != kSentinel) lo = min(lo, uk[i]), hi = max(hi, uk[i]);
#pragma unroll 1
      for (uint32_t i = lane; i < nUO; i += 32) lo = min(lo, UO.k[i]), hi = max(hi, UO.k[i]);
      {  // exact warp min / max of u64
        uint64_t l = lo, h = hi;
#pragma unroll
        for (int o = 16; o; o >>= 1) {
          l = min(l, __shfl_xor_sync(kFull, l, o));
          h = max(h, __shfl_xor_sync(kFull, h, o));
        }
        lo = l, hi = h;
      }
      const uint64_t hmax = hi;
      lo = max(lo, thr);  // count(>= lo) >= ef; find the largest such key
      if (count_gt(hi - 1) >= ef) {
        lo = hi;
      } else {
#pragma unroll 1
        for (int it = 0; it < bis_it && hi - lo > 1; ++it) {
          const uint64_t mid = key_mid(lo, hi);
          if (count_gt(mid - 1) >= ef) lo = mid;
          else hi = mid;
        }
      }
      if (lo <= thr) return;
      thr = lo;
#pragma unroll
      for (int i = 0; i < kUR; ++i)
        if (uid[i] != kSentinel && uk[i] < thr) uk[i] = 0, uid[i] = kSentinel, ufree |= 1u << i;
      {  // drop this lane's list entries below thr (stable squeeze)
        uint32_t w2 = 0;
#pragma unroll
        for (int i = 0; i < kFR; ++i) {
          if (uint32_t(i) < fcnt) {
            const uint64_t x = Fl_k[i * 32 + lane];
            const uint32_t v = Fl_i[i * 32 + lane];
            if (x >= thr) {
              Fl_k[w2 * 32 + lane] = x, Fl_i[w2 * 32 + lane] = v;
              ++w2;
            }
          }
        }
#pragma unroll
        for (int i = 0; i < kFR; ++i)
          if (uint32_t(i) >= w2 && uint32_t(i) < fcnt)
            Fl_k[i * 32 + lane] = 0, Fl_i[i * 32 + lane] = kSentinel;
        fcnt = w2;
        lane_head();
      }
      auto squeeze = [&](Arr& A, uint32_t& cnt) {
        uint32_t w = 0;
#pragma unroll 1
        for (uint32_t c0 = 0; c0 < cnt; c0 += 32) {
          const uint32_t i = c0 + lane;
          const bool in = i < cnt;
          const uint64_t x = in ? A.k[i] : 0;
          const uint32_t id = in ? A.id[i] : 0;
          const bool kp = in && x >= thr;
          const uint32_t bm = __ballot_sync(kFull, kp);
          __syncwarp();
          if (kp) {
            const uint32_t o = w + __popc(bm & lanemask_lt(lane));
            A.k[o] = x, A.id[o] = id;
          }
          w += __popc(bm);
          __syncwarp();
        }
        cnt = w;
      };
      if (nUO) squeeze(UO, nUO);
      if (nFO) {
        squeeze(FO, nFO);
        fo_rescan();
      }
      nU = __reduce_add_sync(kFull, uint32_t(kUR) - __popc(ufree)) + nUO;
      // pivot: the largest key with >= ef - 48 entries at or above it
      // (bisection between thr and the U max), then its exact count; the
      // slack is how many inserts above it the pivot survives (48 measured
      // best of 24 / 32 / 48 / 64)
      const uint32_t pslack = (a.flags >> 23) & 15u ? ((a.flags >> 23) & 15u) * 8u : 48u;
      if (ef > pslack) {
        uint64_t plo = thr, phi = hmax;
        const uint32_t target = ef - pslack;
        if (count_gt(phi - 1) >= target) {
          plo = phi;
        } else {
#pragma unroll 1
          for (int it = 0; it < bis_it && phi - plo > 1; ++it) {
            const uint64_t mid = key_mid(plo, phi);
            if (count_gt(mid - 1) >= target) plo = mid;
            else phi = mid;
          }
        }
        H = plo;
        cH = count_gt(H - 1);
        if (cH >= ef) H = ~0ull;
      }
    };
    // visit lane-held candidates in commit order (:393-399)
    // pre: candidates from this warp's own expansion were filtered against
    // the visited set with nothing committed since, so the re-check is moot
    auto visit = [&](bool cand, uint64_t x, uint32_t v, bool msk, bool pre) {
      const bool isnew = cand && (pre || !((vis[v >> 5] >> (v & 31)) & 1u));
      if (isnew) atomicOr(vis + (v >> 5), 1u << (v & 31));
      const uint32_t nm = __ballot_sync(kFull, isnew);
      scanned += __popc(nm);
      u_total += __popc(__ballot_sync(kFull, isnew && !msk));
      const bool inF = isnew && x >= thr;
      insert_F(inF, x, v);
      insert_U(inF && !msk, x, v);
      if (u_total >= ef && nU >= ef + kSlackU) {
        const uint64_t t0 = clock64();
        compact();
        cyc_comp += clock64() - t0;
      }
    };

    // ---- entry (:379-384), then the loop; every visit goes through ONE
    // call site (the commit path must stay small in the i-cache) ----
    bool cand;
    uint64_t cx;
    uint32_t cv;
    bool cm, pre = true;  // the entry is unvisited
    {
      const uint32_t entry = uint32_t(g.entry);
      cx = 0;
      if constexpr (TP) {
        if (lane == 0) {
          const float4* r4 = reinterpret_cast<const float4*>(keys + size_t(entry) * D);
          double acc = 0.0;
#pragma unroll
          for (int c = 0; c < D / 4; ++c) {
            const float4 kk = __ldg(r4 + c);
            acc = fma(qd[4 * c + 0], (double)kk.x, acc);
            acc = fma(qd[4 * c + 1], (double)kk.y, acc);
            acc = fma(qd[4 * c + 2], (double)kk.z, acc);
            acc = fma(qd[4 * c + 3], (double)kk.w, acc);
          }
          cx = okey(acc);
        }
      } else {
        if (lane == 0) {
          fence_proxy_async();
          mbar_arrive_expect_tx(bar, uint32_t(D) * 4u);
          bulk_g2s(tile, keys + size_t(entry) * D, uint32_t(D) * 4u, bar);
        }
        __syncwarp();
        mbar_wait(bar, phase);
        phase ^= 1u;
        if (lane == 0) cx = okey(row_dot<D>(qd, tile));
      }
      cand = lane == 0;
      cv = entry;
      cm = masked_id(entry);
    }
    // DUO: this warp starts each expansion - the node's adjacency row and
    // the new-neighbour filter (against its visited bits as they are: the
    // neighbours it is about to visit are dropped again at commit time),
    // then per-lane L2 prefetches of the new key rows and of their own
    // adjacency rows (vector prefetches: the bulk forms issue lane by lane)
    // - and posts it; the expansion warp runs the dot chains on those rows
    // and returns the packet while this warp visits the previous one.
    uint32_t dseq = 0;
    uint32_t spec_v = kSentinel;  // DUO: this lane's neighbour of the speculated top
    uint32_t spec_node = kSentinel, spec_row = kSentinel;  // (its id and adjacency entry)
    auto duo_issue = [&](uint32_t p) {
      ++dseq;
      if (p != kSentinel) {
        const uint64_t ti0 = clock64();
        // the speculated runner-up's adjacency row is already in registers
        const uint32_t v = p == spec_node ? spec_row
                                          : lane < M ? __ldg(adj + size_t(p) * M + lane) : kSentinel;
        const uint32_t grp = __match_any_sync(kFull, v);
        c_usp += clock64() - ti0;  // (dbg: the adjacency-row wait)
        const bool isnew = v != kSentinel && uint32_t(__ffs(grp) - 1) == lane &&
                           !((vis[v >> 5] >> (v & 31)) & 1u);
        if (isnew) {
          const char* r = reinterpret_cast<const char*>(keys + size_t(v) * D);
#pragma unroll
          for (int l = 0; l < D * 4 / 128; ++l) prefetch_l2(r + 128 * l);
        }
        const uint32_t nm = __ballot_sync(kFull, isnew);
        duo_rv[lane] = v;
        if (lane == 0) duo_rf[0] = nm;
        __syncwarp();
        if (lane == 0) {
          __threadfence_block();
          *duo_req = (uint64_t(dseq) << 32) | p;
        }
        // (the best new neighbour is likely a top soon: its adjacency row,
        // the first load of its issue, to L2 now)
        if (isnew && !(a.flags & 2u))  // (the row's first line; a straddling tail comes with the load)
          prefetch_l2(adj + size_t(v) * M);
        c_fsp += clock64() - ti0;  // (dbg: the whole issue)
      } else if (lane == 0) {
        __threadfence_block();
        *duo_req = (uint64_t(dseq) << 32) | p;
      }
    };
    if constexpr (DUO) duo_issue(g.entry);  // the entry is the first top

    // The next top is known before the visit: the best of this expansion's
    // new children >= thr and the frontier after the pop (the visit only
    // inserts those children; a compaction can only end the search). Found
    // early (one argmax over per-lane bests and FO's best), it steers the
    // work that would otherwise wait for the loop top: DUO posts it to the
    // expansion warp, latency mode takes its packet now or hints it.
    bool have_next = false, early_took = false;
    uint64_t nk = 0, w_n = 0;
    uint32_t nid = kSentinel, sl_n = 0;
    auto next_top = [&](bool inf, uint64_t x, uint32_t v) {
      uint64_t k0 = hk;
      uint32_t i0 = hi;
      if (inf && better(x, v, k0, i0)) k0 = x, i0 = v;
      warp_best(k0, i0);
      if (nFO && better(fo_k, fo_id, k0, i0)) k0 = fo_k, i0 = fo_id;
      nk = k0, nid = i0, have_next = true;
    };
    // latency mode: take the next top's packet now if ready, else hint it
    // when no helper holds it (its expansion overlaps the visit)
    auto early_lookup = [&]() {
      early_took = false;
      if constexpr (!TP) {
        if (nid == kSentinel) return;
        sl_n = slot_of(nid);
        w_n = *reinterpret_cast<volatile unsigned long long*>(slotw + sl_n);
        const uint64_t w1 = *reinterpret_cast<volatile unsigned long long*>(slotw + sl_n + 1);
        if (uint32_t(w_n) != nid && uint32_t(w1) == nid) w_n = w1, ++sl_n;
        bool t = false;
        if (lane == 0) {
          if (uint32_t(w_n) == nid && uint32_t(w_n >> 32) == sREADY)
            t = atomicCAS(slotw + sl_n, slotword(nid, sREADY), slotword(nid, sTAKEN)) ==
                slotword(nid, sREADY);
          else if (uint32_t(w_n) != nid && !(a.flags & 8u))
            push_hint(nk, nid);
        }
        early_took = __shfl_sync(kFull, t, 0);
      }
    };

    uint64_t cy[5] = {0, 0, 0, 0, 0};
    uint64_t tq = clock64();
    for (;;) {
      visit(cand, cx, cv, cm, pre);
      PIPE_TICK(3)
      if constexpr (DUO) {  // the speculative prefetch (see below), after the visit
        if (spec_v != kSentinel && !((vis[spec_v >> 5] >> (spec_v & 31)) & 1u)) {
          const char* r = reinterpret_cast<const char*>(keys + size_t(spec_v) * D);
#pragma unroll
          for (int l = 0; l < D * 4 / 128; ++l) prefetch_l2(r + 128 * l);
        }
        spec_v = kSentinel;
      }
      // frontier top (:387): lane heads vs the best overflow entry
      uint64_t tk;
      uint32_t tid;
      bool from_fo;
      if (have_next) {  // (p sits in FO iff FO's best is p: ids are unique)
        tk = nk, tid = nid, have_next = false;
        from_fo = nFO && fo_id == tid;
      } else {
        tk = hk, tid = hi;
        warp_best(tk, tid);
        from_fo = nFO && better(fo_k, fo_id, tk, tid);
        if (from_fo) tk = fo_k, tid = fo_id;
      }
      if (tid == kSentinel) break;  // frontier exhausted
      if (u_total >= ef) {          // :390
        if (tk < thr) break;
        if (!(tk >= H && cH < ef) && count_gt(tk) >= ef) break;
      }
      PIPE_TICK(0)
      // the top's packet: look it up and take a ready one (READY -> TAKEN)
      // BEFORE the pop, which it does not depend on, so the pop's shuffles
      // run in the shadow of the loads and the CAS; an in-flight packet is
      // awaited after the pop
      uint32_t sl = 0;
      uint64_t w = 0;
      bool took = false;
      if (!TP && early_took) {
        sl = sl_n, w = w_n, took = lane == 0, early_took = false;
      } else if constexpr (!TP) {
        sl = slot_of(tid);
        w = *reinterpret_cast<volatile unsigned long long*>(slotw + sl);
        const uint64_t w1 = *reinterpret_cast<volatile unsigned long long*>(slotw + sl + 1);
        if (uint32_t(w) != tid && uint32_t(w1) == tid) w = w1, ++sl;
        if (lane == 0 && uint32_t(w) == tid && uint32_t(w >> 32) == sREADY)
          took = atomicCAS(slotw + sl, slotword(tid, sREADY), slotword(tid, sTAKEN)) ==
                 slotword(tid, sREADY);
      }
      // pop (:391)
      if (from_fo) {
        ++c_fopop;
        if (lane == 0) {
          --nFO;
          FO.k[fo_ix] = FO.k[nFO], FO.id[fo_ix] = FO.id[nFO];
        }
        nFO = __shfl_sync(kFull, nFO, 0);
        __syncwarp();
        fo_rescan();
      } else {
        // the owner's new head: kFR lanes read its other entries (one each,
        // from the list as it was) and 3 REDUX pick the best; meanwhile the
        // owner lane's last entry fills the hole (its stores follow the
        // loads in program order)
        const uint32_t owner = __ffs(__ballot_sync(kFull, hi == tid)) - 1;
        const uint32_t fc0 = __shfl_sync(kFull, fcnt, owner);
        const uint32_t hp = __shfl_sync(kFull, hpos, owner);
        uint64_t x = 0;
        uint32_t v = kSentinel;
        if (lane < uint32_t(kFR)) x = Fl_k[lane * 32 + owner], v = Fl_i[lane * 32 + owner];
        const bool live = lane < fc0 && lane != hp;
        if (!live) x = 0, v = kSentinel;
        if (lane == owner) {
          --fcnt;
          if (hpos != fcnt) {
            Fl_k[hpos * 32 + lane] = Fl_k[fcnt * 32 + lane];
            Fl_i[hpos * 32 + lane] = Fl_i[fcnt * 32 + lane];
          }
          Fl_k[fcnt * 32 + lane] = 0, Fl_i[fcnt * 32 + lane] = kSentinel;
        }
        const uint32_t mine = v;
        warp_best(x, v);
        const uint32_t pos = __ffs(__ballot_sync(kFull, live && mine == v)) - 1;
        // (the old last entry now sits in the hole)
        if (lane == owner) hk = x, hi = v, hpos = fcnt ? (pos == fcnt ? hp : pos) : 0;
      }
      ++expanded;
      PIPE_TICK(1)
      if constexpr (TP) {
        ++c_miss;
        if constexpr (DUO) {
          // tid's packet (requested when tid was found to be the next top)
          if (*duo_rdy != dseq) {
            const uint64_t tw0 = clock64();
            while (*duo_rdy != dseq) {
            }
            c_wait += clock64() - tw0;
          }
          __threadfence_block();
          const uint32_t nm = duo_flags[0], mm = duo_flags[1];
          cv = duo_pi[lane];
          cx = duo_pk[lane];
          // exact filter now (only this warp writes the visited bits), so
          // visit() need not re-check
          cand = ((nm >> lane) & 1u) && !((vis[cv >> 5] >> (cv & 31)) & 1u);
          cm = (mm >> lane) & 1u;
          // the next top is known before the visit: the best new child >= thr
          // vs the frontier's best (compaction can only end the search), so
          // the expansion warp starts on it while this warp does the visit
          next_top(cand && cx >= thr, cx, cv);
          duo_issue(nid);
          if (!(a.flags & (1u << 27))) {
            // speculation two links ahead: the runner-up (the best of the
            // frontier and these children other than nid) is the top after
            // nid unless one of nid's children beats it; its adjacency row
            // (an L2 hit: prefetched when it was found) is requested now and
            // its new neighbours' key rows are prefetched after the visit
            const bool inf2 = cand && cx >= thr && cv != nid;
            uint64_t k2 = hi != nid ? hk : 0;
            uint32_t i2 = hi != nid ? hi : kSentinel;
            if (inf2 && better(cx, cv, k2, i2)) k2 = cx, i2 = cv;
            warp_best(k2, i2);
            if (nFO && fo_id != nid && better(fo_k, fo_id, k2, i2)) i2 = fo_id;
            spec_v = (i2 != kSentinel && lane < M) ? __ldg(adj + size_t(i2) * M + lane)
                                                   : 0xFFFFFFFFu;
            spec_node = i2, spec_row = spec_v;
          }
        } else {
          expand(tid, cv, cx, cand, cm);
        }
        pre = true;
        PIPE_TICK(2)
        if constexpr (VS && !DUO) {  // the new frontier nodes' adjacency rows go to L2 now
          if ((M * 4) % 16 == 0 && !(a.flags & 2u) && cand && cx >= thr)
            bulk_prefetch_l2(adj + size_t(cv) * M, M * 4);
        }
        continue;
      }
      // hit (taken above, or in flight: wait, then take) or expand inline
      bool hit = __shfl_sync(kFull, took, 0);
      if (!hit && uint32_t(w) == tid && uint32_t(w >> 32) == sBUSY) {
        const uint64_t tw0 = clock64();
        do {
          __nanosleep(20);
          w = *reinterpret_cast<volatile unsigned long long*>(slotw + sl);
        } while (uint32_t(w >> 32) == sBUSY && uint32_t(w) == tid);
        c_wait += clock64() - tw0;
        if (lane == 0 && uint32_t(w) == tid && uint32_t(w >> 32) == sREADY)
          took = atomicCAS(slotw + sl, slotword(tid, sREADY), slotword(tid, sTAKEN)) ==
                 slotword(tid, sREADY);
        hit = __shfl_sync(kFull, took, 0);
      }
      // expanded bit after the take: helpers may evict packets of expanded nodes
      if (lane == 0) atomicOr(expd + (tid >> 5), 1u << (tid & 31));
      PIPE_TICK(2)
      if (hit) {
        ++c_hit;
        __threadfence_block();
        const uint32_t j = (lane + rot) & 31u;
        // all four loads at once (the entry loads do not wait for the count)
        const uint32_t cnt = pk_cnt[sl], mb = pk_mb[sl];
        const uint32_t pv = pk_id[sl * 32 + j];
        const uint64_t px = pk_k[sl * 32 + j];
        cand = j < cnt;
        cv = cand ? pv : kSentinel;
        cx = cand ? px : 0;
        cm = cand && ((mb >> j) & 1u);
        __syncwarp();
        if (lane == 0) st_release_cta(slotw + sl, slotword(kSentinel, sFREE));
        rot += cnt;
        // other packets may have visited these since: the exact filter now
        // (only this warp writes the visited bits), then the next top
        cand = cand && !((vis[cv >> 5] >> (cv & 31)) & 1u);
        pre = true;
        if (a.flags & 262144u) {
          next_top(cand && cx >= thr, cx, cv);
          early_lookup();
        }
      } else {
        ++c_miss;
#ifdef RA_PIPE_MISSCLASS
        // 1: a child of the node just visited from a packet, 2: a child of an
        // inline expansion (miss chain), 3: older
        if (__any_sync(kFull, cand && cv == tid)) cy[4] += pre ? (1ull << 20) : 1ull;
        else cy[4] += 1ull << 40;
#endif
        expand(tid, cv, cx, cand, cm);
        pre = true;
        if (a.flags & 262144u) {
          next_top(cand && cx >= thr, cx, cv);
          early_lookup();
        }
        if (!(a.flags & (8u | 32768u))) {
          // the likely next tops are this node's best children, which no
          // helper has seen: hint the best two so helpers start on them now
          uint64_t k1 = cand ? cx : 0;
          uint32_t i1 = cand ? cv : kSentinel;
          warp_best(k1, i1);
          uint64_t k2 = (cand && cv != i1) ? cx : 0;
          uint32_t i2 = (cand && cv != i1) ? cv : kSentinel;
          warp_best(k2, i2);
          if (lane == 0) {
            if (i1 != kSentinel) push_hint(k1, i1);
            if (i2 != kSentinel) push_hint(k2, i2);
          }
        }
      }
    }
    if constexpr (DUO) {  // stop the expansion warp; its tile is free after the barrier
      if (lane == 0) *duo_req = (uint64_t(dseq + 1) << 32) | kSentinel;
      pair_sync(qslot);
      c_hit = duo_pk[0];  // its busy / dot cycles (dbg); c_fsp / c_usp: this warp's issue / adjacency wait
      cy_dot = duo_pk[3];
    }
    // ---- result (:402-410): the pool's top min(k, |pool|), best-first ----
    uint32_t p2 = 32;
    while (p2 < nU) p2 <<= 1;
    bool fin_smem;
    uint8_t* fin_base = TP ? fo_base : smem + lay.tiles_off();
    if constexpr (TP) {
      if (VS && !DUO) {  // this warp's (dead) row tile (DUO has none)
        fin_smem = PipeLayout::arr_bytes(p2) <= lay.tile_bytes();
        fin_base = wbase + lay.tp_tile_off();
      } else {
        fin_smem = p2 <= lay.capO;  // this warp's (dead) FO region
      }
    } else {
      ctrl[0] = 1;  // helpers stop
      __syncwarp();
      // (fused attention: leave room for >= 8 staged V rows behind the array)
      fin_smem = PipeLayout::arr_bytes(p2) + 16 +
                     (a.fa.out ? (40 + 32 * (size_t(D) + 2)) * 8 + 8 * (size_t(D) * 4 + 8)
                                      : 0) <=
                 size_t(kPW) * lay.tile_bytes();
      if (lane == 0) {
        ctrl[4] = p2;
        ctrl[5] = fin_smem;
      }
      __syncthreads();  // helpers are done with their tiles (and TMA)
    }
    // A: shared memory when it fits, else FO's (dead) half of the HBM slot
    Arr A = fin_smem ? Arr::at(fin_base, p2) : Arr::at(spill_slot, p2);
    uint32_t w = 0;
#pragma unroll
    for (int i = 0; i < kUR; ++i) {
      const bool kp = uid[i] != kSentinel;
      const uint32_t bm = __ballot_sync(kFull, kp);
      if (kp) {
        const uint32_t o = w + __popc(bm & lanemask_lt(lane));
        A.k[o] = uk[i], A.id[o] = uid[i];
      }
      w += __popc(bm);
    }
    for (uint32_t i = lane; i < nUO; i += 32) A.k[w + i] = UO.k[i], A.id[w + i] = UO.id[i];
    w += nUO;
    for (uint32_t i = w + lane; i < p2; i += 32) A.k[i] = 0, A.id[i] = kSentinel;
    if (a.dbg && lane == 0) {
      uint64_t* d = a.dbg + size_t(b) * 12;
      d[0] = c_miss, d[1] = c_wait, d[2] = clock64() - t_begin, d[3] = expanded;
      d[4] = c_hit, d[5] = TP ? 0 : ctrl[8], d[6] = c_comp;
      d[7] = cy[0], d[8] = cy[1], d[9] = cy[2], d[10] = cy[3], d[11] = cyc_comp;
#ifndef RA_PIPE_PROFILE
      if (TP) {  // overflow anatomy: FO / UO spill rounds, FO pops, moved to HBM
        d[7] = c_fsp, d[8] = c_fopop, d[9] = (fo_g ? 1u : 0u) | (uo_g ? 2u : 0u), d[10] = c_usp;
        if (DUO) d[9] = cy_dot;
        d[5] = pk_fo, d[11] = pk_uo;  // peak overflow sizes
      }
#else
      if (TP) d[5] = cy_adj, d[11] = cy_tma;
#endif
#ifdef RA_PIPE_MISSCLASS
      d[9] = cy[4];
#endif
      (void)c_comp, (void)c_fopop, (void)c_fsp, (void)c_usp;
    }
    const uint32_t pool = uint32_t(u_total < ef ? u_total : ef);
    if (lane == 0) {
      a.scanned[b] = scanned;
      if (a.scanned_own) a.scanned_own[b] = scanned;
      if (a.expanded) a.expanded[b] = expanded;
    }
    if constexpr (TP) {
      __syncwarp();
      if (p2 <= 256) {  // (A in shared memory or in the HBM slot)
        // pool in registers (element lane * 8 + i), warp bitonic sort
        uint64_t sk8[8];
        uint32_t si8[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const uint32_t e = lane * 8 + i;
          sk8[i] = e < p2 ? A.k[e] : 0;
          si8[i] = e < p2 ? A.id[e] : kSentinel;
        }
        warp_sort256(sk8, si8, lane);
        const uint32_t take = pool < k ? pool : k;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const uint32_t r = lane * 8 + i;
          if (r < k) {
            const bool have = r < take;
            const double sc = have ? okey_inv(sk8[i]) : __longlong_as_double(0x7ff8000000000000ll);
            a.ids[size_t(b) * k + r] = have ? si8[i] : kSentinel;
            a.scores[size_t(b) * k + r] = have ? (float)sc : __int_as_float(0x7fc00000);
            if (a.scores64) a.scores64[size_t(b) * k + r] = sc;
          }
        }
        for (uint32_t r = 256 + lane; r < k; r += 32) {  // k beyond the pool
          a.ids[size_t(b) * k + r] = kSentinel;
          a.scores[size_t(b) * k + r] = __int_as_float(0x7fc00000);
          if (a.scores64) a.scores64[size_t(b) * k + r] = __longlong_as_double(0x7ff8000000000000ll);
        }
        if (lane == 0) {
          a.n_out[b] = take;
          a.truncated[b] = take < k;
        }
        return;
      }
      for (uint32_t kk = 2; kk <= p2; kk <<= 1) {
        for (uint32_t j = kk >> 1; j > 0; j >>= 1) {
          for (uint32_t i = lane; i < p2; i += 32) {
            const uint32_t pj = i ^ j;
            if (pj > i) {
              const bool desc = (i & kk) == 0;
              const uint64_t xi = A.k[i], xp = A.k[pj];
              const uint32_t ii = A.id[i], ip = A.id[pj];
              if (desc ? better(xp, ip, xi, ii) : better(xi, ii, xp, ip)) {
                A.k[i] = xp, A.k[pj] = xi;
                A.id[i] = ip, A.id[pj] = ii;
              }
            }
          }
          __syncwarp();
        }
      }
      const uint32_t take = pool < k ? pool : k;
      for (uint32_t r = lane; r < k; r += 32) {
        const bool have = r < take;
        const double s = have ? okey_inv(A.k[r]) : __longlong_as_double(0x7ff8000000000000ll);
        a.ids[size_t(b) * k + r] = have ? A.id[r] : kSentinel;
        a.scores[size_t(b) * k + r] = have ? (float)s : __int_as_float(0x7fc00000);
        if (a.scores64) a.scores64[size_t(b) * k + r] = s;
      }
      if (lane == 0) {
        a.n_out[b] = take;
        a.truncated[b] = take < k;
      }
      return;
    } else {
      if (lane == 0) ctrl[7] = pool;
      __syncthreads();
    }
  } else if constexpr (DUO) {
    // =================== DUO expansion warp ===================
    // expands exactly the nodes the commit warp posts (each is the next top
    // or the search is over), so its expansion overlaps the commit warp's
    // visit of the previous packet; filtering against the visited bits here
    // is a hint (the commit warp re-filters)
    uint64_t busy = 0;
    for (uint32_t hseq = 1;; ++hseq) {
      uint64_t w;
      do {
        w = *duo_req;
      } while (uint32_t(w >> 32) != hseq);
      const uint32_t p = uint32_t(w);
      if (p == kSentinel) break;
      const uint64_t tb0 = clock64();
      __threadfence_block();
      const uint32_t v = duo_rv[lane], nm = duo_rf[0];
      const bool isnew = (nm >> lane) & 1u;
      // the static-set bit is requested now and used after the chain
      const uint32_t mw = (isnew && a.mask_bits) ? __ldg(a.mask_bits + (v >> 5)) : 0u;
      const uint64_t td0 = clock64();
      uint64_t sk = 0;
      if (isnew) sk = okey(row_dot<D>(qd, keys + size_t(v) * D));  // (rows L2-prefetched)
      const uint32_t mm = __ballot_sync(kFull, isnew && ((mw >> (v & 31)) & 1u));  // (W: not a pool entry)
      cy_dot += clock64() - td0;
      duo_pk[lane] = sk;
      duo_pi[lane] = v;
      if (lane == 0) duo_flags[0] = nm, duo_flags[1] = mm;
      __syncwarp();
      if (lane == 0) {
        __threadfence_block();
        *duo_rdy = hseq;
      }
      busy += clock64() - tb0;
    }
    if (lane == 0) duo_pk[0] = busy, duo_pk[1] = cy_adj, duo_pk[2] = cy_tma, duo_pk[3] = cy_dot;
    pair_sync(qslot);
    return;
  } else if constexpr (!TP) {
    // =================== helper warps ===================
    uint32_t n_exp = 0, n_chain = 0, n_evict = 0;
    if (a.flags & 1u) ctrl[0] = 1;  // profiling: commit warp alone
    const uint32_t chain_max = (a.flags >> 4) & 15u ? (a.flags >> 4) & 15u : kChain;
    const uint32_t pick = (a.flags >> 8) & 31u ? (a.flags >> 8) & 31u : kPick;
    // claim node id's slot: free, or evict a ready packet of a node that is
    // expanded already or ranks below x
    auto try_claim = [&](uint32_t id, uint64_t x, uint32_t& sl) -> bool {
      bool ok = false;
      const uint32_t s0 = slot_of(id);
      sl = s0;
      if (lane == 0) {
        const uint64_t w0 = *reinterpret_cast<volatile unsigned long long*>(slotw + s0);
        const uint64_t w1 = *reinterpret_cast<volatile unsigned long long*>(slotw + s0 + 1);
        if (uint32_t(w0) != id && uint32_t(w1) != id) {
          // a free way first, else the way whose ready packet may be evicted
          // (node expanded already, or ranking below x; the lower rank goes)
          auto rank = [&](uint64_t w, uint32_t s) -> uint64_t {  // 0: unusable
            const uint32_t st = uint32_t(w >> 32);
            if (st == sFREE) return ~0ull;
            if (st != sREADY) return 0;
            if (vbit(expd, uint32_t(w))) return ~0ull - 1;
            const uint64_t nk = pk_nk[s];
            return nk < x ? ~nk : 0;
          };
          const uint64_t r0 = rank(w0, s0), r1 = rank(w1, s0 + 1);
          if (r0 | r1) {
            const bool second = r1 > r0;
            const uint64_t w = second ? w1 : w0;
            sl = s0 + second;
            ok = atomicCAS(slotw + sl, w, slotword(id, sBUSY)) == w;
            n_evict += ok && uint32_t(w >> 32) != sFREE;
          }
        }
        if (ok) pk_nk[sl] = x;
      }
      sl = __shfl_sync(kFull, sl, 0);
      return __shfl_sync(kFull, ok, 0);
    };
    // fused attention: one chunk of W (the tile's MT rows) -> its partial
    // (sum e*v, max, sum e) in the head's scratch row, in W order
    // (bf16 groups: the W rows come from the f32 copy, which holds the same
    // rounded values)
    const bool fused = a.fa.out != nullptr;
    auto wchunk = [&](uint32_t c) {
      const uint32_t r0 = c * a.fa.crows, rows = min(a.fa.crows, a.fa.nW - r0);
      const float* V = a.fa.values[b];
      const uint32_t wid = lane < rows ? a.fa.W[r0 + lane] : 0u;
      fence_proxy_async();
      if (lane == 0) mbar_arrive_expect_tx(bar, rows * uint32_t(D) * 4u);
      __syncwarp();
      if (lane < rows) bulk_g2s(tile + size_t(lane) * RS, keys + size_t(wid) * D, D * 4u, bar);
      mbar_wait(bar, phase);
      phase ^= 1u;
      const double z = lane < rows ? row_dot<D>(qd, tile + size_t(lane) * RS) * a.fa.inv_sqrt_d
                                   : -DBL_MAX;
      double m = z;
#pragma unroll
      for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(kFull, m, o));
      const double e = lane < rows ? exp(z - m) : 0.0;
      __syncwarp();  // every lane is done with the key rows
      fence_proxy_async();
      if (lane == 0) mbar_arrive_expect_tx(bar, rows * uint32_t(D) * 4u);
      __syncwarp();
      if (lane < rows) bulk_g2s(tile + size_t(lane) * RS, V + size_t(wid) * D, D * 4u, bar);
      mbar_wait(bar, phase);
      phase ^= 1u;
      constexpr int kJ = (D + 31) / 32;
      double acc[kJ];
#pragma unroll
      for (int t = 0; t < kJ; ++t) acc[t] = 0.0;
      double se = 0.0;
      for (uint32_t i = 0; i < rows; ++i) {  // W order (partial_attention, attention.cpp:102-128)
        const double ei = __shfl_sync(kFull, e, i);
        se += ei;
#pragma unroll
        for (int t = 0; t < kJ; ++t)
          if (lane + 32 * t < uint32_t(D))
            acc[t] = fma(ei, (double)tile[size_t(i) * RS + lane + 32 * t], acc[t]);
      }
      double* dst = a.fa.chunk + (size_t(b) * a.fa.nchunk + c) * (D + 2);
#pragma unroll
      for (int t = 0; t < kJ; ++t)
        if (lane + 32 * t < uint32_t(D)) dst[lane + 32 * t] = acc[t];
      if (lane == 0) dst[D] = m, dst[D + 1] = se;
      __syncwarp();
    };
    auto next_chunk = [&]() -> uint32_t {
      uint32_t c = 0;
      if (lane == 0) c = atomicAdd(const_cast<uint32_t*>(ctrl) + 13, 1u);
      return __shfl_sync(kFull, c, 0);
    };
    // the helper on the commit warp's scheduler (SMSP = warp % 4) does not
    // pre-expand: its issue slots would be taken from the serial commit path
    // (-2.5% search time measured); it takes W attention chunks or sleeps
    const bool quiet = !(a.flags & 4194304u) && (warp % 4u) == 0u;
    for (;;) {
      if (ctrl[0]) break;
      if (quiet) {
        if (fused && ctrl[13] < a.fa.nchunk) {
          const uint32_t c = next_chunk();
          if (c < a.fa.nchunk) wchunk(c);
        } else {
          __nanosleep(1000);
        }
        continue;
      }
      // the frontier's best `pick` nodes, best first: a tournament over the
      // published per-lane sorted columns (winner lane advances)
      uint64_t ck[kFR];
      uint32_t ci[kFR];
#pragma unroll
      for (int i = 0; i < kFR; ++i) {
        ck[i] = pubf_k[i * 32 + lane];
        ci[i] = pubf_id[i * 32 + lane];
        if (ci[i] >= n) ck[i] = 0, ci[i] = kSentinel;
      }
      // the commit warp's lists are unsorted: odd-even transposition sort
#pragma unroll
      for (int r = 0; r < kFR; ++r) {
#pragma unroll
        for (int i = r & 1; i + 1 < kFR; i += 2) {
          if (better(ck[i + 1], ci[i + 1], ck[i], ci[i])) {
            const uint64_t tk2 = ck[i];
            const uint32_t ti2 = ci[i];
            ck[i] = ck[i + 1], ci[i] = ci[i + 1];
            ck[i + 1] = tk2, ci[i + 1] = ti2;
          }
        }
      }
      auto claimable = [&](uint32_t id) -> bool {
        if (id >= n || vbit(expd, id)) return false;
        const uint32_t s0 = slot_of(id);
        const uint64_t w0 = *reinterpret_cast<volatile unsigned long long*>(slotw + s0);
        const uint64_t w1 = *reinterpret_cast<volatile unsigned long long*>(slotw + s0 + 1);
        return uint32_t(w0) != id && uint32_t(w1) != id;  // not in flight / ready already
      };
      // best claimable hint (kHintN / 32 per lane)
      uint64_t hx = 0;
      uint32_t hid = kSentinel;
      if (!(a.flags & 8u)) {
#pragma unroll
        for (uint32_t t = 0; t < kHintN / 32; ++t) {
          const uint64_t k2 = hint_k[t * 32 + lane];
          const uint32_t i2 = hint_id[t * 32 + lane];
          if (i2 != kSentinel && better(k2, i2, hx, hid) && claimable(i2)) hx = k2, hid = i2;
        }
      }
      warp_best(hx, hid);
      uint32_t got = kSentinel, sl = 0;
      uint64_t gk = 0;
      for (uint32_t r = 0; r < pick; ++r) {
        uint64_t x = ck[0];
        uint32_t id = ci[0];
        warp_best(x, id);
        if (hid != kSentinel && !better(x, id, hx, hid)) {  // the hint ranks first
          if (try_claim(hid, hx, sl)) {
            got = hid, gk = hx;
            break;
          }
          hid = kSentinel, hx = 0;
        }
        if (id == kSentinel) break;
        if (ci[0] == id) {  // winner lane advances
#pragma unroll
          for (int i = 0; i < kFR - 1; ++i) ck[i] = ck[i + 1], ci[i] = ci[i + 1];
          ck[kFR - 1] = 0, ci[kFR - 1] = kSentinel;
        }
        if (!claimable(id)) continue;
        if (try_claim(id, x, sl)) {
          got = id, gk = x;
          break;
        }
      }
      if (got == kSentinel) {
        // idle: a chunk of W attention (by the last helpers only, so the
        // others stay responsive to hints)
        if (fused && ctrl[13] < a.fa.nchunk &&
            warp + ((a.flags >> 19) & 7u ? (a.flags >> 19) & 7u : kPW) >= kPW) {
          const uint32_t c = next_chunk();
          if (c < a.fa.nchunk) wchunk(c);
          continue;
        }
        __nanosleep(64);
        continue;
      }
      for (uint32_t depth = 0;; ++depth) {
        uint32_t v;
        uint64_t x;
        bool isnew;
        bool msk;
        expand(got, v, x, isnew, msk);
        ++n_exp;
        const uint32_t newmask = __ballot_sync(kFull, isnew);
        const uint32_t o = __popc(newmask & lanemask_lt(lane));
        if (isnew) {
          pk_id[sl * 32 + o] = v;
          pk_k[sl * 32 + o] = x;
          // likely future tops: their adjacency rows go to L2 now
          if ((M * 4) % 16 == 0 && !(a.flags & 2u)) bulk_prefetch_l2(adj + size_t(v) * M, M * 4);
        }
        const uint32_t mb = __reduce_or_sync(kFull, msk ? (1u << o) : 0u);
        if (lane == 0) {
          pk_cnt[sl] = __popc(newmask);
          pk_mb[sl] = mb;
        }
        __threadfence_block();
        __syncwarp();
        if (lane == 0)
          *reinterpret_cast<volatile unsigned long long*>(slotw + sl) = slotword(got, sREADY);
        // greedy chain: the best new neighbour is the likely next top
        uint64_t ck2 = isnew ? x : 0;
        uint32_t cid = isnew ? v : kSentinel;
        warp_best(ck2, cid);
        {  // the runner-up (and optionally the third) child: hints for idle helpers
          uint64_t k2 = (isnew && v != cid) ? x : 0;
          uint32_t i2 = (isnew && v != cid) ? v : kSentinel;
          warp_best(k2, i2);
          if (lane == 0 && i2 != kSentinel && !(a.flags & 8u)) push_hint(k2, i2);
          if (a.flags & 131072u) {
            uint64_t k3 = (isnew && v != cid && v != i2) ? x : 0;
            uint32_t i3 = (isnew && v != cid && v != i2) ? v : kSentinel;
            warp_best(k3, i3);
            if (lane == 0 && i3 != kSentinel) push_hint(k3, i3);
          }
        }
        const bool chain = !(depth + 1 >= chain_max || cid == kSentinel || ctrl[0]) &&
                           ((a.flags & 16384u) || ck2 > gk);
        // an unchained best child is still a likely top soon after this
        // packet is committed: a hint for another helper
        if (!chain && lane == 0 && cid != kSentinel && !(a.flags & (8u | 65536u)))
          push_hint(ck2, cid);
        if (!chain) break;
        if (vbit(expd, cid)) break;
        {
          const uint32_t s0 = slot_of(cid);
          const uint64_t w0 = *reinterpret_cast<volatile unsigned long long*>(slotw + s0);
          const uint64_t w1 = *reinterpret_cast<volatile unsigned long long*>(slotw + s0 + 1);
          if (uint32_t(w0) == cid || uint32_t(w1) == cid) break;
        }
        if (!try_claim(cid, ck2, sl)) break;
        got = cid, gk = ck2;
        ++n_chain;
      }
    }
    if (fused)  // W chunks nobody got to during the search
      for (uint32_t c = next_chunk(); c < a.fa.nchunk; c = next_chunk()) wchunk(c);
    if (lane == 0) {
      atomicAdd(const_cast<uint32_t*>(ctrl) + 8, n_exp);
      atomicAdd(const_cast<uint32_t*>(ctrl) + 9, n_chain);
      atomicAdd(const_cast<uint32_t*>(ctrl) + 10, n_evict);
    }
    __syncthreads();  // matches the commit warp's first barrier
    __syncthreads();  // final array gathered
  }

  if constexpr (TP) return;
  // ---- final: CTA bitonic sort of the gathered pool candidates ----
  const uint32_t p2 = ctrl[4];
  const bool fin_smem = ctrl[5];
  Arr A = fin_smem ? Arr::at(smem + lay.tiles_off(), p2) : Arr::at(spill_slot, p2);
  for (uint32_t kk = 2; kk <= p2; kk <<= 1) {
    for (uint32_t j = kk >> 1; j > 0; j >>= 1) {
      for (uint32_t i = threadIdx.x; i < p2; i += blockDim.x) {
        const uint32_t pj = i ^ j;
        if (pj > i) {
          const bool desc = (i & kk) == 0;
          const uint64_t xi = A.k[i], xp = A.k[pj];
          const uint32_t ii = A.id[i], ip = A.id[pj];
          if (desc ? better(xp, ip, xi, ii) : better(xi, ii, xp, ip)) {
            A.k[i] = xp, A.k[pj] = xi;
            A.id[i] = ip, A.id[pj] = ii;
          }
        }
      }
      __syncthreads();
    }
  }
  const uint32_t pool = ctrl[7];
  const uint32_t take = pool < k ? pool : k;
  for (uint32_t r = threadIdx.x; r < k; r += blockDim.x) {
    const bool have = r < take;
    const double s = have ? okey_inv(A.k[r]) : __longlong_as_double(0x7ff8000000000000ll);
    a.ids[size_t(b) * k + r] = have ? A.id[r] : kSentinel;
    a.scores[size_t(b) * k + r] = have ? (float)s : __int_as_float(0x7fc00000);
    if (a.scores64) a.scores64[size_t(b) * k + r] = s;
  }
  if (threadIdx.x == 0) {
    a.n_out[b] = take;
    a.truncated[b] = take < k;
  }
  if (a.fa.out) fused_attention_tail<D>(a, lay, b, A, p2, fin_smem, take, smem);

}

template <int D, bool BF>
bool launch_pipe_d(ra_ctx* ctx, const SearchArgs& a, uint32_t max_n, uint8_t* scratch,
                   bool tp, int tps, int duo) {
  const size_t budget = ctx->smem_optin ? ctx->smem_optin : 227 * 1024;
  uint32_t spill_cap = 32;
  while (spill_cap < max_n) spill_cap <<= 1;
  SearchArgs s = a;
  // RA_PIPE_FLAGS: profiling / tuning switches, read once (0 = the defaults):
  //   bit 0      helpers idle (commit warp alone)
  //   bit 1      no L2 prefetch of new nodes' adjacency rows
  //   bit 3      no hint ring
  //   bits 4-7   chain length (default 3)        bits 8-12  tournament pick (12)
  //   bit 13     throughput mode: no L1 prefetch of key rows
  //   bit 14     chain regardless of the parent's rank
  //   bit 15     no hints from inline expansions   bit 16  no unchained-best hints
  //   bit 17     also hint the third child         bit 18  early next top (latency)
  //   bit 2      plain-loop row dot in the latency-mode expansions
  //   bit 27     DUO: no two-ahead row speculation
  //   bits 19-21 helpers allowed to take W chunks during the search (default all)
  //   bit 22     the commit warp's scheduler partner pre-expands too
  //   bits 23-26 stop-test pivot slack / 8 (default 48)
  //   bits 28-31 thr bisection steps / 4 (default 8)
  static const uint32_t env_flags = [] {
    const char* f = std::getenv("RA_PIPE_FLAGS");
    return f ? uint32_t(std::atoi(f)) : 0u;
  }();
  s.flags = env_flags;
  uint8_t* cur = scratch;
  s.spill = cur;
  cur += (size_t(a.B) * 2 * PipeLayout::arr_bytes(spill_cap) + 255) & ~size_t(255);
  s.vis_global = reinterpret_cast<uint32_t*>(cur);
  if (tp) {
    s.fa.out = nullptr;
    // TPS: visited bitset and a TMA row tile per query warp in shared
    // memory (no HBM bitsets to zero, coalesced 512-B row copies), as many
    // query warps per CTA as the batch needs to fill the SMs in ONE wave.
    // Taken while the batch fits one wave (B <= num_sms x warps that fit);
    // bigger batches keep the 16-warps-per-SM register-row kernel.
    // tps: 0 auto, 1 forced (if it fits), -1 off
#ifndef RA_TPS_ROWS
#define RA_TPS_ROWS 16
#endif
#ifndef RA_TPS_CAPO
#define RA_TPS_CAPO 128
#endif
    // DUO: TPS with a second warp per query that expands the next top while
    // the commit warp visits the previous packet; taken while the batch fits
    // one wave at <= kDuoPairs queries per SM (duo: 0 auto, 1 forced, -1 off)
    if (!BF && duo >= 0) {  // (f32 rows: the commit warp issues f32 row copies)
      PipeLayout ls{uint32_t(D), 0, (max_n + 31) / 32, 1, 64};  // (no row tile)
      ls.duo = 1;
      const uint32_t fit = uint32_t(std::min<size_t>((budget - ls.tp_base()) / ls.tp_warp_bytes(),
                                                     kDuoPairs));
      const uint32_t sms = uint32_t(ctx->num_sms);
      const uint32_t want = (a.B + sms - 1) / sms;
      if (fit >= 1 && (duo == 1 || want <= fit)) {
        const uint32_t wpc = std::max<uint32_t>(1, std::min(fit, want));
        {
          PipeLayout l0 = ls;
          l0.capO = 0;
          const size_t per = (budget - ls.tp_base()) / wpc - l0.tp_warp_bytes();
          ls.capO = uint32_t(std::min<size_t>(per / 24 - 2, 4096)) & ~31u;
        }
        const size_t bytes = ls.tp_base() + wpc * ls.tp_warp_bytes();
        auto kern = k_graph_search_pipe<D, true, true, false, true>;
        static int set_bytes[64] = {};
        if (int(bytes) > set_bytes[ctx->device & 63]) {
          RA_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       int(bytes)));
          set_bytes[ctx->device & 63] = int(bytes);
        }
        kern<<<(a.B + wpc - 1) / wpc, wpc * 64, bytes, ctx->stream>>>(s, ls, spill_cap);
        RA_LAUNCH_CHECK();
        return true;
      }
    }
    if (tps >= 0) {
      // the overflow arrays FO / UO get what the warps leave of the budget
      // (a search that outgrows them moves them to its HBM slot: exact, slow)
      PipeLayout ls{uint32_t(D), std::min<uint32_t>(std::max<uint32_t>(a.max_M, 1), RA_TPS_ROWS),
                    (max_n + 31) / 32, 1, RA_TPS_CAPO};
      const uint32_t fit = uint32_t(std::min<size_t>((budget - ls.tp_base()) / ls.tp_warp_bytes(),
                                                     kTW));
      const uint32_t sms = uint32_t(ctx->num_sms);
      const uint32_t want = (a.B + sms - 1) / sms;
      if (fit >= 1 && (tps == 1 || want <= fit)) {
        const uint32_t wpc = std::max<uint32_t>(1, std::min(fit, want));
        {
          PipeLayout l0 = ls;
          l0.capO = 0;
          const size_t per = (budget - ls.tp_base()) / wpc - l0.tp_warp_bytes();
          ls.capO = uint32_t(std::min<size_t>(per / 24 - 2, 4096)) & ~31u;
        }
        const size_t wb = ls.tp_warp_bytes();
        const size_t bytes = ls.tp_base() + wpc * wb;
        auto kern = k_graph_search_pipe<D, true, true, BF>;
        static int set_bytes[64] = {};
        if (int(bytes) > set_bytes[ctx->device & 63]) {
          RA_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       int(bytes)));
          set_bytes[ctx->device & 63] = int(bytes);
        }
        kern<<<(a.B + wpc - 1) / wpc, wpc * 32, bytes, ctx->stream>>>(s, ls, spill_cap);
        RA_LAUNCH_CHECK();
        return true;
      }
    }
#ifndef RA_TP_CAPO
#define RA_TP_CAPO 256
#endif
    PipeLayout lay{uint32_t(D), std::max<uint32_t>(a.max_M, 1), (max_n + 31) / 32, 0, RA_TP_CAPO};
    const size_t bytes = kTW * lay.tp_warp_bytes();
    auto kern = k_graph_search_pipe<D, false, true, BF>;
    RA_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes)));
    kern<<<(a.B + kTW - 1) / kTW, kTW * 32, bytes, ctx->stream>>>(s, lay, spill_cap);
    RA_LAUNCH_CHECK();
    return true;
  }
  PipeLayout lay{uint32_t(D), std::max<uint32_t>(a.max_M, 1), (max_n + 31) / 32, 1, 0};
  if (s.fa.out) {
    // the fused tail stages the W chunk partials and >= 8 V rows in the
    // helpers' tiles (fused_attention_tail): small-degree graphs get taller
    // tiles so that area always holds them
    const size_t need = (40 + 32 * (size_t(D) + 2)) * 8 + 8 * (size_t(D) * 4 + 8) + 16;
    while (size_t(kPW) * lay.tile_bytes() < need) ++lay.MT;
  }
  if (lay.bytes() + PipeLayout::arr_bytes(512) * 2 > budget) lay.vis_smem = 0;
  const size_t fixed = lay.bytes();
  if (fixed + PipeLayout::arr_bytes(256) * 2 > budget) return false;
  lay.capO = uint32_t(std::min<size_t>((budget - fixed - 64) / 24, 8192)) & ~31u;
  if (lay.bytes() > budget) return false;
  auto kern = lay.vis_smem ? k_graph_search_pipe<D, true, false, BF>
                           : k_graph_search_pipe<D, false, false, BF>;
  {  // the attribute only ever grows; set it when a launch needs more
    static int set_bytes[64][2] = {};  // per device (the attribute is per device)
    int& have = set_bytes[ctx->device & 63][lay.vis_smem ? 1 : 0];
    if (int(lay.bytes()) > have) {
      RA_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   int(lay.bytes())));
      have = int(lay.bytes());
    }
  }
  kern<<<a.B, kPW * 32, lay.bytes(), ctx->stream>>>(s, lay, spill_cap);
  RA_LAUNCH_CHECK();
  return true;
}

}  // namespace

bool pipe_latency_supported(const ra_ctx* ctx, uint32_t d, uint32_t max_M, uint32_t max_n) {
  if (max_M > 32 || max_M == 0) return false;
  if (d != 8 && d != 16 && d != 32 && d != 64 && d != 128) return false;
  const size_t budget = ctx->smem_optin ? ctx->smem_optin : 227 * 1024;
  PipeLayout lay{d, max_M, (max_n + 31) / 32, 1, 0};
  if (lay.bytes() + PipeLayout::arr_bytes(512) * 2 > budget) lay.vis_smem = 0;
  return lay.bytes() + PipeLayout::arr_bytes(256) * 2 <= budget;
}

size_t search_pipe_scratch_bytes(uint32_t B, uint32_t max_n) {
  uint32_t p2 = 32;
  while (p2 < max_n) p2 <<= 1;
  return size_t(B) * 2 * PipeLayout::arr_bytes(p2) + 256 +
         size_t(B) * 2 * ((max_n + 31) / 32) * 4 + 256;
}

// Latency mode (one CTA of helpers per query) while the batch leaves SMs
// idle; throughput mode (8 queries per CTA) once it fills the GPU.
bool launch_graph_search_pipe(ra_ctx* ctx, const SearchArgs& a, uint32_t max_n,
                              uint8_t* scratch, int mode) {
  if (a.max_M > 32 || a.max_M == 0) return false;
  // mode 0 auto, 1 throughput (DUO, else TPS, when it fits one wave), 2
  // latency, 3 throughput with register rows only, 4 TPS forced, 5 DUO forced
  const bool tp = mode == 1 || mode == 3 || mode == 4 || mode == 5 ||
                  (mode == 0 && a.B > 2u * uint32_t(ctx->num_sms));
  const int tps = mode == 3 ? -1 : mode == 4 ? 1 : 0;
  const int duo = mode == 3 || mode == 4 ? -1 : mode == 5 ? 1 : 0;
  if (a.bf16) {  // bf16 rows: d in {32, 64, 128} (16-B multiples)
    switch (a.d) {
      case 128: return launch_pipe_d<128, true>(ctx, a, max_n, scratch, tp, tps, duo);
      case 64: return launch_pipe_d<64, true>(ctx, a, max_n, scratch, tp, tps, duo);
      case 32: return launch_pipe_d<32, true>(ctx, a, max_n, scratch, tp, tps, duo);
      default: return false;
    }
  }
  switch (a.d) {
    case 128: return launch_pipe_d<128, false>(ctx, a, max_n, scratch, tp, tps, duo);
    case 64: return launch_pipe_d<64, false>(ctx, a, max_n, scratch, tp, tps, duo);
    case 32: return launch_pipe_d<32, false>(ctx, a, max_n, scratch, tp, tps, duo);
    case 16: return launch_pipe_d<16, false>(ctx, a, max_n, scratch, tp, tps, duo);
    case 8: return launch_pipe_d<8, false>(ctx, a, max_n, scratch, tp, tps, duo);
    default: return false;
  }
}

}  // namespace ra
