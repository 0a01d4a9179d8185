// Decode hot path of the hybrid two-tier attention step (engine.py:151-195,
// decode mode) for B200 (sm_100a).
//
// HBM layout: K and V of one position are adjacent (KV [B*Hkv, T, 2, D]), so
// every selected archive entry is ONE contiguous 2*D*esz-byte row; the TMA
// unit gathers 4 such rows per tile::gather4 op straight into shared memory.
//
// One persistent kernel per step streams two kinds of work items through
// warp-private TMA pipelines (S stages of SUB=32 rows, mbarrier per stage):
//   * dense items  : the whole attended window [dlo, dhi) of one (batch,
//                    kv-head); all G query heads attend every row
//                    (engine.py:161-164). Item id == bk = b*Hkv + kv-head, so
//                    they are dispatched first; the warp that finishes one
//                    also computes the window weights and the fp64 MAW EMA
//                    (kv_cache.py:171-187, engine.py:177-191) from the dense
//                    scores it stored -- off the tail of the step.
//   * sparse items : SPARSE_ROWS-row slices of the (batch, kv-head) union list
//                    of selected archive rows; each entry carries a G-bit mask
//                    of the query heads whose context/padding contains it
//                    (engine.py:134-149), so every archived row is read once.
// Each item writes (m, z, acc) per query head to a fixed slot; the warp that
// finishes the last item of a (batch, kv-head) folds them in a fixed order
// and applies merge_states(sparse, dense) (attention.py:153-188). Results do
// not depend on which warp ran which item (no float atomics).
//
// Two compute variants:
//   decode_f32_kernel  (float32 storage, the reference-exact path): one key
//       row per lane, fp64 dot products in the reference's sequential order
//       (_core.pyx:59-65), fp64 online softmax, fp32 P.V.
//   decode_bf16_kernel (bfloat16 storage): QK^T and P.V on the tensor cores
//       with mma.sync m16n8k16 (K rows x 8 query heads; V^T x P^T, P split
//       into bf16 hi + lo so P keeps ~16 significant bits), fp32 softmax in
//       the mma fragment layout. The tensor cores are used to cut issue slots
//       of the 8-head GEMV, not for FLOPs: the kernel stays HBM-bound. K|V rows
//       land in 128B-swizzled 32x128-byte tiles so ldmatrix is conflict-free.
#include "hgca_common.cuh"
#include "hgca_internal.h"
#include "hgca_tc.cuh"
#include "hgca_host.h"

#include <cuda.h>

#include <type_traits>

namespace hgca {

// Debug build only (-DHGCA_TIMELINE): per-warp timeline of the decode kernel,
// read back with hgca_debug_timeline (tools/timeline.py).
#ifdef HGCA_TIMELINE
#define TL_SLOTS 20
__device__ unsigned long long g_tl[148 * 16 * TL_SLOTS];
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define TL(...) __VA_ARGS__
__device__ unsigned long long g_tlm[4096 * 8];  // merge kernel: per CTA phase stamps
// step boundary (graph mode): per decode CTA {entry, wait released, previous
// merge grid's last CTA end}; the merge CTAs atomicMax their end into g_mend
__device__ unsigned long long g_gap[1024 * 4];
__device__ unsigned long long g_mend;
#else
#define TL(...)
#endif

#ifndef HGCA_BF16_STAGES
#define HGCA_BF16_STAGES 2
#endif
#ifndef HGCA_LAZY_CLAIM
#define HGCA_LAZY_CLAIM 1
#endif
#ifndef HGCA_F32_STAGES
#define HGCA_F32_STAGES 2
#endif
#ifndef HGCA_F32_NC
#define HGCA_F32_NC 8  // consumer warps per CTA cap (shared memory decides below it)
#endif
#ifndef HGCA_BF16_PAIRS
#define HGCA_BF16_PAIRS 6  // consumer warps per CTA, each paired with its own producer warp
#endif

constexpr int SUB = 32;  // rows per pipeline stage (one per lane)
constexpr uint32_t FULL = 0xffffffffu;
constexpr int SMEM_MAX = 232448;  // dynamic shared memory per CTA on sm_100

// Per-stage descriptor (smem, written by the warp that issued the stage).
struct StageDesc {
  int item, bk, r0, n;
  int first, last, dense, pad;
};

// ------------------------------------------------------------------ step positions
// The step's window range: from the descriptor (eager launches), or -- when
// a.state is set (graph-replayable steps, hgca_decode_desc.state) -- from the
// device-resident step state {dlo, dhi, epoch, arrivals}, which the merge
// kernel advances by one position after every step. Everything derived from
// the range (dense item count, MAW EMA extent) is computed here, on device.
struct StepPos {
  int64_t dlo, dhi, w_old;
  int W, dr, Sd, nd;  // window + kv_in rows, rows per dense item, dense items per (b, kv-head), dense items
  int nf;             // full-length sparse items (they come first, see Cursor)
};
__device__ __forceinline__ int64_t ld_relaxed_i64(const int64_t* p) {
  int64_t v;
  asm volatile("ld.relaxed.gpu.global.s64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ StepPos step_pos(const DecodeArgs& a) {
  StepPos p;
  if (a.state) {
    p.dlo = ld_relaxed_i64(a.state);
    p.dhi = ld_relaxed_i64(a.state + 1);
    p.w_old = p.dhi - 1 - p.dlo;  // a decode step adds exactly one entry
  } else {
    p.dlo = a.dlo;
    p.dhi = a.dhi;
    p.w_old = a.w_old;
  }
  p.W = (int)(p.dhi - p.dlo);
  // dense items (window parts) follow the sparse item granularity the last
  // union rebuild chose for this step size (item_offsets_kernel: long items
  // for big steps, down to one 32-row stage for small ones, so a small step
  // spreads over every warp instead of one warp walking a 256-row window
  // part); before any rebuild, the descriptor's default
  const int chosen = a.item_off[2 * (a.B * a.Hkv + 1)];
  p.dr = chosen >= 16 && chosen <= (int)a.dense_rows ? chosen : (int)a.dense_rows;
#ifndef HGCA_DENSE_DIV
#define HGCA_DENSE_DIV 2
#endif
  // the window parts come right after the full sparse items, so a long one
  // could still run when the short tail items are gone: halve them (at least
  // one 32-row stage; quarter-length parts measured worse at C3)
  p.dr = max(min(p.dr, SUB), p.dr / HGCA_DENSE_DIV);
  p.Sd = (p.W + p.dr - 1) / p.dr;
  p.nd = (int)(a.B * a.Hkv) * p.Sd;
  p.nf = a.item_off[a.B * a.Hkv];
  return p;
}

// ------------------------------------------------------------------ work items
// Item ids: [0, nf) the full-length sparse items (item_tab[id]), then
// [nf, nf + nd) the dense items (bk = (id - nf) / Sd; window rows of part
// (id - nf) % Sd, sp.dr each), then the sparse tail items (item_tab[id - nd]).
// The full sparse items depend only on the last union rebuild, not on the
// step's window range, so a warp whose first item is one of them can start
// gathering it before the previous step's kernels finish (graph mode, see
// producer_prefetch); the short tail items come last so the step ends
// balanced. The cursor walks a warp through items in sub-chunks of SUB rows;
// lane 0 holds the prefetched id of the next item.
struct Cursor {
  int nxt;  // lane 0
  int item, bk, lo, hi, row, dense;
};

__device__ __forceinline__ void cursor_item(Cursor& c, const DecodeArgs& a, const StepPos& sp, int it) {
  c.item = it;
  if (it >= sp.nf && it < sp.nf + sp.nd) {
    c.dense = 1;
    c.bk = (it - sp.nf) / sp.Sd;
    c.lo = ((it - sp.nf) % sp.Sd) * sp.dr;
    c.hi = min(sp.W, c.lo + sp.dr);
  } else {
    c.dense = 0;
    const int4 e = __ldg(a.item_tab + (it < sp.nf ? it : it - sp.nd));
    c.bk = e.x;
    c.lo = e.y;
    c.hi = e.z;
  }
  c.row = c.lo;
}

__device__ __forceinline__ StageDesc cursor_stage(Cursor& c) {
  StageDesc d;
  d.item = c.item;
  d.bk = c.bk;
  d.r0 = c.row;
  d.n = min(SUB, c.hi - c.row);
  d.first = c.row == c.lo;
  d.last = c.row + SUB >= c.hi;
  d.dense = c.dense;
  d.pad = 0;
  c.row += SUB;
  return d;
}

// Static first wave: a warp's first item is its global warp index (cur.nxt
// preset by the caller, no contended atomic before the first gather); every
// later item is atomicAdd(counter) + nwarps, prefetched while the current
// item runs.
__device__ __forceinline__ StageDesc cursor_next_off(Cursor& c, const DecodeArgs& a, const StepPos& sp, int total,
                                                     int lane, int nwarps) {
  if (c.item < 0 || c.row >= c.hi) {
#if HGCA_LAZY_CLAIM
    // claim the next item only once the current one is fully issued: a warp
    // then holds at most one item it has not started, so the last items of
    // the queue go to the warps that are actually about to be free
    if (lane == 0 && c.nxt < 0) c.nxt = atomicAdd(a.counter, 1) + nwarps;
#endif
    const int it = __shfl_sync(FULL, c.nxt, 0);
    if (it >= total) {
      StageDesc d;
      d.item = -1;
      d.bk = d.r0 = d.n = d.first = d.last = d.dense = d.pad = 0;
      return d;
    }
#if HGCA_LAZY_CLAIM
    if (lane == 0) c.nxt = -1;
#else
    if (lane == 0) c.nxt = atomicAdd(a.counter, 1) + nwarps;
#endif
    cursor_item(c, a, sp, it);
  }
  return cursor_stage(c);
}

// kv_in (engine.py:161-163, append_kv kv_cache.py:122-169): the step's new K
// and V rows of (batch, kv-head) bk are written at position dhi-1 by the warp
// that issues the dense sub-chunk holding that row, right before its gather
// (generic-proxy stores fenced before the async-proxy TMA read). Rows are
// stored position-rotated (see rotoff). Every lane writes 16-byte chunks.
template <int D, bool BF16>
__device__ __forceinline__ void write_new_row(const DecodeArgs& a, const StepPos& sp, const StageDesc& d, int lane) {
  if (!a.k_new || !d.dense || d.r0 + d.n != sp.W) return;
  constexpr int ROWB = D * (BF16 ? 2 : 4), CH = 2 * ROWB / 16;  // 16-byte chunks of the K|V row pair
  const int64_t pos = sp.dhi - 1;
  unsigned char* dst = reinterpret_cast<unsigned char*>(const_cast<void*>(a.KV)) + ((int64_t)d.bk * a.T + pos) * 2 * ROWB;
  for (int c = lane; c < CH; c += 32) {
    const unsigned char* src = reinterpret_cast<const unsigned char*>(c < CH / 2 ? a.k_new : a.v_new) +
                               (int64_t)d.bk * ROWB + (c % (CH / 2)) * 16;
    const int pc = (c & ~7) | ((c ^ (int)pos) & 7);  // rotated rows (both storage dtypes)
    *reinterpret_cast<uint4*>(dst + pc * 16) = *reinterpret_cast<const uint4*>(src);
  }
  fence_proxy_async_global();
}

// Union entry of lane's row of sub-chunk d: position | (query-head mask << 24).
// Rows past the sub-chunk end get position 0 and an empty mask.
template <int G>
__device__ __forceinline__ int32_t sub_entry(const StageDesc& d, const DecodeArgs& a, const StepPos& sp, int lane) {
  if (d.item < 0 || lane >= d.n) return 0;
  if (d.dense) return (int32_t)(sp.dlo + d.r0 + lane) | (int32_t)(((1u << G) - 1u) << 24);
  return __ldg(a.u_ent + (int64_t)d.bk * a.T + d.r0 + lane);
}

// ------------------------------------------------------------------ merge kernel
// One CTA per query head (batch, kv-head, g) with D threads, one output dim
// each, launched behind the decode kernel with programmatic dependent launch.
// The partials are head-major, so this head's partials of the (batch,
// kv-head)'s contiguous item ranges (sparse: full items, tail items; dense:
// the window parts) are contiguous: up to three 1-D TMA bulk copies per chunk
// of MERGE_NI items stream them into shared memory while two warps read the
// items' (m, z) and form the fold weights. The fold runs in item order: max,
// one exp per item, weighted sums over the chunk (4 interleaved partial sums,
// combined in a fixed order); chunks of long lists combine with an online
// rescale. Then:
//   * merge_states(sparse, dense)            attention.py:153-188, engine.py:166-169
//   * window weights w = float32(exp(s - m) / z) from the stored dense
//     scores and the dense (m, z)            _core.pyx:81-82
//   * MAW maintenance, 3 separately rounded fp64 ops (kv_cache.py:186), new
//     entries maw = w (engine.py:177-191).
// Fixed order throughout: deterministic. (B*Hq CTAs of ~50 KB: four per SM,
// so the whole merge of a C2/C4 step is one wave.) Long item lists (128K
// context: ~300 items per head) are split over m.split CTAs per head whose
// partials the last to arrive combines in share order (split merge).
constexpr int MERGE_NI = 96;  // items per fold chunk

template <int D>
struct MergeCfg {
  static constexpr int NT = D;                 // threads: one per output dim
  static constexpr int NI = MERGE_NI;
  static constexpr int IPL = NI / 32;          // items per lane in the (m, z) pass
  static constexpr int OFF_W = NI * D * 4;     // accumulators [NI][D] f32, then weights [NI] f64
  static constexpr int OFF_BAR = OFF_W + NI * 8;
  static constexpr int SMEM = OFF_BAR + 16;
  static_assert(NI % 32 == 0 && D % 64 == 0, "merge mapping");
};

template <int D, int G, typename SC>
__global__ void __launch_bounds__(MergeCfg<D>::NT) decode_merge_kernel(const __grid_constant__ DecodeArgs a) {
  using C = MergeCfg<D>;
  const DecodeMergeArgs& m = a.m;
  extern __shared__ __align__(128) unsigned char msm[];
  float* sacc = reinterpret_cast<float*>(msm);
  // fold arithmetic: fp64 on the reference-exact fp32 path; fp32 weights and
  // partial sums on the bf16 path (its 1e-2 contract; the (m, z) stats stay
  // fp64), which takes the fp64 exp / convert / FMA chains off every merge
  using AT = typename std::conditional<sizeof(SC) == 8, double, float>::type;
  AT* sw = reinterpret_cast<AT*>(msm + C::OFF_W);
  uint64_t* bar = reinterpret_cast<uint64_t*>(msm + C::OFF_BAR);
  __shared__ double hM[2], hZ[2], hS[2];  // [0] sparse, [1] dense running stats
  __shared__ int x_last;                  // split merge: this CTA combines the head's partials
  const int S = m.split;                  // CTAs per query head (split merge), 1 = off
  const int js = (int)(blockIdx.x % S);   // this CTA's share of the head's items
  const int64_t bq = blockIdx.x / S;      // b * Hq + kv-head * G + g
  const int64_t b = bq / m.Hq, kvh = (bq % m.Hq) / G, bk = b * m.Hkv + kvh;
  const int g = (int)(bq % m.Hq) % G;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  TL(if (tid == 0) g_tlm[blockIdx.x * 8 + 0] = gtimer();)
  if (tid == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
  }
  // Everything that does not depend on this step's decode grid is read before
  // griddepcontrol.wait: the item ranges (built at the last selection change)
  // and the window MAW (only this kernel writes it).
  // (the step state, in graph mode, was last written by the previous step's
  // merge, which completed before this step's decode grid passed its wait)
  const StepPos sp = step_pos(a);
  const uint64_t epoch = a.state ? (uint64_t)ld_relaxed_i64(a.state + 2) : m.epoch;
  const int64_t BK = m.B * m.Hkv, nd = sp.nd, Sd = sp.Sd;
  const int64_t o0 = m.item_off[bk], o1 = m.item_off[bk + 1];
  const int64_t t0 = m.item_off[BK + 1 + bk], t1 = m.item_off[BK + 1 + bk + 1];
  const int64_t nf = o1 - o0, ns = nf + (t1 - t0), n = ns + Sd;
  // this CTA's items: a contiguous share of the sparse items; the last share
  // also holds the dense (window) items, so its dense stats are final locally
  const int64_t r0 = ns * js / S, r1 = js == S - 1 ? n : ns * (js + 1) / S;
  const bool dense_here = js == S - 1;
  // item ids (see Cursor): full sparse items [0, NF), dense [NF, NF + nd), tails after
  const int64_t NF = sp.nf;
  auto item_id = [&](int64_t i) {
    return i < nf ? o0 + i : (i < ns ? nd + t0 + (i - nf) : NF + bk * Sd + (i - ns));
  };
  const double* pm = m.part_m + g * m.MI;
  const double* pz = m.part_z + g * m.MI;
  const float* pacc = m.part_acc + g * m.MI * D;
  constexpr int EB = 8;  // window entries per thread per epilogue batch (one batch covers 8*D)
  const bool epi = a.maw != nullptr || a.wts_out != nullptr;
  const int64_t W = sp.W, n_el = epi ? W : 0, w_old = sp.w_old;
  const SC* dsc = reinterpret_cast<const SC*>(a.dsc) + bq * a.dsc_ld;
  double* maw = a.maw ? a.maw + bq * a.T + sp.dlo : nullptr;
  SC sv[EB];
  double mo[EB];
  auto maw_load = [&](int64_t x0) {
#pragma unroll
    for (int u = 0; u < EB; ++u) {
      const int64_t j = x0 + u * C::NT + tid;
      mo[u] = (maw && j < n_el && j < w_old) ? maw[j] : 0.0;
    }
  };
  auto dsc_load = [&](int64_t x0) {
#pragma unroll
    for (int u = 0; u < EB; ++u) {
      const int64_t j = x0 + u * C::NT + tid;
      sv[u] = j < n_el ? dsc[j] : (SC)0;
    }
  };
  maw_load(0);
  if (tid < 2) {
    hM[tid] = -INFINITY;
    hZ[tid] = 0.0;
  }
  double acc_s = 0.0, acc_d = 0.0;
  uint32_t phase = 0;
  // ---- window weights + MAW maintenance from the stored dense scores and
  // the dense (m, z) (batches of EB entries per thread; batch 0 is loaded
  // before the folds). Needs only the final dense stats, so it runs inside the
  // last fold chunk, before that chunk's bulk-copy wait (its latency hides
  // the copies); with a push exchange pending it runs after the push, and in
  // a split merge the dense share runs it after publishing its partial.
  bool epi_done = false;
  auto window_epilogue = [&]() {
    epi_done = true;
    const double md = hM[1], zd = hZ[1];
    const bool d_ok = (zd > 0.0) && md != -INFINITY;
    const double rz = 1.0 / zd;
    for (int64_t x0 = 0; x0 < n_el; x0 += (int64_t)EB * C::NT) {
      if (x0) {
        maw_load(x0);
        dsc_load(x0);
      }
#pragma unroll
      for (int u = 0; u < EB; ++u) {
        const int64_t j = x0 + u * C::NT + tid;
        if (j >= n_el) continue;
        float w32;
        if constexpr (sizeof(SC) == 8) {  // fp32 storage: reference-exact fp64 weights (_core.pyx:81-82)
          w32 = d_ok ? (float)(exp((double)sv[u] - md) / zd) : 0.f;
        } else {  // bf16 storage: fp32 math (no bit-exactness contract on this path)
          w32 = d_ok ? __expf((float)sv[u] - (float)md) * (float)rz : 0.f;
        }
        if (a.wts_out) a.wts_out[bq * W + j] = w32;
        if (maw) {
          const double aw = (double)w32;
          maw[j] = j < w_old ? __dadd_rn(__dmul_rn(a.one_minus_alpha, mo[u]), __dmul_rn(a.alpha, aw)) : aw;
        }
      }
    }
  };

  // the mbarrier init and the running stats are visible to every warp before
  // any of them folds (griddepcontrol.wait is not a CTA barrier)
  __syncthreads();
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
  TL(if (tid == 0) g_tlm[blockIdx.x * 8 + 1] = gtimer();)
  // the next step's decode grid may launch now (it waits for this grid in
  // its own griddepcontrol.wait before touching anything)
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  // the decode grid is complete: re-arm its work counter for the next step
  if (blockIdx.x == 0 && tid == 0) *a.counter = 0;
  // One fold pass over the concatenated item list [full items, tail items |
  // dense parts]: the first ns items are sparse, the rest dense.
  for (int64_t c0 = r0; c0 < r1; c0 += C::NI) {
    const int64_t c1 = min(r1, c0 + C::NI), cn = c1 - c0;
    const int64_t lo[3] = {0, nf, ns}, hi[3] = {nf, ns, n};
    if (tid == 0) {
      uint32_t bytes = 0;
      for (int r = 0; r < 3; ++r) {
        const int64_t x0 = max(c0, lo[r]), x1 = min(c1, hi[r]);
        if (x1 > x0) bytes += (uint32_t)((x1 - x0) * D * 4);
      }
      mbar_expect_tx(bar, bytes);
      for (int r = 0; r < 3; ++r) {
        const int64_t x0 = max(c0, lo[r]), x1 = min(c1, hi[r]);
        if (x1 > x0)
          bulk_g2s(sacc + (x0 - c0) * D, pacc + item_id(x0) * D, (uint32_t)((x1 - x0) * D * 4), bar);
      }
    }
    if (c0 == r0 && dense_here) dsc_load(0);  // the window scores of the epilogue: in flight during the fold
    TL(if (tid == 0 && c0 == r0) g_tlm[blockIdx.x * 8 + 6] = gtimer();)
    // the chunk's sparse items [0, ce) (warp 0) and dense items [ce, cn) (warp 1)
    const int64_t ce = min(cn, max((int64_t)0, ns - c0));
    if (wid < 2) {
      const int64_t i0 = wid ? ce : 0, i1 = wid ? cn : ce;
      if (i1 > i0) {  // warp-uniform
        double mv[C::IPL], zv[C::IPL];
#pragma unroll
        for (int u = 0; u < C::IPL; ++u) {
          const int64_t i = i0 + u * 32 + lane;
          mv[u] = -INFINITY;
          zv[u] = 0.0;
          if (i < i1) {
            const int64_t it = item_id(c0 + i);
            mv[u] = pm[it];
            zv[u] = pz[it];
          }
        }
        double mx = -INFINITY;
        if constexpr (sizeof(AT) == 8) {
#pragma unroll
          for (int u = 0; u < C::IPL; ++u) mx = fmax(mx, mv[u]);
          mx = warp_max_f64(mx);
        } else {  // bf16 path: the items' m are fp32 values (exact in fp32): a 32-bit reduction
          float mf = -INFINITY;
#pragma unroll
          for (int u = 0; u < C::IPL; ++u) mf = fmaxf(mf, (float)mv[u]);
#pragma unroll
          for (int o = 16; o; o >>= 1) mf = fmaxf(mf, __shfl_xor_sync(FULL, mf, o));
          mx = mf;
        }
        const double mold = hM[wid], mn = fmax(mold, mx);
        double zl = 0.0;
#pragma unroll
        for (int u = 0; u < C::IPL; ++u) {
          const int64_t i = i0 + u * 32 + lane;
          if (i < i1) {
            double w;
            if constexpr (sizeof(AT) == 8) {
              w = (mv[u] == -INFINITY || mn == -INFINITY) ? 0.0 : exp(mv[u] - mn);
              sw[i] = w;
            } else {
              const float wf = (mv[u] == -INFINITY || mn == -INFINITY) ? 0.f : __expf((float)(mv[u] - mn));
              sw[i] = wf;
              w = wf;
            }
            zl += zv[u] * w;
          }
        }
        zl = warp_sum_f64(zl);
        __syncwarp();  // every lane's read of hM[wid] before lane 0 rewrites it
        if (lane == 0) {
          double so;
          if constexpr (sizeof(AT) == 8)
            so = (mold == -INFINITY || mn == -INFINITY) ? 0.0 : exp(mold - mn);
          else
            so = (mold == -INFINITY || mn == -INFINITY) ? 0.0 : (double)__expf((float)(mold - mn));
          hS[wid] = so;
          hZ[wid] = hZ[wid] * so + zl;
          hM[wid] = mn;
        }
      }
    }
    __syncthreads();
    TL(if (tid == 0 && c0 == r0) g_tlm[blockIdx.x * 8 + 7] = gtimer();)
    if (c1 == n && !m.push_n && S == 1) window_epilogue();  // dense stats final: overlap the copies
    TL(if (tid == 0 && c1 == n) g_tlm[blockIdx.x * 8 + 3] = gtimer();)
    mbar_wait(bar, phase);
    phase ^= 1;
    const float* src = sacc + tid;
    auto dot = [&](int64_t i0, int64_t i1) {  // 4 interleaved partial sums, combined in a fixed order
      AT p0 = 0, p1 = 0, p2 = 0, p3 = 0;
      int64_t i = i0;
      for (; i + 4 <= i1; i += 4) {
        p0 += sw[i] * (AT)src[i * D];
        p1 += sw[i + 1] * (AT)src[(i + 1) * D];
        p2 += sw[i + 2] * (AT)src[(i + 2) * D];
        p3 += sw[i + 3] * (AT)src[(i + 3) * D];
      }
      for (; i < i1; ++i) p0 += sw[i] * (AT)src[i * D];
      return (double)((p0 + p1) + (p2 + p3));
    };
    if (ce > 0) acc_s = acc_s * hS[0] + dot(0, ce);
    if (cn > ce) acc_d = acc_d * hS[1] + dot(ce, cn);
    __syncthreads();  // the next chunk's copies overwrite sacc / sw
  }
  TL(if (tid == 0) g_tlm[blockIdx.x * 8 + 2] = gtimer();)
  if (S > 1) {
    // split merge: every share publishes its partial at once and the last CTA
    // to arrive folds the shares in order (so the result does not depend on
    // arrival order); the dense share runs the window epilogue afterwards,
    // off the output's critical path
    double* xm = m.xmz + (bq * S + js) * 4;
    double* xa = m.xacc + (bq * S + js) * 2 * D;
    xa[tid] = acc_s;
    xa[D + tid] = acc_d;
    if (tid == 0) {
      xm[0] = hM[0];
      xm[1] = hZ[0];
      xm[2] = hM[1];
      xm[3] = hZ[1];
    }
    __threadfence();
    __syncthreads();
    if (tid == 0) x_last = atomicAdd(m.xcnt + bq, 1u) == (unsigned)(S - 1);
    __syncthreads();
    if (x_last) {
      __threadfence();
      const double* xm0 = m.xmz + bq * S * 4;
      const double* xa0 = m.xacc + bq * S * 2 * D;
      double M = -INFINITY;
      for (int j = 0; j < S; ++j) M = fmax(M, __ldcg(xm0 + j * 4));
      double Z = 0.0, A = 0.0;
      for (int j = 0; j < S; ++j) {
        const double mj = __ldcg(xm0 + j * 4);
        const double w = (mj == -INFINITY || M == -INFINITY) ? 0.0 : exp(mj - M);
        Z = fma(__ldcg(xm0 + j * 4 + 1), w, Z);
        A = fma(__ldcg(xa0 + j * 2 * D + tid), w, A);
      }
      acc_s = A;
      acc_d = __ldcg(xa0 + (S - 1) * 2 * D + D + tid);
      __syncthreads();  // every thread has read hM / hZ above (through xm of its own share)
      if (tid == 0) {
        hM[0] = M;
        hZ[0] = Z;
        hM[1] = __ldcg(xm0 + (S - 1) * 4 + 2);
        hZ[1] = __ldcg(xm0 + (S - 1) * 4 + 3);
        m.xcnt[bq] = 0;  // re-armed for the next step
      }
      __syncthreads();
    }
  }
  const double Ms = hM[0], Zs = hZ[0], md = hM[1], zd = hZ[1];
  if (S == 1 || x_last) {
    // merge_states(sparse, dense) (attention.py:153-188) in the equivalent
    // flash form -- both partials rescaled to M = max(m_s, m_d), one exp
    // each, one log -- so the dependent fp64 transcendental chain is three
    // deep instead of five (its latency is the tail of every step); equal to
    // the reference's lse-space form up to fp64 rounding
    const bool s_empty = !(Zs > 0.0) || Ms == -INFINITY;
    const bool d_empty = !(zd > 0.0) || md == -INFINITY;
    const double M = fmax(s_empty ? -INFINITY : Ms, d_empty ? -INFINITY : md);
    const bool both_empty = M == -INFINITY;
    // (bf16 path: fp32 transcendentals, its 1e-2 contract)
    auto exp_ = [](double x) { return sizeof(AT) == 8 ? exp(x) : (double)__expf((float)x); };
    auto log_ = [](double x) { return sizeof(AT) == 8 ? log(x) : (double)__logf((float)x); };
    const double es = s_empty ? 0.0 : exp_(Ms - M), ed = d_empty ? 0.0 : exp_(md - M);
    const double Zt = both_empty ? 1.0 : fma(Zs, es, zd * ed);
    const float ov = both_empty ? 0.f : (float)(fma(acc_s, es, acc_d * ed) / Zt);
    const double lv = both_empty ? -INFINITY : M + log_(Zt);
    const bool want_s = m.out_sparse || m.lse_sparse || (m.push_n && m.push_sparse);
    const double lse_s = (want_s && !s_empty) ? Ms + log_(Zs) : -INFINITY;
    const float os = (want_s && !s_empty) ? (float)(acc_s / Zs) : 0.f;
    m.out[bq * D + tid] = ov;
    if (m.out_sparse) m.out_sparse[bq * D + tid] = os;
    if (tid == 0) {
      m.lse[bq] = lv;
      if (m.lse_sparse) m.lse_sparse[bq] = lse_s;
    }
    if (m.push_n) {
      // one-shot exchange: this head's row of the rank's packed partial goes
      // straight into every destination slot (peer HBM over NVLink); the last
      // CTA to finish publishes the step's epoch once all rows are fenced
      const float pv = m.push_sparse ? os : ov;
      const double pl = m.push_sparse ? lse_s : lv;
      const int64_t lse_off = m.B * m.Hq * D * 4;
      for (int p = 0; p < m.push_n; ++p) {
        reinterpret_cast<float*>(m.push_dst[p])[bq * D + tid] = pv;
        if (tid == 0) reinterpret_cast<double*>(m.push_dst[p] + lse_off)[bq] = pl;
      }
      __threadfence_system();
      __syncthreads();
      if (tid == 0) {
        const unsigned prev = atomicAdd(m.push_cnt, 1u);
        if (prev == gridDim.x / S - 1) {  // every head's combining CTA has pushed
          *m.push_cnt = 0;  // re-armed for the next step (stream order)
          __threadfence_system();
          for (int p = 0; p < m.push_n; ++p)
            asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(m.push_flag[p]), "l"(epoch) : "memory");
        }
      }
    }
  }
  TL(if (tid == 0) g_tlm[blockIdx.x * 8 + 4] = gtimer();)
  if (!epi_done && dense_here) {
    if (r1 == r0) dsc_load(0);  // (no fold chunk ran)
    window_epilogue();
  }
  TL(__syncthreads(); if (tid == 0) { g_tlm[blockIdx.x * 8 + 5] = gtimer(); atomicMax(&g_mend, gtimer()); })
  if (a.state) {
    // graph mode: advance the step state once every CTA has read it (the
    // last CTA to arrive moves dhi and the exchange epoch forward). Every
    // thread consumed its state loads at the top of the kernel, so the
    // arrival needs no fence; the next kernel reads the state after this
    // grid completes (griddepcontrol.wait), which orders the stores.
    __syncthreads();
    if (tid == 0) {
      unsigned long long* arrivals = reinterpret_cast<unsigned long long*>(a.state + 3);
      if (atomicAdd(arrivals, 1ull) == (unsigned long long)gridDim.x - 1) {
        *arrivals = 0;
        a.state[1] = sp.dhi + 1;
        a.state[2] = (int64_t)(epoch + 1);
      }
    }
  }
}

// ------------------------------------------------------------------ producer warp
// Warp-specialized decode CTAs pair every consumer warp with a producer warp
// that runs the consumer's work cursor and fills its S-stage ring: per stage
// the StageDesc + the 32 union entries, kv_in (written before its gather), 8
// tile::gather4 ops of whole K|V row pairs (L2 evict-first), and the item's
// query rows with the first stage of an item. The consumer only computes.
// (A producer costs ~1.1K cycles per stage -- 8 gather4 ops at ~70 cycles
// each plus the cursor, whose atomic and item-table reads are dependent
// global loads -- which used to sit on the fp32 kernel's critical path.)
//
// Producers run ahead of the programmatic-launch wait: in graph mode
// (a.state) a producer whose first item is a full sparse item (rebuild-time
// data only: item table, union entries, archive rows -- nothing the previous
// step's kernels write, and a graph replay starts after all earlier stream
// work) gathers that item's first stages -- its whole ring -- while the
// previous step's merge still runs; the item's queries, the work counter and everything that
// depends on the step's window wait for griddepcontrol.wait.
template <int D, int G, bool BF16, typename C>
__device__ __forceinline__ void decode_producer(const DecodeArgs& a, unsigned char* cw, int first_item, int nwarps,
                                                int lane) {
  constexpr int S = C::S;
  const uint32_t cw_u = smem_u32(cw);
  const unsigned char* Qg = reinterpret_cast<const unsigned char*>(a.q);
  StageDesc* cdesc = reinterpret_cast<StageDesc*>(cw + C::OFF_DESC);
  int32_t* cmeta = reinterpret_cast<int32_t*>(cw + C::OFF_META);
  uint64_t* cfull = reinterpret_cast<uint64_t*>(cw + C::OFF_FULL);
  uint64_t* cempty = reinterpret_cast<uint64_t*>(cw + C::OFF_EMPTY);
  // static first wave: this producer's first item is its consumer's global
  // index; later items come from the work counter (cursor_next_off)
  Cursor cur;
  cur.nxt = first_item;
  cur.item = -1;
  cur.row = cur.hi = cur.lo = cur.bk = cur.dense = 0;
  const uint64_t evict_first = l2_evict_first_policy();
  auto issue_gathers = [&](int s, const StageDesc& d, int32_t ent) {
    const int pos = ent & 0xffffff;
    const int rg = lane & 7;  // 4-row group of this lane's gather4 op
    const int rowbase = d.bk * (int)a.T;
    const int q0 = __shfl_sync(FULL, pos, rg * 4 + 0);
    const int q1 = __shfl_sync(FULL, pos, rg * 4 + 1);
    const int q2 = __shfl_sync(FULL, pos, rg * 4 + 2);
    const int q3 = __shfl_sync(FULL, pos, rg * 4 + 3);
    if (lane == 0) mbar_expect_tx(&cfull[s], C::STAGE + (d.first ? C::QB : 0));
    __syncwarp();
    if (lane < C::NOPS)
      tma_gather4_hint(cw_u + s * C::STAGE + rg * 4 * 2 * C::ROWB, &a.kmap, 0, rowbase + q0, rowbase + q1,
                       rowbase + q2, rowbase + q3, &cfull[s], evict_first);
  };
  auto issue_q = [&](int s, const StageDesc& d) {
    if (lane == 0 && d.first) {
      const int64_t b = d.bk / a.Hkv, kvh = d.bk % a.Hkv;
      bulk_g2s(cw + C::OFF_Q + s * C::QSLOT, Qg + (b * a.Hq + kvh * G) * (int64_t)C::ROWB, C::QB, &cfull[s]);
    }
  };
  int npre = 0;  // stages of the first item gathered before the wait (graph mode)
  StageDesc pend, first;
  int32_t pend_ent = 0;
  if (a.state) {
    StepPos sp0;  // only nf matters for a full sparse item
    sp0.nf = a.item_off[a.B * a.Hkv];
    sp0.nd = 0;
    if (first_item < sp0.nf) {
      cursor_item(cur, a, sp0, first_item);
      for (; npre < S && cur.row < cur.hi; ++npre) {  // fill the whole ring if the item is long enough
        pend = cursor_stage(cur);
        if (npre == 0) first = pend;
        pend_ent = lane < pend.n ? __ldg(a.u_ent + (int64_t)pend.bk * a.T + pend.r0 + lane) : 0;
        if (lane == 0) cdesc[npre] = pend;
        cmeta[npre * SUB + lane] = pend_ent;
        __syncwarp();  // desc/meta stores before lane 0's (release) arrive
        issue_gathers(npre, pend, pend_ent);
      }
    }
  }
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  const StepPos sp = step_pos(a);
  const int total = sp.nd + a.item_off[2 * a.B * a.Hkv + 1];
  if (npre) {
    issue_q(0, first);
#if HGCA_LAZY_CLAIM
    if (lane == 0) cur.nxt = -1;  // the next item is claimed when the prefetched one is fully issued
#else
    if (lane == 0) cur.nxt = atomicAdd(a.counter, 1) + nwarps;  // the prefetched item's deferred fetch
#endif
  }
  pend = cursor_next_off(cur, a, sp, total, lane, nwarps);  // (after prefetched stages: the next one)
  pend_ent = sub_entry<G>(pend, a, sp, lane);
  for (int k = npre;; ++k) {
    const int s = k % S;
    if (k >= S) mbar_wait(&cempty[s], ((k / S) - 1) & 1);
    const StageDesc d = pend;
    const int32_t ent = pend_ent;
    if (lane == 0) cdesc[s] = d;
    cmeta[s * SUB + lane] = ent;
    __syncwarp();  // desc/meta stores before lane 0's (release) arrive
    if (d.item < 0) {
      if (lane == 0) mbar_arrive(&cfull[s]);  // wake the consumer: no more work
      break;
    }
    write_new_row<D, BF16>(a, sp, d, lane);
    issue_gathers(s, d, ent);
    issue_q(s, d);
    pend = cursor_next_off(cur, a, sp, total, lane, nwarps);
    pend_ent = sub_entry<G>(pend, a, sp, lane);
  }
}

// =========================================================== bf16 (tensor-core) kernel
// Warp-specialized CTA: NC consumer warps, each with its own S-stage ring in
// shared memory, and NC producer warps, one per consumer, that run that
// consumer's work cursor and issue its TMA gathers, so the consumers only
// compute. (A producer costs ~1.1K cycles per stage -- 8 gather4 ops at ~70
// cycles each plus the cursor -- so sharing producers between consumers makes
// the producers the bottleneck; measured on B200.)
template <int D, int G, int S_, int NPAIR>
struct Bf16Cfg {
  static constexpr int S = S_;
  static constexpr int ROWB = D * 2;                    // bytes of one K (or V) row
  static constexpr int STAGE = SUB * 2 * ROWB;          // 32 rotated K|V row pairs
  static constexpr int NOPS = SUB / 4;                  // gather4 ops per stage (whole row pairs)
  static constexpr int QB = G * ROWB;                   // raw query block of one item
  static constexpr int QSLOT = (QB + 127) / 128 * 128;
  static constexpr int PT_LD = 40;                      // P^T staging row (floats), conflict-free
  static constexpr int OFF_Q = S * STAGE;
  static constexpr int OFF_PT = OFF_Q + S * QSLOT;
  static constexpr int OFF_META = OFF_PT + 8 * PT_LD * 4;
  static constexpr int OFF_DESC = OFF_META + S * SUB * 4;
  static constexpr int OFF_FULL = OFF_DESC + S * 32;    // mbarriers: stage landed (TMA tx)
  static constexpr int OFF_EMPTY = OFF_FULL + S * 8;    // mbarriers: stage consumed
  static constexpr int OFF_ST = OFF_EMPTY + S * 8;      // final (m, z) per head, fp64
  static constexpr int WARP_SMEM = (OFF_ST + 16 * 8 + 1023) / 1024 * 1024;
  static constexpr int NC0 = (SMEM_MAX - 1024) / WARP_SMEM;
  static constexpr int NC = NC0 > NPAIR ? NPAIR : NC0;  // consumer warps
  static constexpr int NW = 2 * NC;                     // + one producer warp per consumer
  static constexpr int SMEM = NC * WARP_SMEM + 1024;    // + alignment slack
  static_assert(NC >= 1, "bf16 decode pipeline does not fit shared memory");
  static_assert(G <= 8, "at most 8 query heads per kv head");
};

// swizzled byte offset of 16-byte chunk `ch` of row `r` inside a 32x128 B tile
__device__ __forceinline__ uint32_t swz128(int r, int ch) { return (uint32_t)(r * 128 + ((ch ^ (r & 7)) << 4)); }

// bf16 K|V rows are stored rotated by position (write_rows_kernel): 16-byte
// chunk c of the row pair of position p sits at chunk (c & ~7) | ((c ^ p) & 7),
// a permutation inside each 128-byte segment. Byte offset of logical chunk c
// of stage row r holding a position with p & 7 == rot:
template <int D>
__device__ __forceinline__ uint32_t rotoff(int r, int c, int rot) {
  return (uint32_t)(r * 4 * D + (((c & ~7) | ((c ^ rot) & 7)) << 4));
}

template <int D, int G, int S, int NPAIR>
__global__ void __launch_bounds__(Bf16Cfg<D, G, S, NPAIR>::NW * 32, 1)
    decode_bf16_kernel(const __grid_constant__ DecodeArgs a) {
  using C = Bf16Cfg<D, G, S, NPAIR>;
  constexpr int KC = D / 16;  // k16 chunks of the head dim (QK) == m16 tiles of the head dim (PV)
  extern __shared__ unsigned char sm_raw[];
  unsigned char* sm = smem_align1024(sm_raw);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp < C::NC) {  // each consumer warp initialises its own ring's barriers
    unsigned char* wsm = sm + warp * C::WARP_SMEM;
    if (lane < S) {
      mbar_init(reinterpret_cast<uint64_t*>(wsm + C::OFF_FULL) + lane, 1);
      mbar_init(reinterpret_cast<uint64_t*>(wsm + C::OFF_EMPTY) + lane, 1);
    }
    fence_mbar_init();
  }
  TL(const unsigned long long tl_entry = gtimer();)
  __syncthreads();
  if (warp >= C::NC) {  // producers: their own programmatic-launch wait (decode_producer)
    decode_producer<D, G, true, C>(a, sm + (warp - C::NC) * C::WARP_SMEM, (int)blockIdx.x * C::NC + (warp - C::NC),
                                   (int)gridDim.x * C::NC, lane);
    return;
  }
  // This grid may have been launched early behind the previous step's merge
  // (programmatic dependent launch): everything above overlapped its tail;
  // nothing the previous kernels wrote (step state, union lists, work counter,
  // queries, partial slots) is read or written before this wait.
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
  TL(if (threadIdx.x == 0) {
    g_gap[blockIdx.x * 4 + 0] = tl_entry; g_gap[blockIdx.x * 4 + 1] = gtimer();
    g_gap[blockIdx.x * 4 + 2] = *(volatile unsigned long long*)&g_mend;
  })
  // let the merge grid launch now: its CTAs take SMs as decode CTAs exit and
  // wait in griddepcontrol.wait until this whole grid has completed
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");

  // ================================================================== consumer
  unsigned char* wsm = sm + warp * C::WARP_SMEM;
  const uint32_t wsm_u = smem_u32(wsm);
  StageDesc* desc = reinterpret_cast<StageDesc*>(wsm + C::OFF_DESC);
  uint64_t* full = reinterpret_cast<uint64_t*>(wsm + C::OFF_FULL);
  uint64_t* empty = reinterpret_cast<uint64_t*>(wsm + C::OFF_EMPTY);
  int32_t* meta = reinterpret_cast<int32_t*>(wsm + C::OFF_META);
  float* pt = reinterpret_cast<float*>(wsm + C::OFF_PT);
  double* st = reinterpret_cast<double*>(wsm + C::OFF_ST);
  const int g4 = lane >> 2, t4 = lane & 3;      // mma groupID / thread-in-group
  const int hA = 2 * t4, hB = 2 * t4 + 1;       // query heads of this lane's fragment columns
  const float scale = (float)a.scale;
  TL(unsigned long long* tl = g_tl + ((int64_t)blockIdx.x * C::NC + warp) * TL_SLOTS;
     unsigned long long tl_merge = 0, tl_wait = 0, tl_sub = 0, tl_items = 0, tl_qk = 0, tl_pv = 0, tl_v = 0,
                        tl_issue = 0, tl_tma = 0, tl_nmerge = 0, tl_sm = 0, tl_epi = 0, tl_mask = 0,
                        tl_smax = 0, tl_end = 0;
     if (lane == 0) tl[0] = gtimer(););

  // per-item state (fragment layout: this lane owns heads hA, hB)
  uint32_t qf[KC][2];
  float acc[KC][4];
  float mA = -INFINITY, mB = -INFINITY, zA = 0.f, zB = 0.f;

  for (int k = 0;; ++k) {
    const int s = k % S;
    TL(long long c0 = clock64();)
    mbar_wait(&full[s], (k / S) & 1);
    const StageDesc d = desc[s];
    if (d.item < 0) break;
    TL(long long c1 = clock64(); tl_wait += c1 - c0; ++tl_sub;
       if (d.first && lane == 0) { tl[18] = gtimer(); tl[19] = (unsigned long long)d.item; })
#ifdef HGCA_NOCOMPUTE
    // experiment: data movement only (results are garbage)
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
    continue;
#endif
    const uint32_t stg = wsm_u + s * C::STAGE;
    if (d.first) {
      const uint32_t* qw = reinterpret_cast<const uint32_t*>(wsm + C::OFF_Q + s * C::QSLOT);
#pragma unroll
      for (int kc = 0; kc < KC; ++kc) {
        qf[kc][0] = g4 < G ? qw[g4 * (D / 2) + kc * 8 + t4] : 0u;
        qf[kc][1] = g4 < G ? qw[g4 * (D / 2) + kc * 8 + 4 + t4] : 0u;
      }
#pragma unroll
      for (int mt = 0; mt < KC; ++mt) acc[mt][0] = acc[mt][1] = acc[mt][2] = acc[mt][3] = 0.f;
      mA = mB = -INFINITY;
      zA = zB = 0.f;
    }
    TL(long long c2 = clock64(); tl_v += c2 - c1;)
    // ---- S = K Q^T: rows x heads, fp32 accumulate on the tensor cores.
    // ldmatrix row of this lane: K rows h*16 + (mi&1)*8 + (lane&7), k-half mi>>1
    const int mi = lane >> 3;
    float c[2][4];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      c[h][0] = c[h][1] = c[h][2] = c[h][3] = 0.f;
      const int r = h * 16 + (mi & 1) * 8 + (lane & 7);
      const int rot = meta[s * SUB + r] & 7;
#pragma unroll
      for (int kc = 0; kc < KC; ++kc) {
        uint32_t af[4];
        ldsm_x4(stg + rotoff<D>(r, 2 * kc + (mi >> 1), rot), af);
        mma_bf16(c[h], af, qf[kc][0], qf[kc][1]);
      }
    }
    TL(long long c2a = clock64(); tl_sm += c2a - c2;)
    // ---- scale + mask: value j of this lane is row j*8 + g4, heads hA / hB
    float sA[4], sB[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int row = j * 8 + g4;
      const uint32_t qm = (uint32_t)meta[s * SUB + row] >> 24;
      const bool ok = row < d.n;
      const float va = c[j >> 1][(j & 1) * 2 + 0] * scale;
      const float vb = c[j >> 1][(j & 1) * 2 + 1] * scale;
      sA[j] = (ok && hA < G && ((qm >> hA) & 1u)) ? va : -INFINITY;
      sB[j] = (ok && hB < G && ((qm >> hB) & 1u)) ? vb : -INFINITY;
      if (d.dense && ok) {
        float* dsc = reinterpret_cast<float*>(a.dsc);
        const int64_t bq0 = (int64_t)(d.bk / a.Hkv) * a.Hq + (d.bk % a.Hkv) * G;
        if (hA < G) dsc[(bq0 + hA) * a.dsc_ld + d.r0 + row] = va;
        if (hB < G) dsc[(bq0 + hB) * a.dsc_ld + d.r0 + row] = vb;
      }
    }
    TL(long long c2b = clock64(); tl_mask += c2b - c2a;)
    // ---- online softmax (fp32) per head, reduced over the 8 lanes sharing t4
    float xA = fmaxf(fmaxf(sA[0], sA[1]), fmaxf(sA[2], sA[3]));
    float xB = fmaxf(fmaxf(sB[0], sB[1]), fmaxf(sB[2], sB[3]));
#pragma unroll
    for (int o = 4; o < 32; o <<= 1) {
      xA = fmaxf(xA, __shfl_xor_sync(FULL, xA, o));
      xB = fmaxf(xB, __shfl_xor_sync(FULL, xB, o));
    }
    const float nA = fmaxf(mA, xA), nB = fmaxf(mB, xB);
    const float alA = nA == -INFINITY ? 1.f : __expf(mA - nA);
    const float alB = nB == -INFINITY ? 1.f : __expf(mB - nB);
    float pA[4], pB[4], sumA = 0.f, sumB = 0.f;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      pA[j] = sA[j] == -INFINITY ? 0.f : __expf(sA[j] - nA);
      pB[j] = sB[j] == -INFINITY ? 0.f : __expf(sB[j] - nB);
      sumA += pA[j];
      sumB += pB[j];
    }
#pragma unroll
    for (int o = 4; o < 32; o <<= 1) {
      sumA += __shfl_xor_sync(FULL, sumA, o);
      sumB += __shfl_xor_sync(FULL, sumB, o);
    }
    zA = zA * alA + sumA;
    zB = zB * alB + sumB;
    mA = nA;
    mB = nB;
    if (__any_sync(FULL, alA != 1.f || alB != 1.f)) {
#pragma unroll
      for (int mt = 0; mt < KC; ++mt) {
        acc[mt][0] *= alA; acc[mt][1] *= alB; acc[mt][2] *= alA; acc[mt][3] *= alB;
      }
    }
    TL(long long c2c = clock64(); tl_smax += c2c - c2b;)
    // ---- P^T to shared memory (rows x heads -> heads x rows)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int row = j * 8 + g4;
      if (hA < G) pt[hA * C::PT_LD + row] = pA[j];
      if (hB < G) pt[hB * C::PT_LD + row] = pB[j];
    }
    __syncwarp();
    TL(long long c3 = clock64(); tl_qk += c3 - c2;)
    // ---- O^T += V^T P^T: dims x heads; P = hi + lo in bf16
#pragma unroll
    for (int kk = 0; kk < 2; ++kk) {
      uint32_t bh0 = 0, bh1 = 0, bl0 = 0, bl1 = 0;
      if (g4 < G) {
        const float2 p01 = *reinterpret_cast<const float2*>(pt + g4 * C::PT_LD + kk * 16 + 2 * t4);
        const float2 p89 = *reinterpret_cast<const float2*>(pt + g4 * C::PT_LD + kk * 16 + 8 + 2 * t4);
        bh0 = pack_bf16(p01.x, p01.y);
        bh1 = pack_bf16(p89.x, p89.y);
        bl0 = pack_bf16(p01.x - bf16_lo_f(bh0), p01.y - bf16_hi_f(bh0));
        bl1 = pack_bf16(p89.x - bf16_lo_f(bh1), p89.y - bf16_hi_f(bh1));
      }
      // ldmatrix.trans row of this lane: V rows kk*16 + (mi>>1)*8 + (lane&7), dim-half mi&1
      const int r = kk * 16 + (mi >> 1) * 8 + (lane & 7);
      const int rot = meta[s * SUB + r] & 7;
#pragma unroll
      for (int mt = 0; mt < KC; ++mt) {
        uint32_t af[4];
        ldsm_x4_t(stg + rotoff<D>(r, D / 8 + mt * 2 + (mi & 1), rot), af);
        mma_bf16(acc[mt], af, bh0, bh1);
        mma_bf16(acc[mt], af, bl0, bl1);
      }
    }
    TL(long long c4 = clock64(); tl_pv += c4 - c3;)
    TL(long long c4b = clock64();)
    if (d.last) {
      TL(++tl_items;)
      // partial (m, z, acc) of this item; acc[mt][j] = O[head hA|hB][dim mt*16 + g4 (+8)]
      // (head-major partials: head h of item i at h * MI + i)
      const int64_t iA = hA * a.m.MI + d.item, iB = hB * a.m.MI + d.item;
      if (lane < 4) {
        if (hA < G) { a.part_m[iA] = mA; a.part_z[iA] = zA; }
        if (hB < G) { a.part_m[iB] = mB; a.part_z[iB] = zB; }
      }
      float* paA = a.part_acc + iA * D;
      float* paB = a.part_acc + iB * D;
#pragma unroll
      for (int mt = 0; mt < KC; ++mt) {
        if (hA < G) { paA[mt * 16 + g4] = acc[mt][0]; paA[mt * 16 + 8 + g4] = acc[mt][2]; }
        if (hB < G) { paB[mt * 16 + g4] = acc[mt][1]; paB[mt * 16 + 8 + g4] = acc[mt][3]; }
      }
    }
    __syncwarp();
    TL(long long c5 = clock64(); tl_end += c5 - c4b;)
    if (lane == 0) mbar_arrive(&empty[s]);  // stage consumed: the producer may refill it
  }
  TL(if (lane == 0) {
    tl[1] = gtimer(); tl[17] = tl[1];
    tl[2] = tl_merge; tl[3] = tl_wait; tl[4] = tl_sub; tl[5] = tl_items; tl[6] = tl_qk; tl[7] = tl_pv;
    tl[8] = tl_v; tl[9] = tl_issue; tl[10] = tl_tma; tl[11] = tl_mask; tl[12] = tl_sm; tl[13] = tl_epi;
    tl[14] = tl_smax; tl[15] = tl_end; tl[16] = blockIdx.x;
  })
}

// =========================================================== fp32 (reference-exact) kernel
// Warp-specialized like the bf16 kernel: NC consumer warps, each with its own
// S-stage ring, and NC producer warps (decode_producer) that run the
// consumers' cursors and issue their gathers, so the dependent global loads of
// the cursor (work-counter atomic, item table, union entries) and the TMA
// issue stay off the consumer's per-stage critical path (a self-issuing warp
// spent ~2.1K of ~6.8K cycles per stage there at C1).
// fp32 K|V rows are stored position-rotated like the bf16 ones (16-byte chunk
// c of position p at (c & ~7) | ((c ^ p) & 7)), so one tile::gather4 op moves
// four whole 2*D*4-byte row pairs (8 ops per 32-row stage) and both compute
// phases read shared memory without bank conflicts: the score phase (lane =
// row, 16-byte chunks, rows of a quarter-warp in distinct p & 7 classes) and
// P.V (lanes = head dims of one row).
template <int D, int G>
struct F32Cfg {
  static constexpr int ROWB = D * 4;                    // bytes of one K (or V) row
  static constexpr int PAIR = 2 * ROWB;                 // one rotated K|V row pair
  static constexpr int DPL = D / 32;                    // head dims per lane in P.V
  static constexpr int S = HGCA_F32_STAGES;
  static constexpr int STAGE = SUB * PAIR;
  static constexpr int NOPS = SUB / 4;                  // gather4 ops per stage
  static constexpr int QB = G * ROWB;
  static constexpr int QSLOT = QB;                      // (a multiple of 128 bytes)
  static constexpr int OFF_Q = S * STAGE;                   // raw queries [S][G][D] f32
  static constexpr int OFF_QK = OFF_Q + S * QSLOT;          // queries [G][D] fp64
  static constexpr int OFF_ACC = OFF_QK + G * D * 8;        // P.V accumulators [G][D] fp32
  static constexpr int OFF_PF = OFF_ACC + G * D * 4;        // this stage's fp32 weights [32] (P.V broadcast)
  static constexpr int OFF_META = OFF_PF + SUB * 4;         // entries [S][32]
  static constexpr int OFF_DESC = OFF_META + S * SUB * 4;
  static constexpr int OFF_FULL = OFF_DESC + S * 32;        // mbarriers: stage landed (TMA tx)
  static constexpr int OFF_EMPTY = OFF_FULL + S * 8;        // mbarriers: stage consumed
  static constexpr int WARP_SMEM = (OFF_EMPTY + S * 8 + 127) / 128 * 128;
  static constexpr int NC0 = (SMEM_MAX - 1024) / WARP_SMEM;
  static constexpr int NC = NC0 > HGCA_F32_NC ? HGCA_F32_NC : NC0;  // consumer warps
  static constexpr int NW = 2 * NC;                     // + one producer warp per consumer
  static constexpr int SMEM = NC * WARP_SMEM + 1024;
  static_assert(NC >= 1, "fp32 decode pipeline does not fit shared memory");
  static_assert(D == 64 || D == 128, "fp32 decode: head_dim 64 or 128");
  static_assert(QB % 128 == 0, "query slot alignment");
};

template <int D, int G>
__global__ void __launch_bounds__(F32Cfg<D, G>::NW * 32, 1) decode_f32_kernel(const __grid_constant__ DecodeArgs a) {
  using C = F32Cfg<D, G>;
  extern __shared__ unsigned char sm_raw[];
  unsigned char* sm = smem_align1024(sm_raw);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp < C::NC) {  // each consumer warp initialises its own ring's barriers
    unsigned char* wsm = sm + warp * C::WARP_SMEM;
    if (lane < C::S) {
      mbar_init(reinterpret_cast<uint64_t*>(wsm + C::OFF_FULL) + lane, 1);
      mbar_init(reinterpret_cast<uint64_t*>(wsm + C::OFF_EMPTY) + lane, 1);
    }
    fence_mbar_init();
  }
  TL(const unsigned long long tl_entry = gtimer();)
  __syncthreads();
  if (warp >= C::NC) {  // producers: their own programmatic-launch wait (decode_producer)
    decode_producer<D, G, false, C>(a, sm + (warp - C::NC) * C::WARP_SMEM, (int)blockIdx.x * C::NC + (warp - C::NC),
                                    (int)gridDim.x * C::NC, lane);
    return;
  }
  asm volatile("griddepcontrol.wait;\n" ::: "memory");               // see decode_bf16_kernel
  TL(if (threadIdx.x == 0) {
    g_gap[blockIdx.x * 4 + 0] = tl_entry; g_gap[blockIdx.x * 4 + 1] = gtimer();
    g_gap[blockIdx.x * 4 + 2] = *(volatile unsigned long long*)&g_mend;
  })
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");

  // ================================================================== consumer
  unsigned char* wsm = sm + warp * C::WARP_SMEM;
  StageDesc* desc = reinterpret_cast<StageDesc*>(wsm + C::OFF_DESC);
  uint64_t* full = reinterpret_cast<uint64_t*>(wsm + C::OFF_FULL);
  uint64_t* empty = reinterpret_cast<uint64_t*>(wsm + C::OFF_EMPTY);
  int32_t* meta = reinterpret_cast<int32_t*>(wsm + C::OFF_META);
  double* qk = reinterpret_cast<double*>(wsm + C::OFF_QK);
  float* accs = reinterpret_cast<float*>(wsm + C::OFF_ACC);
  TL(unsigned long long* tl = g_tl + ((int64_t)blockIdx.x * C::NC + warp) * TL_SLOTS;
     unsigned long long tl_wait = 0, tl_score = 0, tl_pv = 0, tl_issue = 0, tl_part = 0, tl_sub = 0, tl_items = 0,
                        tl_first = 0;
     if (lane == 0) tl[0] = gtimer(););

  double m_run[G], z_run[G];  // running (m, z) of the current item, per head (warp-uniform)
  for (int k = 0;; ++k) {
    const int s = k % C::S;
    TL(long long c0 = clock64();)
    mbar_wait(&full[s], (k / C::S) & 1);
    const StageDesc d = desc[s];
    if (d.item < 0) break;
    TL(long long c1 = clock64(); tl_wait += c1 - c0; ++tl_sub; if (!tl_first) tl_first = gtimer();)
    const unsigned char* st = wsm + s * C::STAGE;
    const int32_t myent = meta[s * SUB + lane];
    const uint32_t qm = (uint32_t)myent >> 24;
    const uint32_t wq = G == 1 ? 1u : __reduce_or_sync(FULL, qm);
    const int myrot = myent & 7;
    if (d.first) {
      const float* qr = reinterpret_cast<const float*>(wsm + C::OFF_Q + s * C::QSLOT);
      for (int t = lane; t < G * D; t += 32) qk[t] = (double)qr[t];
      for (int t = lane; t < G * D; t += 32) accs[t] = 0.f;
#pragma unroll
      for (int g = 0; g < G; ++g) {
        m_run[g] = -INFINITY;
        z_run[g] = 0.0;
      }
      __syncwarp();
    }
    // ---- scores: lane = row, exact fp64 products summed in the reference's
    // sequential order over the head dimension (_core.pyx:59-65)
    double sacc[G];
#pragma unroll
    for (int g = 0; g < G; ++g) sacc[g] = 0.0;
    {
      // batches of 16 elements: the 16 loads and fp32 -> fp64 conversions are
      // issued ahead of the batch's dependent DFMA chain (the chain is what
      // bounds a stage)
      const unsigned char* kr = st + lane * C::PAIR;
#pragma unroll 2
      for (int c0 = 0; c0 < D / 4; c0 += 4) {
        float4 kv[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int c = c0 + u;
          kv[u] = *reinterpret_cast<const float4*>(kr + (((c & ~7) | ((c ^ myrot) & 7)) << 4));
        }
        double kd[16];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          kd[4 * u + 0] = (double)kv[u].x;
          kd[4 * u + 1] = (double)kv[u].y;
          kd[4 * u + 2] = (double)kv[u].z;
          kd[4 * u + 3] = (double)kv[u].w;
        }
#pragma unroll
        for (int g = 0; g < G; ++g) {
          if (G == 1 || ((wq >> g) & 1u)) {
            const double* qg = qk + g * D + c0 * 4;
#pragma unroll
            for (int e = 0; e < 16; e += 2) {
              const double2 qq = *reinterpret_cast<const double2*>(qg + e);
              sacc[g] = fma(qq.x, kd[e], sacc[g]);  // exact products: one rounding per add
              sacc[g] = fma(qq.y, kd[e + 1], sacc[g]);
            }
          }
        }
      }
    }
    const int64_t b = d.bk / a.Hkv, kvh = d.bk % a.Hkv;
    TL(long long c2 = clock64(); tl_score += c2 - c1;)
    // ---- per active head: online softmax (fp64 exp, the weights the MAW
    // needs) and P.V in fp32 with lanes over head dims
#pragma unroll
    for (int g = 0; g < G; ++g) {
      if (G > 1 && !((wq >> g) & 1u)) continue;
      const double sv = (lane < d.n && ((qm >> g) & 1u)) ? sacc[g] * a.scale : -INFINITY;
      if (d.dense && lane < d.n)
        reinterpret_cast<double*>(a.dsc)[(b * a.Hq + kvh * G + g) * a.dsc_ld + d.r0 + lane] = sv;
      const double cm = warp_max_f64(sv);
      const double mold = m_run[g], mnew = fmax(mold, cm);
      if (mnew == -INFINITY) continue;
      // exp(0) = 1 and exp(-inf) = 0 exactly: skip the fp64 exp when the max
      // did not move or this is the item's first stage (the common case)
      const double scal = mold == -INFINITY ? 0.0 : (mold == mnew ? 1.0 : exp(mold - mnew));
      const double p = sv == -INFINITY ? 0.0 : exp(sv - mnew);
      z_run[g] = z_run[g] * scal + warp_sum_f64(p);
      m_run[g] = mnew;
      float* pfs = reinterpret_cast<float*>(wsm + C::OFF_PF);
      pfs[lane] = (float)p;  // the stage's weights, broadcast to every lane below
      const float sf = (float)scal;
      float acc[C::DPL];
      float* ag = accs + g * D + lane * C::DPL;
#pragma unroll
      for (int i = 0; i < C::DPL; ++i) acc[i] = mold == -INFINITY ? 0.f : ag[i] * sf;
      __syncwarp();
      // V chunk of this lane's dims; 16-byte chunk index inside the row pair
      constexpr int VC0 = D / 4;
      const int vc = VC0 + lane * C::DPL / 4, vo = (lane * C::DPL) % 4;
#pragma unroll 2
      for (int r4 = 0; r4 < SUB; r4 += 4) {
        const float4 p4 = *reinterpret_cast<const float4*>(pfs + r4);  // 4 weights, 4 row rotations per load
        const int4 m4 = *reinterpret_cast<const int4*>(meta + s * SUB + r4);
        const float pr4[4] = {p4.x, p4.y, p4.z, p4.w};
        const int rr4[4] = {m4.x & 7, m4.y & 7, m4.z & 7, m4.w & 7};
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const float pr = pr4[u];
          const float* vr =
              reinterpret_cast<const float*>(st + (r4 + u) * C::PAIR + (((vc & ~7) | ((vc ^ rr4[u]) & 7)) << 4)) + vo;
          if constexpr (C::DPL == 4) {
            const float4 v = *reinterpret_cast<const float4*>(vr);
            acc[0] = fmaf(pr, v.x, acc[0]); acc[1] = fmaf(pr, v.y, acc[1]);
            acc[2] = fmaf(pr, v.z, acc[2]); acc[3] = fmaf(pr, v.w, acc[3]);
          } else {
            const float2 v = *reinterpret_cast<const float2*>(vr);
            acc[0] = fmaf(pr, v.x, acc[0]); acc[1] = fmaf(pr, v.y, acc[1]);
          }
        }
      }
      __syncwarp();  // pfs is rewritten by the next head / stage
#pragma unroll
      for (int i = 0; i < C::DPL; ++i) ag[i] = acc[i];
    }
    TL(long long c3 = clock64(); tl_pv += c3 - c2;)
    __syncwarp();  // every lane's reads of the stage are done
    if (lane == 0) mbar_arrive(&empty[s]);  // the producer may refill it
    if (d.last) {
      TL(++tl_items;)
      for (int t = lane; t < G * D; t += 32) a.part_acc[((t / D) * a.m.MI + d.item) * D + t % D] = accs[t];
      if (lane == 0) {
#pragma unroll
        for (int g = 0; g < G; ++g) {
          a.part_m[g * a.m.MI + d.item] = m_run[g];
          a.part_z[g * a.m.MI + d.item] = z_run[g];
        }
      }
    }
    __syncwarp();
    TL(long long c4 = clock64(); tl_part += c4 - c3;)
  }
  TL(if (lane == 0) {
    tl[1] = gtimer(); tl[2] = tl_sub; tl[3] = tl_wait; tl[4] = tl_score; tl[5] = tl_pv; tl[6] = tl_issue;
    tl[7] = tl_part; tl[8] = tl_first; tl[9] = tl_items; tl[16] = blockIdx.x;
  })
}

// -------------------------------------------------------------- union build
// Per (batch, kv-head): union of the G query heads' selection masks over the
// archive [0, n_arch) as packed entries pos | (query-head mask << 24).
// grouped = 1 orders them by mask value, then position (the fp32 kernel then
// sees mostly single-head sub-chunks); grouped = 0 keeps position order (the
// bf16 kernel computes every head of a row anyway, and position order keeps
// neighbouring rows close in HBM).
__global__ void __launch_bounds__(1024) union_build_kernel(const uint32_t* __restrict__ sel, int64_t Hq, int64_t Hkv,
                                                           int64_t G, int64_t words, int64_t n_arch, int64_t T,
                                                           int32_t* u_ent, int32_t* u_cnt, int grouped) {
  __shared__ unsigned int hist[256];
  __shared__ int wsum[32];
  __shared__ int base_s;
  const int64_t bk = blockIdx.x;
  const int64_t b = bk / Hkv, kvh = bk % Hkv;
  const uint32_t* m0 = sel + (b * Hq + kvh * G) * words;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nwarp = blockDim.x >> 5;
  const int64_t nw = (n_arch + 31) >> 5;
  for (int i = tid; i < 256; i += blockDim.x) hist[i] = 0;
  __syncthreads();
  auto word_masks = [&](int64_t w, uint32_t* mg) -> uint32_t {
    uint32_t any = 0;
    const int64_t rem = n_arch - (w << 5);
    const uint32_t keep = rem >= 32 ? 0xffffffffu : ((1u << rem) - 1u);
    for (int g = 0; g < G; ++g) {
      mg[g] = m0[g * words + w] & keep;
      any |= mg[g];
    }
    return any;
  };
  if (grouped) {
    for (int64_t w = tid; w < nw; w += blockDim.x) {
      uint32_t mg[8];
      uint32_t any = word_masks(w, mg);
      while (any) {
        const int bit = __ffs(any) - 1;
        any &= any - 1;
        uint32_t qm = 0;
        for (int g = 0; g < G; ++g) qm |= ((mg[g] >> bit) & 1u) << g;
        atomicAdd(&hist[qm], 1u);
      }
    }
  }
  __syncthreads();
  if (tid == 0) base_s = 0;
  __syncthreads();
  const int64_t per = (nw + blockDim.x - 1) / blockDim.x;
  if (!grouped && per <= 8) {
    // position order, every word of the list in one pass: thread t owns words
    // [t * per, (t + 1) * per) (all loads in flight at once), one block scan of
    // the per-thread counts, then the thread writes its entries in order (the
    // masks re-read from cache). The chunked loop below needs nw / 1024 rounds of
    // load -> scan -> write latency.
    int c = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int64_t w = tid * per + k;
      if (k < per && w < nw) {
        uint32_t mg[8];
        c += __popc(word_masks(w, mg));
      }
    }
    int incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane == 31) wsum[wid] = incl;
    __syncthreads();
    if (wid == 0) {
      int x = lane < nwarp ? wsum[lane] : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      if (lane < nwarp) wsum[lane] = x;
    }
    __syncthreads();
    int pos = (wid ? wsum[wid - 1] : 0) + (incl - c);
    int32_t* out = u_ent + bk * T;
    for (int k = 0; k < per; ++k) {
      const int64_t w = tid * per + k;
      if (w >= nw) break;
      uint32_t mg[8];
      uint32_t hit = word_masks(w, mg);
      const uint32_t wbase = (uint32_t)(w << 5);
      while (hit) {
        const int bit = __ffs(hit) - 1;
        hit &= hit - 1;
        uint32_t qm = 0;
#pragma unroll
        for (int g = 0; g < 8; ++g)
          if (g < G) qm |= ((mg[g] >> bit) & 1u) << g;
        out[pos++] = (int32_t)((wbase + bit) | (qm << 24));
      }
    }
    if (tid == 0) u_cnt[bk] = wsum[nwarp - 1];
    return;
  }
  const int nbins = grouped ? (1 << G) : 2;
  for (int v = 1; v < nbins; ++v) {
    if (grouped && hist[v] == 0) continue;  // uniform: hist is stable after the barrier
    for (int64_t w0 = 0; w0 < nw; w0 += blockDim.x) {
      const int64_t w = w0 + tid;
      uint32_t hit = 0;
      uint32_t mg[8];
      if (w < nw) {
        uint32_t any = word_masks(w, mg);
        if (!grouped) {
          hit = any;
        } else {
          while (any) {
            const int bit = __ffs(any) - 1;
            any &= any - 1;
            uint32_t qm = 0;
            for (int g = 0; g < G; ++g) qm |= ((mg[g] >> bit) & 1u) << g;
            if (qm == (uint32_t)v) hit |= 1u << bit;
          }
        }
      }
      const int c = __popc(hit);
      int incl = c;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      if (lane == 31) wsum[wid] = incl;
      __syncthreads();
      if (wid == 0) {
        int x = lane < nwarp ? wsum[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int y = __shfl_up_sync(0xffffffffu, x, o);
          if (lane >= o) x += y;
        }
        if (lane < nwarp) wsum[lane] = x;
      }
      __syncthreads();
      int pos = base_s + (wid ? wsum[wid - 1] : 0) + (incl - c);
      while (hit) {
        const int bit = __ffs(hit) - 1;
        hit &= hit - 1;
        uint32_t qm = 0;
        for (int g = 0; g < G; ++g) qm |= ((mg[g] >> bit) & 1u) << g;
        u_ent[bk * T + pos] = (int32_t)((uint32_t)((w << 5) + bit) | (qm << 24));
        ++pos;
      }
      __syncthreads();
      if (tid == 0) base_s += wsum[nwarp - 1];
      __syncthreads();
    }
  }
  if (tid == 0) u_cnt[bk] = base_s;
}

// Union for the bf16 kernel (mode 2): position order (union_build_kernel,
// grouped = 0), then each aligned window of 32 entries -- one decode stage --
// is permuted to (rank within position class, class) order, class = p & 7. The
// bf16 K|V rows are stored rotated by p & 7, so an aligned group of 8 entries
// with 8 distinct classes puts the 8 rows one ldmatrix reads in 8 different
// bank groups; keeping the permutation inside a stage keeps the stage's rows
// as close in HBM as plain position order (interleaving classes over the
// whole list let the j-th entries of different classes drift apart: 2.3%
// slower on C2). One warp per window; keys (rank, class) are unique, the slot
// is the number of smaller keys. Grid (B * Hkv, windows / 32): every window of
// every list is independent, so the whole GPU takes them (one CTA per list
// left ~4/5 of the SMs idle at C3).
__global__ void __launch_bounds__(1024) union_window_classes_kernel(int32_t* u_ent, const int32_t* u_cnt, int64_t T) {
  const int64_t bk = blockIdx.x;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
  const int cnt = u_cnt[bk];
  int32_t* ent = u_ent + bk * T;
  const int w_first = (int)(blockIdx.y * nwarp + wid) * 32;
  for (int w0 = w_first; w0 < cnt; w0 += (int)gridDim.y * nwarp * 32) {
    const int n = min(32, cnt - w0);
    const bool ok = lane < n;
    const int32_t e = ok ? ent[w0 + lane] : 0;
    const int cls = ok ? (e & 7) : 8;  // positions are the low 24 bits; p & 7 = e & 7
    // slot = number of entries with a smaller (rank, class) key: those of a lower
    // rank in any class (min(count_c, rank) per class) plus those of the same
    // rank in a lower class (count_c > rank)
    int rank = 0, slot = 0;
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const uint32_t m = __ballot_sync(FULL, cls == c);
      if (cls == c) rank = __popc(m & ((1u << lane) - 1u));
    }
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const int cnt_c = __popc(__ballot_sync(FULL, cls == c));
      slot += min(cnt_c, rank) + ((c < cls && cnt_c > rank) ? 1 : 0);
    }
    __syncwarp();
    if (ok) ent[w0 + slot] = e;
  }
}

// Sparse work items. Each (b, kv-head) union list [0, u_cnt) is cut into
// full items of `rows` entries over [0, big) and tail items of rows/4 entries
// over [big, u_cnt), big = rows * floor((u_cnt - u_cnt/TAIL_DIV) / rows): the
// last >= 1/TAIL_DIV of every list is small items. Item ids: all full items
// (bk order), then all tail items (bk order), so once the queue reaches the
// tail every warp picks up short items and the warps finish together (the
// tail must hold more work than one full item per warp).
// item_off [2][BK+1]: row 0 = full-item prefix (row 0 [BK] = number of full
// items), row 1 = absolute start of each bk's tail items (row 1 [BK] = total).
#ifndef HGCA_TAIL_DIV
#define HGCA_TAIL_DIV 12  // with lazy claims a twelfth of each list suffices (6 before: round-2 A/B)
#endif
#ifndef HGCA_TAIL_SPLIT
#define HGCA_TAIL_SPLIT 4
#endif
constexpr int TAIL_DIV = HGCA_TAIL_DIV;      // the last >= 1/TAIL_DIV of each list is tail items
constexpr int TAIL_SPLIT = HGCA_TAIL_SPLIT;  // of rows / TAIL_SPLIT entries each
// the host's item capacities (hgca_decode_step, sparse_capacity) assume tail
// items of >= rows / 4 entries, and rows >= 16 keeps them >= 4 entries
static_assert(TAIL_SPLIT >= 1 && TAIL_SPLIT <= 4, "tail items must hold >= rows / 4 entries");
static_assert(TAIL_DIV >= 2, "the tail is at most half of a list");
// tail items hold rows / TAIL_SPLIT entries, but never less than one 32-row
// stage: the short items of small steps (adaptive rows 32-128) would otherwise
// be partial stages whose per-item cost (q load, partial write, merge fold)
// buys no balance
__device__ __forceinline__ int64_t tail_rows(int64_t rows) {
  const int64_t t = rows / TAIL_SPLIT;
  return t >= SUB ? t : (rows < SUB ? rows : SUB);
}
__device__ __forceinline__ void item_counts(int64_t cnt, int64_t rows, int& nbig, int& nsmall) {
  const int64_t big = (cnt - cnt / TAIL_DIV) / rows * rows;
  const int64_t small = tail_rows(rows);
  nbig = (int)(big / rows);
  nsmall = (int)((cnt - big + small - 1) / small);
}

// Item granularity adapts to the step (off[2*(BK+1)] = rows chosen): the
// largest power-of-two fraction of max_rows, not below min_rows, that still
// yields >= target items over the union -- big steps keep long items (few
// partials to fold), small steps get enough items for every warp.
__global__ void item_offsets_kernel(const int32_t* u_cnt, int64_t BK, int64_t max_rows, int64_t min_rows,
                                    int64_t target, int64_t window_rows, int32_t* off) {
  __shared__ int32_t carry[2];
  __shared__ int wsum[2][32];
  __shared__ long long utot;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nwarp = blockDim.x >> 5;
  // the step's work = the unions + the dense windows (window parts use the
  // same granularity), so a big window with a small union keeps long items
  if (tid == 0) utot = (long long)BK * window_rows;
  __syncthreads();
  {
    long long u = 0;
    for (int64_t x = tid; x < BK; x += blockDim.x) u += u_cnt[x];
    for (int o = 16; o; o >>= 1) u += __shfl_xor_sync(0xffffffffu, u, o);
    if (lane == 0) atomicAdd(reinterpret_cast<unsigned long long*>(&utot), (unsigned long long)u);
  }
  if (tid < 2) carry[tid] = 0;
  __syncthreads();
  int64_t rows = max_rows;
  while (rows / 2 >= min_rows && utot < rows * target) rows /= 2;
  if (tid == 0) off[2 * (BK + 1)] = (int32_t)rows;
  for (int pass = 0; pass < 2; ++pass) {
    for (int64_t x0 = 0; x0 < BK; x0 += blockDim.x) {
      const int64_t x = x0 + tid;
      int nb = 0, ns = 0;
      if (x < BK) item_counts(u_cnt[x], rows, nb, ns);
      const int c = pass == 0 ? nb : ns;
      int incl = c;
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      if (lane == 31) wsum[pass][wid] = incl;
      __syncthreads();
      if (wid == 0) {
        int v = lane < nwarp ? wsum[pass][lane] : 0;
        for (int o = 1; o < 32; o <<= 1) {
          const int y = __shfl_up_sync(0xffffffffu, v, o);
          if (lane >= o) v += y;
        }
        if (lane < nwarp) wsum[pass][lane] = v;
      }
      __syncthreads();
      if (x < BK) off[pass * (BK + 1) + x] = carry[pass] + (wid ? wsum[pass][wid - 1] : 0) + (incl - c);
      __syncthreads();
      if (tid == 0) carry[pass] += wsum[pass][nwarp - 1];
      __syncthreads();
    }
    if (tid == 0) {
      off[pass * (BK + 1) + BK] = carry[pass];
      if (pass == 0) carry[1] = carry[0];  // tail items follow all full items
    }
    __syncthreads();
  }
}

// item_tab[id] = (bk, lo, hi, 0) for the full and tail items of bk
__global__ void item_table_kernel(const int32_t* u_cnt, const int32_t* off, int64_t BK, int4* tab) {
  const int64_t bk = blockIdx.x;
  if (bk >= BK) return;
  const int64_t rows = off[2 * (BK + 1)];
  int nb = 0, ns = 0;
  item_counts(u_cnt[bk], rows, nb, ns);
  const int cnt = u_cnt[bk], small = (int)tail_rows(rows), big = nb * (int)rows;
  for (int i = threadIdx.x; i < nb; i += blockDim.x)
    tab[off[bk] + i] = make_int4((int)bk, i * (int)rows, (i + 1) * (int)rows, 0);
  for (int i = threadIdx.x; i < ns; i += blockDim.x)
    tab[off[BK + 1 + bk] + i] = make_int4((int)bk, big + i * small, min(cnt, big + (i + 1) * small), 0);
}

// KV[bh, pos + i, 0, :] = k_new[bh, i, :], KV[bh, pos + i, 1, :] = v_new[bh, i, :];
// rot = 1 (bf16 storage) stores 16-byte chunk c of the row pair at
// (c & ~7) | ((c ^ position) & 7) -- see rotoff().
__global__ void write_rows_kernel(unsigned char* KV, int64_t BH, int64_t T, int64_t rowb, int64_t pos,
                                  const unsigned char* kn, const unsigned char* vn, int64_t n, int rot) {
  const int64_t pieces = rowb / 16;
  const int64_t total = BH * n * pieces;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = t % pieces, row = t / pieces;
    const int64_t bh = row / n, i = row % n;
    const int64_t position = pos + i;
    const int64_t kc = p, vc = pieces + p;
    const int64_t kp = rot ? ((kc & ~7) | ((kc ^ position) & 7)) : kc;
    const int64_t vp = rot ? ((vc & ~7) | ((vc ^ position) & 7)) : vc;
    const int64_t base = (bh * T + position) * 2 * rowb;
    const int64_t src = (bh * n + i) * rowb + p * 16;
    *reinterpret_cast<uint4*>(KV + base + kp * 16) = *reinterpret_cast<const uint4*>(kn + src);
    *reinterpret_cast<uint4*>(KV + base + vp * 16) = *reinterpret_cast<const uint4*>(vn + src);
  }
}

// ------------------------------------------------------------------ launchers
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

// 2-D tensor map over KV viewed as [rows = B*Hkv*T, 2*D elements] for
// tile::gather4: box = one whole (rotated) K|V row pair, no swizzle -- TMA
// gather cost is per gathered row, so whole rows keep it at 8 ops per 32-row
// stage (both storage dtypes).
static int make_row_map(CUtensorMap* map, const void* base, int64_t rows, int64_t D, bool bf16) {
  static EncodeTiledFn encode = nullptr;
  if (!encode) {
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&encode, cudaEnableDefault, &q) != cudaSuccess ||
        !encode)
      return -3000;
  }
  const int esz = bf16 ? 2 : 4;
  cuuint64_t gdim[2] = {(cuuint64_t)(2 * D), (cuuint64_t)rows};
  cuuint64_t gstr[1] = {(cuuint64_t)(2 * D * esz)};
  cuuint32_t box[2] = {(cuuint32_t)(2 * D), 1};
  cuuint32_t es[2] = {1, 1};
  CUresult r = encode(map, bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
                      const_cast<void*>(base), gdim, gstr, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                      CU_TENSOR_MAP_SWIZZLE_NONE,
                      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : -3001;
}

MapCache& map_cache() {
  static MapCache c;
  return c;
}

template <bool BF16, int D, int G>
static int launch_decode_t(const DecodeArgs& a_in, cudaStream_t s) {
  DecodeArgs a = a_in;
  {
    // encoded once per (device, KV buffer): host work only
    const int64_t rows = a.B * a.Hkv * a.T;
    const int rc = map_cache().get(map_key(BF16 ? 1 : 2, a.KV, rows, 2 * D, 0, 0), &a.kmap,
                                   [&](CUtensorMap* m) { return make_row_map(m, a.KV, rows, D, BF16); });
    if (rc) return rc;
  }
  const int nsm = sm_count();
  static DevFlags attr;
  // decode grid: programmatic dependent launch too -- it may start behind the
  // previous step's merge (launch, barrier init) and waits for it in
  // griddepcontrol.wait before reading anything
  cudaLaunchConfig_t dcfg = {};
  dcfg.gridDim = dim3((unsigned)nsm);
  dcfg.stream = s;
  cudaLaunchAttribute dat[1];
  dat[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  dat[0].val.programmaticStreamSerializationAllowed = 1;
  dcfg.attrs = dat;
  dcfg.numAttrs = 1;
  if constexpr (BF16) {
    using C = Bf16Cfg<D, G, HGCA_BF16_STAGES, HGCA_BF16_PAIRS>;
    const int rc = set_smem_dev(decode_bf16_kernel<D, G, HGCA_BF16_STAGES, HGCA_BF16_PAIRS>, C::SMEM, attr);
    if (rc) return rc;
    dcfg.blockDim = dim3(C::NW * 32);
    dcfg.dynamicSmemBytes = C::SMEM;
    const cudaError_t e0 = cudaLaunchKernelEx(&dcfg, decode_bf16_kernel<D, G, HGCA_BF16_STAGES, HGCA_BF16_PAIRS>, a);
    if (e0 != cudaSuccess) return (int)e0;
  } else {
    using C = F32Cfg<D, G>;
    const int rc = set_smem_dev(decode_f32_kernel<D, G>, C::SMEM, attr);
    if (rc) return rc;
    dcfg.blockDim = dim3(C::NW * 32);
    dcfg.dynamicSmemBytes = C::SMEM;
    const cudaError_t e0 = cudaLaunchKernelEx(&dcfg, decode_f32_kernel<D, G>, a);
    if (e0 != cudaSuccess) return (int)e0;
  }
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return (int)e;
  // merge kernel: programmatic dependent launch (its launch overlaps the decode tail)
  cudaLaunchConfig_t cfg = {};
  using SC = typename std::conditional<BF16, float, double>::type;  // dense score type
  static DevFlags mattr;
  {
    const int rc = set_smem_dev(decode_merge_kernel<D, G, SC>, MergeCfg<D>::SMEM, mattr);
    if (rc) return rc;
  }
  cfg.gridDim = dim3((unsigned)(a.B * a.Hq * a.m.split));
  cfg.blockDim = dim3(MergeCfg<D>::NT);
  cfg.dynamicSmemBytes = MergeCfg<D>::SMEM;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return (int)cudaLaunchKernelEx(&cfg, decode_merge_kernel<D, G, SC>, a);
}

template <bool BF16, int D>
static int launch_decode_g(const DecodeArgs& a, cudaStream_t s) {
  switch (a.G) {
    case 1: return launch_decode_t<BF16, D, 1>(a, s);
    case 2: return launch_decode_t<BF16, D, 2>(a, s);
    case 4: return launch_decode_t<BF16, D, 4>(a, s);
    case 8: return launch_decode_t<BF16, D, 8>(a, s);
  }
  return -1000;
}

__global__ void step_state_set_kernel(int64_t* state, int64_t dlo, int64_t dhi, uint64_t epoch) {
  state[0] = dlo;
  state[1] = dhi;
  state[2] = (int64_t)epoch;
  state[3] = 0;
}

int launch_step_state_set(int64_t* state, int64_t dlo, int64_t dhi, uint64_t epoch, cudaStream_t s) {
  step_state_set_kernel<<<1, 1, 0, s>>>(state, dlo, dhi, epoch);
  return (int)cudaGetLastError();
}

int decode_chunk_rows(int dtype, int64_t D) {
  (void)dtype;
  (void)D;
  return SUB;
}

int launch_decode_partial(int dtype, const DecodeArgs& a, cudaStream_t s) {
  // the work counter must be 0 on entry: zeroed by the caller once, then re-armed
  // by every merge kernel (no per-step memset launch)
  if (dtype == kBF16) {
    if (a.D == 128) return launch_decode_g<true, 128>(a, s);
    if (a.D == 64) return launch_decode_g<true, 64>(a, s);
  } else if (dtype == kF32) {
    if (a.D == 128) return launch_decode_g<false, 128>(a, s);
    if (a.D == 64) return launch_decode_g<false, 64>(a, s);
  }
  return -1001;
}

int launch_union_build(const uint32_t* sel, int64_t B, int64_t Hq, int64_t Hkv, int64_t words, int64_t n_arch,
                       int64_t T, int32_t* u_ent, int32_t* u_cnt, int32_t* item_off, int4* item_tab,
                       int64_t sparse_rows, int64_t min_rows, int64_t target, int64_t window_rows, int grouped,
                       cudaStream_t s) {
  const int64_t G = Hq / Hkv;
  union_build_kernel<<<(unsigned)(B * Hkv), 1024, 0, s>>>(sel, Hq, Hkv, G, words, n_arch, T, u_ent, u_cnt,
                                                          (grouped == 1 || grouped == 3) ? 1 : 0);
  if (grouped >= 2) {
    const cudaError_t e0 = cudaGetLastError();
    if (e0 != cudaSuccess) return (int)e0;
    // 8-warp CTAs, ~8 windows per warp at a full archive (the lists are at most n_arch long)
    const unsigned chunks = (unsigned)std::max<int64_t>(1, std::min<int64_t>((n_arch + 2047) / 2048, 65535));
    union_window_classes_kernel<<<dim3((unsigned)(B * Hkv), chunks), 256, 0, s>>>(u_ent, u_cnt, T);
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return (int)e;
  item_offsets_kernel<<<1, 1024, 0, s>>>(u_cnt, B * Hkv, sparse_rows, min_rows, target, window_rows, item_off);
  e = cudaGetLastError();
  if (e != cudaSuccess) return (int)e;
  item_table_kernel<<<(unsigned)(B * Hkv), 128, 0, s>>>(u_cnt, item_off, B * Hkv, item_tab);
  return (int)cudaGetLastError();
}

int launch_write_rows(int dtype, void* KV, int64_t BH, int64_t T, int64_t D, int64_t pos, const void* k_new,
                      const void* v_new, int64_t n, cudaStream_t s) {
  const int64_t esz = dtype == kBF16 ? 2 : (dtype == kF64 ? 8 : 4);
  const int64_t rowb = D * esz;
  if (rowb % 16) return -1002;
  const int64_t total = BH * n * (rowb / 16);
  if (total == 0) return 0;
  const int64_t nb = (total + 255) / 256;
  const int blocks = (int)(nb < 148 * 8 ? nb : 148 * 8);
  write_rows_kernel<<<blocks, 256, 0, s>>>((unsigned char*)KV, BH, T, rowb, pos, (const unsigned char*)k_new,
                                           (const unsigned char*)v_new, n, 1);
  return (int)cudaGetLastError();
}

template <bool BF16, int D, int G>
static void cfg_of(int64_t* o) {
  if constexpr (BF16) {
    using C = Bf16Cfg<D, G, HGCA_BF16_STAGES, HGCA_BF16_PAIRS>;
    o[0] = C::NC; o[1] = C::WARP_SMEM; o[2] = HGCA_BF16_STAGES; o[3] = SUB; o[4] = C::SMEM;
  } else {
    using C = F32Cfg<D, G>;
    o[0] = C::NC; o[1] = C::WARP_SMEM; o[2] = C::S; o[3] = SUB; o[4] = C::SMEM;
  }
}

int decode_config(int dtype, int64_t D, int64_t G, int64_t* o) {
#define HG_CFG(BB, DD)                        \
  switch (G) {                                \
    case 1: cfg_of<BB, DD, 1>(o); return 0;   \
    case 2: cfg_of<BB, DD, 2>(o); return 0;   \
    case 4: cfg_of<BB, DD, 4>(o); return 0;   \
    case 8: cfg_of<BB, DD, 8>(o); return 0;   \
  }                                           \
  return -1;
  if (dtype == kBF16 && D == 128) { HG_CFG(true, 128) }
  if (dtype == kBF16 && D == 64) { HG_CFG(true, 64) }
  if (dtype == kF32 && D == 128) { HG_CFG(false, 128) }
  if (dtype == kF32 && D == 64) { HG_CFG(false, 64) }
#undef HG_CFG
  return -1;
}

}  // namespace hgca

#ifdef HGCA_TIMELINE
extern "C" int hgca_debug_gaps(void* host) {
  return (int)cudaMemcpyFromSymbol(host, hgca::g_gap, sizeof(hgca::g_gap));
}
extern "C" int hgca_debug_timeline_merge(void* host) {
  return (int)cudaMemcpyFromSymbol(host, hgca::g_tlm, sizeof(hgca::g_tlm));
}
extern "C" int hgca_debug_timeline(void* host, int64_t n) {
  const int64_t cap = (int64_t)sizeof(hgca::g_tl) / 8;
  if (n > cap) n = cap;
  if (!host) {
    static unsigned long long zero[148 * 16 * TL_SLOTS];
    return (int)cudaMemcpyToSymbol(hgca::g_tl, zero, sizeof(zero));
  }
  return (int)cudaMemcpyFromSymbol(host, hgca::g_tl, n * 8);
}
#endif
