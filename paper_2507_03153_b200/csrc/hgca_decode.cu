// Decode hot path of the hybrid two-tier attention step (engine.py:151-195,
// decode mode) for B200 (sm_100a).
//
// One persistent kernel (decode_partial_kernel) streams two kinds of work
// items through the same warp-specialized pipeline:
//   * dense items  : contiguous window rows [dlo, dhi) of one (batch, kv-head)
//                    -- all G query heads of the GQA group attend every row
//                    (engine.py:161-164);
//   * sparse items : a slice of the (batch, kv-head) union list of selected
//                    archive rows; each entry carries a G-bit mask of the query
//                    heads whose context/padding contains it (engine.py:134-149,
//                    union-deduplicated so every archived row is read once).
// A producer warp gathers K/V rows with 16-byte cp.async into padded shared
// memory stages (mbarrier full/empty ring); four consumer warps compute
//   * fp64 scores, one row per thread, sequential over the head dimension
//     (exact products, reference summation order: _core.pyx:59-65),
//   * an fp64 online softmax per query head,
//   * fp32 P.V accumulation, one warp per query head, lanes over dims.
// Each item emits (m, z, acc) per query head into a fixed slot, so the result
// is independent of which CTA ran which item (deterministic, no float atomics).
// The warp finishing the last item of a (batch, kv-head) then folds its
// partials in a fixed order, applies the reference merge_states
// (attention.py:153-188) and the fp64 MAW EMA (kv_cache.py:171-187,
// engine.py:177-191) from the stored dense scores -- no second kernel.
#include "hgca_common.cuh"
#include "hgca_internal.h"

#include <cuda.h>

namespace hgca {

// Debug build only (-DHGCA_TIMELINE): per-warp timeline of the decode kernel,
// read back with hgca_debug_timeline (tools/timeline.py).
#ifdef HGCA_TIMELINE
#define TL_SLOTS 12
__device__ unsigned long long g_tl[148 * 16 * TL_SLOTS];
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define TL(...) __VA_ARGS__
#else
#define TL(...)
#endif

template <typename T, int D, int G>
struct DecodeCfg {
  static constexpr int ESZ = (int)sizeof(T);
  static constexpr int ROWB = D * ESZ;
  static constexpr int SUB = 32;                        // rows per sub-chunk (one per lane)
  static constexpr int PIECES = ROWB / 16;
  static constexpr int E = 16 / ESZ;                    // elements per 16-byte piece
  // bf16: K rows gathered by TMA (tile::gather4, 4 rows per op) into dense
  // rows, read with a per-lane piece rotation; QK in fp32 per 16-byte piece
  // (8 exact products) accumulated in fp64; V rows gathered into registers.
  // fp32 (reference-exact path): cp.async into XOR-swizzled rows, per-element
  // fp64 DFMA in the reference's sequential order, V staged in smem.
  static constexpr bool TMA = ESZ == 2;
  static constexpr bool PIECE32 = ESZ == 2;
  static constexpr bool V_SMEM = ESZ == 4;
  static constexpr int DPL = D / 32;                    // dims per lane in P.V
  static constexpr int S = 2;                           // stages per warp
  static constexpr int OFF_V = SUB * ROWB;
  static constexpr int OFF_POS = OFF_V + (V_SMEM ? SUB * ROWB : 0);
  static constexpr int OFF_QM = OFF_POS + SUB * 4;
  static constexpr int STAGE = ((OFF_QM + SUB) + 127) / 128 * 128;
  static constexpr int QRAW = G * ROWB;                 // raw query block of one item
  static constexpr int NQB = S;                         // raw query buffers
  static constexpr int QK_ESZ = PIECE32 ? 4 : 8;
  static constexpr int OFF_QRAW = S * STAGE;
  static constexpr int OFF_QK = OFF_QRAW + NQB * QRAW;  // queries [G][D] (fp32 or fp64)
  static constexpr int OFF_SC = OFF_QK + G * D * QK_ESZ;// scores [G][32] fp64
  static constexpr int OFF_ACC = OFF_SC + G * SUB * 8;  // P.V accumulators [G][D] fp32
  static constexpr int OFF_MZ = OFF_ACC + G * D * 4;    // running (m, z) [G][2] fp64
  static constexpr int OFF_BAR = OFF_MZ + G * 16;       // mbarriers [S]
  static constexpr int OFF_DESC = OFF_BAR + S * 8;       // stage descriptors [S]
  // metadata ring: descriptor + union entries (pos, mask) of the next
  // sub-chunks, fetched with cp.async one issue ahead
  static constexpr int MR = 2;
  static constexpr int MSLOT = 32 + SUB * 4 + SUB;       // desc, pos[32], qm[32]
  static constexpr int OFF_META = ((OFF_DESC + S * 32) + 15) / 16 * 16;
  static constexpr int WARP_SMEM = ((OFF_META + MR * MSLOT) + 127) / 128 * 128;
  static constexpr int NC0 = (232448 - 2048) / WARP_SMEM;
  // <= 8 warps: at most 2 per SM sub-partition, so 255 registers per thread
  static constexpr int NC = NC0 > 8 ? 8 : NC0;
  static constexpr int SMEM = NC * WARP_SMEM;
  static_assert(NC >= 1, "decode warp pipeline does not fit shared memory");
  static_assert(D % 32 == 0, "head_dim must be a multiple of 32");
};

// Per-stage descriptor (smem, written by the warp that issued the stage).
struct StageDesc {
  int item, bk, r0, n;
  int first, last, dense, qbuf;
};

__device__ __forceinline__ int swz(int r, int p) { return (p & ~7) | ((p ^ r) & 7); }

template <typename T>
__device__ __forceinline__ void unpack8(const uint4 v, float* f);
template <>
__device__ __forceinline__ void unpack8<__nv_bfloat16>(const uint4 v, float* f) {
  const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    f[2 * i] = __uint_as_float(w[i] << 16);
    f[2 * i + 1] = __uint_as_float(w[i] & 0xffff0000u);
  }
}

template <typename T, int DPL>
__device__ __forceinline__ void load_v_f32(const unsigned char* p, float* out);
template <>
__device__ __forceinline__ void load_v_f32<float, 4>(const unsigned char* p, float* out) {
  const float4 v = *reinterpret_cast<const float4*>(p);
  out[0] = v.x; out[1] = v.y; out[2] = v.z; out[3] = v.w;
}
template <>
__device__ __forceinline__ void load_v_f32<float, 2>(const unsigned char* p, float* out) {
  const float2 v = *reinterpret_cast<const float2*>(p);
  out[0] = v.x; out[1] = v.y;
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void tma_gather4(void* dst, const CUtensorMap* map, int col, int r0, int r1, int r2,
                                            int r3, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];\n" ::"r"(smem_u32(dst)),
      "l"(map), "r"(col), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
               ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

// ------------------------------------------------------------ in-kernel merge
// Run by the warp that finishes the last work item of (b, kv-head) bk: folds
// the dense and sparse partials of each of the G query heads in a fixed order
// (so the result does not depend on which warp runs it), applies
// merge_states(sparse, dense) (attention.py:153-188, engine.py:166-169) and
// the fp64 MAW maintenance of the attended window from the stored scores:
//   w   = float32(exp(s - m) / z)                     (_core.pyx:81-82)
//   maw = (1-alpha)*maw + alpha*w   (3 roundings)     (kv_cache.py:186)
//   new entries: maw = w                              (engine.py:191)
template <int D, int G>
__device__ __forceinline__ void warp_fold(const DecodeArgs& a, int64_t i0, int64_t i1, int g, int lane,
                                          double& M, double& Z, double* acc) {
  constexpr int DPL = D / 32;
  const uint32_t FULL = 0xffffffffu;
  double mx = -INFINITY;
  for (int64_t i = i0 + lane; i < i1; i += 32) mx = fmax(mx, __ldcg(a.m.part_m + i * G + g));
  M = warp_max_f64(mx);
  double z = 0.0;
#pragma unroll
  for (int k = 0; k < DPL; ++k) acc[k] = 0.0;
  for (int64_t c0 = i0; c0 < i1; c0 += 32) {
    const int64_t i = c0 + lane;
    double w = 0.0;
    if (i < i1) {
      const double mi = __ldcg(a.m.part_m + i * G + g);
      if (mi != -INFINITY) {
        w = exp(mi - M);
        z += __ldcg(a.m.part_z + i * G + g) * w;
      }
    }
    const int n = (int)min((int64_t)32, i1 - c0);
    const float* pa = a.m.part_acc + (c0 * G + g) * D + lane * DPL;
#pragma unroll 8
    for (int jj = 0; jj < n; ++jj) {
      const double wj = __shfl_sync(FULL, w, jj);
      if constexpr (DPL == 4) {
        const float4 v = __ldcg(reinterpret_cast<const float4*>(pa + (int64_t)jj * G * D));
        acc[0] += wj * v.x; acc[1] += wj * v.y; acc[2] += wj * v.z; acc[3] += wj * v.w;
      } else {
        const float2 v = __ldcg(reinterpret_cast<const float2*>(pa + (int64_t)jj * G * D));
        acc[0] += wj * v.x; acc[1] += wj * v.y;
      }
    }
  }
  Z = warp_sum_f64(z);
}

template <int D, int G>
__device__ void warp_merge_bk(const DecodeArgs& a, int64_t bk, int lane) {
  constexpr int DPL = D / 32;
  const DecodeMergeArgs& m = a.m;
  const int64_t b = bk / a.Hkv, kvh = bk % a.Hkv;
  const int64_t d0 = bk * a.Sd, d1 = d0 + a.Sd;
  const int64_t s0 = a.n_dense_items + __ldcg(a.item_off + bk), s1 = a.n_dense_items + __ldcg(a.item_off + bk + 1);
  for (int g = 0; g < G; ++g) {
    const int64_t bq = b * a.Hq + kvh * G + g;
    double Md, Zd, Ms, Zs, ad[DPL], as[DPL];
    warp_fold<D, G>(a, d0, d1, g, lane, Md, Zd, ad);
    warp_fold<D, G>(a, s0, s1, g, lane, Ms, Zs, as);
    const bool s_empty = !(Zs > 0.0);
    const bool d_empty = !(Zd > 0.0);
    const double lse_s = s_empty ? -INFINITY : Ms + log(Zs);
    const double lse_d = d_empty ? -INFINITY : Md + log(Zd);
    const double mm = fmax(lse_s, lse_d);
    const bool both_empty = mm == -INFINITY;
    const double ms = both_empty ? 0.0 : mm;
    const double wa = exp(lse_s - ms), wb = exp(lse_d - ms);
    const double zs = both_empty ? 1.0 : wa + wb;
    const float ca = (float)(wa / zs), cb = (float)(wb / zs);
#pragma unroll
    for (int k = 0; k < DPL; ++k) {
      const int c = lane * DPL + k;
      const float od = d_empty ? 0.f : (float)(ad[k] / Zd);
      const float os = s_empty ? 0.f : (float)(as[k] / Zs);
      m.out[bq * D + c] = __fadd_rn(__fmul_rn(ca, os), __fmul_rn(cb, od));
      if (m.out_sparse) m.out_sparse[bq * D + c] = os;
    }
    if (lane == 0) {
      m.lse[bq] = both_empty ? -INFINITY : ms + log(zs);
      if (m.lse_sparse) m.lse_sparse[bq] = lse_s;
    }
    if (m.maw == nullptr && m.wts_out == nullptr) continue;
#pragma unroll 4
    for (int64_t j = lane; j < m.W; j += 32) {
      const float w32 = d_empty ? 0.f : (float)(exp(__ldcg(m.dsc + bq * m.dsc_ld + j) - Md) / Zd);
      if (m.wts_out) m.wts_out[bq * m.W + j] = w32;
      if (m.maw) {
        double* mp = m.maw + bq * m.T + m.dlo + j;
        const double aw = (double)w32;
        *mp = j < m.w_old ? __dadd_rn(__dmul_rn(m.one_minus_alpha, *mp), __dmul_rn(m.alpha, aw)) : aw;
      }
    }
  }
}

template <typename T, int D, int G>
__global__ void __launch_bounds__(DecodeCfg<T, D, G>::NC * 32, 1) decode_partial_kernel(const __grid_constant__ DecodeArgs a) {
  using C = DecodeCfg<T, D, G>;
  extern __shared__ __align__(128) unsigned char sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t FULL = 0xffffffffu;
  unsigned char* wsm = sm + warp * C::WARP_SMEM;
  StageDesc* desc = reinterpret_cast<StageDesc*>(wsm + C::OFF_DESC);
  uint64_t* bar = reinterpret_cast<uint64_t*>(wsm + C::OFF_BAR);
  double* sc = reinterpret_cast<double*>(wsm + C::OFF_SC);
  float* accs = reinterpret_cast<float*>(wsm + C::OFF_ACC);
  double* mz = reinterpret_cast<double*>(wsm + C::OFF_MZ);
  const int64_t W = a.dhi - a.dlo;
  const int total = (int)(a.n_dense_items + (int64_t)a.item_off[a.B * a.Hkv]);
  const unsigned char* Kg = reinterpret_cast<const unsigned char*>(a.K);
  const unsigned char* Vg = reinterpret_cast<const unsigned char*>(a.V);
  const unsigned char* Qg = reinterpret_cast<const unsigned char*>(a.q);
  if constexpr (C::TMA) {
    if (lane < C::S) mbar_init(&bar[lane], 1);
    fence_mbar_init();
    __syncwarp();
  }
  TL(unsigned long long* tl = g_tl + ((int64_t)blockIdx.x * C::NC + warp) * TL_SLOTS;
     unsigned long long tl_merge = 0, tl_wait = 0, tl_sub = 0, tl_items = 0, tl_qk = 0, tl_pv = 0, tl_v = 0,
                        tl_issue = 0;
     if (lane == 0) tl[0] = gtimer(););

  // ---------------------------------------------------------- load cursor
  // Each warp streams whole work items (dynamic, global counter) through its
  // own S-stage ring. The cursor runs ahead across item boundaries; the union
  // entries (position, query-head mask) of a sub-chunk are loaded one issue
  // ahead (pd2) and its rows are prefetched into L2 (bf16: V) when it becomes
  // pd1, the next sub-chunk to issue.
  int next_item = 0;  // lane 0: id of the item after the current one
  if (lane == 0) next_item = atomicAdd(a.counter, 1);
  int L_item = -1, L_bk = 0, L_hi = 0, L_row = 0, L_lo = 0, L_dense = 0, L_qbuf = C::NQB - 1;
  int meta_slot = 0;  // slot holding the next sub-chunk to issue

  // Form the descriptor of the next sub-chunk into metadata slot ms; its union
  // entries arrive by cp.async (sparse) or are computed (dense).
  auto advance = [&](int ms) {
    unsigned char* slot = wsm + C::OFF_META + ms * C::MSLOT;
    StageDesc d;
    if (L_item < 0 || L_row >= L_hi) {
      const int item = __shfl_sync(FULL, next_item, 0);
      if (item >= total) {
        d.item = -1;
        if (lane == 0) *reinterpret_cast<StageDesc*>(slot) = d;
        return;
      }
      L_item = item;
      if (lane == 0) next_item = atomicAdd(a.counter, 1);
      if (L_item < a.n_dense_items) {
        L_dense = 1;
        L_bk = (int)(L_item / a.Sd);
        L_lo = (int)((L_item % a.Sd) * a.dense_rows);
        L_hi = (int)min(W, (int64_t)L_lo + a.dense_rows);
      } else {
        L_dense = 0;
        const int4 e = __ldg(a.item_tab + (L_item - (int)a.n_dense_items));  // (bk, lo, hi, -)
        L_bk = e.x;
        L_lo = e.y;
        L_hi = e.z;
      }
      L_row = L_lo;
    }
    d.item = L_item;
    d.bk = L_bk;
    d.r0 = L_row;
    d.n = min(C::SUB, L_hi - L_row);
    d.first = L_row == L_lo;
    d.last = L_row + C::SUB >= L_hi;
    d.dense = L_dense;
    d.qbuf = 0;
    if (lane == 0) *reinterpret_cast<StageDesc*>(slot) = d;
    int32_t* mpos = reinterpret_cast<int32_t*>(slot + 32);
    uint8_t* mqm = slot + 32 + C::SUB * 4;
    if (L_dense) {
      mpos[lane] = lane < d.n ? (int32_t)(a.dlo + L_row + lane) : 0;
      mqm[lane] = lane < d.n ? (uint8_t)((1u << G) - 1u) : (uint8_t)0;
    } else {
      // entries past the item end are masked at use (lane >= n); they are
      // stale-but-valid positions of the [B*Hkv, T] union buffer
      if (lane < 8) cp_async16(mpos + lane * 4, a.u_pos + (int64_t)L_bk * a.T + L_row + lane * 4);
      else if (lane < 10) cp_async16(mqm + (lane - 8) * 16, a.u_qm + (int64_t)L_bk * a.T + L_row + (lane - 8) * 16);
    }
    L_row += C::SUB;
  };

  auto issue = [&](int s) {
    unsigned char* st = wsm + s * C::STAGE;
    // this sub-chunk's metadata was fetched one issue ago
    asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    __syncwarp();
    const unsigned char* slot = wsm + C::OFF_META + meta_slot * C::MSLOT;
    StageDesc d = *reinterpret_cast<const StageDesc*>(slot);
    int32_t pos = 0;
    uint32_t qm = 0;
    if (d.item >= 0 && lane < d.n) {
      pos = reinterpret_cast<const int32_t*>(slot + 32)[lane];
      qm = slot[32 + C::SUB * 4 + lane];
    }
    if (d.item >= 0 && d.first) {
      L_qbuf = (L_qbuf + 1) % C::NQB;
      d.qbuf = L_qbuf;
    }
    if (lane == 0) desc[s] = d;
    if (d.item >= 0) {
      reinterpret_cast<int32_t*>(st + C::OFF_POS)[lane] = pos;
      st[C::OFF_QM + lane] = (uint8_t)qm;
      const int64_t b = d.bk / a.Hkv, kvh = d.bk % a.Hkv;
      const unsigned char* qsrc = Qg + (b * a.Hq + kvh * G) * (int64_t)C::ROWB;
      unsigned char* qdst = wsm + C::OFF_QRAW + d.qbuf * C::QRAW;
      if constexpr (C::TMA) {
        // 8 gather4 ops (4 rows each) + the item's queries on this stage's mbarrier
        const int rowbase = d.bk * (int)a.T;
        const int q0 = __shfl_sync(FULL, pos, (lane & 7) * 4 + 0);
        const int q1 = __shfl_sync(FULL, pos, (lane & 7) * 4 + 1);
        const int q2 = __shfl_sync(FULL, pos, (lane & 7) * 4 + 2);
        const int q3 = __shfl_sync(FULL, pos, (lane & 7) * 4 + 3);
        if (lane == 0) mbar_expect_tx(&bar[s], C::SUB * C::ROWB + (d.first ? C::QRAW : 0));
        __syncwarp();
        if (lane < 8)
          tma_gather4(st + lane * 4 * C::ROWB, &a.kmap, 0, rowbase + q0, rowbase + q1, rowbase + q2,
                      rowbase + q3, &bar[s]);
        if (lane == 8 && d.first) bulk_g2s(qdst, qsrc, C::QRAW, &bar[s]);
        if constexpr (!C::V_SMEM) {  // warm L2 with this sub-chunk's V rows
          if (lane < d.n) {
            const int64_t off = ((int64_t)d.bk * a.T + pos) * C::ROWB;
#pragma unroll
            for (int l = 0; l < C::ROWB; l += 128) asm volatile("prefetch.global.L2 [%0];\n" ::"l"(Vg + off + l));
          }
        }
      } else {
        if (d.first)
          for (int t = lane; t < C::QRAW / 16; t += 32) cp_async16(qdst + t * 16, qsrc + t * 16);
        const unsigned char* kbase = Kg + (int64_t)d.bk * a.T * C::ROWB;
        const unsigned char* vbase = Vg + (int64_t)d.bk * a.T * C::ROWB;
#pragma unroll 4
        for (int t = lane; t < C::SUB * C::PIECES; t += 32) {
          const int r = t / C::PIECES, p = t % C::PIECES;
          const int32_t pr = __shfl_sync(FULL, pos, r);
          if (r < d.n) {
            cp_async16(st + r * C::ROWB + swz(r, p) * 16, kbase + (int64_t)pr * C::ROWB + p * 16);
            if (C::V_SMEM) cp_async16(st + C::OFF_V + r * C::ROWB + p * 16, vbase + (int64_t)pr * C::ROWB + p * 16);
          }
        }
        asm volatile("cp.async.commit_group;\n" ::: "memory");
      }
      // fetch the following sub-chunk's metadata into the other slot
      meta_slot ^= 1;
      advance(meta_slot);
      asm volatile("cp.async.commit_group;\n" ::: "memory");
    }
  };

  advance(0);
  asm volatile("cp.async.commit_group;\n" ::: "memory");
#pragma unroll
  for (int s = 0; s < C::S; ++s) issue(s);

  // ---------------------------------------------------------- compute
  for (int k = 0;; ++k) {
    const int s = k % C::S;
    __syncwarp();
    TL(long long c0 = clock64();)
    if constexpr (C::TMA) {
      if (desc[s].item >= 0) mbar_wait(&bar[s], (k / C::S) & 1);
    } else {
      // outstanding groups, oldest first: data(k), meta(k+1)+..., data(k+1), meta(k+2)
      asm volatile("cp.async.wait_group %0;\n" ::"n"(2 * (C::S - 1)) : "memory");
    }
    __syncwarp();
    const StageDesc d = desc[s];
    if (d.item < 0) break;
    TL(long long c1 = clock64(); tl_wait += c1 - c0; ++tl_sub;)
    const unsigned char* st = wsm + s * C::STAGE;
    const int32_t mypos = reinterpret_cast<const int32_t*>(st + C::OFF_POS)[lane];
    const uint32_t qm = st[C::OFF_QM + lane];
    const uint32_t wq = __reduce_or_sync(FULL, qm);
    // ---- V rows of this sub-chunk into registers (bf16), unconditional
    uint2 vreg[C::V_SMEM ? 1 : C::SUB];
    if constexpr (!C::V_SMEM) {
      const unsigned char* vbase = Vg + (int64_t)d.bk * a.T * C::ROWB + lane * C::DPL * C::ESZ;
#pragma unroll
      for (int r = 0; r < C::SUB; ++r) {
        const int32_t pr = __shfl_sync(FULL, mypos, r);
        if constexpr (C::DPL * C::ESZ == 8) {
          vreg[r] = __ldg(reinterpret_cast<const uint2*>(vbase + (int64_t)pr * C::ROWB));
        } else {
          vreg[r].x = __ldg(reinterpret_cast<const uint32_t*>(vbase + (int64_t)pr * C::ROWB));
        }
      }
    }
    TL(long long c2 = clock64(); tl_v += c2 - c1;)
    if (d.first) {
      const T* qr = reinterpret_cast<const T*>(wsm + C::OFF_QRAW + d.qbuf * C::QRAW);
      if constexpr (C::PIECE32) {
        // piece p's first 4 floats at [p*4], last 4 at [D/2 + p*4]: rotated
        // per-lane piece reads then hit distinct banks
        float* qk = reinterpret_cast<float*>(wsm + C::OFF_QK);
        for (int t = lane; t < G * D; t += 32) {
          const int g = t / D, e = t % D, p = e / 8, j = e % 8;
          qk[g * D + (j < 4 ? p * 4 + j : D / 2 + p * 4 + (j - 4))] = to_f32(qr[t]);
        }
      } else {
        double* qk = reinterpret_cast<double*>(wsm + C::OFF_QK);
        for (int t = lane; t < G * D; t += 32) qk[t] = to_f64(qr[t]);
      }
      for (int t = lane; t < G * D; t += 32) accs[t] = 0.f;
      if (lane < G) {
        mz[2 * lane] = -INFINITY;
        mz[2 * lane + 1] = 0.0;
      }
      __syncwarp();
    }
    // ---- scores: lane = row
    double sacc[G];
#pragma unroll
    for (int g = 0; g < G; ++g) sacc[g] = 0.0;
    {
      const unsigned char* krow = st + lane * C::ROWB;
      if constexpr (C::PIECE32) {
        const float* qk = reinterpret_cast<const float*>(wsm + C::OFF_QK);
        if (__popc(wq) == 1) {  // single query head (most union chunks): no per-piece branching
          const int g = __ffs(wq) - 1;
          double s1 = 0.0;
#pragma unroll 4
          for (int i = 0; i < C::PIECES; ++i) {
            const int p = (i + lane) & (C::PIECES - 1);  // rotation: conflict-free dense rows
            float kf[8];
            unpack8<T>(*reinterpret_cast<const uint4*>(krow + p * 16), kf);
            const float4 qa = *reinterpret_cast<const float4*>(qk + g * D + p * 4);
            const float4 qb = *reinterpret_cast<const float4*>(qk + g * D + D / 2 + p * 4);
            float part = qa.x * kf[0];
            part = fmaf(qa.y, kf[1], part);
            part = fmaf(qa.z, kf[2], part);
            part = fmaf(qa.w, kf[3], part);
            part = fmaf(qb.x, kf[4], part);
            part = fmaf(qb.y, kf[5], part);
            part = fmaf(qb.z, kf[6], part);
            part = fmaf(qb.w, kf[7], part);
            s1 += (double)part;
          }
#pragma unroll
          for (int gg = 0; gg < G; ++gg) sacc[gg] = (gg == g) ? s1 : 0.0;
        } else {
#pragma unroll 2
          for (int i = 0; i < C::PIECES; ++i) {
            const int p = (i + lane) & (C::PIECES - 1);
            float kf[8];
            unpack8<T>(*reinterpret_cast<const uint4*>(krow + p * 16), kf);
#pragma unroll
            for (int g = 0; g < G; ++g) {
              if ((wq >> g) & 1u) {
                const float4 qa = *reinterpret_cast<const float4*>(qk + g * D + p * 4);
                const float4 qb = *reinterpret_cast<const float4*>(qk + g * D + D / 2 + p * 4);
                float part = qa.x * kf[0];
                part = fmaf(qa.y, kf[1], part);
                part = fmaf(qa.z, kf[2], part);
                part = fmaf(qa.w, kf[3], part);
                part = fmaf(qb.x, kf[4], part);
                part = fmaf(qb.y, kf[5], part);
                part = fmaf(qb.z, kf[6], part);
                part = fmaf(qb.w, kf[7], part);
                sacc[g] += (double)part;
              }
            }
          }
        }
      } else {
        const double* qk = reinterpret_cast<const double*>(wsm + C::OFF_QK);
#pragma unroll 4
        for (int p = 0; p < C::PIECES; ++p) {
          const uint4 raw = *reinterpret_cast<const uint4*>(krow + swz(lane, p) * 16);
          const double kd[4] = {(double)__uint_as_float(raw.x), (double)__uint_as_float(raw.y),
                                (double)__uint_as_float(raw.z), (double)__uint_as_float(raw.w)};
#pragma unroll
          for (int g = 0; g < G; ++g) {
            if ((wq >> g) & 1u) {
              const double2 qa = *reinterpret_cast<const double2*>(qk + g * D + p * 4);
              const double2 qb = *reinterpret_cast<const double2*>(qk + g * D + p * 4 + 2);
              sacc[g] = fma(qa.x, kd[0], sacc[g]);  // exact products: reference order
              sacc[g] = fma(qa.y, kd[1], sacc[g]);
              sacc[g] = fma(qb.x, kd[2], sacc[g]);
              sacc[g] = fma(qb.y, kd[3], sacc[g]);
            }
          }
        }
      }
    }
    const int64_t b = d.bk / a.Hkv, kvh = d.bk % a.Hkv;
#pragma unroll
    for (int g = 0; g < G; ++g) {
      if (!((wq >> g) & 1u)) continue;
      const double sv = ((qm >> g) & 1u) ? sacc[g] * a.scale : -INFINITY;
      sc[g * C::SUB + lane] = sv;
      if (d.dense && lane < d.n) a.dsc[(b * a.Hq + kvh * G + g) * a.dsc_ld + (mypos - a.dlo)] = sv;
    }
    __syncwarp();
    TL(long long c3 = clock64(); tl_qk += c3 - c2;)
    // ---- per active head (rolled loop): online softmax (fp64) + P.V (fp32)
    for (uint32_t hm = wq; hm; hm &= hm - 1) {
      const int g = __ffs(hm) - 1;
      const double sv = sc[g * C::SUB + lane];
      const double cm = warp_max_f64(sv);
      const double m_old = mz[2 * g];
      const double mnew = fmax(m_old, cm);
      if (mnew == -INFINITY) continue;
      const double scal = exp(m_old - mnew);
      const double p = exp(sv - mnew);
      const double zs = warp_sum_f64(p);
      const float pf = (float)p;
      const float sf = (float)scal;
      float acc[C::DPL];
      float* ag = accs + g * D + lane * C::DPL;
#pragma unroll
      for (int i = 0; i < C::DPL; ++i) acc[i] = ag[i] * sf;
#pragma unroll
      for (int r = 0; r < C::SUB; ++r) {
        const float pr = __shfl_sync(FULL, pf, r);
        if (C::V_SMEM && r >= d.n) break;  // staged V rows past the end are not loaded
        float vv[C::DPL];
        if constexpr (C::V_SMEM) {
          load_v_f32<T, C::DPL>(st + C::OFF_V + r * C::ROWB + lane * C::DPL * C::ESZ, vv);
        } else {
          vv[0] = __uint_as_float(vreg[r].x << 16);
          vv[1] = __uint_as_float(vreg[r].x & 0xffff0000u);
          if constexpr (C::DPL == 4) {
            vv[C::DPL > 2 ? 2 : 0] = __uint_as_float(vreg[r].y << 16);
            vv[C::DPL > 3 ? 3 : 0] = __uint_as_float(vreg[r].y & 0xffff0000u);
          }
        }
#pragma unroll
        for (int i = 0; i < C::DPL; ++i) acc[i] = fmaf(pr, vv[i], acc[i]);
      }
#pragma unroll
      for (int i = 0; i < C::DPL; ++i) ag[i] = acc[i];
      __syncwarp();
      if (lane == 0) {
        mz[2 * g] = mnew;
        mz[2 * g + 1] = mz[2 * g + 1] * scal + zs;
      }
      __syncwarp();
    }
    TL(long long c4 = clock64(); tl_pv += c4 - c3;)
    if (d.last) {
      TL(++tl_items;)
      for (int t = lane; t < G * D; t += 32) a.part_acc[(int64_t)d.item * G * D + t] = accs[t];
      if (lane < G) {
        a.part_m[(int64_t)d.item * G + lane] = mz[2 * lane];
        a.part_z[(int64_t)d.item * G + lane] = mz[2 * lane + 1];
      }
      // the last finished item of this (b, kv-head) merges it
      __threadfence();
      __syncwarp();
      int old = 0;
      if (lane == 0) old = atomicAdd(a.bk_done + d.bk, 1);
      old = __shfl_sync(FULL, old, 0);
      const int n_items = (int)a.Sd + (__ldcg(a.item_off + d.bk + 1) - __ldcg(a.item_off + d.bk));
      if (old == n_items - 1) {
        __threadfence();
        TL(long long m0 = clock64();)
        warp_merge_bk<D, G>(a, d.bk, lane);
        TL(tl_merge += clock64() - m0;)
      }
    }
    __syncwarp();
    TL(long long c5 = clock64();)
    issue(s);
    TL(tl_issue += clock64() - c5;)
  }
  if constexpr (!C::TMA) asm volatile("cp.async.wait_group 0;\n" ::: "memory");
  TL(if (lane == 0) {
    tl[1] = gtimer();
    tl[2] = tl_merge; tl[3] = tl_wait; tl[4] = tl_sub; tl[5] = tl_items; tl[6] = tl_qk; tl[7] = tl_pv;
    tl[8] = tl_v; tl[9] = tl_issue; tl[10] = blockIdx.x; tl[11] = clock64();
  })
}

// --------------------------------------------------------------------- merge
// One CTA per (batch, query head). Folds dense and sparse partials in a fixed
// order, applies merge_states(sparse, dense) (engine.py:166-169), and updates
// the MAW of the attended window positions from the stored fp64 scores:
//   w   = float32(exp(s - m) / z)                     (_core.pyx:81-82)
//   maw = (1-alpha)*maw + alpha*w   (3 roundings)     (kv_cache.py:186)
//   new entries: maw = w                              (engine.py:191)
// -------------------------------------------------------------- union build
// Per (batch, kv-head): union of the G query heads' selection masks over the
// archive [0, n_arch), emitted grouped by query-head mask value (ascending
// mask, then ascending position) so consecutive rows of a chunk share their
// mask and the consumer warps skip inactive heads uniformly.
__global__ void __launch_bounds__(1024) union_build_kernel(const uint32_t* __restrict__ sel,
                                                           int64_t Hq, int64_t Hkv, int64_t G,
                                                           int64_t words, int64_t n_arch, int64_t T,
                                                           int32_t* u_pos, uint8_t* u_qm,
                                                           int32_t* u_cnt) {
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
  __syncthreads();
  if (tid == 0) base_s = 0;
  __syncthreads();
  const int nbins = 1 << G;
  for (int v = 1; v < nbins; ++v) {
    if (hist[v] == 0) continue;  // uniform: hist is stable after the barrier
    for (int64_t w0 = 0; w0 < nw; w0 += blockDim.x) {
      const int64_t w = w0 + tid;
      uint32_t hit = 0;
      if (w < nw) {
        uint32_t mg[8];
        uint32_t any = word_masks(w, mg);
        while (any) {
          const int bit = __ffs(any) - 1;
          any &= any - 1;
          uint32_t qm = 0;
          for (int g = 0; g < G; ++g) qm |= ((mg[g] >> bit) & 1u) << g;
          if (qm == (uint32_t)v) hit |= 1u << bit;
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
        u_pos[bk * T + pos] = (int32_t)((w << 5) + bit);
        u_qm[bk * T + pos] = (uint8_t)v;
        ++pos;
      }
      __syncthreads();
      if (tid == 0) base_s += wsum[nwarp - 1];
      __syncthreads();
    }
  }
  if (tid == 0) u_cnt[bk] = base_s;
}

// item_off[bk] = sum_{x<bk} ceil(u_cnt[x] / rows)  (single CTA, sequential chunks)
__global__ void item_offsets_kernel(const int32_t* u_cnt, int64_t BK, int64_t rows, int32_t* off) {
  __shared__ int32_t carry;
  __shared__ int wsum[32];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nwarp = blockDim.x >> 5;
  if (tid == 0) carry = 0;
  __syncthreads();
  for (int64_t x0 = 0; x0 < BK; x0 += blockDim.x) {
    const int64_t x = x0 + tid;
    const int c = x < BK ? (int)((u_cnt[x] + rows - 1) / rows) : 0;
    int incl = c;
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane == 31) wsum[wid] = incl;
    __syncthreads();
    if (wid == 0) {
      int v = lane < nwarp ? wsum[lane] : 0;
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += y;
      }
      if (lane < nwarp) wsum[lane] = v;
    }
    __syncthreads();
    if (x < BK) off[x] = carry + (wid ? wsum[wid - 1] : 0) + (incl - c);
    __syncthreads();
    if (tid == 0) carry += wsum[nwarp - 1];
    __syncthreads();
  }
  if (tid == 0) off[BK] = carry;
}

// item_tab[item_off[bk] + i] = (bk, i*rows, min(u_cnt[bk], (i+1)*rows), 0)
__global__ void item_table_kernel(const int32_t* u_cnt, const int32_t* off, int64_t BK, int64_t rows,
                                  int4* tab) {
  const int64_t bk = blockIdx.x;
  if (bk >= BK) return;
  const int n = off[bk + 1] - off[bk];
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const int lo = (int)(i * rows);
    tab[off[bk] + i] = make_int4((int)bk, lo, (int)min((int64_t)u_cnt[bk], (int64_t)lo + rows), 0);
  }
}

// K/V[bh, pos + i, :] = new[bh, i, :]  (append_kv into the position buffer)
__global__ void write_rows_kernel(unsigned char* K, unsigned char* V, int64_t BH, int64_t T,
                                  int64_t rowb, int64_t pos, const unsigned char* kn,
                                  const unsigned char* vn, int64_t n) {
  const int64_t pieces = rowb / 16;
  const int64_t total = BH * n * pieces;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = t % pieces, row = t / pieces;
    const int64_t bh = row / n, i = row % n;
    const int64_t dst = (bh * T + pos + i) * rowb + p * 16;
    const int64_t src = (bh * n + i) * rowb + p * 16;
    *reinterpret_cast<uint4*>(K + dst) = *reinterpret_cast<const uint4*>(kn + src);
    *reinterpret_cast<uint4*>(V + dst) = *reinterpret_cast<const uint4*>(vn + src);
  }
}

// ------------------------------------------------------------------ launchers
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

// 2-D tensor map over the K buffer [B*Hkv*T rows, D] for tile::gather4 (box = one row).
static int make_row_map(CUtensorMap* map, const void* base, int64_t rows, int64_t D, int esz) {
  static EncodeTiledFn encode = nullptr;
  if (!encode) {
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&encode, cudaEnableDefault, &q) != cudaSuccess ||
        !encode)
      return -3000;
  }
  cuuint64_t gdim[2] = {(cuuint64_t)D, (cuuint64_t)rows};
  cuuint64_t gstr[1] = {(cuuint64_t)(D * esz)};
  cuuint32_t box[2] = {(cuuint32_t)D, 1};
  cuuint32_t es[2] = {1, 1};
  CUresult r = encode(map, esz == 2 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
                      const_cast<void*>(base), gdim, gstr, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                      CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : -3001;
}

template <typename T, int D, int G>
static int launch_decode_t(const DecodeArgs& a_in, cudaStream_t s) {
  using C = DecodeCfg<T, D, G>;
  DecodeArgs a = a_in;
  if (C::TMA) {
    // cached per K buffer: encoding is host work only
    static const void* cached_base = nullptr;
    static int64_t cached_rows = -1;
    static CUtensorMap cached;
    const int64_t rows = a.B * a.Hkv * a.T;
    if (cached_base != a.K || cached_rows != rows) {
      const int rc = make_row_map(&cached, a.K, rows, D, C::ESZ);
      if (rc) return rc;
      cached_base = a.K;
      cached_rows = rows;
    }
    a.kmap = cached;
  }
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(decode_partial_kernel<T, D, G>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    if (e != cudaSuccess) return -(int)e;
    attr = true;
  }
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  decode_partial_kernel<T, D, G><<<nsm, C::NC * 32, C::SMEM, s>>>(a);
  return (int)cudaGetLastError();
}

template <typename T, int D>
static int launch_decode_g(const DecodeArgs& a, cudaStream_t s) {
  switch (a.G) {
    case 1: return launch_decode_t<T, D, 1>(a, s);
    case 2: return launch_decode_t<T, D, 2>(a, s);
    case 4: return launch_decode_t<T, D, 4>(a, s);
    case 8: return launch_decode_t<T, D, 8>(a, s);
  }
  return -1000;
}

int decode_chunk_rows(int dtype, int64_t D) {
  (void)dtype;
  (void)D;
  return 32;
}

int launch_decode_partial(int dtype, const DecodeArgs& a, cudaStream_t s) {
  // work counter + per-(b, kv-head) finished-item counters
  cudaError_t e = cudaMemsetAsync(a.counter, 0, sizeof(int32_t) * (1 + a.B * a.Hkv), s);
  if (e != cudaSuccess) return (int)e;
  if (dtype == kBF16) {
    if (a.D == 128) return launch_decode_g<__nv_bfloat16, 128>(a, s);
    if (a.D == 64) return launch_decode_g<__nv_bfloat16, 64>(a, s);
  } else if (dtype == kF32) {
    if (a.D == 128) return launch_decode_g<float, 128>(a, s);
    if (a.D == 64) return launch_decode_g<float, 64>(a, s);
  }
  return -1001;
}


int launch_union_build(const uint32_t* sel, int64_t B, int64_t Hq, int64_t Hkv, int64_t words,
                       int64_t n_arch, int64_t T, int32_t* u_pos, uint8_t* u_qm, int32_t* u_cnt,
                       int32_t* item_off, int4* item_tab, int64_t sparse_rows, cudaStream_t s) {
  const int64_t G = Hq / Hkv;
  union_build_kernel<<<(unsigned)(B * Hkv), 1024, 0, s>>>(sel, Hq, Hkv, G, words, n_arch, T, u_pos,
                                                          u_qm, u_cnt);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return (int)e;
  item_offsets_kernel<<<1, 1024, 0, s>>>(u_cnt, B * Hkv, sparse_rows, item_off);
  e = cudaGetLastError();
  if (e != cudaSuccess) return (int)e;
  item_table_kernel<<<(unsigned)(B * Hkv), 128, 0, s>>>(u_cnt, item_off, B * Hkv, sparse_rows, item_tab);
  return (int)cudaGetLastError();
}

int launch_write_rows(int dtype, void* K, void* V, int64_t BH, int64_t T, int64_t D, int64_t pos,
                      const void* k_new, const void* v_new, int64_t n, cudaStream_t s) {
  const int64_t esz = dtype == kBF16 ? 2 : (dtype == kF64 ? 8 : 4);
  const int64_t rowb = D * esz;
  if (rowb % 16) return -1002;
  const int64_t total = BH * n * (rowb / 16);
  if (total == 0) return 0;
  const int64_t nb = (total + 255) / 256;
  const int blocks = (int)(nb < 148 * 8 ? nb : 148 * 8);
  write_rows_kernel<<<blocks, 256, 0, s>>>((unsigned char*)K, (unsigned char*)V, BH, T, rowb, pos,
                                           (const unsigned char*)k_new, (const unsigned char*)v_new, n);
  return (int)cudaGetLastError();
}

}  // namespace hgca

#ifdef HGCA_TIMELINE
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

namespace hgca {
template <typename T, int D, int G>
static void cfg_of(int64_t* o) {
  using C = DecodeCfg<T, D, G>;
  o[0] = C::NC; o[1] = C::WARP_SMEM; o[2] = C::S; o[3] = C::SUB; o[4] = C::SMEM;
}
int decode_config(int dtype, int64_t D, int64_t G, int64_t* o) {
#define HG_CFG(TT, DD)                                       \
  switch (G) {                                               \
    case 1: cfg_of<TT, DD, 1>(o); return 0;                  \
    case 2: cfg_of<TT, DD, 2>(o); return 0;                  \
    case 4: cfg_of<TT, DD, 4>(o); return 0;                  \
    case 8: cfg_of<TT, DD, 8>(o); return 0;                  \
  }                                                          \
  return -1;
  if (dtype == kBF16 && D == 128) { HG_CFG(__nv_bfloat16, 128) }
  if (dtype == kBF16 && D == 64) { HG_CFG(__nv_bfloat16, 64) }
  if (dtype == kF32 && D == 128) { HG_CFG(float, 128) }
  if (dtype == kF32 && D == 64) { HG_CFG(float, 64) }
#undef HG_CFG
  return -1;
}
}  // namespace hgca
