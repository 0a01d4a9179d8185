// Append / re-evaluation step for bfloat16 storage (engine.py:111-132,
// 161-169; sparsifier.py:158-177) on the tensor cores.
//
// An append step attends n_q new queries per query head to (segment 0) the
// whole archive [0, lo) and (segment 1) the window plus the new entries
// [lo, hi), with the reference's merge_states(archive, window) on top, and it
// needs, per query head and position, the mean attention weight over the n_q
// rows (a_cpu -> StoreTier.reevaluate, a_gpu -> the window MAW). The keys are
// consecutive positions, so this is GEMM-shaped: per (batch, kv-head) the
// G * n_q query rows (head-major: row = g * n_q + i) form the M side.
//
//   append_attend_kernel<D, 1>  split-K over chunks of ACHUNK keys: one CTA per
//       (batch x kv-head, row group, segment, chunk); a producer warp TMA-loads
//       32-key stages (2-D tile box, one op per stage) into a ring, each
//       consumer warp owns 16 query rows: S = Q K^T and O += P V on mma.sync
//       m16n8k16 (P as bf16 hi + lo), fp32 online softmax -> (m, z, acc) per row.
//   append_fold_kernel<D>       one warp per (batch x kv-head, row): folds the
//       chunk partials of each segment in chunk order, merge_states, out/lse,
//       and keeps each row's final (m, z) per segment.
//   append_attend_kernel<D, 2>  same tiling, recomputes S with the final
//       statistics: w = exp(s - m) / z, and writes per (query head, position)
//       the mean of w over the head's n_q rows (fixed summation order).
// Deterministic: fixed partition and fixed fold / summation orders.
#include "hgca_common.cuh"
#include "hgca_internal.h"
#include "hgca_host.h"
#include "hgca_tc.cuh"
#include "hgca_umma.cuh"

#include <cuda.h>
#include <cstdlib>
#include <type_traits>

namespace hgca {

constexpr uint32_t FULL_MASK = 0xffffffffu;
constexpr int AK = 32;          // keys per stage
constexpr int ACHUNK = 4096;    // keys per split-K item
constexpr int AS = 4;           // stages in the ring
constexpr int AMAXW = 8;        // consumer warps per CTA -> <= 128 query rows per row group

struct AppendArgs {
  CUtensorMap kmap;             // 2-D tile map over KV [B*Hkv*T rows, 2D], box {2D, 32}
  CUtensorMap kvmap5;           // tcgen05 pass: over KV [B*Hkv*T rows, 2D], box {64, 64}, no swizzle
  CUtensorMap qmap5;            // tcgen05 pass: over q [B*Hq*nq rows, D], box {64, 128}, 128-byte swizzle
  CUtensorMap qmap5h;           // the same with box {64, 64}: a 64-row group loaded twice (split-key pass 1)
  const __nv_bfloat16* q;       // [B*Hq, nq, D]
  int64_t B, Hq, Hkv, G, T, nq;
  float scale;
  int64_t seg_lo[2], seg_hi[2];  // 0 = archive [0, lo), 1 = window + kv_in [lo, hi)
  int64_t nch[2];                // split-K chunks per segment
  int64_t R, RG, n_rg;           // rows per (batch, kv-head), rows per row group, row groups
  int64_t n_items;
  float* part_acc;               // [n_items][RG][D]
  float* part_m;                 // [n_items][RG]
  float* part_z;
  float* fin;                    // [B*Hkv][R][2 segments][m, z]
  float* out;                    // [B*Hq, nq, D]
  double* lse;                   // [B*Hq, nq]
  float* mean[2];                // [B*Hq, mean_ld] mean weights per position, or null
  int64_t mean_ld[2];
  int split_keys;                // pass 1 on 64-row groups: the split-key mode (HGCA_APPEND_SPLIT_KEYS=0: off)
};

template <int D, int PASS>
struct AppendCfg {
  static constexpr int ROWB = 2 * D * 2;                 // bytes of one rotated K|V row pair
  static constexpr int STAGE = AK * ROWB;
  static constexpr int OFF_W = AS * STAGE;               // pass 2: weights [RG <= 128][AK] fp32
  static constexpr int OFF_BAR = OFF_W + (PASS == 2 ? AMAXW * 16 * AK * 4 : 0);
  static constexpr int SMEM = OFF_BAR + 2 * AS * 8 + 1024;  // + alignment slack
};

template <int D>
__device__ __forceinline__ uint32_t arot(int r, int c, int rot) {
  return (uint32_t)(r * 4 * D + (((c & ~7) | ((c ^ rot) & 7)) << 4));
}

// item id -> (bk, row group, segment, chunk)
__device__ __forceinline__ void append_item(const AppendArgs& a, int64_t id, int64_t& bk, int64_t& rg, int& seg,
                                            int64_t& chunk) {
  const int64_t nc = a.nch[0] + a.nch[1];
  const int64_t c = id % nc;
  const int64_t t = id / nc;
  rg = t % a.n_rg;
  bk = t / a.n_rg;
  seg = c < a.nch[0] ? 0 : 1;
  chunk = seg ? c - a.nch[0] : c;
}

template <int D, int PASS>
__global__ void __launch_bounds__((AMAXW + 1) * 32, 1) append_attend_kernel(const __grid_constant__ AppendArgs a) {
  using C = AppendCfg<D, PASS>;
  constexpr int KC = D / 16;
  extern __shared__ unsigned char sm_raw[];
  unsigned char* sm = smem_align1024(sm_raw);
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + C::OFF_BAR);
  uint64_t* empty = full + AS;
  float* wbuf = reinterpret_cast<float*>(sm + C::OFF_W);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int NW = (int)(blockDim.x >> 5) - 1;  // consumer warps
  int64_t bk, rg, chunk;
  int seg;
  append_item(a, blockIdx.x, bk, rg, seg, chunk);
  const int64_t p0 = a.seg_lo[seg] + chunk * ACHUNK;
  const int64_t p1 = min(a.seg_hi[seg], p0 + ACHUNK);
  const int nst = (int)((p1 - p0 + AK - 1) / AK);
  if (threadIdx.x == 0) {
    for (int s = 0; s < AS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NW);
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (warp == NW) {  // ----------------------------------------------- producer
    if (lane == 0) {
      const uint64_t policy = l2_evict_first_policy();
      const int rowbase = (int)(bk * a.T + p0);
      for (int st = 0; st < nst; ++st) {
        const int s = st % AS;
        if (st >= AS) mbar_wait(&empty[s], ((st / AS) - 1) & 1);
        mbar_expect_tx(&full[s], C::STAGE);
        tma_load_2d(smem_u32(sm + s * C::STAGE), &a.kmap, 0, rowbase + st * AK, &full[s], policy);
      }
    }
    return;
  }

  // ------------------------------------------------------------------ consumer
  const int g4 = lane >> 2, t4 = lane & 3, mi = lane >> 3;
  const int r0 = warp * 16;                                   // first row of this warp in the group
  const int64_t rowA = rg * a.RG + r0 + g4, rowB = rowA + 8;  // rows of this lane in the (b, kv-head)
  const bool okA = r0 + g4 < a.RG && rowA < a.R, okB = r0 + g4 + 8 < a.RG && rowB < a.R;
  const int64_t b = bk / a.Hkv, kvh = bk % a.Hkv;
  const __nv_bfloat16* qbase = a.q + (b * a.Hq + kvh * a.G) * a.nq * D;  // rows of this (b, kv-head)
  // Q A-fragments for all k16 chunks (rows r0..r0+15 of the group)
  uint32_t qa[KC][4];
  {
    const uint32_t* qA = reinterpret_cast<const uint32_t*>(qbase + rowA * D);
    const uint32_t* qB = reinterpret_cast<const uint32_t*>(qbase + rowB * D);
#pragma unroll
    for (int kc = 0; kc < KC; ++kc) {
      qa[kc][0] = okA ? qA[kc * 8 + t4] : 0u;
      qa[kc][1] = okB ? qB[kc * 8 + t4] : 0u;
      qa[kc][2] = okA ? qA[kc * 8 + 4 + t4] : 0u;
      qa[kc][3] = okB ? qB[kc * 8 + 4 + t4] : 0u;
    }
  }
  // pass 2: the rows' final statistics of this segment
  float fmA = 0.f, fzA = 1.f, fmB = 0.f, fzB = 1.f;
  if (PASS == 2) {
    if (okA) { fmA = a.fin[((bk * a.R + rowA) * 2 + seg) * 2]; fzA = a.fin[((bk * a.R + rowA) * 2 + seg) * 2 + 1]; }
    if (okB) { fmB = a.fin[((bk * a.R + rowB) * 2 + seg) * 2]; fzB = a.fin[((bk * a.R + rowB) * 2 + seg) * 2 + 1]; }
  }
  const float rzA = 1.f / fzA, rzB = 1.f / fzB;
  // pass 2: the (query head, key) mean targets of this thread, fixed for the item
  // (at most G*AK / 32 = 8 per thread: heads*AK pairs over ceil(RG/16) warps, RG <= 128)
  int64_t mdst[8];
  int mrow[8], mkey[8];
  int n_mt = 0;
  if (PASS == 2 && a.mean[seg]) {
    const int heads = (int)(a.RG / a.nq);  // row groups hold whole heads
    const int64_t g0 = (rg * a.RG) / a.nq;
    for (int t = threadIdx.x; t < heads * AK && n_mt < 8; t += NW * 32) {
      const int hl = t / AK, k = t % AK;
      if (g0 + hl >= a.G) break;
      mrow[n_mt] = hl * (int)a.nq;
      mkey[n_mt] = k;
      mdst[n_mt] = (b * a.Hq + kvh * a.G + g0 + hl) * a.mean_ld[seg] - a.seg_lo[seg] + k;
      ++n_mt;
    }
  }
  const float inv_nq = 1.f / (float)a.nq;
  float o[D / 8][4];
#pragma unroll
  for (int n = 0; n < D / 8; ++n) o[n][0] = o[n][1] = o[n][2] = o[n][3] = 0.f;
  float mA = -INFINITY, mB = -INFINITY, zA = 0.f, zB = 0.f;

  for (int st = 0; st < nst; ++st) {
    const int s = st % AS;
    mbar_wait(&full[s], (st / AS) & 1);
    const uint32_t stg = smem_u32(sm + s * C::STAGE);
    const int64_t kp0 = p0 + (int64_t)st * AK;  // position of key 0 of the stage
    // ---- S = Q K^T for the 32 keys: 4 n-tiles of 8 keys
    float sc[4][4];
#pragma unroll
    for (int n = 0; n < 4; ++n) sc[n][0] = sc[n][1] = sc[n][2] = sc[n][3] = 0.f;
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int key = j * 16 + (mi >> 1) * 8 + (lane & 7);
      const int rot = (int)((kp0 + key) & 7);
#pragma unroll
      for (int kc = 0; kc < KC; ++kc) {
        uint32_t kb[4];
        ldsm_x4(stg + arot<D>(key, 2 * kc + (mi & 1), rot), kb);
        mma_bf16(sc[2 * j], qa[kc], kb[0], kb[1]);
        mma_bf16(sc[2 * j + 1], qa[kc], kb[2], kb[3]);
      }
    }
    // ---- scale + mask (keys past the segment end)
#pragma unroll
    for (int n = 0; n < 4; ++n) {
      const int64_t kpos = kp0 + n * 8 + 2 * t4;
      const bool v0 = kpos < p1, v1 = kpos + 1 < p1;
      sc[n][0] = v0 ? sc[n][0] * a.scale : -INFINITY;
      sc[n][1] = v1 ? sc[n][1] * a.scale : -INFINITY;
      sc[n][2] = v0 ? sc[n][2] * a.scale : -INFINITY;
      sc[n][3] = v1 ? sc[n][3] * a.scale : -INFINITY;
    }
    if constexpr (PASS == 1) {
      // ---- online softmax per row (rows g4 | g4 + 8), reduced over the 4 lanes sharing g4
      float xA = -INFINITY, xB = -INFINITY;
#pragma unroll
      for (int n = 0; n < 4; ++n) {
        xA = fmaxf(xA, fmaxf(sc[n][0], sc[n][1]));
        xB = fmaxf(xB, fmaxf(sc[n][2], sc[n][3]));
      }
#pragma unroll
      for (int off = 1; off < 4; off <<= 1) {
        xA = fmaxf(xA, __shfl_xor_sync(FULL_MASK, xA, off));
        xB = fmaxf(xB, __shfl_xor_sync(FULL_MASK, xB, off));
      }
      const float nA = fmaxf(mA, xA), nB = fmaxf(mB, xB);
      const float alA = nA == -INFINITY ? 1.f : __expf(mA - nA);
      const float alB = nB == -INFINITY ? 1.f : __expf(mB - nB);
      float sA = 0.f, sB = 0.f;
#pragma unroll
      for (int n = 0; n < 4; ++n) {
        sc[n][0] = sc[n][0] == -INFINITY ? 0.f : __expf(sc[n][0] - nA);
        sc[n][1] = sc[n][1] == -INFINITY ? 0.f : __expf(sc[n][1] - nA);
        sc[n][2] = sc[n][2] == -INFINITY ? 0.f : __expf(sc[n][2] - nB);
        sc[n][3] = sc[n][3] == -INFINITY ? 0.f : __expf(sc[n][3] - nB);
        sA += sc[n][0] + sc[n][1];
        sB += sc[n][2] + sc[n][3];
      }
#pragma unroll
      for (int off = 1; off < 4; off <<= 1) {
        sA += __shfl_xor_sync(FULL_MASK, sA, off);
        sB += __shfl_xor_sync(FULL_MASK, sB, off);
      }
      zA = zA * alA + sA;
      zB = zB * alB + sB;
      mA = nA;
      mB = nB;
#pragma unroll
      for (int n = 0; n < D / 8; ++n) {
        o[n][0] *= alA; o[n][1] *= alA; o[n][2] *= alB; o[n][3] *= alB;
      }
      // ---- O += P V: P (rows x 16 keys) as A fragments straight from the S
      // fragments (bf16 hi + lo), V as the B operand via ldmatrix.trans
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        uint32_t ph[4], pl[4];
        ph[0] = pack_bf16(sc[2 * j][0], sc[2 * j][1]);
        ph[1] = pack_bf16(sc[2 * j][2], sc[2 * j][3]);
        ph[2] = pack_bf16(sc[2 * j + 1][0], sc[2 * j + 1][1]);
        ph[3] = pack_bf16(sc[2 * j + 1][2], sc[2 * j + 1][3]);
        pl[0] = pack_bf16(sc[2 * j][0] - bf16_lo_f(ph[0]), sc[2 * j][1] - bf16_hi_f(ph[0]));
        pl[1] = pack_bf16(sc[2 * j][2] - bf16_lo_f(ph[1]), sc[2 * j][3] - bf16_hi_f(ph[1]));
        pl[2] = pack_bf16(sc[2 * j + 1][0] - bf16_lo_f(ph[2]), sc[2 * j + 1][1] - bf16_hi_f(ph[2]));
        pl[3] = pack_bf16(sc[2 * j + 1][2] - bf16_lo_f(ph[3]), sc[2 * j + 1][3] - bf16_hi_f(ph[3]));
        const int key = j * 16 + (mi & 1) * 8 + (lane & 7);
        const int rot = (int)((kp0 + key) & 7);
#pragma unroll
        for (int dp = 0; dp < D / 16; ++dp) {
          uint32_t vb[4];
          ldsm_x4_t(stg + arot<D>(key, D / 8 + 2 * dp + (mi >> 1), rot), vb);
          mma_bf16(o[2 * dp], ph, vb[0], vb[1]);
          mma_bf16(o[2 * dp], pl, vb[0], vb[1]);
          mma_bf16(o[2 * dp + 1], ph, vb[2], vb[3]);
          mma_bf16(o[2 * dp + 1], pl, vb[2], vb[3]);
        }
      }
    } else {
      // ---- pass 2: final weights of the rows, staged for the per-head means
#pragma unroll
      for (int n = 0; n < 4; ++n) {
        const int k0 = n * 8 + 2 * t4;
        wbuf[(r0 + g4) * AK + k0] = sc[n][0] == -INFINITY ? 0.f : __expf(sc[n][0] - fmA) * rzA;
        wbuf[(r0 + g4) * AK + k0 + 1] = sc[n][1] == -INFINITY ? 0.f : __expf(sc[n][1] - fmA) * rzA;
        wbuf[(r0 + g4 + 8) * AK + k0] = sc[n][2] == -INFINITY ? 0.f : __expf(sc[n][2] - fmB) * rzB;
        wbuf[(r0 + g4 + 8) * AK + k0 + 1] = sc[n][3] == -INFINITY ? 0.f : __expf(sc[n][3] - fmB) * rzB;
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);  // stage consumed
    if constexpr (PASS == 2) {
      // all consumers' weights of this stage are in wbuf: per (query head of
      // this row group, key) the mean over the head's nq rows, in row order
      asm volatile("bar.sync 1, %0;\n" ::"r"(NW * 32) : "memory");
      for (int j = 0; j < n_mt; ++j) {
        if (kp0 + mkey[j] >= p1) continue;
        float acc = 0.f;
        for (int i = 0; i < (int)a.nq; ++i) acc += wbuf[(mrow[j] + i) * AK + mkey[j]];
        a.mean[seg][mdst[j] + kp0] = acc * inv_nq;
      }
      asm volatile("bar.sync 1, %0;\n" ::"r"(NW * 32) : "memory");
    }
  }
  if constexpr (PASS == 1) {
    // partial (m, z, acc) of this item's rows
    const int64_t item = blockIdx.x;
    if (t4 == 0) {
      if (r0 + g4 < a.RG) {
        a.part_m[item * a.RG + r0 + g4] = mA;
        a.part_z[item * a.RG + r0 + g4] = zA;
      }
      if (r0 + g4 + 8 < a.RG) {
        a.part_m[item * a.RG + r0 + g4 + 8] = mB;
        a.part_z[item * a.RG + r0 + g4 + 8] = zB;
      }
    }
    float* pa = a.part_acc + item * a.RG * D;
#pragma unroll
    for (int n = 0; n < D / 8; ++n) {
      const int c = n * 8 + 2 * t4;
      if (r0 + g4 < a.RG) { pa[(r0 + g4) * D + c] = o[n][0]; pa[(r0 + g4) * D + c + 1] = o[n][1]; }
      if (r0 + g4 + 8 < a.RG) { pa[(r0 + g4 + 8) * D + c] = o[n][2]; pa[(r0 + g4 + 8) * D + c + 1] = o[n][3]; }
    }
  }
}

// ------------------------------------------------------------------ tcgen05 pass 1
// Same work items and partial outputs as append_attend_kernel<D, 1>, with
// both GEMMs on the 5th-generation tensor cores (D = 128, row groups of 128):
//   warp 0  TMA: the row group's Q once (two 64-column 128-byte-swizzled
//           atoms, 128 rows), then per stage of 64 keys four 64x64 boxes
//           K0 K1 V0 V1 into a 3-stage ring. bf16 rows are stored rotated by
//           position (16-byte chunk c at c ^ (p & 7) inside each 128-byte
//           segment), which IS the 128-byte swizzle of an 8-row-aligned box:
//           stages start at positions rounded down to 8 (the extra keys are
//           masked), so the tiles are canonical SW128 operands as loaded.
//   warp 1  one thread issues S = Q K^T on tcgen05 (M 128, N 64, K-major
//           operands) into a double-buffered TMEM tile; warp 6 one thread
//           issues O += P V (V as the MN-major B operand; P = bf16 hi + lo)
//           into the TMEM accumulator; tcgen05.commit drives the mbarriers.
//   warps 2-5  one thread per row (its TMEM lane): tcgen05.ld the S row,
//           scale + mask, fp32 softmax against a per-row reference max that
//           is only raised when a score exceeds it by more than 8 (p <= e^8,
//           so P and O stay in range); raising it rescales the row's O in
//           TMEM (ld, scale, st -- warp-collective, after the previous P V
//           completed), which happens a few times per row, not per stage.
//           P rows (hi, lo) go to shared memory in the SW128 layout.
// (m, z, acc) per row as the mma.sync kernel writes them (m is the reference
// max: z and acc are relative to it, which is all the fold needs).
constexpr int T5_KEYS = 64;  // keys per stage
#ifndef HGCA_T5_STAGES
#define HGCA_T5_STAGES 4
#endif
constexpr int T5_S = HGCA_T5_STAGES;  // K|V stages in the ring
constexpr float T5_HEADROOM2 = 8.f * 1.4426950408889634f;  // e^8 of headroom, in log2 units

__device__ __forceinline__ float ex2_approx(float x) {  // 2^x; 2^-inf = +0
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// max / sum of a register row with 8 independent chains (a serial chain of
// N dependent FMNMX / FADD was a large part of the per-stage softmax latency)
template <int N>
__device__ __forceinline__ float row_max8(const float (&x)[N]) {
  static_assert(N % 8 == 0, "row_max8");
  float m[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) m[i] = x[i];
#pragma unroll
  for (int j = 8; j < N; j += 8)
#pragma unroll
    for (int i = 0; i < 8; ++i) m[i] = fmaxf(m[i], x[j + i]);
  return fmaxf(fmaxf(fmaxf(m[0], m[1]), fmaxf(m[2], m[3])), fmaxf(fmaxf(m[4], m[5]), fmaxf(m[6], m[7])));
}
template <int N>
__device__ __forceinline__ float row_sum8(const float (&x)[N]) {
  float m[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) m[i] = x[i];
#pragma unroll
  for (int j = 8; j < N; j += 8)
#pragma unroll
    for (int i = 0; i < 8; ++i) m[i] += x[j + i];
  return ((m[0] + m[1]) + (m[2] + m[3])) + ((m[4] + m[5]) + (m[6] + m[7]));
}

struct Tc5Cfg {               // D = 128
  static constexpr int QATOM = 128 * 128;               // 128 rows x 64 bf16 (16 KB)
  static constexpr int KVQ = T5_KEYS * 128;             // 64 keys x 64 bf16 (8 KB)
  static constexpr int STAGE = 4 * KVQ;                 // K0 K1 V0 V1
  static constexpr int PBUF = 128 * 128;                // 128 rows x 64 keys bf16
  static constexpr int OFF_Q = 0;
  static constexpr int OFF_KV = OFF_Q + 2 * QATOM;
  static constexpr int OFF_P = OFF_KV + T5_S * STAGE;   // [2 buffers][hi, lo]
  static constexpr int OFF_BAR = OFF_P + 4 * PBUF;
  static constexpr int NBAR = 1 + 2 * T5_S + 8;         // qfull, full[S], empty[S], sfull[2], pfull[2], pvdone[2], sfree[2]
  static constexpr int OFF_TM = OFF_BAR + NBAR * 8;
  static constexpr int SMEM = OFF_TM + 16 + 1024;       // + alignment slack
  static constexpr int TMEM_COLS = 256;                 // S[2] x 64 | O 128
  static constexpr int THREADS = 7 * 32;               // TMA, QK issuer, 4 softmax warps, PV issuer
};

#ifdef HGCA_TC5_PROF
// debug build: cycle counters summed over CTAs (softmax warp 2): [3] wait sfull,
// [4] wait pvdone, [5] total, [6] stages
__device__ unsigned long long g_tc5prof[8];
#define P5(...) __VA_ARGS__
#else
#define P5(...)
#endif
template <int NCP>  // copies of the row group in the tile: 1, or 2 / 4 in split-key mode
__global__ void __launch_bounds__(Tc5Cfg::THREADS, 1) append_tc5_kernel(const __grid_constant__ AppendArgs a) {
  using C = Tc5Cfg;
  constexpr int D = 128;
  constexpr uint32_t O_COL = 2 * T5_KEYS;
  extern __shared__ unsigned char sm_raw[];
  unsigned char* sm = smem_align1024(sm_raw);
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + C::OFF_BAR);
  uint64_t* qfull = bars;
  uint64_t* full = bars + 1;
  uint64_t* empty = full + T5_S;
  uint64_t* sfull = empty + T5_S;
  uint64_t* pfull = sfull + 2;
  uint64_t* pvdone = pfull + 2;
  uint64_t* sfree = pvdone + 2;  // S buffer read out of TMEM by every softmax warp (QK may overwrite it)
  uint32_t* tm_holder = reinterpret_cast<uint32_t*>(sm + C::OFF_TM);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int64_t bk, rg, chunk;
  int seg;
  append_item(a, blockIdx.x, bk, rg, seg, chunk);
  const int64_t p0 = a.seg_lo[seg] + chunk * ACHUNK;
  const int64_t p1 = min(a.seg_hi[seg], p0 + ACHUNK);
  const int64_t p0a = p0 & ~(int64_t)7;  // 8-aligned stage base: rotation == swizzle phase
  const int nst = (int)((p1 - p0a + T5_KEYS - 1) / T5_KEYS);
  // split-key mode for groups of <= 64 rows: the group is loaded ncp = 2
  // or 4 times (TMEM lanes 0-63 / 64-127, or one lane quarter per copy), copy c's
  // softmax threads take keys [c * 64 / ncp, (c + 1) * 64 / ncp) of every stage
  // (the rest of their P row stays zero), so all four softmax warps work and
  // each row's per-stage chain is 1 / ncp; the copies' (m, z, O) are merged in
  // the epilogue
  constexpr int ncp = NCP;
  constexpr bool dup = ncp > 1;
  const int nsw = dup ? 4 : (int)((a.RG + 31) / 32);
  if (threadIdx.x == 0) {
    mbar_init(qfull, 1);
    for (int s = 0; s < T5_S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&sfull[b], 1);
      mbar_init(&pfull[b], nsw);  // one arrive per softmax warp that owns rows
      mbar_init(&sfree[b], nsw);
    }
    mbar_init(&pvdone[0], 1);
    mbar_init(&pvdone[1], 1);
    fence_mbar_init();
  }
  // Row groups of < 128 rows (e.g. n_q = 16 at G = 4: 64 rows): the softmax
  // warps of the padding quarters skip the stages entirely; their P rows stay
  // zero (written once here), so the padding O rows are zero and unused.
  if (warp >= 2 && warp < 6 && !dup && (warp & 3) * 32 >= a.RG) {
    const int r = (warp & 3) * 32 + lane;
    unsigned char* prow0 = sm + C::OFF_P + (r >> 3) * 1024 + (r & 7) * 128;
#pragma unroll
    for (int bb = 0; bb < 4; ++bb)
#pragma unroll
      for (int c = 0; c < 8; ++c) *reinterpret_cast<uint4*>(prow0 + bb * C::PBUF + c * 16) = make_uint4(0, 0, 0, 0);
    umma::fence_smem_async();
  }
  if (warp >= 2 && warp < 6 && dup) {  // split keys: zero the part of each P row this copy never writes
    const int L = (warp & 3) * 32 + lane, cp = (warp & 3) * ncp / 4, cpc = 8 / ncp;  // 16-byte chunks per copy
    unsigned char* prow0 = sm + C::OFF_P + (L >> 3) * 1024 + (L & 7) * 128;
#pragma unroll
    for (int bb = 0; bb < 4; ++bb)
#pragma unroll
      for (int c = 0; c < 8; ++c)
        if (c / cpc != cp)
          *reinterpret_cast<uint4*>(prow0 + bb * C::PBUF + ((c ^ (L & 7)) << 4)) = make_uint4(0, 0, 0, 0);
    umma::fence_smem_async();
  }
  if (warp == 1) umma::tmem_alloc<C::TMEM_COLS>(smem_u32(tm_holder));
  umma::fence_before_sync();
  __syncthreads();
  umma::fence_after_sync();
  const uint32_t tmem = *tm_holder;
  const uint32_t sQ = smem_u32(sm + C::OFF_Q), sKV = smem_u32(sm + C::OFF_KV), sP = smem_u32(sm + C::OFF_P);

  if (warp == 0) {  // ------------------------------------------------ TMA producer
    if (lane == 0) {
      const uint64_t policy = l2_evict_first_policy();
      const int64_t b = bk / a.Hkv, kvh = bk % a.Hkv;
      const int qrow = (int)((b * a.Hq + kvh * a.G) * a.nq + rg * a.RG);
      mbar_expect_tx(qfull, 2 * C::QATOM);
      if (dup) {  // the group at lanes 0, 128 / ncp, ...: same swizzle phase (multiples of 1 KB apart)
        for (int h = 0; h < 2; ++h)
          for (int cp = 0; cp < ncp; ++cp)
            tma_load_2d(sQ + h * C::QATOM + cp * (128 / ncp) * 128, &a.qmap5h, 64 * h, qrow, qfull, policy);
      } else {
        tma_load_2d(sQ, &a.qmap5, 0, qrow, qfull, policy);
        tma_load_2d(sQ + C::QATOM, &a.qmap5, 64, qrow, qfull, policy);
      }
      const int rowbase = (int)(bk * a.T + p0a);
      for (int st = 0; st < nst; ++st) {
        const int s = st % T5_S;
        if (st >= T5_S) mbar_wait(&empty[s], ((st / T5_S) - 1) & 1);
        mbar_expect_tx(&full[s], C::STAGE);
#pragma unroll
        for (int qd = 0; qd < 4; ++qd)
          tma_load_2d(sKV + s * C::STAGE + qd * C::KVQ, &a.kvmap5, qd * 64, rowbase + st * T5_KEYS, &full[s], policy);
      }
    }
  } else if (warp == 1 || warp == 6) {  // ----------------------------- MMA issuers
    // two issuing threads (tcgen05.mma issue costs tens of cycles each):
    // warp 1 issues S = Q K^T, warp 6 issues O += P V
    if (lane == 0) {
      constexpr uint32_t IDESC_QK = umma::idesc_bf16_f32(128, T5_KEYS, false, false);
      constexpr uint32_t IDESC_PV = umma::idesc_bf16_f32(128, D, false, true);
      if (warp == 1) {
        mbar_wait(qfull, 0);
        umma::fence_after_sync();
        for (int st = 0; st < nst; ++st) {
          const int s = st % T5_S, b = st & 1;
          mbar_wait(&full[s], (st / T5_S) & 1);
          // S buffer b was read out of TMEM by softmax(st-2)
          if (st >= 2) mbar_wait(&sfree[b], ((st - 2) >> 1) & 1);
          umma::fence_after_sync();
          const uint32_t kb = sKV + s * C::STAGE;
#pragma unroll
          for (int k = 0; k < D / 16; ++k) {
            const uint64_t ad = umma::smem_desc(sQ + (k / 4) * C::QATOM + (k % 4) * 32, 16, 1024);
            const uint64_t bd = umma::smem_desc(kb + (k / 4) * C::KVQ + (k % 4) * 32, 16, 1024);
            umma::mma_bf16(tmem + b * T5_KEYS, ad, bd, IDESC_QK, k > 0);
          }
          umma::commit(smem_u32(&sfull[b]));
        }
      } else {
        for (int st = 0; st < nst; ++st) {
          const int s = st % T5_S, b = st & 1;
          // P of stage st written (and so S = Q K^T of stage st complete)
          mbar_wait(&pfull[b], (st >> 1) & 1);
          umma::fence_after_sync();
          const uint32_t vb = sKV + s * C::STAGE + 2 * C::KVQ;  // V0 then V1: the two 64-column atoms
#pragma unroll
          for (int h = 0; h < 2; ++h) {  // P hi, P lo
            const uint32_t pb = sP + (b * 2 + h) * C::PBUF;
#pragma unroll
            for (int j = 0; j < T5_KEYS / 16; ++j) {
              const uint64_t ad = umma::smem_desc(pb + j * 32, 16, 1024);
              const uint64_t bd = umma::smem_desc(vb + j * 16 * 128, C::KVQ, 1024);
              umma::mma_bf16(tmem + O_COL, ad, bd, IDESC_PV, st > 0 || h > 0 || j > 0);
            }
          }
          umma::commit(smem_u32(&pvdone[b]));  // PV(st) -- and every earlier PV -- complete
          umma::commit(smem_u32(&empty[s]));   // K (read by QK(st), complete) and V free
        }
      }
    }
    __syncwarp();
  } else if (dup || (warp & 3) * 32 < a.RG) {  // -------------------- softmax warps (rows)
    const int quarter = warp & 3;
    const int L = quarter * 32 + lane;                   // TMEM lane == P row
    const int hh = dup ? quarter * ncp / 4 : 0;          // split keys: this thread's copy (part of each stage)
    const int r = dup ? L % (128 / ncp) : L;             // row of the group
    const uint32_t tl = (uint32_t)(quarter * 32) << 16;
    // softmax in log2 units: x = s * log2(e), p = 2^(x - mu2) == exp(s - mu2 * ln 2)
    const float sl2 = a.scale * 1.4426950408889634f;
    float mu2 = -INFINITY, z = 0.f;             // reference max (log2 units), sum of p
    const uint32_t prow = (uint32_t)((L >> 3) * 1024 + (L & 7) * 128);
    P5(long long w_s = 0, w_pv = 0, t_s0 = clock64();)
    auto stages = [&](auto nk_c) {
      constexpr int NK = decltype(nk_c)::value;  // keys of a stage this thread takes
      for (int st = 0; st < nst; ++st) {
        const int b = st & 1;
        P5(long long c0 = clock64();)
        mbar_wait(&sfull[b], (st >> 1) & 1);
        P5(w_s += clock64() - c0;)
        umma::fence_after_sync();
        float x[NK];
        {
          uint32_t v[NK / 16][16];  // all loads in flight, one wait
#pragma unroll
          for (int c = 0; c < NK / 16; ++c) umma::ld_32x32b_x16(tmem + tl + b * T5_KEYS + hh * NK + c * 16, v[c]);
          umma::ld_wait();
          umma::fence_before_sync();
          __syncwarp();
          if (lane == 0) mbar_arrive(&sfree[b]);  // S(st) is in registers: QK(st + 2) may overwrite it
#pragma unroll
          for (int c = 0; c < NK / 16; ++c)
#pragma unroll
            for (int j = 0; j < 16; ++j) x[c * 16 + j] = __uint_as_float(v[c][j]);
        }
        const int64_t kp0 = p0a + (int64_t)st * T5_KEYS + hh * NK;
        if (!(kp0 >= p0 && kp0 + NK <= p1)) {  // a partial part (warp-uniform): mask the keys out of range
          const int jlo = (int)max(min(p0 - kp0, (int64_t)NK), (int64_t)0);
          const int jhi = (int)max(min(p1 - kp0, (int64_t)NK), (int64_t)0);
#pragma unroll
          for (int j = 0; j < NK; ++j) x[j] = (j >= jlo && j < jhi) ? x[j] : -INFINITY;
        }
        const float mx = row_max8(x) * sl2;  // the scale is positive: max commutes with it
        float alpha = 1.f;
        if (mx > mu2 + T5_HEADROOM2) {  // raise the reference max (also the first finite score)
          alpha = mu2 == -INFINITY ? 0.f : ex2_approx(mu2 - mx);
          mu2 = mx;
        }
        const float mref = mu2 == -INFINITY ? 0.f : mu2;  // a split-key half may not have seen a key yet
#pragma unroll
        for (int j = 0; j < NK; ++j) x[j] = ex2_approx(fmaf(x[j], sl2, -mref));  // masked keys: 2^-inf = 0
        z = z * alpha + row_sum8(x);
        // P buffer b was last read by PV(st-2)
        P5(long long c1 = clock64();)
        if (st >= 2) mbar_wait(&pvdone[b], ((st - 2) >> 1) & 1);
        P5(w_pv += clock64() - c1;)
        if (st >= 1 && __any_sync(FULL_MASK, alpha != 1.f)) {
          // rescale the rows' O once PV(st-1) has completed (PV(st) waits for this
          // stage's P, released below); warp-collective TMEM ld / st
          mbar_wait(&pvdone[b ^ 1], ((st - 1) >> 1) & 1);
          umma::fence_after_sync();
          {
#pragma unroll
            for (int c0 = 0; c0 < D; c0 += 16) {
              uint32_t v[16];
              umma::ld_32x32b_x16(tmem + tl + O_COL + c0, v);
              umma::ld_wait();
#pragma unroll
              for (int j = 0; j < 16; ++j) v[j] = __float_as_uint(__uint_as_float(v[j]) * alpha);
              umma::st_32x32b_x16(tmem + tl + O_COL + c0, v);
            }
            umma::st_wait();
          }
        }
        unsigned char* ph = sm + C::OFF_P + (b * 2) * C::PBUF + prow;
        unsigned char* pl = ph + C::PBUF;
#pragma unroll
        for (int c = 0; c < NK / 8; ++c) {
          uint32_t hi[4], lo[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            hi[e] = pack_bf16(x[c * 8 + 2 * e], x[c * 8 + 2 * e + 1]);
            lo[e] = pack_bf16(x[c * 8 + 2 * e] - bf16_lo_f(hi[e]), x[c * 8 + 2 * e + 1] - bf16_hi_f(hi[e]));
          }
          const uint32_t off = (uint32_t)(((hh * (NK / 8) + c) ^ (L & 7)) << 4);
          *reinterpret_cast<uint4*>(ph + off) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
          *reinterpret_cast<uint4*>(pl + off) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
        }
        umma::fence_smem_async();  // P (generic stores) -> visible to the tensor core
        umma::fence_before_sync();
        __syncwarp();
        if (lane == 0) mbar_arrive(&pfull[b]);
      }
    };
    stages(std::integral_constant<int, T5_KEYS / NCP>{});
    mbar_wait(&pvdone[(nst - 1) & 1], ((nst - 1) >> 1) & 1);  // the last PV (and all before it)
    P5(if (warp == 2 && lane == 0) { atomicAdd(&g_tc5prof[3], (unsigned long long)w_s);
       atomicAdd(&g_tc5prof[6], (unsigned long long)nst);
       atomicAdd(&g_tc5prof[4], (unsigned long long)w_pv); atomicAdd(&g_tc5prof[5], (unsigned long long)(clock64() - t_s0)); })
    umma::fence_after_sync();
    // this row's partial (m, z, acc), as append_attend_kernel<D, 1> writes it;
    // split keys: the second copy (lanes 64-127) hands its (m, z, O) to the
    // first through shared memory (the P buffers: every PV is complete)
    // split keys: copies 1.. hand their (m, z, O) to copy 0 through shared
    // memory (the P buffers: every PV is complete); copy 0 merges them
    const int rw = 128 / ncp;                             // rows per copy (lanes)
    float* ob = reinterpret_cast<float*>(sm + C::OFF_P);  // [copy - 1][D][rw] column-major: conflict-free
    float* mzb = ob + 3 * D * 32;                         // [copy - 1][rw][2] (past the largest O area)
    float fc[4] = {1.f, 0.f, 0.f, 0.f};
    if (dup) {
      // (ordered already through pfull -> PV -> pvdone; the barrier makes the
      // P-region reuse explicit for the race checker, once per CTA)
      asm volatile("bar.sync 1, 128;\n" ::: "memory");
      if (hh) {
        float* obc = ob + (hh - 1) * D * rw;
#pragma unroll
        for (int c0 = 0; c0 < D; c0 += 16) {
          uint32_t v[16];
          umma::ld_32x32b_x16(tmem + tl + O_COL + c0, v);
          umma::ld_wait();
#pragma unroll
          for (int j = 0; j < 16; ++j) obc[(c0 + j) * rw + r] = __uint_as_float(v[j]);
        }
        mzb[((hh - 1) * rw + r) * 2] = mu2;
        mzb[((hh - 1) * rw + r) * 2 + 1] = z;
      }
      asm volatile("bar.sync 1, 128;\n" ::: "memory");  // the four softmax warps
      if (!hh) {
        float mc[4] = {mu2, -INFINITY, -INFINITY, -INFINITY}, zc[4] = {z, 0.f, 0.f, 0.f};
        float mm = mu2;
#pragma unroll
        for (int c = 1; c < 4; ++c)
          if (c < ncp) {
            mc[c] = mzb[((c - 1) * rw + r) * 2];
            zc[c] = mzb[((c - 1) * rw + r) * 2 + 1];
            mm = fmaxf(mm, mc[c]);
          }
        z = 0.f;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          fc[c] = (c < ncp && mc[c] != -INFINITY) ? ex2_approx(mc[c] - mm) : 0.f;
          z += zc[c] * fc[c];
        }
        mu2 = mm;
      }
    }
    const bool mine = (!dup || !hh) && r < a.RG && rg * a.RG + r < a.R;
    const int64_t item = blockIdx.x;
    float4* pa = reinterpret_cast<float4*>(a.part_acc + (item * a.RG + r) * D);
    if (!dup || !hh) {
#pragma unroll
      for (int c0 = 0; c0 < D; c0 += 16) {
        uint32_t v[16];
        umma::ld_32x32b_x16(tmem + tl + O_COL + c0, v);
        umma::ld_wait();
        float o[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          float acc = __uint_as_float(v[j]) * fc[0];
#pragma unroll
          for (int c = 1; c < 4; ++c)  // unrolled: the copies' loads are independent
            if (c < ncp) acc += ob[((c - 1) * D + c0 + j) * rw + r] * fc[c];
          o[j] = dup ? acc : __uint_as_float(v[j]);
        }
        if (mine) {
#pragma unroll
          for (int j = 0; j < 16; j += 4) pa[(c0 + j) / 4] = make_float4(o[j], o[j + 1], o[j + 2], o[j + 3]);
        }
      }
    }
    if (mine) {
      a.part_m[item * a.RG + r] = mu2 == -INFINITY ? -INFINITY : mu2 * 0.6931471805599453f;  // natural-log units
      a.part_z[item * a.RG + r] = z;
    }
  }
  umma::fence_before_sync();
  __syncthreads();
  if (warp == 1) umma::tmem_dealloc<C::TMEM_COLS>(tmem);
}

// ------------------------------------------------------------------ tcgen05 pass 1, two tiles
// For (batch, kv-head)s with >= 2 row groups of 128 (G * n_q >= 256): one CTA
// takes two row groups (tiles) against the same keys, so each K|V stage is
// loaded once for both, and the tiles' softmax warps (4 each) run side by side
// while the tensor core works on the other tile (as FA4 ping-pongs two Q tiles).
// Per tile: S double-buffered in TMEM; P (bf16 hi, lo: 32 + 32 columns) is
// written back over its own S buffer and P V reads the A operand from TMEM
// (no shared-memory P, so a tile's softmax never waits for its previous P V
// except to rescale O; the freed shared memory holds more K|V stages); O in TMEM.
#ifndef HGCA_X2_STAGES
#define HGCA_X2_STAGES 4
#endif
struct Tc5x2Cfg {              // D = 128
  static constexpr int QATOM = 128 * 128;
  static constexpr int KVQ = T5_KEYS * 128;
  static constexpr int S = HGCA_X2_STAGES;
  static constexpr int STAGE = 4 * KVQ;                 // K0 K1 V0 V1
  static constexpr int OFF_Q = 0;                       // [tile][2 atoms]
  static constexpr int OFF_KV = OFF_Q + 4 * QATOM;
  static constexpr int OFF_BAR = OFF_KV + S * STAGE;    // (P lives in TMEM, over S)
  static constexpr int NBAR = 1 + 2 * S + 2 + 8;        // qfull, full[S], empty[S], sfull[2], pfull[2][2], pvdone[2][2]
  static constexpr int OFF_TM = OFF_BAR + NBAR * 8;
  static constexpr int SMEM = OFF_TM + 16 + 1024;
  static constexpr int TMEM_COLS = 512;                 // S[2 tiles][2] x 64 | O[2 tiles] x 128
  static constexpr int THREADS = 11 * 32;               // TMA, QK, softmax 2-5 (tile 0), PV, softmax 7-10 (tile 1)
};

__global__ void __launch_bounds__(Tc5x2Cfg::THREADS, 1) append_tc5x2_kernel(const __grid_constant__ AppendArgs a) {
  using C = Tc5x2Cfg;
  constexpr int D = 128;
  constexpr uint32_t O_COL = 4 * T5_KEYS;
  extern __shared__ unsigned char sm_raw[];
  unsigned char* sm = smem_align1024(sm_raw);
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + C::OFF_BAR);
  uint64_t* qfull = bars;
  uint64_t* full = bars + 1;
  uint64_t* empty = full + C::S;
  uint64_t* sfull = empty + C::S;
  uint64_t* pfull = sfull + 2;   // [tile][parity]
  uint64_t* pvdone = pfull + 4;  // [tile][parity]
  uint32_t* tm_holder = reinterpret_cast<uint32_t*>(sm + C::OFF_TM);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // item -> (bk, tile pair, segment, chunk)
  const int64_t nc = a.nch[0] + a.nch[1], npair = (a.n_rg + 1) / 2;
  const int64_t cidx = blockIdx.x % nc, t_ = blockIdx.x / nc;
  const int64_t pair = t_ % npair, bk = t_ / npair;
  const int seg = cidx < a.nch[0] ? 0 : 1;
  const int64_t chunk = seg ? cidx - a.nch[0] : cidx;
  bool valid[2];
  valid[0] = true;
  valid[1] = 2 * pair + 1 < a.n_rg;
  const int64_t p0 = a.seg_lo[seg] + chunk * ACHUNK;
  const int64_t p1 = min(a.seg_hi[seg], p0 + ACHUNK);
  const int64_t p0a = p0 & ~(int64_t)7;
  const int nst = (int)((p1 - p0a + T5_KEYS - 1) / T5_KEYS);
  if (threadIdx.x == 0) {
    mbar_init(qfull, 1);
    for (int s = 0; s < C::S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int i = 0; i < 2; ++i) mbar_init(&sfull[i], 1);
    for (int i = 0; i < 4; ++i) {
      mbar_init(&pfull[i], 4);
      mbar_init(&pvdone[i], 1);
    }
    fence_mbar_init();
  }
  if (warp == 1) umma::tmem_alloc<C::TMEM_COLS>(smem_u32(tm_holder));
  umma::fence_before_sync();
  __syncthreads();
  umma::fence_after_sync();
  const uint32_t tmem = *tm_holder;
  const uint32_t sQ = smem_u32(sm + C::OFF_Q), sKV = smem_u32(sm + C::OFF_KV);

  if (warp == 0) {  // ------------------------------------------------ TMA producer
    if (lane == 0) {
      const uint64_t policy = l2_evict_first_policy();
      const int64_t b = bk / a.Hkv, kvh = bk % a.Hkv;
      const int nt = valid[1] ? 2 : 1;
      mbar_expect_tx(qfull, nt * 2 * C::QATOM);
      for (int t = 0; t < nt; ++t) {
        const int qrow = (int)((b * a.Hq + kvh * a.G) * a.nq + (2 * pair + t) * a.RG);
        tma_load_2d(sQ + t * 2 * C::QATOM, &a.qmap5, 0, qrow, qfull, policy);
        tma_load_2d(sQ + t * 2 * C::QATOM + C::QATOM, &a.qmap5, 64, qrow, qfull, policy);
      }
      const int rowbase = (int)(bk * a.T + p0a);
      for (int st = 0; st < nst; ++st) {
        const int s = st % C::S;
        if (st >= C::S) mbar_wait(&empty[s], ((st / C::S) - 1) & 1);
        mbar_expect_tx(&full[s], C::STAGE);
#pragma unroll
        for (int qd = 0; qd < 4; ++qd)
          tma_load_2d(sKV + s * C::STAGE + qd * C::KVQ, &a.kvmap5, qd * 64, rowbase + st * T5_KEYS, &full[s], policy);
      }
    }
  } else if (warp == 1 || warp == 6) {  // ----------------------------- MMA issuers
    if (lane == 0) {
      constexpr uint32_t IDESC_QK = umma::idesc_bf16_f32(128, T5_KEYS, false, false);
      constexpr uint32_t IDESC_PV = umma::idesc_bf16_f32(128, D, false, true);
      if (warp == 1) {  // S = Q K^T for both tiles
        mbar_wait(qfull, 0);
        umma::fence_after_sync();
        for (int st = 0; st < nst; ++st) {
          const int s = st % C::S, b = st & 1;
          mbar_wait(&full[s], (st / C::S) & 1);
          for (int t = 0; t < 2; ++t)  // S[t][b] holds P(st-2) until the tile's PV(st-2) has read it
            if (valid[t] && st >= 2) mbar_wait(&pvdone[t * 2 + b], ((st - 2) >> 1) & 1);
          umma::fence_after_sync();
          const uint32_t kb = sKV + s * C::STAGE;
          for (int t = 0; t < 2; ++t) {
            if (!valid[t]) continue;
#pragma unroll
            for (int k = 0; k < D / 16; ++k) {
              const uint64_t ad = umma::smem_desc(sQ + t * 2 * C::QATOM + (k / 4) * C::QATOM + (k % 4) * 32, 16, 1024);
              const uint64_t bd = umma::smem_desc(kb + (k / 4) * C::KVQ + (k % 4) * 32, 16, 1024);
              umma::mma_bf16(tmem + (t * 2 + b) * T5_KEYS, ad, bd, IDESC_QK, k > 0);
            }
          }
          umma::commit(smem_u32(&sfull[b]));
        }
      } else {  // O[t] += P[t] V
        for (int st = 0; st < nst; ++st) {
          const int s = st % C::S, b = st & 1;
          const uint32_t vb = sKV + s * C::STAGE + 2 * C::KVQ;
          for (int t = 0; t < 2; ++t) {
            if (!valid[t]) continue;
            mbar_wait(&pfull[t * 2 + b], (st >> 1) & 1);
            umma::fence_after_sync();
#pragma unroll
            for (int h = 0; h < 2; ++h) {  // P hi in columns 0-31 of S[t][b], P lo in 32-63
#pragma unroll
              for (int j = 0; j < T5_KEYS / 16; ++j) {
                const uint64_t bd = umma::smem_desc(vb + j * 16 * 128, C::KVQ, 1024);
                umma::mma_bf16_ts(tmem + O_COL + t * D, tmem + (t * 2 + b) * T5_KEYS + h * 32 + j * 8, bd, IDESC_PV,
                                  st > 0 || h > 0 || j > 0);
              }
            }
            umma::commit(smem_u32(&pvdone[t * 2 + b]));
          }
          umma::commit(smem_u32(&empty[s]));  // both tiles' QK (complete) and PV of this stage
        }
      }
    }
    __syncwarp();
  } else {  // ------------------------------------------------------- softmax warps
    const int t = warp >= 7 ? 1 : 0;
    if (valid[t]) {
      const int quarter = warp & 3;
      const int r = quarter * 32 + lane;
      const uint32_t tl = (uint32_t)(quarter * 32) << 16;
      const float sl2 = a.scale * 1.4426950408889634f;
      float mu2 = -INFINITY, z = 0.f;
      for (int st = 0; st < nst; ++st) {
        const int b = st & 1;
        mbar_wait(&sfull[b], (st >> 1) & 1);
        umma::fence_after_sync();
        float x[T5_KEYS];
        {
          uint32_t v[4][16];
#pragma unroll
          for (int c = 0; c < 4; ++c) umma::ld_32x32b_x16(tmem + tl + (t * 2 + b) * T5_KEYS + c * 16, v[c]);
          umma::ld_wait();
#pragma unroll
          for (int c = 0; c < 4; ++c)
#pragma unroll
            for (int j = 0; j < 16; ++j) x[c * 16 + j] = __uint_as_float(v[c][j]);
        }
        const int64_t kp0 = p0a + (int64_t)st * T5_KEYS;
        if (!(kp0 >= p0 && kp0 + T5_KEYS <= p1)) {
          const int jlo = (int)max(p0 - kp0, (int64_t)0), jhi = (int)min(p1 - kp0, (int64_t)T5_KEYS);
#pragma unroll
          for (int j = 0; j < T5_KEYS; ++j) x[j] = (j >= jlo && j < jhi) ? x[j] : -INFINITY;
        }
        const float mx = row_max8(x) * sl2;
        float alpha = 1.f;
        if (mx > mu2 + T5_HEADROOM2) {
          alpha = mu2 == -INFINITY ? 0.f : ex2_approx(mu2 - mx);
          mu2 = mx;
        }
#pragma unroll
        for (int j = 0; j < T5_KEYS; ++j) x[j] = ex2_approx(fmaf(x[j], sl2, -mu2));
        z = z * alpha + row_sum8(x);
        if (st >= 1 && __any_sync(FULL_MASK, alpha != 1.f)) {
          // rescale O once the tile's PV(st-1) has completed (PV(st) waits for this stage's P)
          mbar_wait(&pvdone[t * 2 + (b ^ 1)], ((st - 1) >> 1) & 1);
          umma::fence_after_sync();
#pragma unroll
          for (int c0 = 0; c0 < D; c0 += 16) {
            uint32_t v[16];
            umma::ld_32x32b_x16(tmem + tl + O_COL + t * D + c0, v);
            umma::ld_wait();
#pragma unroll
            for (int j = 0; j < 16; ++j) v[j] = __float_as_uint(__uint_as_float(v[j]) * alpha);
            umma::st_32x32b_x16(tmem + tl + O_COL + t * D + c0, v);
          }
        }
        {  // P(st) as bf16 hi / lo pairs over this row's S columns: the A operand of PV from TMEM
          uint32_t hi[32], lo[32];
#pragma unroll
          for (int e = 0; e < 32; ++e) {
            hi[e] = pack_bf16(x[2 * e], x[2 * e + 1]);
            lo[e] = pack_bf16(x[2 * e] - bf16_lo_f(hi[e]), x[2 * e + 1] - bf16_hi_f(hi[e]));
          }
          const uint32_t sc = tmem + tl + (t * 2 + b) * T5_KEYS;
          umma::st_32x32b_x16(sc, *reinterpret_cast<const uint32_t(*)[16]>(&hi[0]));
          umma::st_32x32b_x16(sc + 16, *reinterpret_cast<const uint32_t(*)[16]>(&hi[16]));
          umma::st_32x32b_x16(sc + 32, *reinterpret_cast<const uint32_t(*)[16]>(&lo[0]));
          umma::st_32x32b_x16(sc + 48, *reinterpret_cast<const uint32_t(*)[16]>(&lo[16]));
          umma::st_wait();
        }
        umma::fence_before_sync();
        __syncwarp();
        if (lane == 0) mbar_arrive(&pfull[t * 2 + b]);
      }
      mbar_wait(&pvdone[t * 2 + ((nst - 1) & 1)], ((nst - 1) >> 1) & 1);
      umma::fence_after_sync();
      const int64_t rg = 2 * pair + t;
      const bool mine = r < a.RG && rg * a.RG + r < a.R;
      const int64_t item = (bk * a.n_rg + rg) * nc + cidx;  // the (bk, row group, segment, chunk) item
      float4* pa = reinterpret_cast<float4*>(a.part_acc + (item * a.RG + r) * D);
#pragma unroll
      for (int c0 = 0; c0 < D; c0 += 16) {
        uint32_t v[16];
        umma::ld_32x32b_x16(tmem + tl + O_COL + t * D + c0, v);
        umma::ld_wait();
        if (mine) {
#pragma unroll
          for (int j = 0; j < 16; j += 4)
            pa[(c0 + j) / 4] = make_float4(__uint_as_float(v[j]), __uint_as_float(v[j + 1]),
                                           __uint_as_float(v[j + 2]), __uint_as_float(v[j + 3]));
        }
      }
      if (mine) {
        a.part_m[item * a.RG + r] = mu2 == -INFINITY ? -INFINITY : mu2 * 0.6931471805599453f;
        a.part_z[item * a.RG + r] = z;
      }
    }
  }
  umma::fence_before_sync();
  __syncthreads();
  if (warp == 1) umma::tmem_dealloc<C::TMEM_COLS>(tmem);
}

// ------------------------------------------------------------------ tcgen05 pass 2
// The per-(query head, position) mean weights for a 128-row group on the
// tensor cores: S = Q K^T as in pass 1, the rows' final weights
// w = exp(s - m) / z (m, z from the fold), and the per-head sums as a GEMM,
// MEAN[head, key] = A . W with A[head, row] = 1 when the row belongs to the
// head (heads padded to M = 128, K = the 128 rows) and W [rows, 64 keys] as
// the MN-major B operand written by the row threads (bf16 hi + lo). Warp 4
// (TMEM lanes 0-31 = the heads) reads MEAN one stage behind and stores
// mean / n_q. Only K is loaded.
struct Tc5MCfg {               // D = 128
  static constexpr int QATOM = 128 * 128;
  static constexpr int KQ = T5_KEYS * 128;              // 64 keys x 64 bf16
  static constexpr int S = 4;                           // K stages
  static constexpr int STAGE = 2 * KQ;                  // K0 K1
  static constexpr int WBUF = 128 * 128;                // 128 rows x 64 keys bf16
  static constexpr int OFF_Q = 0;
  static constexpr int OFF_K = OFF_Q + 2 * QATOM;
  static constexpr int OFF_W = OFF_K + S * STAGE;       // [2 buffers][hi, lo]
  static constexpr int OFF_A = OFF_W + 4 * WBUF;        // head-membership matrix, 2 atoms
  static constexpr int OFF_BAR = OFF_A + 2 * QATOM;
  static constexpr int NBAR = 1 + 2 * S + 8;            // qfull, full[S], empty[S], sfull[2], wfull[2], mdone[2], sfree[2]
  static constexpr int OFF_TM = OFF_BAR + NBAR * 8;
  static constexpr int SMEM = OFF_TM + 16 + 1024;
  static constexpr int TMEM_COLS = 256;                 // S[2] x 64 | MEAN[2] x 64
  static constexpr int THREADS = 11 * 32;              // TMA, QK issuer, 4 row warps, GEMM issuer, 4 more row warps
};
// Row warps of pass 2: warps 2-5 and 7-10, two per TMEM lane quarter (warp w
// may only touch lanes 32*(w%4)..+31): the pair of a quarter splits every
// stage's 64 keys (half 0: warps 2-5, half 1: warps 7-10), so a row's
// per-stage work (S read, weights, W hi/lo) is halved. Quarters past the row
// group (e.g. rows 64-127 for n_q = 16 at G = 4) idle.
__device__ __forceinline__ bool tc5m_row_warp(int warp) { return (warp >= 2 && warp < 6) || warp >= 7; }
__device__ __forceinline__ int tc5m_half(int warp) { return warp >= 7 ? 1 : 0; }

__global__ void __launch_bounds__(Tc5MCfg::THREADS, 1) append_tc5_mean_kernel(const __grid_constant__ AppendArgs a) {
  using C = Tc5MCfg;
  constexpr int D = 128;
  constexpr uint32_t M_COL = 2 * T5_KEYS;
  extern __shared__ unsigned char sm_raw[];
  unsigned char* sm = smem_align1024(sm_raw);
  int64_t bk, rg, chunk;
  int seg;
  append_item(a, blockIdx.x, bk, rg, seg, chunk);
  if (!a.mean[seg]) return;  // (uniform) no means wanted for this segment
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + C::OFF_BAR);
  uint64_t* qfull = bars;
  uint64_t* full = bars + 1;
  uint64_t* empty = full + C::S;
  uint64_t* sfull = empty + C::S;
  uint64_t* wfull = sfull + 2;
  uint64_t* mdone = wfull + 2;
  uint64_t* sfree = mdone + 2;  // S buffer read out of TMEM by every row warp (QK may overwrite it)
  uint32_t* tm_holder = reinterpret_cast<uint32_t*>(sm + C::OFF_TM);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t p0 = a.seg_lo[seg] + chunk * ACHUNK;
  const int64_t p1 = min(a.seg_hi[seg], p0 + ACHUNK);
  const int64_t p0a = p0 & ~(int64_t)7;
  const int nst = (int)((p1 - p0a + T5_KEYS - 1) / T5_KEYS);
  const int nq = (int)a.nq, heads = (int)(a.RG / a.nq);
  const int64_t g0 = rg * a.RG / a.nq, b_ = bk / a.Hkv, kvh = bk % a.Hkv;
  if (threadIdx.x == 0) {
    mbar_init(qfull, 1);
    for (int s = 0; s < C::S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&sfull[b], 1);
      mbar_init(&wfull[b], 2 * (int)((a.RG + 31) / 32));  // one arrive per row warp that owns rows
      mbar_init(&sfree[b], 2 * (int)((a.RG + 31) / 32));
      mbar_init(&mdone[b], 1);
    }
    fence_mbar_init();
  }
  // padding quarters (row groups of < 128 rows): their W rows stay zero
  // (A is zero there too, but 0 * garbage could be NaN) and they skip the stages
  if (tc5m_row_warp(warp) && (warp & 3) * 32 >= a.RG) {
    const int r = (warp & 3) * 32 + lane, c0 = tc5m_half(warp) * 4;
    unsigned char* wrow0 = sm + C::OFF_W + (r >> 3) * 1024 + (r & 7) * 128;
#pragma unroll
    for (int bb = 0; bb < 4; ++bb)
#pragma unroll
      for (int c = c0; c < c0 + 4; ++c) *reinterpret_cast<uint4*>(wrow0 + bb * C::WBUF + c * 16) = make_uint4(0, 0, 0, 0);
  }
  if (warp >= 2 && warp < 6) {  // head-membership matrix A [128 heads][128 rows], K-major SW128 (row warps)
    const int h = threadIdx.x - 64;
    unsigned char* arow = sm + C::OFF_A + (h >> 3) * 1024 + (h & 7) * 128;
#pragma unroll
    for (int c = 0; c < 16; ++c) {  // 16-byte chunk c of the row: rows 8c .. 8c+7 (atom c / 8)
      uint32_t v[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int r0 = c * 8 + 2 * e;
        const float x0 = (h < heads && r0 / nq == h) ? 1.f : 0.f;
        const float x1 = (h < heads && (r0 + 1) / nq == h) ? 1.f : 0.f;
        v[e] = pack_bf16(x0, x1);
      }
      *reinterpret_cast<uint4*>(arow + (c >> 3) * C::QATOM + (((c & 7) ^ (h & 7)) << 4)) = make_uint4(v[0], v[1], v[2], v[3]);
    }
    umma::fence_smem_async();
  }
  if (warp == 1) umma::tmem_alloc<C::TMEM_COLS>(smem_u32(tm_holder));
  umma::fence_before_sync();
  __syncthreads();
  umma::fence_after_sync();
  const uint32_t tmem = *tm_holder;
  const uint32_t sQ = smem_u32(sm + C::OFF_Q), sK = smem_u32(sm + C::OFF_K), sW = smem_u32(sm + C::OFF_W),
                 sA = smem_u32(sm + C::OFF_A);

  if (warp == 0) {  // ------------------------------------------------ TMA producer
    if (lane == 0) {
      const uint64_t policy = l2_evict_first_policy();
      const int qrow = (int)((b_ * a.Hq + kvh * a.G) * a.nq + rg * a.RG);
      mbar_expect_tx(qfull, 2 * C::QATOM);
      tma_load_2d(sQ, &a.qmap5, 0, qrow, qfull, policy);
      tma_load_2d(sQ + C::QATOM, &a.qmap5, 64, qrow, qfull, policy);
      const int rowbase = (int)(bk * a.T + p0a);
      for (int st = 0; st < nst; ++st) {
        const int s = st % C::S;
        if (st >= C::S) mbar_wait(&empty[s], ((st / C::S) - 1) & 1);
        mbar_expect_tx(&full[s], C::STAGE);
        tma_load_2d(sK + s * C::STAGE, &a.kvmap5, 0, rowbase + st * T5_KEYS, &full[s], policy);
        tma_load_2d(sK + s * C::STAGE + C::KQ, &a.kvmap5, 64, rowbase + st * T5_KEYS, &full[s], policy);
      }
    }
  } else if (warp == 1 || warp == 6) {  // ----------------------------- MMA issuers
    // warp 1 issues S = Q K^T, warp 6 the head-sum GEMM MEAN = A . W
    if (lane == 0) {
      constexpr uint32_t IDESC_QK = umma::idesc_bf16_f32(128, T5_KEYS, false, false);
      constexpr uint32_t IDESC_M = umma::idesc_bf16_f32(128, T5_KEYS, false, true);
      if (warp == 1) {
        mbar_wait(qfull, 0);
        umma::fence_after_sync();
        for (int st = 0; st < nst; ++st) {
          const int s = st % C::S, b = st & 1;
          mbar_wait(&full[s], (st / C::S) & 1);
          if (st >= 2) mbar_wait(&sfree[b], ((st - 2) >> 1) & 1);  // S buffer b read out by the rows of stage st-2
          umma::fence_after_sync();
          const uint32_t kb = sK + s * C::STAGE;
#pragma unroll
          for (int k = 0; k < D / 16; ++k) {
            const uint64_t ad = umma::smem_desc(sQ + (k / 4) * C::QATOM + (k % 4) * 32, 16, 1024);
            const uint64_t bd = umma::smem_desc(kb + (k / 4) * C::KQ + (k % 4) * 32, 16, 1024);
            umma::mma_bf16(tmem + b * T5_KEYS, ad, bd, IDESC_QK, k > 0);
          }
          umma::commit(smem_u32(&sfull[b]));
          umma::commit(smem_u32(&empty[s]));  // K is read by this GEMM only
        }
      } else {
        const int ksteps = (int)((a.RG + 15) / 16);  // rows past the group are zero: skip their K steps
        for (int st = 0; st < nst; ++st) {
          const int b = st & 1;
          mbar_wait(&wfull[b], (st >> 1) & 1);
          umma::fence_after_sync();
#pragma unroll
          for (int h = 0; h < 2; ++h) {  // W hi, W lo
            const uint32_t wb = sW + (b * 2 + h) * C::WBUF;
#pragma unroll
            for (int k = 0; k < 8; ++k) {  // 16 rows per step
              if (k < ksteps) {
                const uint64_t ad = umma::smem_desc(sA + (k / 4) * C::QATOM + (k % 4) * 32, 16, 1024);
                const uint64_t bd = umma::smem_desc(wb + k * 16 * 128, C::WBUF, 1024);
                umma::mma_bf16(tmem + M_COL + b * T5_KEYS, ad, bd, IDESC_M, h > 0 || k > 0);
              }
            }
          }
          umma::commit(smem_u32(&mdone[b]));
        }
      }
    }
    __syncwarp();
  } else if (tc5m_row_warp(warp) && (warp & 3) * 32 < a.RG) {  // ------- row warps (rows x half the keys)
    const int quarter = warp & 3;
    const int half = tc5m_half(warp);
    constexpr int HK = T5_KEYS / 2;  // keys per row warp per stage
    const int r = quarter * 32 + lane;
    const uint32_t tl = (uint32_t)(quarter * 32) << 16;
    const float sl2 = a.scale * 1.4426950408889634f;
    float m2 = INFINITY, rz = 0.f;  // padding rows: weight 0
    if (r < a.RG && rg * a.RG + r < a.R) {
      const float* f = a.fin + ((bk * a.R + rg * a.RG + r) * 2 + seg) * 2;
      m2 = f[0] * 1.4426950408889634f;
      rz = 1.f / f[1];
    }
    const float inv_nq = 1.f / (float)nq;
    auto readout = [&](int j) {  // warp with TMEM lanes 0-31 = the heads
      const int b = j & 1;
      mbar_wait(&mdone[b], (j >> 1) & 1);
      umma::fence_after_sync();
      uint32_t v[4][16];
#pragma unroll
      for (int c = 0; c < 4; ++c) umma::ld_32x32b_x16(tmem + tl + M_COL + b * T5_KEYS + c * 16, v[c]);
      umma::ld_wait();
      if (lane < heads && g0 + lane < a.G) {
        const int64_t kp0 = p0a + (int64_t)j * T5_KEYS;
        float* dst = a.mean[seg] + (b_ * a.Hq + kvh * a.G + g0 + lane) * a.mean_ld[seg] - a.seg_lo[seg] + kp0;
        const bool aligned = ((reinterpret_cast<uintptr_t>(dst) & 15) == 0);
        if (kp0 >= p0 && kp0 + T5_KEYS <= p1 && aligned) {  // whole stage in range: 16-byte stores
#pragma unroll
          for (int c = 0; c < 4; ++c)
#pragma unroll
            for (int e = 0; e < 16; e += 4)
              *reinterpret_cast<float4*>(dst + c * 16 + e) =
                  make_float4(__uint_as_float(v[c][e]) * inv_nq, __uint_as_float(v[c][e + 1]) * inv_nq,
                              __uint_as_float(v[c][e + 2]) * inv_nq, __uint_as_float(v[c][e + 3]) * inv_nq);
        } else {
          const int jlo = (int)max(p0 - kp0, (int64_t)0), jhi = (int)min(p1 - kp0, (int64_t)T5_KEYS);
#pragma unroll
          for (int c = 0; c < 4; ++c)
#pragma unroll
            for (int e = 0; e < 16; ++e)
              if (c * 16 + e >= jlo && c * 16 + e < jhi) dst[c * 16 + e] = __uint_as_float(v[c][e]) * inv_nq;
        }
      }
    };
    const uint32_t prow = (uint32_t)((r >> 3) * 1024 + (r & 7) * 128);
    for (int st = 0; st < nst; ++st) {
      const int b = st & 1;
      mbar_wait(&sfull[b], (st >> 1) & 1);
      umma::fence_after_sync();
      float x[HK];
      {
        uint32_t v[2][16];
#pragma unroll
        for (int c = 0; c < 2; ++c) umma::ld_32x32b_x16(tmem + tl + b * T5_KEYS + half * HK + c * 16, v[c]);
        umma::ld_wait();
        umma::fence_before_sync();
        __syncwarp();
        if (lane == 0) mbar_arrive(&sfree[b]);  // S(st) is in registers: QK(st + 2) may overwrite it
#pragma unroll
        for (int c = 0; c < 2; ++c)
#pragma unroll
          for (int j = 0; j < 16; ++j) x[c * 16 + j] = __uint_as_float(v[c][j]);
      }
      const int64_t kp0 = p0a + (int64_t)st * T5_KEYS + half * HK;
      if (kp0 >= p0 && kp0 + HK <= p1) {
#pragma unroll
        for (int j = 0; j < HK; ++j) x[j] = ex2_approx(fmaf(x[j], sl2, -m2)) * rz;
      } else {
        const int jlo = (int)max(p0 - kp0, (int64_t)0), jhi = (int)min(p1 - kp0, (int64_t)HK);
#pragma unroll
        for (int j = 0; j < HK; ++j) {
          const float w = ex2_approx(fmaf(x[j], sl2, -m2)) * rz;
          x[j] = (j >= jlo && j < jhi) ? w : 0.f;
        }
      }
      if (st >= 2) mbar_wait(&mdone[b], ((st - 2) >> 1) & 1);  // W buffer b read by MEAN(st-2)
      unsigned char* wh = sm + C::OFF_W + (b * 2) * C::WBUF + prow;
      unsigned char* wl = wh + C::WBUF;
#pragma unroll
      for (int c = 0; c < HK / 8; ++c) {
        uint32_t hi[4], lo[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          hi[e] = pack_bf16(x[c * 8 + 2 * e], x[c * 8 + 2 * e + 1]);
          lo[e] = pack_bf16(x[c * 8 + 2 * e] - bf16_lo_f(hi[e]), x[c * 8 + 2 * e + 1] - bf16_hi_f(hi[e]));
        }
        const uint32_t off = (uint32_t)(((c + half * (HK / 8)) ^ (r & 7)) << 4);
        *reinterpret_cast<uint4*>(wh + off) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
        *reinterpret_cast<uint4*>(wl + off) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
      }
      umma::fence_smem_async();
      umma::fence_before_sync();
      __syncwarp();
      if (lane == 0) mbar_arrive(&wfull[b]);
      if (quarter == 0 && half == 0 && st >= 1) readout(st - 1);
    }
    if (quarter == 0 && half == 0) readout(nst - 1);
  }
  umma::fence_before_sync();
  __syncthreads();
  if (warp == 1) umma::tmem_dealloc<C::TMEM_COLS>(tmem);
}

// ------------------------------------------------------------------ tcgen05 pass 2, two tiles
// The mean-weight pass for two 128-row groups of a (batch, kv-head) per CTA:
// one K stream, one head-membership matrix (the tiles have the same head
// layout), per tile: S double-buffered, W (hi, lo) single-buffered, MEAN
// double-buffered in TMEM, its own row warps and readout warp.
struct Tc5Mx2Cfg {             // D = 128
  static constexpr int QATOM = 128 * 128;
  static constexpr int KQ = T5_KEYS * 128;
  static constexpr int S = 4;
  static constexpr int STAGE = 2 * KQ;                  // K0 K1
  static constexpr int WBUF = 128 * 128;
  static constexpr int OFF_Q = 0;                       // [tile][2 atoms]
  static constexpr int OFF_K = OFF_Q + 4 * QATOM;
  static constexpr int OFF_W = OFF_K + S * STAGE;       // [tile][hi, lo]
  static constexpr int OFF_A = OFF_W + 4 * WBUF;
  static constexpr int OFF_BAR = OFF_A + 2 * QATOM;
  static constexpr int NBAR = 1 + 2 * S + 2 + 8;        // qfull, full[S], empty[S], sfull[2], wfull[2][2], mdone[2][2]
  static constexpr int OFF_TM = OFF_BAR + NBAR * 8;
  static constexpr int SMEM = OFF_TM + 16 + 1024;
  static constexpr int TMEM_COLS = 512;                 // S[2][2] x 64 | MEAN[2][2] x 64
  static constexpr int THREADS = 11 * 32;
};

__global__ void __launch_bounds__(Tc5Mx2Cfg::THREADS, 1) append_tc5_mean_x2_kernel(const __grid_constant__ AppendArgs a) {
  using C = Tc5Mx2Cfg;
  constexpr int D = 128;
  constexpr uint32_t M_COL = 4 * T5_KEYS;
  extern __shared__ unsigned char sm_raw[];
  unsigned char* sm = smem_align1024(sm_raw);
  const int64_t nc = a.nch[0] + a.nch[1], npair = (a.n_rg + 1) / 2;
  const int64_t cidx = blockIdx.x % nc, t_ = blockIdx.x / nc;
  const int64_t pair = t_ % npair, bk = t_ / npair;
  const int seg = cidx < a.nch[0] ? 0 : 1;
  const int64_t chunk = seg ? cidx - a.nch[0] : cidx;
  if (!a.mean[seg]) return;
  bool valid[2];
  valid[0] = true;
  valid[1] = 2 * pair + 1 < a.n_rg;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + C::OFF_BAR);
  uint64_t* qfull = bars;
  uint64_t* full = bars + 1;
  uint64_t* empty = full + C::S;
  uint64_t* sfull = empty + C::S;
  uint64_t* wfull = sfull + 2;   // [tile][parity]
  uint64_t* mdone = wfull + 4;   // [tile][parity]
  uint32_t* tm_holder = reinterpret_cast<uint32_t*>(sm + C::OFF_TM);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t p0 = a.seg_lo[seg] + chunk * ACHUNK;
  const int64_t p1 = min(a.seg_hi[seg], p0 + ACHUNK);
  const int64_t p0a = p0 & ~(int64_t)7;
  const int nst = (int)((p1 - p0a + T5_KEYS - 1) / T5_KEYS);
  const int nq = (int)a.nq, heads = (int)(a.RG / a.nq);
  const int64_t b_ = bk / a.Hkv, kvh = bk % a.Hkv;
  if (threadIdx.x == 0) {
    mbar_init(qfull, 1);
    for (int s = 0; s < C::S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int i = 0; i < 2; ++i) mbar_init(&sfull[i], 1);
    for (int i = 0; i < 4; ++i) {
      mbar_init(&wfull[i], 4);
      mbar_init(&mdone[i], 1);
    }
    fence_mbar_init();
  }
  if (warp >= 2 && warp < 6) {  // head-membership matrix A [128 heads][128 rows], K-major SW128
    const int h = threadIdx.x - 64;
    unsigned char* arow = sm + C::OFF_A + (h >> 3) * 1024 + (h & 7) * 128;
#pragma unroll
    for (int c = 0; c < 16; ++c) {
      uint32_t v[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int r0 = c * 8 + 2 * e;
        const float x0 = (h < heads && r0 / nq == h) ? 1.f : 0.f;
        const float x1 = (h < heads && (r0 + 1) / nq == h) ? 1.f : 0.f;
        v[e] = pack_bf16(x0, x1);
      }
      *reinterpret_cast<uint4*>(arow + (c >> 3) * C::QATOM + (((c & 7) ^ (h & 7)) << 4)) = make_uint4(v[0], v[1], v[2], v[3]);
    }
    umma::fence_smem_async();
  }
  if (warp == 1) umma::tmem_alloc<C::TMEM_COLS>(smem_u32(tm_holder));
  umma::fence_before_sync();
  __syncthreads();
  umma::fence_after_sync();
  const uint32_t tmem = *tm_holder;
  const uint32_t sQ = smem_u32(sm + C::OFF_Q), sK = smem_u32(sm + C::OFF_K), sW = smem_u32(sm + C::OFF_W),
                 sA = smem_u32(sm + C::OFF_A);

  if (warp == 0) {  // ------------------------------------------------ TMA producer
    if (lane == 0) {
      const uint64_t policy = l2_evict_first_policy();
      const int nt = valid[1] ? 2 : 1;
      mbar_expect_tx(qfull, nt * 2 * C::QATOM);
      for (int t = 0; t < nt; ++t) {
        const int qrow = (int)((b_ * a.Hq + kvh * a.G) * a.nq + (2 * pair + t) * a.RG);
        tma_load_2d(sQ + t * 2 * C::QATOM, &a.qmap5, 0, qrow, qfull, policy);
        tma_load_2d(sQ + t * 2 * C::QATOM + C::QATOM, &a.qmap5, 64, qrow, qfull, policy);
      }
      const int rowbase = (int)(bk * a.T + p0a);
      for (int st = 0; st < nst; ++st) {
        const int s = st % C::S;
        if (st >= C::S) mbar_wait(&empty[s], ((st / C::S) - 1) & 1);
        mbar_expect_tx(&full[s], C::STAGE);
        tma_load_2d(sK + s * C::STAGE, &a.kvmap5, 0, rowbase + st * T5_KEYS, &full[s], policy);
        tma_load_2d(sK + s * C::STAGE + C::KQ, &a.kvmap5, 64, rowbase + st * T5_KEYS, &full[s], policy);
      }
    }
  } else if (warp == 1 || warp == 6) {  // ----------------------------- MMA issuers
    if (lane == 0) {
      constexpr uint32_t IDESC_QK = umma::idesc_bf16_f32(128, T5_KEYS, false, false);
      constexpr uint32_t IDESC_M = umma::idesc_bf16_f32(128, T5_KEYS, false, true);
      if (warp == 1) {
        mbar_wait(qfull, 0);
        umma::fence_after_sync();
        for (int st = 0; st < nst; ++st) {
          const int s = st % C::S, b = st & 1;
          mbar_wait(&full[s], (st / C::S) & 1);
          for (int t = 0; t < 2; ++t)  // S[t][b] was read by the tile's rows of stage st-2
            if (valid[t] && st >= 2) mbar_wait(&wfull[t * 2 + b], ((st - 2) >> 1) & 1);
          umma::fence_after_sync();
          const uint32_t kb = sK + s * C::STAGE;
          for (int t = 0; t < 2; ++t) {
            if (!valid[t]) continue;
#pragma unroll
            for (int k = 0; k < D / 16; ++k) {
              const uint64_t ad = umma::smem_desc(sQ + t * 2 * C::QATOM + (k / 4) * C::QATOM + (k % 4) * 32, 16, 1024);
              const uint64_t bd = umma::smem_desc(kb + (k / 4) * C::KQ + (k % 4) * 32, 16, 1024);
              umma::mma_bf16(tmem + (t * 2 + b) * T5_KEYS, ad, bd, IDESC_QK, k > 0);
            }
          }
          umma::commit(smem_u32(&sfull[b]));
          umma::commit(smem_u32(&empty[s]));  // K is read by these GEMMs only
        }
      } else {
        for (int st = 0; st < nst; ++st) {
          const int b = st & 1;
          for (int t = 0; t < 2; ++t) {
            if (!valid[t]) continue;
            mbar_wait(&wfull[t * 2 + b], (st >> 1) & 1);
            umma::fence_after_sync();
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const uint32_t wb = sW + (t * 2 + h) * C::WBUF;
#pragma unroll
              for (int k = 0; k < 8; ++k) {
                const uint64_t ad = umma::smem_desc(sA + (k / 4) * C::QATOM + (k % 4) * 32, 16, 1024);
                const uint64_t bd = umma::smem_desc(wb + k * 16 * 128, C::WBUF, 1024);
                umma::mma_bf16(tmem + M_COL + (t * 2 + b) * T5_KEYS, ad, bd, IDESC_M, h > 0 || k > 0);
              }
            }
            umma::commit(smem_u32(&mdone[t * 2 + b]));
          }
        }
      }
    }
    __syncwarp();
  } else {  // ------------------------------------------------------- row warps
    const int t = warp >= 7 ? 1 : 0;
    if (valid[t]) {
      const int quarter = warp & 3;
      const int r = quarter * 32 + lane;
      const uint32_t tl = (uint32_t)(quarter * 32) << 16;
      const float sl2 = a.scale * 1.4426950408889634f;
      const int64_t rg = 2 * pair + t, g0 = rg * a.RG / a.nq;
      float m2 = INFINITY, rz = 0.f;
      if (r < a.RG && rg * a.RG + r < a.R) {
        const float* f = a.fin + ((bk * a.R + rg * a.RG + r) * 2 + seg) * 2;
        m2 = f[0] * 1.4426950408889634f;
        rz = 1.f / f[1];
      }
      const float inv_nq = 1.f / (float)nq;
      auto readout = [&](int j) {  // the warp whose TMEM lanes 0-31 hold the heads
        const int b = j & 1;
        mbar_wait(&mdone[t * 2 + b], (j >> 1) & 1);
        umma::fence_after_sync();
        uint32_t v[4][16];
#pragma unroll
        for (int c = 0; c < 4; ++c) umma::ld_32x32b_x16(tmem + tl + M_COL + (t * 2 + b) * T5_KEYS + c * 16, v[c]);
        umma::ld_wait();
        if (lane < heads && g0 + lane < a.G) {
          const int64_t kp0 = p0a + (int64_t)j * T5_KEYS;
          float* dst = a.mean[seg] + (b_ * a.Hq + kvh * a.G + g0 + lane) * a.mean_ld[seg] - a.seg_lo[seg] + kp0;
          const bool aligned = ((reinterpret_cast<uintptr_t>(dst) & 15) == 0);
          if (kp0 >= p0 && kp0 + T5_KEYS <= p1 && aligned) {
#pragma unroll
            for (int c = 0; c < 4; ++c)
#pragma unroll
              for (int e = 0; e < 16; e += 4)
                *reinterpret_cast<float4*>(dst + c * 16 + e) =
                    make_float4(__uint_as_float(v[c][e]) * inv_nq, __uint_as_float(v[c][e + 1]) * inv_nq,
                                __uint_as_float(v[c][e + 2]) * inv_nq, __uint_as_float(v[c][e + 3]) * inv_nq);
          } else {
            const int jlo = (int)max(p0 - kp0, (int64_t)0), jhi = (int)min(p1 - kp0, (int64_t)T5_KEYS);
#pragma unroll
            for (int c = 0; c < 4; ++c)
#pragma unroll
              for (int e = 0; e < 16; ++e)
                if (c * 16 + e >= jlo && c * 16 + e < jhi) dst[c * 16 + e] = __uint_as_float(v[c][e]) * inv_nq;
          }
        }
      };
      const uint32_t prow = (uint32_t)((r >> 3) * 1024 + (r & 7) * 128);
      for (int st = 0; st < nst; ++st) {
        const int b = st & 1;
        mbar_wait(&sfull[b], (st >> 1) & 1);
        umma::fence_after_sync();
        float x[T5_KEYS];
        {
          uint32_t v[4][16];
#pragma unroll
          for (int c = 0; c < 4; ++c) umma::ld_32x32b_x16(tmem + tl + (t * 2 + b) * T5_KEYS + c * 16, v[c]);
          umma::ld_wait();
#pragma unroll
          for (int c = 0; c < 4; ++c)
#pragma unroll
            for (int j = 0; j < 16; ++j) x[c * 16 + j] = __uint_as_float(v[c][j]);
        }
        const int64_t kp0 = p0a + (int64_t)st * T5_KEYS;
        if (kp0 >= p0 && kp0 + T5_KEYS <= p1) {
#pragma unroll
          for (int j = 0; j < T5_KEYS; ++j) x[j] = ex2_approx(fmaf(x[j], sl2, -m2)) * rz;
        } else {
          const int jlo = (int)max(p0 - kp0, (int64_t)0), jhi = (int)min(p1 - kp0, (int64_t)T5_KEYS);
#pragma unroll
          for (int j = 0; j < T5_KEYS; ++j) {
            const float w = ex2_approx(fmaf(x[j], sl2, -m2)) * rz;
            x[j] = (j >= jlo && j < jhi) ? w : 0.f;
          }
        }
        if (st >= 1) mbar_wait(&mdone[t * 2 + (b ^ 1)], ((st - 1) >> 1) & 1);  // W (single buffer) read by MEAN(st-1)
        unsigned char* wh = sm + C::OFF_W + (t * 2) * C::WBUF + prow;
        unsigned char* wl = wh + C::WBUF;
#pragma unroll
        for (int c = 0; c < T5_KEYS / 8; ++c) {
          uint32_t hi[4], lo[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            hi[e] = pack_bf16(x[c * 8 + 2 * e], x[c * 8 + 2 * e + 1]);
            lo[e] = pack_bf16(x[c * 8 + 2 * e] - bf16_lo_f(hi[e]), x[c * 8 + 2 * e + 1] - bf16_hi_f(hi[e]));
          }
          const uint32_t off = (uint32_t)((c ^ (r & 7)) << 4);
          *reinterpret_cast<uint4*>(wh + off) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
          *reinterpret_cast<uint4*>(wl + off) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
        }
        umma::fence_smem_async();
        umma::fence_before_sync();
        __syncwarp();
        if (lane == 0) mbar_arrive(&wfull[t * 2 + b]);
        if (quarter == 0 && st >= 1) readout(st - 1);
      }
      if (quarter == 0) readout(nst - 1);
    }
  }
  umma::fence_before_sync();
  __syncthreads();
  if (warp == 1) umma::tmem_dealloc<C::TMEM_COLS>(tmem);
}

// ------------------------------------------------------------------ tcgen05 pass 2, key-major
// The mean-weight pass with the GEMM transposed: S^T = K Q^T puts 128 keys on
// the TMEM lanes and NT row groups (NT * RG <= 256 query rows) on the
// columns, so every thread owns one key and sums its weights
// w = 2^(s * scale * log2e - (m2 + log2 z)) over each head's n_q columns in
// registers: no cross-row reduction, no second GEMM, no weight tile in shared
// memory. The per-row constants c = m2 + log2 z (from the fold) sit in
// shared memory and are read as broadcasts. Only K is loaded; the two
// accumulators are double-buffered so the QK of stage st + 1 overlaps the
// exponentials of stage st. Warps: 0 TMA, 1 MMA issuer, 2-17 four sets of
// four key warps (lane quarter = warp % 4): sets 0 / 2 take the even stages
// (accumulator 0), sets 1 / 3 the odd ones, and the two sets of an
// accumulator split its columns at a head boundary.
template <int NT>
struct Tc5KCfg {               // D = 128
  static constexpr int KEYS = 128;                      // keys per stage (the M = 128 tile)
  static constexpr int QH = NT * 128 * 128;             // one 64-column half of Q: NT*128 rows x 128 B
  static constexpr int KH = KEYS * 128;                 // one 64-column half of a K stage
  static constexpr int S = 4;
  static constexpr int STAGE = 2 * KH;
  static constexpr int OFF_Q = 0;
  static constexpr int OFF_K = OFF_Q + 2 * QH;
  static constexpr int OFF_C = OFF_K + S * STAGE;       // c[NT * 128] fp32
  static constexpr int OFF_BAR = OFF_C + NT * 128 * 4;
  static constexpr int NBAR = 1 + 2 * S + 4;            // qfull, full[S], empty[S], afull[2], afree[2]
  static constexpr int OFF_TM = OFF_BAR + NBAR * 8;
  static constexpr int SMEM = OFF_TM + 16 + 1024;
  static constexpr int ACOLS = NT * 128;                // TMEM columns per accumulator
  static constexpr int TMEM_COLS = 2 * ACOLS;
  static constexpr int THREADS = 18 * 32;             // TMA, MMA, 4 x 4 key warps
};

template <int NT>
__global__ void __launch_bounds__(Tc5KCfg<NT>::THREADS, 1) append_tc5_mean_k_kernel(const __grid_constant__ AppendArgs a) {
  using C = Tc5KCfg<NT>;
  constexpr int D = 128;
  extern __shared__ unsigned char sm_raw[];
  unsigned char* sm = smem_align1024(sm_raw);
  const int64_t nc = a.nch[0] + a.nch[1], ngrp = (a.n_rg + NT - 1) / NT;
  const int64_t cidx = blockIdx.x % nc, t_ = blockIdx.x / nc;
  const int64_t rg0 = (t_ % ngrp) * NT, bk = t_ / ngrp;
  const int seg = cidx < a.nch[0] ? 0 : 1;
  const int64_t chunk = seg ? cidx - a.nch[0] : cidx;
  if (!a.mean[seg]) return;  // (uniform) no means wanted for this segment
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + C::OFF_BAR);
  uint64_t* qfull = bars;
  uint64_t* full = bars + 1;
  uint64_t* empty = full + C::S;
  uint64_t* afull = empty + C::S;
  uint64_t* afree = afull + 2;
  float* cst = reinterpret_cast<float*>(sm + C::OFF_C);
  uint32_t* tm_holder = reinterpret_cast<uint32_t*>(sm + C::OFF_TM);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t p0 = a.seg_lo[seg] + chunk * ACHUNK;
  const int64_t p1 = min(a.seg_hi[seg], p0 + ACHUNK);
  const int64_t p0a = p0 & ~(int64_t)7;
  const int nst = (int)((p1 - p0a + C::KEYS - 1) / C::KEYS);
  const int64_t row0 = rg0 * a.RG;                          // first query row (of the bk's R) in this CTA
  const int ncol = (int)min((int64_t)NT * a.RG, a.R - row0);  // whole heads (RG and R are multiples of n_q)
  const int npad = (ncol + 15) & ~15;                       // MMA N
  const int64_t b_ = bk / a.Hkv, kvh = bk % a.Hkv;
  if (threadIdx.x == 0) {
    mbar_init(qfull, 1);
    for (int s = 0; s < C::S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&afull[b], 1);
      mbar_init(&afree[b], 8);  // the 2 x 4 key warps of accumulator b
    }
    fence_mbar_init();
  }
  if (warp >= 2) {  // per-row exponent offsets c = m * log2e + log2 z
    for (int j = threadIdx.x - 64; j < NT * 128; j += 512) {
      float c = INFINITY;
      if (j < ncol) {
        const float* f = a.fin + ((bk * a.R + row0 + j) * 2 + seg) * 2;
        c = f[0] * 1.4426950408889634f + log2f(f[1]);
      }
      cst[j] = c;
    }
  }
  if (warp == 1) umma::tmem_alloc<C::TMEM_COLS>(smem_u32(tm_holder));
  umma::fence_before_sync();
  __syncthreads();
  umma::fence_after_sync();
  const uint32_t tmem = *tm_holder;
  const uint32_t sQ = smem_u32(sm + C::OFF_Q), sK = smem_u32(sm + C::OFF_K);

  if (warp == 0) {  // ------------------------------------------------ TMA producer
    if (lane == 0) {
      const uint64_t policy = l2_evict_first_policy();
      const int qrow = (int)((b_ * a.Hq + kvh * a.G) * a.nq + row0);
      mbar_expect_tx(qfull, 2 * C::QH);
#pragma unroll
      for (int t = 0; t < NT; ++t) {
        tma_load_2d(sQ + t * 128 * 128, &a.qmap5, 0, qrow + t * 128, qfull, policy);
        tma_load_2d(sQ + C::QH + t * 128 * 128, &a.qmap5, 64, qrow + t * 128, qfull, policy);
      }
      const int rowbase = (int)(bk * a.T + p0a);
      for (int st = 0; st < nst; ++st) {
        const int s = st % C::S;
        if (st >= C::S) mbar_wait(&empty[s], ((st / C::S) - 1) & 1);
        mbar_expect_tx(&full[s], C::STAGE);
        const uint32_t kb = sK + s * C::STAGE;
        const int r = rowbase + st * C::KEYS;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          tma_load_2d(kb + h * C::KH, &a.kvmap5, 64 * h, r, &full[s], policy);
          tma_load_2d(kb + h * C::KH + T5_KEYS * 128, &a.kvmap5, 64 * h, r + T5_KEYS, &full[s], policy);
        }
      }
    }
  } else if (warp == 1) {  // ------------------------------------------- MMA issuer
    if (lane == 0) {
      const uint32_t idesc = umma::idesc_bf16_f32(128, npad, false, false);
      mbar_wait(qfull, 0);
      umma::fence_after_sync();
      for (int st = 0; st < nst; ++st) {
        const int s = st % C::S, b = st & 1;
        mbar_wait(&full[s], (st / C::S) & 1);
        if (st >= 2) mbar_wait(&afree[b], ((st - 2) >> 1) & 1);  // accumulator b read out (stage st - 2)
        umma::fence_after_sync();
        const uint32_t kb = sK + s * C::STAGE;
#pragma unroll
        for (int k = 0; k < D / 16; ++k) {
          const uint64_t ad = umma::smem_desc(kb + (k / 4) * C::KH + (k % 4) * 32, 16, 1024);
          const uint64_t bd = umma::smem_desc(sQ + (k / 4) * C::QH + (k % 4) * 32, 16, 1024);
          umma::mma_bf16(tmem + b * C::ACOLS, ad, bd, idesc, k > 0);
        }
        umma::commit(smem_u32(&afull[b]));
        umma::commit(smem_u32(&empty[s]));
      }
    }
    __syncwarp();
  } else {  // ---------------------------------------------------------- key warps
    const int set = (warp - 2) >> 2, quarter = warp & 3;
    const int b = set & 1;  // this set's stages st = b, b + 2, ... (accumulator b)
    const uint32_t tl = (uint32_t)(quarter * 32) << 16;
    const float sl2 = a.scale * 1.4426950408889634f;
    const float inv_nq = 1.f / (float)a.nq;
    const int nq = (int)a.nq;
    const int64_t ld = a.mean_ld[seg];
    const int W = nq % 32 == 0 ? 32 : nq % 8 == 0 ? 8 : nq % 4 == 0 ? 4 : 0;  // columns per sum group
    // the two sets of an accumulator split its columns at a head boundary
    // (when that boundary is a 32-column one; else the first set takes all)
    const int csplit = (ncol / nq / 2) * nq;
    const bool split = csplit > 0 && csplit % 32 == 0;
    const int cbeg = (set >> 1) ? (split ? csplit : ncol) : 0;
    const int cend = (set >> 1) ? ncol : (split ? csplit : ncol);
    float* const mrow = a.mean[seg] + (b_ * a.Hq + kvh * a.G + (row0 + cbeg) / a.nq) * ld - a.seg_lo[seg];
    for (int st = b; st < nst; st += 2) {
      const int64_t key = p0a + (int64_t)st * C::KEYS + quarter * 32 + lane;
      const bool mine = key >= p0 && key < p1;
      float* mp = mrow + key;
      mbar_wait(&afull[b], (st >> 1) & 1);
      umma::fence_after_sync();
      if (cbeg >= cend) {  // (uniform) nothing for this set
        umma::fence_before_sync();
        __syncwarp();
        if (lane == 0) mbar_arrive(&afree[b]);
        continue;
      }
      float hs = 0.f;
      int left = nq;
      for (int c0 = cbeg; c0 < cend; c0 += 32) {
        float x[32];
        {
          uint32_t v[2][16];
          umma::ld_32x32b_x16(tmem + tl + b * C::ACOLS + c0, v[0]);
          umma::ld_32x32b_x16(tmem + tl + b * C::ACOLS + c0 + 16, v[1]);
          umma::ld_wait();
          if (c0 + 32 >= cend) {  // the accumulator is in registers: QK(st + 2) may overwrite it
            umma::fence_before_sync();
            __syncwarp();
            if (lane == 0) mbar_arrive(&afree[b]);
          }
#pragma unroll
          for (int e = 0; e < 32; ++e) x[e] = __uint_as_float(v[e >> 4][e & 15]);
        }
        // exponents first, then the exponentials: independent chains for the scheduler
#pragma unroll
        for (int e4 = 0; e4 < 8; ++e4) {
          const float4 c4 = *reinterpret_cast<const float4*>(cst + c0 + e4 * 4);
          x[e4 * 4 + 0] = fmaf(x[e4 * 4 + 0], sl2, -c4.x);
          x[e4 * 4 + 1] = fmaf(x[e4 * 4 + 1], sl2, -c4.y);
          x[e4 * 4 + 2] = fmaf(x[e4 * 4 + 2], sl2, -c4.z);
          x[e4 * 4 + 3] = fmaf(x[e4 * 4 + 3], sl2, -c4.w);
        }
#pragma unroll
        for (int e = 0; e < 32; ++e) x[e] = ex2_approx(x[e]);
        // heads of n_q columns end on group boundaries: a tree per group of W columns, then
        // the groups accumulate into the head's sum
        auto flush = [&]() {
          if (mine) *mp = hs * inv_nq;
          mp += ld;
          hs = 0.f;
          left = nq;
        };
        if (W == 32) {  // whole chunks of one head: one check per chunk
          float g8[4];
#pragma unroll
          for (int g = 0; g < 4; ++g)
            g8[g] = ((x[g * 8] + x[g * 8 + 1]) + (x[g * 8 + 2] + x[g * 8 + 3])) +
                    ((x[g * 8 + 4] + x[g * 8 + 5]) + (x[g * 8 + 6] + x[g * 8 + 7]));
          hs += (g8[0] + g8[1]) + (g8[2] + g8[3]);
          if ((left -= 32) == 0) flush();
        } else if (W == 8) {
#pragma unroll
          for (int g = 0; g < 4; ++g)
            if (c0 + g * 8 < cend) {
              hs += ((x[g * 8] + x[g * 8 + 1]) + (x[g * 8 + 2] + x[g * 8 + 3])) +
                    ((x[g * 8 + 4] + x[g * 8 + 5]) + (x[g * 8 + 6] + x[g * 8 + 7]));
              if ((left -= 8) == 0) flush();
            }
        } else if (W == 4) {
#pragma unroll
          for (int g = 0; g < 8; ++g)
            if (c0 + g * 4 < cend) {
              hs += (x[g * 4] + x[g * 4 + 1]) + (x[g * 4 + 2] + x[g * 4 + 3]);
              if ((left -= 4) == 0) flush();
            }
        } else {  // other n_q: column by column
#pragma unroll
          for (int e = 0; e < 32; ++e) {
            if (c0 + e < cend) {
              hs += x[e];
              if (--left == 0) flush();
            }
          }
        }
      }
    }
  }
  umma::fence_before_sync();
  __syncthreads();
  if (warp == 1) umma::tmem_dealloc<C::TMEM_COLS>(tmem);
}

// One warp per (b, kv-head, row): fold the chunk partials of both segments,
// merge_states(archive, window) (attention.py:153-188), out / lse, and the
// row's final (m, z) per segment for pass 2.
template <int D>
__global__ void __launch_bounds__(256) append_fold_kernel(const __grid_constant__ AppendArgs a) {
  constexpr int DPL = D / 32;
  const int lane = threadIdx.x & 31;
  const int64_t wid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t BK = a.B * a.Hkv;
  if (wid >= BK * a.R) return;
  const int64_t bk = wid / a.R, row = wid % a.R;
  const int64_t rg = row / a.RG, rr = row % a.RG;
  const int64_t nc = a.nch[0] + a.nch[1];
  const int64_t base = (bk * a.n_rg + rg) * nc;
  float so[2][DPL];
  double lse_seg[2];
  for (int seg = 0; seg < 2; ++seg) {
    const int64_t c0 = seg ? a.nch[0] : 0, c1 = seg ? nc : a.nch[0];
    float M = -INFINITY;
    for (int64_t c = c0; c < c1; ++c) M = fmaxf(M, a.part_m[(base + c) * a.RG + rr]);
    float Z = 0.f, acc[DPL];
#pragma unroll
    for (int k = 0; k < DPL; ++k) acc[k] = 0.f;
    if (M != -INFINITY) {
      for (int64_t c = c0; c < c1; ++c) {
        const float mc = a.part_m[(base + c) * a.RG + rr];
        if (mc == -INFINITY) continue;
        const float w = __expf(mc - M);
        Z += a.part_z[(base + c) * a.RG + rr] * w;
        const float* pa = a.part_acc + ((base + c) * a.RG + rr) * D + lane * DPL;
#pragma unroll
        for (int k = 0; k < DPL; ++k) acc[k] += w * pa[k];
      }
    }
    const bool empty = !(Z > 0.f);
#pragma unroll
    for (int k = 0; k < DPL; ++k) so[seg][k] = empty ? 0.f : acc[k] / Z;
    lse_seg[seg] = empty ? -INFINITY : (double)M + log((double)Z);
    if (lane == 0) {
      a.fin[((bk * a.R + row) * 2 + seg) * 2] = M;
      a.fin[((bk * a.R + row) * 2 + seg) * 2 + 1] = empty ? 1.f : Z;
    }
  }
  const double mm = fmax(lse_seg[0], lse_seg[1]);
  const bool both_empty = mm == -INFINITY;
  const double ms = both_empty ? 0.0 : mm;
  const double wa = exp(lse_seg[0] - ms), wb = exp(lse_seg[1] - ms);
  const double zs = both_empty ? 1.0 : wa + wb;
  const float ca = (float)(wa / zs), cb = (float)(wb / zs);
  const int64_t b = bk / a.Hkv, kvh = bk % a.Hkv;
  const int64_t g = row / a.nq, i = row % a.nq;
  const int64_t orow = (b * a.Hq + kvh * a.G + g) * a.nq + i;
#pragma unroll
  for (int k = 0; k < DPL; ++k)
    a.out[orow * D + lane * DPL + k] = __fadd_rn(__fmul_rn(ca, so[0][k]), __fmul_rn(cb, so[1][k]));
  if (lane == 0) a.lse[orow] = both_empty ? -INFINITY : ms + log(zs);
}

// ------------------------------------------------------------------ launcher
typedef CUresult (*EncodeTiledFnA)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static int make_tile_map(CUtensorMap* map, const void* base, int64_t rows, int64_t D) {
  static EncodeTiledFnA encode = nullptr;
  if (!encode) {
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&encode, cudaEnableDefault, &q) != cudaSuccess ||
        !encode)
      return -3000;
  }
  cuuint64_t gdim[2] = {(cuuint64_t)(2 * D), (cuuint64_t)rows};
  cuuint64_t gstr[1] = {(cuuint64_t)(2 * D * 2)};
  cuuint32_t box[2] = {(cuuint32_t)(2 * D), (cuuint32_t)AK};
  cuuint32_t es[2] = {1, 1};
  CUresult r = encode(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), gdim, gstr, box, es,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : -3001;
}

// 2-D bf16 map [rows, cols] with a (box_cols x box_rows) box
static int make_map2d(CUtensorMap* map, const void* base, int64_t rows, int64_t cols, int box_cols, int box_rows,
                      CUtensorMapSwizzle swz) {
  static EncodeTiledFnA encode = nullptr;
  if (!encode) {
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&encode, cudaEnableDefault, &q) != cudaSuccess ||
        !encode)
      return -3000;
  }
  cuuint64_t gdim[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t gstr[1] = {(cuuint64_t)(cols * 2)};
  cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = encode(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), gdim, gstr, box, es,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : -3001;
}

// Layout of the caller's workspace for one append step (all sizes in bytes).
struct AppendPlan {
  int64_t R, RG, n_rg, nch0, nch1, n_items;
  int64_t off_acc, off_m, off_z, off_fin, bytes;
};

static AppendPlan append_plan(int64_t B, int64_t Hq, int64_t Hkv, int64_t D, int64_t nq, int64_t lo, int64_t hi) {
  AppendPlan p{};
  const int64_t G = Hq / Hkv;
  p.R = G * nq;
  // row groups of <= AMAXW*16 rows holding whole query heads (nq <= 128)
  const int64_t heads_per_group = (AMAXW * 16) / nq;
  p.RG = (heads_per_group >= G ? G : heads_per_group) * nq;
  p.n_rg = (p.R + p.RG - 1) / p.RG;
  p.nch0 = (lo + ACHUNK - 1) / ACHUNK;
  p.nch1 = (hi - lo + ACHUNK - 1) / ACHUNK;
  p.n_items = B * Hkv * p.n_rg * (p.nch0 + p.nch1);
  auto al = [](int64_t x) { return (x + 255) / 256 * 256; };
  p.off_acc = 0;
  p.off_m = al(p.n_items * p.RG * D * 4);
  p.off_z = p.off_m + al(p.n_items * p.RG * 4);
  p.off_fin = p.off_z + al(p.n_items * p.RG * 4);
  p.bytes = p.off_fin + al(B * Hkv * p.R * 4 * 4);
  return p;
}

int64_t append_ws_bytes(int64_t B, int64_t Hq, int64_t Hkv, int64_t D, int64_t nq, int64_t lo, int64_t hi) {
  if (nq < 1 || nq > AMAXW * 16 || Hkv < 1 || Hq % Hkv) return -1;
  return append_plan(B, Hq, Hkv, D, nq, lo, hi).bytes;
}

template <int D>
static int launch_append_d(const void* KV, int64_t B, int64_t Hq, int64_t Hkv, int64_t T, const void* q, int64_t nq,
                           double scale, int64_t lo, int64_t hi, float* out, double* lse, float* mean_archive,
                           float* mean_window, void* ws, cudaStream_t s) {
  using C1 = AppendCfg<D, 1>;
  using C2 = AppendCfg<D, 2>;
  const AppendPlan p = append_plan(B, Hq, Hkv, D, nq, lo, hi);
  AppendArgs a{};
  {
    const int64_t rows = B * Hkv * T;
    const int rc = map_cache().get(map_key(10 + (int)D, KV, rows, 2 * D, 0, 0), &a.kmap,
                                   [&](CUtensorMap* m) { return make_tile_map(m, KV, rows, D); });
    if (rc) return rc;
  }
  a.q = reinterpret_cast<const __nv_bfloat16*>(q);
  a.B = B; a.Hq = Hq; a.Hkv = Hkv; a.G = Hq / Hkv; a.T = T; a.nq = nq;
  a.scale = (float)scale;
  a.seg_lo[0] = 0; a.seg_hi[0] = lo; a.seg_lo[1] = lo; a.seg_hi[1] = hi;
  a.nch[0] = p.nch0; a.nch[1] = p.nch1;
  a.R = p.R; a.RG = p.RG; a.n_rg = p.n_rg; a.n_items = p.n_items;
  unsigned char* w = reinterpret_cast<unsigned char*>(ws);
  a.part_acc = reinterpret_cast<float*>(w + p.off_acc);
  a.part_m = reinterpret_cast<float*>(w + p.off_m);
  a.part_z = reinterpret_cast<float*>(w + p.off_z);
  a.fin = reinterpret_cast<float*>(w + p.off_fin);
  a.out = out; a.lse = lse;
  a.mean[0] = mean_archive; a.mean_ld[0] = lo;
  a.mean[1] = mean_window; a.mean_ld[1] = hi - lo;
  static DevFlags attr1, attr2;
  {
    int e = set_smem_dev(append_attend_kernel<D, 1>, C1::SMEM, attr1);
    if (e) return e;
    e = set_smem_dev(append_attend_kernel<D, 2>, C2::SMEM, attr2);
    if (e) return e;
  }
  const int nw = (int)((p.RG + 15) / 16);
  if constexpr (D == 128) {  // pass 1 on tcgen05
    {
      const int64_t rows = B * Hkv * T;
      const int rc5 = map_cache().get(map_key(20, KV, rows, 2 * D, 64, T5_KEYS), &a.kvmap5, [&](CUtensorMap* m) {
        return make_map2d(m, KV, rows, 2 * D, 64, T5_KEYS, CU_TENSOR_MAP_SWIZZLE_NONE);
      });
      if (rc5) return rc5;
      const int rc = make_map2d(&a.qmap5, q, B * Hq * nq, D, 64, 128, CU_TENSOR_MAP_SWIZZLE_128B);
      if (rc) return rc;
      const char* sk = getenv("HGCA_APPEND_SPLIT_KEYS");
      a.split_keys = !(sk && *sk == '0');
      // split keys: one box per copy of the group (64 rows for 2 copies, 32 for 4)
      const int rch = make_map2d(&a.qmap5h, q, B * Hq * nq, D, 64, p.RG > 32 ? 64 : 32, CU_TENSOR_MAP_SWIZZLE_128B);
      if (rch) return rch;
    }
    static DevFlags attr5[3];
    const int ncp = !a.split_keys ? 1 : p.RG <= 32 ? 4 : p.RG <= 64 ? 2 : 1;
    auto tc5k = ncp == 4 ? append_tc5_kernel<4> : ncp == 2 ? append_tc5_kernel<2> : append_tc5_kernel<1>;
    if (const int e5 = set_smem_dev(tc5k, Tc5Cfg::SMEM, attr5[ncp >> 1])) return e5;
    // every row group: >= 64 rows as one tile, smaller ones in split-key mode (2 or 4 copies of
    // the group fill the 128-row tile); without split keys groups of < 64 rows stay on mma.sync
    const char* force_mma = getenv("HGCA_APPEND_MMA_SYNC");  // A/B switch: 1 = the mma.sync pass for every group
    const bool tc5 = (p.RG >= 64 || a.split_keys) && !(force_mma && *force_mma && *force_mma != '0');
    static DevFlags attr52;
    if (const int e52 = set_smem_dev(append_tc5x2_kernel, Tc5x2Cfg::SMEM, attr52)) return e52;
    const bool two_tiles = tc5 && p.RG == 128 && p.n_rg >= 2;  // pairs of 128-row groups share the K|V stream
    if (p.n_items > 0 && two_tiles)
      append_tc5x2_kernel<<<(unsigned)(B * Hkv * ((p.n_rg + 1) / 2) * (p.nch0 + p.nch1)), Tc5x2Cfg::THREADS,
                            Tc5x2Cfg::SMEM, s>>>(a);
    else if (p.n_items > 0 && tc5)
      tc5k<<<(unsigned)p.n_items, Tc5Cfg::THREADS, Tc5Cfg::SMEM, s>>>(a);
    else if (p.n_items > 0)
      append_attend_kernel<D, 1><<<(unsigned)p.n_items, (nw + 1) * 32, C1::SMEM, s>>>(a);
  } else {
    if (p.n_items > 0) append_attend_kernel<D, 1><<<(unsigned)p.n_items, (nw + 1) * 32, C1::SMEM, s>>>(a);
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return (int)e;
  const int64_t warps = B * Hkv * p.R;
  append_fold_kernel<D><<<(unsigned)((warps * 32 + 255) / 256), 256, 0, s>>>(a);
  e = cudaGetLastError();
  if (e != cudaSuccess) return (int)e;
  if ((mean_archive || mean_window) && p.n_items > 0) {
    bool tc5_mean = false;
    if constexpr (D == 128) {
      // key-major tcgen05 pass for every row group (default); HGCA_APPEND_MEAN_OLD=1: the
      // row-major pass with the head-sum GEMM (groups of >= 64 rows); HGCA_APPEND_MMA_SYNC=1:
      // the mma.sync pass. Two row groups per CTA share the K stream (HGCA_APPEND_MEAN_NT=1: one)
      const char* force_mma = getenv("HGCA_APPEND_MMA_SYNC");
      const char* old_mean = getenv("HGCA_APPEND_MEAN_OLD");
      const char* nt_env = getenv("HGCA_APPEND_MEAN_NT");
      const bool forced = force_mma && *force_mma && *force_mma != '0';
      const bool oldm = old_mean && *old_mean && *old_mean != '0';
      const bool km = !forced && !oldm;
      const bool km2 = km && p.n_rg >= 2 && !(nt_env && *nt_env == '1');
      const bool rowmajor = !forced && oldm && p.RG >= 64;
      tc5_mean = km || rowmajor;
      static DevFlags attr_m, attr_m2, attr_k1, attr_k2;
      const int64_t nc = p.nch0 + p.nch1;
      if (km2) {
        if (const int ek = set_smem_dev(append_tc5_mean_k_kernel<2>, Tc5KCfg<2>::SMEM, attr_k2)) return ek;
        append_tc5_mean_k_kernel<2><<<(unsigned)(B * Hkv * ((p.n_rg + 1) / 2) * nc), Tc5KCfg<2>::THREADS,
                                      Tc5KCfg<2>::SMEM, s>>>(a);
      } else if (km) {
        if (const int ek = set_smem_dev(append_tc5_mean_k_kernel<1>, Tc5KCfg<1>::SMEM, attr_k1)) return ek;
        append_tc5_mean_k_kernel<1><<<(unsigned)(B * Hkv * p.n_rg * nc), Tc5KCfg<1>::THREADS, Tc5KCfg<1>::SMEM, s>>>(a);
      } else if (rowmajor) {
        if (const int em = set_smem_dev(append_tc5_mean_kernel, Tc5MCfg::SMEM, attr_m)) return em;
        if (const int em2 = set_smem_dev(append_tc5_mean_x2_kernel, Tc5Mx2Cfg::SMEM, attr_m2)) return em2;
        if (p.RG == 128 && p.n_rg >= 2)  // pairs of 128-row groups share the K stream
          append_tc5_mean_x2_kernel<<<(unsigned)(B * Hkv * ((p.n_rg + 1) / 2) * nc), Tc5Mx2Cfg::THREADS,
                                      Tc5Mx2Cfg::SMEM, s>>>(a);
        else
          append_tc5_mean_kernel<<<(unsigned)p.n_items, Tc5MCfg::THREADS, Tc5MCfg::SMEM, s>>>(a);
      }
    }
    if (!tc5_mean) append_attend_kernel<D, 2><<<(unsigned)p.n_items, (nw + 1) * 32, C2::SMEM, s>>>(a);
  }
  return (int)cudaGetLastError();
}

int launch_append_bf16(const void* KV, int64_t B, int64_t Hq, int64_t Hkv, int64_t T, int64_t D, const void* q,
                       int64_t nq, double scale, int64_t lo, int64_t hi, float* out, double* lse, float* mean_archive,
                       float* mean_window, void* ws, cudaStream_t s) {
  if (D == 128)
    return launch_append_d<128>(KV, B, Hq, Hkv, T, q, nq, scale, lo, hi, out, lse, mean_archive, mean_window, ws, s);
  if (D == 64)
    return launch_append_d<64>(KV, B, Hq, Hkv, T, q, nq, scale, lo, hi, out, lse, mean_archive, mean_window, ws, s);
  return -1001;
}

#ifdef HGCA_TC5_PROF
extern "C" int hgca_debug_tc5prof(unsigned long long* out8) {
  cudaDeviceSynchronize();
  return (int)cudaMemcpyFromSymbol(out8, g_tc5prof, sizeof(unsigned long long) * 8);
}
#endif

}  // namespace hgca
