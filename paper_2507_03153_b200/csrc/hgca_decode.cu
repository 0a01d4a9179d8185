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
// decode_merge_kernel then folds the partials in a fixed order, applies the
// reference merge_states (attention.py:153-188) and the fp64 MAW EMA
// (kv_cache.py:171-187, engine.py:177-191) from the stored dense scores.
#include "hgca_common.cuh"
#include "hgca_internal.h"

namespace hgca {

template <typename T, int D, int G>
struct DecodeCfg {
  static constexpr int ESZ = (int)sizeof(T);
  static constexpr int ROWB = D * ESZ;
  static constexpr int CH = ROWB <= 256 ? 128 : 64;    // rows per stage (<= consumer threads)
  static constexpr int KRS = ROWB + 16;                 // padded K row: conflict-free row-per-thread reads
  static constexpr int VRS = ROWB;
  static constexpr int PIECES = ROWB / 16;
  static constexpr int E = 16 / ESZ;                    // elements per 16-byte piece
  static constexpr int QB = G * ROWB;                   // raw query bytes staged per chunk
  static constexpr int OFF_V = CH * KRS;
  static constexpr int OFF_Q = OFF_V + CH * VRS;
  static constexpr int OFF_POS = OFF_Q + QB;
  static constexpr int OFF_QM = OFF_POS + CH * 4;
  static constexpr int STAGE = ((OFF_QM + CH) + 127) / 128 * 128;
  static constexpr int GW = G < 4 ? G : 4;              // distinct heads across the 4 PV warps
  static constexpr int NPV = 4 / GW;                    // warps sharing one head in P.V
  static constexpr int HPW = G > 4 ? G / 4 : 1;         // heads per PV warp
  static constexpr int DPL = D / 32;                    // dims per lane in P.V
  static constexpr int FIXED = G * D * 8 + G * CH * 8 + G * CH * 4 + 4 * D * 4 + 256;
  static constexpr int SMAX = 232448 - 1024;
  static constexpr int S0 = (SMAX - FIXED) / STAGE;
  static constexpr int S = S0 > 4 ? 4 : S0;
  static constexpr int SMEM = S * STAGE + FIXED;
  static_assert(S >= 2, "decode stage does not fit shared memory");
  static_assert(D % 32 == 0, "head_dim must be a multiple of 32");
};

template <typename T>
__device__ __forceinline__ void load_piece_f64(const unsigned char* p, double* out);
template <>
__device__ __forceinline__ void load_piece_f64<float>(const unsigned char* p, double* out) {
  const float4 v = *reinterpret_cast<const float4*>(p);
  out[0] = (double)v.x; out[1] = (double)v.y; out[2] = (double)v.z; out[3] = (double)v.w;
}
template <>
__device__ __forceinline__ void load_piece_f64<__nv_bfloat16>(const unsigned char* p, double* out) {
  const uint4 v = *reinterpret_cast<const uint4*>(p);
  const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    out[2 * i] = (double)__uint_as_float(w[i] << 16);
    out[2 * i + 1] = (double)__uint_as_float(w[i] & 0xffff0000u);
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
template <>
__device__ __forceinline__ void load_v_f32<__nv_bfloat16, 4>(const unsigned char* p, float* out) {
  const uint2 v = *reinterpret_cast<const uint2*>(p);
  out[0] = __uint_as_float(v.x << 16); out[1] = __uint_as_float(v.x & 0xffff0000u);
  out[2] = __uint_as_float(v.y << 16); out[3] = __uint_as_float(v.y & 0xffff0000u);
}
template <>
__device__ __forceinline__ void load_v_f32<__nv_bfloat16, 2>(const unsigned char* p, float* out) {
  const uint32_t v = *reinterpret_cast<const uint32_t*>(p);
  out[0] = __uint_as_float(v << 16); out[1] = __uint_as_float(v & 0xffff0000u);
}

template <typename T, int D, int G>
__global__ void __launch_bounds__(160, 1) decode_partial_kernel(const DecodeArgs a) {
  using C = DecodeCfg<T, D, G>;
  extern __shared__ __align__(128) unsigned char sm[];
  unsigned char* stages = sm;
  double* qsh = reinterpret_cast<double*>(sm + C::S * C::STAGE);  // [G][D]
  double* sc = qsh + G * D;                                        // [G][CH]
  float* pf = reinterpret_cast<float*>(sc + G * C::CH);            // [G][CH]
  float* accbuf = pf + G * C::CH;                                  // [4][D]
  __shared__ __align__(8) uint64_t full[C::S], empty[C::S];
  __shared__ int st_item[C::S], st_chunk[C::S], st_nvalid[C::S], st_last[C::S];
  __shared__ double m_sh[G], z_sh[G], scal_sh[G];

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t BK = a.B * a.Hkv;
  const int64_t W = a.dhi - a.dlo;
  if (tid == 0) {
    for (int s = 0; s < C::S; ++s) {
      mbar_init(&full[s], 64);
      mbar_init(&empty[s], 4);
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (warp == 4) {
    // ---------------------------------------------------------------- producer
    const int64_t total = a.n_dense_items + (int64_t)a.item_off[BK];
    const unsigned char* Kg = reinterpret_cast<const unsigned char*>(a.K);
    const unsigned char* Vg = reinterpret_cast<const unsigned char*>(a.V);
    const unsigned char* Qg = reinterpret_cast<const unsigned char*>(a.q);
    int k = 0;
    while (true) {
      int item = 0;
      if (lane == 0) item = atomicAdd(a.counter, 1);
      item = __shfl_sync(0xffffffffu, item, 0);
      if (item >= total) {
        const int s = k % C::S;
        if (k >= C::S) mbar_wait(&empty[s], ((k / C::S) - 1) & 1);
        if (lane == 0) st_item[s] = -1;
        __syncwarp();
        cp_async_mbar_arrive_noinc(&full[s]);
        mbar_arrive(&full[s]);
        break;
      }
      int64_t bk, lo, hi;
      const bool dense = item < a.n_dense_items;
      if (dense) {
        bk = item / a.Sd;
        lo = (item % a.Sd) * a.dense_rows;
        hi = min(W, lo + a.dense_rows);
      } else {
        const int x = item - (int)a.n_dense_items;
        int64_t l = 0, r = BK;  // largest bk with item_off[bk] <= x
        while (r - l > 1) {
          const int64_t mid = (l + r) >> 1;
          if (a.item_off[mid] <= x) l = mid; else r = mid;
        }
        bk = l;
        lo = (int64_t)(x - a.item_off[bk]) * a.sparse_rows;
        hi = min((int64_t)a.u_cnt[bk], lo + a.sparse_rows);
      }
      const int64_t b = bk / a.Hkv, kvh = bk % a.Hkv;
      const int nchunks = (int)((hi - lo + C::CH - 1) / C::CH);
      const unsigned char* qsrc = Qg + (b * a.Hq + kvh * G) * (int64_t)C::ROWB;
      const unsigned char* kbase = Kg + bk * a.T * (int64_t)C::ROWB;
      const unsigned char* vbase = Vg + bk * a.T * (int64_t)C::ROWB;
      for (int c = 0; c < nchunks; ++c, ++k) {
        const int s = k % C::S;
        if (k >= C::S) mbar_wait(&empty[s], ((k / C::S) - 1) & 1);
        unsigned char* st = stages + s * C::STAGE;
        int32_t* pos_s = reinterpret_cast<int32_t*>(st + C::OFF_POS);
        uint8_t* qm_s = st + C::OFF_QM;
        const int64_t r0 = lo + (int64_t)c * C::CH;
        const int nvalid = (int)min((int64_t)C::CH, hi - r0);
        for (int r = lane; r < C::CH; r += 32) {
          int32_t pos = 0;
          uint8_t qm = 0;
          if (r < nvalid) {
            if (dense) {
              pos = (int32_t)(a.dlo + r0 + r);
              qm = (uint8_t)((1u << G) - 1u);
            } else {
              pos = a.u_pos[bk * a.T + r0 + r];
              qm = a.u_qm[bk * a.T + r0 + r];
            }
          }
          pos_s[r] = pos;
          qm_s[r] = qm;
        }
        if (lane == 0) {
          st_item[s] = item;
          st_chunk[s] = c;
          st_nvalid[s] = nvalid;
          st_last[s] = (c == nchunks - 1) ? (dense ? 2 : 1) : 0;
        }
        __syncwarp();
        for (int t = lane; t < nvalid * C::PIECES; t += 32) {
          const int r = t / C::PIECES, p = t % C::PIECES;
          const int64_t off = (int64_t)pos_s[r] * C::ROWB + p * 16;
          cp_async16(st + r * C::KRS + p * 16, kbase + off);
          cp_async16(st + C::OFF_V + r * C::VRS + p * 16, vbase + off);
        }
        for (int t = lane; t < C::QB / 16; t += 32) cp_async16(st + C::OFF_Q + t * 16, qsrc + t * 16);
        cp_async_mbar_arrive_noinc(&full[s]);
        mbar_arrive(&full[s]);
      }
    }
    return;
  }

  // ------------------------------------------------------------------ consumers
  float acc[C::HPW][C::DPL];
  const int g0 = warp % C::GW, rsub = warp / C::GW;
  int k = 0;
  while (true) {
    const int s = k % C::S;
    mbar_wait(&full[s], (k / C::S) & 1);
    const int item = st_item[s];
    if (item < 0) break;
    const unsigned char* st = stages + s * C::STAGE;
    const int32_t* pos_s = reinterpret_cast<const int32_t*>(st + C::OFF_POS);
    const uint8_t* qm_s = st + C::OFF_QM;
    const int c = st_chunk[s], nvalid = st_nvalid[s], last = st_last[s];
    if (c == 0) {
      for (int t = tid; t < G * D; t += 128) {
        const T* qr = reinterpret_cast<const T*>(st + C::OFF_Q);
        qsh[t] = to_f64(qr[t]);
      }
      if (tid < G) {
        m_sh[tid] = -INFINITY;
        z_sh[tid] = 0.0;
      }
#pragma unroll
      for (int j = 0; j < C::HPW; ++j)
#pragma unroll
        for (int i = 0; i < C::DPL; ++i) acc[j][i] = 0.f;
      named_sync(1, 128);
    }
    // ---- scores: one row per thread, fp64, sequential over d
    if (tid < C::CH) {
      const int r = tid;
      const uint32_t qm = qm_s[r];
      const uint32_t wq = __reduce_or_sync(0xffffffffu, qm);
      double sacc[G];
#pragma unroll
      for (int g = 0; g < G; ++g) sacc[g] = 0.0;
      if (wq) {
        const unsigned char* krow = st + r * C::KRS;
#pragma unroll 2
        for (int p = 0; p < C::PIECES; ++p) {
          double kd[C::E];
          load_piece_f64<T>(krow + p * 16, kd);
#pragma unroll
          for (int g = 0; g < G; ++g) {
            if ((wq >> g) & 1u) {
              const double* qg = qsh + g * D + p * C::E;
#pragma unroll
              for (int e = 0; e < C::E; ++e) sacc[g] = fma(qg[e], kd[e], sacc[g]);
            }
          }
        }
      }
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const double sv = ((qm >> g) & 1u) ? sacc[g] * a.scale : -INFINITY;
        sc[g * C::CH + r] = sv;
      }
      if (item < a.n_dense_items && r < nvalid) {
        const int64_t bk = item / a.Sd;
        const int64_t b = bk / a.Hkv, kvh = bk % a.Hkv;
        const int64_t j = pos_s[r] - a.dlo;
#pragma unroll
        for (int g = 0; g < G; ++g) a.dsc[(b * a.Hq + kvh * G + g) * a.dsc_ld + j] = sc[g * C::CH + r];
      }
    }
    named_sync(1, 128);
    // ---- online softmax update (fp64), warp w owns heads w, w+4
    for (int g = warp; g < G; g += 4) {
      double cm = -INFINITY;
      for (int r = lane; r < C::CH; r += 32) cm = fmax(cm, sc[g * C::CH + r]);
      cm = warp_max_f64(cm);
      const double m_old = m_sh[g];
      const double mnew = fmax(m_old, cm);
      double zs = 0.0;
      double scal = 1.0;
      if (mnew == -INFINITY) {
        for (int r = lane; r < C::CH; r += 32) pf[g * C::CH + r] = 0.f;
      } else {
        scal = exp(m_old - mnew);
        for (int r = lane; r < C::CH; r += 32) {
          const double p = exp(sc[g * C::CH + r] - mnew);
          zs += p;
          pf[g * C::CH + r] = (float)p;
        }
      }
      zs = warp_sum_f64(zs);
      __syncwarp();
      if (lane == 0) {
        z_sh[g] = z_sh[g] * scal + zs;
        m_sh[g] = mnew;
        scal_sh[g] = scal;
      }
    }
    named_sync(1, 128);
    // ---- P.V (fp32): warp handles heads g0 + 4j over rows r = rsub (mod NPV)
#pragma unroll
    for (int j = 0; j < C::HPW; ++j) {
      const int g = g0 + 4 * j;
      const float sf = (float)scal_sh[g];
#pragma unroll
      for (int i = 0; i < C::DPL; ++i) acc[j][i] *= sf;
      const float* pg = pf + g * C::CH;
      for (int r = rsub; r < nvalid; r += C::NPV) {
        const float p = pg[r];
        if (p != 0.f) {
          float vv[C::DPL];
          load_v_f32<T, C::DPL>(st + C::OFF_V + r * C::VRS + lane * C::DPL * C::ESZ, vv);
#pragma unroll
          for (int i = 0; i < C::DPL; ++i) acc[j][i] = fmaf(p, vv[i], acc[j][i]);
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
    if (last) {
      // ---- emit this item's partial (fixed slot `item`)
      if (C::NPV == 1) {
#pragma unroll
        for (int j = 0; j < C::HPW; ++j) {
          const int g = g0 + 4 * j;
          float* dst = a.part_acc + ((int64_t)item * G + g) * D + lane * C::DPL;
#pragma unroll
          for (int i = 0; i < C::DPL; ++i) dst[i] = acc[j][i];
        }
      } else {
#pragma unroll
        for (int i = 0; i < C::DPL; ++i) accbuf[warp * D + lane * C::DPL + i] = acc[0][i];
        named_sync(1, 128);
        if (rsub == 0) {
          float* dst = a.part_acc + ((int64_t)item * G + g0) * D + lane * C::DPL;
#pragma unroll
          for (int i = 0; i < C::DPL; ++i) {
            float t = 0.f;
            for (int w2 = 0; w2 < C::NPV; ++w2) t += accbuf[(g0 + w2 * C::GW) * D + lane * C::DPL + i];
            dst[i] = t;
          }
        }
      }
      if (tid < G) {
        a.part_m[(int64_t)item * G + tid] = m_sh[tid];
        a.part_z[(int64_t)item * G + tid] = z_sh[tid];
      }
      named_sync(1, 128);
    }
    ++k;
  }
}

// --------------------------------------------------------------------- merge
// One CTA per (batch, query head). Folds dense and sparse partials in a fixed
// order, applies merge_states(sparse, dense) (engine.py:166-169), and updates
// the MAW of the attended window positions from the stored fp64 scores:
//   w   = float32(exp(s - m) / z)                     (_core.pyx:81-82)
//   maw = (1-alpha)*maw + alpha*w   (3 roundings)     (kv_cache.py:186)
//   new entries: maw = w                              (engine.py:191)
__global__ void __launch_bounds__(128) decode_merge_kernel(const DecodeMergeArgs a) {
  const int64_t bq = blockIdx.x;
  const int64_t b = bq / a.Hq, h = bq % a.Hq;
  const int64_t kvh = h / a.G, g = h % a.G;
  const int64_t bk = b * a.Hkv + kvh;
  const int tid = threadIdx.x;
  __shared__ double Md_s, Zd_s;
  // dense fold
  double Md = -INFINITY;
  for (int64_t i = 0; i < a.Sd; ++i) Md = fmax(Md, a.part_m[(bk * a.Sd + i) * a.G + g]);
  double Zd = 0.0;
  for (int64_t i = 0; i < a.Sd; ++i) {
    const double mi = a.part_m[(bk * a.Sd + i) * a.G + g];
    if (mi != -INFINITY) Zd += a.part_z[(bk * a.Sd + i) * a.G + g] * exp(mi - Md);
  }
  // sparse fold
  const int64_t i0 = a.n_dense_items + a.item_off[bk], i1 = a.n_dense_items + a.item_off[bk + 1];
  double Ms = -INFINITY;
  for (int64_t i = i0; i < i1; ++i) Ms = fmax(Ms, a.part_m[i * a.G + g]);
  double Zs = 0.0;
  for (int64_t i = i0; i < i1; ++i) {
    const double mi = a.part_m[i * a.G + g];
    if (mi != -INFINITY) Zs += a.part_z[i * a.G + g] * exp(mi - Ms);
  }
  const bool s_empty = !(Zs > 0.0);
  const bool d_empty = !(Zd > 0.0);
  const double lse_s = s_empty ? -INFINITY : Ms + log(Zs);
  const double lse_d = d_empty ? -INFINITY : Md + log(Zd);
  // merge_states coefficients (attention.py:170-182)
  const double m = fmax(lse_s, lse_d);
  const bool both_empty = m == -INFINITY;
  const double ms = both_empty ? 0.0 : m;
  const double wa = exp(lse_s - ms), wb = exp(lse_d - ms);
  const double zs = both_empty ? 1.0 : wa + wb;
  const float ca = (float)(wa / zs), cb = (float)(wb / zs);
  for (int64_t c = tid; c < a.D; c += blockDim.x) {
    double ad = 0.0, as = 0.0;
    for (int64_t i = 0; i < a.Sd; ++i) {
      const double mi = a.part_m[(bk * a.Sd + i) * a.G + g];
      if (mi != -INFINITY) ad += (double)a.part_acc[((bk * a.Sd + i) * a.G + g) * a.D + c] * exp(mi - Md);
    }
    for (int64_t i = i0; i < i1; ++i) {
      const double mi = a.part_m[i * a.G + g];
      if (mi != -INFINITY) as += (double)a.part_acc[(i * a.G + g) * a.D + c] * exp(mi - Ms);
    }
    const float od = d_empty ? 0.f : (float)(ad / Zd);
    const float os = s_empty ? 0.f : (float)(as / Zs);
    a.out[bq * a.D + c] = __fadd_rn(__fmul_rn(ca, os), __fmul_rn(cb, od));
    if (a.out_sparse) a.out_sparse[bq * a.D + c] = os;
  }
  if (tid == 0) {
    a.lse[bq] = both_empty ? -INFINITY : ms + log(zs);
    if (a.lse_sparse) a.lse_sparse[bq] = lse_s;
    Md_s = Md;
    Zd_s = Zd;
  }
  __syncthreads();
  if (a.maw == nullptr && a.wts_out == nullptr) return;
  for (int64_t j = tid; j < a.W; j += blockDim.x) {
    const float w32 = d_empty ? 0.f : (float)(exp(a.dsc[bq * a.dsc_ld + j] - Md_s) / Zd_s);
    if (a.wts_out) a.wts_out[bq * a.W + j] = w32;
    if (a.maw) {
      double* mp = a.maw + bq * a.T + a.dlo + j;
      const double aw = (double)w32;
      *mp = j < a.w_old ? __dadd_rn(__dmul_rn(a.one_minus_alpha, *mp), __dmul_rn(a.alpha, aw)) : aw;
    }
  }
}

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
template <typename T, int D, int G>
static int launch_decode_t(const DecodeArgs& a, cudaStream_t s) {
  using C = DecodeCfg<T, D, G>;
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
  decode_partial_kernel<T, D, G><<<nsm, 160, C::SMEM, s>>>(a);
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
  const int64_t esz = dtype == kBF16 ? 2 : 4;
  return D * esz <= 256 ? 128 : 64;
}

int launch_decode_partial(int dtype, const DecodeArgs& a, cudaStream_t s) {
  cudaError_t e = cudaMemsetAsync(a.counter, 0, sizeof(int32_t), s);
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

int launch_decode_merge(const DecodeMergeArgs& a, cudaStream_t s) {
  decode_merge_kernel<<<(unsigned)(a.B * a.Hq), 128, 0, s>>>(a);
  return (int)cudaGetLastError();
}

int launch_union_build(const uint32_t* sel, int64_t B, int64_t Hq, int64_t Hkv, int64_t words,
                       int64_t n_arch, int64_t T, int32_t* u_pos, uint8_t* u_qm, int32_t* u_cnt,
                       int32_t* item_off, int64_t sparse_rows, cudaStream_t s) {
  const int64_t G = Hq / Hkv;
  union_build_kernel<<<(unsigned)(B * Hkv), 1024, 0, s>>>(sel, Hq, Hkv, G, words, n_arch, T, u_pos,
                                                          u_qm, u_cnt);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return (int)e;
  item_offsets_kernel<<<1, 1024, 0, s>>>(u_cnt, B * Hkv, sparse_rows, item_off);
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
