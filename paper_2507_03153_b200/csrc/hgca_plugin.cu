// Reference-exact attention, merge and selection kernels behind the tierkv
// backend contract (backends.py:8-20). These serve the drop-in plugin path
// (attend / attend_indexed / merge_states / select_salient / pack_head_groups)
// and the engine's append/re-evaluation path; the decode hot path lives in
// hgca_decode.cu.
//
// Numerics follow _core.pyx:56-82: scores are sequential fp64 dot products of
// exactly-converted inputs (so every product is exact and the sum rounds in the
// reference's order), softmax statistics and weights are fp64, weights and
// outputs are rounded to the input dtype at the end.
#include "hgca_common.cuh"
#include "hgca_internal.h"

namespace hgca {

// s += (double)q * (double)k. For fp32/bf16 inputs the product is exact in
// fp64, so one fused multiply-add rounds exactly like the reference's separate
// multiply and add; for fp64 inputs the two roundings are kept explicitly.
template <typename T>
__device__ __forceinline__ double dot_step(double s, double q, T k) {
  return fma(q, to_f64(k), s);
}
template <>
__device__ __forceinline__ double dot_step<double>(double s, double q, double k) {
  return __dadd_rn(s, __dmul_rn(q, k));
}

// Output / weight element type: the input dtype for the reference's float32 /
// float64 contract; float32 for bfloat16 storage (no reference contract).
template <typename T> struct OutT { using type = T; };
template <> struct OutT<__nv_bfloat16> { using type = float; };

// Element c of a rotated row (position p): 16-byte chunk (c / epc) sits at
// (chunk & ~7) | ((chunk ^ p) & 7) -- the engine's bf16 K|V layout.
__device__ __forceinline__ int64_t rot_elem(int64_t c, int64_t p, int64_t epc) {
  const int64_t ch = c / epc;
  return (((ch & ~7) | ((ch ^ p) & 7)) * epc) + c % epc;
}

// One CTA per (query row i, head bh). K/V rows for head bh start at
//   kv + kv_head_index(bh) * ld_head + row0 * ld_row
// (row stride ld_row: d for plain [.., n, d] buffers, 2d for the engine's
// interleaved K|V rows) and are either the first n rows (dense) or the rows
// listed in idx.
template <typename T>
__global__ void __launch_bounds__(256) attend_rows_kernel(AttendArgs a) {
  using O = typename OutT<T>::type;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* qs = reinterpret_cast<double*>(smem_raw);  // [d]
  double* red = qs + a.d;                            // [blockDim]
  const int i = blockIdx.x;
  const int64_t bh = blockIdx.y;
  const int tid = threadIdx.x, nt = blockDim.x;
  const int64_t d = a.d;
  const int64_t b = bh / a.Hq, h = bh % a.Hq;
  const int64_t kvh = b * a.Hkv + h / a.G;
  const T* q = reinterpret_cast<const T*>(a.q) + (bh * a.nq + i) * d;
  const int64_t ldr = a.ld_row;
  const T* k = reinterpret_cast<const T*>(a.k) + kvh * a.ld_head + a.row0 * ldr;
  const T* v = reinterpret_cast<const T*>(a.v) + kvh * a.ld_head + a.row0 * ldr;
  const int64_t* idx = a.idx ? a.idx + (a.idx_off ? a.idx_off[bh] : 0) : nullptr;
  const int64_t n = a.idx_cnt ? a.idx_cnt[bh] : a.n;
  O* out = reinterpret_cast<O*>(a.out) + (bh * a.nq + i) * d;
  double* lse = a.lse + bh * a.nq + i;
  double* sc = a.ws + (bh * a.nq + i) * a.ws_ld;
  O* wts = a.wts ? reinterpret_cast<O*>(a.wts) + (bh * a.nq + i) * a.wts_ld : nullptr;

  if (n == 0) {
    for (int64_t c = tid; c < d; c += nt) out[c] = from_f64<O>(0.0);
    if (tid == 0) *lse = -INFINITY;
    return;
  }
  for (int64_t c = tid; c < d; c += nt) qs[c] = to_f64(q[c]);
  __syncthreads();
  // scores: one key row per thread, sequential over c (_core.pyx:59-67)
  double m = -INFINITY;
  for (int64_t j = tid; j < n; j += nt) {
    const int64_t r = idx ? idx[j] : j;
    const T* kr = k + r * ldr;
    double s = 0.0;
    if (a.rot) {
      const int64_t p = a.row0 + r, epc = 16 / (int64_t)sizeof(T);
      for (int64_t c = 0; c < d; ++c) s = dot_step<T>(s, qs[c], kr[rot_elem(c, p, epc)]);
    } else {
      for (int64_t c = 0; c < d; ++c) s = dot_step<T>(s, qs[c], kr[c]);
    }
    s = s * a.scale;
    sc[j] = s;
    m = fmax(m, s);
  }
  red[tid] = m;
  __syncthreads();
  for (int o = nt / 2; o > 0; o >>= 1) {
    if (tid < o) red[tid] = fmax(red[tid], red[tid + o]);
    __syncthreads();
  }
  m = red[0];
  __syncthreads();
  // w = exp(s - m), z = sum w (fixed-shape tree)  (_core.pyx:68-74)
  double z = 0.0;
  for (int64_t j = tid; j < n; j += nt) {
    double w = exp(sc[j] - m);
    sc[j] = w;
    z += w;
  }
  red[tid] = z;
  __syncthreads();
  for (int o = nt / 2; o > 0; o >>= 1) {
    if (tid < o) red[tid] += red[tid + o];
    __syncthreads();
  }
  z = red[0];
  __syncthreads();
  // acc[c] = sum_j w_j * v[j][c]; sequential in j per segment (_core.pyx:75-76),
  // segments combined in order. One segment (exact reference order) for n < 512.
  int nseg = (int)(nt / d);
  if (nseg < 1) nseg = 1;
  if (n < 512) nseg = 1;
  const int64_t seg_len = (n + nseg - 1) / nseg;
  double* part = red;  // reuse: [nseg * d] must fit in blockDim doubles -> d*nseg <= nt
  for (int64_t t = tid; t < (int64_t)nseg * d; t += nt) {
    const int64_t c = t % d, sg = t / d;
    const int64_t j0 = sg * seg_len, j1 = min(n, j0 + seg_len);
    double acc = 0.0;
    for (int64_t j = j0; j < j1; ++j) {
      const int64_t r = idx ? idx[j] : j;
      const int64_t cc = a.rot ? rot_elem(c, a.row0 + r, 16 / (int64_t)sizeof(T)) : c;
      acc = __dadd_rn(acc, __dmul_rn(sc[j], to_f64(v[r * ldr + cc])));
    }
    if (nseg == 1) {
      out[c] = from_f64<O>(acc / z);
    } else {
      part[t] = acc;
    }
  }
  if (nseg > 1) {
    __syncthreads();
    for (int64_t c = tid; c < d; c += nt) {
      double acc = 0.0;
      for (int sg = 0; sg < nseg; ++sg) acc += part[sg * d + c];
      out[c] = from_f64<O>(acc / z);
    }
  }
  if (tid == 0) *lse = m + log(z);
  if (wts)
    for (int64_t j = tid; j < n; j += nt) wts[j] = from_f64<O>(sc[j] / z);
}

// merge_states (attention.py:153-188): coefficients in fp64, cast to the
// output dtype, then ca*a + cb*b in that dtype with separate roundings.
template <typename T>
__global__ void merge_states_kernel(MergeArgs a) {
  const int64_t r = blockIdx.x;
  const double la = a.lse_a[r], lb = a.lse_b[r];
  const double m = fmax(la, lb);
  const bool both_empty = isinf(m) && m < 0;
  const double ms = both_empty ? 0.0 : m;
  const double wa = exp(la - ms), wb = exp(lb - ms);
  const double zs = both_empty ? 1.0 : wa + wb;
  const T ca = from_f64<T>(wa / zs), cb = from_f64<T>(wb / zs);
  const T* oa = reinterpret_cast<const T*>(a.out_a) + r * a.d;
  const T* ob = reinterpret_cast<const T*>(a.out_b) + r * a.d;
  T* o = reinterpret_cast<T*>(a.out) + r * a.d;
  for (int64_t c = threadIdx.x; c < a.d; c += blockDim.x) o[c] = ca * oa[c] + cb * ob[c];
  if (threadIdx.x == 0) a.lse[r] = both_empty ? -INFINITY : ms + log(zs);
  if (a.w_out) {
    const T* wa_ = reinterpret_cast<const T*>(a.w_a) + r * a.na;
    const T* wb_ = reinterpret_cast<const T*>(a.w_b) + r * a.nb;
    T* wo = reinterpret_cast<T*>(a.w_out) + r * (a.na + a.nb);
    for (int64_t j = threadIdx.x; j < a.na; j += blockDim.x) wo[j] = ca * wa_[j];
    for (int64_t j = threadIdx.x; j < a.nb; j += blockDim.x) wo[a.na + j] = cb * wb_[j];
  }
}

// fp32 products must not be contracted into FMAs to match numpy's separately
// rounded multiply and add.
template <>
__global__ void merge_states_kernel<float>(MergeArgs a) {
  const int64_t r = blockIdx.x;
  const double la = a.lse_a[r], lb = a.lse_b[r];
  const double m = fmax(la, lb);
  const bool both_empty = isinf(m) && m < 0;
  const double ms = both_empty ? 0.0 : m;
  const double wa = exp(la - ms), wb = exp(lb - ms);
  const double zs = both_empty ? 1.0 : wa + wb;
  const float ca = (float)(wa / zs), cb = (float)(wb / zs);
  const float* oa = reinterpret_cast<const float*>(a.out_a) + r * a.d;
  const float* ob = reinterpret_cast<const float*>(a.out_b) + r * a.d;
  float* o = reinterpret_cast<float*>(a.out) + r * a.d;
  for (int64_t c = threadIdx.x; c < a.d; c += blockDim.x)
    o[c] = __fadd_rn(__fmul_rn(ca, oa[c]), __fmul_rn(cb, ob[c]));
  if (threadIdx.x == 0) a.lse[r] = both_empty ? -INFINITY : ms + log(zs);
  if (a.w_out) {
    const float* wa_ = reinterpret_cast<const float*>(a.w_a) + r * a.na;
    const float* wb_ = reinterpret_cast<const float*>(a.w_b) + r * a.nb;
    float* wo = reinterpret_cast<float*>(a.w_out) + r * (a.na + a.nb);
    for (int64_t j = threadIdx.x; j < a.na; j += blockDim.x) wo[j] = __fmul_rn(ca, wa_[j]);
    for (int64_t j = threadIdx.x; j < a.nb; j += blockDim.x) wo[a.na + j] = __fmul_rn(cb, wb_[j]);
  }
}
template <>
__global__ void merge_states_kernel<double>(MergeArgs a) {
  const int64_t r = blockIdx.x;
  const double la = a.lse_a[r], lb = a.lse_b[r];
  const double m = fmax(la, lb);
  const bool both_empty = isinf(m) && m < 0;
  const double ms = both_empty ? 0.0 : m;
  const double wa = exp(la - ms), wb = exp(lb - ms);
  const double zs = both_empty ? 1.0 : wa + wb;
  const double ca = wa / zs, cb = wb / zs;
  const double* oa = reinterpret_cast<const double*>(a.out_a) + r * a.d;
  const double* ob = reinterpret_cast<const double*>(a.out_b) + r * a.d;
  double* o = reinterpret_cast<double*>(a.out) + r * a.d;
  for (int64_t c = threadIdx.x; c < a.d; c += blockDim.x)
    o[c] = __dadd_rn(__dmul_rn(ca, oa[c]), __dmul_rn(cb, ob[c]));
  if (threadIdx.x == 0) a.lse[r] = both_empty ? -INFINITY : ms + log(zs);
  if (a.w_out) {
    const double* wa_ = reinterpret_cast<const double*>(a.w_a) + r * a.na;
    const double* wb_ = reinterpret_cast<const double*>(a.w_b) + r * a.nb;
    double* wo = reinterpret_cast<double*>(a.w_out) + r * (a.na + a.nb);
    for (int64_t j = threadIdx.x; j < a.na; j += blockDim.x) wo[j] = __dmul_rn(ca, wa_[j]);
    for (int64_t j = threadIdx.x; j < a.nb; j += blockDim.x) wo[a.na + j] = __dmul_rn(cb, wb_[j]);
  }
}

// ------------------------------------------------------------------ selection
// Strict threshold maw > thr over positions [p0, p1) of each row
// (select_salient, sparsifier.py:32-42). One thread per 32-position word; the
// word is read-modify-written by a single thread (no atomics). assign=1 clears
// the row's bits in [p0, p1) first (re-evaluation), assign=0 ORs (ingest).
// keep (optional, [words]) restricts selection to the positions this rank
// owns under sequence sharding (block-cyclic archive shards).
__global__ void threshold_mask_kernel(const double* __restrict__ maw, int64_t rows, int64_t ld,
                                      int64_t p0, int64_t p1, double thr, uint32_t* mask,
                                      int64_t words, int assign, const uint32_t* __restrict__ keep) {
  const int64_t w0 = p0 >> 5, w1 = (p1 + 31) >> 5;
  const int64_t nw = w1 - w0;
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nw * rows) return;
  const int64_t r = t / nw, w = w0 + t % nw;
  uint32_t bits = 0, inrange = 0;
  const double* row = maw + r * ld;
#pragma unroll 4
  for (int b = 0; b < 32; ++b) {
    const int64_t p = (w << 5) + b;
    if (p >= p0 && p < p1) {
      inrange |= 1u << b;
      if (row[p] > thr) bits |= 1u << b;
    }
  }
  if (keep) bits &= keep[w];
  uint32_t* mw = mask + r * words + w;
  const uint32_t old = *mw;
  *mw = assign ? ((old & ~inrange) | bits) : (old | bits);
}

// Compact set bits of (mask_a | mask_b) over [0, n) into ascending int64
// indices; flags[j] = 1 when the entry came only from mask_b (padding).
__global__ void __launch_bounds__(1024) mask_to_indices_kernel(
    const uint32_t* __restrict__ mask_a, const uint32_t* __restrict__ mask_b, int64_t words,
    int64_t n, int64_t* idx_out, int64_t ld_out, uint8_t* flags_out, int64_t* counts) {
  __shared__ int wsum[32];
  __shared__ int64_t base_s;
  const int64_t r = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nwarp = blockDim.x >> 5;
  const int64_t nw = (n + 31) >> 5;
  if (tid == 0) base_s = 0;
  __syncthreads();
  for (int64_t w0 = 0; w0 < nw; w0 += blockDim.x) {
    const int64_t w = w0 + tid;
    uint32_t a = 0, b = 0;
    if (w < nw) {
      a = mask_a ? mask_a[r * words + w] : 0u;
      b = mask_b ? mask_b[r * words + w] : 0u;
      const int64_t rem = n - (w << 5);
      if (rem < 32) {
        const uint32_t keep = rem <= 0 ? 0u : ((1u << rem) - 1u);
        a &= keep;
        b &= keep;
      }
    }
    const uint32_t bits = a | b;
    const int c = __popc(bits);
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
    int64_t pos = base_s + (wid ? wsum[wid - 1] : 0) + (incl - c);
    uint32_t bb = bits;
    while (bb) {
      const int bit = __ffs(bb) - 1;
      bb &= bb - 1;
      idx_out[r * ld_out + pos] = (w << 5) + bit;
      if (flags_out) flags_out[r * ld_out + pos] = ((a >> bit) & 1u) ? 0 : 1;
      ++pos;
    }
    __syncthreads();
    if (tid == 0) base_s += wsum[nwarp - 1];
    __syncthreads();
  }
  if (tid == 0 && counts) counts[r] = base_s;
}

__global__ void popcount_rows_kernel(const uint32_t* __restrict__ mask, int64_t rows, int64_t words,
                                     int64_t n, int64_t* counts) {
  const int64_t r = blockIdx.x;
  const int64_t nw = (n + 31) >> 5;
  int c = 0;
  for (int64_t w = threadIdx.x; w < nw; w += blockDim.x) {
    uint32_t x = mask[r * words + w];
    const int64_t rem = n - (w << 5);
    if (rem < 32) x &= (1u << rem) - 1u;
    c += __popc(x);
  }
  c = warp_sum_i32(c);
  __shared__ int s[32];
  if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    int64_t t = 0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) t += s[i];
    counts[r] = t;
  }
}

// Padding targets (sparsifier.py:209-217): heads are grouped g at a time within
// each batch element; need = max(count in group) - count.
__global__ void group_need_kernel(const int64_t* counts, int64_t B, int64_t H, int64_t g,
                                  int64_t* need) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= B * H) return;
  const int64_t b = t / H, h = t % H;
  const int64_t lo = (h / g) * g, hi = min(H, lo + g);
  int64_t mx = 0;
  for (int64_t x = lo; x < hi; ++x) mx = max(mx, counts[b * H + x]);
  need[t] = mx - counts[t];
}

// Top-k by (maw descending, position ascending) among candidates [0, n) not in
// `exclude` (the padding order of sparsifier.py:219-226; also the topk(f)
// extension). One CTA per row: MSB-first 8-bit radix select on the 64-bit
// monotone key, then the lowest positions among keys equal to the boundary.
__global__ void __launch_bounds__(1024) topk_mask_kernel(const double* __restrict__ maw, int64_t ld,
                                                         int64_t n, const int64_t* __restrict__ kk,
                                                         const uint32_t* __restrict__ exclude,
                                                         uint32_t* out, int64_t words) {
  __shared__ unsigned int hist[256];
  __shared__ uint64_t prefix_s;
  __shared__ int64_t remain_s;
  __shared__ int wsum[32];
  __shared__ int64_t base_s;
  const int64_t r = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nwarp = blockDim.x >> 5;
  const double* row = maw + r * ld;
  const uint32_t* ex = exclude ? exclude + r * words : nullptr;
  uint32_t* o = out + r * words;
  int64_t k = kk[r];
  // number of candidates
  if (k <= 0) return;
  auto is_cand = [&](int64_t p) -> bool { return !(ex && ((ex[p >> 5] >> (p & 31)) & 1u)); };
  uint64_t prefix = 0;
  if (tid == 0) remain_s = k;
  __syncthreads();
  int64_t ncand_total = 0;
  {
    int c = 0;
    for (int64_t p = tid; p < n; p += blockDim.x) c += is_cand(p) ? 1 : 0;
    c = warp_sum_i32(c);
    if (lane == 0) wsum[wid] = c;
    __syncthreads();
    for (int i = 0; i < nwarp; ++i) ncand_total += wsum[i];
    __syncthreads();
  }
  if (k >= ncand_total) {  // every candidate is taken
    for (int64_t w = tid; w < ((n + 31) >> 5); w += blockDim.x) {
      uint32_t bits = 0;
      for (int b = 0; b < 32; ++b) {
        const int64_t p = (w << 5) + b;
        if (p < n && is_cand(p)) bits |= 1u << b;
      }
      o[w] |= bits;
    }
    return;
  }
  for (int shift = 56; shift >= 0; shift -= 8) {
    for (int i = tid; i < 256; i += blockDim.x) hist[i] = 0;
    __syncthreads();
    const uint64_t hmask = shift == 56 ? 0ull : (~0ull << (shift + 8));
    for (int64_t p = tid; p < n; p += blockDim.x) {
      if (!is_cand(p)) continue;
      const uint64_t key = f64_key(row[p]);
      if ((key & hmask) != (prefix & hmask)) continue;
      atomicAdd(&hist[(key >> shift) & 0xFF], 1u);
    }
    __syncthreads();
    if (tid == 0) {
      int64_t rem = remain_s;
      int dsel = 0;
      for (int dgt = 255; dgt >= 0; --dgt) {
        if ((int64_t)hist[dgt] >= rem) {
          dsel = dgt;
          break;
        }
        rem -= hist[dgt];
      }
      remain_s = rem;
      prefix_s = prefix | ((uint64_t)dsel << shift);
    }
    __syncthreads();
    prefix = prefix_s;
  }
  // prefix == boundary key T; take all keys > T and the first `remain` (by
  // position) keys == T.
  const uint64_t T = prefix;
  const int64_t take_eq = remain_s;
  if (tid == 0) base_s = 0;
  __syncthreads();
  const int64_t nw = (n + 31) >> 5;
  for (int64_t w0 = 0; w0 < nw; w0 += blockDim.x) {
    const int64_t w = w0 + tid;
    uint32_t gt = 0, eq = 0;
    if (w < nw) {
      for (int b = 0; b < 32; ++b) {
        const int64_t p = (w << 5) + b;
        if (p >= n || !is_cand(p)) continue;
        const uint64_t key = f64_key(row[p]);
        if (key > T) gt |= 1u << b;
        else if (key == T) eq |= 1u << b;
      }
    }
    const int c = __popc(eq);
    int incl = c;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, off);
      if (lane >= off) incl += y;
    }
    if (lane == 31) wsum[wid] = incl;
    __syncthreads();
    if (wid == 0) {
      int x = lane < nwarp ? wsum[lane] : 0;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, off);
        if (lane >= off) x += y;
      }
      if (lane < nwarp) wsum[lane] = x;
    }
    __syncthreads();
    int64_t rank = base_s + (wid ? wsum[wid - 1] : 0) + (incl - c);
    uint32_t take = gt;
    uint32_t e = eq;
    while (e) {
      const int bit = __ffs(e) - 1;
      e &= e - 1;
      if (rank < take_eq) take |= 1u << bit;
      ++rank;
    }
    if (w < nw && take) o[w] |= take;
    __syncthreads();
    if (tid == 0) base_s += wsum[nwarp - 1];
    __syncthreads();
  }
}

int launch_attend(int dtype, const AttendArgs& a, int64_t BH, cudaStream_t s) {
  if (a.nq == 0 || BH == 0) return 0;
  const int threads = 256;
  const size_t smem = (size_t)(a.d + threads) * sizeof(double);
  dim3 grid((unsigned)a.nq, (unsigned)BH);
  if (dtype == kF32)
    attend_rows_kernel<float><<<grid, threads, smem, s>>>(a);
  else if (dtype == kF64)
    attend_rows_kernel<double><<<grid, threads, smem, s>>>(a);
  else if (dtype == kBF16)
    attend_rows_kernel<__nv_bfloat16><<<grid, threads, smem, s>>>(a);
  else
    return -2000;
  return (int)cudaGetLastError();
}

int launch_merge(int dtype, const MergeArgs& a, cudaStream_t s) {
  if (a.rows == 0) return 0;
  if (dtype == kF32)
    merge_states_kernel<float><<<(unsigned)a.rows, 128, 0, s>>>(a);
  else if (dtype == kF64)
    merge_states_kernel<double><<<(unsigned)a.rows, 128, 0, s>>>(a);
  else
    return -2001;
  return (int)cudaGetLastError();
}


int launch_threshold_mask(const double* maw, int64_t rows, int64_t ld, int64_t p0, int64_t p1,
                          double thr, uint32_t* mask, int64_t words, int assign, const uint32_t* keep,
                          cudaStream_t s) {
  const int64_t nw = ((p1 + 31) >> 5) - (p0 >> 5);
  const int64_t total = nw * rows;
  if (total == 0) return 0;
  threshold_mask_kernel<<<(unsigned)((total + 255) / 256), 256, 0, s>>>(maw, rows, ld, p0, p1, thr,
                                                                         mask, words, assign, keep);
  return (int)cudaGetLastError();
}

int launch_mask_to_indices(const uint32_t* a, const uint32_t* b, int64_t rows, int64_t words,
                           int64_t n, int64_t* idx, int64_t ld, uint8_t* flags, int64_t* counts,
                           cudaStream_t s) {
  mask_to_indices_kernel<<<(unsigned)rows, 1024, 0, s>>>(a, b, words, n, idx, ld, flags, counts);
  return (int)cudaGetLastError();
}

int launch_popcount_rows(const uint32_t* mask, int64_t rows, int64_t words, int64_t n,
                         int64_t* counts, cudaStream_t s) {
  popcount_rows_kernel<<<(unsigned)rows, 256, 0, s>>>(mask, rows, words, n, counts);
  return (int)cudaGetLastError();
}

int launch_group_need(const int64_t* counts, int64_t B, int64_t H, int64_t g, int64_t* need,
                      cudaStream_t s) {
  group_need_kernel<<<(unsigned)((B * H + 255) / 256), 256, 0, s>>>(counts, B, H, g, need);
  return (int)cudaGetLastError();
}

int launch_topk_mask(const double* maw, int64_t rows, int64_t ld, int64_t n, const int64_t* k,
                     const uint32_t* exclude, uint32_t* out, int64_t words, cudaStream_t s) {
  topk_mask_kernel<<<(unsigned)rows, 1024, 0, s>>>(maw, ld, n, k, exclude, out, words);
  return (int)cudaGetLastError();
}


// MAW maintenance from dense / archive weight rows w [BH, nq, w_ld] (float32):
//   a_j = (sum_i (double)w[i][j]) / nq   (numpy mean over rows: sequential
//                                          row sum, then divide; engine.py:177, 181)
//   mode 0: j <  w_old -> maw = (1-alpha)*maw + alpha*a  (kv_cache.py:186)
//           j >= w_old -> maw = a                        (init_maw, engine.py:191)
//   mode 1: maw = a                                      (reevaluate, sparsifier.py:174)
__global__ void maw_update_kernel(const float* __restrict__ w, int64_t BH, int64_t nq, int64_t W,
                                  int64_t w_ld, double* maw, int64_t T, int64_t p0, int64_t w_old,
                                  double one_minus_alpha, double alpha, int mode) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= BH * W) return;
  const int64_t bh = t / W, j = t % W;
  double s = 0.0;
  for (int64_t i = 0; i < nq; ++i) s += (double)w[(bh * nq + i) * w_ld + j];
  const double a = s / (double)nq;
  double* mp = maw + bh * T + p0 + j;
  if (mode == 0 && j < w_old)
    *mp = __dadd_rn(__dmul_rn(one_minus_alpha, *mp), __dmul_rn(alpha, a));
  else
    *mp = a;
}

// f64 EMA of fp64 weights a [rows, lda] into maw [rows, ld] over [0, n):
// (1 - alpha) * maw + alpha * a with three separately rounded ops
// (kv_cache.py:186) -- WindowCache.update_maw.
__global__ void maw_ema_kernel(double* maw, int64_t rows, int64_t ld, int64_t n, const double* __restrict__ a,
                               int64_t lda, double one_minus_alpha, double alpha) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < rows * n;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = t / n, j = t % n;
    double* mp = maw + r * ld + j;
    *mp = __dadd_rn(__dmul_rn(one_minus_alpha, *mp), __dmul_rn(alpha, a[r * lda + j]));
  }
}

int launch_maw_ema(double* maw, int64_t rows, int64_t ld, int64_t n, const double* a, int64_t lda, double alpha,
                   cudaStream_t s) {
  const int64_t total = rows * n;
  if (total == 0) return 0;
  const int64_t nb = (total + 255) / 256;
  maw_ema_kernel<<<(unsigned)(nb < 148 * 16 ? nb : 148 * 16), 256, 0, s>>>(maw, rows, ld, n, a, lda, 1.0 - alpha,
                                                                           alpha);
  return (int)cudaGetLastError();
}

int launch_maw_update(const float* w, int64_t BH, int64_t nq, int64_t W, int64_t w_ld, double* maw,
                      int64_t T, int64_t p0, int64_t w_old, double alpha, int mode, cudaStream_t s) {
  const int64_t total = BH * W;
  if (total == 0) return 0;
  maw_update_kernel<<<(unsigned)((total + 255) / 256), 256, 0, s>>>(w, BH, nq, W, w_ld, maw, T, p0, w_old,
                                                                    1.0 - alpha, alpha, mode);
  return (int)cudaGetLastError();
}

}  // namespace hgca
