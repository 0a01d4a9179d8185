// extern "C" boundary of libhgca_b200.so (declared in include/hgca_b200.h).
// Validation mirrors the reference's ContractError checks (attention.py:94-114,
// 133-144; sparsifier.py:38-39) and maps them to HGCA_EINVAL.
#include <cstdarg>
#include <cstdio>
#include <cstring>

#include "hgca_common.cuh"
#include "hgca_internal.h"

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include "../../include/hgca_b200.h"

namespace hgca {

static thread_local char g_err[512] = "";

static int fail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

static int cuda_status(int e, const char* what) {
  if (e == 0) return HGCA_OK;
  if (e > 0) return fail(HGCA_ECUDA, "%s: %s", what, cudaGetErrorString((cudaError_t)e));
  return fail(HGCA_EINVAL, "%s: unsupported configuration (code %d)", what, e);
}

__global__ void merge_partials_kernel(const float* outs, const double* lses, int64_t P, int64_t rows,
                                      int64_t d, float* out, double* lse) {
  const int64_t r = blockIdx.x;
  double M = -INFINITY;
  for (int64_t p = 0; p < P; ++p) M = fmax(M, lses[p * rows + r]);
  if (M == -INFINITY) {
    for (int64_t c = threadIdx.x; c < d; c += blockDim.x) out[r * d + c] = 0.f;
    if (threadIdx.x == 0) lse[r] = -INFINITY;
    return;
  }
  double Z = 0.0;
  for (int64_t p = 0; p < P; ++p) Z += exp(lses[p * rows + r] - M);
  for (int64_t c = threadIdx.x; c < d; c += blockDim.x) {
    double acc = 0.0;
    for (int64_t p = 0; p < P; ++p) {
      const double w = exp(lses[p * rows + r] - M);
      if (w != 0.0) acc += w * (double)outs[(p * rows + r) * d + c];
    }
    out[r * d + c] = (float)(acc / Z);
  }
  if (threadIdx.x == 0) lse[r] = M + log(Z);
}

// P-way merge of packed per-rank partials (the receive buffer of the
// sequence-sharded allgather): partial p holds out [rows, d] f32 at
// parts + p*stride and lse [rows] f64 right after it. Same fold as
// merge_partials_kernel, in rank order, so every rank computes identical bits.
__global__ void merge_packed_kernel(const unsigned char* parts, int64_t P, int64_t rows, int64_t d,
                                    int64_t stride, float* out, double* lse, const int32_t* err) {
  const int64_t r = blockIdx.x;
  if (err && *(volatile const int32_t*)err) {  // a peer's partial never arrived: poison, never merge stale data
    for (int64_t c = threadIdx.x; c < d; c += blockDim.x) out[r * d + c] = __int_as_float(0x7fc00000);
    if (threadIdx.x == 0) lse[r] = __longlong_as_double(0x7ff8000000000000LL);
    return;
  }
  const int64_t lse_off = rows * d * 4;
  auto L = [&](int64_t p) { return reinterpret_cast<const double*>(parts + p * stride + lse_off)[r]; };
  double M = -INFINITY;
  for (int64_t p = 0; p < P; ++p) M = fmax(M, L(p));
  if (M == -INFINITY) {
    for (int64_t c = threadIdx.x; c < d; c += blockDim.x) out[r * d + c] = 0.f;
    if (threadIdx.x == 0) lse[r] = -INFINITY;
    return;
  }
  double Z = 0.0;
  for (int64_t p = 0; p < P; ++p) Z += exp(L(p) - M);
  for (int64_t c = threadIdx.x; c < d; c += blockDim.x) {
    double acc = 0.0;
    for (int64_t p = 0; p < P; ++p) {
      const double w = exp(L(p) - M);
      if (w != 0.0) acc += w * (double)reinterpret_cast<const float*>(parts + p * stride)[r * d + c];
    }
    out[r * d + c] = (float)(acc / Z);
  }
  if (threadIdx.x == 0) lse[r] = M + log(Z);
}

// One CTA, one thread per flag: spin (acquire, system scope) until every
// peer has published this step's epoch, or the timeout passes.
__global__ void wait_flags_kernel(const unsigned long long* flags, int64_t n, unsigned long long epoch,
                                  long long timeout_ns, int32_t* err) {
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    long long t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (;;) {
      unsigned long long v;
      asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(flags + i) : "memory");
      if (v >= epoch) break;
      long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if (t - t0 > timeout_ns) {
        if (err) atomicExch(err, 1);
        break;
      }
      __nanosleep(64);
    }
  }
}

}  // namespace hgca

using namespace hgca;

static inline cudaStream_t S(hgca_stream_t s) { return reinterpret_cast<cudaStream_t>(s); }

extern "C" {

int hgca_version(void) { return 1; }
const char* hgca_last_error(void) { return g_err; }

int64_t hgca_attend_ws_bytes(int64_t rows, int64_t nkeys) {
  return (rows > 0 ? rows : 1) * (nkeys > 0 ? nkeys : 1) * (int64_t)sizeof(double);
}

int hgca_attend_dense(int dtype, const void* q, const void* k, const void* v, int64_t H, int64_t nq,
                      int64_t nkv, int64_t d, double scale, int keep_weights, void* out,
                      double* lse, void* weights, void* ws, hgca_stream_t stream) {
  if (dtype != HGCA_DTYPE_F32 && dtype != HGCA_DTYPE_F64)
    return fail(HGCA_EINVAL, "attend_dense: dtype must be float32 or float64");
  if (H < 0 || nq < 0 || nkv < 0 || d < 1) return fail(HGCA_EINVAL, "attend_dense: bad shape");
  if (!(scale > 0)) return fail(HGCA_EINVAL, "attend_dense: scale must be > 0");
  if (!q || !out || !lse || (nkv > 0 && (!k || !v || !ws)) || (keep_weights && nkv > 0 && !weights))
    return fail(HGCA_EINVAL, "attend_dense: null pointer");
  AttendArgs a{};
  a.q = q; a.k = k; a.v = v;
  a.Hq = H; a.Hkv = H; a.G = 1;
  a.nq = nq; a.d = d; a.ld_head = nkv * d; a.ld_row = d; a.row0 = 0; a.n = nkv;
  a.scale = scale;
  a.out = out; a.lse = lse;
  a.wts = keep_weights ? weights : nullptr; a.wts_ld = nkv;
  a.ws = reinterpret_cast<double*>(ws); a.ws_ld = nkv;
  return cuda_status(launch_attend(dtype, a, H, S(stream)), "attend_dense");
}

int hgca_attend_indexed(int dtype, const void* q, const void* k, const void* v, const int64_t* idx,
                        int64_t n, int64_t M, int64_t nq, int64_t d, double scale, int keep_weights,
                        void* out, double* lse, void* weights, void* ws, hgca_stream_t stream) {
  if (dtype != HGCA_DTYPE_F32 && dtype != HGCA_DTYPE_F64)
    return fail(HGCA_EINVAL, "attend_indexed: dtype must be float32 or float64");
  if (n < 0 || M < 0 || nq < 0 || d < 1) return fail(HGCA_EINVAL, "attend_indexed: bad shape");
  if (!(scale > 0)) return fail(HGCA_EINVAL, "attend_indexed: scale must be > 0");
  if (!q || !out || !lse || (n > 0 && (!k || !v || !idx || !ws)) || (keep_weights && n > 0 && !weights))
    return fail(HGCA_EINVAL, "attend_indexed: null pointer");
  AttendArgs a{};
  a.q = q; a.k = k; a.v = v;
  a.Hq = 1; a.Hkv = 1; a.G = 1;
  a.nq = nq; a.d = d; a.ld_head = M * d; a.ld_row = d; a.row0 = 0; a.n = n;
  a.idx = idx;
  a.scale = scale;
  a.out = out; a.lse = lse;
  a.wts = keep_weights ? weights : nullptr; a.wts_ld = n;
  a.ws = reinterpret_cast<double*>(ws); a.ws_ld = n;
  return cuda_status(launch_attend(dtype, a, 1, S(stream)), "attend_indexed");
}

int hgca_attend_indexed_heads(int dtype, const void* q, const void* k, const void* v, int64_t H,
                              int64_t M, const int64_t* idx, const int64_t* idx_off,
                              const int64_t* idx_cnt, int64_t max_n, int64_t nq, int64_t d,
                              double scale, void* out, double* lse, void* weights, void* ws,
                              hgca_stream_t stream) {
  if (dtype != HGCA_DTYPE_F32 && dtype != HGCA_DTYPE_F64 && dtype != HGCA_DTYPE_BF16)
    return fail(HGCA_EINVAL, "attend_indexed_heads: bad dtype");
  if (H < 0 || M < 0 || nq < 0 || d < 1 || max_n < 0)
    return fail(HGCA_EINVAL, "attend_indexed_heads: bad shape");
  if (!q || !out || !lse || !idx_off || !idx_cnt || (max_n > 0 && (!k || !v || !idx || !ws)))
    return fail(HGCA_EINVAL, "attend_indexed_heads: null pointer");
  AttendArgs a{};
  a.q = q; a.k = k; a.v = v;
  a.Hq = H; a.Hkv = H; a.G = 1;
  a.nq = nq; a.d = d; a.ld_head = M * d; a.ld_row = d; a.row0 = 0; a.n = 0;
  a.idx = idx; a.idx_off = idx_off; a.idx_cnt = idx_cnt;
  a.scale = scale;
  a.out = out; a.lse = lse;
  a.wts = weights; a.wts_ld = max_n;
  a.ws = reinterpret_cast<double*>(ws); a.ws_ld = max_n > 0 ? max_n : 1;
  return cuda_status(launch_attend(dtype, a, H, S(stream)), "attend_indexed_heads");
}

int hgca_attend_gqa(int dtype, const void* q, const void* KV, int64_t B, int64_t Hq, int64_t Hkv, int64_t T,
                    int64_t row0, int64_t n, int64_t nq, int64_t d, double scale, void* out, double* lse,
                    void* weights, int64_t wts_ld, void* ws, hgca_stream_t stream) {
  if (B < 1 || Hq < 1 || Hkv < 1 || Hq % Hkv || d < 1 || n < 0 || row0 < 0 || row0 + n > T)
    return fail(HGCA_EINVAL, "attend_gqa: bad shape (B=%lld Hq=%lld Hkv=%lld row0=%lld n=%lld T=%lld)",
                (long long)B, (long long)Hq, (long long)Hkv, (long long)row0, (long long)n,
                (long long)T);
  if (weights && wts_ld < n) return fail(HGCA_EINVAL, "attend_gqa: wts_ld < n");
  AttendArgs a{};
  if (dtype != HGCA_DTYPE_F32 && dtype != HGCA_DTYPE_BF16)
    return fail(HGCA_EINVAL, "attend_gqa: storage dtype must be float32 or bfloat16");
  const int64_t esz = dtype == HGCA_DTYPE_BF16 ? 2 : 4;
  a.q = q; a.k = KV; a.v = reinterpret_cast<const unsigned char*>(KV) + d * esz;
  a.Hq = Hq; a.Hkv = Hkv; a.G = Hq / Hkv;
  a.nq = nq; a.d = d; a.ld_head = T * 2 * d; a.ld_row = 2 * d; a.row0 = row0; a.n = n;
  a.rot = 1;  // the engine stores K|V rows position-rotated (both storage dtypes)
  a.scale = scale;
  a.out = out; a.lse = lse;
  a.wts = weights; a.wts_ld = wts_ld;
  a.ws = reinterpret_cast<double*>(ws); a.ws_ld = n > 0 ? n : 1;
  return cuda_status(launch_attend(dtype, a, B * Hq, S(stream)), "attend_gqa");
}

int hgca_attend_gqa_indexed(int dtype, const void* q, const void* KV, int64_t B, int64_t Hq, int64_t Hkv,
                            int64_t T, const int64_t* idx, const int64_t* idx_off, const int64_t* idx_cnt,
                            int64_t max_n, int64_t nq, int64_t d, double scale, void* out, double* lse,
                            void* weights, void* ws, hgca_stream_t stream) {
  if (B < 1 || Hq < 1 || Hkv < 1 || Hq % Hkv || d < 1 || nq < 0 || max_n < 0 || max_n > T)
    return fail(HGCA_EINVAL, "attend_gqa_indexed: bad shape");
  if (dtype != HGCA_DTYPE_F32 && dtype != HGCA_DTYPE_BF16)
    return fail(HGCA_EINVAL, "attend_gqa_indexed: storage dtype must be float32 or bfloat16");
  if (!q || !KV || !out || !lse || !idx_off || !idx_cnt || (max_n > 0 && (!idx || !ws)))
    return fail(HGCA_EINVAL, "attend_gqa_indexed: null pointer");
  const int64_t esz = dtype == HGCA_DTYPE_BF16 ? 2 : 4;
  AttendArgs a{};
  a.q = q; a.k = KV; a.v = reinterpret_cast<const unsigned char*>(KV) + d * esz;
  a.Hq = Hq; a.Hkv = Hkv; a.G = Hq / Hkv;
  a.nq = nq; a.d = d; a.ld_head = T * 2 * d; a.ld_row = 2 * d; a.row0 = 0; a.n = 0;
  a.rot = 1;
  a.idx = idx; a.idx_off = idx_off; a.idx_cnt = idx_cnt;
  a.scale = scale;
  a.out = out; a.lse = lse;
  a.wts = weights; a.wts_ld = max_n;
  a.ws = reinterpret_cast<double*>(ws); a.ws_ld = max_n > 0 ? max_n : 1;
  return cuda_status(launch_attend(dtype, a, B * Hq, S(stream)), "attend_gqa_indexed");
}

int hgca_merge_states(int dtype, const void* out_a, const double* lse_a, const void* out_b,
                      const double* lse_b, int64_t rows, int64_t d, void* out, double* lse,
                      const void* w_a, const void* w_b, int64_t na, int64_t nb, void* w_out,
                      hgca_stream_t stream) {
  if (dtype != HGCA_DTYPE_F32 && dtype != HGCA_DTYPE_F64)
    return fail(HGCA_EINVAL, "merge_states: dtype must be float32 or float64");
  if (rows < 0 || d < 0 || na < 0 || nb < 0) return fail(HGCA_EINVAL, "merge_states: bad shape");
  if (w_out && ((na > 0 && !w_a) || (nb > 0 && !w_b)))
    return fail(HGCA_EINVAL, "merge_states: null weight rows");
  MergeArgs a{};
  a.out_a = out_a; a.lse_a = lse_a; a.out_b = out_b; a.lse_b = lse_b;
  a.rows = rows; a.d = d; a.out = out; a.lse = lse;
  a.w_a = w_a; a.w_b = w_b; a.na = na; a.nb = nb; a.w_out = w_out;  // w_a / w_b may be NULL only when na / nb == 0
  return cuda_status(launch_merge(dtype, a, S(stream)), "merge_states");
}

int hgca_merge_partials(const float* outs, const double* lses, int64_t P, int64_t rows, int64_t d,
                        float* out, double* lse, hgca_stream_t stream) {
  if (P < 1 || rows < 0 || d < 1) return fail(HGCA_EINVAL, "merge_partials: bad shape");
  if (rows == 0) return HGCA_OK;
  merge_partials_kernel<<<(unsigned)rows, 128, 0, S(stream)>>>(outs, lses, P, rows, d, out, lse);
  return cuda_status((int)cudaGetLastError(), "merge_partials");
}

int hgca_merge_packed(const void* parts, int64_t P, int64_t rows, int64_t d, int64_t stride_bytes, float* out,
                      double* lse, hgca_stream_t stream) {
  if (P < 1 || rows < 0 || d < 1 || stride_bytes < rows * d * 4 + rows * 8 || (rows * d * 4) % 8 ||
      stride_bytes % 8)
    return fail(HGCA_EINVAL, "merge_packed: bad shape");
  if (rows == 0) return HGCA_OK;
  merge_packed_kernel<<<(unsigned)rows, 128, 0, S(stream)>>>(reinterpret_cast<const unsigned char*>(parts), P,
                                                            rows, d, stride_bytes, out, lse, nullptr);
  return cuda_status((int)cudaGetLastError(), "merge_packed");
}

int hgca_peer_alloc(int64_t bytes, void** ptr, void* handle64) {
  if (bytes < 1 || !ptr || !handle64) return fail(HGCA_EINVAL, "peer_alloc: bad arguments");
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
  int rc = cuda_status((int)cudaMalloc(ptr, (size_t)bytes), "peer_alloc: cudaMalloc");
  if (rc) return rc;
  rc = cuda_status((int)cudaMemset(*ptr, 0, (size_t)bytes), "peer_alloc: memset");
  if (rc) return rc;
  // the zeroed boxes and flags must be in place before any rank's kernels (on
  // other, non-blocking streams -- or in other processes) write into them
  rc = cuda_status((int)cudaDeviceSynchronize(), "peer_alloc: sync");
  if (rc) return rc;
  cudaIpcMemHandle_t h;
  rc = cuda_status((int)cudaIpcGetMemHandle(&h, *ptr), "peer_alloc: cudaIpcGetMemHandle");
  if (rc) return rc;
  memcpy(handle64, &h, 64);
  return HGCA_OK;
}

int hgca_peer_open(const void* handle64, void** ptr) {
  if (!handle64 || !ptr) return fail(HGCA_EINVAL, "peer_open: bad arguments");
  cudaIpcMemHandle_t h;
  memcpy(&h, handle64, 64);
  return cuda_status((int)cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess), "peer_open");
}

int hgca_peer_close(void* ptr) { return cuda_status((int)cudaIpcCloseMemHandle(ptr), "peer_close"); }

int hgca_peer_free(void* ptr) { return cuda_status((int)cudaFree(ptr), "peer_free"); }

int hgca_merge_packed_wait(const void* parts, int64_t P, int64_t rows, int64_t d, int64_t stride_bytes,
                           const uint64_t* flags, uint64_t epoch, int64_t timeout_ms, int32_t* err, float* out,
                           double* lse, hgca_stream_t stream) {
  if (!flags || P < 1 || timeout_ms < 0) return fail(HGCA_EINVAL, "merge_packed_wait: bad arguments");
  wait_flags_kernel<<<1, 32, 0, S(stream)>>>(reinterpret_cast<const unsigned long long*>(flags), P,
                                             (unsigned long long)epoch, (long long)timeout_ms * 1000000LL, err);
  const int rc = cuda_status((int)cudaGetLastError(), "merge_packed_wait");
  if (rc) return rc;
  if (rows < 0 || d < 1 || stride_bytes < rows * d * 4 + rows * 8 || (rows * d * 4) % 8 || stride_bytes % 8)
    return fail(HGCA_EINVAL, "merge_packed_wait: bad shape");
  if (rows == 0) return HGCA_OK;
  // on a timeout the wait kernel raised *err: the merge then writes NaN instead of folding stale slots
  merge_packed_kernel<<<(unsigned)rows, 128, 0, S(stream)>>>(reinterpret_cast<const unsigned char*>(parts), P,
                                                            rows, d, stride_bytes, out, lse, err);
  return cuda_status((int)cudaGetLastError(), "merge_packed_wait");
}

int hgca_select_threshold(const double* maw, int64_t rows, int64_t ld, int64_t p0, int64_t p1,
                          double beta, int64_t divisor, uint32_t* mask, int64_t words, int assign,
                          const uint32_t* keep, hgca_stream_t stream) {
  if (divisor < 1) return fail(HGCA_EINVAL, "divisor must be >= 1, got %lld", (long long)divisor);
  if (p0 < 0 || p1 < p0 || p1 > ld || words * 32 < p1 || rows < 0)
    return fail(HGCA_EINVAL, "select_threshold: bad range");
  if (rows == 0 || p1 == p0) return HGCA_OK;
  const double thr = beta / (double)divisor;  // IEEE fp64, like beta / divisor in Python
  const int64_t nw = ((p1 + 31) >> 5) - (p0 >> 5);
  const int64_t total = nw * rows;
  (void)total;
  return cuda_status(launch_threshold_mask(maw, rows, ld, p0, p1, thr, mask, words, assign, keep, S(stream)),
                     "select_threshold");
}

int hgca_mask_to_indices(const uint32_t* mask_a, const uint32_t* mask_b, int64_t rows, int64_t words,
                         int64_t n, int64_t* idx, int64_t ld, uint8_t* flags, int64_t* counts,
                         hgca_stream_t stream) {
  if (rows < 0 || n < 0 || words * 32 < n || ld < n) return fail(HGCA_EINVAL, "mask_to_indices: bad shape");
  if (rows == 0) return HGCA_OK;
  return cuda_status(launch_mask_to_indices(mask_a, mask_b, rows, words, n, idx, ld, flags, counts, S(stream)),
                     "mask_to_indices");
}

int hgca_popcount_rows(const uint32_t* mask, int64_t rows, int64_t words, int64_t n, int64_t* counts,
                       hgca_stream_t stream) {
  if (rows < 0 || words * 32 < n) return fail(HGCA_EINVAL, "popcount_rows: bad shape");
  if (rows == 0) return HGCA_OK;
  return cuda_status(launch_popcount_rows(mask, rows, words, n, counts, S(stream)), "popcount_rows");
}

int hgca_group_need(const int64_t* counts, int64_t B, int64_t H, int64_t g, int64_t* need,
                    hgca_stream_t stream) {
  if (B < 0 || H < 0 || g < 1) return fail(HGCA_EINVAL, "group_need: bad shape");
  if (B * H == 0) return HGCA_OK;
  return cuda_status(launch_group_need(counts, B, H, g, need, S(stream)), "group_need");
}

int hgca_select_topk(const double* maw, int64_t rows, int64_t ld, int64_t n, const int64_t* k,
                     const uint32_t* exclude, uint32_t* out, int64_t words, hgca_stream_t stream) {
  if (rows < 0 || n < 0 || n > ld || words * 32 < n) return fail(HGCA_EINVAL, "select_topk: bad shape");
  if (rows == 0 || n == 0) return HGCA_OK;
  return cuda_status(launch_topk_mask(maw, rows, ld, n, k, exclude, out, words, S(stream)), "select_topk");
}

int hgca_write_rows(int dtype, void* KV, int64_t BH, int64_t T, int64_t d, int64_t pos, const void* k_new,
                    const void* v_new, int64_t n, hgca_stream_t stream) {
  if (pos < 0 || n < 0 || pos + n > T) return fail(HGCA_EINVAL, "write_rows: position range exceeds buffer");
  return cuda_status(launch_write_rows(dtype, KV, BH, T, d, pos, k_new, v_new, n, S(stream)), "write_rows");
}

int hgca_decode_chunk_rows(int dtype, int64_t d) { return decode_chunk_rows(dtype, d); }

#ifndef HGCA_BF16_ITEM_ROWS
#define HGCA_BF16_ITEM_ROWS 256  // longest bf16 work item (rows); the fp32 kernel's is 64
#endif
#ifndef HGCA_F32_ITEM_ROWS
#define HGCA_F32_ITEM_ROWS 64  // longest fp32 work item (rows)
#endif
static int64_t dense_rows_of(int dtype) { return dtype == HGCA_DTYPE_F32 ? HGCA_F32_ITEM_ROWS : HGCA_BF16_ITEM_ROWS; }
// the shortest work item (one 32-row pipeline stage): step-adaptive items
// (hgca_union_build_items with item_target > 0) never go below it, and the
// dense items follow the chosen sparse granularity
static constexpr int64_t kMinItemRows = 32;

int hgca_item_rows(int dtype, int64_t* out2) {
  if (!out2 || (dtype != HGCA_DTYPE_F32 && dtype != HGCA_DTYPE_BF16))
    return fail(HGCA_EINVAL, "item_rows: storage dtype must be float32 or bfloat16");
  out2[0] = kMinItemRows;         // shortest dense item (capacity of the partial buffers)
  out2[1] = dense_rows_of(dtype);  // longest item
  return HGCA_OK;
}

int hgca_decode_config(int dtype, int64_t d, int64_t group, int64_t* out5) {
  if (!out5 || decode_config(dtype, d, group, out5)) return fail(HGCA_EINVAL, "decode_config: unsupported");
  return HGCA_OK;
}

int hgca_maw_update(const float* w, int64_t BH, int64_t nq, int64_t W, int64_t w_ld, double* maw,
                    int64_t T, int64_t p0, int64_t w_old, double alpha, int mode, hgca_stream_t stream) {
  if (BH < 0 || nq < 1 || W < 0 || w_ld < W || p0 < 0 || p0 + W > T || (mode != 0 && mode != 1))
    return fail(HGCA_EINVAL, "maw_update: bad shape");
  if (!(alpha >= 0.0 && alpha <= 1.0)) return fail(HGCA_EINVAL, "alpha must be in [0, 1], got %g", alpha);
  return cuda_status(launch_maw_update(w, BH, nq, W, w_ld, maw, T, p0, w_old, alpha, mode, S(stream)),
                     "maw_update");
}

int hgca_maw_ema(double* maw, int64_t rows, int64_t ld, int64_t n, const double* a, int64_t lda, double alpha,
                 hgca_stream_t stream) {
  if (rows < 0 || n < 0 || ld < n || lda < n || (rows * n > 0 && (!maw || !a)))
    return fail(HGCA_EINVAL, "maw_ema: bad shape");
  if (!(alpha >= 0.0 && alpha <= 1.0)) return fail(HGCA_EINVAL, "alpha must be in [0, 1], got %g", alpha);
  return cuda_status(launch_maw_ema(maw, rows, ld, n, a, lda, alpha, S(stream)), "maw_ema");
}

int hgca_union_build_items_w(const uint32_t* sel_mask, int64_t B, int64_t Hq, int64_t Hkv, int64_t words,
                             int64_t n_arch, int64_t T, int32_t* u_ent, int32_t* u_cnt, int32_t* item_off,
                             int32_t* item_tab, int64_t max_rows, int64_t min_rows, int64_t item_target,
                             int64_t window_rows, int grouped, hgca_stream_t stream) {
  if (window_rows < 0 || window_rows > T) return fail(HGCA_EINVAL, "union_build: bad window_rows");
  if (B < 1 || Hkv < 1 || Hq % Hkv || Hq / Hkv > 8 || n_arch < 0 || n_arch > T || words * 32 < n_arch ||
      max_rows < 16 || max_rows % 16 || min_rows < 16 || min_rows % 16 || min_rows > max_rows || item_target < 0 ||
      T >= (1 << 24))
    return fail(HGCA_EINVAL, "union_build: bad shape");
  if (!item_tab || !u_ent || !u_cnt || !item_off) return fail(HGCA_EINVAL, "union_build: null output");
  return cuda_status(launch_union_build(sel_mask, B, Hq, Hkv, words, n_arch, T, u_ent, u_cnt, item_off,
                                        reinterpret_cast<int4*>(item_tab), max_rows, min_rows, item_target,
                                        window_rows, (grouped == 2 || grouped == 3) ? grouped : (grouped ? 1 : 0),
                                        S(stream)),
                     "union_build");
}

int hgca_union_build_items(const uint32_t* sel_mask, int64_t B, int64_t Hq, int64_t Hkv, int64_t words,
                           int64_t n_arch, int64_t T, int32_t* u_ent, int32_t* u_cnt, int32_t* item_off,
                           int32_t* item_tab, int64_t max_rows, int64_t min_rows, int64_t item_target, int grouped,
                           hgca_stream_t stream) {
  return hgca_union_build_items_w(sel_mask, B, Hq, Hkv, words, n_arch, T, u_ent, u_cnt, item_off, item_tab,
                                  max_rows, min_rows, item_target, 0, grouped, stream);
}

int hgca_union_build(const uint32_t* sel_mask, int64_t B, int64_t Hq, int64_t Hkv, int64_t words,
                     int64_t n_arch, int64_t T, int32_t* u_ent, int32_t* u_cnt, int32_t* item_off,
                     int32_t* item_tab, int64_t sparse_rows, int grouped, hgca_stream_t stream) {
  return hgca_union_build_items(sel_mask, B, Hq, Hkv, words, n_arch, T, u_ent, u_cnt, item_off, item_tab,
                                sparse_rows, sparse_rows, 0, grouped, stream);
}

static int decode_prepare(const hgca_decode_desc* d, DecodeArgs& a, DecodeMergeArgs& m) {
  if (!d) return fail(HGCA_EINVAL, "decode_step: null descriptor");
  if (d->dtype != HGCA_DTYPE_F32 && d->dtype != HGCA_DTYPE_BF16)
    return fail(HGCA_EINVAL, "decode_step: storage dtype must be float32 or bfloat16");
  if (d->B < 1 || d->Hkv < 1 || d->Hq % d->Hkv) return fail(HGCA_EINVAL, "decode_step: bad heads");
  const int64_t G = d->Hq / d->Hkv;
  if (G != 1 && G != 2 && G != 4 && G != 8) return fail(HGCA_EINVAL, "decode_step: Hq/Hkv must be 1, 2, 4 or 8");
  if (d->D != 64 && d->D != 128) return fail(HGCA_EINVAL, "decode_step: head_dim must be 64 or 128");
  if (d->T < 1 || d->T >= (1 << 24)) return fail(HGCA_EINVAL, "decode_step: T must be in [1, 2^24)");
  const int64_t W = d->dhi - d->dlo;
  if (d->dlo < 0 || W < 1 || d->dhi > d->T || d->w_old < 0 || d->w_old > W || d->dsc_ld < W)
    return fail(HGCA_EINVAL, "decode_step: bad dense range");
  // graph mode: the range comes from the device state at run time; size the
  // item capacity check for the largest window the scratch allows
  const int64_t Wcap = d->state ? d->dsc_ld : W;
  if (d->sparse_rows < 16 || d->sparse_rows % 16)
    return fail(HGCA_EINVAL, "decode_step: sparse_rows must be a positive multiple of 16");
  const int64_t DR = dense_rows_of(d->dtype);
  // dense items (window parts) per (batch, kv-head): as short as kMinItemRows when the union
  // rebuild chose short items (the kernels read the chosen size from item_off)
  const int64_t Sd = (Wcap + kMinItemRows - 1) / kMinItemRows;
  const int64_t n_dense = d->B * d->Hkv * Sd;
  // every item but the last full and last tail item of a list holds >= sparse_rows/4 rows; adaptive
  // items (hgca_union_build_items, rows >= union / item_target): <= 5/3 item_target + 5 per list
  if (d->item_target < 0) return fail(HGCA_EINVAL, "decode_step: item_target must be >= 0");
  const int64_t BKd = d->B * d->Hkv;
  const int64_t max_sparse = BKd * ((4 * d->T + d->sparse_rows - 1) / d->sparse_rows + 2) +
                             (d->item_target ? (5 * d->item_target + 2) / 3 + 5 * BKd : 0);
  if (d->max_items < n_dense + max_sparse)
    return fail(HGCA_EINVAL, "decode_step: partial buffers hold %lld items, need %lld",
                (long long)d->max_items, (long long)(n_dense + max_sparse));
  if (!d->KV || !d->q || !d->u_ent || !d->u_cnt || !d->item_off || !d->item_tab || !d->dsc || !d->part_m ||
      !d->part_z || !d->part_acc || !d->counter || !d->out || !d->lse)
    return fail(HGCA_EINVAL, "decode_step: null pointer");
  if (!(d->alpha >= 0.0 && d->alpha <= 1.0)) return fail(HGCA_EINVAL, "alpha must be in [0, 1], got %g", d->alpha);
  a = DecodeArgs{};
  if ((d->k_new == nullptr) != (d->v_new == nullptr)) return fail(HGCA_EINVAL, "decode_step: k_new and v_new go together");
  a.KV = d->KV; a.q = d->q;
  a.k_new = d->k_new; a.v_new = d->v_new;
  a.B = d->B; a.Hq = d->Hq; a.Hkv = d->Hkv; a.G = G; a.D = d->D; a.T = d->T;
  a.scale = d->scale;
  a.dlo = d->dlo; a.dhi = d->dhi;
  a.u_ent = d->u_ent; a.u_cnt = d->u_cnt; a.item_off = d->item_off;
  a.item_tab = reinterpret_cast<const int4*>(d->item_tab);
  a.sparse_rows = d->sparse_rows;
  a.dsc = d->dsc; a.dsc_ld = d->dsc_ld;
  a.part_m = d->part_m; a.part_z = d->part_z; a.part_acc = d->part_acc;
  a.counter = d->counter;
  a.n_dense_items = n_dense;
  a.Sd = Sd;
  a.dense_rows = DR;
  a.w_old = d->w_old;
  a.maw = d->maw;
  a.one_minus_alpha = 1.0 - d->alpha; a.alpha = d->alpha;
  a.wts_out = d->wts_out;
  a.state = d->state;
  m = DecodeMergeArgs{};
  m.B = d->B; m.Hq = d->Hq; m.Hkv = d->Hkv; m.G = G; m.D = d->D;
  m.n_dense_items = n_dense; m.item_off = d->item_off;
  m.part_m = d->part_m; m.part_z = d->part_z; m.part_acc = d->part_acc; m.MI = d->max_items;
  m.out = d->out; m.lse = d->lse;
  m.out_sparse = d->out_sparse; m.lse_sparse = d->lse_sparse;
  if (d->push_n < 0 || d->push_n > 8 || (d->push_n && !d->push_cnt))
    return fail(HGCA_EINVAL, "decode_step: push_n must be in [0, 8] with a push counter");
  m.push_n = d->push_n;
  m.push_sparse = d->push_sparse ? 1 : 0;
  for (int p = 0; p < d->push_n; ++p) {
    if (!d->push_dst[p] || !d->push_flag[p]) return fail(HGCA_EINVAL, "decode_step: null push slot %d", p);
    m.push_dst[p] = static_cast<unsigned char*>(d->push_dst[p]);
    m.push_flag[p] = reinterpret_cast<unsigned long long*>(d->push_flag[p]);
  }
  m.epoch = d->epoch;
  m.push_cnt = d->push_cnt;
  m.split = 1;
  if (d->merge_split > 1) {
    if (d->merge_split > 16 || !d->merge_scratch)
      return fail(HGCA_EINVAL, "decode_step: merge_split must be in [1, 16] with a merge_scratch");
    unsigned char* xs = static_cast<unsigned char*>(d->merge_scratch);
    const int64_t heads = d->B * d->Hq, cnt_b = (heads * 4 + 255) / 256 * 256;
    m.split = (int)d->merge_split;
    m.xcnt = reinterpret_cast<unsigned int*>(xs);
    m.xmz = reinterpret_cast<double*>(xs + cnt_b);
    m.xacc = reinterpret_cast<double*>(xs + cnt_b + heads * d->merge_split * 4 * 8);
  }
  return HGCA_OK;
}

int64_t hgca_append_ws_bytes(int64_t B, int64_t Hq, int64_t Hkv, int64_t D, int64_t nq, int64_t lo, int64_t hi) {
  if (B < 1 || lo < 0 || hi <= lo) return -1;
  return append_ws_bytes(B, Hq, Hkv, D, nq, lo, hi);
}

int hgca_append_bf16(const void* KV, int64_t B, int64_t Hq, int64_t Hkv, int64_t T, int64_t D, const void* q,
                     int64_t nq, double scale, int64_t lo, int64_t hi, float* out, double* lse, float* mean_archive,
                     float* mean_window, void* ws, int64_t ws_bytes, hgca_stream_t stream) {
  if (B < 1 || Hkv < 1 || Hq % Hkv || Hq / Hkv > 8 || (D != 64 && D != 128))
    return fail(HGCA_EINVAL, "append_bf16: bad heads / head_dim");
  if (nq < 1 || nq > 128) return fail(HGCA_EINVAL, "append_bf16: n_q must be in [1, 128], got %lld", (long long)nq);
  if (lo < 0 || hi <= lo || hi > T) return fail(HGCA_EINVAL, "append_bf16: bad position range");
  if (!KV || !q || !out || !lse || !ws) return fail(HGCA_EINVAL, "append_bf16: null pointer");
  const int64_t need = append_ws_bytes(B, Hq, Hkv, D, nq, lo, hi);
  if (need < 0 || ws_bytes < need)
    return fail(HGCA_EINVAL, "append_bf16: workspace holds %lld bytes, needs %lld", (long long)ws_bytes,
                (long long)need);
  return cuda_status(launch_append_bf16(KV, B, Hq, Hkv, T, D, q, nq, scale, lo, hi, out, lse, mean_archive,
                                        mean_window, ws, S(stream)),
                     "append_bf16");
}

// HGCA_HOST_PROF=1 (diagnostics): host time of the host-buffer step's parts,
// averaged and printed to stderr every 64 calls
namespace {
struct HostProf {
  bool on = getenv("HGCA_HOST_PROF") != nullptr;
  double t[5] = {0, 0, 0, 0, 0};
  long n = 0;
};
HostProf& host_prof() {
  static HostProf p;
  return p;
}
double now_us() {
  return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now().time_since_epoch()).count();
}
}  // namespace

static int decode_step_host_impl(const hgca_decode_desc* d, const void* in_host, void* in_dev, int64_t in_bytes,
                                 void* out_host, const void* out_dev, int64_t out_bytes, hgca_stream_t stream,
                                 bool sync) {
  HostProf& hp = host_prof();
  double tp0 = hp.on ? now_us() : 0.0, tp1 = 0, tp2 = 0, tp3 = 0;
  if (in_bytes < 0 || out_bytes < 0 || (in_bytes && (!in_host || !in_dev)) || (out_bytes && (!out_host || !out_dev)))
    return fail(HGCA_EINVAL, "decode_step_host: bad staging buffers");
  DecodeArgs a;
  DecodeMergeArgs m;
  int rc = decode_prepare(d, a, m);
  if (rc) return rc;
  a.m = m;
  cudaStream_t s = S(stream);
  if (hp.on) tp1 = now_us();
  if (in_bytes) {
    rc = cuda_status((int)cudaMemcpyAsync(in_dev, in_host, (size_t)in_bytes, cudaMemcpyHostToDevice, s),
                     "decode_step_host: H2D");
    if (rc) return rc;
  }
  if (hp.on) tp2 = now_us();
  // Results straight to the host: when out_host is pinned and mapped (UVA), the
  // merge kernel writes out / lse (which the descriptor places inside
  // out_dev) into their mirror locations in out_host over the bus, so no D2H
  // copy sits on the step's critical path. Otherwise: staged + copied.
  bool direct = false;
  if (out_bytes) {
    void* mapped = nullptr;
    const char* od = static_cast<const char*>(out_dev);
    const char* po = reinterpret_cast<const char*>(m.out);
    const char* pl = reinterpret_cast<const char*>(m.lse);
    const int64_t nb_out = m.B * m.Hq * m.D * 4, nb_lse = m.B * m.Hq * 8;
    const bool inside = po >= od && po + nb_out <= od + out_bytes && pl >= od && pl + nb_lse <= od + out_bytes;
    if (inside && cudaHostGetDevicePointer(&mapped, out_host, 0) == cudaSuccess && mapped) {
      a.m.out = reinterpret_cast<float*>(static_cast<char*>(mapped) + (po - od));
      a.m.lse = reinterpret_cast<double*>(static_cast<char*>(mapped) + (pl - od));
      direct = true;
    } else {
      (void)cudaGetLastError();  // not mapped: clear the lookup error, use the staged copy
    }
  }
  if (hp.on) tp3 = now_us();
  rc = cuda_status(launch_decode_partial(d->dtype, a, s), "decode_step_host");
  if (rc) return rc;
  if (hp.on) {
    const double tp4 = now_us();
    hp.t[0] += tp1 - tp0; hp.t[1] += tp2 - tp1; hp.t[2] += tp3 - tp2; hp.t[3] += tp4 - tp3;
    if (++hp.n % 64 == 0)
      fprintf(stderr, "[hgca host prof] us/call: prepare %.2f H2D-issue %.2f map %.2f launch(2 kernels) %.2f\n",
              hp.t[0] / hp.n, hp.t[1] / hp.n, hp.t[2] / hp.n, hp.t[3] / hp.n);
  }
  if (out_bytes && !direct) {
    rc = cuda_status((int)cudaMemcpyAsync(out_host, out_dev, (size_t)out_bytes, cudaMemcpyDeviceToHost, s),
                     "decode_step_host: D2H");
    if (rc) return rc;
  }
  return sync ? cuda_status((int)cudaStreamSynchronize(s), "decode_step_host: sync") : 0;
}

int hgca_decode_step_host(const hgca_decode_desc* d, const void* in_host, void* in_dev, int64_t in_bytes,
                          void* out_host, const void* out_dev, int64_t out_bytes, hgca_stream_t stream) {
  return decode_step_host_impl(d, in_host, in_dev, in_bytes, out_host, out_dev, out_bytes, stream, true);
}

int hgca_decode_step_host_async(const hgca_decode_desc* d, const void* in_host, void* in_dev, int64_t in_bytes,
                                void* out_host, const void* out_dev, int64_t out_bytes, hgca_stream_t stream) {
  return decode_step_host_impl(d, in_host, in_dev, in_bytes, out_host, out_dev, out_bytes, stream, false);
}

int64_t hgca_merge_scratch_bytes(int64_t B, int64_t Hq, int64_t D, int64_t split) {
  if (B < 1 || Hq < 1 || D < 1 || split < 1 || split > 16) return -1;
  const int64_t heads = B * Hq, cnt_b = (heads * 4 + 255) / 256 * 256;
  return cnt_b + heads * split * 4 * 8 + heads * split * 2 * D * 8;
}

int hgca_step_state_set(int64_t* state, int64_t dlo, int64_t dhi, uint64_t epoch, hgca_stream_t stream) {
  if (!state || dlo < 0 || dhi <= dlo) return fail(HGCA_EINVAL, "step_state_set: bad state or range");
  return cuda_status(launch_step_state_set(state, dlo, dhi, epoch, S(stream)), "step_state_set");
}

int hgca_decode_step(const hgca_decode_desc* d, hgca_stream_t stream) {
  DecodeArgs a;
  DecodeMergeArgs m;
  int rc = decode_prepare(d, a, m);
  if (rc) return rc;
  a.m = m;
  return cuda_status(launch_decode_partial(d->dtype, a, S(stream)), "decode_step");
}

}  // extern "C"
