// Internal argument blocks and launchers (not part of the C ABI).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace hgca {

// Generic reference-exact attention (attend / attend_indexed / append path).
struct AttendArgs {
  const void* q;        // [BH, nq, d]
  const void* k;        // kv rows for head bh at k + kvh*ld_head + row0*d
  const void* v;
  int64_t Hq, Hkv, G;   // bh = b*Hq + h; kvh = b*Hkv + h/G
  int64_t nq, d;
  int64_t ld_head;      // elements between consecutive kv heads
  int64_t ld_row;       // elements between consecutive kv rows (d, or 2d for interleaved K|V rows)
  int rot;              // 1: rows are the engine's position-rotated bf16 K|V pairs (see write_rows_kernel)
  int64_t row0;         // first row (dense) / base for idx
  int64_t n;            // dense key count (when idx == nullptr and idx_cnt == nullptr)
  const int64_t* idx;      // optional gathered rows (concatenated per head)
  const int64_t* idx_off;  // optional per-head offsets into idx
  const int64_t* idx_cnt;  // optional per-head counts
  double scale;
  void* out;            // [BH, nq, d]
  double* lse;          // [BH, nq]
  void* wts;            // optional [BH, nq, wts_ld]
  int64_t wts_ld;
  double* ws;           // scores workspace [BH, nq, ws_ld]
  int64_t ws_ld;
};

struct MergeArgs {
  const void* out_a;
  const double* lse_a;
  const void* out_b;
  const double* lse_b;
  int64_t rows, d;
  void* out;
  double* lse;
  const void* w_a;  // optional weight rows [rows, na] / [rows, nb]
  const void* w_b;
  int64_t na, nb;
  void* w_out;      // [rows, na + nb]
};

struct DecodeMergeArgs {
  int64_t B, Hq, Hkv, G, D;
  int64_t n_dense_items;  // = B*Hkv*Sd dense items (window parts), ids first
  const int32_t* item_off;
  const double* part_m;   // [G, MI] head-major item partials
  const double* part_z;   // [G, MI]
  const float* part_acc;  // [G, MI, D]
  int64_t MI;             // item stride of the partials (descriptor max_items)
  float* out;             // [B*Hq, D]
  double* lse;            // [B*Hq]
  float* out_sparse;      // optional sparse partial out [B*Hq, D] (for sharded merges)
  double* lse_sparse;
  // one-shot exchange: this rank's packed partial pushed into push_n slots
  int push_n, push_sparse;
  unsigned char* push_dst[8];
  unsigned long long* push_flag[8];
  unsigned long long epoch;
  unsigned int* push_cnt;
  // split merge (long item lists): `split` CTAs per query head each fold a
  // contiguous share of the sparse items (the last also the dense ones) into a
  // partial in the scratch; the last to arrive combines them in split order
  int split;
  unsigned int* xcnt;     // [B*Hq] arrival counters (0 between steps)
  double* xmz;            // [B*Hq, split, 4]: m_s, z_s, m_d, z_d
  double* xacc;           // [B*Hq, split, 2, D]: acc_s, acc_d
};

// Fused decode step: dense window items + sparse union chunks, merged in-kernel.
struct DecodeArgs {
  DecodeMergeArgs m;      // fold / merge_states parameters (decode_merge_kernel)
  CUtensorMap kmap;       // row map over KV [B*Hkv*T rows, 2D] for TMA gather4, set by the launcher
  const void* KV;         // [B*Hkv, T, 2, D] storage dtype: K row then V row per position
  const void* q;          // [B*Hq, D] storage dtype (decode: one query row)
  const void* k_new;      // optional [B*Hkv, D] kv_in rows written at position dhi-1 by the kernel
  const void* v_new;
  int64_t B, Hq, Hkv, G, D, T;
  double scale;
  int64_t dlo, dhi;       // dense positions [dlo, dhi)
  const int32_t* u_ent;   // [B*Hkv, T] union entries pos | (query-head mask << 24)
  const int32_t* u_cnt;   // [B*Hkv]
  const int32_t* item_off;// [B*Hkv + 1] sparse item prefix
  const int4* item_tab;   // [sparse items] (bk, lo, hi, 0)
  int64_t sparse_rows;    // rows per sparse item
  void* dsc;              // [B*Hq, dsc_ld] dense scores (fp64 for fp32 storage, fp32 for bf16)
  int64_t dsc_ld;
  double* part_m;         // [G, m.MI] head-major: one head's items are contiguous
  double* part_z;         // [G, m.MI]
  float* part_acc;        // [G, m.MI, D]
  int32_t* counter;       // work counter (0 on entry; re-armed by the merge kernel)
  int64_t n_dense_items;  // B*Hkv*Sd
  int64_t Sd;             // dense items (window parts of dense_rows rows) per (batch, kv-head)
  int64_t dense_rows;     // window rows per dense item (hgca_item_rows)
  // merge-kernel epilogue: window weights + MAW maintenance
  int64_t w_old;          // window entries before this step (EMA'd); the rest are new
  double* maw;            // [B*Hq, T] or nullptr (no MAW maintenance)
  double one_minus_alpha, alpha;
  float* wts_out;         // optional dense weights [B*Hq, dhi - dlo]
  // graph mode (optional): device step state {dlo, dhi, epoch, arrivals};
  // when set the kernels take the window range from it (dlo/dhi/w_old above
  // are ignored) and the merge kernel advances dhi and epoch after the step
  int64_t* state;
};



int launch_attend(int dtype, const AttendArgs& a, int64_t BH, cudaStream_t s);
int launch_merge(int dtype, const MergeArgs& a, cudaStream_t s);
int launch_threshold_mask(const double* maw, int64_t rows, int64_t ld, int64_t p0, int64_t p1,
                          double thr, uint32_t* mask, int64_t words, int assign, const uint32_t* keep,
                          cudaStream_t s);
int launch_mask_to_indices(const uint32_t* a, const uint32_t* b, int64_t rows, int64_t words,
                           int64_t n, int64_t* idx, int64_t ld, uint8_t* flags, int64_t* counts,
                           cudaStream_t s);
int launch_popcount_rows(const uint32_t* mask, int64_t rows, int64_t words, int64_t n,
                         int64_t* counts, cudaStream_t s);
int launch_group_need(const int64_t* counts, int64_t B, int64_t H, int64_t g, int64_t* need,
                      cudaStream_t s);
int launch_topk_mask(const double* maw, int64_t rows, int64_t ld, int64_t n, const int64_t* k,
                     const uint32_t* exclude, uint32_t* out, int64_t words, cudaStream_t s);

int launch_decode_partial(int dtype, const DecodeArgs& a, cudaStream_t s);
int launch_union_build(const uint32_t* sel, int64_t B, int64_t Hq, int64_t Hkv, int64_t words,
                       int64_t n_arch, int64_t T, int32_t* u_ent, int32_t* u_cnt, int32_t* item_off,
                       int4* item_tab, int64_t sparse_rows, int64_t min_rows, int64_t target, int64_t window_rows,
                       int grouped, cudaStream_t s);
int launch_write_rows(int dtype, void* KV, int64_t BH, int64_t T, int64_t D, int64_t pos,
                      const void* k_new, const void* v_new, int64_t n, cudaStream_t s);
int decode_chunk_rows(int dtype, int64_t D);
int launch_step_state_set(int64_t* state, int64_t dlo, int64_t dhi, uint64_t epoch, cudaStream_t s);
int64_t append_ws_bytes(int64_t B, int64_t Hq, int64_t Hkv, int64_t D, int64_t nq, int64_t lo, int64_t hi);
int launch_append_bf16(const void* KV, int64_t B, int64_t Hq, int64_t Hkv, int64_t T, int64_t D, const void* q,
                       int64_t nq, double scale, int64_t lo, int64_t hi, float* out, double* lse, float* mean_archive,
                       float* mean_window, void* ws, cudaStream_t s);
int decode_config(int dtype, int64_t D, int64_t G, int64_t* out);
int launch_maw_ema(double* maw, int64_t rows, int64_t ld, int64_t n, const double* a, int64_t lda, double alpha,
                   cudaStream_t s);
int launch_maw_update(const float* w, int64_t BH, int64_t nq, int64_t W, int64_t w_ld, double* maw,
                      int64_t T, int64_t p0, int64_t w_old, double alpha, int mode, cudaStream_t s);

}  // namespace hgca
