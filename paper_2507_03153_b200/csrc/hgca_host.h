// Host-side launch state shared by the launchers: per-device "attribute set"
// flags and a thread-safe cache of encoded TMA tensor maps. Both are keyed by
// the current device, so one process may drive engines on several GPUs, and
// the map cache holds one entry per (device, buffer, geometry) -- a
// multi-layer engine encodes each layer's map once, not once per switch.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>

#include <atomic>
#include <mutex>

namespace hgca {

inline int current_device() {
  int dev = 0;
  cudaGetDevice(&dev);
  return dev;
}

// SM count of the current device, cached per ordinal (< 64).
inline int sm_count() {
  static std::atomic<int> cache[64];
  const int dev = current_device() & 63;
  int n = cache[dev].load(std::memory_order_relaxed);
  if (n <= 0) {
    n = 148;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    cache[dev].store(n, std::memory_order_relaxed);
  }
  return n;
}

// One bit per device ordinal (< 64): set once the kernel's attribute is set there.
struct DevFlags {
  std::atomic<uint64_t> bits{0};
};

template <typename K>
inline int set_smem_dev(K kernel, int bytes, DevFlags& f) {
  const int dev = current_device();
  const uint64_t bit = 1ull << (dev & 63);
  if (f.bits.load(std::memory_order_acquire) & bit) return 0;
  const cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e != cudaSuccess) return (int)e;
  f.bits.fetch_or(bit, std::memory_order_release);
  return 0;
}

struct MapKey {
  int dev, kind;
  const void* base;
  int64_t rows, cols, box0, box1;
  bool operator==(const MapKey& o) const { return memcmp(this, &o, sizeof(MapKey)) == 0; }
};

// Encoded tensor maps keyed by MapKey; `encode(CUtensorMap*)` runs on a miss.
// 512 entries, round-robin replacement, one mutex (lookups are a few hundred ns).
class MapCache {
 public:
  template <typename Enc>
  int get(const MapKey& k, CUtensorMap* out, Enc encode) {
    std::lock_guard<std::mutex> lock(mu_);
    if (last_ < n_ && keys_[last_] == k) {  // the common case: the same layer again
      *out = maps_[last_];
      return 0;
    }
    for (int i = 0; i < n_; ++i)
      if (keys_[i] == k) {
        *out = maps_[i];
        last_ = i;
        return 0;
      }
    CUtensorMap m;
    const int rc = encode(&m);
    if (rc) return rc;
    const int slot = n_ < kCap ? n_++ : (next_++ % kCap);
    last_ = slot;
    keys_[slot] = k;
    maps_[slot] = m;
    *out = m;
    return 0;
  }

 private:
  static constexpr int kCap = 512;
  std::mutex mu_;
  MapKey keys_[kCap];
  CUtensorMap maps_[kCap];
  int n_ = 0, next_ = 0, last_ = 0;
};

inline MapKey map_key(int kind, const void* base, int64_t rows, int64_t cols, int64_t box0, int64_t box1) {
  MapKey k;
  memset(&k, 0, sizeof(k));
  k.dev = current_device();
  k.kind = kind;
  k.base = base;
  k.rows = rows;
  k.cols = cols;
  k.box0 = box0;
  k.box1 = box1;
  return k;
}

MapCache& map_cache();  // one per process (hgca_decode.cu)

}  // namespace hgca
