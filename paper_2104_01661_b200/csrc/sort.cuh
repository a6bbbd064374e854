// sort.cuh -- CUB radix sorts with the item count narrowed to 32 bits when it
// fits: the 64-bit-offset instantiation measured ~1.9x slower on B200 (65 M
// (key, value) pairs, 22-bit keys: 3.43 vs 1.83 ms, the PageRank plan's sort),
// and the double-buffer form (no internal alternate arrays).
#pragma once

#include <cub/cub.cuh>

#include <climits>

#include "common.cuh"

namespace gbx {

template <typename K, typename V>
inline void radix_sort_pairs(cudaStream_t s, cub::DoubleBuffer<K>& k, cub::DoubleBuffer<V>& v,
                             int64_t m, int begin_bit, int end_bit) {
  if (m <= 0) return;
  size_t tb = 0;
  if (m < INT_MAX) {
    const int mi = static_cast<int>(m);
    GBX_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, k, v, mi, begin_bit, end_bit, s));
    Tmp<uint8_t> t(tb, s);
    GBX_CUDA(cub::DeviceRadixSort::SortPairs(t.p, tb, k, v, mi, begin_bit, end_bit, s));
  } else {
    GBX_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, k, v, m, begin_bit, end_bit, s));
    Tmp<uint8_t> t(tb, s);
    GBX_CUDA(cub::DeviceRadixSort::SortPairs(t.p, tb, k, v, m, begin_bit, end_bit, s));
  }
}

template <typename K>
inline void radix_sort_keys(cudaStream_t s, cub::DoubleBuffer<K>& k, int64_t m, int begin_bit,
                            int end_bit) {
  if (m <= 0) return;
  size_t tb = 0;
  if (m < INT_MAX) {
    const int mi = static_cast<int>(m);
    GBX_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tb, k, mi, begin_bit, end_bit, s));
    Tmp<uint8_t> t(tb, s);
    GBX_CUDA(cub::DeviceRadixSort::SortKeys(t.p, tb, k, mi, begin_bit, end_bit, s));
  } else {
    GBX_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tb, k, m, begin_bit, end_bit, s));
    Tmp<uint8_t> t(tb, s);
    GBX_CUDA(cub::DeviceRadixSort::SortKeys(t.p, tb, k, m, begin_bit, end_bit, s));
  }
}

// separate input / output arrays (the inputs are left untouched)
template <typename K, typename V>
inline void radix_sort_pairs(cudaStream_t s, const K* kin, K* kout, const V* vin, V* vout,
                             int64_t m, int begin_bit, int end_bit) {
  if (m <= 0) return;
  size_t tb = 0;
  if (m < INT_MAX) {
    const int mi = static_cast<int>(m);
    GBX_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, kin, kout, vin, vout, mi, begin_bit,
                                             end_bit, s));
    Tmp<uint8_t> t(tb, s);
    GBX_CUDA(cub::DeviceRadixSort::SortPairs(t.p, tb, kin, kout, vin, vout, mi, begin_bit,
                                             end_bit, s));
  } else {
    GBX_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, kin, kout, vin, vout, m, begin_bit,
                                             end_bit, s));
    Tmp<uint8_t> t(tb, s);
    GBX_CUDA(cub::DeviceRadixSort::SortPairs(t.p, tb, kin, kout, vin, vout, m, begin_bit,
                                             end_bit, s));
  }
}

}  // namespace gbx
