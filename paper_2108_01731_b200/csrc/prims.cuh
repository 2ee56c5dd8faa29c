// prims.cuh -- thin stream-ordered wrappers over CUB device primitives
// (scan / select / radix sort / run-length).  Used for the bookkeeping
// around the hand-written kernels; temp storage comes from the pool.
#pragma once
#include <cub/cub.cuh>

#include "common.cuh"

namespace lcc {

template <class InIt, class OutIt, class Pred>
inline void select_if(InIt in, OutIt out, int64_t* d_count, int64_t n, Pred pred, cudaStream_t s) {
    size_t bytes = 0;
    LCC_CUDA(cub::DeviceSelect::If(nullptr, bytes, in, out, d_count, n, pred, s));
    Buf<unsigned char> tmp(bytes, s);
    LCC_CUDA(cub::DeviceSelect::If(tmp.get(), bytes, in, out, d_count, n, pred, s));
}

template <class InIt, class FlagIt, class OutIt>
inline void select_flagged(InIt in, FlagIt flags, OutIt out, int64_t* d_count, int64_t n,
                           cudaStream_t s) {
    size_t bytes = 0;
    LCC_CUDA(cub::DeviceSelect::Flagged(nullptr, bytes, in, flags, out, d_count, n, s));
    Buf<unsigned char> tmp(bytes, s);
    LCC_CUDA(cub::DeviceSelect::Flagged(tmp.get(), bytes, in, flags, out, d_count, n, s));
}

template <class InIt, class OutIt>
inline void exclusive_sum(InIt in, OutIt out, int64_t n, cudaStream_t s) {
    size_t bytes = 0;
    LCC_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, in, out, n, s));
    Buf<unsigned char> tmp(bytes, s);
    LCC_CUDA(cub::DeviceScan::ExclusiveSum(tmp.get(), bytes, in, out, n, s));
}

template <class InIt, class OutIt>
inline void inclusive_sum(InIt in, OutIt out, int64_t n, cudaStream_t s) {
    size_t bytes = 0;
    LCC_CUDA(cub::DeviceScan::InclusiveSum(nullptr, bytes, in, out, n, s));
    Buf<unsigned char> tmp(bytes, s);
    LCC_CUDA(cub::DeviceScan::InclusiveSum(tmp.get(), bytes, in, out, n, s));
}

template <class InIt, class OutT>
inline void device_sum(InIt in, OutT* out, int64_t n, cudaStream_t s) {
    size_t bytes = 0;
    LCC_CUDA(cub::DeviceReduce::Sum(nullptr, bytes, in, out, n, s));
    Buf<unsigned char> tmp(bytes, s);
    LCC_CUDA(cub::DeviceReduce::Sum(tmp.get(), bytes, in, out, n, s));
}

// Stable LSD radix sort of 64-bit keys restricted to bits [0, end_bit).
inline void sort_keys(uint64_t* keys_in, uint64_t* keys_out, int64_t n, int end_bit,
                      cudaStream_t s) {
    size_t bytes = 0;
    LCC_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, bytes, keys_in, keys_out, n, 0, end_bit, s));
    Buf<unsigned char> tmp(bytes, s);
    LCC_CUDA(cub::DeviceRadixSort::SortKeys(tmp.get(), bytes, keys_in, keys_out, n, 0, end_bit, s));
}

// Double-buffered variants: no n-sized temp copy (peak = the two buffers);
// the sorted run is in db.Current() afterwards.
inline void sort_keys_db(cub::DoubleBuffer<uint64_t>& db, int64_t n, int end_bit, cudaStream_t s) {
    size_t bytes = 0;
    LCC_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, bytes, db, n, 0, end_bit, s));
    Buf<unsigned char> tmp(bytes, s);
    LCC_CUDA(cub::DeviceRadixSort::SortKeys(tmp.get(), bytes, db, n, 0, end_bit, s));
}

template <class V>
inline void sort_pairs_db(cub::DoubleBuffer<uint64_t>& dk, cub::DoubleBuffer<V>& dv, int64_t n, int end_bit,
                          cudaStream_t s) {
    size_t bytes = 0;
    LCC_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, dk, dv, n, 0, end_bit, s));
    Buf<unsigned char> tmp(bytes, s);
    LCC_CUDA(cub::DeviceRadixSort::SortPairs(tmp.get(), bytes, dk, dv, n, 0, end_bit, s));
}

template <class V>
inline void sort_pairs(uint64_t* keys_in, uint64_t* keys_out, V* vals_in, V* vals_out, int64_t n,
                       int end_bit, cudaStream_t s) {
    size_t bytes = 0;
    LCC_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, keys_in, keys_out, vals_in, vals_out,
                                             n, 0, end_bit, s));
    Buf<unsigned char> tmp(bytes, s);
    LCC_CUDA(cub::DeviceRadixSort::SortPairs(tmp.get(), bytes, keys_in, keys_out, vals_in,
                                             vals_out, n, 0, end_bit, s));
}

inline int bit_width(uint64_t x) {
    int b = 0;
    while (x) { ++b; x >>= 1; }
    return b;
}

}  // namespace lcc
