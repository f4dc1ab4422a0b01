// K2: stable LSD radix sort of (global row, bag) pairs. The onesweep
// machinery is CUB's (CCCL 2.8, namespaced asb_cub), driven through our own
// policy hub (digit width, CTA size and items per thread are macros so the
// tuning can be A/B-ed with `make variant`). Measured on B200 at cfg2
// (36.5M pairs, 26-bit keys): CUB's default dispatch 1.21 ms; this hub with
// 8-bit digits, 384 threads x 23 items 0.86 ms; 9-bit digits (3 passes) 1.14 ms
// (the wider ranking costs more than the saved pass); 10-bit exceeds 48 KB smem.
#pragma once

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/dispatch/dispatch_radix_sort.cuh>

#ifndef ASB_SORT_BITS
#define ASB_SORT_BITS 8
#endif
#ifndef ASB_SORT_THREADS
#define ASB_SORT_THREADS 384
#endif
#ifndef ASB_SORT_ITEMS
#define ASB_SORT_ITEMS 23
#endif

namespace asb {

namespace cubns = CUB_NS_QUALIFIER;

template <int BITS, int THREADS, int ITEMS>
struct SortPolicyHub {
  using Base = typename cubns::detail::radix::policy_hub<unsigned, int, int>::Policy1000;
  struct Policy : cubns::ChainedPolicy<1000, Policy, Policy> {
    static constexpr bool ONESWEEP = true;
    static constexpr int ONESWEEP_RADIX_BITS = BITS;
    using HistogramPolicy = cubns::AgentRadixSortHistogramPolicy<128, 16, 1, unsigned, BITS>;
    using ExclusiveSumPolicy = cubns::AgentRadixSortExclusiveSumPolicy<256, BITS>;
    using OnesweepPolicy =
        cubns::AgentRadixSortOnesweepPolicy<THREADS, ITEMS, unsigned, 1, cubns::RADIX_RANK_MATCH_EARLY_COUNTS_ANY,
                                            cubns::BLOCK_SCAN_RAKING_MEMOIZE, cubns::RADIX_SORT_STORE_DIRECT, BITS>;
    // never run on sm_100 (onesweep path), required for instantiation
    using ScanPolicy = typename Base::ScanPolicy;
    using DownsweepPolicy = typename Base::DownsweepPolicy;
    using AltDownsweepPolicy = typename Base::AltDownsweepPolicy;
    using UpsweepPolicy = typename Base::UpsweepPolicy;
    using AltUpsweepPolicy = typename Base::AltUpsweepPolicy;
    using SingleTilePolicy = typename Base::SingleTilePolicy;
    using SegmentedPolicy = typename Base::SegmentedPolicy;
    using AltSegmentedPolicy = typename Base::AltSegmentedPolicy;
  };
  using MaxPolicy = Policy;
};

using SortDispatch = cubns::DispatchRadixSort<false, unsigned, int, int,
                                              SortPolicyHub<ASB_SORT_BITS, ASB_SORT_THREADS, ASB_SORT_ITEMS>>;

// keys_in/vals_in are left intact; the sorted pairs land in keys_out/vals_out.
inline cudaError_t sort_pairs(void* tmp, size_t& tmp_bytes, const unsigned* keys_in, unsigned* keys_out,
                              const int* vals_in, int* vals_out, int n, int end_bit, cudaStream_t s) {
  cubns::DoubleBuffer<unsigned> k(const_cast<unsigned*>(keys_in), keys_out);
  cubns::DoubleBuffer<int> v(const_cast<int*>(vals_in), vals_out);
  return SortDispatch::Dispatch(tmp, tmp_bytes, k, v, n, 0, end_bit, false, s);
}

constexpr int sort_passes(int end_bit) { return (end_bit + ASB_SORT_BITS - 1) / ASB_SORT_BITS; }

}  // namespace asb
