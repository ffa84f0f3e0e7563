// Fixed log-spaced latency bins shared by the DES (producer) and the summary select (consumer).
//
// The DES adds every measurement-window latency to a per-(replica, tenant) histogram as it emits
// it (one fire-and-forget RED per completion, fused into the producer).  Bins are the top 18 bits
// of the order-preserving key of the FP64 value -- sign, exponent and 6 mantissa bits, i.e. 64
// bins per binary octave -- offset so bin 0 starts at 2^-10 ms; values below clamp into bin 0,
// values at or above 2^22 ms into the last bin.  Bins are monotone in the value, so the select
// kernel knows from the histogram alone which bins hold the nearest-rank targets and finishes with
// ONE streaming pass over the samples (engine.cpp:800-816 ranks, exact).
#pragma once

#include <stdint.h>

#include "glibc_math.h"

namespace mg {

constexpr int kHistBins = 2048;
constexpr int kHistShift = 46;
// okey(2^-10) >> kHistShift: positive doubles map to bits | 2^63
constexpr uint64_t kHistBase = ((1ull << 63) | (static_cast<uint64_t>(1023 - 10) << 52)) >> kHistShift;

MG_HD uint64_t lat_key(double x) {
    uint64_t b;
    std::memcpy(&b, &x, 8);
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
MG_HD uint32_t lat_bin_of_key(uint64_t key) {
    const uint64_t v = key >> kHistShift;
    if (v < kHistBase) return 0;
    const uint64_t d = v - kHistBase;
    return d >= static_cast<uint64_t>(kHistBins) ? static_cast<uint32_t>(kHistBins - 1) : static_cast<uint32_t>(d);
}
MG_HD uint32_t lat_bin(double x) { return lat_bin_of_key(lat_key(x)); }
// [lo, lo + 2^kHistShift) is exactly the key range of an interior bin (0 < b < kHistBins - 1)
MG_HD uint64_t lat_bin_lo(uint32_t b) { return (kHistBase + b) << kHistShift; }

}  // namespace mg
