// mh/layout.hpp -- Morton-hybrid geometry (reference: layout.hpp:42-99).
// n = 2^m * t; tiles numbered along the Z curve, row-major inside a tile.
// The codec calls the library's host planner (mhg_encode / mhg_extract).
#pragma once

#include <cstdint>

#include "mh/abi.hpp"

namespace mh {

using Index = std::uint64_t;

namespace detail {

/// Bit k of x moved to bit 2k (x < 2^32): the tile Z-index is
/// dilate(tile row) << 1 | dilate(tile column) (reference: layout.hpp:15-33).  Spread by
/// halving strides with the usual magic masks; undilate gathers the even bits back.
constexpr std::uint64_t dilate(std::uint64_t x) {
    constexpr std::uint64_t mask[5] = {0x0000ffff0000ffffull, 0x00ff00ff00ff00ffull, 0x0f0f0f0f0f0f0f0full,
                                       0x3333333333333333ull, 0x5555555555555555ull};
    x &= 0xffffffffull;
    for (int s = 0; s < 5; ++s) x = (x | (x << (16 >> s))) & mask[s];
    return x;
}

constexpr std::uint64_t undilate(std::uint64_t x) {
    constexpr std::uint64_t mask[5] = {0x3333333333333333ull, 0x0f0f0f0f0f0f0f0full, 0x00ff00ff00ff00ffull,
                                       0x0000ffff0000ffffull, 0x00000000ffffffffull};
    x &= 0x5555555555555555ull;
    for (int s = 0; s < 5; ++s) x = (x | (x >> (1 << s))) & mask[s];
    return x;
}

static_assert(dilate(0b1011) == 0b1000101 && undilate(0b1000101) == 0b1011, "bit dilation");
static_assert(dilate(0xffffffffull) == 0x5555555555555555ull, "bit dilation, 32 bits");
static_assert(undilate(dilate(0x9e3779b9ull)) == 0x9e3779b9ull, "dilation round trip");
static_assert(undilate(0xffffffffffffffffull) == 0xffffffffull, "odd bits are ignored");

}  // namespace detail

struct Layout {
    std::uint64_t n = 1;
    std::uint64_t t = 1;
    unsigned grid_log2 = 0;
    std::uint64_t tile = 1;
    std::uint64_t total = 1;

    Layout() = default;
    Layout(std::uint64_t side, std::uint64_t tile_side) : n(side), t(tile_side) {
        gpu::check(mhg_layout_check(side, tile_side));  // invalid_argument
        for (std::uint64_t g = side / tile_side; g > 1; g >>= 1) ++grid_log2;
        tile = t * t;
        total = n * n;
    }

    std::uint64_t tdiv(std::uint64_t v) const { return v / t; }
    std::uint64_t tmod(std::uint64_t v) const { return v % t; }
    std::uint64_t tilediv(std::uint64_t v) const { return v / tile; }
    std::uint64_t tilemod(std::uint64_t v) const { return v % tile; }
};

inline Index encode(const Layout& lay, std::uint64_t i, std::uint64_t j) {
    Index z = 0;
    gpu::check(mhg_encode(lay.n, lay.t, i, j, &z));  // out_of_range outside the matrix
    return z;
}

inline std::uint64_t extract_i(const Layout& lay, Index z) {
    std::uint64_t i = 0, j = 0;
    gpu::check(mhg_extract(lay.n, lay.t, z, &i, &j));
    return i;
}

inline std::uint64_t extract_j(const Layout& lay, Index z) {
    std::uint64_t i = 0, j = 0;
    gpu::check(mhg_extract(lay.n, lay.t, z, &i, &j));
    return j;
}

}  // namespace mh
