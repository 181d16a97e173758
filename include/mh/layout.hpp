// mh/layout.hpp -- Morton-hybrid geometry (reference: layout.hpp:42-99).
// n = 2^m * t; tiles numbered along the Z curve, row-major inside a tile.
// The codec calls the library's host planner (mhg_encode / mhg_extract).
#pragma once

#include <cstdint>

#include "mh/abi.hpp"

namespace mh {

using Index = std::uint64_t;

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
