// mh/field.hpp -- prime field GF(q), q < 2^31 (reference: field.hpp:23-55).
// Host-side scalar helpers; bulk arithmetic runs in the GPU epilogue.
#pragma once

#include <cstdint>

#include "mh/abi.hpp"

namespace mh {

/// Prime modulus 2 <= q < 2^31 with the Barrett constant floor((2^64-1)/q).
struct Modulus {
    std::uint32_t q = 2;
    std::uint64_t mu = std::uint64_t(1) << 63;

    Modulus() = default;
    explicit Modulus(std::uint32_t prime) : q(prime) {
        gpu::check(mhg_modulus_check(prime));  // invalid_argument on range / primality
        mu = prime == 2 ? (std::uint64_t(1) << 63) : ~std::uint64_t(0) / prime;
    }
};

/// Canonical residue in [0, q).
struct Fp {
    std::uint32_t v = 0;
    friend bool operator==(Fp a, Fp b) { return a.v == b.v; }
    friend bool operator!=(Fp a, Fp b) { return a.v != b.v; }
};

inline Fp add(Fp a, Fp b, const Modulus& m) {
    const std::uint32_t s = a.v + b.v;
    return Fp{s >= m.q ? s - m.q : s};
}

inline Fp mul(Fp a, Fp b, const Modulus& m) {
    return Fp{std::uint32_t((std::uint64_t(a.v) * b.v) % m.q)};
}

}  // namespace mh
