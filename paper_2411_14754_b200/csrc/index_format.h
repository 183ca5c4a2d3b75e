// Host-side index model and the `.suco` byte format (README.md:138-146,
// index.hpp:87-98): little-endian magic "SUCO", version u32 = 1, header
// (n u64, d u32, N_s u32, k_half u32, iterations u32, seed u64, mode u32),
// per-subspace dimension lists, then per subspace: first-half centroids f32,
// second-half centroids f32, IMI offsets u64 (k_half^2 + 1), IMI ids u32 (n).
#pragma once

#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/suco_b200.h"

namespace suco_gpu {

struct Status {
    int code;
    std::string msg;
};

[[noreturn]] inline void raise(int code, std::string msg) { throw Status{code, std::move(msg)}; }

struct HostLayout {
    uint32_t d = 0, ns = 0;
    std::vector<uint32_t> dims;   // concatenated, subspace order
    std::vector<uint32_t> sizes;  // ns
    std::vector<uint32_t> split;  // ns: first-half count = size / 2
    uint32_t start(uint32_t s) const {
        uint32_t p = 0;
        for (uint32_t i = 0; i < s; ++i) p += sizes[i];
        return p;
    }
    uint32_t h1(uint32_t s) const { return split[s]; }
    uint32_t h2(uint32_t s) const { return sizes[s] - split[s]; }
};

// sample_subspaces (subspace.cpp:10-44); throws CONFIG like the reference.
HostLayout sample_subspaces(uint32_t d, uint32_t ns, uint32_t mode, uint64_t seed);

struct HostIndex {
    uint64_t n = 0;
    uint32_t d = 0;
    suco_index_params p{};
    HostLayout layout;
    std::vector<std::vector<float>> cent1, cent2;      // ns
    std::vector<std::vector<uint64_t>> offsets;        // ns x (K+1)
    std::vector<std::vector<uint32_t>> ids;            // ns x n
};

// deserialize_index (index.cpp:191-293), CorruptIndexError -> SUCO_ERR_FORMAT.
HostIndex parse_index(const unsigned char* bytes, uint64_t len);
// serialize_index (index.cpp:147-170).
std::vector<unsigned char> serialize(const HostIndex& x);

// rng.hpp helpers used by the host side of the build (seeding only).
uint64_t splitmix64(uint64_t x);
uint64_t derive_seed(uint64_t seed, uint64_t stream);

struct Mt64 {  // std::mt19937_64
    uint64_t mt[312];
    int idx;
    explicit Mt64(uint64_t seed);
    uint64_t next();
    uint64_t uniform_below(uint64_t bound);
    double uniform_unit();
};

}  // namespace suco_gpu
