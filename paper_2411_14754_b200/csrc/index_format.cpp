// Host-side layout sampling, seeding helpers and the `.suco` byte format.
// This is host logic of the boundary (validation + persistence), not the
// compute path: it parses/produces exactly the reference's bytes so a GPU
// index round-trips with reference-built files.
#include "index_format.h"

#include <cmath>
#include <cstring>
#include <numeric>

namespace suco_gpu {

uint64_t splitmix64(uint64_t x) {  // rng.hpp:14-19
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}

uint64_t derive_seed(uint64_t seed, uint64_t stream) { return splitmix64(seed ^ splitmix64(stream)); }

Mt64::Mt64(uint64_t seed) {
    mt[0] = seed;
    for (int i = 1; i < 312; ++i) mt[i] = 6364136223846793005ULL * (mt[i - 1] ^ (mt[i - 1] >> 62)) + uint64_t(i);
    idx = 312;
}

uint64_t Mt64::next() {
    if (idx >= 312) {
        for (int i = 0; i < 312; ++i) {
            const uint64_t x = (mt[i] & 0xFFFFFFFF80000000ULL) | (mt[(i + 1) % 312] & 0x7FFFFFFFULL);
            uint64_t xa = x >> 1;
            if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
            mt[i] = mt[(i + 156) % 312] ^ xa;
        }
        idx = 0;
    }
    uint64_t x = mt[idx++];
    x ^= (x >> 29) & 0x5555555555555555ULL;
    x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
    x ^= (x << 37) & 0xFFF7EEE000000000ULL;
    return x ^ (x >> 43);
}

uint64_t Mt64::uniform_below(uint64_t bound) {  // rng.hpp:27-33
    const uint64_t threshold = (0 - bound) % bound;
    for (;;) {
        const uint64_t r = next();
        if (r >= threshold) return r % bound;
    }
}

double Mt64::uniform_unit() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }  // rng.hpp:36-38

HostLayout sample_subspaces(uint32_t d, uint32_t ns, uint32_t mode, uint64_t seed) {
    if (ns < 2) raise(SUCO_ERR_CONFIG, "sample_subspaces: need at least 2 subspaces, got " + std::to_string(ns));
    const uint32_t s = d / ns;
    if (s < 2) {
        raise(SUCO_ERR_CONFIG, "sample_subspaces: floor(d/num_subspaces) = " + std::to_string(s) +
                                   " leaves a subspace half empty (d=" + std::to_string(d) +
                                   ", num_subspaces=" + std::to_string(ns) + ")");
    }
    HostLayout L;
    L.d = d;
    L.ns = ns;
    L.dims.resize(d);
    std::iota(L.dims.begin(), L.dims.end(), 0u);
    if (mode == 1) {  // deterministic_shuffle, rng.hpp:50-56
        Mt64 g(seed);
        for (uint64_t i = d; i > 1; --i) std::swap(L.dims[i - 1], L.dims[g.uniform_below(i)]);
    }
    L.sizes.resize(ns);
    L.split.resize(ns);
    for (uint32_t i = 0; i < ns; ++i) {
        const uint32_t b = s * i, e = (i + 1 == ns) ? d : s * (i + 1);
        L.sizes[i] = e - b;
        L.split[i] = (e - b) / 2;
    }
    return L;
}

namespace {

struct Reader {
    const unsigned char* p;
    uint64_t len, pos = 0;
    void need(uint64_t c, const char* section) {
        if (len - pos < c) {
            raise(SUCO_ERR_CORRUPT_INDEX, std::string("index file truncated in section '") + section + "' at byte offset " +
                                       std::to_string(pos));
        }
    }
    uint32_t u32(const char* section) {
        need(4, section);
        const uint32_t v = uint32_t(p[pos]) | (uint32_t(p[pos + 1]) << 8) | (uint32_t(p[pos + 2]) << 16) |
                           (uint32_t(p[pos + 3]) << 24);
        pos += 4;
        return v;
    }
    uint64_t u64(const char* section) {
        const uint64_t lo = u32(section);
        return lo | (uint64_t(u32(section)) << 32);
    }
};

[[noreturn]] void corrupt(const std::string& section, const std::string& detail) {
    raise(SUCO_ERR_CORRUPT_INDEX, "index section '" + section + "': " + detail);
}

struct Writer {
    std::vector<unsigned char> b;
    void u32(uint32_t v) {
        for (int i = 0; i < 4; ++i) b.push_back(static_cast<unsigned char>(v >> (8 * i)));
    }
    void u64(uint64_t v) {
        u32(static_cast<uint32_t>(v));
        u32(static_cast<uint32_t>(v >> 32));
    }
};

}  // namespace

HostIndex parse_index(const unsigned char* bytes, uint64_t len) {
    Reader r{bytes, len};
    r.need(4, "magic");
    if (std::memcmp(bytes, "SUCO", 4) != 0) corrupt("magic", "bad magic bytes");
    r.pos = 4;
    const uint32_t version = r.u32("version");
    if (version != 1) corrupt("version", "unsupported format version " + std::to_string(version));
    HostIndex x;
    x.n = r.u64("header");
    const uint32_t d = r.u32("header");
    const uint32_t ns = r.u32("header");
    x.p.num_subspaces = ns;
    x.p.k_half = r.u32("header");
    x.p.iterations = r.u32("header");
    x.p.seed = r.u64("header");
    const uint32_t mode = r.u32("header");
    if (x.n < 1) corrupt("header", "n must be >= 1");
    if (x.n > 0xFFFFFFFFULL) corrupt("header", "n exceeds 32-bit point-id capacity");
    if (d < 1) corrupt("header", "d must be >= 1");
    if (ns < 2) corrupt("header", "subspace count must be >= 2");
    if (x.p.k_half < 1) corrupt("header", "k_half must be >= 1");
    if (x.p.iterations < 1) corrupt("header", "iterations must be >= 1");
    if (x.n < x.p.k_half) corrupt("header", "n smaller than k_half");
    if (mode > 1) corrupt("header", "unknown subspace mode " + std::to_string(mode));
    x.p.mode = mode;
    x.d = d;
    HostLayout& L = x.layout;
    L.d = d;
    L.ns = ns;
    L.sizes.resize(ns);
    L.split.resize(ns);
    std::vector<bool> seen(d, false);
    for (uint32_t s = 0; s < ns; ++s) {
        const uint32_t count = r.u32("layout");
        if (count < 2) corrupt("layout", "subspace " + std::to_string(s) + " has < 2 dimensions");
        L.sizes[s] = count;
        L.split[s] = count / 2;
        for (uint32_t j = 0; j < count; ++j) {
            const uint32_t dim = r.u32("layout");
            if (dim >= d) corrupt("layout", "dimension index " + std::to_string(dim) + " >= d");
            if (seen[dim]) corrupt("layout", "dimension " + std::to_string(dim) + " repeated");
            seen[dim] = true;
            L.dims.push_back(dim);
        }
    }
    for (uint32_t dim = 0; dim < d; ++dim) {
        if (!seen[dim]) corrupt("layout", "dimension " + std::to_string(dim) + " missing");
    }
    const uint32_t k = x.p.k_half;
    const uint64_t cells = uint64_t(k) * k;
    x.cent1.resize(ns);
    x.cent2.resize(ns);
    x.offsets.resize(ns);
    x.ids.resize(ns);
    std::vector<bool> id_seen;
    for (uint32_t s = 0; s < ns; ++s) {
        for (int half = 0; half < 2; ++half) {
            auto& c = half == 0 ? x.cent1[s] : x.cent2[s];
            c.resize(size_t(k) * (half == 0 ? L.h1(s) : L.h2(s)));
            for (float& v : c) {
                const uint32_t u = r.u32("centroids");
                std::memcpy(&v, &u, 4);
                if (!std::isfinite(v)) corrupt("centroids", "non-finite centroid value");
            }
        }
        auto& off = x.offsets[s];
        off.resize(cells + 1);
        for (uint64_t c = 0; c <= cells; ++c) {
            off[c] = r.u64("imi offsets");
            if (c == 0 && off[0] != 0) corrupt("imi offsets", "first offset must be 0");
            if (c > 0 && off[c] < off[c - 1]) corrupt("imi offsets", "offsets decrease at cell " + std::to_string(c - 1));
        }
        if (off[cells] != x.n) corrupt("imi offsets", "offsets do not cover n points");
        auto& ids = x.ids[s];
        ids.resize(x.n);
        id_seen.assign(x.n, false);
        for (uint64_t i = 0; i < x.n; ++i) {
            const uint32_t id = r.u32("imi ids");
            if (id >= x.n) corrupt("imi ids", "point id " + std::to_string(id) + " >= n");
            if (id_seen[id]) corrupt("imi ids", "point id " + std::to_string(id) + " repeated");
            id_seen[id] = true;
            ids[i] = id;
        }
    }
    if (r.pos != len) corrupt("trailer", std::to_string(len - r.pos) + " trailing bytes");
    return x;
}

std::vector<unsigned char> serialize(const HostIndex& x) {
    Writer w;
    const uint32_t ns = x.layout.ns;
    const uint64_t cells = uint64_t(x.p.k_half) * x.p.k_half;
    uint64_t total = 48 + 4ull * (ns + x.d);
    for (uint32_t s = 0; s < ns; ++s) {
        total += 4 * (x.cent1[s].size() + x.cent2[s].size()) + 8 * (cells + 1) + 4 * x.n;
    }
    w.b.reserve(total);
    for (char c : {'S', 'U', 'C', 'O'}) w.b.push_back(static_cast<unsigned char>(c));
    w.u32(1);
    w.u64(x.n);
    w.u32(x.d);
    w.u32(x.p.num_subspaces);
    w.u32(x.p.k_half);
    w.u32(x.p.iterations);
    w.u64(x.p.seed);
    w.u32(x.p.mode);
    uint32_t pos = 0;
    for (uint32_t s = 0; s < ns; ++s) {
        w.u32(x.layout.sizes[s]);
        for (uint32_t j = 0; j < x.layout.sizes[s]; ++j) w.u32(x.layout.dims[pos + j]);
        pos += x.layout.sizes[s];
    }
    for (uint32_t s = 0; s < ns; ++s) {
        for (const float v : x.cent1[s]) {
            uint32_t u;
            std::memcpy(&u, &v, 4);
            w.u32(u);
        }
        for (const float v : x.cent2[s]) {
            uint32_t u;
            std::memcpy(&u, &v, 4);
            w.u32(u);
        }
        for (const uint64_t o : x.offsets[s]) w.u64(o);
        for (const uint32_t id : x.ids[s]) w.u32(id);
    }
    return w.b;
}

}  // namespace suco_gpu
