// C-ABI, vecs I/O (io.cpp:99-210) and device upload straight from vecs files.
#include <cuda_runtime.h>
#include <stdint.h>

#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "capi_internal.h"

using namespace suco_gpu;

// ------------------------------------------------------------------ vecs I/O (io.cpp:99-210)
// Record framing shared by fvecs / bvecs / ivecs: [dim i32 LE][dim elements]. Parsed in order
// with the reference's checks and messages (io.cpp:46-85, 99-137), so the first error wins
// exactly as there. Rows stream through two pinned staging buffers straight into device memory.
namespace {

constexpr int32_t kVecsMaxDim = 1 << 20;
constexpr double kVecsMaxExactInt = 16777216.0;  // 2^24

size_t vecs_elem(int kind) { return kind == 1 ? 1 : 4; }

uint32_t le32(const unsigned char* p) {
    return uint32_t(p[0]) | (uint32_t(p[1]) << 8) | (uint32_t(p[2]) << 16) | (uint32_t(p[3]) << 24);
}

struct VecsFile {
    FILE* f = nullptr;
    uint64_t size = 0;
    ~VecsFile() {
        if (f) std::fclose(f);
    }
};

void vecs_open(VecsFile& vf, const std::string& path) {
    vf.f = std::fopen(path.c_str(), "rb");
    if (!vf.f) raise(SUCO_ERR_FORMAT, "cannot open file: " + path);
    std::fseek(vf.f, 0, SEEK_END);
    vf.size = static_cast<uint64_t>(std::ftell(vf.f));
    std::fseek(vf.f, 0, SEEK_SET);
    if (vf.size == 0) raise(SUCO_ERR_FORMAT, "empty file: " + path);
}

// Streams records [0, limit) through `sink(first_record, count, float rows)`; returns n, sets d.
template <typename Sink>
uint64_t vecs_stream(const std::string& path, int kind, uint64_t limit, uint32_t& d, float* stage_a, float* stage_b,
                     uint64_t stage_rows, Sink&& sink) {
    VecsFile vf;
    vecs_open(vf, path);
    const size_t es = vecs_elem(kind);
    std::vector<unsigned char> buf;
    uint64_t pos = 0, record = 0;
    d = 0;
    float* stage[2] = {stage_a, stage_b};
    int which = 0;
    uint64_t in_stage = 0, stage_first = 0;
    while (pos < vf.size && record < limit) {
        unsigned char hdr[4];
        if (vf.size - pos < 4) {
            raise(SUCO_ERR_FORMAT, path + ": truncated record header at byte offset " + std::to_string(pos) +
                                       " (record " + std::to_string(record) + ")");
        }
        if (std::fread(hdr, 1, 4, vf.f) != 4) raise(SUCO_ERR_FORMAT, "failed reading file: " + path);
        const int32_t dim = static_cast<int32_t>(le32(hdr));
        if (dim <= 0 || dim > kVecsMaxDim) {
            raise(SUCO_ERR_FORMAT, path + ": record " + std::to_string(record) + " declares invalid dimension " +
                                       std::to_string(dim));
        }
        if (record == 0) {
            d = static_cast<uint32_t>(dim);
            buf.resize(size_t(d) * es);
        } else if (static_cast<uint32_t>(dim) != d) {
            raise(SUCO_ERR_FORMAT, path + ": record " + std::to_string(record) + " has dimension " +
                                       std::to_string(dim) + ", expected " + std::to_string(d));
        }
        pos += 4;
        const uint64_t body = uint64_t(dim) * es;
        if (vf.size - pos < body) {
            raise(SUCO_ERR_FORMAT, path + ": truncated record body at byte offset " + std::to_string(pos) +
                                       " (record " + std::to_string(record) + ")");
        }
        if (std::fread(buf.data(), 1, body, vf.f) != body) raise(SUCO_ERR_FORMAT, "failed reading file: " + path);
        float* row = stage[which] + in_stage * d;
        for (uint32_t j = 0; j < d; ++j) {
            float v = 0.f;
            if (kind == 0) {
                const uint32_t bits = le32(buf.data() + 4 * size_t(j));
                std::memcpy(&v, &bits, 4);
                if (!std::isfinite(v)) {
                    raise(SUCO_ERR_FORMAT, path + ": non-finite value in record " + std::to_string(record));
                }
            } else if (kind == 1) {
                v = static_cast<float>(buf[j]);
            } else {
                const int32_t iv = static_cast<int32_t>(le32(buf.data() + 4 * size_t(j)));
                if (iv > int32_t(kVecsMaxExactInt) || iv < -int32_t(kVecsMaxExactInt)) {
                    raise(SUCO_ERR_FORMAT, path + ": record " + std::to_string(record) + " holds " +
                                               std::to_string(iv) + ", too large to load into floats exactly");
                }
                v = static_cast<float>(iv);
            }
            row[j] = v;
        }
        pos += body;
        ++record;
        if (++in_stage == stage_rows) {
            sink(stage_first, in_stage, stage[which], which);
            which ^= 1;
            stage_first = record;
            in_stage = 0;
        }
    }
    if (record == 0) raise(SUCO_ERR_FORMAT, path + ": no records within the read limit");
    if (in_stage) sink(stage_first, in_stage, stage[which], which);
    return record;
}

// Upper bound on the records of a vecs file (for the device allocation): every record has the
// first record's dim. Exact unless the file is malformed (then the parse raises anyway).
uint64_t vecs_bound(const std::string& path, int kind, uint64_t limit, uint32_t* dim) {
    VecsFile vf;
    vecs_open(vf, path);
    unsigned char hdr[4];
    if (vf.size < 4 || std::fread(hdr, 1, 4, vf.f) != 4) {
        raise(SUCO_ERR_FORMAT, path + ": truncated record header at byte offset 0 (record 0)");
    }
    const int32_t d0 = static_cast<int32_t>(le32(hdr));
    if (d0 <= 0 || d0 > kVecsMaxDim) {
        raise(SUCO_ERR_FORMAT, path + ": record 0 declares invalid dimension " + std::to_string(d0));
    }
    *dim = static_cast<uint32_t>(d0);
    const uint64_t stride = 4 + uint64_t(d0) * vecs_elem(kind);
    const uint64_t n = (vf.size + stride - 1) / stride;
    return std::min(n, limit);
}

void check_kind(int kind) {
    if (kind < 0 || kind > 2) raise(SUCO_ERR_CONTRACT, "vecs kind must be 0 (fvecs), 1 (bvecs) or 2 (ivecs)");
}

// Streams a vecs file into x->data (n x d f32 on the device).
void stream_vecs_into(suco_gpu_index* x, const std::string& path, int kind, uint64_t limit, uint64_t* n_out,
                      uint32_t* d_out) {
    uint32_t d0 = 0;
    const uint64_t nmax = vecs_bound(path, kind, limit, &d0);
    x->data.reserve(nmax * d0);
    const uint64_t rows = std::max<uint64_t>(1, (32ull << 20) / (uint64_t(d0) * 4));  // 32 MB stages
    float* pin[2] = {nullptr, nullptr};
    cudaEvent_t done[2] = {nullptr, nullptr};
    try {
        for (int i = 0; i < 2; ++i) {
            CUDA_TRY(cudaMallocHost(&pin[i], rows * d0 * 4));
            CUDA_TRY(cudaEventCreateWithFlags(&done[i], cudaEventDisableTiming));
            CUDA_TRY(cudaEventRecord(done[i], x->own));
        }
        uint32_t d = 0;
        // a stage is refilled only after its previous copy finished (event), so parsing the next
        // chunk overlaps the copy of the last one
        auto wait_stage = [&](int w) { CUDA_TRY(cudaEventSynchronize(done[w])); };
        wait_stage(0);
        const uint64_t n = vecs_stream(path, kind, limit, d, pin[0], pin[1], rows,
                                       [&](uint64_t first, uint64_t cnt, const float* rowsp, int w) {
            CUDA_TRY(cudaMemcpyAsync(x->data.p + first * d, rowsp, cnt * d * 4, cudaMemcpyHostToDevice, x->own));
            CUDA_TRY(cudaEventRecord(done[w], x->own));
            wait_stage(w ^ 1);
        });
        CUDA_TRY(cudaStreamSynchronize(x->own));
        *n_out = n;
        *d_out = d;
    } catch (...) {
        for (int i = 0; i < 2; ++i) {
            if (pin[i]) cudaFreeHost(pin[i]);
            if (done[i]) cudaEventDestroy(done[i]);
        }
        throw;
    }
    for (int i = 0; i < 2; ++i) {
        cudaFreeHost(pin[i]);
        cudaEventDestroy(done[i]);
    }
}

}  // namespace

int suco_read_vecs(const char* path, int kind, uint64_t limit, float* out, uint64_t cap_rows, uint64_t* n,
                   uint32_t* d) {
    return guarded([&] {
        if (!path || !n || !d) raise(SUCO_ERR_CONTRACT, "null argument");
        check_kind(kind);
        if (!out) {  // size query: parse the framing, keep nothing
            uint32_t dd = 0;
            const uint64_t rows = 4096;
            std::vector<float> a, b;
            uint32_t d0 = 0;
            vecs_bound(path, kind, limit, &d0);
            a.resize(rows * d0);
            b.resize(rows * d0);
            *n = vecs_stream(path, kind, limit, dd, a.data(), b.data(), rows, [](uint64_t, uint64_t, const float*, int) {});
            *d = dd;
            return;
        }
        uint32_t d0 = 0;
        vecs_bound(path, kind, limit, &d0);
        const uint64_t rows = 4096;
        std::vector<float> a(rows * d0), b(rows * d0);
        uint32_t dd = 0;
        *n = vecs_stream(path, kind, limit, dd, a.data(), b.data(), rows,
                         [&](uint64_t first, uint64_t cnt, const float* rowsp, int) {
            if (first + cnt > cap_rows) raise(SUCO_ERR_CONTRACT, "output buffer holds fewer rows than the file");
            std::memcpy(out + first * dd, rowsp, cnt * dd * 4);
        });
        *d = dd;
    });
}

int suco_write_vecs(const char* path, int kind, uint64_t n, uint32_t d, const float* values) {
    return guarded([&] {
        if (!path || !values) raise(SUCO_ERR_CONTRACT, "null argument");
        check_kind(kind);
        if (n < 1 || d < 1) raise(SUCO_ERR_CONTRACT, "write_vecs: n and d must be >= 1");
        std::vector<unsigned char> rec(4 + size_t(d) * vecs_elem(kind));
        rec[0] = static_cast<unsigned char>(d);
        rec[1] = static_cast<unsigned char>(d >> 8);
        rec[2] = static_cast<unsigned char>(d >> 16);
        rec[3] = static_cast<unsigned char>(d >> 24);
        for (uint64_t i = 0; i < n * d; ++i) {  // validate before touching the file (io.cpp:139-160)
            const float v = values[i];
            if (kind == 1 && !(v == std::trunc(v) && v >= 0.f && v <= 255.f)) {
                raise(SUCO_ERR_CONTRACT, "write_vecs: bvecs values must be integers in [0, 255]");
            }
            if (kind == 2 && !(v == std::trunc(v) && std::fabs(v) <= kVecsMaxExactInt)) {
                raise(SUCO_ERR_CONTRACT, "write_vecs: ivecs values must be integers with |v| <= 2^24");
            }
        }
        FILE* f = std::fopen(path, "wb");
        if (!f) raise(SUCO_ERR_INTERNAL, std::string("cannot open file for writing: ") + path);
        bool ok = true;
        for (uint64_t r = 0; r < n && ok; ++r) {
            for (uint32_t j = 0; j < d; ++j) {
                const float v = values[r * d + j];
                if (kind == 0) {
                    std::memcpy(rec.data() + 4 + 4 * size_t(j), &v, 4);
                } else if (kind == 1) {
                    rec[4 + j] = static_cast<unsigned char>(v);
                } else {
                    const int32_t iv = static_cast<int32_t>(v);
                    std::memcpy(rec.data() + 4 + 4 * size_t(j), &iv, 4);
                }
            }
            ok = std::fwrite(rec.data(), 1, rec.size(), f) == rec.size();
        }
        ok = (std::fclose(f) == 0) && ok;
        if (!ok) raise(SUCO_ERR_INTERNAL, std::string("failed writing file: ") + path);
    });
}

int suco_gpu_build_index_from_vecs(const char* path, int kind, uint64_t limit, const suco_index_params* params,
                                   int device, suco_gpu_index** out) {
    return guarded([&] {
        if (!out || !path) raise(SUCO_ERR_CONTRACT, "null argument");
        *out = nullptr;
        if (!params) raise(SUCO_ERR_CONTRACT, "index params are null");
        check_kind(kind);
        DeviceGuard g(device);
        suco_gpu_index* x = new_index_on(device);
        try {
            uint64_t n = 0;
            uint32_t d = 0;
            stream_vecs_into(x, path, kind, limit, &n, &d);
            upload_data(x, nullptr, n, d);
            build_core(x, n, d, params);
        } catch (...) {
            delete x;
            throw;
        }
        *out = x;
    });
}

int suco_gpu_load_index_from_vecs(const unsigned char* bytes, uint64_t len, const char* path, int kind, uint64_t limit,
                                  int device, suco_gpu_index** out) {
    return guarded([&] {
        if (!out || !path) raise(SUCO_ERR_CONTRACT, "null argument");
        *out = nullptr;
        HostIndex h = parse_index(bytes, len);  // FORMAT first, like load_index + read_vecs in suco_cli.cpp:241-244
        check_kind(kind);
        DeviceGuard g(device);
        suco_gpu_index* x = new_index_on(device);
        try {
            uint64_t n = 0;
            uint32_t d = 0;
            stream_vecs_into(x, path, kind, limit, &n, &d);
            if (h.n != n) {
                raise(SUCO_ERR_INCOMPATIBLE, "index was built from n = " + std::to_string(h.n) +
                                                 " points but dataset has n = " + std::to_string(n));
            }
            if (h.d != d) {
                raise(SUCO_ERR_INCOMPATIBLE, "index was built for d = " + std::to_string(h.d) +
                                                 " but dataset has d = " + std::to_string(d));
            }
            x->host = std::move(h);
            upload_data(x, nullptr, n, d);
            load_core(x, n);
        } catch (...) {
            delete x;
            throw;
        }
        *out = x;
    });
}
