// Drop-in use of the B200 path from C++ through include/suco_b200.hpp, the way
// the reference CLI drives its own library: `suco build` (suco_cli.cpp:199-221)
// then `suco query` (suco_cli.cpp:238-251 -> run_suco_batch, suco_cli.cpp:95-114).
//
//   gpu_batch <n> <d> <base.f32> <nq> <queries.f32> <alpha> <beta> <k> <out.bin>
//
// Raw little-endian float32 row-major inputs. Writes nq*k u32 ids then nq*k
// f64 distances to out.bin, plus the serialized index to out.bin.suco, and
// prints one JSON line. The GPU tests run it against the C oracle.
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <iostream>
#include <vector>

#include "suco_b200.hpp"

static std::vector<float> read_f32(const char* path, std::size_t count) {
    std::vector<float> v(count);
    std::ifstream f(path, std::ios::binary);
    if (!f.read(reinterpret_cast<char*>(v.data()), static_cast<std::streamsize>(count * sizeof(float)))) {
        throw std::runtime_error(std::string("cannot read ") + path);
    }
    return v;
}

int main(int argc, char** argv) {
    if (argc != 10) {
        std::fprintf(stderr, "usage: %s n d base.f32 nq queries.f32 alpha beta k out.bin\n", argv[0]);
        return 2;
    }
    try {
        const std::uint64_t n = std::strtoull(argv[1], nullptr, 10);
        const std::uint32_t d = static_cast<std::uint32_t>(std::strtoul(argv[2], nullptr, 10));
        const std::uint64_t nq = std::strtoull(argv[4], nullptr, 10);
        const std::vector<float> base = read_f32(argv[3], n * d);
        const std::vector<float> queries = read_f32(argv[5], nq * d);
        const suco::gpu::CollisionParams cp{std::strtod(argv[6], nullptr), std::strtod(argv[7], nullptr),
                                            static_cast<std::uint32_t>(std::strtoul(argv[8], nullptr, 10))};

        // suco::build_index(data, params) -> suco::gpu::build_index(rows, n, d, params)
        const auto t0 = std::chrono::steady_clock::now();
        suco::gpu::GpuIndex index = suco::gpu::build_index(base, n, d, suco::gpu::IndexParams{4, 16, 3, 42});
        const auto t1 = std::chrono::steady_clock::now();
        // save_index/load_index round trip: identical bytes, identical answers
        const std::vector<unsigned char> bytes = suco::gpu::serialize_index(index);
        suco::gpu::GpuIndex loaded = suco::gpu::load_index(bytes, base, n, d);
        // run_suco_batch(index, base, queries, params) -> one batched call
        const std::vector<suco::gpu::QueryResult> results = loaded.knn_query_batch(queries, nq, cp);
        const auto t2 = std::chrono::steady_clock::now();
        // per-query form (suco::knn_query) agrees with the batch
        for (std::uint64_t q = 0; q < std::min<std::uint64_t>(nq, 4); ++q) {
            const auto one = suco::gpu::knn_query(index, std::span<const float>(queries.data() + q * d, d), cp);
            for (std::uint32_t i = 0; i < cp.k; ++i) {
                if (one.entries[i].id != results[q].entries[i].id ||
                    one.entries[i].distance != results[q].entries[i].distance) {
                    std::fprintf(stderr, "batch/single mismatch at query %llu\n", static_cast<unsigned long long>(q));
                    return 1;
                }
            }
        }
        std::ofstream out(argv[9], std::ios::binary);
        for (const auto& r : results)
            for (const auto& e : r.entries) out.write(reinterpret_cast<const char*>(&e.id), 4);
        for (const auto& r : results)
            for (const auto& e : r.entries) out.write(reinterpret_cast<const char*>(&e.distance), 8);
        std::ofstream(std::string(argv[9]) + ".suco", std::ios::binary)
            .write(reinterpret_cast<const char*>(bytes.data()), static_cast<std::streamsize>(bytes.size()));
        std::cout << "{\"n\": " << n << ", \"queries\": " << nq << ", \"index_bytes\": " << bytes.size()
                  << ", \"build_s\": " << std::chrono::duration<double>(t1 - t0).count()
                  << ", \"query_s\": " << std::chrono::duration<double>(t2 - t1).count() << "}\n";
        return 0;
    } catch (const suco::gpu::ConfigError& e) {  // exit codes of suco_cli.cpp:695-706
        std::cerr << "configuration error: " << e.what() << "\n";
        return 2;
    } catch (const suco::gpu::FormatError& e) {
        std::cerr << "format error: " << e.what() << "\n";
        return 3;
    } catch (const suco::gpu::IncompatibilityError& e) {
        std::cerr << "incompatibility: " << e.what() << "\n";
        return 4;
    } catch (const std::exception& e) {
        std::cerr << "error: " << e.what() << "\n";
        return 1;
    }
}
