// SPDX-License-Identifier: Apache-2.0
//
// On-disk POD files of the ember graph store (edges_<split>.bin,
// bucket_offsets.bin, node_part_<k>.bin = rows x d theta then rows x d Adagrad state,
// relations.bin). Source-compatible with the reference's proj/include/ember/binary_io.h (same
// function names, element types and error behaviour: IoError on open / size / short-IO failures),
// re-implemented here on C stdio so it builds as C++17 as well as C++20 (no <span> required:
// the pointer + count overloads below are what the span versions forward to).
//
// Little-endian 32-bit floats for parameters and optimizer state, 32-bit unsigned ids for
// edges, 64-bit unsigned offsets (the machines this runs on are little-endian).
#pragma once

#include <cstdint>
#include <cstdio>
#include <string>
#include <vector>

#if __cplusplus >= 202002L
#include <span>
#endif

#include "ember/common.h"

namespace ember {

static_assert(sizeof(float) == 4, "on-disk floats are 32-bit");

namespace detail {
struct File {
    std::FILE* f = nullptr;
    File(const std::string& path, const char* mode) : f(std::fopen(path.c_str(), mode)) {}
    ~File() {
        if (f) std::fclose(f);
    }
    File(const File&) = delete;
    File& operator=(const File&) = delete;
};

inline std::uint64_t file_bytes(std::FILE* f, const std::string& path) {
    if (std::fseek(f, 0, SEEK_END) != 0) throw IoError("seek failed: " + path);
    const long n = std::ftell(f);
    if (n < 0) throw IoError("tell failed: " + path);
    std::rewind(f);
    return static_cast<std::uint64_t>(n);
}
}  // namespace detail

// Writes count elements (truncating the file).
template <typename T>
void write_pod_file(const std::string& path, const T* data, std::size_t count) {
    detail::File out(path, "wb");
    if (!out.f) throw IoError("cannot open for write: " + path);
    if (count && std::fwrite(data, sizeof(T), count, out.f) != count) throw IoError("write failed: " + path);
    if (std::fflush(out.f) != 0) throw IoError("write failed: " + path);
}

// Reads the whole file; its size must be a multiple of sizeof(T).
template <typename T>
std::vector<T> read_pod_file(const std::string& path) {
    detail::File in(path, "rb");
    if (!in.f) throw IoError("cannot open for read: " + path);
    const std::uint64_t bytes = detail::file_bytes(in.f, path);
    if (bytes % sizeof(T) != 0)
        throw IoError("file size " + std::to_string(bytes) + " not a multiple of element size: " + path);
    std::vector<T> data(bytes / sizeof(T));
    if (!data.empty() && std::fread(data.data(), sizeof(T), data.size(), in.f) != data.size())
        throw IoError("read failed: " + path);
    return data;
}

// Reads exactly count elements into out; a file of any other size is an error.
template <typename T>
void read_pod_file_exact(const std::string& path, T* out, std::size_t count) {
    detail::File in(path, "rb");
    if (!in.f) throw IoError("cannot open for read: " + path);
    const std::uint64_t bytes = detail::file_bytes(in.f, path);
    if (bytes != count * sizeof(T))
        throw IoError("file " + path + " has " + std::to_string(bytes) + " bytes, expected " +
                      std::to_string(count * sizeof(T)));
    if (count && std::fread(out, sizeof(T), count, in.f) != count) throw IoError("read failed: " + path);
}

#if __cplusplus >= 202002L
template <typename T>
void write_pod_file(const std::string& path, std::span<const T> data) {
    write_pod_file(path, data.data(), data.size());
}
template <typename T>
void read_pod_file_exact(const std::string& path, std::span<T> out) {
    read_pod_file_exact(path, out.data(), out.size());
}
#endif

}  // namespace ember
