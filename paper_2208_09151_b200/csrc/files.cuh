// files.cuh -- byte images of the runtime files, written asynchronously (files.cu).
#pragma once

#include <string>
#include <vector>

#include "gx_internal.cuh"

namespace gx {

constexpr uint32_t kPackBlob = 0, kPackWiden = 1, kPackCopy8 = 2;

struct PackOp {
    uint64_t dst;     // byte offset in the image
    const void* src;  // device source (blob: byte offset into the header blob)
    uint64_t n;       // bytes (blob) or items (widen: u32 -> u64, copy8: 8-byte items)
    uint32_t kind;
};

// Files appended back to back: add_file, then its pieces in file order.
struct FileImage {
    std::vector<std::string> paths;
    std::vector<uint64_t> starts;
    std::vector<uint8_t> blob;
    std::vector<PackOp> ops;
    uint64_t total = 0;
    uint64_t add_file(const std::string& path);
    void header(const void* p, uint64_t n);
    void widen(const uint32_t* d_src, uint64_t n);
    void copy8(const void* d_src, uint64_t n);
    template <class T>
    void value(T v) {
        header(&v, sizeof v);
    }
};

// pack on ctx->stream, D2H on a side stream in chunks, pwrite by host threads
void write_file_image(gx_ctx* ctx, FileImage& im);

}  // namespace gx
