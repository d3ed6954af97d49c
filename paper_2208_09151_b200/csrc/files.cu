// files.cu -- the runtime-file writers (FORMATS.md: ids / adj / init / update;
// sampler.hpp:123-182, changeset.hpp:409-454) as one asynchronous pipeline.
//
// The reference writes each file from host vectors with a BinWriter. Here the
// byte image of every file of a call is assembled on the device by one pack
// kernel -- headers (magic + counts, built on the host) copied from a small
// blob, u32 device ids widened to the format's u64, (src, dst) u32 pairs copied
// -- into one staging buffer; a side copy stream moves it to pinned host
// memory in chunks (double-buffered), and a pool of host threads pwrite()s the
// parts of every file a chunk holds as soon as it lands. Packing, D2H and file
// writes overlap; the bytes are the reference's (tests/test_gpu_files.py).
#include <fcntl.h>
#include <unistd.h>

#include <thread>

#include "files.cuh"

namespace gx {

__global__ void k_pack_files(const PackOp* __restrict__ ops, uint32_t nops, const uint8_t* __restrict__ blob,
                             uint8_t* __restrict__ img) {
    for (uint32_t o = blockIdx.x; o < nops; o += gridDim.x) {
        const PackOp op = ops[o];
        // every piece starts 4-byte aligned (headers are 8 / 4 / 8 bytes), not
        // always 8: adj files carry a u32 layer count, so stores are u32
        uint32_t* d = reinterpret_cast<uint32_t*>(img + op.dst);
        if (op.kind == kPackWiden) {  // u32 -> u64 (little-endian: low word, then 0)
            const uint32_t* s = static_cast<const uint32_t*>(op.src);
            for (uint64_t i = threadIdx.x; i < op.n; i += blockDim.x) {
                d[2 * i] = s[i];
                d[2 * i + 1] = 0u;
            }
        } else if (op.kind == kPackCopy8) {  // (src, dst) u32 pairs
            const uint2* s = static_cast<const uint2*>(op.src);
            for (uint64_t i = threadIdx.x; i < op.n; i += blockDim.x) {
                const uint2 v = s[i];
                d[2 * i] = v.x;
                d[2 * i + 1] = v.y;
            }
        } else {  // header bytes from the blob (op.src = offset into it)
            const uint64_t b0 = reinterpret_cast<uint64_t>(op.src);
            for (uint64_t i = threadIdx.x; i < op.n; i += blockDim.x) img[op.dst + i] = blob[b0 + i];
        }
    }
}

uint64_t FileImage::add_file(const std::string& path) {
    paths.push_back(path);
    starts.push_back(total);
    return total;
}

void FileImage::header(const void* p, uint64_t n) {
    const uint64_t at = blob.size();
    blob.insert(blob.end(), static_cast<const uint8_t*>(p), static_cast<const uint8_t*>(p) + n);
    ops.push_back({total, reinterpret_cast<const void*>(at), n, kPackBlob});
    total += n;
}

void FileImage::widen(const uint32_t* d_src, uint64_t n) {
    if (n) ops.push_back({total, d_src, n, kPackWiden});
    total += 8 * n;
}

void FileImage::copy8(const void* d_src, uint64_t n) {
    if (n) ops.push_back({total, d_src, n, kPackCopy8});
    total += 8 * n;
}

namespace {
struct Fd {
    int fd = -1;
    ~Fd() {
        if (fd >= 0) ::close(fd);
    }
};
void pwrite_all(int fd, const uint8_t* p, uint64_t n, uint64_t off, const std::string& path) {
    while (n) {
        const ssize_t w = ::pwrite(fd, p, n, (off_t)off);
        if (w <= 0) fail(GX_RUNTIME_ERROR, "short write: " + path);
        p += w;
        n -= (uint64_t)w;
        off += (uint64_t)w;
    }
}
}  // namespace

void write_file_image(gx_ctx* ctx, FileImage& im) {
    const size_t F = im.paths.size();
    im.starts.push_back(im.total);  // file f = [starts[f], starts[f + 1])
    std::vector<Fd> fds(F);
    for (size_t f = 0; f < F; ++f) {
        fds[f].fd = ::open(im.paths[f].c_str(), O_WRONLY | O_CREAT | O_TRUNC, 0644);
        if (fds[f].fd < 0) fail(GX_RUNTIME_ERROR, "cannot open for write: " + im.paths[f]);
    }
    if (!im.total) return;
    cudaStream_t st = ctx->stream;
    DevBuf<uint8_t> img(im.total), blob(std::max<size_t>(im.blob.size(), 1));
    DevBuf<PackOp> ops(std::max<size_t>(im.ops.size(), 1));
    GX_CUDA(cudaMemcpyAsync(blob.p, im.blob.data(), im.blob.size(), cudaMemcpyHostToDevice, st));
    GX_CUDA(cudaMemcpyAsync(ops.p, im.ops.data(), im.ops.size() * sizeof(PackOp), cudaMemcpyHostToDevice, st));
    if (!im.ops.empty()) {
        k_pack_files<<<std::min<size_t>(im.ops.size(), (size_t)ctx->num_sms * 8), 256, 0, st>>>(
            ops.p, (uint32_t)im.ops.size(), blob.p, img.p);
        GX_CHECK_LAUNCH();
    }
    // chunked D2H on a side stream into two pinned buffers; chunk k's writes
    // run while chunk k + 1 is in flight
    static const uint64_t CH = (uint64_t)env_int("GX_FILE_CHUNK_MB", 64) << 20;
    const uint64_t chunk = std::min<uint64_t>(im.total, CH);
    const uint64_t nchunks = (im.total + chunk - 1) / chunk;
    PinBuf<uint8_t> pin[2];
    pin[0].alloc(chunk);
    if (nchunks > 1) pin[1].alloc(chunk);
    cudaStream_t cp;
    GX_CUDA(cudaStreamCreateWithFlags(&cp, cudaStreamNonBlocking));
    cudaEvent_t packed, landed[2];
    GX_CUDA(cudaEventCreateWithFlags(&packed, cudaEventDisableTiming));
    for (auto& e : landed) GX_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    auto cleanup = [&] {
        cudaEventDestroy(packed);
        for (auto& e : landed) cudaEventDestroy(e);
        cudaStreamDestroy(cp);
    };
    try {
        GX_CUDA(cudaEventRecord(packed, st));
        GX_CUDA(cudaStreamWaitEvent(cp, packed, 0));
        auto issue = [&](uint64_t k) {
            const uint64_t lo = k * chunk, n = std::min(chunk, im.total - lo);
            GX_CUDA(cudaMemcpyAsync(pin[k & 1].p, img.p + lo, n, cudaMemcpyDeviceToHost, cp));
            GX_CUDA(cudaEventRecord(landed[k & 1], cp));
        };
        issue(0);
        static const int nthreads = std::max(1, env_int("GX_FILE_THREADS", 8));
        size_t fbegin = 0;  // first file overlapping the current chunk
        for (uint64_t k = 0; k < nchunks; ++k) {
            GX_CUDA(cudaEventSynchronize(landed[k & 1]));
            if (k + 1 < nchunks) issue(k + 1);  // the other buffer is free: its writes finished
            const uint64_t lo = k * chunk, hi = std::min(im.total, lo + chunk);
            while (fbegin < F && im.starts[fbegin + 1] <= lo) ++fbegin;
            size_t fend = fbegin;
            while (fend < F && im.starts[fend] < hi) ++fend;
            const uint8_t* base = pin[k & 1].p;
            auto work = [&](size_t f0, size_t f1) {
                for (size_t f = f0; f < f1; ++f) {
                    const uint64_t a = std::max(lo, im.starts[f]), b = std::min(hi, im.starts[f + 1]);
                    if (b > a) pwrite_all(fds[f].fd, base + (a - lo), b - a, a - im.starts[f], im.paths[f]);
                }
            };
            const size_t nf = fend - fbegin;
            const int T = (int)std::min<size_t>(nthreads, std::max<size_t>(nf / 4, 1));
            if (T <= 1) {
                work(fbegin, fend);
            } else {
                std::vector<std::thread> ts;
                std::vector<std::exception_ptr> errs(T);
                for (int t = 0; t < T; ++t)
                    ts.emplace_back([&, t] {
                        try {
                            work(fbegin + nf * t / T, fbegin + nf * (t + 1) / T);
                        } catch (...) {
                            errs[t] = std::current_exception();
                        }
                    });
                for (auto& th : ts) th.join();
                for (auto& e : errs)
                    if (e) std::rethrow_exception(e);
            }
        }
        GX_CUDA(cudaStreamSynchronize(cp));
    } catch (...) {
        cudaStreamSynchronize(cp);
        cleanup();
        throw;
    }
    cleanup();
    for (size_t f = 0; f < F; ++f) {
        const int fd = fds[f].fd;
        fds[f].fd = -1;
        if (::close(fd) != 0) fail(GX_RUNTIME_ERROR, "close failed: " + im.paths[f]);
    }
}

}  // namespace gx
