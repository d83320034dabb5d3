// rawio.cu -- the RawF64 matrix file ("SKLR", the reference's interchange format,
// src/matrix_io.cpp:141-200) read straight into device memory, or a row shard of it.
//
// Header: "SKLR" | u32 rows | u32 cols | u32 reserved | rows*cols little-endian
// doubles, column-major.  Validation is the reference's load_raw, message for message
// and byte offset for byte offset (FormatError -> FQB_ERR_FORMAT + fqb_last_error +
// *err_offset).  Only the file's size and header are read to validate, then the rows
// [row0, row0 + rows) of each column (one contiguous run per column) are read with
// pread by several threads into pinned staging panels of whole columns, and every
// filled panel goes to the device with one cudaMemcpy2DAsync while the next is read
// (three panels in flight).  A row-sharded rank thus reads and uploads only its own
// slab; a host destination is filled by the same threads
// directly, without staging.
#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <climits>
#include <cstdint>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "engine.hpp"

namespace farqb {

namespace {

struct Fd {
    int fd = -1;
    ~Fd() {
        if (fd >= 0) ::close(fd);
    }
};

uint32_t u32le(const unsigned char* b) {
    return uint32_t(b[0]) | (uint32_t(b[1]) << 8) | (uint32_t(b[2]) << 16) | (uint32_t(b[3]) << 24);
}

// the reference's checks (matrix_io.cpp:141-165), on the file size and header only
void validate(int fd, int64_t* rows_out, int64_t* cols_out) {
    struct stat st;
    if (::fstat(fd, &st) != 0) throw Error(kStatusInvalid, "cannot stat matrix file");
    const uint64_t size = uint64_t(st.st_size);
    unsigned char h[16];
    const ssize_t got = size >= 16 ? ::pread(fd, h, 16, 0) : 0;
    if (size < 16 || got != 16) throw FormatFailure("truncated header, need 16 bytes", int64_t(size));
    if (std::memcmp(h, "SKLR", 4) != 0) throw FormatFailure("bad magic, expected SKLR", 0);
    const uint64_t rows = u32le(h + 4), cols = u32le(h + 8);
    if (rows > uint64_t(INT_MAX)) throw FormatFailure("dimension overflow in row count", 4);
    if (cols > uint64_t(INT_MAX)) throw FormatFailure("dimension overflow in column count", 8);
    if (cols != 0 && rows > (UINT64_MAX / 8) / cols) throw FormatFailure("dimension overflow in payload size", 4);
    const uint64_t need = rows * cols * 8;
    if (size - 16 < need)
        throw FormatFailure("truncated payload: expected " + std::to_string(need) + " bytes, found " +
                                std::to_string(size - 16),
                            int64_t(size));
    if (size - 16 > need) throw FormatFailure("trailing bytes after payload", int64_t(16 + need));
    *rows_out = int64_t(rows);
    *cols_out = int64_t(cols);
}

// columns [c0, c1) of rows [row0, row0 + rows) into dst (ld), by `threads` readers
void read_columns(int fd, int64_t m, int64_t row0, int64_t rows, int64_t c0, int64_t c1, double* dst, int64_t ld,
                  int threads) {
    std::atomic<int64_t> next{c0};
    std::atomic<bool> failed{false};
    auto work = [&]() {
        for (int64_t j; !failed && (j = next.fetch_add(1)) < c1;) {
            char* p = reinterpret_cast<char*>(dst + (j - c0) * ld);
            int64_t left = rows * 8;
            off_t off = off_t(16 + (j * m + row0) * 8);
            while (left > 0) {
                const ssize_t r = ::pread(fd, p, size_t(std::min<int64_t>(left, int64_t(1) << 30)), off);
                if (r <= 0) {
                    failed = true;
                    return;
                }
                p += r;
                off += r;
                left -= r;
            }
        }
    };
    const int nt = int(std::max<int64_t>(1, std::min<int64_t>(threads, c1 - c0)));
    std::vector<std::thread> pool;
    for (int t = 1; t < nt; ++t) pool.emplace_back(work);
    work();
    for (auto& t : pool) t.join();
    if (failed) throw Error(kStatusInvalid, "read error in matrix file");
}

int reader_threads() {
    const unsigned hw = std::thread::hardware_concurrency();
    return int(std::max(1u, std::min(hw ? hw : 4u, 16u)));
}

}  // namespace

void raw_header(const char* path, int64_t* rows, int64_t* cols) {
    Fd f;
    f.fd = ::open(path, O_RDONLY);
    if (f.fd < 0) throw Error(kStatusInvalid, std::string("cannot open ") + path);
    validate(f.fd, rows, cols);
}

void load_raw_rows(Handle* h, const char* path, int64_t row0, int64_t rows, double* dst, int64_t ld,
                   bool dst_on_device) {
    Fd f;
    f.fd = ::open(path, O_RDONLY);
    if (f.fd < 0) throw Error(kStatusInvalid, std::string("cannot open ") + path);
    int64_t m = 0, n = 0;
    validate(f.fd, &m, &n);
    if (row0 < 0 || rows < 0 || row0 + rows > m) throw Error(kStatusDimension, "row range outside the matrix");
    if (ld < std::max<int64_t>(rows, 1)) throw Error(kStatusDimension, "leading dimension too small");
    if (rows == 0 || n == 0) return;
    const int threads = reader_threads();
    if (!dst_on_device) {
        read_columns(f.fd, m, row0, rows, 0, n, dst, ld, threads);
        return;
    }
    if (!h) throw Error(kStatusInvalid, "a device destination needs a handle");
    // three pinned panels of whole columns, ~64 MB each, refilled once their upload is done
    constexpr int kPanels = 3;
    const int64_t col_bytes = rows * 8;
    const int64_t per_panel = std::max<int64_t>(1, (int64_t(64) << 20) / col_bytes);
    cudaStream_t s = h->stream;
    double* stage[kPanels] = {};
    cudaEvent_t done[kPanels] = {};
    struct Cleanup {
        double** st;
        cudaEvent_t* ev;
        ~Cleanup() {
            for (int i = 0; i < kPanels; ++i) {
                if (ev[i]) {
                    cudaEventSynchronize(ev[i]);
                    cudaEventDestroy(ev[i]);
                }
                if (st[i]) cudaFreeHost(st[i]);
            }
        }
    } cleanup{stage, done};
    for (int i = 0; i < kPanels; ++i) {
        FQB_CUDA(cudaMallocHost(reinterpret_cast<void**>(&stage[i]), size_t(per_panel * col_bytes)));
        FQB_CUDA(cudaEventCreateWithFlags(&done[i], cudaEventDisableTiming));
    }
    bool used[kPanels] = {};
    int k = 0;
    for (int64_t c0 = 0; c0 < n; c0 += per_panel, k = (k + 1) % kPanels) {
        const int64_t c1 = std::min(n, c0 + per_panel);
        if (used[k]) FQB_CUDA(cudaEventSynchronize(done[k]));   // its previous upload has landed
        read_columns(f.fd, m, row0, rows, c0, c1, stage[k], rows, threads);
        FQB_CUDA(cudaMemcpy2DAsync(dst + c0 * ld, size_t(ld) * 8, stage[k], size_t(rows) * 8, size_t(rows) * 8,
                                   size_t(c1 - c0), cudaMemcpyHostToDevice, s));
        FQB_CUDA(cudaEventRecord(done[k], s));
        used[k] = true;
    }
    FQB_CUDA(cudaStreamSynchronize(s));
}

}  // namespace farqb
