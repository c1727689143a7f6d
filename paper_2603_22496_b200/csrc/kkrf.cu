// KKRF container I/O: the reference's binary RF format
// (rffile.py:1-26, write_container 74-113, read_container 116-178), read
// straight into device memory for the throughput path.
//
// Layout (little-endian): 59-byte head "<4sHB3I5d" (magic "KKRF", u16
// version, u8 kind, u32 N, channels, T, f64 fs, fc, c, pitch, t0), N f64
// transmit angles, M f64 receive angles (kind 2 only), then the C-order
// payload (float32 for kind 0, complex64 for kinds 1/2).  Validation and its
// error texts stay in the Python mirror (rffile.py) so they match the
// reference word for word; this file moves bytes.
//
// Payload streaming: the file is read in 16 MiB chunks into two pinned
// buffers; chunk i's host->device copy (cudaMemcpyAsync on the caller's
// stream) overlaps the read of chunk i+1.  Writes mirror it (device->host
// copy of chunk i+1 overlaps the write of chunk i).  Both return with the
// stream's copies complete.

#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <atomic>
#include <cerrno>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "common.cuh"

namespace kkb {
namespace {

constexpr size_t kChunk = 16u << 20;
constexpr size_t kHead = 59;

std::mutex g_io_mu;  // the staging buffers are shared by all callers
void *g_pinned[2] = {nullptr, nullptr};
cudaEvent_t g_ev[2];

int ensure_staging() {
    if (g_pinned[0]) return KKB_OK;
    for (int i = 0; i < 2; ++i) {
        KKB_TRY_CUDA(cudaHostAlloc(&g_pinned[i], kChunk, cudaHostAllocDefault), "cudaHostAlloc(kkrf)");
        KKB_TRY_CUDA(cudaEventCreateWithFlags(&g_ev[i], cudaEventDisableTiming), "event(kkrf)");
    }
    return KKB_OK;
}

int io_error(const char *what, const char *path) {
    set_error("%s %s: %s", what, path, strerror(errno));
    return KKB_ERR_IO;
}

// read exactly n bytes at offset (short file -> KKB_ERR_FORMAT)
int pread_full(int fd, void *dst, size_t n, long long off, const char *path) {
    char *p = static_cast<char *>(dst);
    while (n > 0) {
        ssize_t r = pread(fd, p, n, (off_t)off);
        if (r < 0) {
            if (errno == EINTR) continue;
            return io_error("read", path);
        }
        if (r == 0) {
            set_error("%s: unexpected end of file", path);
            return KKB_ERR_FORMAT;
        }
        p += r;
        n -= (size_t)r;
        off += r;
    }
    return KKB_OK;
}

int write_full(int fd, const void *src, size_t n, const char *path) {
    const char *p = static_cast<const char *>(src);
    while (n > 0) {
        ssize_t r = write(fd, p, n);
        if (r < 0) {
            if (errno == EINTR) continue;
            return io_error("write", path);
        }
        p += r;
        n -= (size_t)r;
    }
    return KKB_OK;
}

template <typename T>
T get_le(const unsigned char *b) {
    T v;
    memcpy(&v, b, sizeof(T));  // x86-64 / aarch64 hosts are little-endian
    return v;
}
template <typename T>
void put_le(unsigned char *b, T v) {
    memcpy(b, &v, sizeof(T));
}

struct Fd {
    int fd = -1;
    ~Fd() {
        if (fd >= 0) close(fd);
    }
};

}  // namespace
}  // namespace kkb

using namespace kkb;

extern "C" int kkb_kkrf_read_header(const char *path, kkb_kkrf_header *h) {
    if (!path || !h) {
        set_error("kkrf_read_header: null argument");
        return KKB_ERR_ARG;
    }
    Fd f;
    f.fd = open(path, O_RDONLY);
    if (f.fd < 0) return io_error("open", path);
    struct stat st;
    if (fstat(f.fd, &st) != 0) return io_error("stat", path);
    memset(h, 0, sizeof(*h));
    h->file_bytes = (long long)st.st_size;
    if ((size_t)st.st_size < kHead) {
        set_error("%s: truncated header", path);
        return KKB_ERR_FORMAT;
    }
    unsigned char b[kHead];
    int rc = pread_full(f.fd, b, kHead, 0, path);
    if (rc) return rc;
    memcpy(h->magic, b, 4);
    h->version = get_le<uint16_t>(b + 4);
    h->kind = b[6];
    h->num_transmits = get_le<uint32_t>(b + 7);
    h->num_channels = get_le<uint32_t>(b + 11);
    h->num_samples = get_le<uint32_t>(b + 15);
    h->sampling_frequency = get_le<double>(b + 19);
    h->center_frequency = get_le<double>(b + 27);
    h->sound_speed = get_le<double>(b + 35);
    h->pitch = get_le<double>(b + 43);
    h->start_time = get_le<double>(b + 51);
    h->head_bytes = (long long)kHead;
    return KKB_OK;
}

extern "C" int kkb_kkrf_read_bytes(const char *path, long long offset, long long bytes, void *dst,
                                   int dst_is_device, void *stream) {
    if (!path || (bytes > 0 && !dst) || offset < 0 || bytes < 0) {
        set_error("kkrf_read_bytes: bad argument");
        return KKB_ERR_ARG;
    }
    Fd f;
    f.fd = open(path, O_RDONLY);
    if (f.fd < 0) return io_error("open", path);
    if (!dst_is_device) return pread_full(f.fd, dst, (size_t)bytes, offset, path);
    std::lock_guard<std::mutex> lk(g_io_mu);
    int rc = ensure_staging();
    if (rc) return rc;
    cudaStream_t s = as_stream(stream);
    char *d = static_cast<char *>(dst);
    long long done = 0;
    for (int i = 0; done < bytes; ++i) {
        const int k = i & 1;
        const size_t n = (size_t)std::min<long long>((long long)kChunk, bytes - done);
        if (i >= 2) KKB_TRY_CUDA(cudaEventSynchronize(g_ev[k]), "kkrf staging wait");
        rc = pread_full(f.fd, g_pinned[k], n, offset + done, path);
        if (rc) {
            cudaStreamSynchronize(s);
            return rc;
        }
        KKB_TRY_CUDA(cudaMemcpyAsync(d + done, g_pinned[k], n, cudaMemcpyHostToDevice, s), "kkrf H2D");
        KKB_TRY_CUDA(cudaEventRecord(g_ev[k], s), "kkrf record");
        done += (long long)n;
    }
    KKB_TRY_CUDA(cudaStreamSynchronize(s), "kkrf H2D sync");
    return KKB_OK;
}

// Parallel ensemble ingest: `threads` reader threads, each with its own pair
// of pinned 16 MiB staging buffers and its own stream, take files round-robin
// (pread from the page cache / disk into pinned memory, async H2D into the
// frame's slot).  Slots persist across calls (one ensemble read at a time).
namespace {
struct ReadSlot {
    void *pinned[2] = {nullptr, nullptr};
    cudaEvent_t ev[2] = {nullptr, nullptr};
    cudaStream_t st = nullptr;
};
std::mutex g_ens_mu;
std::vector<ReadSlot> g_slots;

int ensure_slots(int n, int dev) {
    while ((int)g_slots.size() < n) {
        ReadSlot r;
        cudaSetDevice(dev);
        for (int i = 0; i < 2; ++i) {
            KKB_TRY_CUDA(cudaHostAlloc(&r.pinned[i], kChunk, cudaHostAllocDefault), "cudaHostAlloc(kkrf slot)");
            KKB_TRY_CUDA(cudaEventCreateWithFlags(&r.ev[i], cudaEventDisableTiming), "event(kkrf slot)");
        }
        KKB_TRY_CUDA(cudaStreamCreateWithFlags(&r.st, cudaStreamNonBlocking), "stream(kkrf slot)");
        g_slots.push_back(r);
    }
    return KKB_OK;
}

int read_one(ReadSlot &r, int &i, const char *path, long long offset, long long bytes, char *d) {
    Fd f;
    f.fd = open(path, O_RDONLY);
    if (f.fd < 0) return io_error("open", path);
    for (long long done = 0; done < bytes; ++i) {
        const int k = i & 1;
        const size_t n = (size_t)std::min<long long>((long long)kChunk, bytes - done);
        if (i >= 2) KKB_TRY_CUDA(cudaEventSynchronize(r.ev[k]), "kkrf slot wait");
        int rc = pread_full(f.fd, r.pinned[k], n, offset + done, path);
        if (rc) return rc;
        KKB_TRY_CUDA(cudaMemcpyAsync(d + done, r.pinned[k], n, cudaMemcpyHostToDevice, r.st), "kkrf H2D");
        KKB_TRY_CUDA(cudaEventRecord(r.ev[k], r.st), "kkrf record");
        done += (long long)n;
    }
    return KKB_OK;
}
}  // namespace

extern "C" int kkb_kkrf_read_ensemble(const char *const *paths, const long long *offsets_host,
                                      int n_files, long long frame_bytes, void *dst, int threads,
                                      void *stream) {
    if (!paths || !offsets_host || n_files < 0 || frame_bytes < 0 || (n_files && frame_bytes && !dst) ||
        threads < 1 || threads > 64) {
        set_error("kkrf_read_ensemble: bad argument (1 <= threads <= 64)");
        return KKB_ERR_ARG;
    }
    if (!n_files || !frame_bytes) return KKB_OK;
    std::lock_guard<std::mutex> lk(g_ens_mu);
    int dev = 0;
    KKB_TRY_CUDA(cudaGetDevice(&dev), "cudaGetDevice");
    threads = std::min(threads, n_files);
    int rc = ensure_slots(threads, dev);
    if (rc) return rc;
    // the destination may still be in use by work queued on the caller's stream
    cudaEvent_t ready;
    KKB_TRY_CUDA(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming), "event(kkrf ready)");
    cudaEventRecord(ready, as_stream(stream));
    std::atomic<int> next{0}, first_err{0};
    std::vector<std::string> err_msg(threads);
    auto worker = [&](int t) {
        cudaSetDevice(dev);
        ReadSlot &r = g_slots[t];
        cudaStreamWaitEvent(r.st, ready, 0);
        int i = 0;
        for (int f; (f = next.fetch_add(1)) < n_files && !first_err.load();) {
            const int e = read_one(r, i, paths[f], offsets_host[f], frame_bytes,
                                   static_cast<char *>(dst) + (size_t)f * frame_bytes);
            if (e) {
                int z = 0;
                if (first_err.compare_exchange_strong(z, e)) err_msg[t] = kkb_last_error();
            }
        }
        cudaStreamSynchronize(r.st);
    };
    std::vector<std::thread> pool;
    for (int t = 1; t < threads; ++t) pool.emplace_back(worker, t);
    worker(0);
    for (auto &th : pool) th.join();
    cudaEventDestroy(ready);
    if (first_err.load()) {
        for (auto &m : err_msg)
            if (!m.empty()) set_error("%s", m.c_str());
        return first_err.load();
    }
    return KKB_OK;
}

extern "C" int kkb_kkrf_write(const char *path, const kkb_kkrf_header *h, const double *tx_host,
                              const double *rx_host, const void *payload, long long payload_bytes,
                              int payload_is_device, void *stream) {
    if (!path || !h || (h->num_transmits && !tx_host) || (h->kind == 2 && h->num_channels && !rx_host) ||
        payload_bytes < 0 || (payload_bytes > 0 && !payload)) {
        set_error("kkrf_write: bad argument");
        return KKB_ERR_ARG;
    }
    unsigned char b[kHead];
    memcpy(b, h->magic, 4);
    put_le<uint16_t>(b + 4, h->version);
    b[6] = h->kind;
    put_le<uint32_t>(b + 7, h->num_transmits);
    put_le<uint32_t>(b + 11, h->num_channels);
    put_le<uint32_t>(b + 15, h->num_samples);
    put_le<double>(b + 19, h->sampling_frequency);
    put_le<double>(b + 27, h->center_frequency);
    put_le<double>(b + 35, h->sound_speed);
    put_le<double>(b + 43, h->pitch);
    put_le<double>(b + 51, h->start_time);
    Fd f;
    f.fd = open(path, O_WRONLY | O_CREAT | O_TRUNC, 0644);
    if (f.fd < 0) return io_error("open", path);
    int rc = write_full(f.fd, b, kHead, path);
    if (!rc) rc = write_full(f.fd, tx_host, sizeof(double) * h->num_transmits, path);
    if (!rc && h->kind == 2) rc = write_full(f.fd, rx_host, sizeof(double) * h->num_channels, path);
    if (rc) return rc;
    if (!payload_is_device) return write_full(f.fd, payload, (size_t)payload_bytes, path);
    std::lock_guard<std::mutex> lk(g_io_mu);
    rc = ensure_staging();
    if (rc) return rc;
    cudaStream_t s = as_stream(stream);
    const char *src = static_cast<const char *>(payload);
    // copy chunk i+1 while chunk i is written
    const long long nchunks = (payload_bytes + (long long)kChunk - 1) / (long long)kChunk;
    auto issue = [&](long long i) -> int {
        const int k = (int)(i & 1);
        const long long off = i * (long long)kChunk;
        const size_t n = (size_t)std::min<long long>((long long)kChunk, payload_bytes - off);
        KKB_TRY_CUDA(cudaMemcpyAsync(g_pinned[k], src + off, n, cudaMemcpyDeviceToHost, s), "kkrf D2H");
        KKB_TRY_CUDA(cudaEventRecord(g_ev[k], s), "kkrf record");
        return KKB_OK;
    };
    if (nchunks > 0 && (rc = issue(0))) return rc;
    for (long long i = 0; i < nchunks; ++i) {
        const int k = (int)(i & 1);
        KKB_TRY_CUDA(cudaEventSynchronize(g_ev[k]), "kkrf D2H wait");
        if (i + 1 < nchunks && (rc = issue(i + 1))) return rc;
        const long long off = i * (long long)kChunk;
        const size_t n = (size_t)std::min<long long>((long long)kChunk, payload_bytes - off);
        rc = write_full(f.fd, g_pinned[k], n, path);
        if (rc) {
            cudaStreamSynchronize(s);
            return rc;
        }
    }
    return KKB_OK;
}
