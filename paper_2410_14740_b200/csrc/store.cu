// store.cu -- NEXT-1: the SSD -> DRAM tier of M2Cache (host code only, part of libm2c).
//
// Paper (§5.4): the full model lives on SSD; a DRAM cache holds layers in two
// areas -- a FIXED area with the first n layers and a DYNAMIC area managed FIFO for the
// upcoming ones -- and a pattern-aware preloader moves WHOLE LAYERS (not
// neurons: neuron-level SSD reads were rejected for their mapping overhead) at
// least two layers ahead of the computation, because loading one layer takes about twice
// as long as computing it.  I/O threads do the reads.
//
// Here the SSD is a packed layer-major file of the host tier (every layer's three packed
// tiers, exactly the bytes of the pinned host tier, each layer padded to 4 KiB for O_DIRECT),
// the DRAM cache is caller-owned pinned memory cut into frames, and one I/O thread preloads
// layers `lookahead` ahead of the layer the decode loop asks for.  The decode loop (host side
// of m2c_decode_step) calls acquire(l) before enqueuing layer l's miss fill: it blocks until
// layer l is resident and returns its frame; release(l, event) records when the GPU has
// finished reading the frame, and the I/O thread synchronises on that event before it
// overwrites the frame (FIFO replacement).  Results do not depend on the store: the frames
// hold the same bytes as the in-memory host tier (tests/test_gpu_parity.py).
#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <chrono>
#include <condition_variable>
#include <cstring>
#include <deque>
#include <mutex>
#include <thread>
#include <vector>

#include "m2c_internal.cuh"

namespace m2c {

constexpr size_t kAlign = 4096;
static size_t round_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

struct Store {
    int fd = -1;
    bool direct = false;
    int n_layers = 0, n_fixed = 0, n_dyn = 0, ahead = 2;
    size_t layer_bytes = 0, frame_bytes = 0;
    uint8_t *frames = nullptr;            // caller-owned pinned memory
    // frame state
    std::vector<int> frame_layer;         // layer held by each frame (-1 none)
    std::vector<int> frame_ready;         // 1 when the read completed
    std::vector<cudaEvent_t> frame_done;  // recorded after the GPU's last read of the frame
    std::vector<int> frame_used;          // 1 if frame_done has been recorded since the load
    std::vector<int> layer_frame;         // frame of each layer (-1 not resident / in flight)
    std::deque<int> fifo;                 // dynamic frames in load order (oldest first)
    int wanted = 0;                       // the layer the decode loop is waiting for / at
    bool stop = false;
    std::mutex mu;
    std::condition_variable cv;
    std::thread io;
    // stats
    int64_t bytes_read = 0, loads = 0;
    double io_s = 0.0, stall_s = 0.0;

    bool read_layer(int l, uint8_t *dst) {
        const off_t off = (off_t)l * (off_t)frame_bytes;
        size_t done = 0;
        while (done < frame_bytes) {
            const ssize_t r = pread(fd, dst + done, frame_bytes - done, off + (off_t)done);
            if (r <= 0) return false;
            done += (size_t)r;
        }
        return true;
    }

    // is layer c inside the window [wanted, wanted + ahead] (decode order, wrapping)?
    bool in_window(int c) const { return (c - wanted + n_layers) % n_layers <= ahead; }

    // the preloader: keep the window's layers resident -- the first missing one is loaded
    // next, into a free dynamic frame or else the oldest (FIFO) frame whose layer has left
    // the window, once the GPU is done reading it; nothing to do -> sleep
    void run() {
        std::unique_lock<std::mutex> lk(mu);
        while (!stop) {
            int l = -1;
            for (int dd = 0; dd <= ahead && dd < n_layers; dd++) {
                const int c = (wanted + dd) % n_layers;
                if (c >= n_fixed && layer_frame[c] < 0) {
                    l = c;
                    break;
                }
            }
            if (l < 0 || n_dyn == 0) {
                cv.wait(lk);
                continue;
            }
            int f = -1;
            for (int i = n_fixed; i < n_fixed + n_dyn; i++)
                if (frame_layer[i] < 0) {
                    f = i;
                    break;
                }
            if (f < 0) {
                auto it = fifo.begin();
                while (it != fifo.end() && in_window(frame_layer[*it])) ++it;
                if (it == fifo.end()) {  // every frame holds a layer still needed: wait
                    cv.wait(lk);
                    continue;
                }
                const int old = *it;
                fifo.erase(it);
                const bool used = frame_used[old];
                cudaEvent_t ev = frame_done[old];
                layer_frame[frame_layer[old]] = -1;
                frame_layer[old] = -1;
                frame_ready[old] = 0;
                lk.unlock();
                if (used) cudaEventSynchronize(ev);  // the GPU has finished reading it
                lk.lock();
                f = old;
            }
            frame_layer[f] = l;
            frame_ready[f] = 0;
            frame_used[f] = 0;
            layer_frame[l] = f;
            fifo.push_back(f);
            lk.unlock();
            const auto t0 = std::chrono::steady_clock::now();
            const bool ok = read_layer(l, frames + (size_t)f * frame_bytes);
            const double dt = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
            lk.lock();
            io_s += dt;
            if (ok) {
                bytes_read += (int64_t)frame_bytes;
                loads++;
            }
            frame_ready[f] = ok ? 1 : -1;
            cv.notify_all();
        }
    }

    // decode loop: block until layer l is resident; returns its frame or nullptr on I/O error
    uint8_t *acquire(int l) {
        std::unique_lock<std::mutex> lk(mu);
        wanted = l;  // the window starts here: the preloader loads l first if it is missing
        cv.notify_all();
        const auto t0 = std::chrono::steady_clock::now();
        cv.wait(lk, [&] { return layer_frame[l] >= 0 && frame_ready[layer_frame[l]] != 0; });
        stall_s += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        const int f = layer_frame[l];
        return frame_ready[f] > 0 ? frames + (size_t)f * frame_bytes : nullptr;
    }
    void release(int l, cudaStream_t st) {
        std::unique_lock<std::mutex> lk(mu);
        const int f = layer_frame[l];
        if (f < 0) return;
        cudaEventRecord(frame_done[f], st);
        frame_used[f] = 1;
        wanted = (l + 1) % n_layers;
        cv.notify_all();
    }
};

m2c_status store_open(m2c_ctx *c, const char *path, int n_fixed, int n_dyn, int ahead, void *frames,
                      size_t frames_bytes, size_t layer_bytes) {
    Store *s = new Store();
    s->n_layers = c->desc.n_layers;
    s->n_fixed = n_fixed;
    s->n_dyn = n_dyn;
    s->ahead = ahead;
    s->layer_bytes = layer_bytes;
    s->frame_bytes = round_up(layer_bytes, kAlign);
    s->frames = static_cast<uint8_t *>(frames);
    if (frames_bytes < (size_t)(n_fixed + n_dyn) * s->frame_bytes) {
        delete s;
        return fail(M2C_ERR_CAPACITY, "store: frames smaller than (n_fixed + n_dynamic) x frame bytes");
    }
    s->fd = open(path, O_RDONLY | O_DIRECT);
    s->direct = s->fd >= 0;
    if (s->fd < 0 || (reinterpret_cast<uintptr_t>(frames) % kAlign)) {
        if (s->fd >= 0) close(s->fd);
        s->fd = open(path, O_RDONLY);
        s->direct = false;
    }
    if (s->fd < 0) {
        delete s;
        return fail(M2C_ERR_INVALID_ARG, std::string("store: cannot open ") + path);
    }
    struct stat stt;
    if (fstat(s->fd, &stt) != 0 || (size_t)stt.st_size < (size_t)s->n_layers * s->frame_bytes) {
        close(s->fd);
        delete s;
        return fail(M2C_ERR_STATE, "store: file shorter than n_layers x frame bytes (m2c_store_write first)");
    }
    const int nf = n_fixed + n_dyn;
    s->frame_layer.assign(nf, -1);
    s->frame_ready.assign(nf, 0);
    s->frame_used.assign(nf, 0);
    s->frame_done.resize(nf);
    s->layer_frame.assign(s->n_layers, -1);
    for (int i = 0; i < nf; i++) cudaEventCreateWithFlags(&s->frame_done[i], cudaEventDisableTiming);
    // the fixed area: the first n_fixed layers, loaded once
    for (int l = 0; l < n_fixed && l < s->n_layers; l++) {
        if (!s->read_layer(l, s->frames + (size_t)l * s->frame_bytes)) {
            for (cudaEvent_t e : s->frame_done) cudaEventDestroy(e);
            close(s->fd);
            delete s;
            return fail(M2C_ERR_STATE, "store: read of a fixed-area layer failed");
        }
        s->frame_layer[l] = l;
        s->frame_ready[l] = 1;
        s->layer_frame[l] = l;
        s->bytes_read += (int64_t)s->frame_bytes;
        s->loads++;
    }
    s->io = std::thread([s] { s->run(); });
    c->store = s;
    return M2C_OK;
}

void store_close(m2c_ctx *c) {
    Store *s = static_cast<Store *>(c->store);
    if (!s) return;
    {
        std::lock_guard<std::mutex> lk(s->mu);
        s->stop = true;
    }
    s->cv.notify_all();
    if (s->io.joinable()) s->io.join();
    for (cudaEvent_t e : s->frame_done) cudaEventDestroy(e);
    if (s->fd >= 0) close(s->fd);
    delete s;
    c->store = nullptr;
}

uint8_t *store_acquire(m2c_ctx *c, int l) { return static_cast<Store *>(c->store)->acquire(l); }
void store_release(m2c_ctx *c, int l, cudaStream_t st) { static_cast<Store *>(c->store)->release(l, st); }

void store_stats(m2c_ctx *c, int64_t *bytes, int64_t *loads, double *io_s, double *stall_s) {
    Store *s = static_cast<Store *>(c->store);
    std::lock_guard<std::mutex> lk(s->mu);
    *bytes = s->bytes_read;
    *loads = s->loads;
    *io_s = s->io_s;
    *stall_s = s->stall_s;
}

// the packed file: layer l at offset l x round_up(layer_bytes, 4 KiB); the layer's host tier
// region (three packed tiers, m2c_layer_footprint's host bytes) verbatim
m2c_status store_write(m2c_ctx *c, const char *path, size_t layer_bytes) {
    const size_t fb = round_up(layer_bytes, kAlign);
    const int fd = open(path, O_WRONLY | O_CREAT | O_TRUNC, 0644);
    if (fd < 0) return fail(M2C_ERR_INVALID_ARG, std::string("store_write: cannot create ") + path);
    std::vector<uint8_t> pad(fb - layer_bytes, 0);
    for (int l = 0; l < c->desc.n_layers; l++) {
        const LayerState &L = c->layers[l];
        if (!L.loaded || L.mode == 0 || !L.host_base) {
            close(fd);
            return fail(M2C_ERR_STATE, "store_write: every layer must be loaded in LRU/ATU mode");
        }
        size_t done = 0;
        while (done < layer_bytes) {
            const ssize_t w = pwrite(fd, L.host_base + done, layer_bytes - done, (off_t)l * (off_t)fb + (off_t)done);
            if (w <= 0) {
                close(fd);
                return fail(M2C_ERR_STATE, "store_write: write failed");
            }
            done += (size_t)w;
        }
        if (!pad.empty() && pwrite(fd, pad.data(), pad.size(), (off_t)l * (off_t)fb + (off_t)layer_bytes) < 0) {
            close(fd);
            return fail(M2C_ERR_STATE, "store_write: write failed");
        }
    }
    fsync(fd);
    close(fd);
    return M2C_OK;
}

}  // namespace m2c
