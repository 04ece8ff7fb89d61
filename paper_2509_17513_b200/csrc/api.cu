// C ABI entry points (include/gsv_b200.h): sessions, layer-prefix decode of
// a container into HBM with the reference's validation order, frame
// materialisation and rendering.
//
// read_layers (container.py:260-310) raises the FIRST error met while
// walking group -> layer -> channel entry -> {read, header, structure,
// decode+CRC, plane count, valid count}, then the group-level checks of
// _assemble_frames.  Here the host walks the directory and every payload's
// structure in that order (stopping at the first structural error, as the
// reference would), the GPU decodes and CRC-checks every run before that
// point, and the earliest failure in the reference's order is reported.
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <chrono>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "gsv_internal.h"

using namespace gsv;

// u8 staging buffers per aux stream for host outputs: the render of frame j
// on a stream waits for the read-back of frame j - kU8Bufs on it
constexpr int kU8Bufs = 3;

struct gsv_session {
    int device = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    RenderWork work;
    // frame-parallel rendering: independent frames on auxiliary streams, each
    // with its own workspace, so the many small latency-bound kernels of a
    // frame overlap with other frames' kernels
    std::vector<cudaStream_t> aux;
    std::vector<RenderWork*> aux_work;
    std::vector<uint8_t*> aux_u8;  // staging for host u8 outputs: kU8Bufs buffers per aux stream
    std::vector<size_t> aux_u8_cap;
    // read-back of host u8 outputs: per aux stream a copy stream, and per
    // staging buffer "rendered" / "copied" events, so the D2H of frame j
    // overlaps the rendering of frame j+1 on the same aux stream
    std::vector<cudaStream_t> aux_copy;
    std::vector<cudaEvent_t> ev_rendered, ev_copied, ev_copy_join;
    std::vector<int> aux_flip;
    cudaEvent_t ev_fork = nullptr;
    std::vector<cudaEvent_t> ev_join;
    int64_t kcap_hint = 0;
    // gsv_render_sequence_host: group uploads on their own stream into a ring
    // of device slots; per slot an "uploaded" event and per (slot, aux
    // stream) a "rendered" event
    cudaStream_t copy_in = nullptr;
    cudaStream_t check = nullptr;  // the groups' CRC kernels (validation, off the render path)
    cudaEvent_t ev_prep = nullptr;
    std::vector<cudaEvent_t> ev_up, ev_slot_done;
    // the payload slots, kept across calls (grow-only: cudaMalloc / cudaFree
    // synchronise, so they are not taken from the pool on every call)
    std::vector<uint8_t*> seq_slot;
    std::vector<size_t> seq_slot_cap;
    std::vector<cudaEvent_t> ev_plane;  // first group uploaded plane-major: frame f's planes landed
    // closed videos whose buffers may still be read by enqueued work: freed
    // once the event recorded at close has completed (gsv_video_close does
    // not synchronise, so the next open's host work overlaps the GPU tail)
    std::vector<std::pair<cudaEvent_t, gsv_video*>> graveyard;
    std::vector<cudaEvent_t> free_events;
};

namespace {

// Device blocks are recycled through a process-wide pool: opening a
// container and its descriptor uploads would otherwise cudaMalloc/cudaFree
// (both synchronising) on every call.  A block goes back to the pool when its
// owner is destroyed -- gsv_video_close synchronises the session first, so no
// kernel still uses it -- and is reused for a request of at most its size
// and at least half of it.  The pool is emptied when cudaMalloc fails.
std::mutex g_pool_mu;
std::multimap<size_t, void*> g_pool;  // capacity -> block

void pool_put(void* p, size_t cap) {
    if (!p) return;
    std::lock_guard<std::mutex> lk(g_pool_mu);
    g_pool.emplace(cap, p);
}

void* pool_get(size_t bytes, size_t* cap) {
    {
        std::lock_guard<std::mutex> lk(g_pool_mu);
        auto it = g_pool.lower_bound(bytes);
        if (it != g_pool.end() && it->first <= 2 * bytes + (1u << 20)) {
            void* p = it->second;
            *cap = it->first;
            g_pool.erase(it);
            return p;
        }
    }
    void* p = nullptr;
    if (cudaMalloc(&p, bytes) != cudaSuccess) {
        cudaGetLastError();
        std::lock_guard<std::mutex> lk(g_pool_mu);
        for (auto& kv : g_pool) cudaFree(kv.second);
        g_pool.clear();
        if (cudaMalloc(&p, bytes) != cudaSuccess) return nullptr;
    }
    *cap = bytes;
    return p;
}

struct DevBuf {
    void* p = nullptr;
    size_t n = 0;    // bytes requested
    size_t cap = 0;  // bytes of the block
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    ~DevBuf() { pool_put(p, cap); }
    int alloc(size_t bytes) {
        n = bytes;
        if (p && bytes <= cap) return GSV_OK;
        pool_put(p, cap);
        p = nullptr;
        cap = 0;
        if (bytes == 0) return GSV_OK;
        p = pool_get(bytes, &cap);
        if (!p) return fail(GSV_E_CUDA, "cudaMalloc: out of memory");
        return GSV_OK;
    }
    template <class T>
    T* as() const {
        return reinterpret_cast<T*>(p);
    }
};

// Pinned host staging for the small descriptor uploads and read-backs of a
// container open: a pageable cudaMemcpyAsync is synchronous and queues behind
// the big transfers other streams have in flight (frame read-backs, other
// groups' payload uploads), so the open's small copies go through this
// per-thread pinned bump buffer instead.  reset() at the start of an open
// (the previous open synchronised before returning).
struct PinnedStage {
    uint8_t* p = nullptr;
    size_t cap = 0, used = 0;
    // outgrown buffers: copies enqueued from them may still be in flight, so
    // they are freed only at reset(), which callers invoke with the work that
    // used the stage drained (cudaFreeHost can synchronise the device: never
    // called while a pipeline is being enqueued)
    std::vector<uint8_t*> retired;
    ~PinnedStage() {
        if (p) cudaFreeHost(p);
        for (uint8_t* q : retired) cudaFreeHost(q);
    }
    void reset() {
        used = 0;
        for (uint8_t* q : retired) cudaFreeHost(q);
        retired.clear();
    }
    uint8_t* reserve(size_t n, cudaStream_t) {
        const size_t need = ((used + 255) & ~size_t(255)) + n;
        if (need > cap) {  // grow into a fresh buffer; the old one is retired
            if (p) retired.push_back(p);
            cap = std::max(need * 2, (size_t)8 << 20);
            p = nullptr;
            if (cudaMallocHost(reinterpret_cast<void**>(&p), cap) != cudaSuccess) {
                p = nullptr;
                cap = 0;
                return nullptr;
            }
            used = 0;
        }
        used = (used + 255) & ~size_t(255);
        uint8_t* q = p + used;
        used += n;
        return q;
    }
};
thread_local PinnedStage t_stage;

// Zero-copy descriptor uploads (gsv_render_sequence_host): the copy engine
// runs host-to-device copies in submission order, so a small descriptor
// upload enqueued after a group's multi-hundred-MB payload upload would wait
// for it.  With this flag set, upload() has a kernel read the pinned staging
// buffer over PCIe instead (UVA: pinned host memory is device-addressable),
// and memsets are kernels too, so the copy engine carries payloads only.
thread_local bool t_zero_copy = false;

__global__ void stage_copy_kernel(uint8_t* __restrict__ dst, const uint8_t* __restrict__ src, size_t n) {
    const size_t n16 = n / 16;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16; i += (size_t)gridDim.x * blockDim.x)
        reinterpret_cast<uint4*>(dst)[i] = reinterpret_cast<const uint4*>(src)[i];
    for (size_t i = n16 * 16 + blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
         i += (size_t)gridDim.x * blockDim.x)
        dst[i] = src[i];
}
__global__ void zero_kernel(uint32_t* __restrict__ p, size_t words) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < words; i += (size_t)gridDim.x * blockDim.x)
        p[i] = 0u;
}
int zero_async(void* p, size_t bytes, cudaStream_t s) {  // bytes: a multiple of 4
    if (!t_zero_copy) {
        GSV_CUDA(cudaMemsetAsync(p, 0, bytes, s));
        return GSV_OK;
    }
    zero_kernel<<<(unsigned)std::min<size_t>((bytes / 4 + 255) / 256, 148), 256, 0, s>>>(
        reinterpret_cast<uint32_t*>(p), bytes / 4);
    count_launch();
    GSV_CUDA(cudaGetLastError());
    return GSV_OK;
}

template <class T>
int upload(DevBuf& b, const std::vector<T>& v, cudaStream_t s) {
    int rc = b.alloc(std::max<size_t>(v.size(), 1) * sizeof(T));
    if (rc) return rc;
    if (v.empty()) return GSV_OK;
    const size_t n = v.size() * sizeof(T);
    uint8_t* h = t_stage.reserve(n, s);
    if (h && t_zero_copy) {  // staging and device blocks are 256-B aligned
        memcpy(h, v.data(), n);
        stage_copy_kernel<<<(unsigned)std::min<size_t>((n / 16 + 255) / 256 + 1, 148), 256, 0, s>>>(
            reinterpret_cast<uint8_t*>(b.p), h, n);
        count_launch();
        GSV_CUDA(cudaGetLastError());
    } else if (h) {
        memcpy(h, v.data(), n);
        GSV_CUDA(cudaMemcpyAsync(b.p, h, n, cudaMemcpyHostToDevice, s));
    } else {
        GSV_CUDA(cudaMemcpyAsync(b.p, v.data(), n, cudaMemcpyHostToDevice, s));
    }
    return GSV_OK;
}

uint32_t rd32(const uint8_t* p) {
    uint32_t v;
    memcpy(&v, p, 4);
    return v;
}
uint16_t rd16(const uint8_t* p) {
    uint16_t v;
    memcpy(&v, p, 2);
    return v;
}

// An error candidate in the reference's evaluation order.
struct ErrKey {
    int64_t order = INT64_MAX;  // entry sequence number (group-level checks after the group's entries)
    int phase = 0;              // 0 structure, 1 crc, 2 plane count / valid count
    int kind = GSV_OK;
    std::string msg;
    bool set() const { return kind != GSV_OK; }
    bool before(int64_t o, int ph) const { return !set() || o < order || (o == order && ph < phase); }
};

// Host-side structural parse of one payload blob (codec.py:80-92, 226-258,
// 183-223 minus the decoding itself).  Appends the run's PlaneRefs with
// *offsets* relative to the blob start in `samples`/`coded` (patched to device
// addresses by the caller).  Returns "" or the CodecError message.
struct ParsedRun {
    RunDesc rd{};
    std::vector<PlaneRef> planes;    // pointers hold blob-relative offsets (+1, 0 = none)
    std::vector<uint32_t> rc_plane;  // indices (within planes) of range-coded planes
};

std::string parse_payload(const uint8_t* blob, size_t size, bool check_size, ParsedRun* out) {
    if (size < 14) return "payload header truncated";
    const int codec = blob[0], bits = blob[1];
    const uint32_t w = rd16(blob + 2), h = rd16(blob + 4), count = rd16(blob + 6);
    const uint32_t length = rd32(blob + 10);
    const uint64_t end = 14ull + length + 4ull;
    if (size < end) return "payload body truncated";
    if (check_size && end != size) return "payload size disagrees with directory";
    if (bits != 8 && bits != 16 && bits != 32) return "bad bit width " + std::to_string(bits);
    const uint32_t item = bits / 8;
    const uint64_t hw = (uint64_t)w * h;
    const uint64_t plane_bytes = hw * item;
    const uint64_t expect_raw = (uint64_t)count * plane_bytes;
    if (plane_bytes > 0xFFFFFFFFull) return "plane too large";
    RunDesc& r = out->rd;
    r.checksum = rd32(blob + 14 + length);
    r.plane_bytes = (uint32_t)plane_bytes;
    r.w = (uint16_t)w;
    r.h = (uint16_t)h;
    r.count = (uint16_t)count;
    r.bits = (uint8_t)bits;
    out->planes.clear();
    out->rc_plane.clear();
    const uint64_t body = 14;
    auto raw_run = [&](uint64_t at) {
        r.kind = 0;
        for (uint32_t f = 0; f < count; f++) {
            PlaneRef p{};
            p.samples = reinterpret_cast<const uint8_t*>(at + f * plane_bytes + 1);
            p.f = f;
            p.mode = 1;
            out->planes.push_back(p);
        }
    };
    if (codec == 0) {
        if (length != expect_raw) return "raw body length mismatch";
        raw_run(body);
        return "";
    }
    if (codec == 1) {
        if (length == 0) return "empty reference-coder body";
        const int flag = blob[body];
        const uint64_t coded = body + 1, clen = (uint64_t)length - 1;
        if (flag == 1) {
            if (clen != expect_raw) return "raw fallback length mismatch";
            raw_run(coded);
            return "";
        }
        if (flag != 0) return "unknown body flag " + std::to_string(flag);
        if (clen < count) return "per-plane mode table truncated";
        r.kind = 1;
        uint64_t pos = count;
        for (uint32_t f = 0; f < count; f++) {
            const int mode = blob[coded + f];
            PlaneRef p{};
            p.f = f;
            if (mode == 1) {
                const uint64_t e = pos + plane_bytes;
                if (e > clen) return "raw plane block truncated";
                p.samples = reinterpret_cast<const uint8_t*>(coded + pos + 1);
                p.mode = 1;
                pos = e;
            } else if (mode == 0) {
                if (pos + 4 > clen) return "coded plane length truncated";
                const uint32_t blen = rd32(blob + coded + pos);
                pos += 4;
                const uint64_t e = pos + blen;
                if (e > clen) return "coded plane block truncated";
                p.coded = reinterpret_cast<const uint8_t*>(coded + pos + 1);
                p.coded_len = blen;
                p.mode = 0;
                out->rc_plane.push_back(f);
                pos = e;
            } else {
                return "unknown plane mode " + std::to_string(mode);
            }
            out->planes.push_back(p);
        }
        if (pos != clen) return "trailing bytes after the last plane block";
        return "";
    }
    if (codec == 2) return "external codec payload: no plugin registered";
    return "unknown codec id " + std::to_string(codec);
}

// A set of runs resident on the device, decoded and CRC-checked.
struct RunSet {
    std::vector<RunDesc> runs;
    std::vector<PlaneRef> planes;  // device addresses
    DevBuf d_runs, d_planes, d_planebuf, d_rc, d_chunk, d_crc, d_jobs;
    std::vector<uint32_t> crc;     // computed CRC per run
    std::vector<uint32_t> key;     // channel (attribute << 8 | component) per run: decode order

    // planes of `pr` (blob-relative) -> device addresses at dev_blob; RC outputs
    // are assigned later by finalize().
    void add(ParsedRun& pr, const uint8_t* dev_blob, uint32_t chan = 0) {
        RunDesc r = pr.rd;
        key.push_back(chan);
        r.plane_base = (uint32_t)planes.size();
        const uint32_t run_id = (uint32_t)runs.size();
        for (auto p : pr.planes) {
            if (p.samples) p.samples = dev_blob + (reinterpret_cast<uintptr_t>(p.samples) - 1);
            if (p.coded) p.coded = dev_blob + (reinterpret_cast<uintptr_t>(p.coded) - 1);
            p.run = run_id;
            planes.push_back(p);
        }
        runs.push_back(r);
    }

    uint32_t* hcrc = nullptr;      // pinned read-back of the CRCs (deferred mode)

    // launch() state kept between prepare() and launch()
    std::vector<CopyJob> jobs;
    int n_cls[3] = {0, 0, 0};
    uint32_t nchunks = 0;

    // allocate RC outputs, upload descriptors, decode, CRC, read CRCs back
    // (deferred: the read-back is only enqueued; fetch_crc() after a sync).
    int decode(cudaStream_t s, bool deferred = false) {
        if (int rc = prepare(s)) return rc;
        return launch(s, deferred);
    }
    // descriptors and output storage: host work + small uploads only
    int prepare(cudaStream_t s) {
        // every plane of a range-coded run gets 16-B aligned storage: RC planes
        // are decoded there, RAW planes are copied there (aligned predictors)
        size_t buf = 0;
        std::vector<size_t> off(planes.size(), 0);
        for (size_t i = 0; i < planes.size(); i++) {
            if (runs[planes[i].run].kind == 1) {
                off[i] = buf;
                buf += (runs[planes[i].run].plane_bytes + 15) & ~size_t(15);
            }
        }
        int rc = d_planebuf.alloc(buf + 64);
        if (rc) return rc;
        jobs.clear();
        for (size_t i = 0; i < planes.size(); i++) {
            if (runs[planes[i].run].kind != 1) continue;
            uint8_t* dst = d_planebuf.as<uint8_t>() + off[i];
            if (planes[i].mode == 1)
                jobs.push_back(CopyJob{planes[i].samples, dst, runs[planes[i].run].plane_bytes});
            planes[i].samples = dst;
        }
        if ((rc = upload(d_jobs, jobs, s))) return rc;
        std::vector<uint32_t> rc_runs[3];
        for (size_t i = 0; i < runs.size(); i++) {
            if (runs[i].kind != 1) continue;
            const int nb = runs[i].bits / 8;
            rc_runs[nb == 1 ? 0 : (nb == 2 ? 1 : 2)].push_back((uint32_t)i);
        }
        // lanes of a decoder warp run in lock-step: runs of one channel
        // (same statistics, same fast/slow paths) share warps
        const char* eo = getenv("GSV_RC_ORDER");
        if (!eo || atoi(eo) != 0)
            for (auto& v : rc_runs)
                std::stable_sort(v.begin(), v.end(), [&](uint32_t a, uint32_t b) { return key[a] < key[b]; });
        std::vector<uint32_t> rc_all;
        for (int b = 0; b < 3; b++) rc_all.insert(rc_all.end(), rc_runs[b].begin(), rc_runs[b].end());
        std::vector<uint32_t> chunk_prefix(planes.size() + 1, 0);
        for (size_t i = 0; i < planes.size(); i++) {
            const uint32_t pb = runs[planes[i].run].plane_bytes;
            chunk_prefix[i + 1] = chunk_prefix[i] + (pb + kCrcChunk - 1) / kCrcChunk;
        }
        if ((rc = upload(d_runs, runs, s))) return rc;
        if ((rc = upload(d_planes, planes, s))) return rc;
        if ((rc = upload(d_rc, rc_all, s))) return rc;
        if ((rc = upload(d_chunk, chunk_prefix, s))) return rc;
        if ((rc = d_crc.alloc(std::max<size_t>(runs.size(), 1) * 4))) return rc;
        if ((rc = zero_async(d_crc.p, std::max<size_t>(runs.size(), 1) * 4, s))) return rc;
        for (int b = 0; b < 3; b++) n_cls[b] = (int)rc_runs[b].size();
        nchunks = chunk_prefix.back();
        return GSV_OK;
    }
    // the decode kernels (copy of RAW planes, range decode, CRC) and the CRC
    // read-back; the payload bytes must be on the device by now (stream order)
    int launch(cudaStream_t s, bool deferred) {
        launch_planes(s);
        return launch_check(s, deferred);
    }
    // what rendering needs: RAW planes of range-coded runs copied to aligned
    // storage, range-coded planes decoded
    void launch_planes(cudaStream_t s) {
        prof_mark(ST_RCDEC, s);
        launch_copy_planes(d_jobs.as<CopyJob>(), (int)jobs.size(), s);
        if (!jobs.empty()) count_launch();
        launch_rc_decode(d_runs.as<RunDesc>(), d_rc.as<uint32_t>(), n_cls, d_planes.as<PlaneRef>(), s);
        if (n_cls[0] + n_cls[1] + n_cls[2]) count_launch();
    }
    // validation only: the CRC of every run and its read-back
    int launch_check(cudaStream_t s, bool deferred) {
        prof_mark(ST_CRC, s);
        launch_crc(d_runs.as<RunDesc>(), d_planes.as<PlaneRef>(), (int)planes.size(),
                   d_chunk.as<uint32_t>(), nchunks, d_crc.as<uint32_t>(), s);
        if (nchunks) count_launch();
        prof_mark(ST_COUNT, s);
        crc.assign(runs.size(), 0);
        hcrc = runs.empty() ? nullptr : reinterpret_cast<uint32_t*>(t_stage.reserve(runs.size() * 4, s));
        if (!runs.empty()) {
            if (!hcrc && deferred) return fail(GSV_E_CUDA, "pinned staging unavailable");
            GSV_CUDA(cudaMemcpyAsync(hcrc ? (void*)hcrc : (void*)crc.data(), d_crc.p, runs.size() * 4,
                                     cudaMemcpyDeviceToHost, s));
        }
        GSV_CUDA(cudaGetLastError());
        if (deferred) return GSV_OK;
        GSV_CUDA(cudaStreamSynchronize(s));
        fetch_crc();
        return GSV_OK;
    }
    void fetch_crc() {
        if (hcrc) memcpy(crc.data(), hcrc, runs.size() * 4);
        hcrc = nullptr;
    }
};

}  // namespace

struct gsv_video {
    gsv_session* s = nullptr;
    Container c;
    int k = 0;
    int nslots = 0;
    DevBuf d_payload;             // staged bytes (empty when resident)
    RunSet runs;
    DevBuf d_slots;               // [frame (group-major)][layer][slot]
    std::vector<size_t> frame_base;  // by group-major frame number
    std::vector<std::vector<uint32_t>> layer_off;  // per group prefix sums
    int64_t frame_total = 0;
    // deferred open (gsv_render_sequence_host): errors that need the CRCs are
    // resolved by finish_open() after the stream has drained
    ErrKey stop, pending;
    std::vector<int64_t> run_order;
    // per run (group index as decode_video names it, layer, attribute,
    // component): the error-message prefix, formatted only when needed
    struct RunTag {
        int g, l, attr;
        unsigned comp;
    };
    std::vector<RunTag> run_tag;
};

namespace {
// free the closed videos whose work has completed (or all, waiting, if wait)
void reap_closed(gsv_session* s, bool wait) {
    size_t keep = 0;
    for (size_t i = 0; i < s->graveyard.size(); i++) {
        auto& g = s->graveyard[i];
        if (wait) cudaEventSynchronize(g.first);
        if (wait || cudaEventQuery(g.first) == cudaSuccess) {
            delete g.second;
            s->free_events.push_back(g.first);
        } else {
            s->graveyard[keep++] = g;
        }
    }
    s->graveyard.resize(keep);
    cudaGetLastError();  // cudaEventQuery's cudaErrorNotReady is not an error
}
std::string run_label(const gsv_video::RunTag& t) {
    char nm[96];
    snprintf(nm, sizeof nm, "group %d layer %d channel %s[%u]: ", t.g, t.l + 1, attr_name(t.attr), t.comp);
    return nm;
}
}  // namespace

namespace {

// The error decode_video would raise first (in the reference's order: entry
// sequence, then phase), given the CRCs; GSV_OK when the container is clean.
int finish_open(gsv_video* v) {
    ErrKey best = v->stop;
    if (v->pending.set() && (!best.set() || v->pending.order < best.order ||
                             (v->pending.order == best.order && v->pending.phase < best.phase)))
        best = v->pending;
    for (size_t r = 0; r < v->runs.runs.size(); r++) {
        if (v->runs.crc[r] != v->runs.runs[r].checksum) {
            const int64_t o = v->run_order[r];
            if (!best.set() || o < best.order || (o == best.order && 1 < best.phase))
                best = {o, 1, GSV_E_CODEC, run_label(v->run_tag[r]) + "checksum mismatch (corrupt or truncated payload)"};
            break;  // runs are in order: the first mismatch is the earliest
        }
    }
    if (best.set()) return fail(best.kind, best.msg);
    return GSV_OK;
}

// deferred: nothing synchronises -- the decode, CRC, table uploads and the
// CRC read-back are enqueued on the session stream, the pinned staging is not
// reset (the caller resets it once it has drained the stream), frame tables
// are built whatever the CRCs say, and finish_open() reports the error after
// a sync.  Structural errors found on the host still fail at once.
// prepare_only (implies deferred): host work and descriptor uploads only;
// open_launch() enqueues the decode kernels later, once the payload bytes have
// been uploaded (gsv_render_sequence_host enqueues every group's descriptor
// uploads before the big payload uploads, so they never queue behind them).
int open_video(gsv_session* s, const uint8_t* data, size_t len, const uint8_t* dev_data,
               int up_to_layer, gsv_video** out, const std::vector<int>* sel = nullptr, bool deferred = false,
               bool prepare_only = false) {
    if (prepare_only) deferred = true;
    reap_closed(s, false);
    *out = nullptr;
    if (!deferred) t_stage.reset();
    static const bool dbg_t = getenv("GSV_DEBUG_OPEN_TIMING") != nullptr;  // dev: phase times to stderr
    auto T = [&](const char* what) {
        static thread_local std::chrono::steady_clock::time_point last;
        const auto now = std::chrono::steady_clock::now();
        if (dbg_t && what) fprintf(stderr, "[open] %s %.2f ms\n", what,
                                   std::chrono::duration<double, std::milli>(now - last).count());
        last = now;
    };
    T(nullptr);
    gsv_video* v = new gsv_video();
    v->s = s;
    auto bail = [&](int rc) {
        delete v;
        return rc;
    };
    int rc = parse_container(data, len, &v->c);
    if (rc) return bail(rc);
    // container index of each opened group (error messages name the group as
    // decode_video of the whole container would)
    std::vector<int> gidx(v->c.groups.size());
    for (size_t g = 0; g < gidx.size(); g++) gidx[g] = (int)g;
    if (sel) gidx = *sel;
    if (sel) {  // keep the selected groups only, in list order (only their bytes are staged)
        const int G0 = (int)v->c.groups.size();
        if (sel->empty()) return bail(fail(GSV_E_INVALID_INPUT, "empty group list"));
        std::vector<char> seen(G0, 0);
        std::vector<GroupDir> keep;
        for (int g : *sel) {
            if (g < 0 || g >= G0)
                return bail(fail(GSV_E_INVALID_INPUT,
                                 "group " + std::to_string(g) + " out of range 0.." + std::to_string(G0 - 1)));
            if (seen[g]) return bail(fail(GSV_E_INVALID_INPUT, "group " + std::to_string(g) + " listed twice"));
            seen[g] = 1;
            keep.push_back(v->c.groups[g]);
        }
        uint32_t next = 0;  // frames numbered from 0, group after group in list order
        for (GroupDir& gd : keep) {
            gd.start_frame = next;
            next += gd.frame_count;
        }
        v->c.groups = std::move(keep);
    }
    const Container& c = v->c;
    const int L = c.layer_count;
    const int k = up_to_layer == -1 ? L : up_to_layer;
    if (k < 1 || k > L) {
        return bail(fail(GSV_E_INVALID_INPUT, "layer " + std::to_string(up_to_layer) + " out of range 1.." +
                                                  std::to_string(L)));
    }
    if (k > kMaxLayers) return bail(fail(GSV_E_INVALID_INPUT, "more than 64 layers decoded"));
    v->k = k;
    cudaStream_t st = s->stream;

    // ---- stage the layer-prefix bytes of every group -----------------------
    const int G = (int)c.groups.size();
    std::vector<uint64_t> lo(G, 0), hi(G, 0), dev_base(G, 0);
    uint64_t total = 0;
    for (int g = 0; g < G; g++) {
        bool any = false;
        for (int l = 0; l < k; l++)
            for (const Entry& e : c.groups[g].channels[l]) {
                if (e.offset >= len) continue;
                const uint64_t end = e.size > len - e.offset ? len : e.offset + e.size;
                if (!any) {
                    lo[g] = e.offset;
                    hi[g] = end;
                    any = true;
                } else {
                    lo[g] = std::min(lo[g], e.offset);
                    hi[g] = std::max(hi[g], end);
                }
            }
        dev_base[g] = total;
        total += ((hi[g] - lo[g]) + 15) & ~15ull;
    }
    if (!dev_data) {
        if ((rc = v->d_payload.alloc(total + 64))) return bail(rc);
        for (int g = 0; g < G; g++)
            if (hi[g] > lo[g])
                GSV_CUDA(cudaMemcpyAsync(v->d_payload.as<uint8_t>() + dev_base[g], data + lo[g], hi[g] - lo[g],
                                         cudaMemcpyHostToDevice, st));
    }
    auto dev_addr = [&](int g, uint64_t off) -> const uint8_t* {
        if (dev_data) return dev_data + off;
        return v->d_payload.as<uint8_t>() + dev_base[g] + (off - lo[g]);
    };

    T("parse+stage");
    // ---- walk entries in the reference's order ----------------------------
    const int shdim_ok = c.sh_degree <= 3;
    const int shdim = shdim_ok ? 3 * (c.sh_degree + 1) * (c.sh_degree + 1) : 0;
    v->nslots = 11 + shdim;
    ErrKey& stop = v->stop;        // first structural / group-level error (walk stops there)
    ErrKey& pending = v->pending;  // first post-CRC error (plane count, valid count)
    std::vector<int64_t>& run_order = v->run_order;      // entry sequence number of each run
    std::vector<gsv_video::RunTag>& run_tag = v->run_tag;  // "group g layer l channel a[c]"
    struct SlotRef { int run = -1; const Entry* e = nullptr; };
    std::vector<std::vector<std::vector<SlotRef>>> slots(G);
    int64_t seq = 0;
    ParsedRun pr;
    for (int g = 0; g < G && !stop.set(); g++) {
        const GroupDir& gd = c.groups[g];
        slots[g].assign(k, std::vector<SlotRef>(v->nslots));
        for (int l = 0; l < k && !stop.set(); l++) {
            const uint32_t n_l = gd.layer_counts[l];
            for (const Entry& e : gd.channels[l]) {
                const int64_t o = seq++;
                const gsv_video::RunTag tag{gidx[g], l, (int)e.attr, (unsigned)e.comp};
                if (e.offset > len || e.size > len - e.offset) {
                    stop = {o, 0, GSV_E_FORMAT,
                            "unexpected end of container (wanted " + std::to_string(e.size) + " bytes)"};
                    break;
                }
                std::string m = parse_payload(data + e.offset, e.size, true, &pr);
                if (!m.empty()) {
                    stop = {o, 0, GSV_E_CODEC, run_label(tag) + m};
                    break;
                }
                const int run_id = (int)v->runs.runs.size();
                v->runs.add(pr, dev_addr(g, e.offset), (uint32_t)e.attr << 8 | e.comp);
                run_order.push_back(o);
                run_tag.push_back(tag);
                if (pr.rd.count != gd.frame_count) {
                    if (pending.before(o, 2))
                        pending = {o, 2, GSV_E_FORMAT,
                                   run_label(tag) + "expected " + std::to_string(gd.frame_count) +
                                       " planes, got " + std::to_string(pr.rd.count)};
                } else if (!(n_l > 0 && (uint64_t)n_l <= (uint64_t)pr.rd.w * pr.rd.h)) {
                    if (pending.before(o, 2)) pending = {o, 2, GSV_E_INVALID_INPUT, "valid_count out of range"};
                }
                const int sl = shdim_ok ? slot_of(e.attr, e.comp, shdim) : -1;
                if (sl >= 0) slots[g][l][sl] = {run_id, &e};  // later duplicates win (dict semantics)
            }
        }
        if (stop.set()) break;
        const int64_t o = seq++;  // _assemble_frames of group g
        if (!shdim_ok) {
            stop = {o, 0, GSV_E_INVALID_INPUT, "sh_degree must be 0..3, got " + std::to_string(c.sh_degree)};
            break;
        }
        if (gd.frame_count >= 1) {
            for (int l = 0; l < k && !stop.set(); l++)
                for (int sl = 0; sl < v->nslots; sl++)
                    if (slots[g][l][sl].run < 0) {
                        static const char* an[] = {"position", "rotation", "scales", "opacity", "sh"};
                        int attr, comp;
                        if (sl < 3) { attr = 0; comp = sl; }
                        else if (sl < 7) { attr = 1; comp = sl - 3; }
                        else if (sl < 10) { attr = 2; comp = sl - 7; }
                        else if (sl == 10) { attr = 3; comp = 0; }
                        else { attr = 4; comp = sl - 11; }
                        stop = {o, 0, GSV_E_FORMAT, std::string("missing channel ") + an[attr] + "[" +
                                                        std::to_string(comp) + "]"};
                        break;
                    }
        }
    }

    T("walk");
    // a structural error stops the walk: decode_video raises it unless an
    // earlier entry's CRC fails, so such an open is resolved synchronously
    if (stop.set()) deferred = prepare_only = false;
    // ---- decode + CRC on the GPU ------------------------------------------
    if (prepare_only) {
        if ((rc = v->runs.prepare(st))) return bail(rc);
    } else if ((rc = v->runs.decode(st, deferred))) {
        return bail(rc);
    }
    T("decode+crc");
    if (!deferred && (rc = finish_open(v))) return bail(rc);

    // ---- frame tables: per frame, per layer, per slot the resolved plane ----
    std::vector<SlotDesc> sd;
    v->frame_base.clear();
    v->layer_off.resize(G);
    for (int g = 0; g < G; g++) {
        auto& lo2 = v->layer_off[g];
        lo2.assign(k + 1, 0);
        for (int l = 0; l < k; l++) lo2[l + 1] = lo2[l] + c.groups[g].layer_counts[l];
        v->frame_total += c.groups[g].frame_count;
    }
    for (int g = 0; g < G; g++) {
        for (int f = 0; f < c.groups[g].frame_count; f++) {
            v->frame_base.push_back(sd.size());
            for (int l = 0; l < k; l++)
                for (int sl = 0; sl < v->nslots; sl++) {
                    SlotDesc d{};
                    const SlotRef& ref = slots[g][l][sl];
                    if (ref.run >= 0) {
                        const RunDesc& rd = v->runs.runs[ref.run];
                        d.samples = v->runs.planes[rd.plane_base + f].samples;
                        d.rmin = (double)ref.e->rmin;
                        d.span = (double)ref.e->rmax - (double)ref.e->rmin;
                        d.dir_bits = ref.e->bits;
                        d.bits = rd.bits;
                    }
                    sd.push_back(d);
                }
        }
    }
    T("frame tables");
    if ((rc = upload(v->d_slots, sd, st))) return bail(rc);
    if (!deferred) GSV_CUDA(cudaStreamSynchronize(st));
    T("upload");
    *out = v;
    return GSV_OK;
}

int frame_src(gsv_video* v, int t, FrameSrc* src) {
    const Container& c = v->c;
    for (size_t g = 0; g < c.groups.size(); g++) {
        const GroupDir& gd = c.groups[g];
        if ((int64_t)gd.start_frame <= t && t < (int64_t)gd.start_frame + gd.frame_count) {
            memset(src, 0, sizeof *src);
            size_t fi = 0;  // group-major frame number of (g, t - start)
            for (size_t h = 0; h < g; h++) fi += c.groups[h].frame_count;
            src->slots = v->d_slots.as<SlotDesc>() + v->frame_base[fi + (t - gd.start_frame)];
            src->nlayers = v->k;
            src->nslots = v->nslots;
            src->sh_degree = c.sh_degree;
            for (int l = 0; l <= v->k; l++) src->layer_off[l] = v->layer_off[g][l];
            return GSV_OK;
        }
    }
    return fail(GSV_E_INVALID_INPUT,
                "frame " + std::to_string(t) + " out of range 0.." + std::to_string(v->frame_total - 1));
}

}  // namespace

extern "C" {

int gsv_session_create(int device, uintptr_t stream, gsv_session** out) {
    *out = nullptr;
    GSV_CUDA(cudaSetDevice(device));
    gsv_session* s = new gsv_session();
    s->device = device;
    if (stream) {
        s->stream = reinterpret_cast<cudaStream_t>(stream);
    } else {
        cudaError_t e = cudaStreamCreateWithFlags(&s->stream, cudaStreamNonBlocking);
        if (e != cudaSuccess) {
            delete s;
            return fail(GSV_E_CUDA, std::string("cudaStreamCreate: ") + cudaGetErrorString(e));
        }
        s->own_stream = true;
    }
    *out = s;
    return GSV_OK;
}

void gsv_session_destroy(gsv_session* s) {
    if (!s) return;
    cudaSetDevice(s->device);
    cudaStreamSynchronize(s->stream);
    reap_closed(s, true);
    for (cudaEvent_t e : s->free_events) cudaEventDestroy(e);
    for (size_t i = 0; i < s->aux.size(); i++) {
        cudaStreamSynchronize(s->aux[i]);
        cudaStreamSynchronize(s->aux_copy[i]);
        work_free(s->aux_work[i]);
        delete s->aux_work[i];
        for (int b = 0; b < kU8Bufs; b++) {
            if (s->aux_u8[kU8Bufs * i + b]) cudaFree(s->aux_u8[kU8Bufs * i + b]);
            cudaEventDestroy(s->ev_rendered[kU8Bufs * i + b]);
            cudaEventDestroy(s->ev_copied[kU8Bufs * i + b]);
        }
        cudaStreamDestroy(s->aux[i]);
        cudaStreamDestroy(s->aux_copy[i]);
        cudaEventDestroy(s->ev_join[i]);
        cudaEventDestroy(s->ev_copy_join[i]);
    }
    if (s->ev_fork) cudaEventDestroy(s->ev_fork);
    if (s->copy_in) {
        cudaStreamSynchronize(s->copy_in);
        cudaStreamDestroy(s->copy_in);
    }
    if (s->check) {
        cudaStreamSynchronize(s->check);
        cudaStreamDestroy(s->check);
    }
    if (s->ev_prep) cudaEventDestroy(s->ev_prep);
    for (cudaEvent_t e : s->ev_up) cudaEventDestroy(e);
    for (cudaEvent_t e : s->ev_plane) cudaEventDestroy(e);
    for (uint8_t* p : s->seq_slot)
        if (p) cudaFree(p);
    for (cudaEvent_t e : s->ev_slot_done) cudaEventDestroy(e);
    work_free(&s->work);
    if (s->own_stream) cudaStreamDestroy(s->stream);
    delete s;
}

long long gsv_kernel_launches(void) { return __atomic_load_n(&gsv::g_launches, __ATOMIC_RELAXED); }

int gsv_profile_enable(int enable) {
    gsv::prof_enable(enable != 0);
    return GSV_OK;
}

int gsv_profile_read(double* ms, long long* marks, int max_stages) {
    return gsv::prof_read(ms, marks, max_stages);
}

int gsv_session_sync(gsv_session* s) {
    GSV_CUDA(cudaStreamSynchronize(s->stream));
    return GSV_OK;
}

int gsv_video_open(gsv_session* s, const uint8_t* data, size_t len, int up_to_layer, gsv_video** out) {
    GSV_CUDA(cudaSetDevice(s->device));
    return open_video(s, data, len, nullptr, up_to_layer, out);
}

int gsv_video_open_resident(gsv_session* s, const uint8_t* data, size_t len, const uint8_t* dev_data,
                            int up_to_layer, gsv_video** out) {
    GSV_CUDA(cudaSetDevice(s->device));
    if (!dev_data) return fail(GSV_E_INVALID_INPUT, "dev_data is NULL");
    return open_video(s, data, len, dev_data, up_to_layer, out);
}

int gsv_video_open_groups(gsv_session* s, const uint8_t* data, size_t len, int up_to_layer, int g0, int g1,
                          gsv_video** out) {
    GSV_CUDA(cudaSetDevice(s->device));
    *out = nullptr;
    gsv_info info;
    if (int rc = gsv_read_info(data, len, &info)) return rc;
    if (g0 < 0 || g1 > info.group_count || g0 >= g1)
        return fail(GSV_E_INVALID_INPUT, "group range [" + std::to_string(g0) + ", " + std::to_string(g1) +
                                             ") out of range 0.." + std::to_string(info.group_count));
    std::vector<int> sel;
    for (int g = g0; g < g1; g++) sel.push_back(g);
    return open_video(s, data, len, nullptr, up_to_layer, out, &sel);
}

int gsv_video_open_group_list(gsv_session* s, const uint8_t* data, size_t len, const uint8_t* dev_data,
                              int up_to_layer, const int32_t* groups, int ngroups, gsv_video** out) {
    GSV_CUDA(cudaSetDevice(s->device));
    *out = nullptr;
    if (ngroups < 0 || (ngroups > 0 && !groups)) return fail(GSV_E_INVALID_INPUT, "invalid group list");
    std::vector<int> sel(groups, groups + ngroups);
    return open_video(s, data, len, dev_data, up_to_layer, out, &sel);
}


void gsv_video_close(gsv_video* v) {
    if (!v) return;
    gsv_session* s = v->s;
    cudaEvent_t e = nullptr;
    if (!s->free_events.empty()) {
        e = s->free_events.back();
        s->free_events.pop_back();
    } else if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) {
        e = nullptr;
    }
    if (!e || cudaEventRecord(e, s->stream) != cudaSuccess) {  // fall back to a synchronous close
        if (e) s->free_events.push_back(e);
        cudaGetLastError();
        cudaStreamSynchronize(s->stream);
        delete v;
        return;
    }
    s->graveyard.emplace_back(e, v);
    reap_closed(s, false);
}

int gsv_video_frame_count(const gsv_video* v) { return (int)v->frame_total; }
int gsv_video_decoded_layers(const gsv_video* v) { return v->k; }

int gsv_video_group_of(const gsv_video* v, int t) {
    for (size_t g = 0; g < v->c.groups.size(); g++) {
        const GroupDir& gd = v->c.groups[g];
        if ((int64_t)gd.start_frame <= t && t < (int64_t)gd.start_frame + gd.frame_count) return (int)g;
    }
    return -1;
}

int64_t gsv_video_group_splats(const gsv_video* v, int g) {
    if (g < 0 || g >= (int)v->layer_off.size()) return -1;
    return v->layer_off[g][v->k];
}

int gsv_video_frame_values(gsv_video* v, int t, double* pos, double* rot, double* scl, double* opac,
                           double* sh) {
    FrameSrc src;
    int rc = frame_src(v, t, &src);
    if (rc) return rc;
    launch_dequant_frame(src, pos, rot, scl, opac, sh, v->s->stream);
    count_launch();
    GSV_CUDA(cudaGetLastError());
    return GSV_OK;
}

int gsv_video_frame_codes(gsv_video* v, int t, uint32_t* out) {
    FrameSrc src;
    int rc = frame_src(v, t, &src);
    if (rc) return rc;
    launch_frame_codes(src, out, v->s->stream);
    count_launch();
    GSV_CUDA(cudaGetLastError());
    return GSV_OK;
}

int gsv_video_render(gsv_video* v, int t, const gsv_camera* cam, float* out_rgb, uint8_t* out_rgb8,
                     gsv_render_stats* stats) {
    FrameSrc src;
    int rc = frame_src(v, t, &src);
    if (rc) return rc;
    if (cam->width < 1 || cam->height < 1) return fail(GSV_E_INVALID_INPUT, "image dimensions must be >= 1");
    return render_planes(src, make_cam(*cam), &v->s->work, out_rgb, out_rgb8, stats, v->s->stream);
}

namespace {

// Aux streams, their workspaces, u8 staging buffers and events for
// frame-parallel rendering (created on first use, grown on demand).
int ensure_aux(gsv_session* s, int nstreams, size_t img8, bool host_out) {
    while ((int)s->aux.size() < nstreams) {
        cudaStream_t st;
        GSV_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
        cudaEvent_t e;
        GSV_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        s->aux.push_back(st);
        s->aux_work.push_back(new RenderWork());
        s->ev_join.push_back(e);
        cudaStream_t cs;
        GSV_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
        s->aux_copy.push_back(cs);
        cudaEvent_t cj;
        GSV_CUDA(cudaEventCreateWithFlags(&cj, cudaEventDisableTiming));
        s->ev_copy_join.push_back(cj);
        s->aux_flip.push_back(0);
        for (int b = 0; b < kU8Bufs; b++) {
            s->aux_u8.push_back(nullptr);
            s->aux_u8_cap.push_back(0);
            cudaEvent_t er, ec;
            GSV_CUDA(cudaEventCreateWithFlags(&er, cudaEventDisableTiming));
            GSV_CUDA(cudaEventCreateWithFlags(&ec, cudaEventDisableTiming));
            GSV_CUDA(cudaEventRecord(ec, cs));  // buffer free
            s->ev_rendered.push_back(er);
            s->ev_copied.push_back(ec);
        }
    }
    if (!s->ev_fork) GSV_CUDA(cudaEventCreateWithFlags(&s->ev_fork, cudaEventDisableTiming));
    const int64_t khint = std::max(s->kcap_hint, s->work.cap_k);
    for (int i = 0; i < nstreams; i++) {
        if (s->aux_work[i]->cap_k < khint) {
            int rc = work_reserve(s->aux_work[i], 1, khint, 0, 0);
            if (rc) return rc;
        }
        for (int b = 0; b < kU8Bufs && host_out; b++) {
            const int q = kU8Bufs * i + b;
            if (s->aux_u8_cap[q] < img8) {
                GSV_CUDA(cudaStreamSynchronize(s->aux_copy[i]));
                if (s->aux_u8[q]) cudaFree(s->aux_u8[q]);
                GSV_CUDA(cudaMalloc(&s->aux_u8[q], img8));
                s->aux_u8_cap[q] = img8;
            }
        }
    }
    return GSV_OK;
}

// Enqueue frames[0..count) of v on the aux streams (frame j on stream
// (first + j) % nstreams), forked from the session stream; host_rgb8 outputs
// go through the per-stream double-buffered u8 staging and a copy stream.
// Nothing is joined back into the session stream.
int enqueue_frames(gsv_video* v, const int32_t* frames, int count, const CamDev& cd, size_t img8,
                   float* const* out_rgb, uint8_t* const* out_rgb8, uint8_t* const* host_rgb8, int nstreams,
                   int first, const cudaEvent_t* frame_ready = nullptr) {
    gsv_session* s = v->s;
    GSV_CUDA(cudaEventRecord(s->ev_fork, s->stream));
    for (int i = 0; i < nstreams; i++) GSV_CUDA(cudaStreamWaitEvent(s->aux[i], s->ev_fork, 0));
    for (int j = 0; j < count; j++) {
        const int i = (first + j) % nstreams;
        if (frame_ready) GSV_CUDA(cudaStreamWaitEvent(s->aux[i], frame_ready[j], 0));  // its planes landed
        FrameSrc src;
        int rc = frame_src(v, frames[j], &src);
        if (rc) return rc;
        uint8_t* o8 = out_rgb8 ? out_rgb8[j] : nullptr;
        const bool to_host = host_rgb8 && host_rgb8[j];
        int q = 0;
        if (to_host) {
            q = kU8Bufs * i + s->aux_flip[i];
            s->aux_flip[i] = (s->aux_flip[i] + 1) % kU8Bufs;
            GSV_CUDA(cudaStreamWaitEvent(s->aux[i], s->ev_copied[q], 0));  // staging buffer free
            o8 = s->aux_u8[q];
        }
        rc = render_planes(src, cd, s->aux_work[i], out_rgb ? out_rgb[j] : nullptr, o8,
                           reinterpret_cast<gsv_render_stats*>(1), s->aux[i]);
        if (rc) return rc;
        if (to_host) {
            GSV_CUDA(cudaEventRecord(s->ev_rendered[q], s->aux[i]));
            GSV_CUDA(cudaStreamWaitEvent(s->aux_copy[i], s->ev_rendered[q], 0));
            GSV_CUDA(cudaMemcpyAsync(host_rgb8[j], o8, img8, cudaMemcpyDeviceToHost, s->aux_copy[i]));
            GSV_CUDA(cudaEventRecord(s->ev_copied[q], s->aux_copy[i]));
        }
    }
    return GSV_OK;
}

// Counters of every aux workspace read back, and the aux (and copy) streams
// joined into the session stream.
int join_aux(gsv_session* s, int nstreams, bool host_out) {
    for (int i = 0; i < nstreams; i++) {
        if (int rc = readback_counters(s->aux_work[i], s->aux[i])) return rc;
        GSV_CUDA(cudaEventRecord(s->ev_join[i], s->aux[i]));
        GSV_CUDA(cudaStreamWaitEvent(s->stream, s->ev_join[i], 0));
        if (host_out) {
            GSV_CUDA(cudaEventRecord(s->ev_copy_join[i], s->aux_copy[i]));
            GSV_CUDA(cudaStreamWaitEvent(s->stream, s->ev_copy_join[i], 0));
        }
    }
    return GSV_OK;
}

// After a synchronised batch: the largest key count any aux workspace needed
// beyond its capacity (0: every frame fitted).
int64_t aux_key_overflow(gsv_session* s, int nstreams) {
    int64_t need = 0;
    for (int i = 0; i < nstreams; i++) {
        RenderWork* w = s->aux_work[i];
        if (w->h_ctr && (int64_t)w->h_ctr[9] > w->cap_k) need = std::max(need, (int64_t)w->h_ctr[9]);
    }
    return need;
}

}  // namespace

int gsv_video_render_batch(gsv_video* v, const int32_t* frames, int count, const gsv_camera* cam,
                           float* const* out_rgb, uint8_t* const* out_rgb8, uint8_t* const* host_rgb8,
                           int nstreams, int check) {
    gsv_session* s = v->s;
    if (count <= 0) return GSV_OK;
    if (cam->width < 1 || cam->height < 1) return fail(GSV_E_INVALID_INPUT, "image dimensions must be >= 1");
    nstreams = std::max(1, std::min(nstreams, 32));
    const CamDev cd = make_cam(*cam);
    const size_t img8 = (size_t)cam->width * cam->height * 3;
    for (int attempt = 0; attempt < 4; attempt++) {
        if (int rc = ensure_aux(s, nstreams, img8, host_rgb8 != nullptr)) return rc;
        if (int rc = enqueue_frames(v, frames, count, cd, img8, out_rgb, out_rgb8, host_rgb8, nstreams, 0)) return rc;
        if (int rc = join_aux(s, nstreams, host_rgb8 != nullptr)) return rc;
        if (!check) return GSV_OK;
        GSV_CUDA(cudaStreamSynchronize(s->stream));
        const int64_t need = aux_key_overflow(s, nstreams);
        if (need == 0) return GSV_OK;
        s->kcap_hint = need + need / 4 + 1024;  // grow and render the batch again
    }
    return fail(GSV_E_NOMEM, "tile key buffer could not be sized");
}

// ---------------------------------------------------------------------------
// Decode + render a whole sequence from host bytes into host u8 frames: the
// reference's decode_video + render_set + write_ppm of every frame
// (pipeline.py:350-359, render.py:382-385, 165-169; cli.py:122-131 per frame)
// as one pipelined call.  Raw groups (codec 0, or codec 1's whole-run raw
// fallback) go through a ring of kSeqSlots device slots: group g's
// layer-prefix bytes are uploaded on the copy stream while earlier groups
// render, its runs are opened (CRC enqueued, not waited for) on the session
// stream once they have landed, and its frames render on the aux streams with
// their read-back; nothing on the host waits until the end, where every
// group's CRC is checked and the first error in decode order is returned
// (the frames written so far are then undefined, as decode_video would have
// raised before rendering).  Sequences with range-coded runs are opened whole
// (every run of every group decodes in parallel) and then rendered.
// ---------------------------------------------------------------------------
namespace {
constexpr int kSeqSlots = 3;

struct VideoList {
    std::vector<gsv_video*> v;
    ~VideoList() {
        for (gsv_video* x : v) delete x;
    }
};

// Plane-major upload of a raw group: its runs of one sample width in one
// layer follow each other with a constant stride in the container (header,
// count x plane, CRC), so plane f of all of them is one 2-D copy.  Returns
// the copies grouped by plane (empty when the layout is not regular).
struct PlaneCopy {
    uint64_t src_off;  // container offset of plane f of the first run
    uint64_t pitch, width, height;
};
std::vector<std::vector<PlaneCopy>> plane_major_plan(const uint8_t* data, const GroupDir& gd, int k) {
    const int F = gd.frame_count;
    std::vector<std::vector<PlaneCopy>> plan(F);
    for (int l = 0; l < k; l++) {
        const auto& ents = gd.channels[l];
        size_t i = 0;
        while (i < ents.size()) {
            const uint8_t* b = data + ents[i].offset;
            const uint64_t hdr = b[0] == 0 ? 14 : 15;  // codec 0 body / codec 1 raw-fallback body
            const uint64_t pb = (uint64_t)rd16(b + 2) * rd16(b + 4) * (b[1] / 8);
            // the longest run of entries with the same layout at a constant stride
            size_t j = i + 1;
            uint64_t stride = 0;
            while (j < ents.size()) {
                const uint8_t* c = data + ents[j].offset;
                const uint64_t hj = c[0] == 0 ? 14 : 15;
                const uint64_t pj = (uint64_t)rd16(c + 2) * rd16(c + 4) * (c[1] / 8);
                const uint64_t st = ents[j].offset - ents[j - 1].offset;
                if (hj != hdr || pj != pb || (j > i + 1 && st != stride) || ents[j].offset < ents[j - 1].offset)
                    break;
                stride = st;
                j++;
            }
            if (j == i + 1) stride = pb;  // a single run: the pitch is irrelevant
            if (stride < pb) return {};
            for (int f = 0; f < F; f++)
                plan[f].push_back(PlaneCopy{ents[i].offset + hdr + (uint64_t)f * pb, stride, pb, (uint64_t)(j - i)});
            i = j;
        }
    }
    return plan;
}

bool group_is_raw(const uint8_t* data, size_t len, const GroupDir& gd, int k) {
    for (int l = 0; l < k; l++)
        for (const Entry& e : gd.channels[l]) {
            if (e.offset > len || e.size > len - e.offset || e.size < 15) return false;
            const uint8_t* b = data + e.offset;
            if (!(b[0] == 0 || (b[0] == 1 && b[14] == 1))) return false;
        }
    return true;
}
}  // namespace

int gsv_render_sequence_host(gsv_session* s, const uint8_t* data, size_t len, int up_to_layer,
                             const int32_t* groups, int ngroups, const gsv_camera* cam,
                             uint8_t* const* host_rgb8, int nstreams, int64_t* frames_out) {
    if (!host_rgb8) return fail(GSV_E_INVALID_INPUT, "host_rgb8 is NULL");
    return gsv_render_sequence(s, data, len, nullptr, up_to_layer, groups, ngroups, nullptr, nullptr, cam, nullptr,
                               nullptr, host_rgb8, nstreams, frames_out);
}

int gsv_render_sequence(gsv_session* s, const uint8_t* data, size_t len, const uint8_t* dev_data, int up_to_layer,
                        const int32_t* groups, int ngroups, const int32_t* frame_begin, const int32_t* frame_end,
                        const gsv_camera* cam, float* const* out_rgb, uint8_t* const* out_rgb8,
                        uint8_t* const* host_rgb8, int nstreams, int64_t* frames_out) {
    const auto t_entry = std::chrono::steady_clock::now();
    GSV_CUDA(cudaSetDevice(s->device));
    if (frames_out) *frames_out = 0;
    if (!out_rgb && !out_rgb8 && !host_rgb8) return fail(GSV_E_INVALID_INPUT, "no output array given");
    const bool host_out = host_rgb8 != nullptr;
    const bool resident = dev_data != nullptr;
    if (cam->width < 1 || cam->height < 1) return fail(GSV_E_INVALID_INPUT, "image dimensions must be >= 1");
    nstreams = std::max(1, std::min(nstreams, 32));
    Container c;
    if (int rc = parse_container(data, len, &c)) return rc;
    std::vector<int> sel;
    if (groups && ngroups > 0) sel.assign(groups, groups + ngroups);
    else
        for (int g = 0; g < (int)c.groups.size(); g++) sel.push_back(g);
    std::vector<char> seen(c.groups.size(), 0);
    for (int g : sel) {
        if (g < 0 || g >= (int)c.groups.size())
            return fail(GSV_E_INVALID_INPUT, "group " + std::to_string(g) + " out of range 0.." +
                                                 std::to_string((int)c.groups.size() - 1));
        if (seen[g]++) return fail(GSV_E_INVALID_INPUT, "group " + std::to_string(g) + " listed twice");
    }
    // frames [fb, fe) of each listed group (group-relative; all by default)
    std::vector<int32_t> fb(sel.size(), 0), fe(sel.size(), 0);
    for (size_t gi = 0; gi < sel.size(); gi++) {
        const int fc = c.groups[sel[gi]].frame_count;
        fb[gi] = frame_begin ? frame_begin[gi] : 0;
        fe[gi] = frame_end ? frame_end[gi] : fc;
        if (fb[gi] < 0 || fe[gi] > fc || fb[gi] >= fe[gi])
            return fail(GSV_E_INVALID_INPUT, "frames [" + std::to_string(fb[gi]) + ", " + std::to_string(fe[gi]) +
                                                 ") out of range for group " + std::to_string(sel[gi]) +
                                                 " (0.." + std::to_string(fc) + ")");
    }
    const int L = c.layer_count;
    const int k = up_to_layer == -1 ? L : up_to_layer;
    if (k < 1 || k > L)
        return fail(GSV_E_INVALID_INPUT,
                    "layer " + std::to_string(up_to_layer) + " out of range 1.." + std::to_string(L));
    const CamDev cd = make_cam(*cam);
    const size_t img8 = (size_t)cam->width * cam->height * 3;
    bool raw = true;
    for (int g : sel) raw = raw && group_is_raw(data, len, c.groups[g], k);

    if (!raw || sel.size() < 2) {
        gsv_video* v = nullptr;
        if (int rc = open_video(s, data, len, dev_data, k, &v, &sel)) return rc;
        std::vector<int32_t> fr;  // the video numbers frames group after group in list order
        int32_t base = 0;
        for (size_t gi = 0; gi < sel.size(); gi++) {
            for (int32_t f = fb[gi]; f < fe[gi]; f++) fr.push_back(base + f);
            base += c.groups[sel[gi]].frame_count;
        }
        int rc = gsv_video_render_batch(v, fr.data(), (int)fr.size(), cam, out_rgb, out_rgb8, host_rgb8, nstreams, 1);
        cudaStreamSynchronize(s->stream);
        if (!rc && frames_out) *frames_out = (int64_t)fr.size();
        delete v;
        return rc;
    }

    // ---- raw groups: the upload / open / render pipeline -------------------
    const int G = (int)sel.size();
    std::vector<uint64_t> lo(G, 0), hi(G, 0);
    uint64_t slot_bytes = 0;
    for (int gi = 0; gi < G; gi++) {
        bool any = false;
        for (int l = 0; l < k; l++)
            for (const Entry& e : c.groups[sel[gi]].channels[l]) {
                const uint64_t end = e.offset + e.size;  // in range: group_is_raw checked it
                lo[gi] = any ? std::min(lo[gi], e.offset) : e.offset;
                hi[gi] = any ? std::max(hi[gi], end) : end;
                any = true;
            }
        slot_bytes = std::max(slot_bytes, hi[gi] - lo[gi]);
    }
    // Every group gets its own slot when the prefix bytes fit comfortably in
    // HBM (a quarter of the free memory): then all uploads are enqueued before
    // any render, so the copy engine streams the container at PCIe rate no
    // matter how far the host's render enqueue runs ahead.  Otherwise a ring
    // of kSeqSlots slots, each reused once its group has rendered.
    uint64_t total = 0;
    for (int gi = 0; gi < G; gi++) total += ((hi[gi] - lo[gi]) + 255) & ~255ull;
    // free HBM: queried only when the slots the session already holds are
    // too small (cudaMemGetInfo can take milliseconds while copies run)
    uint64_t held = 0;
    for (size_t r = 0; r < s->seq_slot_cap.size() && r < (size_t)G; r++) held += s->seq_slot_cap[r];
    size_t mfree = 0, mtot = 0;
    if (!resident && held < total) cudaMemGetInfo(&mfree, &mtot);
    const char* ring_env = getenv("GSV_SEQ_RING");  // tests: force the ring of slots
    const bool fits = held >= total || total <= (held + mfree) / 4;
    const bool all_slots = resident || (fits && !(ring_env && atoi(ring_env) != 0));
    const int R = all_slots ? G : std::min(kSeqSlots, G);
    if (!s->copy_in) GSV_CUDA(cudaStreamCreateWithFlags(&s->copy_in, cudaStreamNonBlocking));
    if (!s->check) GSV_CUDA(cudaStreamCreateWithFlags(&s->check, cudaStreamNonBlocking));
    if (!s->ev_prep) GSV_CUDA(cudaEventCreateWithFlags(&s->ev_prep, cudaEventDisableTiming));
    while ((int)s->ev_up.size() < R) {
        cudaEvent_t e;
        GSV_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        s->ev_up.push_back(e);
    }
    while ((int)s->ev_slot_done.size() < kSeqSlots * 33) {
        cudaEvent_t e;
        GSV_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        s->ev_slot_done.push_back(e);
    }
    if ((int)s->seq_slot.size() < R) {
        s->seq_slot.resize(R, nullptr);
        s->seq_slot_cap.resize(R, 0);
    }
    for (int r = 0; r < R && !resident; r++) {
        const size_t want = (all_slots ? hi[r] - lo[r] : slot_bytes) + 64;
        if (s->seq_slot_cap[r] < want) {
            if (s->seq_slot[r]) cudaFree(s->seq_slot[r]);
            s->seq_slot[r] = nullptr;
            s->seq_slot_cap[r] = 0;
            const size_t cap = want + want / 8;  // slack: group sizes vary a little between calls
            if (cudaMalloc(&s->seq_slot[r], cap) != cudaSuccess) {
                cudaGetLastError();
                return fail(GSV_E_CUDA, "cudaMalloc: out of memory (sequence payload slots)");
            }
            s->seq_slot_cap[r] = cap;
        }
    }
    const std::vector<uint8_t*>& slot = s->seq_slot;
    // device base address of group gi's payload offsets: its slot (which holds
    // bytes [lo, hi) of the container), or the resident container itself
    auto dev_base = [&](int gi) -> const uint8_t* { return resident ? dev_data : slot[gi % R] - lo[gi]; };
    // the pinned staging of the deferred opens is reset once, with the
    // session stream drained (nothing of an earlier call still reads it)
    const auto t_sync = std::chrono::steady_clock::now();
    GSV_CUDA(cudaStreamSynchronize(s->stream));
    const auto t_reset = std::chrono::steady_clock::now();
    t_stage.reset();
    // dev: GSV_DEBUG_SEQ_TIMING=1 prints a per-group timeline (CUDA events)
    static const bool dbg = getenv("GSV_DEBUG_SEQ_TIMING") != nullptr;
    struct Mark {
        const char* what;
        int g;
        cudaEvent_t e;
        double host_ms;
    };
    std::vector<Mark> marks;
    const auto h0 = std::chrono::steady_clock::now();
    if (dbg)
        fprintf(stderr, "[seq] host: setup (parse, slots, sync) %.3f ms (to sync %.3f, sync %.3f, stage reset %.3f)\n",
                std::chrono::duration<double, std::milli>(h0 - t_entry).count(),
                std::chrono::duration<double, std::milli>(t_sync - t_entry).count(),
                std::chrono::duration<double, std::milli>(t_reset - t_sync).count(),
                std::chrono::duration<double, std::milli>(h0 - t_reset).count());
    auto mark = [&](const char* what, int g, cudaStream_t st) {
        if (!dbg) return;
        cudaEvent_t e;
        cudaEventCreate(&e);
        cudaEventRecord(e, st);
        marks.push_back({what, g, e, std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - h0).count()});
    };
    for (int attempt = 0; attempt < 4; attempt++) {
        if (int rc = ensure_aux(s, nstreams, img8, host_out)) return rc;
        VideoList vids;
        mark("start", -1, s->stream);
        int err = GSV_OK;
        int64_t fo = 0;
        // GSV_SEQ_PLANE_MAJOR=1: the first group goes up plane-major (plane f
        // of every run, then f + 1, ...: 2-D copies over the runs' constant
        // stride) so that its frame f can render as soon as its planes have
        // landed.  Off: the copy engine moves the 2-D copies at ~24 GB/s
        // against 55 for one contiguous copy, which delays every later group
        // (measured 76 vs 73 ms per config-2 step)
        static const bool pm_env = getenv("GSV_SEQ_PLANE_MAJOR") && atoi(getenv("GSV_SEQ_PLANE_MAJOR")) != 0;
        std::vector<std::vector<PlaneCopy>> pm0;
        if (pm_env && !resident) pm0 = plane_major_plan(data, c.groups[sel[0]], k);
        const bool plane_major = !pm0.empty();
        if (plane_major)
            while (s->ev_plane.size() < pm0.size()) {
                cudaEvent_t e;
                GSV_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
                s->ev_plane.push_back(e);
            }
        auto upload_group = [&](int gi) -> int {
            const int r = gi % R;
            if (gi >= R)  // ring: the slot's previous group has rendered
                for (int i = 0; i < nstreams; i++)
                    GSV_CUDA(cudaStreamWaitEvent(s->copy_in, s->ev_slot_done[(r % kSeqSlots) * 33 + i], 0));
            if (gi >= R) GSV_CUDA(cudaStreamWaitEvent(s->copy_in, s->ev_slot_done[(r % kSeqSlots) * 33 + 32], 0));
            if (gi == 0 && plane_major) {
                for (size_t f = 0; f < pm0.size(); f++) {
                    for (const PlaneCopy& pc : pm0[f])
                        GSV_CUDA(cudaMemcpy2DAsync(slot[r] + (pc.src_off - lo[0]), pc.pitch, data + pc.src_off,
                                                   pc.pitch, pc.width, pc.height, cudaMemcpyHostToDevice,
                                                   s->copy_in));
                    GSV_CUDA(cudaEventRecord(s->ev_plane[f], s->copy_in));
                }
            } else {
                GSV_CUDA(cudaMemcpyAsync(slot[r], data + lo[gi], hi[gi] - lo[gi], cudaMemcpyHostToDevice,
                                         s->copy_in));
            }
            GSV_CUDA(cudaEventRecord(s->ev_up[r], s->copy_in));
            mark("uploaded", gi, s->copy_in);
            return GSV_OK;
        };
        // every payload upload first when every group has a slot (the copy
        // engine streams the container from t = 0), else each one in the loop
        // once its ring slot is free; a group's descriptors go up by zero-copy
        // kernels on the session stream (never queued behind a payload), just
        // before the group's kernels
        // (all groups' descriptor kernels run at the start, while group 0's
        // payload is still uploading: a later group's kernels would otherwise
        // queue for SMs behind the renders of the groups before it, and its
        // frames could not start until those drained)
        // (resident: no payload copies, so the descriptors go by ordinary
        // copies, group by group, each just before its frames)
        auto prepare = [&](int gi) -> int {
            gsv_video* v = nullptr;
            const std::vector<int> one{sel[gi]};
            const int e = open_video(s, data, len, dev_base(gi), k, &v, &one, true, true);
            if (!e) vids.v.push_back(v);
            return e;
        };
        if (!resident) {
            if (all_slots)
                for (int gi = 0; gi < G && !err; gi++) err = upload_group(gi);
            t_zero_copy = true;
            for (int gi = 0; gi < G && !err; gi++) err = prepare(gi);
            t_zero_copy = false;
            // the CRC stream sees every group's descriptors and zeroed CRC slots
            if (!err) {
                GSV_CUDA(cudaEventRecord(s->ev_prep, s->stream));
                GSV_CUDA(cudaStreamWaitEvent(s->check, s->ev_prep, 0));
            }
            mark("prepared", -1, s->stream);
        }
        for (int gi = 0; gi < G && !err; gi++) {
            const int r = gi % R;
            if (resident) {
                if ((err = prepare(gi))) break;
                GSV_CUDA(cudaEventRecord(s->ev_prep, s->stream));
                GSV_CUDA(cudaStreamWaitEvent(s->check, s->ev_prep, 0));
            }
            gsv_video* v = vids.v[gi];
            if (!all_slots && (err = upload_group(gi))) break;
            // (the plane-major first group: its frames wait for their own planes)
            if (!resident && !(gi == 0 && plane_major)) GSV_CUDA(cudaStreamWaitEvent(s->stream, s->ev_up[r], 0));
            // renders fork before the group's CRC (validation only): they never
            // wait for the CRC kernel, which runs as SM resources free up
            v->runs.launch_planes(s->stream);
            mark("fork", gi, s->stream);
            std::vector<int32_t> fr;
            for (int32_t f = fb[gi]; f < fe[gi]; f++) fr.push_back(f);
            err = enqueue_frames(v, fr.data(), (int)fr.size(), cd, img8, out_rgb ? out_rgb + fo : nullptr,
                                 out_rgb8 ? out_rgb8 + fo : nullptr, host_rgb8 ? host_rgb8 + fo : nullptr, nstreams,
                                 (int)(fo % nstreams),
                                 (gi == 0 && plane_major) ? s->ev_plane.data() + fb[gi] : nullptr);
            if (err) break;
            for (int i = 0; i < nstreams && dbg; i++) mark("rendered", gi, s->aux[i]);
            for (int i = 0; i < nstreams && dbg && host_out; i++) mark("copied", gi, s->aux_copy[i]);
            // the group's CRC on its own stream: no render or later open waits for it
            if (!resident) GSV_CUDA(cudaStreamWaitEvent(s->check, s->ev_up[r], 0));
            if ((err = v->runs.launch_check(s->check, true))) break;
            if (!all_slots) {  // the slot is free once the group has rendered and its CRC has run
                for (int i = 0; i < nstreams; i++) GSV_CUDA(cudaEventRecord(s->ev_slot_done[r * 33 + i], s->aux[i]));
                GSV_CUDA(cudaEventRecord(s->ev_slot_done[r * 33 + 32], s->check));
            }
            fo += fe[gi] - fb[gi];
        }
        // drain everything before any buffer goes back to the pool
        const int jr = join_aux(s, nstreams, host_out);
        mark("joined", -1, s->stream);
        mark("checked", -1, s->check);
        cudaStreamSynchronize(s->copy_in);
        cudaStreamSynchronize(s->check);
        if (dbg) fprintf(stderr, "[seq] host: synced copy+check at %.3f ms\n",
                         std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - h0).count());
        if (dbg) {
            cudaDeviceSynchronize();
            for (const Mark& m : marks) {
                float t = 0;
                cudaEventElapsedTime(&t, marks[0].e, m.e);
                fprintf(stderr, "[seq] %-9s g%-3d gpu %8.3f ms  host-enqueued %8.3f ms\n", m.what, m.g, t, m.host_ms);
            }
            for (const Mark& m : marks) cudaEventDestroy(m.e);
            marks.clear();
            cudaGetLastError();
        }
        const cudaError_t se = cudaStreamSynchronize(s->stream);
        if (err) return err;
        if (jr) return jr;
        if (se != cudaSuccess) return fail(GSV_E_CUDA, std::string("render pipeline: ") + cudaGetErrorString(se));
        for (gsv_video* v : vids.v) {
            v->runs.fetch_crc();
            if (int rc = finish_open(v)) return rc;  // groups in decode order: the first error
        }
        if (dbg) fprintf(stderr, "[seq] host: checked at %.3f ms\n",
                         std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - h0).count());
        const int64_t need = aux_key_overflow(s, nstreams);
        if (need == 0) {
            if (frames_out) *frames_out = fo;
            return GSV_OK;
        }
        s->kcap_hint = need + need / 4 + 1024;  // grow and run the sequence again
    }
    return fail(GSV_E_NOMEM, "tile key buffer could not be sized");
}

int gsv_session_check_capacity(gsv_session* s) {
    GSV_CUDA(cudaStreamSynchronize(s->stream));
    for (size_t i = 0; i < s->aux.size(); i++) {
        GSV_CUDA(cudaStreamSynchronize(s->aux[i]));
        const RenderWork* w = s->aux_work[i];
        if (w->h_ctr && (int64_t)w->h_ctr[9] > w->cap_k)
            return fail(GSV_E_NOMEM, "tile key capacity exceeded in an unchecked batch (stream " +
                                         std::to_string(i) + ": " + std::to_string(w->h_ctr[9]) + " > " +
                                         std::to_string(w->cap_k) + ")");
    }
    return GSV_OK;
}

int gsv_render_soa(gsv_session* s, int64_t n, int sh_degree, const double* pos, const double* rot,
                   const double* scl, const double* opac, const double* sh, const gsv_camera* cam,
                   float* out_rgb, uint8_t* out_rgb8, gsv_render_stats* stats) {
    if (sh_degree < 0 || sh_degree > 3)
        return fail(GSV_E_INVALID_INPUT, "sh_degree must be 0..3, got " + std::to_string(sh_degree));
    if (cam->width < 1 || cam->height < 1) return fail(GSV_E_INVALID_INPUT, "image dimensions must be >= 1");
    SoaSrc src{pos, rot, scl, opac, sh, sh_degree, n};
    return render_soa(src, make_cam(*cam), &s->work, out_rgb, out_rgb8, stats, s->stream);
}

int gsv_render_splats2d(gsv_session* s, int64_t n, const double* means, const double* cov2d,
                        const double* depth, const double* colors, const double* opac,
                        const gsv_camera* cam, float* out_rgb, uint8_t* out_rgb8, gsv_render_stats* stats) {
    if (n < 0) return fail(GSV_E_INVALID_INPUT, "negative splat count");
    if (cam->width < 1 || cam->height < 1) return fail(GSV_E_INVALID_INPUT, "image dimensions must be >= 1");
    Splat2DSrc src{means, cov2d, depth, colors, opac, n};
    return render_splats2d(src, make_cam(*cam), &s->work, out_rgb, out_rgb8, stats, s->stream);
}

int gsv_sqdiff(gsv_session* s, const void* a, const void* b, int64_t n, int is_f64, double* out) {
    double* d = nullptr;
    GSV_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&d), sizeof(double), s->stream));
    if (is_f64)
        launch_sqdiff_f64(static_cast<const double*>(a), static_cast<const double*>(b), n, d, s->stream);
    else
        launch_sqdiff_f32(static_cast<const float*>(a), static_cast<const float*>(b), n, d, s->stream);
    count_launch(1);
    GSV_CUDA(cudaMemcpyAsync(out, d, sizeof(double), cudaMemcpyDeviceToHost, s->stream));
    GSV_CUDA(cudaFreeAsync(d, s->stream));
    GSV_CUDA(cudaStreamSynchronize(s->stream));
    return GSV_OK;
}

int gsv_ssim(gsv_session* s, const void* a, const void* b, int height, int width, int is_f64, double* out) {
    if (height < 11 || width < 11) return fail(GSV_E_INVALID_INPUT, "image smaller than the SSIM window");
    return ssim_device(a, b, height, width, is_f64 != 0, out, s->stream);
}

int gsv_project_debug(gsv_session* s, int64_t n, int sh_degree, const double* pos, const double* rot,
                      const double* scl, const double* opac, const double* sh, const gsv_camera* cam,
                      int32_t* rects, double* depth, int32_t* order, int32_t* tile_count,
                      int64_t* n_visible) {
    if (sh_degree < 0 || sh_degree > 3)
        return fail(GSV_E_INVALID_INPUT, "sh_degree must be 0..3, got " + std::to_string(sh_degree));
    SoaSrc src{pos, rot, scl, opac, sh, sh_degree, n};
    return project_debug(src, make_cam(*cam), &s->work, rects, depth, order, tile_count, n_visible,
                         s->stream);
}

int gsv_video_project_debug(gsv_video* v, int t, const gsv_camera* cam, int32_t* rects, double* depth,
                            int32_t* order, int32_t* tile_count, int64_t* n_visible) {
    FrameSrc src;
    int rc = frame_src(v, t, &src);
    if (rc) return rc;
    if (cam->width < 1 || cam->height < 1) return fail(GSV_E_INVALID_INPUT, "image dimensions must be >= 1");
    return project_debug_planes(src, make_cam(*cam), &v->s->work, rects, depth, order, tile_count, n_visible,
                                v->s->stream);
}

int gsv_fold_deltas(gsv_session* s, int64_t n, int shdim, double* pos, double* rot, double* scl,
                    double* opac, double* sh, int nd, const double* const* d_trans,
                    const double* const* d_rot, const double* const* d_scl,
                    const double* const* d_opac, const double* const* d_sh) {
    if (nd <= 0 || n <= 0) return GSV_OK;
    GSV_CUDA(cudaSetDevice(s->device));
    t_stage.reset();
    // the delta table and the zero-quaternion flag share one pooled block;
    // the flag comes back through the pinned staging buffer
    std::vector<FoldTab> tab(nd + 1);
    for (int d = 0; d < nd; d++) tab[d] = FoldTab{d_trans[d], d_rot[d], d_scl[d], d_opac[d], d_sh[d]};
    tab[nd] = FoldTab{};  // zeroed: the flag word
    DevBuf d_tab;
    int rc = upload(d_tab, tab, s->stream);
    if (rc) return rc;
    int* bad = reinterpret_cast<int*>(d_tab.as<FoldTab>() + nd);
    launch_fold_all(n, shdim, pos, rot, scl, opac, sh, d_tab.as<FoldTab>(), nd, bad, s->stream);  // one pass
    count_launch(1);
    int* h = reinterpret_cast<int*>(t_stage.reserve(sizeof(int), s->stream));
    int hv = 0;
    GSV_CUDA(cudaMemcpyAsync(h ? h : &hv, bad, sizeof(int), cudaMemcpyDeviceToHost, s->stream));
    GSV_CUDA(cudaStreamSynchronize(s->stream));
    if (h) hv = *h;
    if (hv) return fail(GSV_E_INVALID_INPUT, "zero quaternion cannot be normalized");
    return GSV_OK;
}

// ---- encoder ---------------------------------------------
int gsv_quantize_channels(gsv_session* s, gsv_quant_channel* ch, int nch) {
    if (nch < 0 || (nch > 0 && !ch)) return fail(GSV_E_INVALID_INPUT, "invalid channel list");
    if (nch == 0) return GSV_OK;
    std::vector<QuantChannel> qc(nch);
    uint64_t max_values = 0, max_samples = 0;
    for (int i = 0; i < nch; i++) {
        const gsv_quant_channel& c = ch[i];
        if (c.bits != 8 && c.bits != 16 && c.bits != 32) return fail(GSV_E_INVALID_INPUT, "bits must be one of (8, 16, 32)");
        if (c.frames == 0 || c.n == 0) return fail(GSV_E_INVALID_INPUT, "empty channel");
        if ((uint64_t)c.width * c.height < c.n) return fail(GSV_E_INVALID_INPUT, "plane smaller than the channel");
        if (c.frame_stride < c.n) return fail(GSV_E_INVALID_INPUT, "frame stride smaller than the channel");
        qc[i] = QuantChannel{c.values, c.planes, c.frame_stride, c.frames, c.n, c.width, c.height, c.bits};
        max_values = std::max<uint64_t>(max_values, (uint64_t)c.frames * c.n);
        max_samples = std::max<uint64_t>(max_samples, (uint64_t)c.frames * c.width * c.height);
    }
    cudaStream_t st = s->stream;
    DevBuf d_ch, d_red, d_rng;
    int rc = upload(d_ch, qc, st);
    if (rc) return rc;
    if ((rc = d_red.alloc((size_t)nch * 3 * 8))) return rc;
    if ((rc = d_rng.alloc((size_t)nch * 2 * 4))) return rc;
    std::vector<unsigned long long> init((size_t)nch * 3);
    for (int i = 0; i < nch; i++) {
        init[3 * i] = ~0ull;
        init[3 * i + 1] = 0ull;
        init[3 * i + 2] = 0ull;
    }
    GSV_CUDA(cudaMemcpyAsync(d_red.p, init.data(), init.size() * 8, cudaMemcpyHostToDevice, st));
    launch_quantize(d_ch.as<QuantChannel>(), nch, max_values, max_samples, d_red.as<unsigned long long>(),
                    d_rng.as<float>(), st);
    count_launch(3);
    std::vector<unsigned long long> red((size_t)nch * 3);
    std::vector<float> rng((size_t)nch * 2);
    GSV_CUDA(cudaMemcpyAsync(red.data(), d_red.p, red.size() * 8, cudaMemcpyDeviceToHost, st));
    GSV_CUDA(cudaMemcpyAsync(rng.data(), d_rng.p, rng.size() * 4, cudaMemcpyDeviceToHost, st));
    GSV_CUDA(cudaStreamSynchronize(st));
    GSV_CUDA(cudaGetLastError());
    for (int i = 0; i < nch; i++) {
        if (red[3 * i + 2]) return fail(GSV_E_INVALID_INPUT, "non-finite channel values");
        ch[i].range_min = rng[2 * i];
        ch[i].range_max = rng[2 * i + 1];
    }
    return GSV_OK;
}

uint64_t gsv_encode_body_capacity(uint32_t count, uint32_t width, uint32_t height, uint32_t bits) {
    const uint64_t plane = (uint64_t)width * height * (bits / 8);
    return plane * count + plane + count + 64;
}

int gsv_encode_runs(gsv_session* s, gsv_encode_run* runs, int nruns) {
    if (nruns < 0 || (nruns > 0 && !runs)) return fail(GSV_E_INVALID_INPUT, "invalid run list");
    if (nruns == 0) return GSV_OK;
    cudaStream_t st = s->stream;
    uint64_t nplan = 0, nchunks = 0;
    std::vector<uint32_t> by_class[3];
    for (int i = 0; i < nruns; i++) {
        const gsv_encode_run& r = runs[i];
        if (r.bits != 8 && r.bits != 16 && r.bits != 32) return fail(GSV_E_INVALID_INPUT, "bits must be one of (8, 16, 32)");
        if (r.count == 0 || r.width == 0 || r.height == 0 || r.count > 0xFFFF || r.width > 0xFFFF || r.height > 0xFFFF)
            return fail(GSV_E_INVALID_INPUT, "plane run exceeds u16 geometry limits");
        nplan += r.count;
        by_class[r.bits == 8 ? 0 : (r.bits == 16 ? 1 : 2)].push_back((uint32_t)i);
    }
    DevBuf d_snap, d_off, d_runs, d_order, d_res, d_prefix, d_rd, d_pl, d_chunk, d_crc;
    size_t snap_words = 0;
    for (int i = 0; i < nruns; i++) snap_words += 256u * (runs[i].bits / 8);
    int rc;
    if ((rc = d_snap.alloc(snap_words * 4))) return rc;
    if ((rc = d_off.alloc(nplan * 8))) return rc;
    std::vector<EncRun> er(nruns);
    std::vector<RunDesc> rd(nruns);
    std::vector<PlaneRef> pl;
    std::vector<uint32_t> plane_prefix(nruns + 1, 0), chunk_prefix;
    pl.reserve(nplan);
    chunk_prefix.reserve(nplan + 1);
    chunk_prefix.push_back(0);
    size_t so = 0, po = 0;
    for (int i = 0; i < nruns; i++) {
        const gsv_encode_run& r = runs[i];
        const uint32_t pb = r.width * r.height * (r.bits / 8);
        er[i] = EncRun{r.samples, r.body, d_off.as<uint64_t>() + po, d_snap.as<uint32_t>() + so,
                       r.count, r.width, r.height, r.bits};
        so += 256u * (r.bits / 8);
        po += r.count;
        plane_prefix[i + 1] = plane_prefix[i] + r.count;
        RunDesc d{};
        d.plane_bytes = pb;
        d.plane_base = (uint32_t)pl.size();
        d.w = (uint16_t)r.width;
        d.h = (uint16_t)r.height;
        d.count = (uint16_t)r.count;
        d.bits = (uint8_t)r.bits;
        rd[i] = d;
        for (uint32_t f = 0; f < r.count; f++) {
            PlaneRef p{};
            p.samples = r.samples + (size_t)f * pb;
            p.run = (uint32_t)i;
            p.f = f;
            pl.push_back(p);
            nchunks += (pb + kCrcChunk - 1) / kCrcChunk;
            chunk_prefix.push_back((uint32_t)nchunks);
        }
    }
    std::vector<uint32_t> order;
    for (auto& c : by_class) order.insert(order.end(), c.begin(), c.end());
    const int n_cls[3] = {(int)by_class[0].size(), (int)by_class[1].size(), (int)by_class[2].size()};
    if ((rc = upload(d_runs, er, st))) return rc;
    if ((rc = upload(d_order, order, st))) return rc;
    if ((rc = upload(d_prefix, plane_prefix, st))) return rc;
    if ((rc = upload(d_rd, rd, st))) return rc;
    if ((rc = upload(d_pl, pl, st))) return rc;
    if ((rc = upload(d_chunk, chunk_prefix, st))) return rc;
    if ((rc = d_res.alloc((size_t)nruns * sizeof(EncResult)))) return rc;
    if ((rc = d_crc.alloc((size_t)nruns * 4))) return rc;
    GSV_CUDA(cudaMemsetAsync(d_crc.p, 0, (size_t)nruns * 4, st));
    launch_rc_encode(d_runs.as<EncRun>(), d_order.as<uint32_t>(), n_cls, d_res.as<EncResult>(),
                     d_prefix.as<uint32_t>(), nruns, (uint32_t)nplan, st);
    count_launch(2);
    launch_crc(d_rd.as<RunDesc>(), d_pl.as<PlaneRef>(), (int)pl.size(), d_chunk.as<uint32_t>(),
               (uint32_t)nchunks, d_crc.as<uint32_t>(), st);
    if (nchunks) count_launch();
    std::vector<EncResult> res(nruns);
    std::vector<uint32_t> crc(nruns);
    GSV_CUDA(cudaMemcpyAsync(res.data(), d_res.p, res.size() * sizeof(EncResult), cudaMemcpyDeviceToHost, st));
    GSV_CUDA(cudaMemcpyAsync(crc.data(), d_crc.p, crc.size() * 4, cudaMemcpyDeviceToHost, st));
    GSV_CUDA(cudaStreamSynchronize(st));
    GSV_CUDA(cudaGetLastError());
    for (int i = 0; i < nruns; i++) {
        runs[i].body_len = res[i].body_len;
        runs[i].checksum = crc[i];
    }
    return GSV_OK;
}

int gsv_decode_payload_host(gsv_session* s, const uint8_t* blob, size_t len, uint32_t* samples,
                            size_t capacity, int32_t* hdr) {
    if (len >= 14) {
        hdr[0] = blob[0];
        hdr[1] = blob[1];
        hdr[2] = rd16(blob + 2);
        hdr[3] = rd16(blob + 4);
        hdr[4] = rd16(blob + 6);
    }
    ParsedRun pr;
    std::string m = parse_payload(blob, len, false, &pr);
    if (!m.empty()) return fail(GSV_E_CODEC, m);
    const size_t nsamp = (size_t)pr.rd.count * pr.rd.w * pr.rd.h;
    if (nsamp > capacity) return fail(GSV_E_INVALID_INPUT, "output buffer too small");
    DevBuf d_blob;
    int rc = d_blob.alloc(len + 64);
    if (rc) return rc;
    GSV_CUDA(cudaMemcpyAsync(d_blob.p, blob, len, cudaMemcpyHostToDevice, s->stream));
    RunSet rs;
    rs.add(pr, d_blob.as<uint8_t>());
    if ((rc = rs.decode(s->stream))) return rc;
    if (rs.crc[0] != rs.runs[0].checksum)
        return fail(GSV_E_CODEC, "checksum mismatch (corrupt or truncated payload)");
    // planes -> host u32 samples
    const uint32_t item = pr.rd.bits / 8, pb = rs.runs[0].plane_bytes;
    std::vector<uint8_t> tmp((size_t)pb * pr.rd.count + 1);
    for (uint32_t f = 0; f < pr.rd.count; f++)
        if (pb) GSV_CUDA(cudaMemcpyAsync(tmp.data() + (size_t)f * pb, rs.planes[f].samples, pb,
                                         cudaMemcpyDeviceToHost, s->stream));
    GSV_CUDA(cudaStreamSynchronize(s->stream));
    for (size_t i = 0; i < nsamp; i++) {
        uint32_t x = 0;
        for (uint32_t b = 0; b < item; b++) x |= (uint32_t)tmp[i * item + b] << (8 * b);
        samples[i] = x;
    }
    return GSV_OK;
}

}  // extern "C"
