// Host side of the container format: error plumbing, header/directory
// parsing (container.py:35-41, 151-191) and the synthetic-input encoder
// tooling (codec.py:105-180, _rc.py:55-118, 249-279).
#include <stdio.h>
#include <string.h>

#include <string>
#include <vector>

#include "gsv_internal.h"

#include <mutex>

namespace gsv {

long long g_launches = 0;

// ---- stage profiler ---------------------------------------------------------
namespace {
struct Prof {
    std::mutex mu;
    bool enabled = false;
    std::vector<std::pair<int, cudaEvent_t>> marks;
    std::vector<cudaEvent_t> pool;
    double ms[ST_COUNT + 1] = {0};
    long long n[ST_COUNT + 1] = {0};
};
Prof& prof() {
    static Prof p;
    return p;
}
}  // namespace

void prof_enable(bool on) {
    Prof& p = prof();
    std::lock_guard<std::mutex> g(p.mu);
    p.enabled = on;
    for (int i = 0; i <= ST_COUNT; i++) p.ms[i] = 0, p.n[i] = 0;
}

void prof_mark(int stage, cudaStream_t s) {
    Prof& p = prof();
    if (!p.enabled) return;
    std::lock_guard<std::mutex> g(p.mu);
    cudaEvent_t e;
    if (!p.pool.empty()) {
        e = p.pool.back();
        p.pool.pop_back();
    } else {
        cudaEventCreate(&e);
    }
    cudaEventRecord(e, s);
    p.marks.emplace_back(stage, e);
}

int prof_read(double* ms, long long* marks, int max_stages) {
    Prof& p = prof();
    std::lock_guard<std::mutex> g(p.mu);
    for (size_t i = 0; i + 1 < p.marks.size(); i++) {
        const int st = p.marks[i].first;
        if (st >= ST_COUNT) continue;
        cudaEventSynchronize(p.marks[i + 1].second);
        float t = 0;
        cudaEventElapsedTime(&t, p.marks[i].second, p.marks[i + 1].second);
        p.ms[st] += t;
        p.n[st] += 1;
    }
    for (auto& m : p.marks) p.pool.push_back(m.second);
    p.marks.clear();
    for (int i = 0; i < max_stages && i < ST_COUNT; i++) {
        ms[i] = p.ms[i];
        marks[i] = p.n[i];
    }
    return GSV_OK;
}

static thread_local int g_err_kind = GSV_OK;
static thread_local std::string g_err_msg;

void set_error(int kind, const std::string& msg) {
    g_err_kind = kind;
    g_err_msg = msg;
}

int fail(int kind, const std::string& msg) {
    set_error(kind, msg);
    return kind;
}

const char* attr_name(int attr) {
    static const char* names[] = {"position", "rotation", "scales", "opacity", "sh"};
    return (attr >= 0 && attr < 5) ? names[attr] : "?";
}

int slot_of(int attr, int comp, int shdim) {
    switch (attr) {
        case 0: return comp < 3 ? comp : -1;
        case 1: return comp < 4 ? 3 + comp : -1;
        case 2: return comp < 3 ? 7 + comp : -1;
        case 3: return comp < 1 ? 10 : -1;
        case 4: return comp < shdim ? 11 + comp : -1;
    }
    return -1;
}

namespace {
struct Cursor {
    const uint8_t* p;
    size_t len, pos;
    bool take(size_t n, const uint8_t** out) {
        if (pos + n > len) {
            char b[96];
            snprintf(b, sizeof b, "unexpected end of container (wanted %zu bytes)", n);
            set_error(GSV_E_FORMAT, b);
            return false;
        }
        *out = p + pos;
        pos += n;
        return true;
    }
};
template <class T>
T rd(const uint8_t* p) {
    T v;
    memcpy(&v, p, sizeof v);
    return v;
}
}  // namespace

// read_structure (container.py:151-191), same checks in the same order.
int parse_container(const uint8_t* data, size_t len, Container* out) {
    Cursor c{data, len, 0};
    const uint8_t* h;
    if (!c.take(42, &h)) return GSV_E_FORMAT;
    Container ci;
    ci.version = rd<uint16_t>(h + 4);
    ci.layer_count = h[6];
    ci.sh_degree = h[7];
    uint16_t ngroups = rd<uint16_t>(h + 8);
    ci.fps_num = rd<uint16_t>(h + 10);
    ci.fps_den = rd<uint16_t>(h + 12);
    for (int i = 0; i < 6; i++) ci.bounds[i] = rd<float>(h + 14 + 4 * i);
    ci.flags = rd<uint32_t>(h + 38);
    if (memcmp(h, "GSV1", 4) != 0) return fail(GSV_E_FORMAT, "not a gsv container (bad magic)");
    if (ci.version != 1) {
        return fail(GSV_E_FORMAT, "unsupported container version " + std::to_string(ci.version));
    }
    if (ci.layer_count < 1) return fail(GSV_E_FORMAT, "layer count must be >= 1");
    const int L = ci.layer_count;
    uint64_t last = 0;
    bool last_inf = false;
    ci.groups.resize(ngroups);
    for (int g = 0; g < ngroups; g++) {
        GroupDir& gd = ci.groups[g];
        const uint8_t* f;
        if (!c.take(8, &f)) return GSV_E_FORMAT;
        gd.start_frame = rd<uint32_t>(f);
        gd.frame_count = rd<uint16_t>(f + 4);
        gd.position_bits = f[6];
        const uint8_t* lc;
        if (!c.take(4 * (size_t)L, &lc)) return GSV_E_FORMAT;
        gd.layer_counts.resize(L);
        for (int l = 0; l < L; l++) gd.layer_counts[l] = rd<uint32_t>(lc + 4 * l);
        gd.channels.resize(L);
        for (int l = 0; l < L; l++) {
            const uint8_t* nb;
            if (!c.take(2, &nb)) return GSV_E_FORMAT;
            uint16_t nch = rd<uint16_t>(nb);
            gd.channels[l].resize(nch);
            for (int e = 0; e < nch; e++) {
                const uint8_t* ep;
                if (!c.take(28, &ep)) return GSV_E_FORMAT;
                Entry& en = gd.channels[l][e];
                en.attr = ep[0];
                en.comp = rd<uint16_t>(ep + 1);
                en.bits = ep[3];
                en.offset = rd<uint64_t>(ep + 4);
                en.size = rd<uint64_t>(ep + 12);
                en.rmin = rd<float>(ep + 20);
                en.rmax = rd<float>(ep + 24);
                if (en.attr > 4) {
                    return fail(GSV_E_FORMAT, "unknown attribute code " + std::to_string(en.attr));
                }
                // offset + size as an unbounded integer (the reference's Python
                // ints): a sum past 2^64 makes every later offset smaller
                if (last_inf || en.offset < last) return fail(GSV_E_FORMAT, "payload offsets are not increasing");
                last_inf = en.size > UINT64_MAX - en.offset;
                last = last_inf ? UINT64_MAX : en.offset + en.size;
            }
        }
    }
    ci.header_bytes = c.pos;
    *out = std::move(ci);
    return GSV_OK;
}

// ---------------------------------------------------------------------------
// Encoder tooling (produces synthetic benchmark inputs; not on the decode
// path).  Restates _rc.encode_bittree (_rc.py:55-118), plane_residuals
// (_rc.py:249-279) and _encode_reference_body (codec.py:137-163).
// ---------------------------------------------------------------------------
namespace {
struct RcEnc {
    uint64_t low = 0;
    uint32_t rng = 0xFFFFFFFFu;
    uint32_t cache = 0;
    uint64_t cache_size = 1;
    uint8_t* out;
    size_t pos = 0, limit;
    bool overflow = false;
    bool shift_low() {
        if (pos + cache_size > limit) { overflow = true; return false; }
        uint32_t lo32 = (uint32_t)low;
        uint32_t carry = (uint32_t)(low >> 32);
        if (lo32 < 0xFF000000u || carry != 0) {
            out[pos++] = (uint8_t)(cache + carry);
            for (uint64_t i = 1; i < cache_size; i++) out[pos++] = (uint8_t)(0xFF + carry);
            cache = (lo32 >> 24) & 0xFF;
            cache_size = 0;
        }
        cache_size++;
        low = (uint64_t)(lo32 & 0x00FFFFFFu) << 8;
        return true;
    }
};
}  // namespace

static int64_t encode_bittree(const uint8_t* data, size_t num, int nbytes, int32_t* probs,
                              uint8_t* out, size_t cap) {
    RcEnc e;
    e.out = out;
    e.limit = cap >= 8 ? cap - 8 : 0;
    for (size_t i = 0; i < num; i++) {
        for (int b = 0; b < nbytes; b++) {
            uint32_t byte = data[i * nbytes + b];
            int32_t* tree = probs + 256 * b;
            uint32_t ctx = 1;
            for (int bp = 7; bp >= 0; bp--) {
                uint32_t bit = (byte >> bp) & 1;
                uint32_t p = (uint32_t)tree[ctx];
                uint32_t bound = (e.rng >> 12) * p;
                if (bit == 0) {
                    e.rng = bound;
                    tree[ctx] = (int32_t)(p + ((4096 - p) >> 4));
                } else {
                    e.low += bound;
                    e.rng -= bound;
                    tree[ctx] = (int32_t)(p - (p >> 4));
                }
                ctx = (ctx << 1) | bit;
                while (e.rng < (1u << 24)) {
                    if (!e.shift_low()) return -1;
                    e.rng <<= 8;
                }
            }
        }
    }
    for (int i = 0; i < 5; i++)
        if (!e.shift_low()) return -1;
    return (int64_t)e.pos;
}

static void init_probs(int32_t* probs, int nbytes) {
    for (int b = 0; b < nbytes; b++) {
        for (int i = 0; i < 256; i++) probs[256 * b + i] = 2048;
        for (int ctx = 1; ctx < 256; ctx <<= 1) probs[256 * b + ctx] = 3686;
    }
}

}  // namespace gsv

using namespace gsv;

extern "C" {

const char* gsv_last_error(void) { return g_err_msg.c_str(); }
int gsv_last_error_kind(void) { return g_err_kind; }
int gsv_abi_version(void) { return GSV_ABI_VERSION; }

uint32_t gsv_crc32(const uint8_t* p, size_t n) {
    static uint32_t table[256];
    static bool ready = false;
    if (!ready) {
        for (uint32_t i = 0; i < 256; i++) {
            uint32_t c = i;
            for (int k = 0; k < 8; k++) c = (c & 1) ? (0xEDB88320u ^ (c >> 1)) : (c >> 1);
            table[i] = c;
        }
        ready = true;
    }
    uint32_t crc = 0xFFFFFFFFu;
    for (size_t i = 0; i < n; i++) crc = table[(crc ^ p[i]) & 0xFF] ^ (crc >> 8);
    return ~crc;
}

int gsv_read_info(const uint8_t* data, size_t len, gsv_info* out) {
    Container c;
    int rc = parse_container(data, len, &c);
    if (rc) return rc;
    out->version = c.version;
    out->layer_count = c.layer_count;
    out->sh_degree = c.sh_degree;
    out->group_count = (int32_t)c.groups.size();
    out->fps_num = c.fps_num;
    out->fps_den = c.fps_den;
    out->flags = c.flags;
    for (int i = 0; i < 6; i++) out->bounds[i] = c.bounds[i];
    out->header_bytes = c.header_bytes;
    return GSV_OK;
}

int gsv_read_group(const uint8_t* data, size_t len, int group, gsv_group_info* out) {
    Container c;
    int rc = parse_container(data, len, &c);
    if (rc) return rc;
    if (group < 0 || group >= (int)c.groups.size()) return fail(GSV_E_INVALID_INPUT, "group out of range");
    if (c.layer_count > 64) return fail(GSV_E_INVALID_INPUT, "more than 64 layers");
    const GroupDir& g = c.groups[group];
    memset(out, 0, sizeof *out);
    out->start_frame = g.start_frame;
    out->frame_count = g.frame_count;
    out->position_bits = g.position_bits;
    for (int l = 0; l < c.layer_count; l++) {
        out->layer_counts[l] = g.layer_counts[l];
        out->channel_counts[l] = (uint32_t)g.channels[l].size();
    }
    return GSV_OK;
}

int gsv_read_entry(const uint8_t* data, size_t len, int group, int layer, int entry,
                   gsv_entry_info* out) {
    Container c;
    int rc = parse_container(data, len, &c);
    if (rc) return rc;
    if (group < 0 || group >= (int)c.groups.size() || layer < 0 || layer >= c.layer_count ||
        entry < 0 || entry >= (int)c.groups[group].channels[layer].size())
        return fail(GSV_E_INVALID_INPUT, "entry out of range");
    const Entry& e = c.groups[group].channels[layer][entry];
    out->attribute = e.attr;
    out->component = e.comp;
    out->bits = e.bits;
    out->offset = e.offset;
    out->size = e.size;
    out->range_min = e.rmin;
    out->range_max = e.rmax;
    return GSV_OK;
}

int gsv_read_directory(const uint8_t* data, size_t len, gsv_group_info* groups, size_t group_cap,
                       gsv_entry_info* entries, size_t entry_cap, size_t* n_entries) {
    Container c;
    int rc = parse_container(data, len, &c);
    if (rc) return rc;
    if (c.layer_count > 64) return fail(GSV_E_INVALID_INPUT, "more than 64 layers");
    size_t ne = 0;
    for (const GroupDir& g : c.groups)
        for (int l = 0; l < c.layer_count; l++) ne += g.channels[l].size();
    if (n_entries) *n_entries = ne;
    if (c.groups.size() > group_cap || ne > entry_cap) return fail(GSV_E_INVALID_INPUT, "directory buffers too small");
    size_t k = 0;
    for (size_t gi = 0; gi < c.groups.size(); gi++) {
        const GroupDir& g = c.groups[gi];
        gsv_group_info* o = groups + gi;
        memset(o, 0, sizeof *o);
        o->start_frame = g.start_frame;
        o->frame_count = g.frame_count;
        o->position_bits = g.position_bits;
        for (int l = 0; l < c.layer_count; l++) {
            o->layer_counts[l] = g.layer_counts[l];
            o->channel_counts[l] = (uint32_t)g.channels[l].size();
            for (const Entry& e : g.channels[l]) {
                gsv_entry_info* q = entries + k++;
                q->attribute = e.attr;
                q->component = e.comp;
                q->bits = e.bits;
                q->offset = e.offset;
                q->size = e.size;
                q->range_min = e.rmin;
                q->range_max = e.rmax;
            }
        }
    }
    return GSV_OK;
}

// _encode_reference_body (codec.py:137-163) -> body bytes (flag + modes + blocks),
// or the whole-run raw fallback.  samples: count*h*w values < 2^bits.
int64_t gsv_encode_reference_body(const uint32_t* samples, int count, int h, int w, int bits,
                                  uint8_t* out, size_t capacity) {
    const int item = bits / 8, nbytes = bits / 8;
    const size_t hw = (size_t)h * (size_t)w;
    const size_t raw_len = (size_t)count * hw * item;
    if (capacity < raw_len + 1) return -2;
    std::vector<int32_t> probs(256 * nbytes), snap;
    init_probs(probs.data(), nbytes);
    std::vector<uint8_t> data(hw * nbytes);
    std::vector<uint8_t> enc(hw * nbytes * 10 + 64);
    std::vector<uint8_t> body;
    body.reserve(raw_len + 1 + count);
    body.push_back(0);
    std::vector<uint8_t> modes(count);
    std::vector<std::vector<uint8_t>> blocks(count);
    const int64_t half = (int64_t)1 << (bits - 1), full = (int64_t)1 << bits;
    const int64_t def = (int64_t)128 << (bits - 8);
    for (int f = 0; f < count; f++) {
        const uint32_t* plane = samples + (size_t)f * hw;
        const uint32_t* prev = f > 0 ? samples + (size_t)(f - 1) * hw : plane;
        for (size_t idx = 0; idx < hw; idx++) {
            size_t y = idx / w, x = idx % w;
            int64_t pred;
            if (f > 0) pred = prev[idx];
            else if (x > 0) pred = plane[idx - 1];
            else if (y > 0) pred = plane[idx - w];
            else pred = def;
            int64_t r = (int64_t)plane[idx] - pred;
            r = ((r + half) % full + full) % full - half;
            uint64_t z = r >= 0 ? (uint64_t)(2 * r) : (uint64_t)(-2 * r - 1);
            for (int b = 0; b < nbytes; b++) data[idx * nbytes + b] = (uint8_t)(z >> (8 * b));
        }
        snap = probs;
        int64_t n = encode_bittree(data.data(), hw, nbytes, probs.data(), enc.data(), enc.size());
        while (n > 0 && enc[n - 1] == 0) n--;
        const size_t raw_plane = hw * item;
        if (n < 0 || (size_t)n + 4 >= raw_plane) {
            probs = snap;
            modes[f] = 1;
            blocks[f].resize(raw_plane);
            for (size_t i = 0; i < hw; i++)
                for (int b = 0; b < item; b++) blocks[f][i * item + b] = (uint8_t)(plane[i] >> (8 * b));
        } else {
            modes[f] = 0;
            blocks[f].resize(4 + n);
            uint32_t nn = (uint32_t)n;
            memcpy(blocks[f].data(), &nn, 4);
            memcpy(blocks[f].data() + 4, enc.data(), n);
        }
    }
    body.insert(body.end(), modes.begin(), modes.end());
    for (auto& b : blocks) body.insert(body.end(), b.begin(), b.end());
    if (body.size() > raw_len + 1) {
        out[0] = 1;
        for (size_t i = 0; i < (size_t)count * hw; i++)
            for (int b = 0; b < item; b++) out[1 + i * item + b] = (uint8_t)(samples[i] >> (8 * b));
        return (int64_t)(raw_len + 1);
    }
    if (body.size() > capacity) return -2;
    memcpy(out, body.data(), body.size());
    return (int64_t)body.size();
}

}  // extern "C"
