// Internal declarations shared by the libgsv_b200 translation units.
//
// Data layout in HBM:
//   * payload bytes are staged verbatim (one contiguous copy per group
//     layer-prefix segment, container.py:65-70); codec-0 / raw-fallback /
//     RAW-mode planes are consumed in place, so decoding them is zero-copy;
//   * range-coded planes are decoded into `plane_buf` (16-B aligned planes);
//   * every (run, frame) has a PlaneRef giving the device address of its
//     little-endian samples, so the projection reads codes straight from the
//     planes and dequantizes in registers (the fp64 SoA the reference builds,
//     container.py:229-257, is only materialised on request).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stddef.h>

#include <string>
#include <vector>

#include "../../include/gsv_b200.h"

namespace gsv {

// ---- error plumbing --------------------------------------------------------
void set_error(int kind, const std::string& msg);
int fail(int kind, const std::string& msg);
#define GSV_CUDA(call)                                                              \
    do {                                                                            \
        cudaError_t e_ = (call);                                                    \
        if (e_ != cudaSuccess)                                                      \
            return ::gsv::fail(GSV_E_CUDA, std::string(#call) + ": " +              \
                                               cudaGetErrorString(e_));             \
    } while (0)

// ---- container directory (container.py:35-41, 151-191) ----------------------
struct Entry {
    uint8_t attr;      // 0 position, 1 rotation, 2 scales, 3 opacity, 4 sh
    uint16_t comp;
    uint8_t bits;      // directory bit width (used for dequantization)
    uint64_t offset;
    uint64_t size;
    float rmin, rmax;
};

struct GroupDir {
    uint32_t start_frame;
    uint16_t frame_count;
    uint8_t position_bits;
    std::vector<uint32_t> layer_counts;
    std::vector<std::vector<Entry>> channels;  // [layer][entry]
};

struct Container {
    uint16_t version = 0;
    uint8_t layer_count = 0;
    uint8_t sh_degree = 0;
    uint16_t fps_num = 0, fps_den = 0;
    float bounds[6] = {0};
    uint32_t flags = 0;
    std::vector<GroupDir> groups;
    uint64_t header_bytes = 0;  // header + directory
};

int parse_container(const uint8_t* data, size_t len, Container* out);
const char* attr_name(int attr);

// slot of (attr, comp) in the per-splat attribute vector:
// position 0-2, rotation 3-6, scales 7-9, opacity 10, sh 11.. ; -1 if unused
int slot_of(int attr, int comp, int shdim);
inline int slot_count(int sh_degree) { return 11 + 3 * (sh_degree + 1) * (sh_degree + 1); }
constexpr int kMaxSlots = 11 + 48;
constexpr int kMaxLayers = 64;
constexpr int kMaxDevices = 64;  // per-device attribute state
constexpr int kCtrWords = 32;  // device counters per render workspace

// ---- device descriptors ------------------------------------------------------
// One decodable (group, layer, entry) payload.
struct RunDesc {
    uint32_t checksum;
    uint32_t plane_bytes;  // h*w*item
    uint32_t plane_base;   // first PlaneRef of this run
    uint16_t w, h, count;
    uint8_t bits;          // payload bit width
    uint8_t kind;          // 0: raw samples in place, 1: per-plane (codec 1, flag 0)
};

// One plane of one run.
struct PlaneRef {
    const uint8_t* samples;  // little-endian samples (device; may be unaligned)
    const uint8_t* coded;    // range-coded block (mode 0) or nullptr
    uint32_t coded_len;
    uint32_t run;
    uint32_t f;              // index inside the run
    uint32_t mode;           // 0: range coded, 1: raw
};

// One (frame, layer, slot): where that frame's codes live and how to
// dequantize them (quantize.py:114-117 with span = rmax - rmin).
struct SlotDesc {
    const uint8_t* samples;  // little-endian plane samples of this frame (device)
    double rmin, span;       // directory range (f32 values promoted), rmax - rmin
    uint8_t dir_bits;        // directory bit width -> top = 2^bits - 1
    uint8_t bits;            // payload sample width
    uint16_t pad0;
    uint32_t pad1;
};

// A frame's source: its resolved slots [nlayers][nslots].
struct FrameSrc {
    const SlotDesc* slots;
    int32_t nlayers;
    int32_t nslots;
    int32_t sh_degree;
    uint32_t layer_off[kMaxLayers + 1];  // prefix sums of layer counts
};

// fp64 SoA source (render_set / render_progressive inputs)
struct SoaSrc {
    const double* pos;   // (n,3)
    const double* rot;   // (n,4)
    const double* scl;   // (n,3)
    const double* opac;  // (n)
    const double* sh;    // (n,shdim)
    int32_t sh_degree;
    int64_t n;
};

// projected splats (render(list[Splat2D]) inputs), device fp64
struct Splat2DSrc {
    const double* means;   // (n,2)
    const double* cov;     // (n,2,2)
    const double* depth;   // (n)
    const double* colors;  // (n,3)
    const double* opac;    // (n)
    int64_t n;
};

// Camera as the kernels see it (render.py:43-120)
struct CamDev {
    double R[9];
    double t[3];
    double center[3];
    double fx, fy, cx, cy, near_;
    float bg[3];
    int32_t width, height;
};

// 64-byte splat record consumed by the compositor:
//   fx0, fy0, fx1, fy1 : the integer rect [x0, x1) x [y0, y1) as floats (exact)
//   ox, oy             : mean - rect origin (px)
//   ca, cb, cc         : -log2(e)/2 * (a, 2b, c) of the conic inverse
//                        (render.py:346-349): alpha = op * 2^(ca dx^2 + cb dx dy + cc dy^2)
//   r, g, b            : SH colour in [0, 1];  op : opacity
//   rx, ry             : x0 | x1 << 16, y0 | y1 << 16 (u16 each; tile binning)
//   lop                : log2(op) as float bits (-inf for op = 0)
struct __align__(16) SplatRec {
    float fx0, fy0, fx1, fy1;
    float ox, oy, ca, cb;
    float cc, r, g, b;
    float op;
    uint32_t rx, ry;
    uint32_t pad;  // lop
};

// ---- workspace for one in-flight render ----------------------------------
struct RenderWork {
    int64_t cap_n = 0;    // splat capacity
    int64_t cap_k = 0;    // key capacity
    int cap_tiles = 0;
    // per splat
    uint64_t* dkey[2] = {nullptr, nullptr};  // depth sort keys (ping-pong)
    uint32_t* didx[2] = {nullptr, nullptr};  // splat indices (ping-pong)
    SplatRec* rec = nullptr;                 // by splat index
    uint2* rect = nullptr;                   // (rx, ry) of rec, by splat index: the compact copy
                                             // the binning / key-emission gathers read
    uint64_t* tie_k = nullptr;               // depth tie fix-up of long runs: key scratch
    uint32_t* tie_runs = nullptr;            // long runs of equal truncated keys (start, end)
    // per key
    uint32_t* tkey[2] = {nullptr, nullptr};
    uint32_t* tval[2] = {nullptr, nullptr};
    // per tile / per pixel
    uint8_t* tile_done = nullptr;            // saturated tiles
    uint32_t* open_mask = nullptr;           // bit per tile: still open (later rounds' emission)
    uint32_t* r1_bc = nullptr;               // round-1 binning: per (rank block, tile) counts / offsets
    uint32_t* r1_off = nullptr;              // round-1 binning: tile ranges (ntiles + 1)
    size_t r1_bc_cap = 0, r1_off_cap = 0;
    float4* state = nullptr;                 // per pixel (C.rgb, T) carried across rounds
    int64_t cap_pix = 0;
    // decoupled look-back scan state of the fused key emission
    unsigned long long* status = nullptr;
    unsigned int* ticket = nullptr;
    uint32_t epoch = 0;
    // radix sort scratch (sort.cuh SortScratch)
    uint32_t* sort_ghist = nullptr;              // 4 x 256 digit counts + ticket
    unsigned long long* sort_status = nullptr;   // look-back status words
    int64_t sort_status_cap = 0;
    uint32_t sort_epoch = 0;
    // device counters: [0] n_visible, [1] n_keys, [2..3] depth min (u64), [4..5] depth max,
    // [6] key overflow flag, [8..] radix pass state
    unsigned long long* ctr = nullptr;
    unsigned long long* h_ctr = nullptr;     // pinned mirror
};

int work_reserve(RenderWork* w, int64_t n, int64_t k, int tiles, int64_t npix);
void work_free(RenderWork* w);

// ---- encoder (encode.cu) ----
// one channel of one group: (frames, n) fp64 values -> padded w*h planes
struct QuantChannel {
    const double* values;   // value (f, j) at values[f * frame_stride + j]
    uint8_t* planes;
    uint64_t frame_stride;
    uint32_t frames, n, w, h, bits;
};
// one run to range-code: count planes of w*h LE samples
struct EncRun {
    const uint8_t* samples;
    uint8_t* body;       // payload body buffer (capacity per gsv_encode_body_capacity)
    uint64_t* blk_off;   // per plane: offset of its block in the body
    uint32_t* snap;      // NB*256 words: model snapshot
    uint32_t count, w, h, bits;
};
struct EncResult {
    uint64_t body_len;
    uint32_t whole_raw;
    uint32_t pad;
};
struct EncClasses {
    int n[3];
    int off[3];
    int blk[4];
    int lanes;  // runs per warp
};
void launch_quantize(const QuantChannel* d_ch, int nch, uint64_t max_values, uint64_t max_samples,
                     unsigned long long* d_red, float* d_ranges, cudaStream_t s);
void launch_rc_encode(const EncRun* d_runs, const uint32_t* d_order, const int* n_per_class,
                      EncResult* d_res, const uint32_t* d_plane_prefix, int nruns, uint32_t nplanes,
                      cudaStream_t s);

// byte copy job (RAW planes of range-coded runs -> aligned storage)
struct CopyJob {
    const uint8_t* src;
    uint8_t* dst;
    uint32_t bytes;
};

// ---- kernels (host launchers) -------------------------------------------------
// rc_decode.cu
void launch_copy_planes(const CopyJob* jobs, int njobs, cudaStream_t s);
// decode.cu
// rc_runs: run indices grouped by sample width (1, 2, 4 bytes), n_per_class[3]
void launch_rc_decode(const RunDesc* runs, const uint32_t* rc_runs, const int* n_per_class,
                      const PlaneRef* planes, cudaStream_t s);
// CRC-32 work unit: a chunk of this many bytes of one plane (the last chunk
// of a plane may be shorter); chunk counts per plane are built on the host.
constexpr uint32_t kCrcChunk = 4096;
void launch_crc(const RunDesc* runs, const PlaneRef* planes, int nplanes,
                const uint32_t* plane_chunk_prefix, uint32_t nchunks, uint32_t* run_crc,
                cudaStream_t s);
void launch_dequant_frame(const FrameSrc& src, double* pos, double* rot, double* scl,
                          double* opac, double* sh, cudaStream_t s);
void launch_frame_codes(const FrameSrc& src, uint32_t* out, cudaStream_t s);

// composite.cu
// One depth-rank round; `first` starts from (C, T) = (0, 1), `last` writes the
// final image of every tile still open (saturated tiles are written when they
// saturate).
int composite_rows();  // pixel rows per lane of the compositor (GSV_COMPOSITE_ROWS: 2, 4, 8)
void launch_composite_round(const uint32_t* keys, const uint32_t* tile_off, const uint32_t* ranks,
                            const unsigned long long* nkeys, const SplatRec* recs, float4* state,
                            uint8_t* tile_done, const CamDev& cam, bool first, bool last, float* out_rgb,
                            uint8_t* out_rgb8, cudaStream_t s);

// render.cu: full per-frame pipeline
int render_planes(const FrameSrc& src, const CamDev& cam, RenderWork* w, float* out_rgb,
                  uint8_t* out_rgb8, gsv_render_stats* stats, cudaStream_t s);
// counters of w to its pinned mirror on s (after an enqueue-only batch)
int readback_counters(RenderWork* w, cudaStream_t s);
int render_soa(const SoaSrc& src, const CamDev& cam, RenderWork* w, float* out_rgb,
               uint8_t* out_rgb8, gsv_render_stats* stats, cudaStream_t s);
int render_splats2d(const Splat2DSrc& src, const CamDev& cam, RenderWork* w, float* out_rgb,
                    uint8_t* out_rgb8, gsv_render_stats* stats, cudaStream_t s);
// sum of squared differences of two device arrays (fp32 or fp64), into *out (device)
void launch_sqdiff_f32(const float* a, const float* b, int64_t n, double* out, cudaStream_t s);
void launch_sqdiff_f64(const double* a, const double* b, int64_t n, double* out, cudaStream_t s);
// mean SSIM of two device (H, W, 3) images (fp32 or fp64) on stream s
int ssim_device(const void* a, const void* b, int H, int W, bool f64, double* out_mean, cudaStream_t s);
int project_debug(const SoaSrc& src, const CamDev& cam, RenderWork* w, int32_t* rects,
                  double* depth, int32_t* order, int32_t* tile_count, int64_t* n_visible,
                  cudaStream_t s);
int project_debug_planes(const FrameSrc& src, const CamDev& cam, RenderWork* w, int32_t* rects,
                         double* depth, int32_t* order, int32_t* tile_count, int64_t* n_visible,
                         cudaStream_t s);
struct FoldTab {  // one frame delta (motion.py:58-141), device pointers
    const double* dt;
    const double* dq;
    const double* ds;
    const double* dop;
    const double* dsh;
};
void launch_fold_all(int64_t n, int shdim, double* pos, double* rot, double* scl, double* opac, double* sh,
                     const FoldTab* tab, int nd, int* bad, cudaStream_t s);
void launch_fold(int64_t n, int shdim, double* pos, double* rot, double* scl, double* opac,
                 double* sh, const double* dt, const double* dq, const double* ds,
                 const double* dop, const double* dsh, int* bad, cudaStream_t s);

CamDev make_cam(const gsv_camera& c);
constexpr int kTile = 16;
// per-strip state between depth-rank rounds (RenderWork::tile_done: 4 bytes
// per tile, one per strip of the compositor; bytes past the strip count are
// kTileSaturated, so a tile is saturated iff its word is 0x01010101)
constexpr uint8_t kTileOpen = 0;       // (C, T) of its pixels live in `state`
constexpr uint8_t kTileSaturated = 1;  // every pixel T < 1e-4: written out, gets no more keys
constexpr uint8_t kTileBlank = 2;
constexpr uint32_t kTileAllSat = 0x01010101u;      // no key yet: written out as background, state implied (0, 1)

// ---- launch accounting and stage profiling (bench instrumentation) ---------
extern long long g_launches;  // kernels launched by this library (all threads)
inline void count_launch(int n = 1) { __atomic_fetch_add(&g_launches, (long long)n, __ATOMIC_RELAXED); }

enum Stage { ST_PROJECT = 0, ST_DSORT, ST_EMIT, ST_TSORT, ST_RANGES, ST_COMPOSITE, ST_RCDEC, ST_CRC,
             ST_COUNT };
// When enabled, mark(stage) records an event on the stream; the interval up to
// the next mark is charged to `stage` (ST_COUNT = idle / end).
void prof_mark(int stage, cudaStream_t s);
void prof_enable(bool on);
int prof_read(double* ms, long long* marks, int max_stages);

}  // namespace gsv
