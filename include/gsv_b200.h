/*
 * gsv_b200.h -- C ABI of libgsv_b200.so, the B200-native decode-and-render
 * path of the `gsv` (4DGCPro) reference package.
 *
 * Plain pointers and sizes only (no torch / C++ types).  Every entry point
 * replaces one reference interface; paths are relative to
 * /root/reference/pkg/src/gsv/.  The reference is pure Python, so the
 * reference-side binding is a ctypes stub; the package
 * paper_2509_17513_b200 is exactly that stub plus the reference's
 * dataclasses.
 *
 * Errors: every int-returning call returns GSV_OK or one of GSV_E_*; the
 * matching message (the reference's exception text, e.g.
 * "group 0 layer 3 channel sh[4]: checksum mismatch (corrupt or truncated
 * payload)") is available from gsv_last_error() on the calling thread.
 * GSV_E_INVALID_INPUT / FORMAT / CODEC map to the reference's
 * InvalidInputError / FormatError / CodecError (errors.py:8-17).
 *
 * Pointers documented as "device" are CUDA device addresses on the
 * session's device; "host" pointers are ordinary (ideally pinned) memory.
 * All device work is issued on the session stream; calls that return host
 * data synchronise that stream.
 */
#ifndef GSV_B200_H
#define GSV_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GSV_ABI_VERSION 1

enum {
    GSV_OK = 0,
    GSV_E_INVALID_INPUT = 1, /* errors.InvalidInputError */
    GSV_E_FORMAT = 2,        /* errors.FormatError */
    GSV_E_CODEC = 3,         /* errors.CodecError */
    GSV_E_CUDA = 4,          /* CUDA runtime failure (no reference counterpart) */
    GSV_E_NOMEM = 5
};

typedef struct gsv_session gsv_session; /* one CUDA device + stream + scratch */
typedef struct gsv_video gsv_video;     /* a decoded layer prefix, resident in HBM */

/* Camera (render.py:43-120): x_cam = R x_world + t, pinhole fx fy cx cy. */
typedef struct gsv_camera {
    double rotation[9]; /* row-major world-to-camera */
    double translation[3];
    double fx, fy, cx, cy;
    double near_plane;
    double background[3];
    int32_t width, height;
} gsv_camera;

/* Header of a container (container.py:73-81) */
typedef struct gsv_info {
    int32_t version, layer_count, sh_degree, group_count;
    int32_t fps_num, fps_den;
    uint32_t flags;
    float bounds[6];
    uint64_t header_bytes; /* header + directory size */
} gsv_info;

typedef struct gsv_group_info { /* container.py:54-70 */
    uint32_t start_frame;
    uint32_t frame_count;
    uint32_t position_bits;
    uint32_t layer_counts[64];    /* first layer_count entries valid */
    uint32_t channel_counts[64];  /* entries per layer */
} gsv_group_info;

typedef struct gsv_entry_info { /* container.py:44-51 */
    int32_t attribute; /* quantize.py:23-30 codes */
    int32_t component;
    int32_t bits;
    uint64_t offset, size;
    float range_min, range_max;
} gsv_entry_info;

/* Per-render statistics (exposed for tests and the roofline accounting). */
typedef struct gsv_render_stats {
    int64_t n_splats;   /* splats projected (layer prefix size) */
    int64_t n_visible;  /* survivors of project_set's culls */
    int64_t n_keys;     /* (tile, splat) overlaps of the visible splats */
    int32_t tiles_x, tiles_y;
    int64_t n_keys_emitted; /* keys actually emitted (saturated tiles get none in later rounds) */
} gsv_render_stats;

const char* gsv_last_error(void);
int gsv_last_error_kind(void);
int gsv_abi_version(void);

/* ---- sessions ---------------------------------------------------------- */
/* stream: a cudaStream_t (0 = the session creates its own non-blocking stream). */
int gsv_session_create(int device, uintptr_t stream, gsv_session** out);
void gsv_session_destroy(gsv_session* s);
/* Block until all work issued on the session stream has finished. */
int gsv_session_sync(gsv_session* s);

/* ---- container structure (read_structure / read_container_info,
 *      container.py:151-196); host only ------------------------------------ */
int gsv_read_info(const uint8_t* data, size_t len, gsv_info* out);
int gsv_read_group(const uint8_t* data, size_t len, int group, gsv_group_info* out);
int gsv_read_entry(const uint8_t* data, size_t len, int group, int layer, int entry,
                   gsv_entry_info* out);
/* the whole directory in one parse: groups[group_count] and every entry in
 * (group, layer, entry) order; *n_entries gets the entry count (also when the
 * buffers are too small, which fails with GSV_E_INVALID_INPUT). */
int gsv_read_directory(const uint8_t* data, size_t len, gsv_group_info* groups, size_t group_cap,
                       gsv_entry_info* entries, size_t entry_cap, size_t* n_entries);

/* ---- decode (read_layers / decode_video, container.py:260-310,
 *      pipeline.py:350-359) --------------------------------------------------
 * gsv_video_open: host container bytes; stages the layer-prefix payload
 * bytes of every group into HBM (only layers <= up_to_layer are copied,
 * mirroring the reference's prefix reads), range-decodes and CRC-checks
 * every run on the GPU and validates the result in the reference's error
 * order.  up_to_layer == -1 means all layers (decode_video's None).
 * gsv_video_open_resident: same, but `dev_data` already holds the whole
 * container in HBM (only `data` is read on the host, for the directory);
 * the device allocation must extend at least 64 bytes past the container
 * (the decoders read whole 16-byte chunks). */
int gsv_video_open(gsv_session* s, const uint8_t* data, size_t len, int up_to_layer,
                   gsv_video** out);
int gsv_video_open_resident(gsv_session* s, const uint8_t* data, size_t len,
                            const uint8_t* dev_data, int up_to_layer, gsv_video** out);
/* groups [g0, g1) only (a streaming player's unit): only their layer-prefix
 * bytes are staged and decoded; frames are numbered 0.. within the range. */
int gsv_video_open_groups(gsv_session* s, const uint8_t* data, size_t len, int up_to_layer, int g0,
                          int g1, gsv_video** out);
/* an arbitrary list of groups (a shard of a sequence: e.g. the
 * longest-processing-time assignment of groups to ranks), opened in list
 * order; frames are numbered 0.. group after group in that order.  dev_data:
 * NULL (stage the groups' layer-prefix bytes from `data`) or the whole
 * container resident in HBM as for gsv_video_open_resident.  Groups must be
 * in range and distinct. */
int gsv_video_open_group_list(gsv_session* s, const uint8_t* data, size_t len, const uint8_t* dev_data,
                              int up_to_layer, const int32_t* groups, int ngroups, gsv_video** out);
/* Does not wait: the video's device memory is released once the work
 * enqueued on its session so far has completed (reaped by later opens and
 * closes, or gsv_session_destroy).  Host outputs of earlier render_batch
 * calls are complete after gsv_session_sync. */
void gsv_video_close(gsv_video* v);
int gsv_video_frame_count(const gsv_video* v);
int gsv_video_decoded_layers(const gsv_video* v);
/* DecodedVideo.frame(t) (container.py:219-223): group index of frame t, or -1 */
int gsv_video_group_of(const gsv_video* v, int t);
/* number of splats of every frame of group g at this layer prefix */
int64_t gsv_video_group_splats(const gsv_video* v, int g);
/* fp64 SoA of frame t (device outputs): pos (n,3) rot (n,4) scl (n,3) opac (n) sh (n,shdim) */
int gsv_video_frame_values(gsv_video* v, int t, double* pos, double* rot, double* scl,
                           double* opac, double* sh);
/* decoded integer samples of frame t, (layer, slot) order, u32 (device), for parity tests:
 * out[(layer_base + j) * nslots + slot] for splat j of that layer. */
int gsv_video_frame_codes(gsv_video* v, int t, uint32_t* out);

/* ---- render (render_set / render_progressive, render.py:382-398) --------
 * Output: fp32 RGB (height, width, 3) in [0,1] (device), optional u8 RGB
 * rounded like write_ppm (render.py:165-169).  Either output may be NULL. */
int gsv_video_render(gsv_video* v, int t, const gsv_camera* cam, float* out_rgb,
                     uint8_t* out_rgb8, gsv_render_stats* stats);
/* Render `count` frames of v (frames[j]) frame-parallel on `nstreams`
 * auxiliary streams (joined back into the session stream).  Per frame j:
 * out_rgb[j] (device fp32), out_rgb8[j] (device u8) and/or host_rgb8[j]
 * (host, ideally pinned, u8 copied D2H on the frame's stream); any array or
 * entry may be NULL.  check != 0: synchronise and verify the tile-key
 * capacity, re-rendering the batch after growing it if needed; check == 0:
 * fully asynchronous (capacity learnt from earlier renders). */
int gsv_video_render_batch(gsv_video* v, const int32_t* frames, int count, const gsv_camera* cam,
                           float* const* out_rgb, uint8_t* const* out_rgb8,
                           uint8_t* const* host_rgb8, int nstreams, int check);
/* after unchecked batches: GSV_OK, or GSV_E_NOMEM if any frame overflowed */
int gsv_session_check_capacity(gsv_session* s);
/* Decode + render every frame of the listed groups (all groups when groups
 * is NULL) straight from host container bytes into host u8 RGB frames
 * (host_rgb8[j]: frame j in group-list order, group-major; pinned memory
 * makes the copies asynchronous): the reference's decode_video(path, k)
 * followed by render_set + write_ppm's rounding of every frame
 * (pipeline.py:350-359, render.py:382-385, 165-169; cli.py:122-131 per
 * frame), pipelined in one call -- group uploads, opens and renders with
 * read-back overlap; CRC and structural errors are reported as decode_video
 * raises them (first in decode order), after the pipeline has drained.
 * frames_out (may be NULL): frames written.  The session keeps the device
 * payload slots (the container's layer-prefix bytes) for its next call. */
int gsv_render_sequence_host(gsv_session* s, const uint8_t* data, size_t len, int up_to_layer,
                             const int32_t* groups, int ngroups, const gsv_camera* cam,
                             uint8_t* const* host_rgb8, int nstreams, int64_t* frames_out);
/* The general form: dev_data (may be NULL) holds the whole container already
 * in HBM (then nothing is uploaded; `data` is still read for the directory
 * and payload headers); frame_begin / frame_end (may be NULL: whole groups)
 * give per listed group the group-relative frames [b, e) to render (a
 * rank's pieces of a sharded sequence; the group is still opened, and its
 * CRC checked, whole); per output frame j any of out_rgb[j] (device fp32),
 * out_rgb8[j] (device u8), host_rgb8[j] (host u8); at least one array. */
int gsv_render_sequence(gsv_session* s, const uint8_t* data, size_t len, const uint8_t* dev_data,
                        int up_to_layer, const int32_t* groups, int ngroups, const int32_t* frame_begin,
                        const int32_t* frame_end, const gsv_camera* cam, float* const* out_rgb,
                        uint8_t* const* out_rgb8, uint8_t* const* host_rgb8, int nstreams, int64_t* frames_out);
/* render an fp64 SoA Gaussian set resident in HBM (render_set) */
int gsv_render_soa(gsv_session* s, int64_t n, int sh_degree, const double* pos,
                   const double* rot, const double* scl, const double* opac, const double* sh,
                   const gsv_camera* cam, float* out_rgb, uint8_t* out_rgb8,
                   gsv_render_stats* stats);
/* render(list[Splat2D]) (render.py:359-379) on device fp64 arrays:
 * means (n,2), cov2d (n,2,2), depth (n), colors (n,3), opacities (n);
 * rects from cov2d as render() computes them, stable depth order. */
int gsv_render_splats2d(gsv_session* s, int64_t n, const double* means, const double* cov2d,
                        const double* depth, const double* colors, const double* opac,
                        const gsv_camera* cam, float* out_rgb, uint8_t* out_rgb8,
                        gsv_render_stats* stats);
/* psnr (metrics.py:31-38) building block: sum over n elements of (a - b)^2
 * in fp64, a and b device arrays of fp32 (is_f64 = 0) or fp64; *out is host. */
int gsv_sqdiff(gsv_session* s, const void* a, const void* b, int64_t n, int is_f64, double* out);
/* ssim (metrics.py:48-65): mean SSIM of the channel-mean images of two
 * device (height, width, 3) images, fp32 (is_f64 = 0) or fp64; *out is host. */
int gsv_ssim(gsv_session* s, const void* a, const void* b, int height, int width, int is_f64,
             double* out);
/* reconstruct_frame's fold (motion.py:165-235), in place on device SoA arrays:
 * for each of nd deltas (device pointer tables on the host side):
 *   q <- normalize(dq * q); p += dt; s <- max(s + ds, 1e-7);
 *   o <- clip(o + do, 0, 1); sh += dsh
 * Delta rows beyond n are ignored (FrameDelta.prefix). */
int gsv_fold_deltas(gsv_session* s, int64_t n, int shdim, double* pos, double* rot,
                    double* scl, double* opac, double* sh, int nd,
                    const double* const* d_trans, const double* const* d_rot,
                    const double* const* d_scl, const double* const* d_opac,
                    const double* const* d_sh);
/* projection outputs for parity tests (device): for every splat i,
 * rect[i] = (x0,x1,y0,y1) or all zero when culled, depth[i], order[r] = i of
 * depth-rank r (visible splats first, stable), tile_count[i]. */
int gsv_project_debug(gsv_session* s, int64_t n, int sh_degree, const double* pos,
                      const double* rot, const double* scl, const double* opac,
                      const double* sh, const gsv_camera* cam, int32_t* rects, double* depth,
                      int32_t* order, int32_t* tile_count, int64_t* n_visible);

/* the same for frame t of a decoded video, through the production projection
 * (integer codes dequantised in registers from the code planes) -- the path
 * gsv_video_render and gsv_video_render_batch run */
int gsv_video_project_debug(gsv_video* v, int t, const gsv_camera* cam, int32_t* rects, double* depth,
                            int32_t* order, int32_t* tile_count, int64_t* n_visible);

/* ---- codec (decode_planes, codec.py:226-263): one payload, host buffers --
 * hdr receives codec, bits, width, height, count; samples (count*h*w) as u32. */
int gsv_decode_payload_host(gsv_session* s, const uint8_t* blob, size_t len,
                            uint32_t* samples, size_t capacity, int32_t* hdr);

/* ---- encoder: GPU quantisation + codec-1 range coding --
 * gsv_quantize_channels: quantize_channel (quantize.py:79-106, f32 range
 * cover quantize.py:62-76) of nch channels of one group, each channel a
 * (frames, n) block of fp64 values on the device (value (f, j) at
 * values[f * frame_stride + j]), written as frames padded planes
 * (flatten_to_plane, quantize.py:160-167) of width*height LE samples at
 * `planes` (device); range_min / range_max receive the stored f32 range.
 * Non-finite input -> GSV_E_INVALID_INPUT "non-finite channel values".
 * Synchronises the session stream. */
typedef struct gsv_quant_channel {
    const double* values;       /* device */
    uint8_t* planes;            /* device: frames * width * height * bits/8 bytes */
    uint64_t frame_stride;      /* elements between frames (>= n) */
    uint32_t frames, n, width, height, bits;
    float range_min, range_max; /* out */
} gsv_quant_channel;
int gsv_quantize_channels(gsv_session* s, gsv_quant_channel* ch, int nch);

/* gsv_encode_runs: for every run, the codec-1 payload body of
 * _encode_reference_body (codec.py:137-163: per-plane range coding through
 * encode_bittree, _rc.py:55-118, RAW planes where coding does not pay, the
 * whole-run raw fallback) into `body` (device, gsv_encode_body_capacity
 * bytes), and the payload CRC-32 of the samples (encode_planes,
 * codec.py:166-180).  body_len / checksum are written back; the payload is
 * header `<BBHHHHI` + body[0:body_len] + checksum.  Synchronises. */
typedef struct gsv_encode_run {
    const uint8_t* samples; /* device: count * width * height LE samples */
    uint8_t* body;          /* device */
    uint32_t count, width, height, bits;
    uint64_t body_len;      /* out */
    uint32_t checksum;      /* out */
    uint32_t reserved;
} gsv_encode_run;
uint64_t gsv_encode_body_capacity(uint32_t count, uint32_t width, uint32_t height, uint32_t bits);
int gsv_encode_runs(gsv_session* s, gsv_encode_run* runs, int nruns);

/* ---- instrumentation ------------------------------------------------------
 * gsv_kernel_launches: kernels launched by this library so far (process-wide).
 * gsv_profile_enable(1) resets and starts stage timing with CUDA events on the
 * launching streams; gsv_profile_read fills per-stage total ms and interval
 * counts for stages 0..7 = project, depth sort, key emission, tile sort,
 * tile ranges, composite, range decode, CRC. */
long long gsv_kernel_launches(void);
int gsv_profile_enable(int enable);
int gsv_profile_read(double* ms, long long* intervals, int max_stages);

/* ---- synthetic input tooling (encoder side; not on the decode path) ------
 * Range-code one run of planes like codec.py:105-180 (codec 1) into `out`
 * (payload body, without the 14-B header / CRC).  Returns body length or <0. */
int64_t gsv_encode_reference_body(const uint32_t* samples, int count, int h, int w, int bits,
                                  uint8_t* out, size_t capacity);
uint32_t gsv_crc32(const uint8_t* data, size_t len);

#ifdef __cplusplus
}
#endif
#endif /* GSV_B200_H */
