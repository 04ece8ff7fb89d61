/*
 * gsv_oracle.c -- CPU restatement of the reference decode/render path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library, and
 * only as the checker (or as the timed CPU baseline).  The product path in
 * paper_2509_17513_b200/ never links or calls it.
 *
 * Every function restates one reference function (paths relative to
 * /root/reference/pkg/src/gsv/).  Floating point follows the reference's
 * evaluation order exactly, including where numpy delegates to OpenBLAS
 * (measured here: `P @ R.T` and stacked 3x3 `@` are fma chains
 * fma(a2,b2, fma(a1,b1, a0*b0)); einsum and elementwise numpy ops are plain
 * left-to-right mul/add).  Build with -ffp-contract=off so that only the
 * explicit fma() calls fuse.
 *
 * Parity pinning: tests/golden/ holds fixtures produced by the real reference
 * (tests/golden/make_golden.py); tests/test_oracle_golden.py checks this file
 * against them (decoded samples and fp64 values bit-exact, rects / order
 * exact, images to 1e-12).
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define OC_EXPORT __attribute__((visibility("default")))

/* ---- error codes shared with the Python wrapper -------------------------- */
enum { OC_OK = 0, OC_E_CODEC = 3, OC_E_INVALID = 1, OC_E_NOMEM = 5 };

static void set_err(char *err, int errlen, const char *msg) {
    if (err && errlen > 0) snprintf(err, (size_t)errlen, "%s", msg);
}

/* ---- CRC-32 (zlib / ISO-HDLC), as used at codec.py:260-262 -------------- */
static uint32_t crc_table[256];
static int crc_ready = 0;

static void crc_init(void) {
    for (uint32_t i = 0; i < 256; i++) {
        uint32_t c = i;
        for (int k = 0; k < 8; k++) c = (c & 1) ? (0xEDB88320u ^ (c >> 1)) : (c >> 1);
        crc_table[i] = c;
    }
    crc_ready = 1;
}

OC_EXPORT uint32_t oc_crc32_update(uint32_t crc, const uint8_t *p, size_t n) {
    if (!crc_ready) crc_init();
    crc = ~crc;
    for (size_t i = 0; i < n; i++) crc = crc_table[(crc ^ p[i]) & 0xFF] ^ (crc >> 8);
    return ~crc;
}

OC_EXPORT uint32_t oc_crc32(const uint8_t *p, size_t n) { return oc_crc32_update(0, p, n); }

/* ---- adaptive binary range decoder (_rc.py:36-42, 121-155, 304-317) ----- */
#define PROB_ONE 4096u
#define PROB_INIT 2048u
#define PROB_INIT_ZERO_PATH 3686u
#define ADAPT_SHIFT 4
#define RC_TOP (1u << 24)

OC_EXPORT void oc_new_bittree_probs(int32_t *probs, int nbytes) {
    for (int b = 0; b < nbytes; b++) {
        for (int i = 0; i < 256; i++) probs[b * 256 + i] = (int32_t)PROB_INIT;
        for (int ctx = 1; ctx < 256; ctx <<= 1) probs[b * 256 + ctx] = (int32_t)PROB_INIT_ZERO_PATH;
    }
}

/* decode_bittree: fills out[num*nbytes]; bytes past the block read as 0. */
OC_EXPORT size_t oc_decode_bittree(const uint8_t *buf, size_t n, int32_t *probs,
                                   uint8_t *out, size_t num, int nbytes) {
    size_t pos = 1; /* the first emitted byte is always zero */
    uint32_t code = 0;
    for (int i = 0; i < 4; i++) {
        uint32_t nx = pos < n ? buf[pos] : 0;
        code = (code << 8) | nx;
        pos++;
    }
    uint32_t rng = 0xFFFFFFFFu;
    for (size_t i = 0; i < num; i++) {
        for (int b = 0; b < nbytes; b++) {
            int32_t *tree = probs + b * 256;
            uint32_t ctx = 1;
            for (int k = 0; k < 8; k++) {
                uint32_t p = (uint32_t)tree[ctx];
                uint32_t bound = (rng >> 12) * p;
                if (code < bound) {
                    rng = bound;
                    tree[ctx] = (int32_t)(p + ((PROB_ONE - p) >> ADAPT_SHIFT));
                    ctx = ctx << 1;
                } else {
                    code -= bound;
                    rng -= bound;
                    tree[ctx] = (int32_t)(p - (p >> ADAPT_SHIFT));
                    ctx = (ctx << 1) | 1u;
                }
                while (rng < RC_TOP) {
                    uint32_t nx = pos < n ? buf[pos] : 0;
                    code = (code << 8) | nx;
                    pos++;
                    rng <<= 8;
                }
            }
            out[i * (size_t)nbytes + (size_t)b] = (uint8_t)(ctx & 0xFF);
        }
    }
    return pos;
}

/* byte assembly + unzigzag + plane_from_residuals (codec.py:214-217,
 * _rc.py:282-301, 326-328).  prev may be NULL when has_prev == 0. */
static void plane_from_bytes(const uint8_t *data, int nbytes, const uint32_t *prev,
                             int has_prev, int h, int w, int bits, uint32_t *plane) {
    const int64_t def = (int64_t)128 << (bits - 8);
    const uint64_t mask = (bits == 32) ? 0xFFFFFFFFull : ((1ull << bits) - 1ull);
    size_t idx = 0;
    for (int y = 0; y < h; y++) {
        for (int x = 0; x < w; x++, idx++) {
            uint64_t z = 0;
            for (int b = 0; b < nbytes; b++) z |= (uint64_t)data[idx * nbytes + b] << (8 * b);
            int64_t r = (z & 1u) ? -(int64_t)((z + 1) / 2) : (int64_t)(z / 2);
            int64_t pred;
            if (has_prev) pred = prev[idx];
            else if (x > 0) pred = plane[idx - 1];
            else if (y > 0) pred = plane[idx - (size_t)w];
            else pred = def;
            plane[idx] = (uint32_t)((uint64_t)(pred + r) & mask);
        }
    }
}

static uint32_t rd_le(const uint8_t *p, int item) {
    if (item == 1) return p[0];
    if (item == 2) return (uint32_t)p[0] | ((uint32_t)p[1] << 8);
    return (uint32_t)p[0] | ((uint32_t)p[1] << 8) | ((uint32_t)p[2] << 16) | ((uint32_t)p[3] << 24);
}

static void wr_le(uint8_t *p, uint32_t v, int item) {
    for (int i = 0; i < item; i++) p[i] = (uint8_t)(v >> (8 * i));
}

/*
 * oc_decode_payload: CodedPayload.from_bytes + decode_planes
 * (codec.py:80-92, 183-263).  `hdr` receives codec, bits, w, h, count.
 * Samples (count*h*w, promoted to u32) go to `out` if out_cap suffices.
 * Returns 0 or OC_E_CODEC with the reference's message in `err`.
 * `consumed` receives the payload end offset (caller compares with size).
 */
OC_EXPORT int oc_decode_payload(const uint8_t *blob, size_t len, uint32_t *out, size_t out_cap,
                                int32_t *hdr, size_t *consumed, char *err, int errlen) {
    char msg[160];
    if (len < 14) { set_err(err, errlen, "payload header truncated"); return OC_E_CODEC; }
    int codec = blob[0], bits = blob[1];
    int w = (int)rd_le(blob + 2, 2), h = (int)rd_le(blob + 4, 2), count = (int)rd_le(blob + 6, 2);
    uint32_t length = rd_le(blob + 10, 4);
    size_t end = 14 + (size_t)length + 4;
    hdr[0] = codec; hdr[1] = bits; hdr[2] = w; hdr[3] = h; hdr[4] = count;
    if (len < end) { set_err(err, errlen, "payload body truncated"); return OC_E_CODEC; }
    *consumed = end;
    const uint8_t *body = blob + 14;
    uint32_t checksum = rd_le(blob + 14 + length, 4);
    if (bits != 8 && bits != 16 && bits != 32) {
        snprintf(msg, sizeof msg, "bad bit width %d", bits);
        set_err(err, errlen, msg);
        return OC_E_CODEC;
    }
    const int item = bits / 8;
    const size_t hw = (size_t)h * (size_t)w;
    const size_t nsamp = (size_t)count * hw;
    const size_t expect_raw = nsamp * (size_t)item;
    if (nsamp > out_cap) { set_err(err, errlen, "output buffer too small"); return OC_E_INVALID; }
    if (codec == 0) {
        if (length != expect_raw) { set_err(err, errlen, "raw body length mismatch"); return OC_E_CODEC; }
        for (size_t i = 0; i < nsamp; i++) out[i] = rd_le(body + i * item, item);
    } else if (codec == 1) {
        if (length == 0) { set_err(err, errlen, "empty reference-coder body"); return OC_E_CODEC; }
        int flag = body[0];
        const uint8_t *coded = body + 1;
        size_t clen = (size_t)length - 1;
        if (flag == 1) {
            if (clen != expect_raw) { set_err(err, errlen, "raw fallback length mismatch"); return OC_E_CODEC; }
            for (size_t i = 0; i < nsamp; i++) out[i] = rd_le(coded + i * item, item);
        } else if (flag == 0) {
            if (clen < (size_t)count) { set_err(err, errlen, "per-plane mode table truncated"); return OC_E_CODEC; }
            size_t pos = (size_t)count;
            int nbytes = bits / 8;
            int32_t probs[4 * 256];
            oc_new_bittree_probs(probs, nbytes);
            uint8_t *data = (uint8_t *)malloc(hw * (size_t)nbytes + 1);
            if (!data) return OC_E_NOMEM;
            for (int f = 0; f < count; f++) {
                uint32_t *plane = out + (size_t)f * hw;
                const uint32_t *prev = f > 0 ? out + (size_t)(f - 1) * hw : out;
                int mode = coded[f];
                if (mode == 1) {
                    size_t e = pos + hw * (size_t)item;
                    if (e > clen) { free(data); set_err(err, errlen, "raw plane block truncated"); return OC_E_CODEC; }
                    for (size_t i = 0; i < hw; i++) plane[i] = rd_le(coded + pos + i * item, item);
                    pos = e;
                } else if (mode == 0) {
                    if (pos + 4 > clen) { free(data); set_err(err, errlen, "coded plane length truncated"); return OC_E_CODEC; }
                    uint32_t blen = rd_le(coded + pos, 4);
                    pos += 4;
                    size_t e = pos + blen;
                    if (e > clen) { free(data); set_err(err, errlen, "coded plane block truncated"); return OC_E_CODEC; }
                    oc_decode_bittree(coded + pos, blen, probs, data, hw, nbytes);
                    pos = e;
                    plane_from_bytes(data, nbytes, prev, f > 0, h, w, bits, plane);
                } else {
                    free(data);
                    snprintf(msg, sizeof msg, "unknown plane mode %d", mode);
                    set_err(err, errlen, msg);
                    return OC_E_CODEC;
                }
            }
            free(data);
            if (pos != clen) { set_err(err, errlen, "trailing bytes after the last plane block"); return OC_E_CODEC; }
        } else {
            snprintf(msg, sizeof msg, "unknown body flag %d", flag);
            set_err(err, errlen, msg);
            return OC_E_CODEC;
        }
    } else if (codec == 2) {
        set_err(err, errlen, "external codec payload: no plugin registered");
        return OC_E_CODEC;
    } else {
        snprintf(msg, sizeof msg, "unknown codec id %d", codec);
        set_err(err, errlen, msg);
        return OC_E_CODEC;
    }
    /* CRC-32 of the little-endian sample bytes, all planes incl. padding */
    uint32_t crc = 0;
    uint8_t tmp[4096];
    size_t i = 0;
    while (i < nsamp) {
        size_t m = 0;
        while (i < nsamp && m + (size_t)item <= sizeof tmp) { wr_le(tmp + m, out[i], item); m += (size_t)item; i++; }
        crc = oc_crc32_update(crc, tmp, m);
    }
    if (crc != checksum) {
        set_err(err, errlen, "checksum mismatch (corrupt or truncated payload)");
        return OC_E_CODEC;
    }
    return OC_OK;
}

/* dequantize_codes (quantize.py:114-117): rmin + code/top*(rmax-rmin) */
OC_EXPORT void oc_dequantize(const uint32_t *codes, size_t n, int bits, double rmin, double rmax,
                             double *out, size_t out_stride) {
    const double top = (double)((bits == 32) ? 4294967295.0 : (double)((1ull << bits) - 1ull));
    const double span = rmax - rmin;
    for (size_t i = 0; i < n; i++) out[i * out_stride] = rmin + ((double)codes[i] / top) * span;
}

/* ---- projection (render.py:185-287) -------------------------------------- */
typedef struct {
    double R[9];   /* world-to-camera rotation, row-major */
    double t[3];
    double fx, fy, cx, cy;
    double near_;
    double bg[3];
    int32_t width, height;
} oc_camera;

static const double SH_C0 = 0.28209479177387814;
static const double SH_C1 = 0.4886025119029199;
static const double SH_C2[5] = {1.0925484305920792, -1.0925484305920792, 0.31539156525252005,
                                -1.0925484305920792, 0.5462742152960396};
static const double SH_C3[7] = {-0.5900435899266435, 2.890611442640554, -0.4570457994644658,
                                0.3731763325901154, -0.4570457994644658, 1.445305721320277,
                                -0.5900435899266435};

static double np_max(double a, double b) { return (a != a) ? a : ((b != b) ? b : (a >= b ? a : b)); }
static double np_min(double a, double b) { return (a != a) ? a : ((b != b) ? b : (a <= b ? a : b)); }
static double np_clip01(double v) { return np_min(np_max(v, 0.0), 1.0); }

/* 3x3 @ 3x3 as OpenBLAS evaluates it: C[i][k] = fma(a2,b2, fma(a1,b1, a0*b0)) */
static void mm3(const double *A, const double *B, double *C) {
    for (int i = 0; i < 3; i++)
        for (int k = 0; k < 3; k++)
            C[i * 3 + k] = fma(A[i * 3 + 2], B[6 + k], fma(A[i * 3 + 1], B[3 + k], A[i * 3 + 0] * B[k]));
}

/* eval_sh_colors (render.py:202-237) for one splat; center = -R^T t */
static void sh_color(const double *pos, const double *sh, int deg, const double *center, double *rgb) {
    double col[3];
    for (int c = 0; c < 3; c++) col[c] = SH_C0 * sh[c];
    if (deg >= 1) {
        double dx = pos[0] - center[0], dy = pos[1] - center[1], dz = pos[2] - center[2];
        double nrm = sqrt((dx * dx + dy * dy) + dz * dz);
        if (nrm == 0.0) nrm = 1.0;
        double x = dx / nrm, y = dy / nrm, z = dz / nrm;
        for (int c = 0; c < 3; c++)
            col[c] = ((col[c] - (SH_C1 * y) * sh[3 + c]) + (SH_C1 * z) * sh[6 + c]) - (SH_C1 * x) * sh[9 + c];
        if (deg >= 2) {
            double xx = x * x, yy = y * y, zz = z * z, xy = x * y, yz = y * z, xz = x * z;
            for (int c = 0; c < 3; c++) {
                double v = col[c];
                v = v + (SH_C2[0] * xy) * sh[12 + c];
                v = v + (SH_C2[1] * yz) * sh[15 + c];
                v = v + (SH_C2[2] * ((2.0 * zz - xx) - yy)) * sh[18 + c];
                v = v + (SH_C2[3] * xz) * sh[21 + c];
                v = v + (SH_C2[4] * (xx - yy)) * sh[24 + c];
                col[c] = v;
            }
            if (deg >= 3) {
                for (int c = 0; c < 3; c++) {
                    double v = col[c];
                    v = v + ((SH_C3[0] * y) * (3.0 * xx - yy)) * sh[27 + c];
                    v = v + ((SH_C3[1] * xy) * z) * sh[30 + c];
                    v = v + ((SH_C3[2] * y) * ((4.0 * zz - xx) - yy)) * sh[33 + c];
                    v = v + ((SH_C3[3] * z) * ((2.0 * zz - 3.0 * xx) - 3.0 * yy)) * sh[36 + c];
                    v = v + ((SH_C3[4] * x) * ((4.0 * zz - xx) - yy)) * sh[39 + c];
                    v = v + ((SH_C3[5] * z) * (xx - yy)) * sh[42 + c];
                    v = v + ((SH_C3[6] * x) * (xx - 3.0 * yy)) * sh[45 + c];
                    col[c] = v;
                }
            }
        }
    }
    for (int c = 0; c < 3; c++) rgb[c] = np_clip01(col[c] + 0.5);
}

/*
 * oc_project: project_set for every splat (no compaction; `alive` marks the
 * survivors).  Arrays are SoA-by-row like the reference: pos (n,3), rot (n,4),
 * scales (n,3), sh (n, shdim).  Outputs: means (n,2), cov2d (n,4: 00,01,10,11),
 * depth (n), colors (n,3), rects (n,4: x0,x1,y0,y1), alive (n).
 */
OC_EXPORT void oc_project(int64_t n, const double *pos, const double *rot, const double *scl,
                          const double *sh, int deg, const oc_camera *cam, double *means,
                          double *cov2d, double *depth, double *colors, int64_t *rects,
                          uint8_t *alive) {
    const double *R = cam->R;
    double RT[9];
    for (int i = 0; i < 3; i++)
        for (int j = 0; j < 3; j++) RT[i * 3 + j] = R[j * 3 + i];
    double center[3];
    for (int i = 0; i < 3; i++) {
        const double m0 = -R[0 * 3 + i], m1 = -R[1 * 3 + i], m2 = -R[2 * 3 + i];
        center[i] = fma(m2, cam->t[2], fma(m1, cam->t[1], m0 * cam->t[0]));
    }
    const int shdim = 3 * (deg + 1) * (deg + 1);
    for (int64_t i = 0; i < n; i++) {
        const double *p = pos + 3 * i;
        double cp[3];
        for (int r = 0; r < 3; r++)
            cp[r] = fma(R[r * 3 + 2], p[2], fma(R[r * 3 + 1], p[1], R[r * 3 + 0] * p[0])) + cam->t[r];
        const double d = cp[2];
        int al = d > cam->near_;
        /* _quat_to_rotmats */
        const double *q = rot + 4 * i;
        double qn = sqrt(((q[0] * q[0] + q[1] * q[1]) + q[2] * q[2]) + q[3] * q[3]);
        double w = q[0] / qn, x = q[1] / qn, y = q[2] / qn, z = q[3] / qn;
        double m[9];
        m[0] = 1 - 2 * (y * y + z * z);
        m[1] = 2 * (x * y - w * z);
        m[2] = 2 * (x * z + w * y);
        m[3] = 2 * (x * y + w * z);
        m[4] = 1 - 2 * (x * x + z * z);
        m[5] = 2 * (y * z - w * x);
        m[6] = 2 * (x * z - w * y);
        m[7] = 2 * (y * z + w * x);
        m[8] = 1 - 2 * (x * x + y * y);
        const double *s = scl + 3 * i;
        double s2[3] = {s[0] * s[0], s[1] * s[1], s[2] * s[2]};
        /* einsum("nij,nj,nkj->nik"): sum over j of (m_ij * s2_j) * m_kj */
        double cw[9];
        for (int a = 0; a < 3; a++)
            for (int k = 0; k < 3; k++)
                cw[a * 3 + k] = ((m[a * 3 + 0] * s2[0]) * m[k * 3 + 0] + (m[a * 3 + 1] * s2[1]) * m[k * 3 + 1]) +
                                (m[a * 3 + 2] * s2[2]) * m[k * 3 + 2];
        double tmp[9], cc[9];
        mm3(R, cw, tmp);
        mm3(tmp, RT, cc);
        const double zz = al ? d : 1.0;
        const double u = cam->fx * cp[0] / zz + cam->cx;
        const double v = cam->fy * cp[1] / zz + cam->cy;
        double J[6] = {cam->fx / zz, 0.0, -cam->fx * cp[0] / (zz * zz),
                       0.0, cam->fy / zz, -cam->fy * cp[1] / (zz * zz)};
        /* einsum("nab,nbc,ndc->nad"): b outer, c inner, plain products */
        double c2[4];
        for (int a = 0; a < 2; a++)
            for (int dd = 0; dd < 2; dd++) {
                double acc = 0.0;
                int first = 1;
                for (int b = 0; b < 3; b++)
                    for (int c = 0; c < 3; c++) {
                        double pr = (J[a * 3 + b] * cc[b * 3 + c]) * J[dd * 3 + c];
                        if (first) { acc = pr; first = 0; } else acc = acc + pr;
                    }
                c2[a * 2 + dd] = acc;
            }
        c2[0] += 0.3;
        c2[3] += 0.3;
        const double A = c2[0], B = c2[1], C = c2[3];
        const double hm = (A - C) / 2;
        const double lam = (A + C) / 2 + sqrt(hm * hm + B * B);
        const double radius = ceil(3.0 * sqrt(np_max(lam, 0.0)));
        const double x0 = np_max(floor(u - radius), 0.0);
        const double x1 = np_min(floor(u + radius) + 1, (double)cam->width);
        const double y0 = np_max(floor(v - radius), 0.0);
        const double y1 = np_min(floor(v + radius) + 1, (double)cam->height);
        al = al && (x0 < x1) && (y0 < y1);
        alive[i] = (uint8_t)al;
        means[2 * i] = u;
        means[2 * i + 1] = v;
        for (int k = 0; k < 4; k++) cov2d[4 * i + k] = c2[k];
        depth[i] = d;
        if (al) {
            rects[4 * i] = (int64_t)x0; rects[4 * i + 1] = (int64_t)x1;
            rects[4 * i + 2] = (int64_t)y0; rects[4 * i + 3] = (int64_t)y1;
        } else {
            rects[4 * i] = rects[4 * i + 1] = rects[4 * i + 2] = rects[4 * i + 3] = 0;
        }
        sh_color(p, sh + (int64_t)shdim * i, deg, center, colors + 3 * i);
    }
}

/*
 * oc_composite: _composite_arrays + _composite (render.py:301-356) over
 * splats already in depth order.  cov2d (m,4) -> conic inverse inside.
 * img (H,W,3) fp64 output, clipped to [0,1].  evals (optional) counts
 * evaluated (pixel, splat) pairs (T >= 1e-4 at test time).
 */
OC_EXPORT void oc_composite(int64_t m, const double *means, const double *cov2d,
                            const double *colors, const double *opac, const int64_t *rects,
                            int width, int height, const double *bg, double *img, double *trans,
                            int64_t *evals) {
    const size_t npix = (size_t)width * (size_t)height;
    for (size_t i = 0; i < npix * 3; i++) img[i] = 0.0;
    for (size_t i = 0; i < npix; i++) trans[i] = 1.0;
    int64_t ev = 0;
    for (int64_t i = 0; i < m; i++) {
        const double *c = cov2d + 4 * i;
        const double det = c[0] * c[3] - c[1] * c[1];
        const double ia = c[3] / det, ib = -c[1] / det, ic = c[0] / det;
        const int64_t x0 = rects[4 * i], x1 = rects[4 * i + 1], y0 = rects[4 * i + 2], y1 = rects[4 * i + 3];
        const double mx = means[2 * i], my = means[2 * i + 1];
        const double op = opac[i];
        const double cr = colors[3 * i], cg = colors[3 * i + 1], cb = colors[3 * i + 2];
        for (int64_t y = y0; y < y1; y++) {
            const double dy = (double)y - my;
            for (int64_t x = x0; x < x1; x++) {
                const size_t pix = (size_t)y * (size_t)width + (size_t)x;
                const double t = trans[pix];
                if (t < 1e-4) continue;
                ev++;
                const double dx = (double)x - mx;
                double power = -0.5 * (ia * dx * dx + 2.0 * ib * dx * dy + ic * dy * dy);
                if (power > 0.0) power = 0.0;
                double alpha = op * exp(power);
                if (alpha > 0.99) alpha = 0.99;
                if (alpha <= 0.0) continue;
                const double wgt = t * alpha;
                img[3 * pix] += wgt * cr;
                img[3 * pix + 1] += wgt * cg;
                img[3 * pix + 2] += wgt * cb;
                trans[pix] = t * (1.0 - alpha);
            }
        }
    }
    for (size_t p = 0; p < npix; p++) {
        const double t = trans[p];
        for (int k = 0; k < 3; k++) img[3 * p + k] = np_clip01(img[3 * p + k] + t * bg[k]);
    }
    if (evals) *evals = ev;
}

/* ---- delta folding (motion.py:24-46, 165-193, 218-235) ------------------- */
/*
 * In place over n splats for `nd` deltas; delta arrays are concatenated
 * (nd, stride_n, ...) with the first n rows of each used (FrameDelta.prefix).
 * Returns 0, or 1 if a zero quaternion would be normalised
 * (quat_normalize raises InvalidInputError).
 */
OC_EXPORT int oc_fold_deltas(int64_t n, double *pos, double *rot, double *scl, double *opac,
                             double *sh, int shdim, int nd, const int64_t *delta_len,
                             const double *const *d_trans, const double *const *d_rot,
                             const double *const *d_scl, const double *const *d_opac,
                             const double *const *d_sh) {
    for (int d = 0; d < nd; d++) {
        (void)delta_len;
        const double *dt = d_trans[d], *dq = d_rot[d], *ds = d_scl[d], *dop = d_opac[d], *dsh = d_sh[d];
        /* apply_rigid: rotations = normalize(dq * q); positions += t */
        for (int64_t i = 0; i < n; i++) {
            const double aw = dq[4 * i], ax = dq[4 * i + 1], ay = dq[4 * i + 2], az = dq[4 * i + 3];
            double *q = rot + 4 * i;
            const double bw = q[0], bx = q[1], by = q[2], bz = q[3];
            const double w = ((aw * bw - ax * bx) - ay * by) - az * bz;
            const double x = ((aw * bx + ax * bw) + ay * bz) - az * by;
            const double y = ((aw * by - ax * bz) + ay * bw) + az * bx;
            const double z = ((aw * bz + ax * by) - ay * bx) + az * bw;
            const double nrm = sqrt(((w * w + x * x) + y * y) + z * z);
            if (nrm == 0.0) return 1;
            q[0] = w / nrm; q[1] = x / nrm; q[2] = y / nrm; q[3] = z / nrm;
        }
        for (int64_t i = 0; i < n; i++)
            for (int k = 0; k < 3; k++) pos[3 * i + k] = pos[3 * i + k] + dt[3 * i + k];
        /* apply_residual */
        for (int64_t i = 0; i < n; i++) {
            for (int k = 0; k < 3; k++) scl[3 * i + k] = np_max(scl[3 * i + k] + ds[3 * i + k], 1e-7);
            opac[i] = np_clip01(opac[i] + dop[i]);
            for (int k = 0; k < shdim; k++) sh[(int64_t)shdim * i + k] = sh[(int64_t)shdim * i + k] + dsh[(int64_t)shdim * i + k];
        }
    }
    return 0;
}
