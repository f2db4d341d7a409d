// sad_codec.cu — the `.sad` container (codec.hpp / codec.cpp of the reference), host side, and the
// decode pipeline: bytes -> sites (host, glibc trig so decoded doubles match the reference bit for
// bit) -> device full refresh -> device render.  Wire format (codec.hpp:9-19, 42-45):
//   "SADF" | u16 version | u32 W | u32 H | u32 count | 10 f32 ranges | count x 16-byte records.
#include "../../include/sad_b200.h"

#include <cmath>
#include <cstdio>
#include <cstring>
#include <limits>
#include <string>
#include <vector>

extern "C" void sad_internal_set_error(const char* msg);  // sad_runtime.cu: shared sad_last_error()

namespace {

constexpr double kPi = 3.14159265358979323846;
constexpr uint16_t kVersion = 1;

sad_status fail(sad_status code, const std::string& m) {
    sad_internal_set_error(m.c_str());
    return code;
}

double dclamp(double v, double lo, double hi) { return v < lo ? lo : (hi < v ? hi : v); }

uint32_t unorm_encode(double value, double lo, double scale, uint32_t max_code) {
    double norm = dclamp((value - lo) / scale, 0.0, 1.0);
    return static_cast<uint32_t>(std::lround(norm * max_code));
}

double unorm_decode(uint32_t code, double lo, double scale, uint32_t max_code) {
    return lo + (static_cast<double>(code) / max_code) * scale;
}

uint16_t f2h(float f) {  // IEEE binary16, round to nearest even (half.hpp:10-36 semantics)
    uint32_t x;
    std::memcpy(&x, &f, 4);
    uint16_t sign = static_cast<uint16_t>((x >> 16) & 0x8000u);
    uint32_t mant = x & 0x7fffffu, e8 = (x >> 23) & 0xffu;
    if (e8 == 255) return sign | 0x7c00u | (mant ? (0x200u | (mant >> 13)) : 0u);
    int e = static_cast<int>(e8) - 112;
    if (e >= 31) return sign | 0x7c00u;
    if (e <= 0) {
        if (e < -10) return sign;
        mant |= 0x800000u;
        int sh = 14 - e;
        uint32_t hm = mant >> sh, rem = mant & ((1u << sh) - 1u), half = 1u << (sh - 1);
        if (rem > half || (rem == half && (hm & 1u))) hm++;
        return static_cast<uint16_t>(sign | hm);
    }
    uint16_t h = static_cast<uint16_t>(sign | (e << 10) | (mant >> 13));
    uint32_t rem = mant & 0x1fffu;
    if (rem > 0x1000u || (rem == 0x1000u && (h & 1u))) h++;
    return h;
}

float h2f(uint16_t h) {
    uint32_t sign = static_cast<uint32_t>(h & 0x8000u) << 16, e = (h >> 10) & 0x1fu, m = h & 0x3ffu, x;
    if (e == 0) {
        if (m == 0) {
            x = sign;
        } else {
            int k = -1;
            do {
                k++;
                m <<= 1;
            } while (!(m & 0x400u));
            x = sign | static_cast<uint32_t>(127 - 15 - k) << 23 | ((m & 0x3ffu) << 13);
        }
    } else if (e == 31) {
        x = sign | 0x7f800000u | (m << 13);
    } else {
        x = sign | ((e - 15 + 127) << 23) | (m << 13);
    }
    float f;
    std::memcpy(&f, &x, 4);
    return f;
}

struct Ranges {  // QuantRanges (codec.hpp:23-28)
    double lt_min = 0, lt_scale = 1e-6, r_min = 0, r_scale = 1e-6;
    double c_min[3] = {0, 0, 0}, c_scale[3] = {1e-6, 1e-6, 1e-6};
};

// compute_ranges (codec.cpp:53-88): min rounded down and scale rounded up through float32 so the
// file's scalars still cover the active population.
Ranges ranges(const sad_sites_view* s) {
    Ranges q;
    bool any = false;
    double lo[5] = {0}, hi[5] = {0};
    for (size_t i = 0; i < s->size; i++) {
        if (!s->active[i]) continue;
        double v[5] = {s->log_tau[i], s->radius[i], s->col_r[i], s->col_g[i], s->col_b[i]};
        for (int k = 0; k < 5; k++) {
            if (!any) {
                lo[k] = hi[k] = v[k];
            } else {
                lo[k] = (v[k] < lo[k]) ? v[k] : lo[k];
                hi[k] = (hi[k] < v[k]) ? v[k] : hi[k];
            }
        }
        any = true;
    }
    if (!any) return q;
    auto cover = [](double lv, double hv, double& mn_o, double& sc_o) {
        float mn = static_cast<float>(lv);
        if (static_cast<double>(mn) > lv) mn = std::nextafterf(mn, -std::numeric_limits<float>::infinity());
        double span = hv - static_cast<double>(mn);
        float sc = static_cast<float>(span < 1e-6 ? 1e-6 : span);
        while (static_cast<double>(mn) + static_cast<double>(sc) < hv)
            sc = std::nextafterf(sc, std::numeric_limits<float>::infinity());
        mn_o = mn;
        sc_o = sc;
    };
    cover(lo[0], hi[0], q.lt_min, q.lt_scale);
    cover(lo[1], hi[1], q.r_min, q.r_scale);
    for (int c = 0; c < 3; c++) cover(lo[2 + c], hi[2 + c], q.c_min[c], q.c_scale[c]);
    return q;
}

void put16(std::vector<uint8_t>& b, uint16_t v) {
    b.push_back(static_cast<uint8_t>(v));
    b.push_back(static_cast<uint8_t>(v >> 8));
}
void put32(std::vector<uint8_t>& b, uint32_t v) {
    for (int i = 0; i < 4; i++) b.push_back(static_cast<uint8_t>(v >> (8 * i)));
}
void putf(std::vector<uint8_t>& b, double v) {
    float f = static_cast<float>(v);
    uint32_t u;
    std::memcpy(&u, &f, 4);
    put32(b, u);
}
uint32_t get32(const uint8_t* p) {
    return static_cast<uint32_t>(p[0]) | (static_cast<uint32_t>(p[1]) << 8) | (static_cast<uint32_t>(p[2]) << 16) |
           (static_cast<uint32_t>(p[3]) << 24);
}
double getf(const uint8_t* p) {
    uint32_t u = get32(p);
    float f;
    std::memcpy(&f, &u, 4);
    return f;
}

}  // namespace

extern "C" {

// write_file (codec.cpp:147-177) into memory: only active sites, ascending id.
sad_status sad_encode(const sad_sites_view* s, int w, int h, uint8_t* out, size_t cap, size_t* nbytes) {
    if (w < 1 || h < 1) return fail(SAD_EINVAL, "write: empty extent");
    size_t count = 0;
    for (size_t i = 0; i < s->size; i++) count += s->active[i] != 0;
    size_t need = 58 + 16 * count;
    *nbytes = need;
    if (!out) return SAD_OK;
    if (cap < need) return fail(SAD_ENOMEM, "encode: buffer too small");
    Ranges q = ranges(s);
    std::vector<uint8_t> b;
    b.reserve(need);
    b.insert(b.end(), {'S', 'A', 'D', 'F'});
    put16(b, kVersion);
    put32(b, static_cast<uint32_t>(w));
    put32(b, static_cast<uint32_t>(h));
    put32(b, static_cast<uint32_t>(count));
    putf(b, q.lt_min);
    putf(b, q.lt_scale);
    putf(b, q.r_min);
    putf(b, q.r_scale);
    for (int c = 0; c < 3; c++) putf(b, q.c_min[c]);
    for (int c = 0; c < 3; c++) putf(b, q.c_scale[c]);
    const double wden = w > 1 ? w - 1.0 : 1.0, hden = h > 1 ? h - 1.0 : 1.0;
    for (size_t i = 0; i < s->size; i++) {
        if (!s->active[i]) continue;
        // pack_site (codec.cpp:90-113)
        uint32_t w0 = unorm_encode(s->x[i], 0.0, wden, 32767) | (unorm_encode(s->y[i], 0.0, hden, 32767) << 15) |
                      (1u << 31);
        uint32_t w1 = unorm_encode(s->col_r[i], q.c_min[0], q.c_scale[0], 2047) |
                      (unorm_encode(s->col_g[i], q.c_min[1], q.c_scale[1], 2047) << 11) |
                      (unorm_encode(s->col_b[i], q.c_min[2], q.c_scale[2], 1023) << 22);
        uint32_t w2 = unorm_encode(s->log_tau[i], q.lt_min, q.lt_scale, 65535) |
                      (unorm_encode(s->radius[i], q.r_min, q.r_scale, 65535) << 16);
        double ang = std::atan2(s->dir_y[i], s->dir_x[i]);
        uint32_t w3 = unorm_encode(ang, -kPi, 2.0 * kPi, 65535) |
                      (static_cast<uint32_t>(f2h(static_cast<float>(s->aniso[i]))) << 16);
        put32(b, w0);
        put32(b, w1);
        put32(b, w2);
        put32(b, w3);
    }
    std::memcpy(out, b.data(), b.size());
    return SAD_OK;
}

// Header of read_file (codec.cpp:179-205), with its exact error messages.
sad_status sad_decode_header(const uint8_t* buf, size_t n, int* w, int* h, uint32_t* count) {
    char msg[96];
    if (n < 18) {
        std::snprintf(msg, sizeof msg, "file truncated at byte %zu, need %zu", n, static_cast<size_t>(18));
        return fail(SAD_EFORMAT, msg);
    }
    if (!(buf[0] == 'S' && buf[1] == 'A' && buf[2] == 'D' && buf[3] == 'F'))
        return fail(SAD_EFORMAT, "bad magic, not a site file");
    uint16_t version = static_cast<uint16_t>(buf[4] | (buf[5] << 8));
    if (version != kVersion) return fail(SAD_EFORMAT, "unknown format version " + std::to_string(version));
    uint32_t ww = get32(buf + 6), hh = get32(buf + 10), c = get32(buf + 14);
    if (ww < 1 || hh < 1 || ww > (1u << 24) || hh > (1u << 24))
        return fail(SAD_EFORMAT, "unreasonable image extent in header");
    size_t need = 58 + 16 * static_cast<size_t>(c);
    if (n != need) {
        std::snprintf(msg, sizeof msg, "file truncated at byte %zu, need %zu", n, need);
        return fail(SAD_EFORMAT, msg);
    }
    *w = static_cast<int>(ww);
    *h = static_cast<int>(hh);
    *count = c;
    return SAD_OK;
}

// read_file + unpack_site (codec.cpp:115-140, 179-222): sites view capacity >= count.
sad_status sad_decode(const uint8_t* buf, size_t n, sad_sites_view* s, int* w, int* h) {
    uint32_t count = 0;
    sad_status rc = sad_decode_header(buf, n, w, h, &count);
    if (rc != SAD_OK) return rc;
    if (s->capacity < count) return fail(SAD_ENOMEM, "decode: sites view capacity too small");
    Ranges q;
    q.lt_min = getf(buf + 18);
    q.lt_scale = getf(buf + 22);
    q.r_min = getf(buf + 26);
    q.r_scale = getf(buf + 30);
    for (int c = 0; c < 3; c++) q.c_min[c] = getf(buf + 34 + 4 * c);
    for (int c = 0; c < 3; c++) q.c_scale[c] = getf(buf + 46 + 4 * c);
    const double wden = *w > 1 ? *w - 1.0 : 1.0, hden = *h > 1 ? *h - 1.0 : 1.0;
    for (uint32_t i = 0; i < count; i++) {
        const uint8_t* r = buf + 58 + 16 * static_cast<size_t>(i);
        uint32_t w0 = get32(r), w1 = get32(r + 4), w2 = get32(r + 8), w3 = get32(r + 12);
        if (!(w0 >> 31)) {  // Site{} defaults, then deactivate (parks at -1,-1)
            s->x[i] = -1.0; s->y[i] = -1.0; s->log_tau[i] = 7.5; s->radius[i] = 1.0;
            s->col_r[i] = s->col_g[i] = s->col_b[i] = 0.0; s->dir_x[i] = 1.0; s->dir_y[i] = 0.0;
            s->aniso[i] = 0.0; s->active[i] = 0; s->frozen[i] = 0;
            continue;
        }
        s->x[i] = unorm_decode(w0 & 0x7fffu, 0.0, wden, 32767);
        s->y[i] = unorm_decode((w0 >> 15) & 0x7fffu, 0.0, hden, 32767);
        s->col_r[i] = dclamp(unorm_decode(w1 & 0x7ffu, q.c_min[0], q.c_scale[0], 2047), 0.0, 1.0);
        s->col_g[i] = dclamp(unorm_decode((w1 >> 11) & 0x7ffu, q.c_min[1], q.c_scale[1], 2047), 0.0, 1.0);
        s->col_b[i] = dclamp(unorm_decode(w1 >> 22, q.c_min[2], q.c_scale[2], 1023), 0.0, 1.0);
        s->log_tau[i] = unorm_decode(w2 & 0xffffu, q.lt_min, q.lt_scale, 65535);
        s->radius[i] = unorm_decode(w2 >> 16, q.r_min, q.r_scale, 65535);
        double ang = unorm_decode(w3 & 0xffffu, -kPi, 2.0 * kPi, 65535);
        s->dir_x[i] = std::cos(ang);
        s->dir_y[i] = std::sin(ang);
        s->aniso[i] = static_cast<double>(h2f(static_cast<uint16_t>(w3 >> 16)));
        s->active[i] = 1;
        s->frozen[i] = 0;
    }
    s->size = count;
    s->generation += 1 + count;
    return SAD_OK;
}

// bpp (codec.cpp:142-145)
sad_status sad_bpp(size_t count, int w, int h, double* out) {
    if (w < 1 || h < 1) return fail(SAD_EINVAL, "bpp: empty extent");
    *out = static_cast<double>(count) * 128.0 / (static_cast<double>(w) * h);
    return SAD_OK;
}

}  // extern "C"
