// sad_device.cuh — device-side building blocks shared by every SAD kernel (sm_100a).
//
// Parity rules: the library is compiled with --fmad=false so every
// float/double add and multiply rounds exactly like the reference's -ffp-contract=off build
// (CMakeLists.txt:15-17); sqrt and division are IEEE round-to-nearest (nvcc defaults); the float
// exponential is a port of glibc's expf that is bit-identical on all 2^32 inputs
// (profiles/expf_port_check.txt); the xorshift/mix32 streams are integer-exact copies of rng.hpp.
#pragma once
#include <cstdint>
#include <cuda_fp16.h>

namespace sadk {

constexpr uint32_t kEmpty = 0xffffffffu;  // CandidateField::kEmpty (types.hpp:85)

// ------------------------------------------------------------------ rng.hpp:12-45
__device__ __forceinline__ uint32_t mix32(uint32_t h) {
    h ^= h >> 16;
    h *= 0x7feb352du;
    h ^= h >> 15;
    h *= 0x846ca68bu;
    h ^= h >> 16;
    return h;
}

// seeded_stream(seed, a, b).s
__device__ __forceinline__ uint32_t seeded_state(uint64_t seed, uint32_t a, uint32_t b) {
    uint32_t h = mix32(static_cast<uint32_t>(seed) ^ 0x9e3779b9u);
    h ^= mix32(static_cast<uint32_t>(seed >> 32) + 0x85ebca6bu);
    h = mix32(h + mix32(a ^ 0x27d4eb2fu));
    h = mix32(h ^ mix32(b + 0x165667b1u));
    return h ? h : 0x6b33a1c9u;
}

__device__ __forceinline__ uint32_t xs_next(uint32_t& s) {
    uint32_t x = s;
    x ^= x << 13;
    x ^= x >> 17;
    x ^= x << 5;
    s = x;
    return x;
}

__device__ __forceinline__ double xs_unit(uint32_t& s) { return (xs_next(s) >> 8) * (1.0 / 16777216.0); }

// ------------------------------------------------------------------ half.hpp + score.cpp:9-22
// IEEE binary16 round trip (RNE), the candidate snapshot's quantisation.
__device__ __forceinline__ double half_rt(double v) {
    return static_cast<double>(__half2float(__float2half_rn(static_cast<float>(v))));
}

// ------------------------------------------------------------------ glibc expf, bit-exact port
// exp(x) = 2^(k/32) * 2^(r/32) with a cubic in r; table entries are bits(2^(i/32)) - (i << 47).
__device__ const unsigned long long kExp2fTab[32] = {
    0x3ff0000000000000ull, 0x3fefd9b0d3158574ull, 0x3fefb5586cf9890full, 0x3fef9301d0125b51ull,
    0x3fef72b83c7d517bull, 0x3fef54873168b9aaull, 0x3fef387a6e756238ull, 0x3fef1e9df51fdee1ull,
    0x3fef06fe0a31b715ull, 0x3feef1a7373aa9cbull, 0x3feedea64c123422ull, 0x3feece086061892dull,
    0x3feebfdad5362a27ull, 0x3feeb42b569d4f82ull, 0x3feeab07dd485429ull, 0x3feea47eb03a5585ull,
    0x3feea09e667f3bcdull, 0x3fee9f75e8ec5f74ull, 0x3feea11473eb0187ull, 0x3feea589994cce13ull,
    0x3feeace5422aa0dbull, 0x3feeb737b0cdc5e5ull, 0x3feec49182a3f090ull, 0x3feed503b23e255dull,
    0x3feee89f995ad3adull, 0x3feeff76f2fb5e47ull, 0x3fef199bdd85529cull, 0x3fef3720dcef9069ull,
    0x3fef5818dcfba487ull, 0x3fef7c97337b9b5full, 0x3fefa4afa2a490daull, 0x3fefd0765b6e4540ull};

__device__ __forceinline__ float sad_expf(float x) {
    uint32_t ux = __float_as_uint(x);
    uint32_t abstop = (ux & 0x7fffffffu) >> 20;
    if (abstop >= 0x42bu) {  // |x| >= 88 (top12 of 88.0f), inf or nan
        if (ux == 0xff800000u) return 0.0f;
        if (abstop >= 0x7f8u) return x + x;
        if (x > 0x1.62e42ep6f) return __int_as_float(0x7f800000);
        if (x < -0x1.9fe368p6f) return 0.0f;
    }
    const double kInvLn2N = 0x1.71547652b82fep0 * 32.0;
    const double kShift = 0x1.8p+52;
    const double kC0 = 0x1.c6af84b912394p-5 / 32.0 / 32.0 / 32.0;
    const double kC1 = 0x1.ebfce50fac4f3p-3 / 32.0 / 32.0;
    const double kC2 = 0x1.62e42ff0c52d6p-1 / 32.0;
    double xd = static_cast<double>(x);
    double z = kInvLn2N * xd;
    double kd = z + kShift;
    uint64_t ki = static_cast<uint64_t>(__double_as_longlong(kd));
    kd -= kShift;
    double r = __fma_rn(kInvLn2N, xd, -kd);
    uint64_t t = __ldg(&kExp2fTab[ki & 31u]);  // L1-cached: lanes index freely without serialising
    t += ki << 47;
    double s = __longlong_as_double(static_cast<long long>(t));
    double zz = __fma_rn(kC0, r, kC1);
    double r2 = r * r;
    double y = __fma_rn(kC2, r, 1.0);
    y = __fma_rn(zz, r2, y);
    y = y * s;
    return static_cast<float>(y);
}

template <typename T> __device__ __forceinline__ T texp(T x);
template <> __device__ __forceinline__ float texp<float>(float x) { return sad_expf(x); }
template <> __device__ __forceinline__ double texp<double>(double x) { return exp(x); }

template <typename T> __device__ __forceinline__ T tsqrt(T x);
template <> __device__ __forceinline__ float tsqrt<float>(float x) { return __fsqrt_rn(x); }
template <> __device__ __forceinline__ double tsqrt<double>(double x) { return __dsqrt_rn(x); }

template <typename T> __device__ __forceinline__ bool tfinite(T x) { return isfinite(static_cast<double>(x)); }
template <> __device__ __forceinline__ bool tfinite<float>(float x) {  // exponent field not all ones
    return (__float_as_uint(x) & 0x7f800000u) != 0x7f800000u;
}

// IEEE round-to-nearest reciprocal: the same value as T(1) / x, with a shorter instruction sequence.
template <typename T> __device__ __forceinline__ T trcp(T x);
template <> __device__ __forceinline__ float trcp<float>(float x) { return __frcp_rn(x); }
template <> __device__ __forceinline__ double trcp<double>(double x) { return __drcp_rn(x); }

// std::max / std::min semantics (NaN-propagating exactly as libstdc++ does)
__device__ __forceinline__ double smax(double a, double b) { return (a < b) ? b : a; }
__device__ __forceinline__ double smin(double a, double b) { return (b < a) ? b : a; }
__device__ __forceinline__ double sclamp(double v, double lo, double hi) { return (v < lo) ? lo : (hi < v) ? hi : v; }

// ------------------------------------------------------------------ Accum (accum.hpp:10-31)
struct DD {
    double hi, lo;
};

__device__ __forceinline__ void dd_add(DD& a, double x) {
    double s = a.hi + x;
    double bb = s - a.hi;
    double err = (a.hi - (s - bb)) + (x - bb);
    a.hi = s;
    a.lo += err;
}

__device__ __forceinline__ void dd_merge(DD& a, const DD& o) {
    dd_add(a, o.hi);
    dd_add(a, o.lo);
}

// Accum::add(Accum) into a 16-byte aligned global (hi, lo) pair with a 128-bit CAS.  The
// compensated sum makes the final hi+lo independent of the arrival order (accum.hpp:5-9).
__device__ __forceinline__ void dd_atomic_merge(double2* addr, DD part) {
    unsigned long long* p = reinterpret_cast<unsigned long long*>(addr);
    unsigned long long ohi = p[0], olo = p[1];
    while (true) {
        DD cur{__longlong_as_double(static_cast<long long>(ohi)), __longlong_as_double(static_cast<long long>(olo))};
        dd_merge(cur, part);
        unsigned long long nhi = static_cast<unsigned long long>(__double_as_longlong(cur.hi));
        unsigned long long nlo = static_cast<unsigned long long>(__double_as_longlong(cur.lo));
        unsigned long long rhi, rlo;
        asm volatile(
            "{\n\t.reg .b128 c, n, o;\n\t"
            "mov.b128 c, {%2, %3};\n\t"
            "mov.b128 n, {%4, %5};\n\t"
            "atom.global.cas.b128 o, [%6], c, n;\n\t"
            "mov.b128 {%0, %1}, o;\n\t}"
            : "=l"(rhi), "=l"(rlo)
            : "l"(ohi), "l"(olo), "l"(nhi), "l"(nlo), "l"(p)
            : "memory");
        if (rhi == ohi && rlo == olo) return;
        ohi = rhi;
        olo = rlo;
    }
}

__device__ __forceinline__ double dd_value(const double2 v) { return v.x + v.y; }

// Orderable 64-bit key of a double for ascending radix sorts; -0.0 is canonicalised to +0.0
// because the reference compares with `<` (budget.cpp:231-235, 297-302).
__device__ __forceinline__ unsigned long long order_key(double d) {
    if (d == 0.0) d = 0.0;
    unsigned long long u = static_cast<unsigned long long>(__double_as_longlong(d));
    return (u & 0x8000000000000000ull) ? ~u : (u | 0x8000000000000000ull);
}

// 4-wide vector of T (float4 / 32-byte double quad)
template <typename T> struct alignas(4 * sizeof(T)) Q4 {
    T x, y, z, w;
};

}  // namespace sadk
