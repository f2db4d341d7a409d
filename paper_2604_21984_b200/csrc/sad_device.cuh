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

#include "sad_log_table.h"

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

// glibc `exp` (double), as built for x86-64 with FMA (the optimized-routines algorithm glibc uses since
// 2.28): exp(x) = 2^(k/128) * exp(r), k = round(x * 128/ln2), r = x - k*ln2/128 in two parts; a 128-entry
// table of (tail, bits(2^(k/128)) - (k << 45)) and a degree-5 polynomial; multiply-adds fused where GCC
// -mfma fuses them.  The table is 2^(i/128) rounded to double and its relative tail, computed at 80
// digits.  Checked against this image's libm: bit-identical on 2e8 random inputs with |x| <= 510
// (profiles/exp_port_check.txt); for |x| > 512 (results < 1e-222 or > 1e222) 0.002% differ by one ulp.
__device__ const uint64_t kExpTab[256] = {
    0x0000000000000000ull, 0x3ff0000000000000ull, 0x3c9b3b4f1a88bf6eull, 0x3feff63da9fb3335ull,
    0xbc7160139cd8dc5dull, 0x3fefec9a3e778061ull, 0xbc905e7a108766d1ull, 0x3fefe315e86e7f85ull,
    0x3c8cd2523567f613ull, 0x3fefd9b0d3158574ull, 0xbc8bce8023f98efaull, 0x3fefd06b29ddf6deull,
    0x3c60f74e61e6c861ull, 0x3fefc74518759bc8ull, 0x3c90a3e45b33d399ull, 0x3fefbe3ecac6f383ull,
    0x3c979aa65d837b6dull, 0x3fefb5586cf9890full, 0x3c8eb51a92fdeffcull, 0x3fefac922b7247f7ull,
    0x3c3ebe3d702f9cd1ull, 0x3fefa3ec32d3d1a2ull, 0xbc6a033489906e0bull, 0x3fef9b66affed31bull,
    0xbc9556522a2fbd0eull, 0x3fef9301d0125b51ull, 0xbc5080ef8c4eea55ull, 0x3fef8abdc06c31ccull,
    0xbc91c923b9d5f416ull, 0x3fef829aaea92de0ull, 0x3c80d3e3e95c55afull, 0x3fef7a98c8a58e51ull,
    0xbc801b15eaa59348ull, 0x3fef72b83c7d517bull, 0xbc8f1ff055de323dull, 0x3fef6af9388c8deaull,
    0x3c8b898c3f1353bfull, 0x3fef635beb6fcb75ull, 0xbc96d99c7611eb26ull, 0x3fef5be084045cd4ull,
    0x3c9aecf73e3a2f60ull, 0x3fef54873168b9aaull, 0xbc8fe782cb86389dull, 0x3fef4d5022fcd91dull,
    0x3c8a6f4144a6c38dull, 0x3fef463b88628cd6ull, 0x3c807a05b0e4047dull, 0x3fef3f49917ddc96ull,
    0x3c968efde3a8a894ull, 0x3fef387a6e756238ull, 0x3c875e18f274487dull, 0x3fef31ce4fb2a63full,
    0x3c80472b981fe7f2ull, 0x3fef2b4565e27cddull, 0xbc96b87b3f71085eull, 0x3fef24dfe1f56381ull,
    0x3c82f7e16d09ab31ull, 0x3fef1e9df51fdee1ull, 0xbc3d219b1a6fbffaull, 0x3fef187fd0dad990ull,
    0x3c8b3782720c0ab4ull, 0x3fef1285a6e4030bull, 0x3c6e149289cecb8full, 0x3fef0cafa93e2f56ull,
    0x3c834d754db0abb6ull, 0x3fef06fe0a31b715ull, 0x3c864201e2ac744cull, 0x3fef0170fc4cd831ull,
    0x3c8fdd395dd3f84aull, 0x3feefc08b26416ffull, 0xbc86a3803b8e5b04ull, 0x3feef6c55f929ff1ull,
    0xbc924aedcc4b5068ull, 0x3feef1a7373aa9cbull, 0xbc9907f81b512d8eull, 0x3feeecae6d05d866ull,
    0xbc71d1e83e9436d2ull, 0x3feee7db34e59ff7ull, 0xbc991919b3ce1b15ull, 0x3feee32dc313a8e5ull,
    0x3c859f48a72a4c6dull, 0x3feedea64c123422ull, 0xbc9312607a28698aull, 0x3feeda4504ac801cull,
    0xbc58a78f4817895bull, 0x3feed60a21f72e2aull, 0xbc7c2c9b67499a1bull, 0x3feed1f5d950a897ull,
    0x3c4363ed60c2ac11ull, 0x3feece086061892dull, 0x3c9666093b0664efull, 0x3feeca41ed1d0057ull,
    0x3c6ecce1daa10379ull, 0x3feec6a2b5c13cd0ull, 0x3c93ff8e3f0f1230ull, 0x3feec32af0d7d3deull,
    0x3c7690cebb7aafb0ull, 0x3feebfdad5362a27ull, 0x3c931dbdeb54e077ull, 0x3feebcb299fddd0dull,
    0xbc8f94340071a38eull, 0x3feeb9b2769d2ca7ull, 0xbc87deccdc93a349ull, 0x3feeb6daa2cf6642ull,
    0xbc78dec6bd0f385full, 0x3feeb42b569d4f82ull, 0xbc861246ec7b5cf6ull, 0x3feeb1a4ca5d920full,
    0x3c93350518fdd78eull, 0x3feeaf4736b527daull, 0x3c7b98b72f8a9b05ull, 0x3feead12d497c7fdull,
    0x3c9063e1e21c5409ull, 0x3feeab07dd485429ull, 0x3c34c7855019c6eaull, 0x3feea9268a5946b7ull,
    0x3c9432e62b64c035ull, 0x3feea76f15ad2148ull, 0xbc8ce44a6199769full, 0x3feea5e1b976dc09ull,
    0xbc8c33c53bef4da8ull, 0x3feea47eb03a5585ull, 0xbc845378892be9aeull, 0x3feea34634ccc320ull,
    0xbc93cedd78565858ull, 0x3feea23882552225ull, 0x3c5710aa807e1964ull, 0x3feea155d44ca973ull,
    0xbc93b3efbf5e2228ull, 0x3feea09e667f3bcdull, 0xbc6a12ad8734b982ull, 0x3feea012750bdabfull,
    0xbc6367efb86da9eeull, 0x3fee9fb23c651a2full, 0xbc80dc3d54e08851ull, 0x3fee9f7df9519484ull,
    0xbc781f647e5a3ecfull, 0x3fee9f75e8ec5f74ull, 0xbc86ee4ac08b7db0ull, 0x3fee9f9a48a58174ull,
    0xbc8619321e55e68aull, 0x3fee9feb564267c9ull, 0x3c909ccb5e09d4d3ull, 0x3feea0694fde5d3full,
    0xbc7b32dcb94da51dull, 0x3feea11473eb0187ull, 0x3c94ecfd5467c06bull, 0x3feea1ed0130c132ull,
    0x3c65ebe1abd66c55ull, 0x3feea2f336cf4e62ull, 0xbc88a1c52fb3cf42ull, 0x3feea427543e1a12ull,
    0xbc9369b6f13b3734ull, 0x3feea589994cce13ull, 0xbc805e843a19ff1eull, 0x3feea71a4623c7adull,
    0xbc94d450d872576eull, 0x3feea8d99b4492edull, 0x3c90ad675b0e8a00ull, 0x3feeaac7d98a6699ull,
    0x3c8db72fc1f0eab4ull, 0x3feeace5422aa0dbull, 0xbc65b6609cc5e7ffull, 0x3feeaf3216b5448cull,
    0x3c7bf68359f35f44ull, 0x3feeb1ae99157736ull, 0xbc93091fa71e3d83ull, 0x3feeb45b0b91ffc6ull,
    0xbc5da9b88b6c1e29ull, 0x3feeb737b0cdc5e5ull, 0xbc6c23f97c90b959ull, 0x3feeba44cbc8520full,
    0xbc92434322f4f9aaull, 0x3feebd829fde4e50ull, 0xbc85ca6cd7668e4bull, 0x3feec0f170ca07baull,
    0x3c71affc2b91ce27ull, 0x3feec49182a3f090ull, 0x3c6dd235e10a73bbull, 0x3feec86319e32323ull,
    0xbc87c50422622263ull, 0x3feecc667b5de565ull, 0x3c8b1c86e3e231d5ull, 0x3feed09bec4a2d33ull,
    0xbc91bbd1d3bcbb15ull, 0x3feed503b23e255dull, 0x3c90cc319cee31d2ull, 0x3feed99e1330b358ull,
    0x3c8469846e735ab3ull, 0x3feede6b5579fdbfull, 0xbc82dfcd978e9db4ull, 0x3feee36bbfd3f37aull,
    0x3c8c1a7792cb3387ull, 0x3feee89f995ad3adull, 0xbc907b8f4ad1d9faull, 0x3feeee07298db666ull,
    0xbc55c3d956dcaebaull, 0x3feef3a2b84f15fbull, 0xbc90a40e3da6f640ull, 0x3feef9728de5593aull,
    0xbc68d6f438ad9334ull, 0x3feeff76f2fb5e47ull, 0xbc91eee26b588a35ull, 0x3fef05b030a1064aull,
    0x3c74ffd70a5fddcdull, 0x3fef0c1e904bc1d2ull, 0xbc91bdfbfa9298acull, 0x3fef12c25bd71e09ull,
    0x3c736eae30af0cb3ull, 0x3fef199bdd85529cull, 0x3c8ee3325c9ffd94ull, 0x3fef20ab5fffd07aull,
    0x3c84e08fd10959acull, 0x3fef27f12e57d14bull, 0x3c63cdaf384e1a67ull, 0x3fef2f6d9406e7b5ull,
    0x3c676b2c6c921968ull, 0x3fef3720dcef9069ull, 0xbc808a1883ccb5d2ull, 0x3fef3f0b555dc3faull,
    0xbc8fad5d3ffffa6full, 0x3fef472d4a07897cull, 0xbc900dae3875a949ull, 0x3fef4f87080d89f2ull,
    0x3c74a385a63d07a7ull, 0x3fef5818dcfba487ull, 0xbc82919e2040220full, 0x3fef60e316c98398ull,
    0x3c8e5a50d5c192acull, 0x3fef69e603db3285ull, 0x3c843a59ac016b4bull, 0x3fef7321f301b460ull,
    0xbc82d52107b43e1full, 0x3fef7c97337b9b5full, 0xbc892ab93b470dc9ull, 0x3fef864614f5a129ull,
    0x3c74b604603a88d3ull, 0x3fef902ee78b3ff6ull, 0x3c83c5ec519d7271ull, 0x3fef9a51fbc74c83ull,
    0xbc8ff7128fd391f0ull, 0x3fefa4afa2a490daull, 0xbc8dae98e223747dull, 0x3fefaf482d8e67f1ull,
    0x3c8ec3bc41aa2008ull, 0x3fefba1bee615a27ull, 0x3c842b94c3a9eb32ull, 0x3fefc52b376bba97ull,
    0x3c8a64a931d185eeull, 0x3fefd0765b6e4540ull, 0xbc8e37bae43be3edull, 0x3fefdbfdad9cbe14ull,
    0x3c77893b4d91cd9dull, 0x3fefe7c1819e90d8ull, 0x3c5305c14160cc89ull, 0x3feff3c22b8f71f1ull,
};

__device__ __forceinline__ double sad_dexp_special(double tmp, uint64_t sbits, uint64_t ki) {
    if ((ki & 0x80000000ull) == 0) {  // k > 0: the exponent of scale may have overflowed
        sbits -= 1009ull << 52;
        const double scale = __longlong_as_double(static_cast<long long>(sbits));
        return 0x1p1009 * __fma_rn(scale, tmp, scale);
    }
    sbits += 1022ull << 52;  // k < 0: care in the subnormal range
    const double scale = __longlong_as_double(static_cast<long long>(sbits));
    // glibc's build does not contract this branch (unlike the k > 0 one): separate multiply and add
    // (host harness over 6e7 inputs in [-745.2, -512]: 0 mismatches; fused: 0.06% off by one ulp)
    double y = __dadd_rn(scale, __dmul_rn(scale, tmp));
    if (y < 1.0) {
        double lo = __dadd_rn(scale - y, __dmul_rn(scale, tmp));
        const double hi = 1.0 + y;
        lo = 1.0 - hi + y + lo;
        y = (hi + lo) - 1.0;
        if (y == 0.0) y = 0.0;
    }
    return 0x1p-1022 * y;
}

__device__ __forceinline__ double sad_dexp(double x) {
    const double kInvLn2N = 0x1.71547652b82fep0 * 128.0, kShift = 0x1.8p52;
    const double kNegLn2hiN = -0x1.62e42fefa0000p-8, kNegLn2loN = -0x1.cf79abc9e3b3ap-47;
    const double C2 = 0x1.ffffffffffdbdp-2, C3 = 0x1.555555555543cp-3, C4 = 0x1.55555cf172b91p-5,
                 C5 = 0x1.1111167a4d017p-7;
    const uint64_t ux = static_cast<uint64_t>(__double_as_longlong(x));
    uint32_t abstop = static_cast<uint32_t>(ux >> 52) & 0x7ffu;
    if (abstop - 0x3c9u >= 0x408u - 0x3c9u) {  // |x| < 2^-54 or |x| >= 512 (top12 thresholds)
        if (abstop - 0x3c9u >= 0x80000000u) return 1.0 + x;
        if (abstop >= 0x409u) {  // |x| >= 1024
            if (ux == 0xfff0000000000000ull) return 0.0;
            if (abstop >= 0x7ffu) return 1.0 + x;
            return (ux >> 63) ? 0.0 : __longlong_as_double(0x7ff0000000000000ll);
        }
        abstop = 0;  // large |x|: special-cased below
    }
    const double z = kInvLn2N * x;
    double kd = z + kShift;
    const uint64_t ki = static_cast<uint64_t>(__double_as_longlong(kd));
    kd -= kShift;
    const double r = __fma_rn(kd, kNegLn2loN, __fma_rn(kd, kNegLn2hiN, x));
    const uint64_t idx = 2 * (ki % 128u);
    const uint64_t top = ki << 45;
    const double tail = __longlong_as_double(static_cast<long long>(__ldg(&kExpTab[idx])));
    const uint64_t sbits = __ldg(&kExpTab[idx + 1]) + top;
    const double r2 = r * r;
    const double tmp = __fma_rn(r2 * r2, __fma_rn(r, C5, C4), __fma_rn(r2, __fma_rn(r, C3, C2), tail + r));
    if (abstop == 0) return sad_dexp_special(tmp, sbits, ki);
    const double scale = __longlong_as_double(static_cast<long long>(sbits));
    return __fma_rn(scale, tmp, scale);
}

// glibc `log` (double), as built for x86-64 with FMA (the optimized-routines algorithm, glibc >= 2.28):
// log(x) = k*ln2 + log(c) + log1p(z/c - 1) over 128 subintervals, plus a separate polynomial near 1; every
// multiply-add GCC fuses under -mfma is an fma here.  The constants (sad_log_table.h) are read from the
// host's libm by tools/gen_log_table.py; a host harness finds 0 mismatches against that libm on 6e7 inputs
// (log-uniform over [e^-700, e^700], densify ratios [1.05, 1e18], the near-1 path), and
// tests/test_libm_port.py checks the device copy.  Used by densify's split anisotropy (budget.cpp:198-199).
__device__ __forceinline__ double sad_dlog(double x) {
    const double Ln2hi = __longlong_as_double(static_cast<long long>(kLogHead[0]));
    const double Ln2lo = __longlong_as_double(static_cast<long long>(kLogHead[1]));
    auto A = [](int i) { return __longlong_as_double(static_cast<long long>(kLogHead[2 + i])); };
    auto B = [](int i) { return __longlong_as_double(static_cast<long long>(kLogHead[7 + i])); };
    uint64_t ix = static_cast<uint64_t>(__double_as_longlong(x));
    const uint32_t top = static_cast<uint32_t>(ix >> 48);
    const uint64_t LO = 0x3feE000000000000ull;  // asuint64(1.0 - 0x1p-4)
    const uint64_t HI = 0x3ff1090000000000ull;  // asuint64(1.0 + 0x1.09p-4)
    if (ix - LO < HI - LO) {
        if (ix == 0x3ff0000000000000ull) return 0.0;
        const double r = x - 1.0, r2 = r * r, r3 = r * r2;
        double i3 = __fma_rn(r, B(8), B(7));
        i3 = __fma_rn(r2, B(9), i3);
        i3 = __fma_rn(r3, B(10), i3);
        double i2 = __fma_rn(r, B(5), B(4));
        i2 = __fma_rn(r2, B(6), i2);
        i2 = __fma_rn(r3, i3, i2);
        double i1 = __fma_rn(r, B(2), B(1));
        i1 = __fma_rn(r2, B(3), i1);
        i1 = __fma_rn(r3, i2, i1);
        double w = r * 0x1p27;
        const double rhi = r + w - w;
        const double rlo = r - rhi;
        const double rr = rhi * rhi;
        const double hi = __fma_rn(rr, B(0), r);
        double lo = __fma_rn(rr, B(0), r - hi);
        lo = __fma_rn(B(0) * rlo, rhi + r, lo);
        double y = __fma_rn(r3, i1, lo);
        return y + hi;
    }
    if (top - 0x0010u >= 0x7ff0u - 0x0010u) {
        if (ix * 2 == 0) return -__longlong_as_double(0x7ff0000000000000ll);
        if (ix == 0x7ff0000000000000ull) return x;
        if ((top & 0x8000u) || (top & 0x7ff0u) == 0x7ff0u) return __longlong_as_double(0x7ff8000000000000ll);
        ix = static_cast<uint64_t>(__double_as_longlong(x * 0x1p52));  // subnormal: normalise
        ix -= 52ull << 52;
    }
    const uint64_t tmp = ix - 0x3fe6000000000000ull;
    const int i = static_cast<int>((tmp >> 45) % 128);
    const int k = static_cast<int>(static_cast<int64_t>(tmp) >> 52);
    const uint64_t iz = ix - (tmp & (0xfffull << 52));
    const double invc = __longlong_as_double(static_cast<long long>(kLogTab[2 * i]));
    const double logc = __longlong_as_double(static_cast<long long>(kLogTab[2 * i + 1]));
    const double z = __longlong_as_double(static_cast<long long>(iz));
    const double r = __fma_rn(z, invc, -1.0);
    const double kd = static_cast<double>(k);
    const double w = __fma_rn(kd, Ln2hi, logc);
    const double hi = w + r;
    const double lo = __fma_rn(kd, Ln2lo, w - hi + r);
    const double r2 = r * r;
    double p = __fma_rn(r, A(2), A(1));
    const double q = __fma_rn(r, A(4), A(3));
    p = __fma_rn(r2, q, p);
    const double t1 = __fma_rn(r2, A(0), lo);
    const double t2 = __fma_rn(r * r2, p, t1);
    return t2 + hi;
}

template <typename T> __device__ __forceinline__ T texp(T x);
template <> __device__ __forceinline__ float texp<float>(float x) { return sad_expf(x); }
template <> __device__ __forceinline__ double texp<double>(double x) { return sad_dexp(x); }

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
