// host_libm.cpp — makes the GPU's log() and exp() reproduce the host libm bit
// for bit.
//
// The reference draws its normals with glibc's log() (rng.hpp:61) and steps
// S with glibc's exp() (heston.hpp:307, via tape.hpp:305 / kernel.hpp:172).
// glibc >= 2.28 implements both with the ARM optimized-routines algorithms
// (log: x = 2^k z, 128-entry (1/c, log c) table, degree-5 polynomial in
// r = z/c - 1; exp: x = k ln2/128 + r, 128-entry 2^(j/128) table, degree-5
// polynomial); on x86-64 CPUs with FMA the ifunc selects the FMA builds,
// whose operation sequences rng.cuh:glibc_log / glibc_exp restate. glibc's
// log rounds the wrong way for about 1 in 10^4 tail arguments, so a
// correctly rounded (or CUDA) log would change some reference draws.
//
// The tables are not shipped with this library: at context creation we
// locate the `__log_data` / `__exp_data` blocks inside the libm this process
// loaded (by their leading constants), then VALIDATE each candidate by
// evaluating the restated sequence on the host against the real log()/exp()
// on 65,536 arguments spanning every table interval of the domain the
// kernels use. Only a table that reproduces libm bit for bit on all of them
// is used (exact_log / exact_exp = 1); otherwise the GPU falls back to CUDA's
// log()/exp() and ltg_rng_exact() reports 0.
#include <dlfcn.h>

#include <cmath>
#include <cstdint>
#include <cstring>
#include <fstream>
#include <string>
#include <vector>

#include "kernels.h"

namespace ltg {

namespace {

double bits2d(uint64_t u) {
    double d;
    std::memcpy(&d, &u, 8);
    return d;
}
uint64_t d2bits(double d) {
    uint64_t u;
    std::memcpy(&u, &d, 8);
    return u;
}

}  // namespace

// host restatements of rng.cuh (std::fma == __fma_rn bit for bit; every
// other operation rounded on its own, as the intrinsics are)
double emulate_log(const RngConsts& K, const RngTables& T, double x) {
    const uint64_t ix = d2bits(x);
    const uint64_t tmp = ix - 0x3fe6000000000000ULL;
    const int i = (int)((tmp >> 45) & 127);
    const int k = (int)((int64_t)tmp >> 52);
    const double z = bits2d(ix - (tmp & 0xfff0000000000000ULL));
    const double invc = T.log_tab[i].x, logc = T.log_tab[i].y;
    const double kd = (double)k;
    const double w = std::fma(kd, K.log_ln2hi, logc);
    const double r = std::fma(z, invc, -1.0);
    const double p12 = std::fma(r, K.log_poly[2], K.log_poly[1]);
    volatile double hi = r + w;
    volatile double r2 = r * r;
    volatile double wh = w - hi;
    volatile double whr = wh + r;
    const double lo = std::fma(kd, K.log_ln2lo, whr);
    volatile double r3 = r * r2;
    const double p34 = std::fma(r, K.log_poly[4], K.log_poly[3]);
    const double lo2 = std::fma(r2, K.log_poly[0], lo);
    const double p = std::fma(p34, r2, p12);
    const double y = std::fma(r3, p, lo2);
    volatile double out = y + hi;
    return out;
}

double emulate_exp(const RngConsts& K, const RngTables& T, double x) {
    const uint32_t abstop = (uint32_t)(d2bits(x) >> 52) & 0x7ffu;
    if (abstop - 0x3c9u >= 0x3fu) {
        if ((int)(abstop - 0x3c9u) < 0) {
            volatile double o = 1.0 + x;
            return o;
        }
        return std::exp(x);
    }
    volatile double kd = std::fma(x, K.exp_invln2N, K.exp_shift);
    const uint64_t ki = d2bits(kd);
    kd = kd - K.exp_shift;
    const double r = std::fma(kd, K.exp_negln2loN, std::fma(kd, K.exp_negln2hiN, x));
    const unsigned idx = 2u * (unsigned)(ki & 127u);
    const double tail = bits2d(T.exp_tab[idx]);
    const uint64_t sbits = T.exp_tab[idx + 1] + (ki << 45);
    const double p23 = std::fma(r, K.exp_poly[1], K.exp_poly[0]);
    volatile double t1 = r + tail;
    volatile double r2 = r * r;
    const double p45 = std::fma(r, K.exp_poly[3], K.exp_poly[2]);
    const double t2 = std::fma(p23, r2, t1);
    volatile double r4 = r2 * r2;
    const double tmp = std::fma(r4, p45, t2);
    const double scale = bits2d(sbits);
    return std::fma(scale, tmp, scale);
}

namespace {

bool read_file(const char* path, std::vector<unsigned char>& buf) {
    std::ifstream f(path, std::ios::binary);
    if (!f) return false;
    buf.assign(std::istreambuf_iterator<char>(f), std::istreambuf_iterator<char>());
    return !buf.empty();
}

uint64_t xorshift(uint64_t& s) {
    s ^= s << 13;
    s ^= s >> 7;
    s ^= s << 17;
    return s;
}

// arguments of log() on the reference's tail path: min(p, 1-p) with
// p = (2n+1) 2^-53, i.e. x in [2^-53, 0.075]
bool validate_log(const RngConsts& K, const RngTables& T) {
    uint64_t s = 0x9E3779B97F4A7C15ULL;
    for (int i = 0; i < 65536; ++i) {
        xorshift(s);
        double x;
        if (i < 4096) {
            // every table interval, both binade halves, at several exponents
            const int e = -(int)(i % 54) - 1;
            const uint64_t mant = ((uint64_t)(i / 54) << 45) ^ (s & ((1ULL << 45) - 1));
            x = std::ldexp(bits2d(0x3ff0000000000000ULL | (mant & 0xfffffffffffffULL)), e);
        } else {
            const uint64_t n = s >> 12;  // 52-bit integer
            x = ((double)(2 * n + 1)) * 0x1p-53;
            if (x > 0.5) x = 1.0 - x;
        }
        if (!(x > 0.0) || x > 0.075) continue;
        if (emulate_log(K, T, x) != std::log(x)) return false;
    }
    return true;
}

// arguments of exp() in the Euler step: drift + diffusion, |x| well below 512;
// cover every table index and magnitudes from 2^-60 to 2^8
bool validate_exp(const RngConsts& K, const RngTables& T) {
    uint64_t s = 0xD1B54A32D192ED03ULL;
    for (int i = 0; i < 65536; ++i) {
        xorshift(s);
        const double u = (double)(s >> 11) * 0x1p-53;          // [0, 1)
        const int e = (int)(i % 69) - 60;                       // 2^-60 .. 2^8
        double x = std::ldexp(u, e);
        if (i & 1) x = -x;
        if (emulate_exp(K, T, x) != std::exp(x)) return false;
    }
    return true;
}

}  // namespace

// Fills the log/exp parts of K and T. Returns a note describing any failure.
std::string discover_glibc_math(RngConsts& K, RngTables& T) {
    std::string note;
    K.exact_log = 0;
    K.exact_exp = 0;
    Dl_info info;
    void* sym = dlsym(RTLD_DEFAULT, "log");
    if (!sym || !dladdr(sym, &info) || !info.dli_fname)
        return "cannot locate the libm that provides log()";
    std::vector<unsigned char> buf;
    if (!read_file(info.dli_fname, buf)) return std::string("cannot read ") + info.dli_fname;
    auto at = [&](size_t off) {
        double d;
        std::memcpy(&d, &buf[off], 8);
        return d;
    };
    // struct log_data { ln2hi, ln2lo, poly[5], poly1[11], tab[128]{invc, logc}, tab2[128] }
    const uint64_t ln2hi = d2bits(0x1.62e42fefa3800p-1), ln2lo = d2bits(0x1.ef35793c76730p-45);
    for (size_t off = 0; off + (18 + 256) * 8 <= buf.size() && !K.exact_log; off += 8) {
        if (d2bits(at(off)) != ln2hi || d2bits(at(off + 8)) != ln2lo) continue;
        RngConsts k = K;
        RngTables t = T;
        k.log_ln2hi = at(off);
        k.log_ln2lo = at(off + 8);
        for (int i = 0; i < 5; ++i) k.log_poly[i] = at(off + 16 + 8 * i);
        for (int i = 0; i < 128; ++i) {
            t.log_tab[i].x = at(off + 144 + 16 * i);
            t.log_tab[i].y = at(off + 144 + 16 * i + 8);
        }
        if (validate_log(k, t)) {
            k.exact_log = 1;
            K = k;
            T = t;
        }
    }
    if (!K.exact_log) note += "no log table reproduces log() bit for bit (CUDA log used); ";
    // struct exp_data { invln2N, shift, negln2hiN, negln2loN, poly[4], ..., tab[2*128] }
    // (the table offset depends on the glibc version: 112 bytes before 2.39,
    // 176 with the exp10 fields of 2.39; both are tried and validated)
    const uint64_t inv = d2bits(0x1.71547652b82fep7), shift = d2bits(0x1.8p52);
    for (size_t off = 0; off + (22 + 256) * 8 <= buf.size() && !K.exact_exp; off += 8) {
        if (d2bits(at(off)) != inv || d2bits(at(off + 8)) != shift) continue;
        for (size_t tab_off : {size_t(176), size_t(112)}) {
            RngConsts k = K;
            RngTables t = T;
            k.exp_invln2N = at(off);
            k.exp_shift = at(off + 8);
            k.exp_negln2hiN = at(off + 16);
            k.exp_negln2loN = at(off + 24);
            for (int i = 0; i < 4; ++i) k.exp_poly[i] = at(off + 32 + 8 * i);
            std::memcpy(t.exp_tab, &buf[off + tab_off], sizeof t.exp_tab);
            if (validate_exp(k, t)) {
                k.exact_exp = 1;
                K = k;
                T = t;
                break;
            }
        }
    }
    if (!K.exact_exp) note += "no exp table reproduces exp() bit for bit (CUDA exp used)";
    return note;
}

// AS241 coefficient rows (rng.hpp:49-58, 65-72, 75-82), highest degree first;
// the denominators' constant terms are 1.0.
void fill_as241(RngConsts& K) {
    static const double num[3][8] = {
        {2.5090809287301226727e+3, 3.3430575583588128105e+4, 6.7265770927008700853e+4,
         4.5921953931549871457e+4, 1.3731693765509461125e+4, 1.9715909503065514427e+3,
         1.3314166789178437745e+2, 3.3871328727963666080e+0},
        {7.74545014278341407640e-4, 2.27238449892691845833e-2, 2.41780725177450611770e-1,
         1.27045825245236838258e+0, 3.64784832476320460504e+0, 5.76949722146069140550e+0,
         4.63033784615654529590e+0, 1.42343711074968357734e+0},
        {2.01033439929228813265e-7, 2.71155556874348757815e-5, 1.24266094738807843860e-3,
         2.65321895265761230930e-2, 2.96560571828504891230e-1, 1.78482653991729133580e+0,
         5.46378491116411436990e+0, 6.65790464350110377720e+0}};
    static const double den[3][8] = {
        {5.2264952788528545610e+3, 2.8729085735721942674e+4, 3.9307895800092710610e+4,
         2.1213794301586595867e+4, 5.3941960214247511077e+3, 6.8718700749205790830e+2,
         4.2313330701600911252e+1, 1.0},
        {1.05075007164441684324e-9, 5.47593808499534494600e-4, 1.51986665636164571966e-2,
         1.48103976427480074590e-1, 6.89767334985100004550e-1, 1.67638483018380384940e+0,
         2.05319162663775882187e+0, 1.0},
        {2.04426310338993978564e-15, 1.42151175831644588870e-7, 1.84631831751005468180e-5,
         7.86869131145613259100e-4, 1.48753612908506148525e-2, 1.36929880922735805310e-1,
         5.99832206555887937690e-1, 1.0}};
    std::memcpy(K.num, num, sizeof num);
    std::memcpy(K.den, den, sizeof den);
    K.lit_uniform = -0x1.fffffffffffffp-1;
    K.lit_qmax = 0.425;
    K.lit_central = 0.180625;
    K.lit_tail1 = 1.6;
}

}  // namespace ltg

// Host-only self-test behind ltg_rng_selftest: discovers the tables and
// compares the restated log/exp against the host libm on n pseudo-random
// arguments each (log: tail arguments (2n+1)*2^-53 folded into (0, 0.075];
// exp: |x| < 2).
extern "C" int ltg_rng_selftest(uint64_t n, uint64_t* mismatches, int* exact) {
    ltg::RngConsts K{};
    ltg::RngTables T{};
    ltg::discover_glibc_math(K, T);
    const bool ok = K.exact_log && K.exact_exp;
    if (exact) *exact = ok ? 1 : 0;
    uint64_t bad = 0, s = 0x243F6A8885A308D3ULL;
    for (uint64_t i = 0; i < n && ok; ++i) {
        s ^= s << 13;
        s ^= s >> 7;
        s ^= s << 17;
        const uint64_t k = s >> 12;
        double x = ((double)(2 * k + 1)) * 0x1p-53;
        if (x > 0.5) x = 1.0 - x;
        if (x > 0.075) x *= 0.075;
        if (ltg::emulate_log(K, T, x) != std::log(x)) ++bad;
        const double y = (x - 0.0375) * 53.0;
        if (ltg::emulate_exp(K, T, y) != std::exp(y)) ++bad;
    }
    if (mismatches) *mismatches = bad;
    return ok ? 0 : 1;
}
