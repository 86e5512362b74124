// Seeded inputs of the `run` command (/root/reference/proj/tools/
// tilemul_main.cpp:236-242): one mt19937_64 stream (the published 64-bit
// Mersenne Twister), uniform(-1, 1) as libstdc++'s
// uniform_real_distribution<double> computes it from one 64-bit draw
// (u = x / 2^64, clamped below 1; v = 2u - 1), operands filled A, then B,
// then C. Used by the CLI and by callers that want the reference's inputs.
#include <cmath>
#include <cstdint>

namespace mmm {

namespace {

struct Mt64 {
    uint64_t s[312];
    int i = 312;
    explicit Mt64(uint64_t seed) {
        s[0] = seed;
        for (int k = 1; k < 312; ++k) s[k] = 6364136223846793005ULL * (s[k - 1] ^ (s[k - 1] >> 62)) + k;
    }
    uint64_t next() {
        if (i >= 312) {
            for (int k = 0; k < 312; ++k) {
                const uint64_t x = (s[k] & 0xFFFFFFFF80000000ULL) | (s[(k + 1) % 312] & 0x7FFFFFFFULL);
                s[k] = s[(k + 156) % 312] ^ (x >> 1) ^ ((x & 1ULL) ? 0xB5026F5AA96619E9ULL : 0ULL);
            }
            i = 0;
        }
        uint64_t y = s[i++];
        y ^= (y >> 29) & 0x5555555555555555ULL;
        y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
        y ^= (y << 37) & 0xFFF7EEE000000000ULL;
        y ^= y >> 43;
        return y;
    }
    double uniform_pm1() {
        double u = static_cast<double>(next()) / 18446744073709551616.0;
        if (u >= 1.0) u = std::nextafter(1.0, 0.0);
        return 2.0 * u + -1.0;
    }
};

}  // namespace

void fill_seeded(uint64_t seed, double* a, int64_t na, double* b, int64_t nb, double* c, int64_t nc) {
    Mt64 g(seed);
    for (int64_t i = 0; i < na; ++i) a[i] = g.uniform_pm1();
    for (int64_t i = 0; b && i < nb; ++i) b[i] = g.uniform_pm1();
    for (int64_t i = 0; c && i < nc; ++i) c[i] = g.uniform_pm1();
}

}  // namespace mmm
