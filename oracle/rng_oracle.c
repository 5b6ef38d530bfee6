/* Oracle (TEST INFRASTRUCTURE, not product code): plain-C restatement of the
 * reference's counter RNG and parameter init so the numpy oracle
 * (oracle/slapo_oracle.py) gets glibc-identical log/cos and therefore
 * bit-identical weights.
 *
 *   splitmix64 / hash_combine / uniform01 / normal01 : proj/include/slapo/rng.hpp:16-46
 *   init_plain (Normal, Uniform)                     : proj/src/module.cpp:412-431
 *   dropout keep test                                 : proj/src/executor.cpp:788-803
 */
#include <math.h>
#include <stdint.h>

static uint64_t splitmix64(uint64_t x) {
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}

uint64_t oracle_hash_combine(uint64_t a, uint64_t b) {
    return splitmix64(a ^ (b + 0x9e3779b97f4a7c15ULL + (a << 6) + (a >> 2)));
}

double oracle_uniform01(uint64_t seed, uint64_t stream, uint64_t index) {
    uint64_t h = splitmix64(oracle_hash_combine(oracle_hash_combine(seed, stream), index));
    return (double)(h >> 11) * 0x1.0p-53;
}

double oracle_normal01(uint64_t seed, uint64_t stream, uint64_t index) {
    double u1 = oracle_uniform01(seed, stream, 2 * index);
    double u2 = oracle_uniform01(seed, stream, 2 * index + 1);
    if (u1 < 1e-300) u1 = 1e-300;
    return sqrt(-2.0 * log(u1)) * cos(2.0 * M_PI * u2);
}

/* init_plain: kind 0 normal, 1 uniform, 2 zeros, 3 ones; f32 != 0 rounds through float. */
void oracle_init_plain(double* out, int64_t n, int kind, uint64_t seed, int f32) {
    for (int64_t i = 0; i < n; ++i) {
        double v = 0.0;
        if (kind == 0) v = 0.1 * oracle_normal01(seed, 0x9a7a, (uint64_t)i);
        else if (kind == 1) v = 0.2 * oracle_uniform01(seed, 0x9a7b, (uint64_t)i) - 0.1;
        else if (kind == 3) v = 1.0;
        out[i] = f32 ? (double)(float)v : v;
    }
}

void oracle_random_tensor(double* out, int64_t n, uint64_t seed, uint64_t stream, int f32) {
    for (int64_t i = 0; i < n; ++i) {
        double v = oracle_normal01(seed, stream, (uint64_t)i);
        out[i] = f32 ? (double)(float)v : v;
    }
}

/* keep[i] = uniform01(stream_seed, 0xd0, i) >= p, stream_seed = hash_combine(exec_seed, node_seed) */
void oracle_dropout_keep(uint8_t* keep, int64_t n, uint64_t exec_seed, uint64_t node_seed, double p) {
    uint64_t s = oracle_hash_combine(exec_seed, node_seed);
    for (int64_t i = 0; i < n; ++i) keep[i] = oracle_uniform01(s, 0xd0, (uint64_t)i) >= p;
}
