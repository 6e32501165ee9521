// Counter-based random numbers for the tuner (product copy; the oracle has its own, task rule ③).
//   mix64(z)        SplitMix64 finaliser of z + 0x9E3779B97F4A7C15
//   draw(s, st, c)  mix64(mix64(s ^ (st * 0xD1B54A32D192ED03)) ^ c)
//   uniform_oc(u)   ((u >> 11) + 1) * 2^-53  in (0, 1]
//   uniform_co(u)   (u >> 11) * 2^-53        in [0, 1)
//   randint(u, n)   ((u >> 11) * n) >> 53    in [0, n)
#pragma once
#include <cstdint>

namespace wpk {

inline uint64_t mix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

inline uint64_t draw(uint64_t seed, uint64_t stream, uint64_t ctr) {
    return mix64(mix64(seed ^ (stream * 0xD1B54A32D192ED03ull)) ^ ctr);
}

inline double uniform_oc(uint64_t u) { return (double)((u >> 11) + 1) * 0x1.0p-53; }
inline double uniform_co(uint64_t u) { return (double)(u >> 11) * 0x1.0p-53; }
inline uint64_t randint(uint64_t u, uint64_t n) {
    return (uint64_t)(((unsigned __int128)(u >> 11) * n) >> 53);
}

struct Rng {
    uint64_t seed, stream, ctr = 0;
    Rng(uint64_t s, uint64_t st) : seed(s), stream(st) {}
    uint64_t next() { return draw(seed, stream, ctr++); }
};

}  // namespace wpk
