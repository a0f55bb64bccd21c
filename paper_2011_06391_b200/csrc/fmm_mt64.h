// fmm_mt64.h — std::mt19937_64 jump-ahead (host), see fmm_mt64.cpp.
#pragma once

#include <cstdint>
#include <vector>

namespace fmm {
namespace mt64 {

constexpr int kN = 312;  // state words
constexpr int kM = 156;  // recurrence offset

// z^J mod P (P: the degree-19937 minimal polynomial of the generator)
struct JumpPoly {
    std::vector<uint64_t> bits;
    int degree = 0;
};

// x_0..x_311 of std::mt19937_64(seed) (its seeding rule)
void seed_window(uint64_t seed, uint64_t* w);
int poly_degree();
JumpPoly jump_poly(uint64_t J);
// out = W_{k+J} from in = W_k (312 words each)
void apply_jump(const JumpPoly& g, const uint64_t* in, uint64_t* out);
// W_p = (x_p .. x_{p+311}) of std::mt19937_64(seed): the next outputs are
// temper(x_{p+312}), temper(x_{p+313}), ... (output j is temper(x_{312+j}))
void window_at(uint64_t seed, uint64_t position, uint64_t* out);
// W_{s*stride} for s in [0, count), count*312 words (host threads)
std::vector<uint64_t> windows(uint64_t seed, uint64_t stride, int64_t count);

}  // namespace mt64
}  // namespace fmm
