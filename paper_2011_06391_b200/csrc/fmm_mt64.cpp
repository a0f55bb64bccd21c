// fmm_mt64.cpp — jump-ahead for std::mt19937_64, so the R-MAT insertion
// stream of rmat_generate (rmat.hpp:32-58: one sequential mt19937_64) can be
// generated on the GPU by many independent sub-streams, bitwise equal to the
// sequential one.
//
// Model. With x_0..x_311 the seeded state array, the generator's words obey
//   x_{k+312} = x_{k+156} ^ ((x_k & UM | x_{k+1} & LM) >> 1) ^ (x_{k+1} & 1 ? A : 0)
// and output j is temper(x_{312+j}). Every bit sequence of the x_k is a linear
// functional of a 19937-bit state under one F2-linear map T, so all of them
// satisfy P(T) = 0 for T's minimal polynomial P (degree 19937; found once by
// Berlekamp-Massey on 2*19937 bits of one bit plane). For a jump of J:
// g(z) = z^J mod P gives x_{k+J+t} = XOR over {i : g_i = 1} of x_{k+i+t} for
// every t, i.e. the window W_{k+J} = (x_{k+J} .. x_{k+J+311}) is the XOR of
// the windows W_{k+i} (Haramoto et al.'s polynomial jump, restated).
#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstring>
#include <mutex>
#include <thread>
#include <vector>

#include "fmm_mt64.h"
#include "fusedmm_cuda.h"

namespace fmm {
namespace mt64 {
namespace {

constexpr uint64_t kA = 0xB5026F5AA96619E9ull;
constexpr uint64_t kUM = 0xFFFFFFFF80000000ull;
constexpr uint64_t kLM = 0x7FFFFFFFull;
constexpr int kDeg = 19937;
constexpr int kWords = (kDeg + 64) / 64 + 1;  // polynomial of degree <= 19937 plus slack

inline uint64_t next_word(uint64_t x0, uint64_t x1, uint64_t xm) {
    const uint64_t y = (x0 & kUM) | (x1 & kLM);
    return xm ^ (y >> 1) ^ ((x1 & 1) ? kA : 0);
}

// x[0..count) continuing the recurrence from a 312-word window
void extend(const uint64_t* w, std::vector<uint64_t>& x, size_t count) {
    x.resize(count);
    std::memcpy(x.data(), w, kN * sizeof(uint64_t));
    for (size_t k = kN; k < count; ++k) x[k] = next_word(x[k - kN], x[k - kN + 1], x[k - kN + kM]);
}

using Poly = std::vector<uint64_t>;  // bit i = coefficient of z^i

inline bool bit(const Poly& p, size_t i) { return (p[i >> 6] >> (i & 63)) & 1; }
inline void flip(Poly& p, size_t i) { p[i >> 6] ^= uint64_t(1) << (i & 63); }

int degree(const Poly& p) {
    for (size_t w = p.size(); w-- > 0;)
        if (p[w]) return static_cast<int>(w * 64 + 63 - __builtin_clzll(p[w]));
    return -1;
}

// Minimal polynomial of the bit sequence s (Berlekamp-Massey over F2),
// returned as the characteristic polynomial (reciprocal of the connection
// polynomial): P(z) = z^L + sum_i c_i z^(L-i).
// bits [off, off+64) of a (zero past the end)
inline uint64_t get64(const Poly& a, size_t off) {
    const size_t w = off >> 6, b = off & 63;
    uint64_t v = w < a.size() ? a[w] >> b : 0;
    if (b && w + 1 < a.size()) v |= a[w + 1] << (64 - b);
    return v;
}

Poly berlekamp_massey(const std::vector<uint8_t>& s) {
    const size_t N = s.size();
    Poly C(N / 64 + 2, 0), B(N / 64 + 2, 0);
    C[0] = B[0] = 1;
    // R bit (N-1-k) = s_k: the discrepancy sum_{i=0..L} c_i s_{n-i} is then
    // the parity of C[0..L] & R[N-1-n ..], word-parallel
    Poly R(N / 64 + 2, 0);
    for (size_t k = 0; k < N; ++k)
        if (s[k]) flip(R, N - 1 - k);
    size_t L = 0, m = 1;
    for (size_t n = 0; n < N; ++n) {
        uint64_t acc = 0;
        const size_t o = N - 1 - n;
        for (size_t w = 0; w * 64 <= L; ++w) {
            uint64_t c = C[w];
            if ((w + 1) * 64 > L + 1) c &= (L + 1 - w * 64 >= 64) ? ~uint64_t(0) : ((uint64_t(1) << (L + 1 - w * 64)) - 1);
            acc ^= c & get64(R, o + w * 64);
        }
        const uint8_t d = static_cast<uint8_t>(__builtin_popcountll(acc) & 1);
        if (!d) {
            ++m;
            continue;
        }
        Poly T;
        const bool grow = 2 * L <= n;
        if (grow) T = C;
        // C ^= B << m
        const size_t ws = m >> 6, bs = m & 63;
        for (size_t w = C.size(); w-- > ws;) {
            uint64_t v = B[w - ws] << bs;
            if (bs && w - ws >= 1) v |= B[w - ws - 1] >> (64 - bs);
            C[w] ^= v;
        }
        if (grow) {
            L = n + 1 - L;
            B.swap(T);
            m = 1;
        } else {
            ++m;
        }
    }
    Poly P(kWords, 0);
    for (size_t i = 0; i <= L; ++i)
        if (bit(C, i)) flip(P, L - i);
    return P;
}

// a mod P in place (a of any length), P monic of degree dP
void reduce(Poly& a, const Poly& P, int dP) {
    for (int i = degree(a); i >= dP; --i) {
        if (!bit(a, static_cast<size_t>(i))) continue;
        // a ^= P << (i - dP)
        const size_t sh = static_cast<size_t>(i - dP), ws = sh >> 6, bs = sh & 63;
        const size_t pw = static_cast<size_t>(dP / 64 + 1);
        for (size_t w = 0; w < pw && w + ws < a.size(); ++w) {
            a[w + ws] ^= P[w] << bs;
            if (bs && w + ws + 1 < a.size()) a[w + ws + 1] ^= P[w] >> (64 - bs);
        }
    }
}

// a^2 over F2: spread the bits (squaring is linear in characteristic 2)
Poly square(const Poly& a) {
    Poly r(2 * a.size() + 1, 0);
    for (size_t w = 0; w < a.size(); ++w) {
        uint64_t v = a[w];
        if (!v) continue;
        auto spread = [](uint32_t x) {
            uint64_t y = x;
            y = (y | (y << 16)) & 0x0000FFFF0000FFFFull;
            y = (y | (y << 8)) & 0x00FF00FF00FF00FFull;
            y = (y | (y << 4)) & 0x0F0F0F0F0F0F0F0Full;
            y = (y | (y << 2)) & 0x3333333333333333ull;
            y = (y | (y << 1)) & 0x5555555555555555ull;
            return y;
        };
        r[2 * w] ^= spread(static_cast<uint32_t>(v));
        r[2 * w + 1] ^= spread(static_cast<uint32_t>(v >> 32));
    }
    return r;
}

struct Model {
    Poly P;
    int dP = 0;
};

const Model& model() {
    static Model M;
    static std::once_flag once;
    std::call_once(once, [] {
        // bit 0 of x_k for 2*19937 + 64 terms from an arbitrary seed
        uint64_t w0[kN];
        seed_window(5489u, w0);
        std::vector<uint64_t> x;
        extend(w0, x, 2 * kDeg + 64 + kN);
        std::vector<uint8_t> s(2 * kDeg + 64);
        for (size_t k = 0; k < s.size(); ++k) s[k] = static_cast<uint8_t>(x[k] & 1);
        M.P = berlekamp_massey(s);
        M.dP = degree(M.P);
    });
    return M;
}

}  // namespace

void seed_window(uint64_t seed, uint64_t* w) {
    w[0] = seed;
    for (int i = 1; i < kN; ++i) w[i] = 6364136223846793005ull * (w[i - 1] ^ (w[i - 1] >> 62)) + static_cast<uint64_t>(i);
}

int poly_degree() { return model().dP; }

JumpPoly jump_poly(uint64_t J) {
    const Model& M = model();
    Poly g(kWords, 0);
    g[0] = 1;  // z^0
    for (int b = 63; b >= 0; --b) {
        g = square(g);
        reduce(g, M.P, M.dP);
        g.resize(kWords);
        if ((J >> b) & 1) {
            // g *= z
            uint64_t carry = 0;
            for (uint64_t& w : g) {
                const uint64_t nc = w >> 63;
                w = (w << 1) | carry;
                carry = nc;
            }
            reduce(g, M.P, M.dP);
        }
    }
    JumpPoly out;
    out.bits = g;
    out.degree = M.dP;
    return out;
}

void apply_jump(const JumpPoly& g, const uint64_t* in, uint64_t* out) {
    std::vector<uint64_t> x;
    extend(in, x, static_cast<size_t>(g.degree) + kN);
    uint64_t acc[kN] = {};
    for (int i = 0; i < g.degree; ++i) {
        if (!((g.bits[static_cast<size_t>(i) >> 6] >> (i & 63)) & 1)) continue;
        const uint64_t* src = x.data() + i;
        for (int k = 0; k < kN; ++k) acc[k] ^= src[k];
    }
    std::memcpy(out, acc, sizeof(acc));
}

void window_at(uint64_t seed, uint64_t position, uint64_t* out) {
    uint64_t w[kN];
    seed_window(seed, w);
    if (position == 0) {
        std::memcpy(out, w, sizeof(w));
        return;
    }
    apply_jump(jump_poly(position), w, out);
}

std::vector<uint64_t> windows(uint64_t seed, uint64_t stride, int64_t count) {
    std::vector<uint64_t> out(static_cast<size_t>(std::max<int64_t>(count, 0)) * kN);
    if (count <= 0) return out;
    seed_window(seed, out.data());
    // chains of C windows: the chain heads by jumps of C*stride (sequential),
    // the rest of each chain by jumps of stride (chains in parallel)
    const int64_t C = 64;
    const int64_t heads = (count + C - 1) / C;
    const JumpPoly gs = jump_poly(stride);
    if (heads > 1) {
        const JumpPoly gc = jump_poly(stride * static_cast<uint64_t>(C));
        for (int64_t h = 1; h < heads; ++h)
            apply_jump(gc, out.data() + (h - 1) * C * kN, out.data() + h * C * kN);
    }
    const int nt = std::max(1, std::min<int>(static_cast<int>(heads), static_cast<int>(std::thread::hardware_concurrency())));
    std::vector<std::thread> th;
    std::atomic<int64_t> next{0};
    for (int t = 0; t < nt; ++t)
        th.emplace_back([&] {
            for (int64_t h; (h = next.fetch_add(1)) < heads;)
                for (int64_t i = h * C + 1; i < std::min(count, (h + 1) * C); ++i)
                    apply_jump(gs, out.data() + (i - 1) * kN, out.data() + i * kN);
        });
    for (auto& x : th) x.join();
    return out;
}

}  // namespace mt64
}  // namespace fmm

extern "C" {

fmm_status fmm_mt64_window(uint64_t seed, uint64_t position, uint64_t* window) {
    if (!window) return FMM_E_INVAL;
    fmm::mt64::window_at(seed, position, window);
    return FMM_OK;
}

}  // extern "C"
