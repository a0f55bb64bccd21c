// fmm_gen.cpp — seeded synthetic inputs for the five BASELINE.json configs
// (host C++, exported as a plain C ABI in libfmm_gen.so).
//
// These are input generators, not part of the fused path. They restate the
// published R-MAT recursive-quadrant algorithm with the reference's RNG
// conventions — std::mt19937_64(seed), u01 = (rng() >> 11) * 2^-53 and the
// quadrant descent of rmat.hpp:32-58 — and the post-processing BASELINE.json
// asks for (self-loops dropped, symmetrised, deduplicated, columns sorted).
// The recipes are written out in SURVEY.md §8(d) and DESIGN.md.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <condition_variable>
#include <deque>
#include <mutex>
#include <thread>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <random>
#include <vector>

namespace {

struct U01 {
    std::mt19937_64 rng;
    explicit U01(uint64_t seed) : rng(seed) {}
    double operator()() { return static_cast<double>(rng() >> 11) * 0x1.0p-53; }
};

// LSD radix sort of 64-bit keys on the low `bits` bits, 16 bits per pass.
void radix_sort(std::vector<uint64_t>& keys, int bits) {
    std::vector<uint64_t> tmp(keys.size());
    for (int shift = 0; shift < bits; shift += 16) {
        std::vector<size_t> cnt(65537, 0);
        for (uint64_t k : keys) ++cnt[((k >> shift) & 0xffff) + 1];
        for (int i = 0; i < 65536; ++i) cnt[i + 1] += cnt[i];
        for (uint64_t k : keys) tmp[cnt[(k >> shift) & 0xffff]++] = k;
        keys.swap(tmp);
    }
}

// keys = (row << 32) | col, sorted -> unique -> CSR
void keys_to_csr(std::vector<uint64_t>& keys, int64_t m, int key_bits, int64_t** row_ptr,
                 int64_t** col, int64_t* nnz) {
    radix_sort(keys, key_bits);
    keys.erase(std::unique(keys.begin(), keys.end()), keys.end());
    *nnz = static_cast<int64_t>(keys.size());
    *row_ptr = static_cast<int64_t*>(std::malloc(sizeof(int64_t) * (m + 1)));
    *col = static_cast<int64_t*>(std::malloc(sizeof(int64_t) * std::max<size_t>(1, keys.size())));
    std::memset(*row_ptr, 0, sizeof(int64_t) * (m + 1));
    for (size_t i = 0; i < keys.size(); ++i) {
        (*row_ptr)[(keys[i] >> 32) + 1]++;
        (*col)[i] = static_cast<int64_t>(keys[i] & 0xffffffffu);
    }
    for (int64_t r = 0; r < m; ++r) (*row_ptr)[r + 1] += (*row_ptr)[r];
}

int bits_for(int64_t m) {
    int b = 0;
    while ((int64_t(1) << b) < m) ++b;
    return b;
}

int num_threads() { return std::max(1, static_cast<int>(std::thread::hardware_concurrency())); }

template <class Fn>
void parallel_for(int64_t n, Fn fn) {
    std::atomic<int64_t> next{0};
    std::vector<std::thread> th;
    const int nt = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(n, num_threads())));
    for (int t = 0; t < nt; ++t)
        th.emplace_back([&] {
            for (int64_t i; (i = next.fetch_add(1)) < n;) fn(i);
        });
    for (auto& x : th) x.join();
}

// MT19937-64 (Matsumoto & Nishimura's published algorithm), bit-identical to
// std::mt19937_64 (checked by fmmgen_mt64_check), with the twist and the
// tempering done over whole 312-word state blocks so the compiler vectorises
// them — the sequential part of R-MAT generation.
struct MT64 {
    static constexpr int N = 312, M = 156;
    static constexpr uint64_t A = 0xB5026F5AA96619E9ull, UM = 0xFFFFFFFF80000000ull, LM = 0x7FFFFFFFull;
    uint64_t mt[N];
    int idx = N;
    explicit MT64(uint64_t seed) {
        mt[0] = seed;
        for (int i = 1; i < N; ++i) mt[i] = 6364136223846793005ull * (mt[i - 1] ^ (mt[i - 1] >> 62)) + i;
    }
    static uint64_t mix(uint64_t hi, uint64_t lo, uint64_t far) {
        const uint64_t y = (hi & UM) | (lo & LM);
        return far ^ (y >> 1) ^ ((y & 1) ? A : 0);
    }
    void twist() {
        for (int i = 0; i < N - M; ++i) mt[i] = mix(mt[i], mt[i + 1], mt[i + M]);
        for (int i = N - M; i < N - 1; ++i) mt[i] = mix(mt[i], mt[i + 1], mt[i + M - N]);
        mt[N - 1] = mix(mt[N - 1], mt[0], mt[M - 1]);
        idx = 0;
    }
    static uint64_t temper(uint64_t y) {
        y ^= (y >> 29) & 0x5555555555555555ull;
        y ^= (y << 17) & 0x71D67FFFEDA60000ull;
        y ^= (y << 37) & 0xFFF7EEE000000000ull;
        y ^= y >> 43;
        return y;
    }
    void fill(uint64_t* out, size_t n) {
        size_t k = 0;
        while (k < n) {
            if (idx == N) twist();
            const size_t take = std::min<size_t>(n - k, static_cast<size_t>(N - idx));
            for (size_t j = 0; j < take; ++j) out[k + j] = temper(mt[idx + j]);
            idx += static_cast<int>(take);
            k += take;
        }
    }
};

struct RawBlock {
    int64_t index = 0, edges = 0;
    std::vector<uint64_t> words;
};

// Bounded producer / consumer queue of raw random blocks.
class WorkQueue {
public:
    explicit WorkQueue(size_t cap) : cap_(cap) {}
    void push(RawBlock&& b) {
        std::unique_lock<std::mutex> lk(mu_);
        not_full_.wait(lk, [&] { return q_.size() < cap_; });
        q_.push_back(std::move(b));
        not_empty_.notify_one();
    }
    bool pop(RawBlock* out) {
        std::unique_lock<std::mutex> lk(mu_);
        not_empty_.wait(lk, [&] { return !q_.empty() || closed_; });
        if (q_.empty()) return false;
        *out = std::move(q_.front());
        q_.pop_front();
        not_full_.notify_one();
        return true;
    }
    void close() {
        std::lock_guard<std::mutex> lk(mu_);
        closed_ = true;
        not_empty_.notify_all();
    }

private:
    size_t cap_;
    bool closed_ = false;
    std::deque<RawBlock> q_;
    std::mutex mu_;
    std::condition_variable not_empty_, not_full_;
};

// Parallel LSD radix sort on the low `bits` bits, 16-bit digits: per-thread
// histograms of contiguous chunks, then a stable scatter.
void parallel_radix_sort(std::vector<uint64_t>& keys, int bits) {
    const int64_t n = static_cast<int64_t>(keys.size());
    const int T = num_threads();
    std::vector<uint64_t> tmp(keys.size());
    std::vector<std::vector<int64_t>> hist(static_cast<size_t>(T), std::vector<int64_t>(65536));
    for (int shift = 0; shift < bits; shift += 16) {
        auto lo = [&](int t) { return n * t / T; };
        parallel_for(T, [&](int64_t t) {
            auto& h = hist[t];
            std::fill(h.begin(), h.end(), 0);
            for (int64_t i = lo(static_cast<int>(t)); i < lo(static_cast<int>(t) + 1); ++i) ++h[(keys[i] >> shift) & 0xffff];
        });
        int64_t run = 0;
        for (int dgt = 0; dgt < 65536; ++dgt)
            for (int t = 0; t < T; ++t) {
                const int64_t c = hist[t][dgt];
                hist[t][dgt] = run;
                run += c;
            }
        parallel_for(T, [&](int64_t t) {
            auto& h = hist[t];
            for (int64_t i = lo(static_cast<int>(t)); i < lo(static_cast<int>(t) + 1); ++i)
                tmp[h[(keys[i] >> shift) & 0xffff]++] = keys[i];
        });
        keys.swap(tmp);
    }
}

// keys = row << scale | col: sort, unique, CSR (int64 row_ptr / col).
void packed_keys_to_csr(std::vector<uint64_t>& keys, int64_t m, int scale, int64_t** row_ptr,
                        int64_t** col, int64_t* nnz) {
    parallel_radix_sort(keys, 2 * scale);
    keys.erase(std::unique(keys.begin(), keys.end()), keys.end());
    const int64_t nk = static_cast<int64_t>(keys.size());
    *nnz = nk;
    *row_ptr = static_cast<int64_t*>(std::malloc(sizeof(int64_t) * (m + 1)));
    *col = static_cast<int64_t*>(std::malloc(sizeof(int64_t) * std::max<int64_t>(1, nk)));
    const uint64_t mask = (uint64_t(1) << scale) - 1;
    int64_t* rp = *row_ptr;
    int64_t* cl = *col;
    parallel_for((nk + (1 << 20) - 1) >> 20, [&](int64_t b) {
        const int64_t e = std::min(nk, (b + 1) << 20);
        for (int64_t i = b << 20; i < e; ++i) cl[i] = static_cast<int64_t>(keys[i] & mask);
    });
    // row_ptr[r] = first position with row >= r (keys sorted)
    int64_t pos = 0;
    for (int64_t r = 0; r <= m; ++r) {
        while (pos < nk && static_cast<int64_t>(keys[pos] >> scale) < r) ++pos;
        rp[r] = pos;
    }
}

}  // namespace

extern "C" {

void fmmgen_free(void* p) { std::free(p); }

// Number of the first n outputs where the bulk MT64 differs from
// std::mt19937_64(seed) (0 expected).
int64_t fmmgen_mt64_check(uint64_t seed, int64_t n) {
    std::mt19937_64 ref(seed);
    MT64 mt(seed);
    std::vector<uint64_t> buf(static_cast<size_t>(n));
    // uneven chunks exercise the block boundaries
    for (int64_t k = 0, step = 1; k < n; k += step, step = step * 3 % 1000 + 1)
        mt.fill(buf.data() + k, static_cast<size_t>(std::min<int64_t>(step, n - k)));
    int64_t bad = 0;
    for (int64_t i = 0; i < n; ++i) bad += buf[i] != ref();
    return bad;
}

// Config 1: n rows, each with exactly k distinct out-neighbours drawn as
// floor(u01*n) until k are distinct (self allowed), sorted ascending; then
// a_uv = u01 drawn in sorted order. X (n x d, optional) continues the same
// stream as U(-1,1): x = -1 + 2*u01.
int fmmgen_er_fixed(int64_t n, int k, uint64_t seed, int64_t* row_ptr, int64_t* col, float* val,
                    float* X, int64_t d) {
    if (n < 1 || k < 0 || k > n) return 1;
    U01 u(seed);
    std::vector<int64_t> pick;
    pick.reserve(k);
    row_ptr[0] = 0;
    for (int64_t r = 0; r < n; ++r) {
        pick.clear();
        while (static_cast<int>(pick.size()) < k) {
            const int64_t v = static_cast<int64_t>(u() * static_cast<double>(n));
            if (std::find(pick.begin(), pick.end(), v) == pick.end()) pick.push_back(v);
        }
        std::sort(pick.begin(), pick.end());
        for (int i = 0; i < k; ++i) {
            col[r * k + i] = pick[i];
            val[r * k + i] = static_cast<float>(u());
        }
        row_ptr[r + 1] = (r + 1) * k;
    }
    if (X)
        for (int64_t i = 0; i < n * d; ++i) X[i] = static_cast<float>(-1.0 + 2.0 * u());
    return 0;
}

// Configs 2, 3, 5: the R-MAT insertion stream of rmat.hpp:24-61 (scale,
// edge_factor * 2^scale insertions, quadrant probabilities a, b, c, 1-a-b-c),
// then self-loops dropped, every (u,v) inserted as (u,v) and (v,u), sorted and
// deduplicated. Arrays are malloc'd; release with fmmgen_free.
int fmmgen_rmat_sym(int scale, int edge_factor, double a, double b, double c, uint64_t seed,
                    int64_t** row_ptr, int64_t** col, int64_t* nnz) {
    if (scale < 1 || scale > 30 || edge_factor < 0) return 1;
    const int64_t nverts = int64_t(1) << scale;
    const int64_t nedges = static_cast<int64_t>(edge_factor) * nverts;
    // The stream is inherently sequential (one mt19937_64), so the main
    // thread only generates raw 64-bit words in bulk while workers run the
    // quadrant descents of whole blocks of insertions; keys are packed as
    // row << scale | col and sorted with a parallel LSD radix sort.
    const double ab = a + b, abc = a + b + c;
    // u01 < t  <=>  (r >> 11) < ceil(t * 2^53)   (exact, t in [0, 1])
    const uint64_t ta = static_cast<uint64_t>(std::ceil(a * 0x1.0p53));
    const uint64_t tab = static_cast<uint64_t>(std::ceil(ab * 0x1.0p53));
    const uint64_t tabc = static_cast<uint64_t>(std::ceil(abc * 0x1.0p53));
    const int64_t kBlockEdges = int64_t(1) << 18;
    const int64_t nblocks = (nedges + kBlockEdges - 1) / kBlockEdges;
    std::vector<std::vector<uint64_t>> block_keys(static_cast<size_t>(nblocks));
    const int workers = std::max(1, static_cast<int>(std::thread::hardware_concurrency()) - 1);
    WorkQueue q(static_cast<size_t>(2 * workers + 2));
    std::vector<std::thread> pool;
    for (int t = 0; t < workers; ++t)
        pool.emplace_back([&] {
            RawBlock blk;
            while (q.pop(&blk)) {
                std::vector<uint64_t>& out = block_keys[blk.index];
                out.reserve(static_cast<size_t>(2 * blk.edges));
                const uint64_t* r = blk.words.data();
                for (int64_t e = 0; e < blk.edges; ++e) {
                    uint64_t row = 0, cl = 0;
                    for (int level = 0; level < scale; ++level) {
                        const uint64_t k = (*r++) >> 11;
                        row <<= 1;
                        cl <<= 1;
                        if (k < ta) {
                        } else if (k < tab) {
                            cl |= 1;
                        } else if (k < tabc) {
                            row |= 1;
                        } else {
                            row |= 1;
                            cl |= 1;
                        }
                    }
                    if (row == cl) continue;
                    out.push_back((row << scale) | cl);
                    out.push_back((cl << scale) | row);
                }
            }
        });
    MT64 mt(seed);
    for (int64_t bi = 0; bi < nblocks; ++bi) {
        RawBlock blk;
        blk.index = bi;
        blk.edges = std::min(kBlockEdges, nedges - bi * kBlockEdges);
        blk.words.resize(static_cast<size_t>(blk.edges * scale));
        mt.fill(blk.words.data(), blk.words.size());
        q.push(std::move(blk));
    }
    q.close();
    for (auto& th : pool) th.join();
    // concatenate
    std::vector<int64_t> off(static_cast<size_t>(nblocks) + 1, 0);
    for (int64_t bi = 0; bi < nblocks; ++bi) off[bi + 1] = off[bi] + static_cast<int64_t>(block_keys[bi].size());
    std::vector<uint64_t> keys(static_cast<size_t>(off[nblocks]));
    parallel_for(nblocks, [&](int64_t bi) {
        std::copy(block_keys[bi].begin(), block_keys[bi].end(), keys.begin() + off[bi]);
        std::vector<uint64_t>().swap(block_keys[bi]);
    });
    packed_keys_to_csr(keys, nverts, scale, row_ptr, col, nnz);
    return 0;
}

// The raw (un-postprocessed) R-MAT insertion stream as COO, for cross-checks
// against the reference generator. rows/cols must hold edge_factor*2^scale.
int fmmgen_rmat_stream(int scale, int edge_factor, double a, double b, double c, uint64_t seed,
                       int64_t* rows, int64_t* cols) {
    if (scale < 1 || scale > 30) return 1;
    const int64_t nedges = static_cast<int64_t>(edge_factor) << scale;
    U01 u(seed);
    const double ab = a + b, abc = a + b + c;
    for (int64_t e = 0; e < nedges; ++e) {
        int64_t row = 0, cl = 0;
        for (int level = 0; level < scale; ++level) {
            const double x = u();
            row <<= 1;
            cl <<= 1;
            if (x < a) {
            } else if (x < ab) {
                cl |= 1;
            } else if (x < abc) {
                row |= 1;
            } else {
                row |= 1;
                cl |= 1;
            }
        }
        rows[e] = row;
        cols[e] = cl;
    }
    return 0;
}

// Config 4: side x side 4-neighbour lattice (v = r*side + c; right and down
// edges) plus, for every v in order, one shortcut w = floor(u01*n) (dropped
// when w == v); symmetrised, deduplicated, sorted. X (n x 2, optional)
// continues the stream: x_v = (c + 0.01*N, r + 0.01*N), normals by
// Box-Muller on two u01 draws (both outputs used).
int fmmgen_lattice(int64_t side, uint64_t seed, int64_t** row_ptr, int64_t** col, int64_t* nnz,
                   float* X) {
    if (side < 1 || side > 46340) return 1;
    const int64_t n = side * side;
    U01 u(seed);
    std::vector<uint64_t> keys;
    keys.reserve(static_cast<size_t>(6 * n));
    auto add = [&](uint64_t p, uint64_t q) {
        keys.push_back((p << 32) | q);
        keys.push_back((q << 32) | p);
    };
    for (int64_t r = 0; r < side; ++r)
        for (int64_t c = 0; c < side; ++c) {
            const uint64_t v = static_cast<uint64_t>(r * side + c);
            if (c + 1 < side) add(v, v + 1);
            if (r + 1 < side) add(v, v + static_cast<uint64_t>(side));
        }
    for (int64_t v = 0; v < n; ++v) {
        const int64_t w = static_cast<int64_t>(u() * static_cast<double>(n));
        if (w != v) add(static_cast<uint64_t>(v), static_cast<uint64_t>(w));
    }
    keys_to_csr(keys, n, 32 + bits_for(n), row_ptr, col, nnz);
    if (X) {
        const double two_pi = 6.283185307179586476925286766559;
        for (int64_t v = 0; v < n; ++v) {
            const double u1 = u(), u2 = u();
            const double rad = std::sqrt(-2.0 * std::log(1.0 - u1));
            const double n0 = rad * std::cos(two_pi * u2), n1 = rad * std::sin(two_pi * u2);
            X[2 * v + 0] = static_cast<float>(static_cast<double>(v % side) + 0.01 * n0);
            X[2 * v + 1] = static_cast<float>(static_cast<double>(v / side) + 0.01 * n1);
        }
    }
    return 0;
}

// X[i] = scale * N(0,1), Box-Muller pairs from a fresh mt19937_64(seed).
// Dense fills are block-parallel: block b (kFillBlock elements) draws from its
// own mt19937_64(block_seed(seed, b)), so the result is independent of the
// thread count and config 5's 4.3e9 values fill in seconds.
}  // extern "C"
namespace {
constexpr int64_t kFillBlock = int64_t(1) << 20;

uint64_t block_seed(uint64_t seed, int64_t b) {
    uint64_t z = seed + 0x9E3779B97F4A7C15ull * static_cast<uint64_t>(b + 1);  // splitmix64
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

template <class Fn>
void parallel_blocks(int64_t count, Fn fn) {
    const int64_t nb = (count + kFillBlock - 1) / kFillBlock;
    const int nt = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(nb, std::thread::hardware_concurrency())));
    std::atomic<int64_t> next{0};
    std::vector<std::thread> th;
    for (int t = 0; t < nt; ++t)
        th.emplace_back([&] {
            for (int64_t b; (b = next.fetch_add(1)) < nb;)
                fn(b, b * kFillBlock, std::min(count, (b + 1) * kFillBlock));
        });
    for (auto& x : th) x.join();
}
}  // namespace
extern "C" {

// X[i] = scale * N(0,1), Box-Muller pairs (both outputs used) per block.
void fmmgen_normal_fill(float* X, int64_t count, double scale, uint64_t seed) {
    const double two_pi = 6.283185307179586476925286766559;
    parallel_blocks(count, [&](int64_t b, int64_t lo, int64_t hi) {
        U01 u(block_seed(seed, b));
        for (int64_t i = lo; i < hi; i += 2) {
            const double u1 = u(), u2 = u();
            const double rad = std::sqrt(-2.0 * std::log(1.0 - u1));
            X[i] = static_cast<float>(scale * rad * std::cos(two_pi * u2));
            if (i + 1 < hi) X[i + 1] = static_cast<float>(scale * rad * std::sin(two_pi * u2));
        }
    });
}

// X[i] = lo + (hi-lo)*u01 per block.
void fmmgen_uniform_fill(float* X, int64_t count, double lo_v, double hi_v, uint64_t seed) {
    parallel_blocks(count, [&](int64_t b, int64_t lo, int64_t hi) {
        U01 u(block_seed(seed, b));
        for (int64_t i = lo; i < hi; ++i) X[i] = static_cast<float>(lo_v + (hi_v - lo_v) * u());
    });
}

}  // extern "C"
