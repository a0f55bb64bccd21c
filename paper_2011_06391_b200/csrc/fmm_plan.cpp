// fmm_plan.cpp — see fmm_plan.h.
#include "fmm_plan.h"

#include <algorithm>
#include <cstdlib>
#include <functional>
#include <queue>
#include <stdexcept>

namespace fmm {

int wide_min(int chunk) {
    static const int env = [] {
        const char* e = std::getenv("FMM_WIDE");
        const int v = e ? std::atoi(e) : 0;
        return (v >= 8 && (v & (v - 1)) == 0) ? v : 0;
    }();
    if (env) return env;
    return std::max(64, std::min(kWideMin, chunk / 16));
}

int wide_level_for(int chunk, int d) {
    static const int env = [] {
        const char* e = std::getenv("FMM_WIDE");
        return e ? std::atoi(e) : 0;
    }();
    int thr = env > 0 ? env : std::max(64, std::min(d >= 64 ? 512 : 128, chunk / 4));
    int k = 0;
    while (k + 1 < kWideLevels && (64 << (k + 1)) <= thr) ++k;
    return k;
}

BandParams choose_bands(int64_t n) {
    BandParams b;
    auto env_int = [](const char* name, int64_t dflt) {
        const char* e = std::getenv(name);
        return e ? static_cast<int64_t>(std::atoll(e)) : dflt;
    };
    if (env_int("FMM_BANDS", 1) == 0) return b;
    const int64_t cols = env_int("FMM_BAND_COLS", 65536);
    // at least 128 bands: X several times the L2 at any d >= 32 (configs 2 and
    // 3, 16-32 bands of this width, lose 7-50% to the extra pieces: r3x)
    if (cols > 0 && n >= 128 * cols) b.band_cols = cols;
    b.min_deg = static_cast<int>(std::max<int64_t>(64, env_int("FMM_BAND_MINDEG", b.min_deg)));
    b.min_len = static_cast<int>(std::max<int64_t>(1, env_int("FMM_BAND_MINLEN", b.min_len)));
    return b;
}

int choose_chunk_edges(int64_t total_nnz) {
    if (const char* e = std::getenv("FMM_CHUNK")) {
        const int v = std::atoi(e);
        if (v >= 32) return v;
    }
    int c = 256;
    while (c < 16384 && static_cast<int64_t>(c) * 16384 * 3 / 2 < total_nnz) c *= 2;
    return c;
}

std::vector<int64_t> part1d(int64_t m, const int64_t* row_ptr, int t) {
    if (t < 1) throw std::invalid_argument("part1d: worker count must be >= 1");
    std::vector<int64_t> b(static_cast<size_t>(t) + 1, 0);
    b[0] = 0;
    b[t] = m;
    const int64_t base = m >= 0 ? row_ptr[0] : 0;
    const int64_t nnz = row_ptr[m] - base;
    if (nnz == 0) {
        for (int i = 1; i < t; ++i) b[i] = m * i / t;
        return b;
    }
    int64_t row = 0;
    for (int i = 1; i < t; ++i) {
        while (row < m && (row_ptr[row] - base) * static_cast<int64_t>(t) <
                              static_cast<int64_t>(i) * nnz)
            ++row;
        b[i] = row;
    }
    return b;
}

std::vector<int64_t> part1d_weighted(int64_t m, const int64_t* row_ptr, int t, double w) {
    if (!(w > 0.0)) return part1d(m, row_ptr, t);
    if (t < 1) throw std::invalid_argument("part1d: worker count must be >= 1");
    std::vector<int64_t> b(static_cast<size_t>(t) + 1, 0);
    b[t] = m;
    const int64_t base = row_ptr[0];
    const long double total = static_cast<long double>(row_ptr[m] - base) + static_cast<long double>(w) * m;
    int64_t row = 0;
    for (int i = 1; i < t; ++i) {
        const long double target = total * i / t;
        while (row < m && static_cast<long double>(row_ptr[row] - base) + static_cast<long double>(w) * row < target)
            ++row;
        b[i] = row;
    }
    return b;
}

std::string validate_row_ptr(int64_t m, const int64_t* row_ptr) {
    if (m < 0) return "negative row count";
    if (row_ptr[0] != 0) return "row_ptr[0] != 0";
    for (int64_t i = 1; i <= m; ++i)
        if (row_ptr[i] < row_ptr[i - 1])
            return "row_ptr not monotone at index " + std::to_string(i);
    return {};
}

namespace {
// Degree bucket: 0 for empty rows, else 1 + 4*floor(log2 deg) + next two bits.
// Degree buckets, monotone in deg: power-of-two below 8, so narrow-degree
// graphs (lattices) keep their natural row order — sequential x_u / Z / CSR
// traffic — and quarter-octaves from 8 up, so rows sharing a warp have
// similar lengths and power-law hubs run first (LPT).
inline int degree_bucket(int64_t deg) {
    if (deg <= 0) return 0;
    const int lg = 63 - __builtin_clzll(static_cast<unsigned long long>(deg));
    if (lg < 3) return 1 + lg;
    return 4 + 4 * (lg - 3) + static_cast<int>((deg >> (lg - 2)) & 3);
}
}  // namespace

ShardPlan build_shard_plan(const int64_t* row_ptr, int64_t row_begin, int64_t row_end, int chunk,
                           const int64_t* col_idx, BandParams bands) {
    ShardPlan P;
    const bool banding = bands.band_cols > 0 && col_idx != nullptr;
    auto is_split = [&](int64_t deg) { return deg > chunk || (banding && deg >= bands.min_deg); };
    P.chunk = chunk;
    P.wide = wide_min(chunk);
    P.row_begin = row_begin;
    P.row_end = row_end;
    P.edge_begin = row_ptr[row_begin];
    P.nnz = row_ptr[row_end] - row_ptr[row_begin];
    const int64_t rows = row_end - row_begin;
    if (rows > INT32_MAX) throw std::invalid_argument("shard has more than 2^31-1 rows");
    P.local_row_ptr.resize(static_cast<size_t>(rows) + 1);
    for (int64_t i = 0; i <= rows; ++i) P.local_row_ptr[i] = row_ptr[row_begin + i] - P.edge_begin;

    // counting sort by (split?, bucket) descending, stable
    constexpr int kBuckets = 1 + 4 * 64 + 4;
    constexpr int kKeys = 2 * kBuckets;
    std::vector<int64_t> count(kKeys + 1, 0);
    auto key_of = [&](int64_t r) {
        const int64_t deg = P.local_row_ptr[r + 1] - P.local_row_ptr[r];
        const int split = is_split(deg) ? 1 : 0;
        // descending: larger key first
        return kKeys - 1 - (split * kBuckets + degree_bucket(deg));
    };
    for (int64_t r = 0; r < rows; ++r) {
        const int64_t deg = P.local_row_ptr[r + 1] - P.local_row_ptr[r];
        if (deg > 0) ++P.nonempty_rows;
        P.max_degree = std::max(P.max_degree, deg);
        if (is_split(deg)) ++P.n_split_rows;
        else {
            if (deg >= P.wide) ++P.n_wide_rows;
            for (int k = 0; k < kWideLevels && deg >= (64 << k); ++k) ++P.n_wide_at[k];
        }
        ++count[key_of(r) + 1];
    }
    for (int k = 0; k < kKeys; ++k) count[k + 1] += count[k];
    P.order.resize(static_cast<size_t>(rows));
    for (int64_t r = 0; r < rows; ++r) P.order[count[key_of(r)]++] = static_cast<int32_t>(r);
    // inside every bucket of degree >= 16, rows by descending exact degree, so
    // the lane groups of a warp end together (configs 2 / 3 / 5: -1 to -2%);
    // lower buckets keep the natural order (lattice locality, config 4)
    {
        auto degree = [&](int32_t r) { return P.local_row_ptr[r + 1] - P.local_row_ptr[r]; };
        int64_t i = 0;
        while (i < rows) {
            const int k = key_of(P.order[i]);
            int64_t j = i + 1;
            while (j < rows && key_of(P.order[j]) == k) ++j;
            if (degree(P.order[i]) >= 16)
                std::stable_sort(P.order.begin() + i, P.order.begin() + j,
                                 [&](int32_t a, int32_t b) { return degree(a) > degree(b); });
            i = j;
        }
    }
    P.items.resize(static_cast<size_t>(rows));
    for (int64_t i = 0; i < rows; ++i) {
        const int32_t r = P.order[i];
        const int64_t e0 = P.local_row_ptr[r];
        const int64_t deg = P.local_row_ptr[r + 1] - e0;
        if (deg > INT32_MAX) throw std::invalid_argument("row degree >= 2^31");
        P.items[i] = {r, static_cast<int32_t>(static_cast<uint32_t>(e0 & 0xffffffffll)),
                      static_cast<int32_t>(e0 >> 32), static_cast<int32_t>(deg)};
    }

    // chunk items for the split prefix, slots assigned row by row; the items
    // then run band-major (a fixed-size chunk counts under its first column's
    // band when the columns are at hand, else under its index)
    int64_t slot = 0;
    P.split_rows.reserve(static_cast<size_t>(P.n_split_rows));
    std::vector<int64_t> item_band;
    std::vector<std::pair<int32_t, int32_t>> pieces;  // {first edge (row-relative), edges}
    for (int64_t i = 0; i < P.n_split_rows; ++i) {
        const int32_t r = P.order[i];
        const int64_t deg = P.local_row_ptr[r + 1] - P.local_row_ptr[r];
        const int64_t* c = col_idx ? col_idx + P.edge_begin + P.local_row_ptr[r] : nullptr;
        pieces.clear();
        bool banded = banding && deg >= bands.min_deg;
        if (banded) {
            auto band_of = [&](int64_t col) { return col < 0 ? int64_t(0) : col / bands.band_cols; };
            int64_t start = 0, cur = band_of(c[0]);
            for (int64_t e = 1; e < deg && banded; ++e) {
                if (c[e] < c[e - 1]) { banded = false; break; }  // unsorted row: fixed chunks
                const int64_t b = band_of(c[e]);
                if (b != cur) {
                    if (e - start >= bands.min_len) {
                        pieces.push_back({static_cast<int32_t>(start), static_cast<int32_t>(e - start)});
                        start = e;
                    }
                    cur = b;
                }
            }
            if (banded) {
                if (deg - start < bands.min_len && !pieces.empty()) pieces.back().second += static_cast<int32_t>(deg - start);
                else pieces.push_back({static_cast<int32_t>(start), static_cast<int32_t>(deg - start)});
                ++P.n_banded_rows;
            } else {
                pieces.clear();
            }
        }
        if (!banded) pieces.push_back({0, static_cast<int32_t>(deg)});
        // no piece longer than the chunk size
        int64_t nch = 0;
        for (const auto& pc : pieces) nch += (pc.second + P.chunk - 1) / P.chunk;
        if (slot + nch > INT32_MAX) throw std::invalid_argument("too many chunk slots");
        const int32_t si = static_cast<int32_t>(P.split_rows.size());
        P.split_rows.push_back({r, static_cast<int32_t>(slot), static_cast<int32_t>(nch), 0});
        int64_t k = 0;
        for (const auto& pc : pieces)
            for (int32_t off = 0; off < pc.second; off += P.chunk, ++k) {
                const int32_t e0 = pc.first + off;
                const int32_t len = std::min<int32_t>(P.chunk, pc.second - off);
                P.chunks.push_back({si, e0, len, static_cast<int32_t>(slot + k)});
                item_band.push_back(c && banding ? std::max<int64_t>(c[e0], 0) / bands.band_cols : 0);
            }
        slot += nch;
    }
    if (banding && P.n_banded_rows > 0) {
        // band-major, longest first inside a band; stable on (row, piece) order
        std::vector<int64_t> idx(P.chunks.size());
        for (size_t q = 0; q < idx.size(); ++q) idx[q] = static_cast<int64_t>(q);
        std::stable_sort(idx.begin(), idx.end(), [&](int64_t a, int64_t b) {
            if (item_band[a] != item_band[b]) return item_band[a] < item_band[b];
            return P.chunks[a].z > P.chunks[b].z;
        });
        std::vector<Int4> sorted(P.chunks.size());
        for (size_t q = 0; q < idx.size(); ++q) sorted[q] = P.chunks[idx[q]];
        P.chunks.swap(sorted);
    }
    P.n_slots = slot;
    return P;
}

}  // namespace fmm
