// fmm_mmio.cpp — MatrixMarket ingestion (mmio.hpp).
//
// fmm_read_matrix_market restates read_matrix_market (mmio.hpp:23-84): the
// header, comment, size-line and entry rules and their error messages
// ("<path>:<line>: <what>") on the host, then the duplicate fold and storage
// order of csr_from_coo on the GPU (fmm_csr_from_coo). fmm_write_matrix_market
// restates write_matrix_market (mmio.hpp:87-99): coordinate real general,
// 1-based, values printed with 17 significant digits.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "fusedmm_cuda.h"

namespace {

void set_msg(char* err, size_t cap, const std::string& msg) {
    if (!err || cap == 0) return;
    const size_t k = std::min(cap - 1, msg.size());
    std::memcpy(err, msg.data(), k);
    err[k] = '\0';
}

struct Parsed {
    int64_t m = 0, n = 0;
    std::vector<int64_t> rows, cols;
    std::vector<float> vals;
};

// A cursor over one line of the file (no terminating newline). The field
// readers follow C++ stream extraction (operator>>) exactly, because the
// reference's error messages depend on where extraction fails: skip
// isspace, then an integer is [+-]digits (overflow fails) and a double is
// the longest [+-]digits[.digits][(e|E)[+-]digits] prefix, which must then
// convert completely ("inf", "nan" and hex floats do not extract).
struct Cursor {
    const char* p;
    const char* end;

    void skip_space() {
        while (p < end && (*p == ' ' || *p == '\t' || *p == '\r' || *p == '\v' || *p == '\f')) ++p;
    }
    bool word(std::string* out) {
        skip_space();
        const char* b = p;
        while (p < end && !(*p == ' ' || *p == '\t' || *p == '\r' || *p == '\v' || *p == '\f')) ++p;
        out->assign(b, p);
        return p > b;
    }
    bool integer(int64_t* out) {
        skip_space();
        bool neg = false;
        if (p < end && (*p == '+' || *p == '-')) neg = *p++ == '-';
        if (p >= end || *p < '0' || *p > '9') return false;
        uint64_t v = 0;
        const uint64_t lim = neg ? uint64_t(INT64_MAX) + 1 : uint64_t(INT64_MAX);
        for (; p < end && *p >= '0' && *p <= '9'; ++p) {
            const uint64_t dgt = static_cast<uint64_t>(*p - '0');
            if (v > (lim - dgt) / 10) return false;  // out of range: extraction fails
            v = v * 10 + dgt;
        }
        *out = neg ? static_cast<int64_t>(0 - v) : static_cast<int64_t>(v);
        return true;
    }
    bool real(double* out) {
        skip_space();
        std::string tok;
        auto digits = [&] {
            size_t k = 0;
            for (; p < end && *p >= '0' && *p <= '9'; ++p, ++k) tok.push_back(*p);
            return k;
        };
        if (p < end && (*p == '+' || *p == '-')) tok.push_back(*p++);
        size_t mant = digits();
        if (p < end && *p == '.') {
            tok.push_back(*p++);
            mant += digits();
        }
        if (mant == 0) return false;
        if (p < end && (*p == 'e' || *p == 'E')) {
            tok.push_back(*p++);
            if (p < end && (*p == '+' || *p == '-')) tok.push_back(*p++);
            if (digits() == 0) return false;  // "1e": the collected token does not convert
        }
        char* stop = nullptr;
        const double v = std::strtod(tok.c_str(), &stop);
        // overflow fails (the stream reports +-max with failbit); underflow
        // to a subnormal or zero is accepted, as by libstdc++'s num_get
        if (*stop != '\0' || v == HUGE_VAL || v == -HUGE_VAL) return false;
        *out = v;
        return true;
    }
};

// The file as lines, numbered from 1 like std::getline: a final line
// without a newline counts, nothing after the last newline does.
class LineReader {
public:
    explicit LineReader(std::string text) : buf_(std::move(text)) {}
    bool next(Cursor* c) {
        if (pos_ >= buf_.size()) return false;
        const size_t nl = buf_.find('\n', pos_);
        const size_t stop = nl == std::string::npos ? buf_.size() : nl;
        c->p = buf_.data() + pos_;
        c->end = buf_.data() + stop;
        pos_ = nl == std::string::npos ? buf_.size() : nl + 1;
        ++lineno_;
        return true;
    }
    long lineno() const { return lineno_; }

private:
    std::string buf_;
    size_t pos_ = 0;
    long lineno_ = 0;
};

bool slurp(const std::string& path, std::string* out) {
    FILE* f = std::fopen(path.c_str(), "rb");
    if (!f) return false;
    char chunk[1 << 16];
    size_t k;
    while ((k = std::fread(chunk, 1, sizeof(chunk), f)) > 0) out->append(chunk, k);
    std::fclose(f);
    return true;
}

// Header, comment, size-line and entry rules of read_matrix_market
// (mmio.hpp:23-84) and its "<path>:<line>: <what>" messages; the duplicate
// fold (csr_from_coo) runs afterwards on the GPU.
bool parse(const std::string& path, Parsed* P, std::string* msg) {
    std::string text;
    if (!slurp(path, &text)) {
        *msg = "cannot open " + path;
        return false;
    }
    auto fail = [&](long line, const std::string& what) {
        *msg = path + ":" + std::to_string(line) + ": " + what;
        return false;
    };
    LineReader lines(std::move(text));
    Cursor cur{};
    if (!lines.next(&cur)) return fail(1, "empty file");
    std::string tok[5];  // banner, object, format, field, symmetry ("" when absent)
    for (std::string& t : tok) cur.word(&t);
    if (tok[0] != "%%MatrixMarket" || tok[1] != "matrix" || tok[2] != "coordinate")
        return fail(1, "malformed MatrixMarket header");
    const std::string& field = tok[3];
    const std::string& symmetry = tok[4];
    const bool pattern = field == "pattern";
    if (!pattern && field != "real" && field != "integer")
        return fail(1, "unsupported field type '" + field + "'");
    const bool symmetric = symmetry == "symmetric";
    if (!symmetric && symmetry != "general") return fail(1, "unsupported symmetry '" + symmetry + "'");
    auto is_skipped = [](const Cursor& c) { return c.p == c.end || *c.p == '%'; };

    int64_t dims[3] = {0, 0, 0};  // m, n, declared entries
    while (lines.next(&cur)) {
        if (is_skipped(cur)) continue;
        // a failed extraction leaves the earlier fields read (m, n may be set)
        int64_t v[3] = {0, 0, 0};
        int k = 0;
        while (k < 3 && cur.integer(&v[k])) dims[k] = v[k], ++k;
        if (k < 3) return fail(lines.lineno(), "malformed size line");
        break;
    }
    const int64_t m = dims[0], n = dims[1], declared = dims[2];
    if (m <= 0 || n < 0) return fail(lines.lineno(), "invalid matrix dimensions");
    P->m = m;
    P->n = n;
    const size_t cap = static_cast<size_t>(std::max<int64_t>(declared, 0)) * (symmetric ? 2 : 1);
    P->rows.reserve(cap);
    P->cols.reserve(cap);
    P->vals.reserve(cap);
    int64_t seen = 0;
    while (lines.next(&cur)) {
        if (is_skipped(cur)) continue;
        int64_t r = 0, c = 0;
        if (!cur.integer(&r) || !cur.integer(&c)) return fail(lines.lineno(), "malformed entry");
        double v = 1.0;
        if (!pattern && !cur.real(&v)) return fail(lines.lineno(), "non-numeric value");
        if (r < 1 || r > m || c < 1 || c > n) return fail(lines.lineno(), "index out of declared bounds");
        const float fv = static_cast<float>(v);
        P->rows.push_back(r - 1);
        P->cols.push_back(c - 1);
        P->vals.push_back(fv);
        if (symmetric && r != c) {  // mirrored off-diagonal entry
            P->rows.push_back(c - 1);
            P->cols.push_back(r - 1);
            P->vals.push_back(fv);
        }
        ++seen;
    }
    if (seen != declared)
        return fail(lines.lineno(), "entry count " + std::to_string(seen) + " does not match declared " +
                                        std::to_string(declared));
    return true;
}

}  // namespace

extern "C" {

fmm_status fmm_read_matrix_market(const char* path, int device, int64_t* m, int64_t* n, int64_t* nnz,
                                  int64_t** row_ptr, int64_t** col_idx, float** values, char* err,
                                  size_t err_cap) {
    if (!path || !m || !n || !nnz || !row_ptr || !col_idx || !values) return FMM_E_INVAL;
    *row_ptr = nullptr;
    *col_idx = nullptr;
    *values = nullptr;
    Parsed P;
    std::string msg;
    if (!parse(path, &P, &msg)) {
        set_msg(err, err_cap, msg);
        return FMM_E_INVAL;
    }
    const int64_t cnt = static_cast<int64_t>(P.rows.size());
    int64_t* rp = static_cast<int64_t*>(std::malloc(sizeof(int64_t) * (P.m + 1)));
    int64_t* cl = static_cast<int64_t*>(std::malloc(sizeof(int64_t) * std::max<int64_t>(cnt, 1)));
    float* vl = static_cast<float*>(std::malloc(sizeof(float) * std::max<int64_t>(cnt, 1)));
    if (!rp || !cl || !vl) {
        std::free(rp);
        std::free(cl);
        std::free(vl);
        return FMM_E_OOM;
    }
    int64_t k = 0;
    const fmm_status st = fmm_csr_from_coo(device, P.m, P.n, cnt, P.rows.data(), P.cols.data(), P.vals.data(), rp,
                                           cl, vl, &k);
    if (st != FMM_OK) {
        std::free(rp);
        std::free(cl);
        std::free(vl);
        set_msg(err, err_cap, std::string("csr_from_coo on the device: ") + fmm_status_string(st));
        return st;
    }
    *m = P.m;
    *n = P.n;
    *nnz = k;
    *row_ptr = rp;
    *col_idx = cl;
    *values = vl;
    return FMM_OK;
}

fmm_status fmm_write_matrix_market(const char* path, int64_t m, int64_t n, const int64_t* row_ptr,
                                   const int64_t* col_idx, const float* values) {
    if (!path || m < 0 || !row_ptr) return FMM_E_INVAL;
    const int64_t nnz = row_ptr[m];
    if (nnz > 0 && (!col_idx || !values)) return FMM_E_INVAL;
    FILE* f = std::fopen(path, "w");
    if (!f) return FMM_E_INVAL;
    std::fprintf(f, "%%%%MatrixMarket matrix coordinate real general\n");
    std::fprintf(f, "%lld %lld %lld\n", static_cast<long long>(m), static_cast<long long>(n),
                 static_cast<long long>(nnz));
    // ostream precision(17) in the default float field prints like %.17g
    for (int64_t u = 0; u < m; ++u)
        for (int64_t p = row_ptr[u]; p < row_ptr[u + 1]; ++p)
            std::fprintf(f, "%lld %lld %.17g\n", static_cast<long long>(u + 1),
                         static_cast<long long>(col_idx[p] + 1), static_cast<double>(values[p]));
    const bool ok = std::ferror(f) == 0;
    return (std::fclose(f) == 0 && ok) ? FMM_OK : FMM_E_INVAL;
}

void fmm_free(void* p) { std::free(p); }

}  // extern "C"
