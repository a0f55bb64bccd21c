// fmm_mmio.cpp — MatrixMarket ingestion (mmio.hpp).
//
// fmm_read_matrix_market restates read_matrix_market (mmio.hpp:23-84): the
// header, comment, size-line and entry rules and their error messages
// ("<path>:<line>: <what>") on the host, then the duplicate fold and storage
// order of csr_from_coo on the GPU (fmm_csr_from_coo). fmm_write_matrix_market
// restates write_matrix_market (mmio.hpp:87-99): coordinate real general,
// 1-based, values printed with 17 significant digits.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <sstream>
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

// mmio.hpp:23-84 up to (not including) the csr_from_coo fold.
bool parse(const std::string& path, Parsed* P, std::string* msg) {
    std::ifstream in(path);
    if (!in) {
        *msg = "cannot open " + path;
        return false;
    }
    auto fail = [&](long line, const std::string& what) {
        *msg = path + ":" + std::to_string(line) + ": " + what;
        return false;
    };
    std::string line;
    long lineno = 0;
    if (!std::getline(in, line)) return fail(1, "empty file");
    ++lineno;
    std::istringstream hdr(line);
    std::string banner, object, format, field, symmetry;
    hdr >> banner >> object >> format >> field >> symmetry;
    if (banner != "%%MatrixMarket" || object != "matrix" || format != "coordinate")
        return fail(1, "malformed MatrixMarket header");
    if (field != "real" && field != "pattern" && field != "integer")
        return fail(1, "unsupported field type '" + field + "'");
    if (symmetry != "general" && symmetry != "symmetric")
        return fail(1, "unsupported symmetry '" + symmetry + "'");
    const bool pattern = field == "pattern";
    const bool symmetric = symmetry == "symmetric";
    int64_t m = 0, n = 0, declared = 0;
    while (std::getline(in, line)) {
        ++lineno;
        if (line.empty() || line[0] == '%') continue;
        std::istringstream sz(line);
        if (!(sz >> m >> n >> declared)) return fail(lineno, "malformed size line");
        break;
    }
    if (m <= 0 || n < 0) return fail(lineno, "invalid matrix dimensions");
    P->m = m;
    P->n = n;
    const size_t reserve = static_cast<size_t>(std::max<int64_t>(declared, 0)) * (symmetric ? 2 : 1);
    P->rows.reserve(reserve);
    P->cols.reserve(reserve);
    P->vals.reserve(reserve);
    int64_t seen = 0;
    while (std::getline(in, line)) {
        ++lineno;
        if (line.empty() || line[0] == '%') continue;
        std::istringstream es(line);
        int64_t r, c;
        if (!(es >> r >> c)) return fail(lineno, "malformed entry");
        double v = 1.0;
        if (!pattern && !(es >> v)) return fail(lineno, "non-numeric value");
        if (r < 1 || r > m || c < 1 || c > n) return fail(lineno, "index out of declared bounds");
        P->rows.push_back(r - 1);
        P->cols.push_back(c - 1);
        P->vals.push_back(static_cast<float>(v));
        if (symmetric && r != c) {
            P->rows.push_back(c - 1);
            P->cols.push_back(r - 1);
            P->vals.push_back(static_cast<float>(v));
        }
        ++seen;
    }
    if (seen != declared)
        return fail(lineno, "entry count " + std::to_string(seen) + " does not match declared " +
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
