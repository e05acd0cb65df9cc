// serialize.cu -- ranking order and ranking CSV (serialize.py:14-21).
//
// Order: scores descending, ties by original id ascending -- the reference's
// np.lexsort((original_ids, -values)).  On the device: a stable radix sort
// by original id, then a stable radix sort by a descending float key (the
// IEEE bit pattern mapped to an order-preserving unsigned key; -0.0 is
// folded onto +0.0, which lexsort treats as equal).
//
// CSV: "vertex_original_id,score" then one row per vertex, written by the
// host like Python's csv.writer (\r\n line ends) with the score formatted as
// repr(float): the shortest round-trip digits (std::to_chars), in fixed
// notation for decimal exponents -4..15 (an integral value gets ".0") and in
// scientific notation otherwise (exponent sign and at least two digits).
#include <cub/cub.cuh>

#include <charconv>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "cubutil.cuh"
#include "internal.cuh"

namespace pr {

__global__ void k_rank_keys(const double *__restrict__ v, const int64_t *__restrict__ idx, int64_t n,
                            unsigned long long *__restrict__ key) {
    GRID_STRIDE(j, n) {
        double x = v[idx[j]];
        if (x == 0.0) x = 0.0;  // -0.0 == +0.0 for the comparison
        unsigned long long u = (unsigned long long)__double_as_longlong(x);
        u = (u >> 63) ? ~u : (u | 0x8000000000000000ull);  // ascending order key
        key[j] = ~u;                                        // descending
    }
}

__global__ void k_iota_i64(int64_t *__restrict__ out, int64_t n) { GRID_STRIDE(i, n) out[i] = i; }

int rank_order(Ctx &ctx, const double *h_values, const int64_t *h_ids, int64_t n, int64_t k, int64_t *h_order) {
    if (n <= 0 || k <= 0) return PR_OK;
    if (k > n) k = n;
    cudaStream_t st = ctx.stream;
    DevBuf v, ids, ids2, idx, idx2, key, key2;
    PR_TRY(ensure(v, 8 * n));
    PR_TRY(ensure(idx, 8 * n));
    PR_TRY(ensure(idx2, 8 * n));
    PR_TRY(ensure(key, 8 * n));
    PR_TRY(ensure(key2, 8 * n));
    PR_CUDA(cudaMemcpyAsync(v.ptr, h_values, 8 * n, cudaMemcpyHostToDevice, st));
    const unsigned grid = (unsigned)(ctx.sm_count * 8);
    k_iota_i64<<<grid, 256, 0, st>>>(idx.as<int64_t>(), n);
    if (h_ids) {
        // secondary key first (stable sorts): original id ascending
        PR_TRY(ensure(ids, 8 * n));
        PR_TRY(ensure(ids2, 8 * n));
        PR_CUDA(cudaMemcpyAsync(ids.ptr, h_ids, 8 * n, cudaMemcpyHostToDevice, st));
        PR_TRY(cub_run(ctx, [&](void *t, size_t &b) {
            return cub::DeviceRadixSort::SortPairs(t, b, ids.as<unsigned long long>(), ids2.as<unsigned long long>(),
                                                   idx.as<int64_t>(), idx2.as<int64_t>(), n, 0, 63, st);
        }));
        std::swap(idx.ptr, idx2.ptr);
        std::swap(idx.bytes, idx2.bytes);
    }
    k_rank_keys<<<grid, 256, 0, st>>>(v.as<double>(), idx.as<int64_t>(), n, key.as<unsigned long long>());
    PR_TRY(cub_run(ctx, [&](void *t, size_t &b) {
        return cub::DeviceRadixSort::SortPairs(t, b, key.as<unsigned long long>(), key2.as<unsigned long long>(),
                                               idx.as<int64_t>(), idx2.as<int64_t>(), n, 0, 64, st);
    }));
    PR_CUDA(cudaMemcpyAsync(h_order, idx2.ptr, 8 * k, cudaMemcpyDeviceToHost, st));
    PR_CUDA(cudaStreamSynchronize(st));
    return PR_OK;
}

// repr(float) of a finite double
static int py_repr(double x, char *out) {
    if (x == 0.0) {
        const char *z = std::signbit(x) ? "-0.0" : "0.0";
        std::strcpy(out, z);
        return (int)std::strlen(z);
    }
    char sci[64];
    auto r = std::to_chars(sci, sci + sizeof(sci), x, std::chars_format::scientific);
    *r.ptr = '\0';
    // sci = [-]d[.ddd]e[+-]XX
    const char *p = sci;
    std::string out_s;
    if (*p == '-') {
        out_s.push_back('-');
        ++p;
    }
    std::string digits;
    while (*p && *p != 'e') {
        if (*p != '.') digits.push_back(*p);
        ++p;
    }
    const int exp10 = std::atoi(p + 1);
    const int nd = (int)digits.size();
    if (exp10 < -4 || exp10 >= 16) {
        out_s.push_back(digits[0]);
        if (nd > 1) {
            out_s.push_back('.');
            out_s.append(digits, 1, std::string::npos);
        }
        char eb[16];
        std::snprintf(eb, sizeof(eb), "e%c%02d", exp10 < 0 ? '-' : '+', exp10 < 0 ? -exp10 : exp10);
        out_s.append(eb);
    } else if (exp10 < 0) {
        out_s.append("0.");
        out_s.append((size_t)(-exp10 - 1), '0');
        out_s.append(digits);
    } else {
        const int int_len = exp10 + 1;
        if (nd <= int_len) {
            out_s.append(digits);
            out_s.append((size_t)(int_len - nd), '0');
            out_s.append(".0");
        } else {
            out_s.append(digits, 0, int_len);
            out_s.push_back('.');
            out_s.append(digits, int_len, std::string::npos);
        }
    }
    std::memcpy(out, out_s.data(), out_s.size());
    out[out_s.size()] = '\0';
    return (int)out_s.size();
}

int format_score(double x, char *out) { return py_repr(x, out); }

int write_ranking_csv(Ctx &ctx, const double *values, const int64_t *ids, int64_t n, const char *path) {
    std::vector<int64_t> order((size_t)(n > 0 ? n : 1));
    PR_TRY(rank_order(ctx, values, ids, n, n, order.data()));
    FILE *fh = std::fopen(path, "wb");
    if (!fh) return fail(PR_ERR_ARG, std::string("cannot open ") + path);
    std::vector<char> buf;
    buf.reserve((size_t)(n > 0 ? n : 1) * 40 + 64);
    const char *head = "vertex_original_id,score\r\n";
    buf.insert(buf.end(), head, head + std::strlen(head));
    char line[96];
    for (int64_t j = 0; j < n; ++j) {
        const int64_t i = order[(size_t)j];
        const int64_t id = ids ? ids[i] : i;
        auto r = std::to_chars(line, line + 32, id);
        *r.ptr++ = ',';
        const int len = py_repr(values[i], r.ptr);
        char *e = r.ptr + len;
        *e++ = '\r';
        *e++ = '\n';
        buf.insert(buf.end(), line, e);
    }
    const size_t wrote = std::fwrite(buf.data(), 1, buf.size(), fh);
    const int closed = std::fclose(fh);
    if (wrote != buf.size() || closed != 0) return fail(PR_ERR_ARG, std::string("write failed: ") + path);
    return PR_OK;
}

}  // namespace pr
