// Integer-mode TSV facts parsing and sorted-dump formatting on the device
// (the data formats either side of the path).
//
// Parse (P/src/io.cpp:44-88, integer mode): lines split on '\n', one trailing
// '\r' stripped, empty lines skipped, fields split on '\t', every field
// std::from_chars-decimal (digits only, any number of leading zeros) and
// <= 2^32 - 1; the field count must equal the arity. Pipeline: one look-back
// compaction finds the line ends, one thread per line parses its fields into
// a staging row, a second compaction keeps the non-empty lines in file order
// and writes the SoA columns the engine consumes directly (no host columns).
// The first bad line (lowest line number, like the reference's sequential
// loop) is re-parsed on the host to build the reference's exact message.
//
// Format (P/src/io.cpp:90-117, no dictionary): one compaction pass computes
// each row's text length, scans it, and writes the row's digits at its offset
// ("v0\tv1\n") — the text is produced in one read of the columns.
#include <string>
#include <vector>

#include "prim.cuh"
#include "tsv.h"

namespace fv {

namespace {

struct NewlineOp {
    const char* bytes;
    u64* pos;
    __device__ u64 value(u64 i) const { return bytes[i] == '\n' ? 1 : 0; }
    __device__ void emit(u64 i, u64 p, u64 v) const {
        if (v) pos[p] = i;
    }
};

enum : u8 { kLineEmpty = 0, kLineOk = 1, kLineBad = 2 };

__global__ void parse_lines_kernel(const char* __restrict__ bytes, u64 nbytes, const u64* __restrict__ nl,
                                   u64 n_nl, u64 lines, u32 arity, u32* __restrict__ vals,
                                   u8* __restrict__ status, unsigned long long* first_bad) {
    for (u64 l = u64(blockIdx.x) * blockDim.x + threadIdx.x; l < lines; l += u64(gridDim.x) * blockDim.x) {
        const u64 b = l == 0 ? 0 : nl[l - 1] + 1;
        u64 e = l < n_nl ? nl[l] : nbytes;
        if (e > b && bytes[e - 1] == '\r') --e;
        if (e == b) {
            status[l] = kLineEmpty;
            continue;
        }
        u32 field = 0;
        u64 v = 0;
        bool digits = false, ok = true;
        for (u64 i = b; i <= e; ++i) {
            const char ch = i < e ? bytes[i] : '\t';  // end of line closes the last field
            if (ch == '\t') {
                if (!digits || v > 0xffffffffull) ok = false;
                if (ok && field < arity) vals[l * arity + field] = static_cast<u32>(v);
                ++field;
                v = 0;
                digits = false;
            } else if (ch >= '0' && ch <= '9') {
                if (v <= 0xffffffffull) v = v * 10 + static_cast<u64>(ch - '0');  // saturates past u32
                digits = true;
            } else {
                ok = false;
            }
        }
        if (field != arity) ok = false;
        status[l] = ok ? kLineOk : kLineBad;
        if (!ok) atomicMin(first_bad, static_cast<unsigned long long>(l));
    }
}

struct KeepLinesOp {
    const u8* status;
    const u32* vals;
    u32 arity;
    u32* const* cols;
    __device__ u64 value(u64 l) const { return status[l] == kLineOk ? 1 : 0; }
    __device__ void emit(u64 l, u64 p, u64 v) const {
        if (!v) return;
        for (u32 j = 0; j < arity; ++j) cols[j][p] = vals[l * arity + j];
    }
};

__device__ __forceinline__ u32 dec_digits(u32 v) {
    u32 d = 1;
    while (v >= 10) {
        v /= 10;
        ++d;
    }
    return d;
}

struct FormatOp {
    const u32* const* cols;
    u32 arity;
    char* out;
    __device__ u64 value(u64 i) const {
        u64 len = arity;  // arity - 1 tabs + newline
        for (u32 j = 0; j < arity; ++j) len += dec_digits(cols[j][i]);
        return len;
    }
    __device__ void emit(u64 i, u64 p, u64) const {
        char* o = out + p;
        for (u32 j = 0; j < arity; ++j) {
            u32 v = cols[j][i];
            const u32 d = dec_digits(v);
            for (u32 k = d; k-- > 0;) {
                o[k] = static_cast<char>('0' + v % 10);
                v /= 10;
            }
            o += d;
            *o++ = j + 1 < arity ? '\t' : '\n';
        }
    }
};

// Reference message for a bad line (P/src/io.cpp:64-80), from its text.
std::string bad_line_message(const std::string& path, u64 line_no, std::string line, u32 arity) {
    if (!line.empty() && line.back() == '\r') line.pop_back();
    std::vector<std::string> fields;
    size_t start = 0;
    for (;;) {
        const size_t tab = line.find('\t', start);
        if (tab == std::string::npos) {
            fields.push_back(line.substr(start));
            break;
        }
        fields.push_back(line.substr(start, tab - start));
        start = tab + 1;
    }
    const std::string where = path + ":" + std::to_string(line_no) + ": ";
    if (fields.size() != arity)
        return where + "expected " + std::to_string(arity) + " tab-separated fields, got " +
               std::to_string(fields.size());
    for (auto& f : fields) {
        bool ok = !f.empty();
        u64 v = 0;
        for (char ch : f) {
            if (ch < '0' || ch > '9') ok = false;
            else if (v <= 0xffffffffull) v = v * 10 + static_cast<u64>(ch - '0');
        }
        if (!ok || v > 0xffffffffull)
            return where + "field '" + f + "' is not an unsigned 32-bit integer (file is in integer mode)";
    }
    return where + "malformed line";
}

}  // namespace

bool tsv_first_line_is_integer(const char* bytes, u64 n, u32 arity) {
    u64 b = 0;
    while (b < n) {
        u64 e = b;
        while (e < n && bytes[e] != '\n') ++e;
        u64 end = e;
        if (end > b && bytes[end - 1] == '\r') --end;
        if (end > b) {
            u32 field = 0;
            bool digits = false;
            u64 v = 0;
            for (u64 i = b; i <= end; ++i) {
                const char ch = i < end ? bytes[i] : '\t';
                if (ch == '\t') {
                    if (!digits || v > 0xffffffffull) return false;
                    ++field;
                    v = 0;
                    digits = false;
                } else if (ch >= '0' && ch <= '9') {
                    if (v <= 0xffffffffull) v = v * 10 + static_cast<u64>(ch - '0');
                    digits = true;
                } else {
                    return false;
                }
            }
            (void)field;  // a field-count mismatch is reported by the parser
            return true;
        }
        b = e + 1;
    }
    return true;  // no non-empty line: nothing to decide (no rows)
}

u64 tsv_parse_u32(Ctx* c, const char* host_bytes, u64 nbytes, u32 arity, const std::string& path,
                  std::vector<DBuf<u32>>& cols) {
    if (arity == 0 || arity > FV_MAX_ARITY) fail(FV_ERR_ARITY, "tsv_parse: unsupported arity");
    cols.clear();
    if (nbytes == 0) {
        for (u32 j = 0; j < arity; ++j) cols.emplace_back(c, 0);
        return 0;
    }
    DBuf<char> bytes(c, nbytes);
    bytes.upload(host_bytes, nbytes);
    DBuf<u64> nl(c, nbytes);  // upper bound: every byte a newline
    u64* d_nnl = c->d_scalars + 30;
    {
        ProfScope prof(c, "tsv_lines", double(nbytes));
        tile_scan(c, NewlineOp{bytes.get(), nl.get()}, nbytes, d_nnl);
    }
    u64 n_nl = 0;
    c->read_scalars(d_nnl, &n_nl, 1);
    const u64 lines = n_nl + (host_bytes[nbytes - 1] != '\n' ? 1 : 0);
    DBuf<u32> vals(c, lines * arity);
    DBuf<u8> status(c, lines);
    u64* d_bad = c->d_scalars + 31;
    FV_CUDA(cudaMemsetAsync(d_bad, 0xff, sizeof(u64), c->stream));
    {
        ProfScope prof(c, "tsv_parse", double(nbytes) + double(lines) * (1.0 + 4.0 * arity));
        const u64 want = ceil_div(lines, 256);
        const unsigned grid = static_cast<unsigned>(want < u64(kNumSMs) * 32 ? (want ? want : 1) : u64(kNumSMs) * 32);
        parse_lines_kernel<<<grid, 256, 0, c->stream>>>(bytes.get(), nbytes, nl.get(), n_nl, lines, arity,
                                                        vals.get(), status.get(),
                                                        reinterpret_cast<unsigned long long*>(d_bad));
        FV_CUDA(cudaGetLastError());
        c->count_launch();
    }
    u64 bad = 0;
    c->read_scalars(d_bad, &bad, 1);
    if (bad != ~u64(0)) {
        u64 range[2] = {0, nbytes};
        if (bad > 0) FV_CUDA(cudaMemcpy(&range[0], nl.get() + bad - 1, 8, cudaMemcpyDeviceToHost));
        if (bad < n_nl) FV_CUDA(cudaMemcpy(&range[1], nl.get() + bad, 8, cudaMemcpyDeviceToHost));
        const u64 b = bad > 0 ? range[0] + 1 : 0;
        fail(FV_ERR_IO, bad_line_message(path, bad + 1, std::string(host_bytes + b, host_bytes + range[1]), arity));
    }
    std::vector<u32*> cp;
    for (u32 j = 0; j < arity; ++j) {
        cols.emplace_back(c, lines);
        cp.push_back(cols.back().get());
    }
    DBuf<u32*> d_cols(c, arity);
    d_cols.upload(cp.data(), arity);
    u64* d_rows = c->d_scalars + 32;
    tile_scan(c, KeepLinesOp{status.get(), vals.get(), arity, d_cols.get()}, lines, d_rows);
    u64 rows = 0;
    c->read_scalars(d_rows, &rows, 1);
    return rows;
}

std::string tsv_format_u32(Ctx* c, const std::vector<const u32*>& cols, u64 n, u32 arity) {
    if (n == 0) return std::string();
    if (arity == 0 || arity > FV_MAX_ARITY) fail(FV_ERR_ARITY, "tsv_format: unsupported arity");
    // Size first (<= 11 bytes per value), then one fused length-scan + write.
    DBuf<char> text(c, n * 11 * arity);
    DBuf<const u32*> d_cols(c, arity);
    d_cols.upload(cols.data(), arity);
    u64* d_len = c->d_scalars + 33;
    {
        ProfScope prof(c, "tsv_format", double(n) * 4.0 * arity);
        tile_scan(c, FormatOp{d_cols.get(), arity, text.get()}, n, d_len);
    }
    u64 len = 0;
    c->read_scalars(d_len, &len, 1);
    c->prof_add_bytes("tsv_format", double(len));
    std::string out(len, '\0');
    text.download(out.data(), len);
    return out;
}

}  // namespace fv
