// colog-on-fvlog: the reference-side binding of INTEGRATION.md §2, compiled.
//
// These four translation units (column.cpp, relation.cpp, kernels.cpp,
// engine.cpp) define every function the reference's hot-path headers declare
// (P/include/colog/{column,relation,kernels,engine}.hpp) on top of the fvlog
// C ABI (include/fvlog.h), so a program built against the UNMODIFIED
// reference headers links against libfvlog.so instead of the reference's
// P/src/{column,relation,kernels,engine}.cpp and runs its hot path on the
// B200. Everything else the reference links (parser, compiler, io, runner,
// oracle) is its own code, unchanged.
//
// The host objects of the reference API (Column, Version, IdPairSet, ...)
// stay host objects — that is the interface — and every data-parallel step
// behind them is one or more fvlog calls on one process-wide context
// (device FVLOG_DEVICE, default 0). Status codes map back to the reference's
// exception types (fvlog.h header comment).
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "colog/relation.hpp"
#include "colog/types.hpp"
#include "fvlog.h"

namespace colog::fvshim {

// The process-wide fvlog context (created on first use).
fv_ctx* ctx();

// FV_OK or throw the reference's exception for the status.
void check(fv_status s, const char* what);

// Owning handles.
struct ColumnH {
    fv_column* p = nullptr;
    ColumnH() = default;
    explicit ColumnH(const std::vector<Value>& raw);
    ColumnH(const ColumnH&) = delete;
    ColumnH& operator=(const ColumnH&) = delete;
    ~ColumnH() { fv_column_free(p); }
};

struct VersionH {
    fv_version* p = nullptr;
    VersionH() = default;
    explicit VersionH(const Version& v);  // upload a host Version's raw columns
    VersionH(const VersionH&) = delete;
    VersionH& operator=(const VersionH&) = delete;
    ~VersionH() { fv_version_free(p); }
};

struct ArrayH {
    fv_array* p = nullptr;
    ArrayH() = default;
    ArrayH(const ArrayH&) = delete;
    ArrayH& operator=(const ArrayH&) = delete;
    ~ArrayH() { fv_array_free(p); }
    template <typename T>
    std::vector<T> read() const {
        std::vector<T> out(p ? fv_array_size(p) : 0);
        if (!out.empty()) check(fv_array_read(p, out.data()), "fv_array_read");
        return out;
    }
};

// Raw columns of a device version (host copies).
std::vector<std::vector<Value>> download_columns(const fv_version* v);
// A host Version over the device version's rows (indexes built on device).
Version download(const fv_version* v);

}  // namespace colog::fvshim
