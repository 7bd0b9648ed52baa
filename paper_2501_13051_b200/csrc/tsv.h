// Device TSV facts parsing / sorted-dump formatting (integer mode; see tsv.cu).
#pragma once

#include <string>
#include <vector>

#include "fv_common.cuh"

namespace fv {

// Mode decision of load_facts (P/src/io.cpp:67-72): true when the first
// non-empty line's fields all parse as u32 (integer mode) or the file has no
// non-empty line; false means dictionary mode (host path).
bool tsv_first_line_is_integer(const char* bytes, u64 n, u32 arity);

// Parse an integer-mode facts file image into device SoA columns (file
// order, duplicates kept). Throws FV_ERR_IO with the reference's message
// ("<path>:<line>: ...") for the first bad line. Returns the row count.
u64 tsv_parse_u32(Ctx* c, const char* host_bytes, u64 nbytes, u32 arity, const std::string& path,
                  std::vector<DBuf<u32>>& cols);

// dump_relation text of n rows given as device columns (already in the
// desired order): "v0\tv1...\n" per row.
std::string tsv_format_u32(Ctx* c, const std::vector<const u32*>& cols, u64 n, u32 arity);

}  // namespace fv
