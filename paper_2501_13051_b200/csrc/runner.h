// TSV I/O + batch runner (P/include/colog/io.hpp, P/include/colog/runner.hpp).
#pragma once

#include <ostream>
#include <string>
#include <vector>

#include "engine.h"
#include "frontend.h"

namespace fv {

struct LoadedFacts {
    std::vector<std::vector<u32>> cols;  // SoA
    u64 rows = 0;
    bool dict_encoded = false;
};

// load_facts (P/src/io.cpp:44-88): integer vs dictionary mode decided by the
// first non-empty line.
LoadedFacts load_facts(const std::string& path, u32 arity, fe::Dictionary& dict);
// dump_relation text (P/src/io.cpp:90-117) for lexicographically sorted rows.
std::string dump_text(const std::vector<u32>& rows_sorted, u32 arity, const fe::Dictionary* dict);

struct RunConfig {
    std::string program_path, facts_dir, out_dir;
    bool print_stats = false;
    std::vector<std::string> dump_relations;
};

int run(Ctx* c, const RunConfig& cfg, std::ostream& out, std::ostream& err);

}  // namespace fv
