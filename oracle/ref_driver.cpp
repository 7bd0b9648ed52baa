// TEST INFRASTRUCTURE — the CPU reference arm / checker, never the product.
//
// Command-line driver for the UNMODIFIED reference engine compiled from
// /root/reference/proj/src/*.cpp (see oracle/Makefile). It replaces the
// reference's CLI11 front end (P/tools/main.cpp:9-43) with plain argv parsing
// and calls colog::run (P/src/runner.cpp:26-92), so its stdout carries the
// reference's own line formats:
//   iter=<k> rel=<r> delta=<n> ms=<t>        (with --stats)
//   rel=<r> rows=<n>
//   iterations=<k> total_ms=<t> workers=<w>
//
// usage: colog_ref run <program.dl> --facts DIR --out DIR [--workers N]
//                      [--stats] [--dump a,b,...]
#include <cstdlib>
#include <cstring>
#include <iostream>
#include <string>

#include "colog/runner.hpp"

int main(int argc, char** argv) {
    if (argc < 3 || std::strcmp(argv[1], "run") != 0) {
        std::cerr << "usage: colog_ref run <program> --facts DIR --out DIR [--workers N] "
                     "[--stats] [--dump a,b]\n";
        return 2;
    }
    colog::RunConfig config;
    config.program_path = argv[2];
    std::string dump_list;
    for (int i = 3; i < argc; ++i) {
        std::string a = argv[i];
        auto need = [&](const char* what) -> std::string {
            if (i + 1 >= argc) {
                std::cerr << "missing value for " << what << "\n";
                std::exit(2);
            }
            return argv[++i];
        };
        if (a == "--facts") config.facts_dir = need("--facts");
        else if (a == "--out") config.out_dir = need("--out");
        else if (a == "--workers") config.workers = static_cast<unsigned>(std::stoul(need("--workers")));
        else if (a == "--stats") config.print_stats = true;
        else if (a == "--dump") dump_list = need("--dump");
        else {
            std::cerr << "unknown option " << a << "\n";
            return 2;
        }
    }
    std::size_t start = 0;
    while (!dump_list.empty() && start <= dump_list.size()) {
        std::size_t comma = dump_list.find(',', start);
        if (comma == std::string::npos) comma = dump_list.size();
        if (comma > start) config.dump_relations.push_back(dump_list.substr(start, comma - start));
        start = comma + 1;
    }
    return colog::run(config, std::cout, std::cerr);
}
