// `fvlog run <program.dl> --facts DIR --out DIR [--device N] [--stats]
//  [--dump a,b]` — CLI compatible with the reference's `colog run`
// (P/tools/main.cpp:9-43): same options and output lines, evaluated on a GPU.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

#include "fvlog.h"

int main(int argc, char** argv) {
    if (argc < 3 || std::strcmp(argv[1], "run") != 0) {
        std::fprintf(stderr,
                     "usage: fvlog run <program> --facts DIR --out DIR [--device N] [--workers N] "
                     "[--stats] [--dump a,b]\n");
        return 2;
    }
    const char* program = argv[2];
    std::string facts, out_dir, dump;
    int device = 0, stats = 0;
    for (int i = 3; i < argc; ++i) {
        std::string a = argv[i];
        auto val = [&]() -> std::string {
            if (i + 1 >= argc) {
                std::fprintf(stderr, "missing value for %s\n", a.c_str());
                std::exit(2);
            }
            return argv[++i];
        };
        if (a == "--facts") facts = val();
        else if (a == "--out") out_dir = val();
        else if (a == "--device") device = std::atoi(val().c_str());
        else if (a == "--workers") (void)val();  // CPU worker count: no GPU analogue
        else if (a == "--stats") stats = 1;
        else if (a == "--dump") dump = val();
        else {
            std::fprintf(stderr, "unknown option %s\n", a.c_str());
            return 2;
        }
    }
    if (facts.empty() || out_dir.empty()) {
        std::fprintf(stderr, "--facts and --out are required\n");
        return 2;
    }
    char* out = nullptr;
    char* err = nullptr;
    const int rc = fv_run(device, program, facts.c_str(), out_dir.c_str(), stats, dump.c_str(), &out, &err);
    if (out) std::fputs(out, stdout);
    if (err) std::fputs(err, stderr);
    fv_free(out);
    fv_free(err);
    return rc;
}
