// TSV facts I/O and the batch runner: the host surface of P/src/io.cpp and
// P/src/runner.cpp (same file layout, mode detection, error texts and output
// line formats), driving the device engine.
#include "runner.h"

#include "tsv.h"

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <charconv>
#include <filesystem>
#include <fstream>
#include <sstream>

namespace fv {

namespace fs = std::filesystem;

namespace {

[[noreturn]] void io_fail(const fs::path& path, size_t line, const std::string& msg) {
    fail(FV_ERR_IO, path.string() + ":" + std::to_string(line) + ": " + msg);
}

bool parse_u32(std::string_view f, u32* out) {
    if (f.empty()) return false;
    u64 v = 0;
    auto [p, ec] = std::from_chars(f.data(), f.data() + f.size(), v);
    if (ec != std::errc{} || p != f.data() + f.size() || v > 0xffffffffull) return false;
    *out = static_cast<u32>(v);
    return true;
}

}  // namespace

LoadedFacts load_facts(const std::string& path_s, u32 arity, fe::Dictionary& dict) {
    const fs::path path(path_s);
    std::ifstream in(path, std::ios::binary);
    if (!in) fail(FV_ERR_IO, "cannot open facts file: " + path.string());
    LoadedFacts out;
    out.cols.resize(arity);
    std::string line;
    size_t line_no = 0;
    bool mode_known = false;
    std::vector<std::string_view> fields;
    while (std::getline(in, line)) {
        ++line_no;
        if (!line.empty() && line.back() == '\r') line.pop_back();
        if (line.empty()) continue;
        fields.clear();
        std::string_view sv(line);
        size_t start = 0;
        while (true) {
            const size_t tab = sv.find('\t', start);
            if (tab == std::string_view::npos) {
                fields.push_back(sv.substr(start));
                break;
            }
            fields.push_back(sv.substr(start, tab - start));
            start = tab + 1;
        }
        if (fields.size() != arity)
            io_fail(path, line_no, "expected " + std::to_string(arity) + " tab-separated fields, got " +
                                       std::to_string(fields.size()));
        if (!mode_known) {
            u32 tmp;
            out.dict_encoded = false;
            for (auto f : fields)
                if (!parse_u32(f, &tmp)) out.dict_encoded = true;
            mode_known = true;
        }
        for (u32 j = 0; j < arity; ++j) {
            u32 v;
            if (out.dict_encoded) {
                v = dict.encode(std::string(fields[j]));
            } else if (!parse_u32(fields[j], &v)) {
                io_fail(path, line_no, "field '" + std::string(fields[j]) +
                                           "' is not an unsigned 32-bit integer (file is in integer mode)");
            }
            out.cols[j].push_back(v);
        }
        ++out.rows;
    }
    return out;
}

std::string dump_text(const std::vector<u32>& rows, u32 arity, const fe::Dictionary* dict) {
    std::ostringstream os;
    const u64 n = arity ? rows.size() / arity : 0;
    if (dict) {
        std::vector<std::vector<std::string>> s(n);
        for (u64 i = 0; i < n; ++i)
            for (u32 j = 0; j < arity; ++j) s[i].push_back(dict->decode(rows[i * arity + j]));
        std::sort(s.begin(), s.end());
        for (auto& r : s) {
            for (u32 j = 0; j < arity; ++j) os << (j ? "\t" : "") << r[j];
            os << '\n';
        }
        return os.str();
    }
    // rows are already lexicographically sorted (FULL invariant)
    for (u64 i = 0; i < n; ++i) {
        for (u32 j = 0; j < arity; ++j) os << (j ? "\t" : "") << rows[i * arity + j];
        os << '\n';
    }
    return os.str();
}

int run(Ctx* c, const RunConfig& cfg, std::ostream& out, std::ostream& err) {
    // FVLOG_TRACE=1: host phase times on stderr (stdout keeps the reference's lines).
    const bool trace = std::getenv("FVLOG_TRACE") != nullptr;
    auto t_last = std::chrono::steady_clock::now();
    auto phase = [&](const char* what) {
        if (!trace) return;
        c->sync();
        const auto now = std::chrono::steady_clock::now();
        std::fprintf(stderr, "[fvlog] run %-12s %.3f ms\n", what,
                     std::chrono::duration<double, std::milli>(now - t_last).count());
        t_last = now;
    };
    try {
        std::ifstream pin(cfg.program_path, std::ios::binary);
        if (!pin) fail(FV_ERR_IO, "cannot open program file: " + cfg.program_path);
        std::ostringstream text;
        text << pin.rdbuf();

        fe::Program prog;
        try {
            prog = fe::parse(text.str());
        } catch (const fe::DiagnosticError& e) {
            err << cfg.program_path << ":" << e.what() << "\n";
            return 1;
        }
        auto diags = fe::validate(prog);
        if (!diags.empty()) {
            for (auto& d : diags) err << cfg.program_path << ":" << fe::format(d) << "\n";
            return 1;
        }
        fe::Dictionary dict;
        fe::resolve_strings(prog, dict);
        phase("parse");
        auto pfacts = fe::program_facts(prog);

        // Host-side staging of the EDB (excluded from the timed span, like
        // the reference's load_facts before evaluate()).
        std::vector<std::vector<u32>> storage;
        std::vector<FactsBlock> blocks;
        std::map<std::string, u32> arity;
        for (auto& d : prog.relations) arity[d.name] = d.arity;
        for (auto& [rel, rows] : pfacts) {
            const u32 a = arity[rel];
            const u64 n = rows.size() / a;
            FactsBlock b{rel, a, n, {}};
            for (u32 j = 0; j < a; ++j) {
                storage.emplace_back(n);
                for (u64 i = 0; i < n; ++i) storage.back()[i] = rows[i * a + j];
            }
            blocks.push_back(std::move(b));
        }
        // Facts files: integer-mode files are parsed on the device straight
        // into EDB columns (tsv.cu); dictionary-mode files (first non-empty
        // line not all integers) go through the host dictionary as before.
        std::vector<LoadedFacts> loaded;
        std::vector<std::string> loaded_rel;
        DeviceEdb file_edb;
        for (auto& d : prog.relations) {
            const fs::path path = fs::path(cfg.facts_dir) / (d.name + ".tsv");
            if (!fs::exists(path)) continue;
            std::ifstream fin(path, std::ios::binary | std::ios::ate);
            if (!fin) fail(FV_ERR_IO, "cannot open facts file: " + path.string());
            std::string bytes(static_cast<size_t>(fin.tellg()), '\0');
            fin.seekg(0);
            if (!bytes.empty() && !fin.read(bytes.data(), static_cast<std::streamsize>(bytes.size())))
                fail(FV_ERR_IO, "cannot read facts file: " + path.string());
            if (tsv_first_line_is_integer(bytes.data(), bytes.size(), d.arity)) {
                DevVersion v;
                v.n = tsv_parse_u32(c, bytes.data(), bytes.size(), d.arity, path.string(), v.cols);
                if (v.n) file_edb.rels.emplace(d.name, std::move(v));
                continue;
            }
            loaded.push_back(load_facts(path.string(), d.arity, dict));
            loaded_rel.push_back(d.name);
        }
        // Fix up column pointers only after all storage is allocated.
        size_t si = 0;
        for (auto& b : blocks)
            for (u32 j = 0; j < b.arity; ++j) b.cols.push_back(storage[si++].data());
        for (size_t k = 0; k < loaded.size(); ++k) {
            FactsBlock b{loaded_rel[k], arity[loaded_rel[k]], loaded[k].rows, {}};
            for (auto& col : loaded[k].cols) b.cols.push_back(col.data());
            blocks.push_back(std::move(b));
        }

        phase("load facts");
        auto plans = fe::compile(prog);
        const auto decls = fe::declarations(prog);
        check_plans(decls, plans);
        // total_ms spans the host-fact upload too, like fv_evaluate and the
        // reference's evaluate(), which seeds from host rows
        // (P/src/runner.cpp:58-61); facts parsed on the device are already
        // resident (their parse is the "load facts" phase, as the
        // reference's TSV load is).
        const auto t_up = std::chrono::steady_clock::now();
        DeviceEdb host_edb = upload_facts(c, decls, blocks);
        c->sync();
        const double upload_ms =
            std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_up).count();
        auto st = evaluate_device(c, decls, plans, {&host_edb, &file_edb});
        st->elapsed_ms += upload_ms;
        phase("evaluate");

        if (cfg.print_stats)
            for (auto& s : st->stats)
                out << "iter=" << s.iteration << " rel=" << s.relation << " delta=" << s.delta_rows
                    << " ms=" << s.elapsed_ms << "\n";
        for (auto& [name, rel] : st->relations) out << "rel=" << name << " rows=" << rel->rows() << "\n";
        out << "iterations=" << st->iterations << " total_ms=" << st->elapsed_ms << " workers=1\n";

        if (!cfg.dump_relations.empty()) {
            fs::create_directories(cfg.out_dir);
            for (auto& name : cfg.dump_relations) {
                auto it = st->relations.find(name);
                if (it == st->relations.end()) {
                    err << "unknown relation in --dump: " << name << "\n";
                    return 1;
                }
                std::ofstream o(fs::path(cfg.out_dir) / (name + ".tsv"), std::ios::binary);
                if (!o) fail(FV_ERR_IO, "cannot open output file: " + (fs::path(cfg.out_dir) / (name + ".tsv")).string());
                // Quirk kept (P/src/runner.cpp:83): a non-empty dictionary
                // decodes every dumped relation (host path); otherwise the
                // sorted rows are formatted on the device.
                if (dict.empty())
                    o << dump_sorted_text(*st, name);
                else
                    o << dump_text(dump_sorted(*st, name), it->second->arity, &dict);
                phase("dump");
            }
        }
        return 0;
    } catch (const std::exception& e) {
        err << "error: " << e.what() << "\n";
        return 1;
    }
}

}  // namespace fv
