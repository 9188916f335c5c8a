// ocldec-b200: command-line front end over the C ABI (include/ocldec_b200.hpp).
//
// Same flags, output file and exit codes as the reference CLI
// (/root/reference/proj/tools/ocldec.cpp:81-177) for the options this path
// supports:
//   ocldec-b200 <input> [-o|--output FILE] [--kernel NAME] [--fold-local-size]
//               [--abi-map FILE] [--dump-cfg] [--dump-regions]
// The output is combined_source() written atomically (temp file + rename,
// ocldec.cpp:35-57) to FILE or <input stem>.cl (ocldec.cpp:59-66).
// Diagnostics go to stderr as "file:line: severity: message"; exit status is 1
// when no kernel was produced or any kernel failed, 0 otherwise.
// --abi-map FILE is parsed first; its diagnostics are printed against FILE and
// any error exits 1 before decompiling (ocldec.cpp:120-131).
// --devices 0,1,... shards the listing across GPUs (one host thread each).
// --dump-cfg / --dump-regions write <out stem>.<kernel>.cfg.dot and
// <out stem>.<kernel>.step<N>.dot next to the output (ocldec.cpp:68-77, 150-165).
#include <cstdio>
#include <cstring>
#include <fstream>
#include <iostream>
#include <sstream>
#include <string>

#include "../include/ocldec_b200.hpp"

namespace {

// The whole file as bytes; on failure err holds the reference CLI's message.
bool slurp(const std::string &path, std::string &out, std::string &err) {
    FILE *f = std::fopen(path.c_str(), "rb");
    if (!f) {
        err = "cannot open '" + path + "' for reading";
        return false;
    }
    out.clear();
    char chunk[1 << 16];
    for (size_t n; (n = std::fread(chunk, 1, sizeof chunk, f)) > 0;)
        out.append(chunk, n);
    std::fclose(f);
    return true;
}

// Temp file beside the target, then rename over it: a failed write never
// leaves a truncated output (the reference CLI's contract, ocldec.cpp:35-57).
bool replace_file(const std::string &path, const std::string &bytes, std::string &err) {
    const std::string part = path + ".tmp";
    FILE *f = std::fopen(part.c_str(), "wb");
    if (!f) {
        err = "cannot open '" + part + "' for writing";
        return false;
    }
    const bool wrote = std::fwrite(bytes.data(), 1, bytes.size(), f) == bytes.size();
    if (std::fclose(f) != 0 || !wrote) {
        err = "write to '" + part + "' failed";
        std::remove(part.c_str());
        return false;
    }
    if (std::rename(part.c_str(), path.c_str()) == 0)
        return true;
    err = "cannot rename '" + part + "' to '" + path + "'";
    std::remove(part.c_str());
    return false;
}

// The path without its extension: a '.' counts only inside the last path
// component (ocldec.cpp:59-77 names the output and dump files this way).
std::string strip_ext(const std::string &path) {
    const size_t cut = path.find_last_of('.');
    const size_t sep = path.find_last_of("/\\");
    const bool has_ext = cut != std::string::npos && (sep == std::string::npos || cut > sep);
    return has_ext ? path.substr(0, cut) : path;
}

std::string dump_stem(const std::string &output, const std::string &kernel) {
    return strip_ext(output) + "." + kernel;
}

std::string default_output(const std::string &input) { return strip_ext(input) + ".cl"; }

int usage(const char *argv0, int code) {
    std::fprintf(code ? stderr : stdout,
                 "Decompiles AMD GCN disassembly listings (CLRX syntax) to OpenCL C on the GPU\n"
                 "Usage: %s input [-o OUTPUT] [--kernel NAME] [--fold-local-size] [--abi-map FILE]\n"
                 "       [--dump-cfg] [--dump-regions] [--device N | --devices N,M,...]\n",
                 argv0);
    return code;
}

} // namespace

int main(int argc, char **argv) {
    std::string input, output, only, abi_path;
    ocldec_b200::DecompileOptions opts;
    for (int i = 1; i < argc; ++i) {
        std::string a = argv[i];
        if (a == "-h" || a == "--help")
            return usage(argv[0], 0);
        if (a == "--version") {
            std::printf("ocldec-b200 (C ABI %d)\n", OCLDEC_B200_ABI_VERSION);
            return 0;
        }
        if ((a == "-o" || a == "--output" || a == "--kernel" || a == "--device" || a == "--abi-map" ||
             a == "--devices") &&
            i + 1 < argc) {
            std::string v = argv[++i];
            if (a == "--abi-map")
                abi_path = v;
            else if (a == "--kernel")
                opts.only_kernel = v;
            else if (a == "--device")
                opts.device = std::atoi(v.c_str());
            else if (a == "--devices") // comma-separated ordinals: shard across them
                for (size_t p0 = 0; p0 <= v.size();) {
                    size_t p1 = v.find(',', p0);
                    if (p1 == std::string::npos)
                        p1 = v.size();
                    opts.devices.push_back(std::atoi(v.substr(p0, p1 - p0).c_str()));
                    p0 = p1 + 1;
                }
            else
                output = v;
            continue;
        }
        if (a == "--fold-local-size") {
            opts.fold_local_size = true;
            continue;
        }
        if (a == "--dump-cfg" || a == "--dump-regions") {
            (a == "--dump-cfg" ? opts.dump_cfg : opts.dump_regions) = true;
            continue;
        }
        if (!a.empty() && a[0] == '-')
            return usage(argv[0], 1);
        if (!input.empty())
            return usage(argv[0], 1);
        input = a;
    }
    if (input.empty())
        return usage(argv[0], 1);

    std::string err, listing;
    if (!slurp(input, listing, err)) {
        std::cerr << "ocldec-b200: error: " << err << "\n";
        return 1;
    }
    if (!abi_path.empty()) {
        if (!slurp(abi_path, opts.abi_map, err)) {
            std::cerr << "ocldec-b200: error: " << err << "\n";
            return 1;
        }
        bool bad = false;
        try {
            for (const auto &d : ocldec_b200::check_abi_map(opts.abi_map)) {
                std::cerr << d.render(abi_path) << "\n";
                bad = bad || d.severity == ocldec_b200::Diagnostic::Error;
            }
        } catch (const std::exception &e) {
            std::cerr << "ocldec-b200: error: " << e.what() << "\n";
            return 1;
        }
        if (bad)
            return 1;
    }
    ocldec_b200::DecompileResult result;
    try {
        result = ocldec_b200::decompile_listing(listing, opts);
    } catch (const std::exception &e) {
        std::cerr << "ocldec-b200: error: " << e.what() << "\n";
        return 1;
    }
    for (const auto &d : result.diagnostics)
        std::cerr << d.render(input) << "\n";
    if (result.kernels.empty()) {
        if (!result.has_errors())
            std::cerr << input << ":0: error: no kernels found\n";
        return 1;
    }
    bool any_failed = false;
    for (const auto &k : result.kernels)
        any_failed = any_failed || k.failed;
    if (output.empty())
        output = default_output(input);
    if (opts.dump_cfg || opts.dump_regions) {
        for (const auto &k : result.kernels) {
            const std::string stem = dump_stem(output, k.name);
            if (opts.dump_cfg && !k.cfg_dot.empty() && !replace_file(stem + ".cfg.dot", k.cfg_dot, err)) {
                std::cerr << "ocldec-b200: error: " << err << "\n";
                return 1;
            }
            for (size_t i = 0; i < k.region_dumps.size(); ++i)
                if (!replace_file(stem + ".step" + std::to_string(i) + ".dot", k.region_dumps[i], err)) {
                    std::cerr << "ocldec-b200: error: " << err << "\n";
                    return 1;
                }
        }
    }
    if (!replace_file(output, result.combined_source(), err)) {
        std::cerr << "ocldec-b200: error: " << err << "\n";
        return 1;
    }
    return any_failed ? 1 : 0;
}
