// ref_tool — thin driver over the UNMODIFIED reference library (satcc_core,
// compiled from /root/reference/proj/src by oracle/Makefile into oracle/_ref/).
//
// TEST INFRASTRUCTURE ONLY.  This binary is the parity checker's ground truth:
// it never sits on the product path.  It exposes two reference entry points
// that the reference's own CLI (proj/tools/satcc_main.cpp) cannot be built
// for here (CLI11 is absent):
//
//   ref_tool opt  <variant> <in.c> <out.c> <metrics.json> [ilp|greedy] [extract_s]
//       optimize_source (proj/include/satcc/pipeline.hpp:64-66) with the CLI's
//       default limits (proj/tools/satcc_main.cpp:37-53); metrics in the
//       satcc-metrics-v1 shape of metrics_json (satcc_main.cpp:89-110).
//
//   ref_tool eval <in.c> <function> <env_in.bin> <env_out.bin>
//       eval_region (proj/include/satcc/interp.hpp:72-74) over the WHOLE body
//       of <function> (not just one anchor iteration as diff_test does,
//       proj/src/oracle.cpp:73-74), with the environment read from / written
//       to the ACSENV1 binary format (oracle/envio.py documents it).
//
//   ref_tool regions <in.c>
//       find_regions (proj/src/ast.cpp:390-398): "<index> <function> <loopvars…>"
//       one line per region — the kernel-registry keys.

#include <cstdint>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <iostream>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "satcc/diag.hpp"
#include "satcc/interp.hpp"
#include "satcc/parser.hpp"
#include "satcc/pipeline.hpp"

using namespace satcc;

namespace {

std::string read_file(const std::string& path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw std::runtime_error("cannot open " + path);
    std::ostringstream ss;
    ss << in.rdbuf();
    return ss.str();
}

std::string json_str(const std::string& s) {
    std::string o = "\"";
    for (char c : s) {
        switch (c) {
            case '"': o += "\\\""; break;
            case '\\': o += "\\\\"; break;
            case '\n': o += "\\n"; break;
            case '\t': o += "\\t"; break;
            default:
                if (static_cast<unsigned char>(c) < 0x20) {
                    char b[8];
                    std::snprintf(b, sizeof b, "\\u%04x", c);
                    o += b;
                } else {
                    o += c;
                }
        }
    }
    return o + "\"";
}

int cmd_opt(int argc, char** argv) {
    if (argc < 6) throw std::runtime_error("usage: opt <variant> <in.c> <out.c> <metrics.json> [ilp|greedy] [extract_s]");
    VariantConfig v = VariantConfig::from_name(argv[2]);
    PipelineLimits lim;  // CLI defaults: 10000 nodes, 10 s, 10 iters, ilp, 30 s
    if (argc > 6) lim.method = std::string(argv[6]) == "greedy" ? ExtractMethod::Greedy : ExtractMethod::Ilp;
    if (argc > 7) lim.extract.max_time = std::stod(argv[7]);
    std::string src = read_file(argv[3]);
    auto [text, fm] = optimize_source(src, argv[3], v, lim);
    {
        std::ofstream o(argv[4], std::ios::binary);
        o << text;
    }
    std::ofstream j(argv[5], std::ios::binary);
    j << "{\n  \"schema\": \"satcc-metrics-v1\",\n  \"variant\": " << json_str(fm.variant)
      << ",\n  \"regions\": [";
    for (size_t i = 0; i < fm.regions.size(); ++i) {
        const RegionMetrics& r = fm.regions[i];
        j << (i ? "," : "") << "\n    {\"region\": " << r.region_index
          << ", \"function\": " << json_str(r.function) << ", \"ssa_ms\": " << r.ssa_ms
          << ", \"sat_ms\": " << r.sat_ms << ", \"extract_ms\": " << r.extract_ms
          << ", \"nodes_final\": " << r.nodes_final << ", \"stop_reason\": " << json_str(r.stop_reason)
          << ", \"objective_before\": " << r.objective_before
          << ", \"objective_after\": " << r.objective_after
          << ", \"static_loads_before\": " << r.static_loads_before
          << ", \"static_loads_after\": " << r.static_loads_after
          << ", \"static_stores\": " << r.static_stores << ", \"fma_count\": " << r.fma_count
          << ", \"method\": " << json_str(r.method)
          << ", \"timed_out\": " << (r.timed_out ? "true" : "false")
          << ", \"error\": " << json_str(r.error) << "}";
    }
    j << "\n  ]\n}\n";
    return 0;
}

// ---- ACSENV1 -------------------------------------------------------------

template <class T>
T rd(std::istream& in) {
    T v{};
    in.read(reinterpret_cast<char*>(&v), sizeof v);
    if (!in) throw std::runtime_error("truncated env file");
    return v;
}
template <class T>
void wr(std::ostream& o, T v) {
    o.write(reinterpret_cast<const char*>(&v), sizeof v);
}
std::string rd_name(std::istream& in) {
    uint32_t n = rd<uint32_t>(in);
    std::string s(n, '\0');
    in.read(s.data(), n);
    return s;
}
void wr_name(std::ostream& o, const std::string& s) {
    wr<uint32_t>(o, static_cast<uint32_t>(s.size()));
    o.write(s.data(), static_cast<std::streamsize>(s.size()));
}

Environment read_env(const std::string& path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw std::runtime_error("cannot open " + path);
    char magic[8];
    in.read(magic, 8);
    if (std::memcmp(magic, "ACSENV1", 8) != 0) throw std::runtime_error("bad env magic");
    Environment env;
    uint32_t ns = rd<uint32_t>(in);
    for (uint32_t i = 0; i < ns; ++i) {
        std::string name = rd_name(in);
        uint8_t t = rd<uint8_t>(in);
        if (t == 0)
            env.scalars[name] = Scalar::of_int(rd<int64_t>(in));
        else
            env.scalars[name] = Scalar::of_double(rd<double>(in));
    }
    uint32_t na = rd<uint32_t>(in);
    for (uint32_t i = 0; i < na; ++i) {
        std::string name = rd_name(in);
        ArrayBuf buf;
        buf.type = rd<uint8_t>(in) == 0 ? Ty::Int : Ty::Double;
        uint32_t nd = rd<uint32_t>(in);
        for (uint32_t d = 0; d < nd; ++d) buf.dims.push_back(rd<int64_t>(in));
        size_t n = buf.size();
        if (buf.type == Ty::Int) {
            buf.iv.resize(n);
            in.read(reinterpret_cast<char*>(buf.iv.data()), static_cast<std::streamsize>(n * 8));
        } else {
            buf.dv.resize(n);
            in.read(reinterpret_cast<char*>(buf.dv.data()), static_cast<std::streamsize>(n * 8));
        }
        if (!in) throw std::runtime_error("truncated array " + name);
        env.arrays[name] = std::move(buf);
    }
    return env;
}

void write_env(const std::string& path, const Environment& env) {
    std::ofstream o(path, std::ios::binary);
    o.write("ACSENV1", 8);
    wr<uint32_t>(o, static_cast<uint32_t>(env.scalars.size()));
    for (auto& [name, s] : env.scalars) {
        wr_name(o, name);
        wr<uint8_t>(o, s.type == Ty::Int ? 0 : 1);
        if (s.type == Ty::Int)
            wr<int64_t>(o, s.i);
        else
            wr<double>(o, s.d);
    }
    wr<uint32_t>(o, static_cast<uint32_t>(env.arrays.size()));
    for (auto& [name, b] : env.arrays) {
        wr_name(o, name);
        wr<uint8_t>(o, b.type == Ty::Int ? 0 : 1);
        wr<uint32_t>(o, static_cast<uint32_t>(b.dims.size()));
        for (long long d : b.dims) wr<int64_t>(o, d);
        if (b.type == Ty::Int)
            o.write(reinterpret_cast<const char*>(b.iv.data()), static_cast<std::streamsize>(b.iv.size() * 8));
        else
            o.write(reinterpret_cast<const char*>(b.dv.data()), static_cast<std::streamsize>(b.dv.size() * 8));
    }
}

const Function& find_fn(const KernelModule& m, const std::string& name) {
    for (auto& it : m.items)
        if (it.kind == TopItem::Kind::Func && it.fn.name == name) return it.fn;
    throw std::runtime_error("no function " + name);
}

int cmd_eval(int argc, char** argv) {
    if (argc < 6) throw std::runtime_error("usage: eval <in.c> <function> <env_in> <env_out>");
    std::string src = read_file(argv[2]);
    KernelModule m = parse(src, argv[2]);
    const Function& fn = find_fn(m, argv[3]);
    Environment env = read_env(argv[4]);
    Environment out = eval_region(*fn.body, std::move(env));
    write_env(argv[5], out);
    return 0;
}

int cmd_regions(int argc, char** argv) {
    if (argc < 3) throw std::runtime_error("usage: regions <in.c>");
    std::string src = read_file(argv[2]);
    KernelModule m = parse(src, argv[2]);
    for (const Region& r : find_regions(m)) {
        std::cout << r.index << " " << r.fn->name;
        for (auto& v : r.enclosing_loop_vars) std::cout << " " << v;
        std::cout << "\n";
    }
    return 0;
}

}  // namespace

int main(int argc, char** argv) {
    if (argc < 2) {
        std::cerr << "usage: ref_tool opt|eval|regions ...\n";
        return 2;
    }
    std::string cmd = argv[1];
    try {
        if (cmd == "opt") return cmd_opt(argc, argv);
        if (cmd == "eval") return cmd_eval(argc, argv);
        if (cmd == "regions") return cmd_regions(argc, argv);
    } catch (const EvalError& e) {
        std::cerr << "EvalError: " << e.what() << "\n";
        return 3;
    } catch (const std::exception& e) {
        std::cerr << "error: " << e.what() << "\n";
        return 1;
    }
    std::cerr << "unknown command " << cmd << "\n";
    return 2;
}
