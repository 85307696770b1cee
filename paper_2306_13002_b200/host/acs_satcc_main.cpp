// acs-satcc — command-line driver over host stage (a) (include/accsat_opt.h),
// option-compatible with the reference CLI's core (proj/tools/satcc_main.cpp):
//
//   acs-satcc [opt] [--variant V] [-o FILE] file        optimized source
//   acs-satcc report [--variant V] [--gpu [--size N]] file...
//                                                       satcc-metrics-v1 JSON (--gpu: plus the
//        B200 execution of every region: GB/s, roofline fraction, skeleton,
//        saturated-vs-original difference; paper_2306_13002_b200/report.py)
//   acs-satcc verify [--variant V] [--trials N] [--tol T] file...
//                                                       satcc-verify-v1 JSON: differential
//        run of original vs optimized region bodies under the reference's
//        interpreter semantics (diff_test, proj/src/oracle.cpp:12-81)
//   acs-satcc [--variant V] [--keep] [--backend cc|b200] -- cmd args...
//                                                       wrapper mode: every
//        existing *.c argument is optimized into <tmp>/<argidx>/<basename> and
//        cmd runs on the substituted paths; exit code propagated (128+signal,
//        127 if exec fails); an unparseable file passes through unchanged
//        (satcc_main.cpp:285-360).  --backend b200: the nest functions of
//        every file run on the B200 instead (paper_2306_13002_b200/jit.py).
//
// Flags: --variant (cse | cse+sat | cse+bulk | accsat, default accsat),
// --max-nodes, --sat-time, --iters, --extract greedy|dag, --no-sat, --no-bulk.
#include <sys/stat.h>
#include <sys/wait.h>
#include <unistd.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <iostream>
#include <sstream>
#include <string>
#include <vector>

#include "../../include/accsat_opt.h"

static std::string read_file(const std::string& p) {
    std::ifstream in(p, std::ios::binary);
    if (!in) throw std::runtime_error("cannot open " + p);
    std::ostringstream ss;
    ss << in.rdbuf();
    return ss.str();
}

int main(int argc, char** argv) {
    std::vector<std::string> args(argv + 1, argv + argc);
    std::string cmd = "opt", variant = "accsat", output;
    acs_opt_limits lim{10000, 10.0, 10, 1, 0.0};
    bool no_sat = false, no_bulk = false, keep = false;
    std::string backend = "cc";   // cc: hand the optimized C to the wrapped compiler; b200: to this backend
    bool gpu = false;             // report --gpu: satcc-metrics-v1 plus the B200 execution of every region
    std::string size;
    std::vector<std::string> files, child;
    size_t i = 0;
    if (!args.empty() && (args[0] == "opt" || args[0] == "report" || args[0] == "verify")) cmd = args[i++];
    int trials = 20;
    double tol_rel = 1e-6;   // satcc's default --tol (proj/tools/satcc_main.cpp:51)
    for (; i < args.size(); ++i) {
        const std::string& a = args[i];
        auto next = [&]() -> std::string {
            if (i + 1 >= args.size()) {
                std::cerr << "acs-satcc: " << a << " needs a value\n";
                std::exit(2);
            }
            return args[++i];
        };
        if (a == "--") {
            child.assign(args.begin() + (long)i + 1, args.end());
            cmd = "wrap";
            break;
        } else if (a == "--variant") variant = next();
        else if (a == "-o") output = next();
        else if (a == "--max-nodes") lim.max_nodes = std::stol(next());
        else if (a == "--sat-time") lim.max_time_s = std::stod(next());
        else if (a == "--iters") lim.max_iters = std::stoi(next());
        else if (a == "--extract") lim.dag_search = next() == "greedy" ? 0 : 1;
        else if (a == "--no-sat") no_sat = true;
        else if (a == "--no-bulk") no_bulk = true;
        else if (a == "--keep") keep = true;
        else if (a == "--backend") backend = next();
        else if (a == "--gpu") gpu = true;
        else if (a == "--size") size = next();
        else if (a == "--trials") trials = std::stoi(next());
        else if (a == "--tol") tol_rel = std::stod(next());
        else files.push_back(a);
    }
    bool sat = variant == "accsat" || variant == "cse+sat", bulk = variant == "accsat" || variant == "cse+bulk";
    if (no_sat) sat = false;
    if (no_bulk) bulk = false;
    std::string v = sat && bulk ? "accsat" : sat ? "cse+sat" : bulk ? "cse+bulk" : "cse";

    auto optimize = [&](const std::string& path, std::string& text, std::string& json) {
        char *t = nullptr, *j = nullptr;
        std::string src = read_file(path);
        int rc = acs_opt_optimize(src.c_str(), path.c_str(), v.c_str(), &lim, &t, &j);
        text = t;
        json = j;
        acs_opt_free(t);
        acs_opt_free(j);
        return rc;
    };

    auto exec_python = [&](std::vector<std::string> py) -> int {
        std::string exe = argv[0];
        std::string dir = exe.find_last_of('/') == std::string::npos ? "." : exe.substr(0, exe.find_last_of('/'));
        const char* pp = std::getenv("PYTHONPATH");
        std::string path = dir + "/.." + (pp ? std::string(":") + pp : "");
        setenv("PYTHONPATH", path.c_str(), 1);
        std::vector<char*> av;
        for (auto& x : py) av.push_back(const_cast<char*>(x.c_str()));
        av.push_back(nullptr);
        execvp(av[0], av.data());
        std::cerr << "acs-satcc: cannot exec python3\n";
        return 127;
    };
    if (cmd == "report" && gpu) {
        std::vector<std::string> py = {"python3", "-m", "paper_2306_13002_b200.report", "--gpu", "--variant", variant};
        if (!size.empty()) {
            py.push_back("--size");
            py.push_back(size);
        }
        py.insert(py.end(), files.begin(), files.end());
        return exec_python(py);
    }
    if (cmd == "wrap" && backend == "b200") {
        // the B200 as the downstream: paper_2306_13002_b200/jit.py builds the
        // file's kernels and stubs the nest functions into acs_eval_host calls
        std::vector<std::string> py = {"python3", "-m", "paper_2306_13002_b200.jit", "wrap", "--variant", variant};
        if (keep) py.push_back("--keep");
        py.push_back("--");
        py.insert(py.end(), child.begin(), child.end());
        return exec_python(py);
    }
    if (cmd == "wrap") {
        if (child.empty()) {
            std::cerr << "acs-satcc: nothing to run after --\n";
            return 2;
        }
        std::string tmp;
        if (keep) {
            tmp = "satcc-cache";
            mkdir(tmp.c_str(), 0755);
        } else {
            char tpl[] = "/tmp/acs-satcc-XXXXXX";
            if (!mkdtemp(tpl)) return 127;
            tmp = tpl;
        }
        for (size_t a = 0; a < child.size(); ++a) {
            const std::string& f = child[a];
            if (f.size() < 2 || f.compare(f.size() - 2, 2, ".c") != 0) continue;
            struct stat st;
            if (stat(f.c_str(), &st) != 0) continue;
            std::string text, json;
            try {
                if (optimize(f, text, json) != 0) {
                    std::cerr << "acs-satcc: warning: " << f << " passed through unchanged: " << json << "\n";
                    continue;
                }
            } catch (const std::exception& e) {
                std::cerr << "acs-satcc: warning: " << f << ": " << e.what() << "\n";
                continue;
            }
            std::string dir = tmp + "/" + std::to_string(a);
            mkdir(dir.c_str(), 0755);
            std::string base = f.substr(f.find_last_of('/') == std::string::npos ? 0 : f.find_last_of('/') + 1);
            std::string out = dir + "/" + base;
            std::ofstream(out, std::ios::binary) << text;
            child[a] = out;
        }
        std::vector<char*> av;
        for (auto& s : child) av.push_back(const_cast<char*>(s.c_str()));
        av.push_back(nullptr);
        pid_t pid = fork();
        if (pid == 0) {
            execvp(av[0], av.data());
            _exit(127);
        }
        int status = 0;
        waitpid(pid, &status, 0);
        if (!keep) {
            std::string rm = "rm -rf '" + tmp + "'";
            if (std::system(rm.c_str()) != 0) std::cerr << "acs-satcc: could not remove " << tmp << "\n";
        }
        if (WIFEXITED(status)) return WEXITSTATUS(status);
        if (WIFSIGNALED(status)) return 128 + WTERMSIG(status);
        return 1;
    }

    if (files.empty()) {
        std::cerr << "usage: acs-satcc [opt|report|verify] [--variant V] file...  |  acs-satcc [flags] -- cmd args...\n";
        return 2;
    }
    if (cmd == "verify") {   // satcc-verify-v1 (proj/tools/satcc_main.cpp:217-283)
        int rc = 0;
        bool all_ok = true;
        std::string out = "{\"schema\": \"satcc-verify-v1\", \"trials\": " + std::to_string(trials) +
                          ", \"tol_rel\": " + std::to_string(tol_rel) + ", \"files\": [";
        bool first = true;
        for (const std::string& f : files) {
            char* j = nullptr;
            std::string src;
            try {
                src = read_file(f);
            } catch (const std::exception& e) {
                std::cerr << "acs-satcc: error: " << e.what() << "\n";
                rc = 1;
                continue;
            }
            int r = acs_opt_verify(src.c_str(), f.c_str(), v.c_str(), &lim, trials, tol_rel, &j);
            std::string js = j;
            acs_opt_free(j);
            if (r == 2) {
                std::cerr << "acs-satcc: error: " << f << ": " << js << "\n";
                rc = 1;
                continue;
            }
            if (r == 1) all_ok = false;
            out += (first ? "" : ", ") + js;
            first = false;
        }
        out += std::string("], \"ok\": ") + (all_ok ? "true" : "false") + "}";
        std::cout << out << "\n";
        if (!all_ok) rc = 1;
        return rc;
    }
    int rc = 0;
    std::string reports = "[";
    for (size_t f = 0; f < files.size(); ++f) {
        std::string text, json;
        try {
            int r = optimize(files[f], text, json);
            if (r) rc = 1;
        } catch (const std::exception& e) {
            std::cerr << "acs-satcc: error: " << e.what() << "\n";
            rc = 1;
            continue;
        }
        if (cmd == "opt") {
            if (!output.empty())
                std::ofstream(output, std::ios::binary) << text;
            else
                std::cout << text;
        } else {
            reports += (f ? ",\n" : "\n") + json;
        }
    }
    if (cmd == "report") std::cout << reports << "]\n";
    return rc;
}
