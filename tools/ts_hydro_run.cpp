// ts_hydro_run — native C++ host driver over the C ABI (no Python, no torch).
//
// The shape of the reference's `taskscope bench` path (tools/main.cpp:94-169 ->
// WorkloadSession::run_benchmark, workload.cpp:595-612) for the real hydro:
// read a key=value workload config (same syntax and error rules as
// parse_workload_config, workload.cpp:382-432), build the mesh, load the
// initial state, time the stepping only, report cells/s = total_cells * steps
// / seconds, and print the per-kernel activity profile the timing hook
// produced (the flat profile Profiler::deliver_activity would build,
// profiler.cpp:298-318).  Single GPU.
//
//   built by `python -m paper_2210_06437_b200.build` (g++ against include/ and
//   libts_hydro.so, rpath to the package directory);
//   tools/ts_hydro_run [config-file]      (defaults: Sedov 16^3 sub-grids, 20 steps)
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <map>
#include <numeric>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "ts_hydro.h"

namespace {

struct RunConfig {
    int nx = 16, ny = 16, nz = 16;
    int steps = 20;
    int species = 0;
    std::string problem = "sedov";
    std::string recon = "ppm";
    std::string periodic;
    double cfl = 0.4, gamma = 1.4;
};

std::string trim(const std::string& s) {
    const auto b = s.find_first_not_of(" \t\r");
    if (b == std::string::npos) return "";
    return s.substr(b, s.find_last_not_of(" \t\r") - b + 1);
}

[[noreturn]] void config_error(int line, const std::string& msg) {
    throw std::runtime_error("workload config line " + std::to_string(line) + ": " + msg);
}

int to_int(const std::string& v, int line, const std::string& key) {
    char* end = nullptr;
    const long x = std::strtol(v.c_str(), &end, 10);
    if (v.empty() || *end != '\0') config_error(line, "bad value '" + v + "' for key '" + key + "'");
    return static_cast<int>(x);
}

RunConfig parse(std::istream& in) {
    RunConfig c;
    std::string raw;
    int line = 0;
    while (std::getline(in, raw)) {
        ++line;
        const std::string t = trim(raw);
        if (t.empty() || t[0] == '#') continue;
        const auto eq = t.find('=');
        if (eq == std::string::npos) config_error(line, "expected key=value");
        const std::string k = trim(t.substr(0, eq)), v = trim(t.substr(eq + 1));
        if (k.empty()) config_error(line, "empty key");
        if (k == "nx") c.nx = to_int(v, line, k);
        else if (k == "ny") c.ny = to_int(v, line, k);
        else if (k == "nz") c.nz = to_int(v, line, k);
        else if (k == "steps") c.steps = to_int(v, line, k);
        else if (k == "species") c.species = to_int(v, line, k);
        else if (k == "problem") c.problem = v;
        else if (k == "recon") c.recon = v;
        else if (k == "periodic") c.periodic = v;
        else if (k == "cfl") c.cfl = std::stod(v);
        else if (k == "gamma") c.gamma = std::stod(v);
        else if (k == "N") { if (v != "8") config_error(line, "N must be 8"); }
        else if (k == "levels" || k == "streams" || k == "seed" || k == "comm_mode" || k == "hydro_iterations" ||
                 k == "gravity_iterations" || k == "kernel_min_ns" || k == "kernel_max_ns") {
        } else config_error(line, "unknown key '" + k + "'");
    }
    return c;
}

void check(int rc, ts_hydro_ctx* ctx, const char* what) {
    if (rc == TS_OK) return;
    std::fprintf(stderr, "%s failed: %s (%s)\n", what, ts_hydro_strerror(rc), ctx ? ts_hydro_last_error(ctx) : "");
    std::exit(1);
}

}  // namespace

int main(int argc, char** argv) {
    RunConfig rc;
    try {
        if (argc > 1) {
            std::ifstream f(argv[1]);
            if (!f) throw std::runtime_error(std::string("cannot open workload config ") + argv[1]);
            rc = parse(f);
        }
    } catch (const std::exception& e) {
        std::fprintf(stderr, "%s\n", e.what());
        return 2;
    }
    const std::map<std::string, int> problems{{"sod", TS_PROBLEM_SOD}, {"sedov", TS_PROBLEM_SEDOV},
                                              {"random", TS_PROBLEM_RANDOM}, {"polytrope", TS_PROBLEM_POLYTROPE},
                                              {"binary", TS_PROBLEM_BINARY}};
    if (!problems.count(rc.problem)) {
        std::fprintf(stderr, "unknown problem '%s'\n", rc.problem.c_str());
        return 2;
    }
    ts_hydro_config cfg;
    ts_hydro_default_config(&cfg);
    cfg.n_species = rc.species;
    cfg.recon = rc.recon == "minmod" ? TS_RECON_MINMOD : TS_RECON_PPM;
    cfg.cfl = rc.cfl;
    cfg.gamma = rc.gamma;
    cfg.dx = 1.0 / (8.0 * rc.nx);
    const int nf = 6 + rc.species;

    const int64_t n = (int64_t)rc.nx * rc.ny * rc.nz;
    std::vector<int64_t> nbr(6 * n);
    std::vector<int32_t> pos(3 * n), owner(n);
    int mask = 0;
    for (char ch : rc.periodic) mask |= 1 << (ch - 'x');
    check(ts_hydro_uniform_mesh(rc.nx, rc.ny, rc.nz, mask, 1, nbr.data(), pos.data(), owner.data()), nullptr,
          "uniform_mesh");

    ts_hydro_ctx* ctx = nullptr;
    check(ts_hydro_create(&cfg, &ctx), nullptr, "create");
    check(ts_hydro_set_mesh(ctx, n, nbr.data(), owner.data(), 1, 0), ctx, "set_mesh");
    std::vector<int64_t> ids(n);
    std::iota(ids.begin(), ids.end(), 0);
    const int32_t dims[3] = {rc.nx, rc.ny, rc.nz};
    std::vector<double> U((size_t)n * nf * 512);
    check(ts_hydro_ic_fill(&cfg, problems.at(rc.problem), n, ids.data(), pos.data(), dims, 2210, U.data()), ctx,
          "ic_fill");
    check(ts_hydro_upload(ctx, 0, n, U.data()), ctx, "upload");
    double dt0 = 0.0;
    check(ts_hydro_compute_dt(ctx, &dt0), ctx, "compute_dt");
    check(ts_hydro_step(ctx, 3), ctx, "warm-up");
    check(ts_hydro_synchronize(ctx), ctx, "synchronize");
    uint64_t nrec = 0;
    check(ts_hydro_flush_activity(ctx, nullptr, 0, &nrec), ctx, "flush");
    std::vector<ts_activity_record> drop(nrec);
    check(ts_hydro_flush_activity(ctx, drop.data(), nrec, &nrec), ctx, "flush");

    // timed region: stepping only (workload.cpp:599-604)
    double ms = 0.0;
    const auto t0 = std::chrono::steady_clock::now();
    check(ts_hydro_time_steps(ctx, (uint64_t)rc.steps, &ms), ctx, "time_steps");
    const double wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();

    check(ts_hydro_flush_activity(ctx, nullptr, 0, &nrec), ctx, "flush");
    std::vector<ts_activity_record> recs(nrec);
    check(ts_hydro_flush_activity(ctx, recs.data(), nrec, &nrec), ctx, "flush");
    struct Entry {
        uint64_t calls = 0, total = 0, min = UINT64_MAX, max = 0;
    };
    std::map<std::string, Entry> prof;
    for (uint64_t i = 0; i < nrec; ++i) {
        const auto& r = recs[i];
        if (r.kind != TS_ACTIVITY_KERNEL) continue;
        auto& e = prof[r.name];
        const uint64_t d = r.end_ns - r.start_ns;
        ++e.calls;
        e.total += d;
        e.min = std::min(e.min, d);
        e.max = std::max(e.max, d);
    }
    double dt_last = 0.0;
    check(ts_hydro_last_dt(ctx, &dt_last), ctx, "last_dt");
    const double cells = (double)n * 512.0;
    std::printf("workload: %s %dx%dx%d sub-grids (%.0f cells), nf=%d, %s, %d steps\n", rc.problem.c_str(), rc.nx,
                rc.ny, rc.nz, cells, nf, rc.recon.c_str(), rc.steps);
    std::printf("cells_per_second (device events) = %.6g   (host wall %.6g)\n", cells * rc.steps / (ms * 1e-3),
                cells * rc.steps / wall);
    std::printf("ms_per_step = %.4f   dt0 = %.6g   dt_last = %.6g\n", ms / rc.steps, dt0, dt_last);
    std::printf("%-24s %8s %12s %10s %10s\n", "kernel", "calls", "total_us", "mean_us", "max_us");
    for (const auto& [name, e] : prof)
        std::printf("%-24s %8llu %12.1f %10.1f %10.1f\n", name.c_str(), (unsigned long long)e.calls, e.total / 1e3,
                    e.total / 1e3 / (double)e.calls, e.max / 1e3);
    ts_hydro_destroy(ctx);
    return 0;
}
