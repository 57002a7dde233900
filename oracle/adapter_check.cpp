// Build check (and, on a GPU box, a run check) of include/ts_hydro_taskscope.hpp
// against the reference's own headers and core: a reference-style Profiler
// receives the B200 kernels' ActivityRecords through deliver_activity.
#include <cstdio>
#include <vector>

#include "ts_hydro_taskscope.hpp"
#ifdef TS_HAVE_EXPORT
#include "taskscope/export.hpp"
#endif

int main(int argc, char** argv) {
    using namespace taskscope;
    ts_hydro_config cfg;
    ts_hydro_default_config(&cfg);
    if (argc < 2) {  // build check only
        std::printf("adapter links: ts_hydro ABI %d\n", ts_hydro_abi_version());
        return 0;
    }
    Profiler profiler;
    CudaHydroDevice dev(cfg, nullptr);
    std::vector<std::int64_t> nbr(6 * 8);
    std::vector<std::int32_t> pos(3 * 8), owner(8);
    ts_hydro_uniform_mesh(2, 2, 2, 7, 1, nbr.data(), pos.data(), owner.data());
    dev.set_mesh(nbr, owner, 1, 0);
    ts_hydro_init_random(dev.ctx(), 1);
    double dt = 0;
    ts_hydro_compute_dt(dev.ctx(), &dt);
    std::vector<CompletionToken> tokens;
    for (int stage = 1; stage <= 3; ++stage) {
        for (std::int64_t g = 0; g < 8; ++g) tokens.push_back(dev.launch_stage(stage, g, 2 + g % 4, 100 + g));
        for (auto& t : tokens) t->wait_blocking();
        tokens.clear();
    }
    ts_hydro_finish_step(dev.ctx());
    // the rest of the step's schedule (workload.cpp:565-569): named gravity
    // launches and a copy, through the SimDevice-shaped calls
    for (std::int64_t g = 0; g < 8; ++g) tokens.push_back(dev.launch_kernel("multipole_kernel", g % 4, 20000, 100 + g));
    tokens.push_back(dev.enqueue_copy(ActivityKind::copy_device_to_host, 1 << 20, 5, 99));
    for (auto& t : tokens) t->wait_blocking();
    const std::uint64_t h = dev.device_alloc(4096);
    dev.device_free(h);
    const auto n = dev.flush_activity(profiler);
    const Snapshot s = profiler.snapshot();
    const auto it = s.profile.find("hydro_stage1_kernel");
    const auto grav = s.profile.find("multipole_kernel");
#ifdef TS_HAVE_EXPORT
    // the reference's own exporters over the real GPU activity: Google trace
    // events (device lanes 10000 + device*1000 + stream) and the profile CSV
    if (argc >= 4) {
        const RunProfile run{s};
        const auto events = write_trace_events(run, argv[2]);
        const auto rows = write_profile_csv(run, argv[3]);
        std::printf("trace events %llu, csv rows %llu\n", (unsigned long long)events, (unsigned long long)rows);
    }
#endif
    std::printf("records %llu, hydro_stage1_kernel calls %llu, multipole_kernel calls %llu\n", (unsigned long long)n,
                (unsigned long long)(it == s.profile.end() ? 0 : it->second.calls),
                (unsigned long long)(grav == s.profile.end() ? 0 : grav->second.calls));
    return (it != s.profile.end() && it->second.calls == 8 && grav != s.profile.end() && grav->second.calls == 8) ? 0
                                                                                                                : 1;
}
