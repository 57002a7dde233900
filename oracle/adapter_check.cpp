// Build check (and, on a GPU box, a run check) of include/ts_hydro_taskscope.hpp
// against the reference's own headers and core: a reference-style Profiler
// receives the B200 kernels' ActivityRecords through deliver_activity.
#include <cstdio>
#include <cstring>
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
    std::vector<std::int64_t> nbr(6 * 64);
    std::vector<std::int32_t> pos(3 * 64), owner(64);
    ts_hydro_uniform_mesh(4, 4, 4, 7, 1, nbr.data(), pos.data(), owner.data());
    dev.set_mesh(nbr, owner, 1, 0);
    ts_hydro_init_random(dev.ctx(), 1);
    double dt = 0;
    ts_hydro_compute_dt(dev.ctx(), &dt);
    // the reference's schedule without any host barrier: every sub-grid's
    // compute_fluxes launches of a step go out on round-robin streams
    // (next_stream, workload.cpp:481-485) in a scrambled sub-grid order; the
    // tokens are awaited only at the end of the run (run_step's drain)
    std::vector<CompletionToken> tokens;
    const int kSteps = 4;
    std::uint32_t stream = 0;
    for (int step = 0; step < kSteps; ++step) {
        for (int stage = 1; stage <= 3; ++stage)
            for (std::int64_t k = 0; k < 64; ++k) {
                const std::int64_t g = (k * 37 + step * 11 + stage * 5) % 64;
                tokens.push_back(dev.launch_stage(stage, g, stream++ % cfg.stream_count, 100 + g));
            }
        ts_hydro_finish_step(dev.ctx());
    }
    for (auto& t : tokens) t->wait_blocking();
    tokens.clear();
    // the same steps batched (ts_hydro_step) on a second context: bitwise equal
    std::vector<double> got((size_t)64 * 6 * 512), want(got.size());
    ts_hydro_download(dev.ctx(), 0, 64, got.data());
    {
        ts_hydro_ctx* ref = nullptr;
        ts_hydro_create(&cfg, &ref);
        ts_hydro_set_mesh(ref, 64, nbr.data(), owner.data(), 1, 0);
        ts_hydro_init_random(ref, 1);
        ts_hydro_step(ref, kSteps);
        ts_hydro_download(ref, 0, 64, want.data());
        ts_hydro_destroy(ref);
    }
    if (std::memcmp(got.data(), want.data(), got.size() * sizeof(double)) != 0) {
        std::printf("drop-in steps differ from the batched steps\n");
        return 1;
    }
    std::printf("drop-in: %d steps x 3 stages x 64 sub-grids on %u streams, no host barrier: bitwise = batched\n",
                kSteps, cfg.stream_count);
    const std::uint64_t hp = dev.host_pinned_alloc(1 << 16);
    if (dev.host_pinned_ptr(hp) == nullptr) return 1;
    dev.host_pinned_free(hp);
    // the rest of the step's schedule (workload.cpp:565-569): named gravity
    // launches and a copy, through the SimDevice-shaped calls
    for (std::int64_t g = 0; g < 8; ++g) tokens.push_back(dev.launch_kernel("multipole_kernel", g % 4, 20000, 100 + g));
    tokens.push_back(dev.enqueue_copy(ActivityKind::copy_device_to_host, 1 << 20, 5, 99));
    for (auto& t : tokens) t->wait_blocking();
    tokens.clear();
    // the whole gravity solve of a step (FMM; records named by kind) and its kick
    const std::vector<std::int32_t> lev(64, 0), posv(pos.begin(), pos.end());
    const std::int32_t dims[3] = {4, 4, 4};
    dev.set_gravity_tree(lev, posv, dims, cfg.dx);
    tokens.push_back(dev.launch_gravity_fmm(3, 500, 1.0, 2, false));
    tokens.push_back(dev.launch_gravity_fmm(4, 501, 1.0, 2, true));
    for (auto& t : tokens) t->wait_blocking();
    const std::uint64_t h = dev.device_alloc(4096);
    dev.device_free(h);
    const auto n = dev.flush_activity(profiler);
    const Snapshot s = profiler.snapshot();
    const auto it = s.profile.find("hydro_stage1_kernel");
    const auto grav = s.profile.find("multipole_kernel");
    const auto p2p = s.profile.find("p2p_kernel");
    const auto root = s.profile.find("multipole_root_kernel");
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
    auto calls = [&](decltype(it) e) { return (unsigned long long)(e == s.profile.end() ? 0 : e->second.calls); };
    std::printf("records %llu, hydro_stage1_kernel calls %llu, multipole_kernel calls %llu (8 named + 2 x 2 FMM), "
                "multipole_root_kernel %llu, p2p_kernel %llu\n",
                (unsigned long long)n, calls(it), calls(grav), calls(root), calls(p2p));
    // 4^3 sub-grids: a root, 8 refined nodes, 64 leaves -> per solve 2 multipole (M2M + M2L of depth 1),
    // 2 multipole_root (M2M + M2L of the root), 1 p2p (the leaves)
    return (calls(it) == 4 * 64 && calls(grav) == 8 + 4 && calls(root) == 4 && calls(p2p) == 2) ? 0 : 1;
}
