// ts_hydro_taskscope.hpp — the reference-side binding a taskscope maintainer
// adds to use the B200 hydro path: a header-only C++ adapter over the C ABI
// (ts_hydro.h) that speaks the reference's own types.
//
//   * CudaHydroDevice::launch_stage(stage, sub-grid, stream, guid) returns a
//     taskscope::CompletionToken fulfilled from the CUDA host callback once
//     the fused stage kernel finished — the replacement for the two
//     SimDevice::launch_kernel awaits in WorkloadSession::fluxes_body
//     (reference proj/core/src/workload.cpp:544-552, device.hpp:57-58);
//   * flush_activity(Profiler&) converts ts_activity_record into
//     taskscope::ActivityRecord on RunClock and calls
//     Profiler::deliver_activity (device.cpp:127-130, profiler.cpp:298-318);
//   * ts_hydro error codes become the reference's exception types
//     (std::invalid_argument / std::runtime_error, device.cpp:26-62).
//
// Include it from code that already builds against the reference headers
// (it needs taskscope/{device,profiler,clock}.hpp); see INTEGRATION.md.
#pragma once

#include <cstdint>
#include <map>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "taskscope/clock.hpp"
#include "taskscope/device.hpp"
#include "taskscope/profiler.hpp"
#include "taskscope/token.hpp"
#include "ts_hydro.h"

namespace taskscope {

class CudaHydroDevice {
public:
    explicit CudaHydroDevice(const ts_hydro_config& cfg, Profiler* sink = nullptr) : sink_(sink) {
        // RunClock is zeroed at its first read: fix the epoch before any device
        // activity so no record predates it (clock.hpp:11-13)
        (void)RunClock::instance().now_ns();
        check(ts_hydro_create(&cfg, &ctx_), "ts_hydro_create");
    }
    ~CudaHydroDevice() {
        if (ctx_ != nullptr) {
            if (sink_ != nullptr) flush_activity(*sink_);
            ts_hydro_destroy(ctx_);
        }
    }
    CudaHydroDevice(const CudaHydroDevice&) = delete;
    CudaHydroDevice& operator=(const CudaHydroDevice&) = delete;

    ts_hydro_ctx* ctx() { return ctx_; }

    // Binds the reference Mesh's neighbour / owner tables (workload.hpp:76-97).
    void set_mesh(const std::vector<std::int64_t>& neighbor_ids, const std::vector<std::int32_t>& owner,
                  std::int32_t world_size, std::int32_t rank) {
        check(ts_hydro_set_mesh(ctx_, static_cast<std::int64_t>(owner.size()), neighbor_ids.data(), owner.data(),
                                world_size, rank),
              "set_mesh");
    }

    // The compute_fluxes drop-in: one fused RK stage of one owned sub-grid.
    CompletionToken launch_stage(int stage, std::int64_t owned_index, std::uint32_t stream_id, Guid guid) {
        auto* promise = new PromiseHandle();
        CompletionToken token = promise->token();
        const int rc = ts_hydro_launch_stage(ctx_, stage, &owned_index, 1, stream_id, guid, &fulfil, promise);
        if (rc != TS_OK) {
            delete promise;
            check(rc, "launch_stage");
        }
        return token;
    }

    // The gravity launch of execute_step_body (workload.cpp:565-569) for a
    // sub-grid gravity_kernel_name calls a p2p_kernel (workload.cpp:365-372):
    // the near-field monopole P2P of that sub-grid, for real.
    CompletionToken launch_gravity_p2p(std::int64_t owned_index, std::uint32_t stream_id, Guid guid,
                                       double G = 1.0, int radius = 4) {
        auto* promise = new PromiseHandle();
        CompletionToken token = promise->token();
        const int rc = ts_hydro_gravity_p2p(ctx_, G, radius, &owned_index, 1, stream_id, guid, &fulfil, promise);
        if (rc != TS_OK) {
            delete promise;
            check(rc, "launch_gravity_p2p");
        }
        return token;
    }

    // The whole gravity solve of a step (the FMM over the octree: every
    // sub-grid's multipole_root / multipole / p2m / p2p work of
    // workload.cpp:565-569 in one call, records named by kind), after the
    // step's hydro of every sub-grid; then, with kick = true, the source term
    // over the last step's dt.  Needs set_gravity_tree.
    CompletionToken launch_gravity_fmm(std::uint32_t stream_id, Guid guid, double G = 1.0, int radius = 2,
                                       bool kick = false) {
        auto* promise = new PromiseHandle();
        CompletionToken token = promise->token();
        int rc = ts_hydro_gravity_fmm(ctx_, G, radius, stream_id, guid, kick ? nullptr : &fulfil, kick ? nullptr : promise);
        if (rc == TS_OK && kick) {
            rc = ts_hydro_gravity_kick(ctx_, -1.0);
            if (rc == TS_OK) rc = ts_hydro_synchronize(ctx_);  // the kick takes no callback: ready on return
            if (rc == TS_OK) {
                promise->set_value();
                delete promise;
                return token;
            }
        }
        if (rc != TS_OK) {
            delete promise;
            check(rc, "launch_gravity_fmm");
        }
        return token;
    }
    void set_gravity_tree(const std::vector<std::int32_t>& level, const std::vector<std::int32_t>& pos,
                          const std::int32_t dims[3], double dx0) {
        check(ts_hydro_set_gravity_tree(ctx_, (std::int64_t)level.size(), level.data(), pos.data(), dims, dx0),
              "set_gravity_tree");
    }

    // The rest of SimDevice's public surface (device.hpp:57-64) on the GPU, so
    // a CudaHydroDevice stands in for the SimDevice a Locality owns: named
    // launches occupy their stream for the requested time (the gravity
    // kernels of workload.cpp:565-569), copies really move `bytes`.
    CompletionToken launch_kernel(const std::string& name, std::uint32_t stream_id, std::uint64_t duration_ns,
                                  Guid guid) {
        auto* promise = new PromiseHandle();
        CompletionToken token = promise->token();
        const int rc = ts_hydro_launch_kernel(ctx_, name.c_str(), stream_id, duration_ns, guid, &fulfil, promise);
        if (rc != TS_OK) {
            delete promise;
            check(rc, "launch_kernel");
        }
        return token;
    }

    CompletionToken enqueue_copy(ActivityKind kind, std::uint64_t bytes, std::uint32_t stream_id, Guid guid) {
        auto* promise = new PromiseHandle();
        CompletionToken token = promise->token();
        const int rc = ts_hydro_enqueue_copy(ctx_, static_cast<std::int32_t>(kind), bytes, stream_id, guid, &fulfil,
                                             promise);
        if (rc != TS_OK) {
            delete promise;
            check(rc, "enqueue_copy");
        }
        return token;
    }

    std::uint64_t device_alloc(std::uint64_t bytes) {
        std::uint64_t h = 0;
        check(ts_hydro_device_alloc(ctx_, bytes, &h), "device_alloc");
        return h;
    }
    void device_free(std::uint64_t handle) { check(ts_hydro_device_free(ctx_, handle), "device_free"); }

    // SimDevice::host_pinned_alloc/free (device.hpp:64-65): handle-based like
    // the reference (handles from 1, device.cpp:171-212); the pinned memory
    // itself is reachable through host_pinned_ptr.
    std::uint64_t host_pinned_alloc(std::uint64_t bytes) {
        void* p = nullptr;
        check(ts_hydro_host_alloc(ctx_, bytes, &p), "host_pinned_alloc");
        std::lock_guard<std::mutex> lk(pinned_mu_);
        const std::uint64_t h = next_pinned_++;
        pinned_[h] = p;
        return h;
    }
    void host_pinned_free(std::uint64_t handle) {
        void* p = nullptr;
        {
            std::lock_guard<std::mutex> lk(pinned_mu_);
            auto it = pinned_.find(handle);
            if (it == pinned_.end()) throw std::invalid_argument("host_pinned_free: unknown host pinned handle");
            p = it->second;
            pinned_.erase(it);
        }
        check(ts_hydro_host_free(ctx_, p), "host_pinned_free");
    }
    void* host_pinned_ptr(std::uint64_t handle) const {
        std::lock_guard<std::mutex> lk(pinned_mu_);
        auto it = pinned_.find(handle);
        return it == pinned_.end() ? nullptr : it->second;
    }

    // SimDevice::flush_activity(Profiler&): at-most-once, RunClock timestamps.
    std::uint64_t flush_activity(Profiler& sink) {
        std::uint64_t n = 0;
        check(ts_hydro_flush_activity(ctx_, nullptr, 0, &n), "flush_activity");
        std::vector<ts_activity_record> recs(n);
        check(ts_hydro_flush_activity(ctx_, recs.data(), n, &n), "flush_activity");
        const auto epoch = static_cast<std::uint64_t>(
            std::chrono::duration_cast<std::chrono::nanoseconds>(RunClock::instance().epoch().time_since_epoch())
                .count());
        for (std::uint64_t i = 0; i < n; ++i) {
            const ts_activity_record& r = recs[i];
            ActivityRecord a;
            a.kind = static_cast<ActivityKind>(r.kind);
            a.name = r.name;
            a.device_id = r.device_id;
            a.stream_id = r.stream_id;
            a.start_ns = r.start_ns > epoch ? r.start_ns - epoch : 0;
            a.end_ns = r.end_ns > epoch ? r.end_ns - epoch : 0;
            if (r.has_bytes) a.bytes = r.bytes;
            a.correlation_guid = r.correlation_guid;
            sink.deliver_activity(a);
        }
        return n;
    }

    // SimDevice::flush_activity() (device.hpp:76-77): to the default sink given
    // at construction; without one the records stay buffered (returns 0).
    std::uint64_t flush_activity() { return sink_ != nullptr ? flush_activity(*sink_) : 0; }

    DeviceMemoryState memory_state() const {
        ts_memory_state m{};
        ts_hydro_memory_state(ctx_, &m);
        return DeviceMemoryState{m.current_device_bytes, m.peak_device_bytes, m.current_host_pinned_bytes,
                                 m.peak_host_pinned_bytes};
    }

    void shutdown() { check(ts_hydro_shutdown(ctx_), "shutdown"); }

private:
    static void fulfil(void* user) {
        auto* promise = static_cast<PromiseHandle*>(user);
        promise->set_value();
        delete promise;
    }

    void check(int rc, const char* what) const {
        if (rc == TS_OK) return;
        const std::string msg = std::string(what) + ": " +
                                (ctx_ != nullptr ? ts_hydro_last_error(ctx_) : ts_hydro_strerror(rc));
        if (rc == TS_EINVAL) throw std::invalid_argument(msg);
        throw std::runtime_error(msg);
    }

    ts_hydro_ctx* ctx_ = nullptr;
    Profiler* sink_ = nullptr;
    mutable std::mutex pinned_mu_;
    std::map<std::uint64_t, void*> pinned_;
    std::uint64_t next_pinned_ = 1;
};

}  // namespace taskscope
