// ORACLE — TEST INFRASTRUCTURE ONLY.
//
// C shim over the reference's own compiled core (built from /root/reference
// sources into oracle/_ref by `make -C oracle ref`).  tests/golden/gen_golden.py
// calls it to draw golden vectors for the data-model pieces of the hot path.
// Nothing here is shipped or timed.

#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <string>

#include "taskscope/distrib.hpp"
#include "taskscope/sampling.hpp"
#include "taskscope/workload.hpp"

using namespace taskscope;

namespace {

LocalityConfig quiet() {
    LocalityConfig cfg;
    cfg.profiler.capture.os_monitor = false;
    cfg.scheduler.worker_count = 1;
    return cfg;
}

// Hand-built uniform mesh from explicit neighbour/owner tables (the shape the
// reference's own tests build, test_workload.cpp:38-54).
Mesh make_mesh(std::int64_t n, const std::int64_t* nbr, const std::int32_t* pos,
               const std::int32_t* owner, int world) {
    Mesh mesh;
    mesh.levels = 1;
    mesh.world_size = world;
    for (std::int64_t i = 0; i < n; ++i) {
        SubGrid g;
        g.grid_id = static_cast<std::uint64_t>(i);
        g.level = 0;
        g.pos = {pos[3 * i], pos[3 * i + 1], pos[3 * i + 2]};
        g.owner = owner[i];
        for (int f = 0; f < kFaceCount; ++f) g.neighbor_ids[f] = nbr[6 * i + f];
        mesh.grids.push_back(std::move(g));
    }
    mesh.finalize();
    return mesh;
}

}  // namespace

extern "C" {

std::uint64_t ref_mix64(std::uint64_t x) { return mix64(x); }
std::uint64_t ref_mix64_2(std::uint64_t a, std::uint64_t b) { return mix64(a, b); }
double ref_cell_value(std::uint64_t g, std::uint64_t s, std::uint64_t i) { return cell_value(g, s, i); }
std::uint64_t ref_face_cell_index(int edge, int face, std::uint64_t j) {
    return face_cell_index(edge, face, j);
}

// build_mesh (workload.cpp:264-327): counts, then owner / level / pos / nbr tables.
std::int64_t ref_build_mesh(int levels, int world, std::uint64_t seed, std::int32_t* owner,
                            std::int32_t* level, std::int32_t* pos, std::int64_t* nbr,
                            std::int64_t cap) {
    try {
        Mesh m = build_mesh(levels, world, seed);
        const auto n = static_cast<std::int64_t>(m.grids.size());
        if (owner != nullptr && n <= cap) {
            for (std::int64_t i = 0; i < n; ++i) {
                const SubGrid& g = m.grids[static_cast<std::size_t>(i)];
                owner[i] = g.owner;
                level[i] = g.level;
                for (int d = 0; d < 3; ++d) pos[3 * i + d] = g.pos[d];
                for (int f = 0; f < 6; ++f) nbr[6 * i + f] = g.neighbor_ids[f];
            }
        }
        return n;
    } catch (const std::exception&) {
        return -1;
    }
}

// gravity_kernel_name (workload.cpp:365-372) of every grid of build_mesh's
// octree: 0 multipole_root_kernel, 1 multipole_kernel, 2 p2m_kernel, 3 p2p_kernel.
std::int64_t ref_gravity_kinds(int levels, int world, std::uint64_t seed, std::int32_t* kind, std::int64_t cap) {
    try {
        Mesh m = build_mesh(levels, world, seed);
        const auto n = static_cast<std::int64_t>(m.grids.size());
        if (kind != nullptr && n <= cap)
            for (std::int64_t i = 0; i < n; ++i) {
                const std::string k = gravity_kernel_name(m, m.grids[static_cast<std::size_t>(i)]);
                kind[i] = k == kKernelMultipoleRoot ? 0 : k == kKernelMultipole ? 1 : k == kKernelP2M ? 2 : 3;
            }
        return n;
    } catch (const std::exception&) {
        return -1;
    }
}

// One reference ghost exchange round at `step` (workload.cpp:572-581) on a
// hand-built mesh; ghosts out as [g][6][N*N] (0 where no neighbour) and the
// number of ghost parcels the transport carried.
int ref_exchange_ghosts(std::int64_t n, const std::int64_t* nbr, const std::int32_t* pos,
                        const std::int32_t* owner, int world, int direct_local, std::uint64_t step,
                        double* ghost, std::uint64_t* parcels) {
    try {
        Mesh mesh = make_mesh(n, nbr, pos, owner, world);
        auto w = World::create_inproc(world, quiet());
        exchange_ghost_cells(mesh, *w, direct_local ? CommMode::direct_local : CommMode::remote_action,
                             step);
        for (std::int64_t i = 0; i < n; ++i)
            for (int f = 0; f < 6; ++f) {
                const auto& layer = mesh.grids[static_cast<std::size_t>(i)].ghost[f];
                double* out = ghost + (i * 6 + f) * 64;
                if (layer.empty())
                    std::memset(out, 0, 64 * sizeof(double));
                else
                    std::memcpy(out, layer.data(), 64 * sizeof(double));
            }
        std::uint64_t sent = 0;
        for (LocalityId r = 0; r < w->size(); ++r) {
            const MessageStats stats = w->locality(r).message_stats();
            const auto it = stats.parcels_sent.find(kActionSetHydroBoundary);
            if (it != stats.parcels_sent.end()) sent += it->second;
        }
        *parcels = sent;
        return 0;
    } catch (const std::exception&) {
        return -1;
    }
}

// Reference cells (cell_value at step) of a hand-built mesh, [g][512].
void ref_fill_cells(std::int64_t n, std::uint64_t step, double* out) {
    for (std::int64_t i = 0; i < n; ++i) {
        SubGrid g;
        g.grid_id = static_cast<std::uint64_t>(i);
        fill_cells(g, step);
        std::memcpy(out + i * 512, g.cells.data(), 512 * sizeof(double));
    }
}

}  // extern "C"
