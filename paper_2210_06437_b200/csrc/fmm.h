// fmm.h — gravity, the whole solve: a cell-based
// fast multipole method over the octree of 8^3 sub-grids.  The reference
// schedules gravity as six launches per sub-grid and step of the kernel
// `gravity_kernel_name` picks (proj/core/src/workload.cpp:365-372, 565-569):
// multipole_root_kernel, multipole_kernel, p2m_kernel, p2p_kernel — timed
// sleeps there.  Numerics contract: DESIGN.md §15 and oracle/fmm_oracle.c
// (bitwise: same operations in the same order, --fmad=false).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

namespace tsh {

constexpr int kFmmRMax = 3;         // interaction radius R (cells) 1..3: reach 2R+1 <= 7 < 8
constexpr int kFmmRootK = 7;        // the root's table spans [-7, 7]^3
constexpr int kFmmChunk = 64;       // a refined node's far sum: chunk sums of 64 entries (ORC_FMM_CHUNK)
constexpr int kFmmSplitMax = 4096;  // (node, chunk) partial sums of one split M2L launch (scratch rows, 168 MB)
constexpr int kFmmNone = -1;        // nb27 code: no source (outside the domain)
// nb27 code <= -2: the slot lies inside a coarser leaf, node id = -2 - code

// One interaction table entry, octant-0 orientation: offset u, |u|^2, and
// (1/|u|, u_x/|u|^3, u_y/|u|^3, u_z/|u|^3) computed with IEEE sqrt / division.
struct FmmEntry {
    int u[3];
    int r2;
    double c[4];
};

// Host tree (fmm_tree.cpp): the refined nodes first (ids 0 .. n_internal - 1,
// by depth: the rows of the expansion array), then the leaves by depth.
struct FmmTree {
    int T = 0;        // virtual depths above hydro level 0
    int max_depth = 0;
    double dx0 = 0.0;  // level-0 cell width; h_d = dx0 2^(T - d)
    std::vector<int> depth, q, leaf, parent, child, nb27;  // q [n][3], child [n][8], nb27 [n][27]
    std::vector<int> int_first;   // refined nodes of depth d = [int_first[d], int_first[d] + n_int[d])
    std::vector<int> n_int;
    int n_internal = 0;
    // gravity_kernel_name's kinds (workload.cpp:365-372): 0 multipole_root_kernel
    // (depth 0), 1 multipole_kernel (refined), 2 p2m_kernel (a leaf with a
    // refined same-depth face neighbour), 3 p2p_kernel (other leaves)
    std::vector<int> kind;
    // leaf node ids at depth >= 1: p2p kind with no refined node among the 26
    // neighbour slots; p2p kind with one across an edge or corner (the leaf
    // kernel then reads refined moments too); p2m kind
    std::vector<int> leaves_p2p, leaves_p2p_restr, leaves_p2m;
    int root_leaf = -1;           // node 0 when the root itself is a leaf (one sub-grid)
    int n() const { return (int)depth.size(); }
};

// Builds the tree from the leaves (hydro level, position at that level);
// returns "" or what is malformed.
std::string fmm_build_tree(int64_t n_leaves, const int32_t* level, const int32_t* pos, const int32_t* dims,
                           double dx0, FmmTree& t);
// Interaction table of radius R (root: the depth-0 table); `far_only` drops
// the near entries (|u|^2 <= R^2).  Same order as orc_fmm_table.
std::vector<FmmEntry> fmm_table(int radius, bool root, bool far_only);

struct FmmArgs {
    const double* U;     // densities: field 0 of row leaf[node] at U + leaf nf 512 (the state, or the
                         // ranks' gathered densities with nf = 1)
    int nf;
    const int* depth;    // device copies of FmmTree's arrays
    const int* q;
    const int* leaf;
    const int* parent;
    const int* child;
    const int* nb27;
    const int* leaf_out;  // a leaf node's output row (owned index), -1 for a leaf another rank owns
    double* M;           // [n][4][512] moments (m, cx, cy, cz)
    double* L;           // [n_internal][10][512] local expansions (phi, g, T xx yy zz xy xz yz)
    double* out;         // [leaf sub-grid][4][512] (phi, gx, gy, gz)
    double* part;        // [kFmmSplitMax][10][512] chunk sums of a split M2L launch
    const FmmEntry* table;
    int n_table;
    int K;               // table reach: tile half-width of the leaf kernel
    const int* list;     // node ids of the launch (list[first + block]); nullptr: first + block
    int first;
    int T;
    double dx0;
    double G;
    unsigned long long* stamp;
};

// Constant-bank tables and shared-memory opt-ins on the current device (once).
cudaError_t fmm_prepare_device();
cudaError_t launch_fmm_moments(const FmmArgs& a, int n_ctas, cudaStream_t s);   // P2M: leaf masses
cudaError_t launch_fmm_restrict(const FmmArgs& a, int n_ctas, cudaStream_t s);  // M2M: one depth of refined nodes
// L2L + M2L of refined nodes a.first .. + n_nodes - 1 (one depth): (chunk,
// node) CTAs + an in-order combine; n_nodes * chunks <= kFmmSplitMax
cudaError_t launch_fmm_m2l_split(const FmmArgs& a, int n_nodes, cudaStream_t s);
// The halves of launch_fmm_m2l_split for a merged solve: one part launch over
// the refined nodes of every depth (rows of a.part in launch order), then the
// per-depth combines in root-first order (a.part offset to the depth's rows).
cudaError_t launch_fmm_m2l_combine(const FmmArgs& a, int n_nodes, cudaStream_t s);
// One part launch for the root (root_node >= 0, its table; rows after the
// deeper ones) and n_nodes listed deeper nodes (a.table, a.list + a.first).
cudaError_t launch_fmm_m2l_part_flat(const FmmArgs& a, int n_nodes, int root_node, const FmmEntry* root_tab,
                                     int n_root_tab, cudaStream_t s);
cudaError_t launch_fmm_leaf(const FmmArgs& a, int n_ctas, bool restricted, cudaStream_t s);  // leaves: L2L + near + far

// Gravity source over dt on the first n sub-grids (dt_dev: the device's
// last-step dt, else dt).
cudaError_t launch_gravity_kick(double* U, int nf, long long n, const double* grav, const double* dt_dev, double dt,
                                unsigned long long* stamp, int sms, cudaStream_t s);

}  // namespace tsh
