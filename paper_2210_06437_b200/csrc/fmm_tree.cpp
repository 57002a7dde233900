// fmm_tree.cpp — host side of the gravity FMM (fmm.h): the octree of 8^3
// sub-grids built from the leaves, its neighbour slots and the interaction
// tables.  The reference's octree (TreeBuilder / build_mesh,
// proj/core/src/workload.cpp:199-327) keeps refined parents as sub-grids
// with `has_children`; here the hydro leaves come in and the refined nodes
// are their ancestors — the same tree.
#include <algorithm>
#include <cmath>
#include <unordered_map>

#include "fmm.h"

namespace tsh {

namespace {

uint64_t key(int d, int x, int y, int z) {
    return ((uint64_t)d << 60) | ((uint64_t)z << 40) | ((uint64_t)y << 20) | (uint64_t)x;
}

}  // namespace

std::string fmm_build_tree(int64_t n_leaves, const int32_t* level, const int32_t* pos, const int32_t* dims,
                           double dx0, FmmTree& t) {
    t = FmmTree{};
    if (n_leaves <= 0) return "no leaves";
    if (!(dx0 > 0.0)) return "dx0 must be positive";
    for (int a = 0; a < 3; ++a)
        if (dims[a] < 1 || dims[a] > (1 << 16)) return "dims must be 1..65536";
    const int mx = std::max(dims[0], std::max(dims[1], dims[2]));
    while ((1 << t.T) < mx) ++t.T;
    t.dx0 = dx0;
    struct Tmp {
        int d, x, y, z;
        int leaf;
    };
    std::unordered_map<uint64_t, int> idx;  // key -> tmp index
    std::vector<Tmp> tmp;
    tmp.reserve((size_t)n_leaves * 2);
    for (int64_t k = 0; k < n_leaves; ++k) {
        const int l = level[k];
        if (l < 0 || l > 16) return "leaf levels must be 0..16";
        for (int a = 0; a < 3; ++a)  // node keys hold 20 bits per coordinate
            if (((int64_t)dims[a] << l) > (1 << 20)) return "more than 2^20 sub-grids along an axis at some level";
        for (int a = 0; a < 3; ++a)
            if (pos[3 * k + a] < 0 || (int64_t)pos[3 * k + a] >= ((int64_t)dims[a] << l))
                return "leaf " + std::to_string(k) + " lies outside the domain";
        const int d = l + t.T;
        for (int e = d; e >= 0; --e) {
            const int s = d - e;
            const uint64_t kk = key(e, pos[3 * k] >> s, pos[3 * k + 1] >> s, pos[3 * k + 2] >> s);
            auto it = idx.find(kk);
            if (it == idx.end()) {
                idx.emplace(kk, (int)tmp.size());
                tmp.push_back({e, pos[3 * k] >> s, pos[3 * k + 1] >> s, pos[3 * k + 2] >> s, e == d ? (int)k : -1});
            } else if (e == d) {
                if (tmp[(size_t)it->second].leaf >= 0) return "leaf " + std::to_string(k) + " is listed twice";
                tmp[(size_t)it->second].leaf = (int)k;
            }
        }
    }
    // a leaf that is also an ancestor of another leaf: overlapping leaves
    for (const Tmp& n : tmp)
        if (n.leaf >= 0) {
            for (int c = 0; c < 8; ++c)
                if (idx.count(key(n.d + 1, 2 * n.x + (c & 1), 2 * n.y + ((c >> 1) & 1), 2 * n.z + (c >> 2))))
                    return "leaf " + std::to_string(n.leaf) + " overlaps finer leaves";
        }
    // order: refined nodes by depth (ids 0 .. n_int - 1, the rows of L), then
    // the leaves by depth; inside a depth by key
    std::vector<int> ord(tmp.size());
    for (size_t i = 0; i < ord.size(); ++i) ord[i] = (int)i;
    std::sort(ord.begin(), ord.end(), [&](int a, int b) {
        const Tmp &A = tmp[(size_t)a], &B = tmp[(size_t)b];
        if ((A.leaf >= 0) != (B.leaf >= 0)) return A.leaf < 0;
        return key(A.d, A.x, A.y, A.z) < key(B.d, B.x, B.y, B.z);
    });
    const int n = (int)ord.size();
    std::unordered_map<uint64_t, int> id;  // key -> node id
    t.depth.resize(n);
    t.q.resize(3 * (size_t)n);
    t.leaf.resize(n);
    t.parent.assign(n, -1);
    t.child.assign(8 * (size_t)n, -1);
    t.nb27.assign(27 * (size_t)n, kFmmNone);
    t.kind.assign(n, 3);
    for (int i = 0; i < n; ++i) {
        const Tmp& m = tmp[(size_t)ord[(size_t)i]];
        t.depth[i] = m.d;
        t.q[3 * i] = m.x;
        t.q[3 * i + 1] = m.y;
        t.q[3 * i + 2] = m.z;
        t.leaf[i] = m.leaf;
        id.emplace(key(m.d, m.x, m.y, m.z), i);
        t.max_depth = std::max(t.max_depth, m.d);
    }
    auto find = [&](int d, int x, int y, int z) -> int {
        if (x < 0 || y < 0 || z < 0) return -1;
        auto it = id.find(key(d, x, y, z));
        return it == id.end() ? -1 : it->second;
    };
    t.int_first.assign((size_t)t.max_depth + 2, 0);
    t.n_int.assign((size_t)t.max_depth + 1, 0);
    for (int i = n - 1; i >= 0; --i)
        if (t.leaf[i] < 0) t.int_first[(size_t)t.depth[i]] = i;
    for (int i = 0; i < n; ++i) {
        const int d = t.depth[i], x = t.q[3 * i], y = t.q[3 * i + 1], z = t.q[3 * i + 2];
        if (t.leaf[i] < 0) ++t.n_int[(size_t)d];
        if (d > 0) {
            const int p = find(d - 1, x >> 1, y >> 1, z >> 1);
            t.parent[i] = p;
            t.child[8 * (size_t)p + ((x & 1) | ((y & 1) << 1) | ((z & 1) << 2))] = i;
        }
        bool refined_nb = false, refined_face = false;
        for (int s = 0; s < 27; ++s) {
            const int X = x + s % 3 - 1, Y = y + (s / 3) % 3 - 1, Z = z + s / 9 - 1;
            int code = kFmmNone;
            const int h = find(d, X, Y, Z);
            if (h >= 0) {
                code = h;
                refined_nb |= t.leaf[h] < 0;
                // the six face slots: gravity_kernel_name's neighbor_ids (workload.cpp:368-370)
                if (s == 4 || s == 10 || s == 12 || s == 14 || s == 16 || s == 22) refined_face |= t.leaf[h] < 0;
            } else if (X >= 0 && Y >= 0 && Z >= 0) {
                for (int e = d - 1; e >= 0; --e) {
                    const int c = find(e, X >> (d - e), Y >> (d - e), Z >> (d - e));
                    if (c < 0) continue;
                    if (t.leaf[c] >= 0) code = -2 - c;
                    break;
                }
            }
            t.nb27[27 * (size_t)i + s] = code;
        }
        t.kind[i] = d == 0 ? 0 : (t.leaf[i] < 0 ? 1 : (refined_face ? 2 : 3));
        if (t.leaf[i] >= 0) {
            if (d == 0) t.root_leaf = i;
            else if (refined_face) t.leaves_p2m.push_back(i);
            else (refined_nb ? t.leaves_p2p_restr : t.leaves_p2p).push_back(i);
        }
    }
    for (int i = 0; i < n; ++i) t.n_internal += t.leaf[i] < 0;
    return "";
}

std::vector<FmmEntry> fmm_table(int radius, bool root, bool far_only) {
    std::vector<FmmEntry> v;
    const int K = root ? kFmmRootK : 2 * radius + 1, R2 = radius * radius;
    for (int z = -K; z <= K; ++z)
        for (int y = -K; y <= K; ++y)
            for (int x = -K; x <= K; ++x) {
                if (x == 0 && y == 0 && z == 0) continue;
                if (!root) {
                    const int px = x >> 1, py = y >> 1, pz = z >> 1;
                    if (px * px + py * py + pz * pz > R2) continue;
                }
                const int r2 = x * x + y * y + z * z;
                if (far_only && r2 <= R2) continue;
                FmmEntry e{};
                e.u[0] = x;
                e.u[1] = y;
                e.u[2] = z;
                e.r2 = r2;
                const double c0 = 1.0 / std::sqrt((double)r2);
                const double c3 = c0 / (double)r2;
                e.c[0] = c0;
                e.c[1] = (double)x * c3;
                e.c[2] = (double)y * c3;
                e.c[3] = (double)z * c3;
                v.push_back(e);
            }
    return v;
}

}  // namespace tsh
