// ts_hydro_ckpt.cpp — persisted state format: an FP64
// field dump plus the mesh, for restart and for offline parity checks of GPU
// runs against the oracle without re-running the CPU path.
//
// The reference persists only profiles (its codec, reference
// proj/core/src/codec.cpp:17-225: a magic/version header, then length-checked
// sections); this file follows the same pattern for the hydro state.  Layout
// (little-endian, no padding between sections):
//
//   header, kHeaderBytes = 128 bytes:
//     0   char[8]  magic "TSHYDRO\0"
//     8   u32      version (1)
//     12  u32      header bytes (128)
//     16  i32      nf, n_species, recon, cells_per_edge (8)
//     32  f64      gamma, cfl, dx, p_floor
//     64  i64      n_grids (global mesh), n_records (sub-grids in this file)
//     80  u64      steps_done
//     88  i32      world, rank (of the writer)
//     96  u64      FNV-1a 64 checksum of the payload
//     104 zero padding
//   payload:
//     i64 neighbor_ids[n_grids][6]   (face order -x,+x,-y,+y,-z,+z; -1 = none)
//     i32 owner[n_grids]
//     i64 global_id[n_records]
//     f64 state[n_records][nf][8][8][8]  (x fastest, workload.cpp:353)
//
// A restart may use a different rank count: every rank reads all files of a
// checkpoint and keeps the records of the sub-grids it owns (ts_hydro_restore).
#include <cstdio>
#include <cstring>
#include <vector>

#include "ts_hydro.h"

namespace {

constexpr char kMagic[8] = {'T', 'S', 'H', 'Y', 'D', 'R', 'O', '\0'};
constexpr uint32_t kVersion = 1;
constexpr uint32_t kHeaderBytes = 128;
constexpr int kCells = 512;

struct Fnv {
    uint64_t h = 0xcbf29ce484222325ull;
    void add(const void* p, size_t n) {
        const unsigned char* b = static_cast<const unsigned char*>(p);
        for (size_t i = 0; i < n; ++i) {
            h ^= b[i];
            h *= 0x100000001b3ull;
        }
    }
};

template <typename T>
void put(unsigned char* buf, size_t off, T v) {
    std::memcpy(buf + off, &v, sizeof(T));
}
template <typename T>
T get(const unsigned char* buf, size_t off) {
    T v;
    std::memcpy(&v, buf + off, sizeof(T));
    return v;
}

struct File {
    FILE* f = nullptr;
    explicit File(FILE* p) : f(p) {}
    ~File() {
        if (f != nullptr) std::fclose(f);
    }
};

size_t payload_bytes(const ts_hydro_checkpoint_header& h) {
    return (size_t)h.n_grids * 6 * 8 + (size_t)h.n_grids * 4 + (size_t)h.n_records * 8 +
           (size_t)h.n_records * (size_t)h.nf * kCells * 8;
}

int read_header(FILE* f, ts_hydro_checkpoint_header* h) {
    unsigned char buf[kHeaderBytes];
    if (std::fread(buf, 1, kHeaderBytes, f) != kHeaderBytes) return TS_EINVAL;
    if (std::memcmp(buf, kMagic, 8) != 0) return TS_EINVAL;
    h->version = get<uint32_t>(buf, 8);
    if (h->version != kVersion || get<uint32_t>(buf, 12) != kHeaderBytes) return TS_EINVAL;
    h->nf = get<int32_t>(buf, 16);
    h->n_species = get<int32_t>(buf, 20);
    h->recon = get<int32_t>(buf, 24);
    h->cells_per_edge = get<int32_t>(buf, 28);
    h->gamma = get<double>(buf, 32);
    h->cfl = get<double>(buf, 40);
    h->dx = get<double>(buf, 48);
    h->p_floor = get<double>(buf, 56);
    h->n_grids = get<int64_t>(buf, 64);
    h->n_records = get<int64_t>(buf, 72);
    h->steps_done = get<uint64_t>(buf, 80);
    h->world = get<int32_t>(buf, 88);
    h->rank = get<int32_t>(buf, 92);
    h->checksum = get<uint64_t>(buf, 96);
    if (h->nf != 6 + h->n_species || h->nf < 6 || h->nf > 11 || h->cells_per_edge != 8 || h->n_grids < 1 ||
        h->n_records < 0 || h->n_records > h->n_grids)
        return TS_EINVAL;
    return TS_OK;
}

}  // namespace

extern "C" {

int ts_hydro_checkpoint_write(const char* path, const ts_hydro_config* cfg, int64_t n_grids,
                              const int64_t* neighbor_ids, const int32_t* owner, int32_t world, int32_t rank,
                              int64_t n_records, const int64_t* global_ids, const double* state,
                              uint64_t steps_done) {
    if (path == nullptr || cfg == nullptr || n_grids < 1 || neighbor_ids == nullptr || owner == nullptr ||
        n_records < 0 || n_records > n_grids || (n_records > 0 && (global_ids == nullptr || state == nullptr)) ||
        cfg->n_species < 0 || cfg->n_species > 5)
        return TS_EINVAL;
    for (int64_t i = 0; i < n_records; ++i)
        if (global_ids[i] < 0 || global_ids[i] >= n_grids) return TS_EINVAL;
    const int32_t nf = 6 + cfg->n_species;
    const size_t state_bytes = (size_t)n_records * (size_t)nf * kCells * sizeof(double);
    Fnv fnv;
    fnv.add(neighbor_ids, (size_t)n_grids * 6 * sizeof(int64_t));
    fnv.add(owner, (size_t)n_grids * sizeof(int32_t));
    if (n_records > 0) {
        fnv.add(global_ids, (size_t)n_records * sizeof(int64_t));
        fnv.add(state, state_bytes);
    }
    unsigned char hdr[kHeaderBytes] = {};
    std::memcpy(hdr, kMagic, 8);
    put<uint32_t>(hdr, 8, kVersion);
    put<uint32_t>(hdr, 12, kHeaderBytes);
    put<int32_t>(hdr, 16, nf);
    put<int32_t>(hdr, 20, cfg->n_species);
    put<int32_t>(hdr, 24, cfg->recon);
    put<int32_t>(hdr, 28, 8);
    put<double>(hdr, 32, cfg->gamma);
    put<double>(hdr, 40, cfg->cfl);
    put<double>(hdr, 48, cfg->dx);
    put<double>(hdr, 56, cfg->p_floor);
    put<int64_t>(hdr, 64, n_grids);
    put<int64_t>(hdr, 72, n_records);
    put<uint64_t>(hdr, 80, steps_done);
    put<int32_t>(hdr, 88, world);
    put<int32_t>(hdr, 92, rank);
    put<uint64_t>(hdr, 96, fnv.h);
    File f(std::fopen(path, "wb"));
    if (f.f == nullptr) return TS_EINVAL;
    bool ok = std::fwrite(hdr, 1, kHeaderBytes, f.f) == kHeaderBytes;
    ok = ok && std::fwrite(neighbor_ids, sizeof(int64_t), (size_t)n_grids * 6, f.f) == (size_t)n_grids * 6;
    ok = ok && std::fwrite(owner, sizeof(int32_t), (size_t)n_grids, f.f) == (size_t)n_grids;
    if (n_records > 0) {
        ok = ok && std::fwrite(global_ids, sizeof(int64_t), (size_t)n_records, f.f) == (size_t)n_records;
        ok = ok && std::fwrite(state, 1, state_bytes, f.f) == state_bytes;
    }
    ok = ok && std::fflush(f.f) == 0;
    return ok ? TS_OK : TS_EINVAL;
}

int ts_hydro_checkpoint_info(const char* path, ts_hydro_checkpoint_header* out) {
    if (path == nullptr || out == nullptr) return TS_EINVAL;
    File f(std::fopen(path, "rb"));
    if (f.f == nullptr) return TS_EINVAL;
    ts_hydro_checkpoint_header h{};
    int rc = read_header(f.f, &h);
    if (rc) return rc;
    // size and checksum of the payload
    Fnv fnv;
    std::vector<unsigned char> buf(1 << 20);
    size_t left = payload_bytes(h), got;
    while (left > 0 && (got = std::fread(buf.data(), 1, left < buf.size() ? left : buf.size(), f.f)) > 0) {
        fnv.add(buf.data(), got);
        left -= got;
    }
    if (left != 0 || std::fgetc(f.f) != EOF) return TS_EINVAL;  // truncated or trailing bytes
    if (fnv.h != h.checksum) return TS_EINVAL;
    *out = h;
    return TS_OK;
}

int ts_hydro_checkpoint_read(const char* path, int64_t* neighbor_ids, int32_t* owner, int64_t* global_ids,
                             double* state) {
    ts_hydro_checkpoint_header h{};
    int rc = ts_hydro_checkpoint_info(path, &h);  // validates size and checksum first
    if (rc) return rc;
    File f(std::fopen(path, "rb"));
    if (f.f == nullptr || std::fseek(f.f, kHeaderBytes, SEEK_SET) != 0) return TS_EINVAL;
    auto section = [&](void* dst, size_t bytes) {
        if (dst != nullptr) return std::fread(dst, 1, bytes, f.f) == bytes;
        return std::fseek(f.f, (long)bytes, SEEK_CUR) == 0;
    };
    bool ok = section(neighbor_ids, (size_t)h.n_grids * 6 * 8);
    ok = ok && section(owner, (size_t)h.n_grids * 4);
    ok = ok && section(global_ids, (size_t)h.n_records * 8);
    ok = ok && section(state, (size_t)h.n_records * (size_t)h.nf * kCells * 8);
    return ok ? TS_OK : TS_EINVAL;
}

}  // extern "C"
