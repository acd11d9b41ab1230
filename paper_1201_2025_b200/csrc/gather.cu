// NCCL score-map gather of the row-strip sharding (north_star: "NCCL is used
// only for the final score-map gather"). Rank g owns output rows [r0_g, r1_g) of every
// map (hsad_strip_plan: quantum-aligned strips); hsad_gather_maps moves each rank's strip
// of each map into the root's full-image map with one grouped ncclSend / ncclRecv per
// (rank, map): NCCL has no gather primitive, and the strips are contiguous row blocks of
// the full map, so the root receives straight into place — no padding, no staging copy.
// The analogue of the reference's worker join (proj/core/src/parallel.hpp:17-40) across
// GPUs.
//
// NCCL is resolved at run time (dlopen "libnccl.so.2": the copy a host process already
// loaded, e.g. torch's, or the system one), so the library has no link-time NCCL
// dependency and a process that never gathers never loads it.
#include <dlfcn.h>

#include <cstdint>
#include <cstring>
#include <type_traits>
#include <mutex>
#include <string>

#include "hsad_internal.h"

namespace hsad_b200 {
namespace {

// the slice of nccl.h this file uses (ABI-stable across NCCL 2.x)
typedef int nccl_result;
typedef void* nccl_comm;
struct nccl_unique_id {
    char internal[128];
};
constexpr int kNcclInt8 = 0;

struct Nccl {
    nccl_result (*send)(const void*, size_t, int, int, nccl_comm, cudaStream_t) = nullptr;
    nccl_result (*recv)(void*, size_t, int, int, nccl_comm, cudaStream_t) = nullptr;
    nccl_result (*group_start)() = nullptr;
    nccl_result (*group_end)() = nullptr;
    nccl_result (*get_unique_id)(nccl_unique_id*) = nullptr;
    nccl_result (*comm_init_rank)(nccl_comm*, int, nccl_unique_id, int) = nullptr;
    nccl_result (*comm_init_all)(nccl_comm*, int, const int*) = nullptr;
    nccl_result (*comm_destroy)(nccl_comm) = nullptr;
    const char* (*error_string)(nccl_result) = nullptr;
    bool ok = false;
};

const Nccl& nccl() {
    static Nccl n;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) return;
        auto sym = [&](auto& fn, const char* name) {
            fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name));
            return fn != nullptr;
        };
        n.ok = sym(n.send, "ncclSend") && sym(n.recv, "ncclRecv") && sym(n.group_start, "ncclGroupStart") &&
               sym(n.group_end, "ncclGroupEnd") && sym(n.get_unique_id, "ncclGetUniqueId") &&
               sym(n.comm_init_rank, "ncclCommInitRank") && sym(n.comm_init_all, "ncclCommInitAll") &&
               sym(n.comm_destroy, "ncclCommDestroy") && sym(n.error_string, "ncclGetErrorString");
    });
    return n;
}

hsad_status nccl_fail(const Nccl& n, nccl_result r, const char* what) {
    return set_error(HSAD_E_NCCL, std::string(what) + " failed: " + (n.error_string ? n.error_string(r) : "?"));
}

#define HSAD_NCCL_TRY(n, expr, what)                  \
    do {                                              \
        nccl_result r__ = (expr);                     \
        if (r__ != 0) return nccl_fail(n, r__, what); \
    } while (0)

}  // namespace
}  // namespace hsad_b200

using namespace hsad_b200;

extern "C" {

hsad_status hsad_nccl_available(void) {
    return nccl().ok ? HSAD_OK : set_error(HSAD_E_NCCL, "libnccl.so.2 not found");
}

hsad_status hsad_nccl_unique_id(uint8_t* id128) {
    const Nccl& n = nccl();
    if (!n.ok) return set_error(HSAD_E_NCCL, "libnccl.so.2 not found");
    if (!id128) return set_error(HSAD_E_INVALID_VALUE, "null id buffer");
    nccl_unique_id id;
    HSAD_NCCL_TRY(n, n.get_unique_id(&id), "ncclGetUniqueId");
    std::memcpy(id128, id.internal, sizeof(id.internal));
    return HSAD_OK;
}

hsad_status hsad_nccl_comm_init_rank(void** comm, int32_t world, const uint8_t* id128, int32_t rank) {
    const Nccl& n = nccl();
    if (!n.ok) return set_error(HSAD_E_NCCL, "libnccl.so.2 not found");
    if (!comm || !id128 || world < 1 || rank < 0 || rank >= world)
        return set_error(HSAD_E_INVALID_VALUE, "bad communicator arguments");
    nccl_unique_id id;
    std::memcpy(id.internal, id128, sizeof(id.internal));
    HSAD_NCCL_TRY(n, n.comm_init_rank(comm, world, id, rank), "ncclCommInitRank");
    return HSAD_OK;
}

hsad_status hsad_nccl_comm_init_all(void** comms, int32_t ndev) {
    const Nccl& n = nccl();
    if (!n.ok) return set_error(HSAD_E_NCCL, "libnccl.so.2 not found");
    if (!comms || ndev < 1) return set_error(HSAD_E_INVALID_VALUE, "bad communicator arguments");
    HSAD_NCCL_TRY(n, n.comm_init_all(comms, ndev, nullptr), "ncclCommInitAll");
    return HSAD_OK;
}

hsad_status hsad_nccl_comm_destroy(void* comm) {
    const Nccl& n = nccl();
    if (!n.ok) return set_error(HSAD_E_NCCL, "libnccl.so.2 not found");
    if (comm) HSAD_NCCL_TRY(n, n.comm_destroy(comm), "ncclCommDestroy");
    return HSAD_OK;
}

hsad_status hsad_gather_maps(void* nccl_comm, int32_t world, int32_t rank, int32_t root, int64_t lines,
                             int64_t samples, const hsad_map_desc* maps, int32_t n_maps, void* stream) {
    if (world < 1 || rank < 0 || rank >= world || root < 0 || root >= world)
        return set_error(HSAD_E_INVALID_VALUE, "rank / root outside [0, world)");
    if (n_maps < 0 || (n_maps > 0 && !maps)) return set_error(HSAD_E_INVALID_VALUE, "bad map list");
    for (int m = 0; m < n_maps; ++m) {
        const int eb = maps[m].elem_bytes;
        if (eb != 1 && eb != 4 && eb != 8) return set_error(HSAD_E_INVALID_VALUE, "elem_bytes must be 1, 4 or 8");
        if (rank == root && !maps[m].d_full) return set_error(HSAD_E_INVALID_VALUE, "root needs full maps");
    }
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    int64_t r0 = 0, r1 = 0;
    hsad_status st = hsad_strip_plan(lines, samples, world, rank, &r0, &r1, nullptr);
    if (st != HSAD_OK) return st;
    const size_t row_px = static_cast<size_t>(samples);
    // the root's own strip: a device copy into place (skipped when it already is)
    if (rank == root)
        for (int m = 0; m < n_maps; ++m) {
            const size_t eb = static_cast<size_t>(maps[m].elem_bytes);
            char* dst = static_cast<char*>(maps[m].d_full) + static_cast<size_t>(r0) * row_px * eb;
            if (r1 > r0 && dst != maps[m].d_strip)
                HSAD_CUDA_TRY(cudaMemcpyAsync(dst, maps[m].d_strip, static_cast<size_t>(r1 - r0) * row_px * eb,
                                              cudaMemcpyDeviceToDevice, s));
        }
    if (world == 1 || n_maps == 0) return HSAD_OK;
    const Nccl& n = nccl();
    if (!n.ok) return set_error(HSAD_E_NCCL, "libnccl.so.2 not found");
    if (!nccl_comm) return set_error(HSAD_E_INVALID_VALUE, "null NCCL communicator");
    HSAD_NCCL_TRY(n, n.group_start(), "ncclGroupStart");
    if (rank == root) {
        for (int g = 0; g < world; ++g) {
            if (g == root) continue;
            int64_t a = 0, b = 0;
            hsad_strip_plan(lines, samples, world, g, &a, &b, nullptr);
            if (b <= a) continue;
            for (int m = 0; m < n_maps; ++m) {
                const size_t eb = static_cast<size_t>(maps[m].elem_bytes);
                char* dst = static_cast<char*>(maps[m].d_full) + static_cast<size_t>(a) * row_px * eb;
                const nccl_result r = n.recv(dst, static_cast<size_t>(b - a) * row_px * eb, kNcclInt8, g,
                                             nccl_comm, s);
                if (r != 0) {
                    n.group_end();
                    return nccl_fail(n, r, "ncclRecv");
                }
            }
        }
    } else if (r1 > r0) {
        for (int m = 0; m < n_maps; ++m) {
            const size_t eb = static_cast<size_t>(maps[m].elem_bytes);
            const nccl_result r = n.send(maps[m].d_strip, static_cast<size_t>(r1 - r0) * row_px * eb, kNcclInt8,
                                         root, nccl_comm, s);
            if (r != 0) {
                n.group_end();
                return nccl_fail(n, r, "ncclSend");
            }
        }
    }
    HSAD_NCCL_TRY(n, n.group_end(), "ncclGroupEnd");
    return HSAD_OK;
}

}  // extern "C"
