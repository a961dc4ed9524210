// sharded.cu -- row-sharded decode over NCCL, behind the C ABI (SURVEY §8b
// "spqr_sharded_create(..., ncclComm_t) + spqr_sharded_matvec", §8e).
//
// One process per GPU.  Rank r of `world` holds the contiguous row band
// [a_r, b_r) of a layer (or of several layers stacked row-wise, e.g. q/k/v:
// the band is cut in the stacked row order, so the gathered y is [q; k; v]),
// aligned to lcm(32, beta2) rows so no cell or statistics group is split.
// spqr_sharded_matvec runs the band through spqr_matvec and all-gathers the y
// bands with ncclAllGather on the caller's stream: in place into y when the
// bands are equal and batch == 1 (every LLaMA shape at N <= 8), else through
// a padded slot per rank and one strided copy per rank.  This is the NCCL
// baseline the north star names; the fused P2P gather (gather.cu) is the
// B200-native alternative.
//
// NCCL is bound at run time (dlopen "libnccl.so.2": the process's already
// loaded NCCL, e.g. torch's, or the system one), so the library itself does
// not depend on NCCL unless these entry points are used.  There is no
// reference counterpart (the reference is single-process CPU code); the
// anchor is BASELINE north_star ("row-sharded ... with an NCCL all-gather of y
// over NVLink") and matvec, kernel.hpp:89-124, per band.
#include <dlfcn.h>
#include <nccl.h>

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <memory>
#include <mutex>
#include <numeric>
#include <string>
#include <vector>

#include "internal.hpp"
#include "spqr_cuda.h"

namespace {

struct NcclError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

struct NcclApi {
    ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
    ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
    ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*comm_count)(const ncclComm_t, int*) = nullptr;
    ncclResult_t (*comm_user_rank)(const ncclComm_t, int*) = nullptr;
    const char* (*error_string)(ncclResult_t) = nullptr;
};

const NcclApi& nccl() {
    static NcclApi api;
    static std::once_flag once;
    static std::string err;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            err = std::string("NCCL: cannot load libnccl.so.2: ") + dlerror();
            return;
        }
        auto sym = [&](auto& fn, const char* name) {
            fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name));
            if (!fn && err.empty()) err = std::string("NCCL: missing symbol ") + name;
        };
        sym(api.get_unique_id, "ncclGetUniqueId");
        sym(api.comm_init_rank, "ncclCommInitRank");
        sym(api.comm_destroy, "ncclCommDestroy");
        sym(api.all_gather, "ncclAllGather");
        sym(api.comm_count, "ncclCommCount");
        sym(api.comm_user_rank, "ncclCommUserRank");
        sym(api.error_string, "ncclGetErrorString");
    });
    if (!err.empty()) throw NcclError(err);
    return api;
}

void nck(ncclResult_t r, const char* what) {
    if (r != ncclSuccess) throw NcclError(std::string("NCCL: ") + what + ": " + nccl().error_string(r));
}
void cck(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw std::runtime_error(std::string("CUDA: ") + what + ": " + cudaGetErrorString(e));
}

// A status from another C-ABI call, passed through unchanged.
struct StatusError : std::runtime_error {
    int status;
    StatusError(int st) : std::runtime_error(spqr_last_error()), status(st) {}
};
void sck(int st) {
    if (st) throw StatusError(st);
}

template <class F>
int nguard(F&& f) {
    try {
        spqr::detail::set_last_error("");
        f();
        return SPQR_OK;
    } catch (const StatusError& e) {
        spqr::detail::set_last_error(e.what());
        return e.status;
    } catch (const NcclError& e) {
        spqr::detail::set_last_error(e.what());
        return SPQR_E_NCCL;
    } catch (const spqr::Error& e) {
        spqr::detail::set_last_error(e.what());
        return spqr::detail::status_of(e);
    } catch (const std::exception& e) {
        spqr::detail::set_last_error(e.what());
        return SPQR_E_CUDA;
    }
}

}  // namespace

struct spqr_sharded {
    ncclComm_t comm = nullptr;
    int rank = 0, world = 1, device = 0;
    std::uint32_t rows = 0, cols = 0;
    std::vector<std::uint32_t> edges;  // world + 1 band edges (stacked rows)
    spqr_layer* band = nullptr;
    float* slots = nullptr;            // [world][batch_cap x band_max] for ragged / batched gathers
    std::size_t slot_cap = 0;          // floats per rank slot
    std::mutex mu;
    ~spqr_sharded() {
        if (band) spqr_layer_destroy(band);
        if (slots) cudaFree(slots);
    }
};

extern "C" {

int spqr_row_bands(uint32_t rows, uint32_t beta2, int world, uint32_t* edges) {
    return nguard([&] {
        if (world < 1 || beta2 == 0) spqr::fail(spqr::Errc::config_invalid, "row bands: world and beta2 must be >= 1");
        // units of lcm(32, beta2) rows (no cell or statistics group is split),
        // band sizes differing by at most one unit, the last band ragged
        const std::uint32_t align = std::lcm<std::uint32_t>(32u, beta2);
        const std::uint32_t units = (rows + align - 1) / align;
        if (static_cast<std::uint32_t>(world) > units)
            spqr::fail(spqr::Errc::config_invalid, "row bands: more ranks than row units (a band would be empty)");
        edges[0] = 0;
        std::uint32_t u = 0;
        for (int k = 0; k < world; ++k) {
            u += units / world + (static_cast<std::uint32_t>(k) < units % world ? 1u : 0u);
            edges[k + 1] = std::min(rows, u * align);
        }
    });
}

int spqr_nccl_unique_id(uint8_t* id_out) {
    return nguard([&] {
        ncclUniqueId id;
        nck(nccl().get_unique_id(&id), "ncclGetUniqueId");
        static_assert(sizeof(id) == SPQR_NCCL_ID_BYTES, "ncclUniqueId size");
        std::memcpy(id_out, &id, sizeof(id));
    });
}

int spqr_nccl_comm_init(const uint8_t* id_in, int world, int rank, int device, void** comm_out) {
    *comm_out = nullptr;
    return nguard([&] {
        if (world < 1 || rank < 0 || rank >= world) spqr::fail(spqr::Errc::config_invalid, "nccl: bad rank / world");
        ncclUniqueId id;
        std::memcpy(&id, id_in, sizeof(id));
        cck(cudaSetDevice(device), "cudaSetDevice");
        ncclComm_t c = nullptr;
        nck(nccl().comm_init_rank(&c, world, id, rank), "ncclCommInitRank");
        *comm_out = c;
    });
}

int spqr_nccl_comm_destroy(void* comm) {
    return nguard([&] {
        if (comm) nck(nccl().comm_destroy(static_cast<ncclComm_t>(comm)), "ncclCommDestroy");
    });
}

int spqr_sharded_create(const uint8_t* const* streams, const size_t* sizes, int count, int rank, int world,
                        void* nccl_comm, const spqr_layer_opts* opts, spqr_sharded** out) {
    *out = nullptr;
    return nguard([&] {
        if (count < 1 || !streams || !sizes) spqr::fail(spqr::Errc::config_invalid, "sharded: no layers");
        if (!nccl_comm) spqr::fail(spqr::Errc::config_invalid, "sharded: no NCCL communicator");
        auto S = std::make_unique<spqr_sharded>();
        S->comm = static_cast<ncclComm_t>(nccl_comm);
        int n = 0, r = 0;
        nck(nccl().comm_count(S->comm, &n), "ncclCommCount");
        nck(nccl().comm_user_rank(S->comm, &r), "ncclCommUserRank");
        if (n != world || r != rank) spqr::fail(spqr::Errc::config_invalid, "sharded: rank / world differ from the communicator's");
        S->rank = rank;
        S->world = world;
        std::vector<spqr_layer_info> infos(count);
        std::vector<std::uint32_t> base(count + 1, 0);
        for (int i = 0; i < count; ++i) {
            sck(spqr_stream_validate(streams[i], sizes[i], &infos[i]));
            if (i > 0 && (infos[i].cols != infos[0].cols || infos[i].beta2 != infos[0].beta2))
                spqr::fail(spqr::Errc::shape_mismatch, "sharded: stacked layers differ in columns or groups");
            if (i + 1 < count && infos[i].rows % 32 != 0)
                spqr::fail(spqr::Errc::shape_mismatch, "sharded: rows of all but the last layer must be a multiple of 32");
            base[i + 1] = base[i] + infos[i].rows;
        }
        S->rows = base[count];
        S->cols = infos[0].cols;
        S->edges.assign(world + 1, 0);
        sck(spqr_row_bands(S->rows, infos[0].beta2, world, S->edges.data()));
        const std::uint32_t a = S->edges[rank], b = S->edges[rank + 1];
        // this rank's part of every member, sliced with spqr_stream_slice_rows
        std::vector<std::vector<std::uint8_t>> parts;
        for (int i = 0; i < count; ++i) {
            const std::uint32_t la = std::max(a, base[i]), lb = std::min(b, base[i + 1]);
            if (la >= lb) continue;
            if (la == base[i] && lb == base[i + 1] && world == 1) {
                parts.emplace_back(streams[i], streams[i] + sizes[i]);
                continue;
            }
            std::size_t len = 0;
            std::vector<std::uint8_t> buf(sizes[i] + 4096);
            sck(spqr_stream_slice_rows(streams[i], sizes[i], la - base[i], lb - base[i], buf.data(), buf.size(), &len));
            buf.resize(len);
            parts.push_back(std::move(buf));
        }
        spqr_layer_opts o{};
        o.device = -1;
        if (opts) o = *opts;
        o.row_begin = o.row_end = 0;
        if (parts.size() == 1) {
            sck(spqr_layer_create(parts[0].data(), parts[0].size(), &o, &S->band));
        } else {
            std::vector<const uint8_t*> ptrs;
            std::vector<size_t> lens;
            for (auto& p : parts) {
                ptrs.push_back(p.data());
                lens.push_back(p.size());
            }
            sck(spqr_layer_create_stacked(ptrs.data(), lens.data(), static_cast<int>(parts.size()), &o, &S->band));
        }
        spqr_layer_info bi;
        spqr_layer_get_info(S->band, &bi);
        S->device = bi.device;
        *out = S.release();
    });
}

int spqr_sharded_band(const spqr_sharded* s, uint32_t* rows, uint32_t* band_begin, uint32_t* band_end,
                      spqr_layer** band_layer) {
    if (rows) *rows = s->rows;
    if (band_begin) *band_begin = s->edges[s->rank];
    if (band_end) *band_end = s->edges[s->rank + 1];
    if (band_layer) *band_layer = s->band;
    return SPQR_OK;
}

int spqr_sharded_matvec(spqr_sharded* s, const void* x_dev, int x_dtype, float* y_dev, int batch, void* cuda_stream) {
    return nguard([&] {
        if (batch < 1) spqr::fail(spqr::Errc::shape_mismatch, "sharded: batch must be >= 1");
        std::lock_guard<std::mutex> lk(s->mu);  // the slots and the band layer's workspace
        auto st = static_cast<cudaStream_t>(cuda_stream);
        const std::uint32_t a = s->edges[s->rank];
        std::uint32_t mx = 0;
        bool equal = true;
        for (int k = 0; k < s->world; ++k) {
            const std::uint32_t w = s->edges[k + 1] - s->edges[k];
            if (k && w != mx) equal = false;
            mx = std::max(mx, w);
        }
        if (batch == 1 && equal) {  // in place: rank r's band is y[r*mx, (r+1)*mx)
            sck(spqr_matvec(s->band, x_dev, x_dtype, y_dev + a, 1, cuda_stream));
            if (s->world > 1) nck(nccl().all_gather(y_dev + a, y_dev, mx, ncclFloat32, s->comm, st), "ncclAllGather");
            return;
        }
        const std::size_t slot = static_cast<std::size_t>(batch) * mx;
        if (slot > s->slot_cap) {
            cck(cudaStreamSynchronize(st), "sync before slot growth");
            if (s->slots) cudaFree(s->slots);
            s->slots = nullptr;
            cck(cudaMalloc(&s->slots, slot * s->world * sizeof(float)), "cudaMalloc sharded slots");
            s->slot_cap = slot;
        }
        float* mine = s->slots + static_cast<std::size_t>(s->rank) * slot;  // [batch][b - a]
        sck(spqr_matvec(s->band, x_dev, x_dtype, mine, batch, cuda_stream));
        if (s->world > 1) nck(nccl().all_gather(mine, s->slots, slot, ncclFloat32, s->comm, st), "ncclAllGather");
        for (int k = 0; k < s->world; ++k) {  // slot k = [batch][band_k] -> y[:, edges[k] ...]
            const std::uint32_t w = s->edges[k + 1] - s->edges[k];
            cck(cudaMemcpy2DAsync(y_dev + s->edges[k], sizeof(float) * s->rows,
                                  s->slots + static_cast<std::size_t>(k) * slot, sizeof(float) * w, sizeof(float) * w,
                                  batch, cudaMemcpyDeviceToDevice, st),
                "gather compaction");
        }
    });
}

void spqr_sharded_destroy(spqr_sharded* s) { delete s; }

}  // extern "C"
