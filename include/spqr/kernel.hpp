// spqr/kernel.hpp -- decode-side compute on the B200 (drop-in API).
//
// Same names and signatures as the reference's kernel.hpp:17-226:
//   dequantize_full, TilePlan, build_tile_plan, matvec (x2), matvec_naive,
//   BenchResult, bench_matvec
// but every compute call runs hand-written sm_100a kernels through the C ABI
// in spqr_cuda.h; there is no CPU fallback (a missing GPU / extension throws).
//
// DeviceLayer is the explicit handle: the layer is validated, transcoded to
// its HBM layout and uploaded once; matvec/dequantize on it never re-upload.
// The SpqrTensor overloads upload a transient DeviceLayer per call -- correct
// but slow; hold a DeviceLayer on hot paths.
#pragma once

#include <cstdint>
#include <memory>
#include <span>
#include <vector>

#include "spqr/format.hpp"
#include "spqr/types.hpp"

struct spqr_layer;

namespace spqr {

class DeviceLayer {
public:
    explicit DeviceLayer(std::span<const std::uint8_t> stream, int device = -1);
    explicit DeviceLayer(const SpqrTensor& t, int device = -1);
    DeviceLayer(DeviceLayer&&) noexcept;
    DeviceLayer& operator=(DeviceLayer&&) noexcept;
    ~DeviceLayer();

    std::uint32_t rows() const;
    std::uint32_t cols() const;
    bool fast_path() const;
    std::size_t payload_bytes() const;
    spqr_layer* handle() const { return h_; }

    // Device-buffer forms (asynchronous on `cuda_stream`).
    void matvec_device(const void* x_dev, bool x_is_f16, float* y_dev, int batch,
                       void* cuda_stream = nullptr) const;
    void dequantize_device(float* w_dev, void* cuda_stream = nullptr) const;
    std::vector<std::uint8_t> export_stream() const;

private:
    spqr_layer* h_ = nullptr;
};

// Work partition summary (kept for API compatibility, kernel.hpp:30-84).  On
// the GPU the partition is computed once per DeviceLayer; build_tile_plan
// returns the reference's 64-row x beta1 tiling of the tensor for callers that
// inspect it (tile_outlier_count etc.).
struct TilePlan {
    struct Tile {
        std::uint32_t r0, r1, c0, c1, block;
        std::size_t slice_offset;
    };
    std::uint32_t tile_rows = 64;
    std::vector<Tile> tiles;
    std::vector<std::pair<std::uint32_t, std::uint32_t>> slices;
    std::size_t tile_outlier_count(std::size_t tile_index) const;
};
TilePlan build_tile_plan(const SpqrTensor& t, std::uint32_t tile_rows = 64);

DenseTensor dequantize_full(const SpqrTensor& t);
DenseTensor dequantize_full(const DeviceLayer& layer);

// The tensor is uploaded on its first matvec and the device layer cached by
// tensor identity (address + sampled fingerprint, LRU): later calls with the
// same tensor cost the host-buffer matvec only.  A tensor modified in place
// after its first matvec needs clear_device_cache().
std::vector<float> matvec(const SpqrTensor& t, std::span<const float> x, const TilePlan& plan);
std::vector<float> matvec(const SpqrTensor& t, std::span<const float> x);
void clear_device_cache();
std::size_t device_cache_size();
std::vector<float> matvec(const DeviceLayer& layer, std::span<const float> x);
std::vector<float> matvec_naive(const SpqrTensor& t, std::span<const float> x);

struct BenchResult {
    double tiled_ns_per_op = 0.0;  // fused GPU kernel, CUDA-event timed
    double naive_ns_per_op = 0.0;  // GPU dequantize + dense product
    double dense_ns_per_op = 0.0;  // dense fp16 GEMV of the same shape
    int repeats = 0;
    bool low_confidence = false;
};
BenchResult bench_matvec(const SpqrTensor& t, std::span<const float> x, int repeats);

namespace detail {
double relative_l2(std::span<const float> a, std::span<const float> b);
}

}  // namespace spqr
