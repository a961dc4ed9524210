// host_api.cpp -- the C++ drop-in API of kernel.hpp on top of the C ABI.
//
// Mirrors /root/reference/proj/include/spqr/kernel.hpp:17-226 name for name.
// Compute goes to the GPU through spqr_cuda.h; a missing device or a failed
// launch throws (SPQR_E_CUDA is surfaced as std::runtime_error), never falls
// back to a CPU loop.
#include <list>
#include <memory>
#include <mutex>
#include <algorithm>
#include <chrono>
#include <cmath>
#include <stdexcept>

#include "internal.hpp"
#include "spqr/kernel.hpp"

namespace spqr {

namespace {
void check(int rc) {
    if (rc == SPQR_OK) return;
    const std::string msg = spqr_last_error();
    if (rc >= 1 && rc <= 16) {
        // message already carries the "<ErrcName>: " prefix
        const auto colon = msg.find(": ");
        throw Error(static_cast<Errc>(rc - 1), colon == std::string::npos ? msg : msg.substr(colon + 2));
    }
    throw std::runtime_error(msg.empty() ? "spqr: CUDA failure" : msg);
}
}  // namespace

DeviceLayer::DeviceLayer(std::span<const std::uint8_t> stream, int device) {
    spqr_layer_opts o{};
    o.device = device;
    check(spqr_layer_create(stream.data(), stream.size(), &o, &h_));
}

DeviceLayer::DeviceLayer(const SpqrTensor& t, int device) : DeviceLayer(encode(t), device) {}

DeviceLayer::DeviceLayer(DeviceLayer&& o) noexcept : h_(o.h_) { o.h_ = nullptr; }
DeviceLayer& DeviceLayer::operator=(DeviceLayer&& o) noexcept {
    if (this != &o) {
        spqr_layer_destroy(h_);
        h_ = o.h_;
        o.h_ = nullptr;
    }
    return *this;
}
DeviceLayer::~DeviceLayer() { spqr_layer_destroy(h_); }

namespace {
spqr_layer_info info_of(const spqr_layer* h) {
    spqr_layer_info i{};
    check(spqr_layer_get_info(h, &i));
    return i;
}
}  // namespace

std::uint32_t DeviceLayer::rows() const { return info_of(h_).rows; }
std::uint32_t DeviceLayer::cols() const { return info_of(h_).cols; }
bool DeviceLayer::fast_path() const { return info_of(h_).fast_path != 0; }
std::size_t DeviceLayer::payload_bytes() const { return info_of(h_).payload_bytes; }

void DeviceLayer::matvec_device(const void* x_dev, bool x_is_f16, float* y_dev, int batch, void* st) const {
    check(spqr_matvec(h_, x_dev, x_is_f16 ? SPQR_F16 : SPQR_F32, y_dev, batch, st));
}

void DeviceLayer::dequantize_device(float* w_dev, void* st) const { check(spqr_dequantize(h_, w_dev, st)); }

std::vector<std::uint8_t> DeviceLayer::export_stream() const {
    std::size_t n = 0;
    const int rc = spqr_layer_export_stream(h_, nullptr, 0, &n);
    if (rc != SPQR_E_BUFFER_TOO_SMALL) check(rc);
    std::vector<std::uint8_t> out(n);
    check(spqr_layer_export_stream(h_, out.data(), out.size(), &n));
    return out;
}

// ------------------------------------------------------------- TilePlan ----
std::size_t TilePlan::tile_outlier_count(std::size_t i) const {
    const Tile& t = tiles[i];
    std::size_t c = 0;
    for (std::uint32_t r = t.r0; r < t.r1; ++r) {
        const auto& s = slices[t.slice_offset + (r - t.r0)];
        c += s.second - s.first;
    }
    return c;
}

TilePlan build_tile_plan(const SpqrTensor& t, std::uint32_t tile_rows) {
    if (tile_rows == 0) fail(Errc::config_invalid, "tile rows must be >= 1");
    TilePlan plan;
    plan.tile_rows = tile_rows;
    std::vector<std::uint32_t> rs(t.rows + 1, 0);
    for (const Outlier& o : t.outliers.items) rs[o.row + 1]++;
    for (std::uint32_t r = 0; r < t.rows; ++r) rs[r + 1] += rs[r];
    const std::uint32_t nb = (t.cols + t.beta1 - 1) / t.beta1;
    const auto& it = t.outliers.items;
    for (std::uint32_t r0 = 0; r0 < t.rows; r0 += tile_rows) {
        const std::uint32_t r1 = std::min(t.rows, r0 + tile_rows);
        for (std::uint32_t k = 0; k < nb; ++k) {
            const std::uint32_t c0 = k * t.beta1, c1 = std::min(t.cols, c0 + t.beta1);
            plan.tiles.push_back({r0, r1, c0, c1, k, plan.slices.size()});
            for (std::uint32_t r = r0; r < r1; ++r) {
                // columns are sorted within a row: binary-search the [c0, c1) slice
                auto lo = std::lower_bound(it.begin() + rs[r], it.begin() + rs[r + 1], c0,
                                           [](const Outlier& o, std::uint32_t c) { return o.col < c; });
                auto hi = std::lower_bound(lo, it.begin() + rs[r + 1], c1,
                                           [](const Outlier& o, std::uint32_t c) { return o.col < c; });
                plan.slices.emplace_back(static_cast<std::uint32_t>(lo - it.begin()),
                                         static_cast<std::uint32_t>(hi - it.begin()));
            }
        }
    }
    return plan;
}

// ------------------------------------------------------ dequantize/matvec --
DenseTensor dequantize_full(const DeviceLayer& layer) {
    const std::uint32_t m = layer.rows(), n = layer.cols();
    std::vector<float> host(static_cast<std::size_t>(m) * n);
    // device buffer via the C ABI's own allocation-free entry point: stage
    // through a transient allocation owned here
    float* dev = nullptr;
    check(spqr_dev_alloc(reinterpret_cast<void**>(&dev), host.size() * sizeof(float)));
    try {
        check(spqr_dequantize(layer.handle(), dev, nullptr));
        check(spqr_dev_copy_to_host(host.data(), dev, host.size() * sizeof(float)));
    } catch (...) {
        spqr_dev_free(dev);
        throw;
    }
    spqr_dev_free(dev);
    return DenseTensor(m, n, std::move(host));
}

DenseTensor dequantize_full(const SpqrTensor& t) { return dequantize_full(DeviceLayer(t)); }

std::vector<float> matvec(const DeviceLayer& layer, std::span<const float> x) {
    if (x.size() != layer.cols()) fail(Errc::shape_mismatch, "vector length must equal columns");
    std::vector<float> y(layer.rows());
    check(spqr_matvec_host(layer.handle(), x.data(), y.data(), 1));
    return y;
}

// matvec(const SpqrTensor&, x[, plan]) is a per-token call in the reference
// (kernel.hpp:89, :126): the tensor is uploaded on first use and the device
// layer cached by tensor identity -- address, shape, widths, group sizes,
// outlier count and a fingerprint sampled from the codes, statistics and
// outliers ("upload on first use, cached by tensor identity").  A
// tensor modified in place after its first matvec must be re-created or the
// cache cleared (clear_device_cache).  LRU, kDeviceCacheCap entries.
namespace {
constexpr std::size_t kDeviceCacheCap = 1024;
struct CacheKey {
    const SpqrTensor* addr;
    std::uint64_t fp;
    bool operator==(const CacheKey&) const = default;
};
std::uint64_t fingerprint(const SpqrTensor& t) {
    std::uint64_t h = 1469598103934665603ull;
    auto mix = [&](std::uint64_t v) {
        h ^= v;
        h *= 1099511628211ull;
    };
    mix(t.rows); mix(t.cols); mix(static_cast<std::uint64_t>(t.weight_bits) << 16 | t.scale_bits << 8 | t.zero_bits);
    mix(t.beta1); mix(t.beta2); mix(t.outliers.items.size());
    mix(reinterpret_cast<std::uintptr_t>(t.codes.codes.data()));
    auto sample = [&](const auto& v) {  // up to 4096 evenly spaced elements
        const std::size_t n = v.size(), step = std::max<std::size_t>(1, n / 4096);
        for (std::size_t i = 0; i < n; i += step) mix(static_cast<std::uint64_t>(v[i]));
        if (n) mix(static_cast<std::uint64_t>(v[n - 1]));
    };
    sample(t.codes.codes);
    const std::size_t nb = t.stats.blocks.size(), bstep = std::max<std::size_t>(1, nb / 64);
    for (std::size_t k = 0; k < nb; k += bstep) {
        const auto& b = t.stats.blocks[k];
        sample(b.scale_codes);
        sample(b.zero_codes);
        for (const auto& gsc : b.groups) mix(static_cast<std::uint64_t>(gsc.scale_s) << 16 | gsc.scale_z);
    }
    const std::size_t no = t.outliers.items.size(), ostep = std::max<std::size_t>(1, no / 4096);
    for (std::size_t i = 0; i < no; i += ostep) {
        const auto& o = t.outliers.items[i];
        mix(static_cast<std::uint64_t>(o.row) << 32 | o.col);
        mix(o.value16);
    }
    return h;
}
std::mutex g_cache_mu;
std::list<std::pair<CacheKey, std::shared_ptr<DeviceLayer>>> g_cache;  // front = most recent
std::shared_ptr<DeviceLayer> cached_layer(const SpqrTensor& t) {
    const CacheKey key{&t, fingerprint(t)};
    {
        std::lock_guard<std::mutex> lk(g_cache_mu);
        for (auto it = g_cache.begin(); it != g_cache.end(); ++it)
            if (it->first == key) {
                g_cache.splice(g_cache.begin(), g_cache, it);
                return it->second;
            }
    }
    auto layer = std::make_shared<DeviceLayer>(t);  // outside the lock: the upload takes milliseconds
    std::lock_guard<std::mutex> lk(g_cache_mu);
    g_cache.emplace_front(key, layer);
    while (g_cache.size() > kDeviceCacheCap) g_cache.pop_back();
    return layer;
}
}  // namespace

void clear_device_cache() {
    std::lock_guard<std::mutex> lk(g_cache_mu);
    g_cache.clear();
}

std::size_t device_cache_size() {
    std::lock_guard<std::mutex> lk(g_cache_mu);
    return g_cache.size();
}

std::vector<float> matvec(const SpqrTensor& t, std::span<const float> x, const TilePlan&) {
    if (x.size() != t.cols) fail(Errc::shape_mismatch, "vector length must equal columns");
    return matvec(*cached_layer(t), x);
}

std::vector<float> matvec(const SpqrTensor& t, std::span<const float> x) {
    if (x.size() != t.cols) fail(Errc::shape_mismatch, "vector length must equal columns");
    return matvec(*cached_layer(t), x);
}

// Reference path: full (bit-exact) dequantization on the GPU, then the dense
// product accumulated in binary64 on the host, as kernel.hpp:131-142 does.
std::vector<float> matvec_naive(const SpqrTensor& t, std::span<const float> x) {
    if (x.size() != t.cols) fail(Errc::shape_mismatch, "vector length must equal columns");
    const DenseTensor w = dequantize_full(t);
    std::vector<float> out(t.rows);
    for (std::uint32_t r = 0; r < t.rows; ++r) {
        double acc = 0.0;
        for (std::uint32_t c = 0; c < t.cols; ++c) acc += static_cast<double>(w(r, c)) * x[c];
        out[r] = static_cast<float>(acc);
    }
    return out;
}

namespace detail {
double relative_l2(std::span<const float> a, std::span<const float> b) {
    double num = 0.0, den = 0.0;
    for (std::size_t i = 0; i < a.size(); ++i) {
        const double d = static_cast<double>(a[i]) - b[i];
        num += d * d;
        den += static_cast<double>(b[i]) * b[i];
    }
    return den == 0.0 ? std::sqrt(num) : std::sqrt(num / den);
}
}  // namespace detail

// Timing is informational; correctness is asserted first (kernel.hpp:185-226):
// the fused kernel must agree with dequantize-then-multiply within 1e-6.
BenchResult bench_matvec(const SpqrTensor& t, std::span<const float> x, int repeats) {
    if (repeats < 1) fail(Errc::config_invalid, "repeats must be >= 1");
    const DeviceLayer layer(t);
    const std::vector<float> y_fast = matvec(layer, x);
    const std::vector<float> y_naive = matvec_naive(t, x);
    if (detail::relative_l2(y_fast, y_naive) > 1e-6)
        fail(Errc::shape_mismatch, "tiled and naive matvec disagree; refusing to time");
    BenchResult res;
    res.repeats = repeats;
    res.low_confidence = repeats == 1;
    double ns[3] = {0, 0, 0};
    check(spqr_bench_layer(layer.handle(), repeats, ns));
    res.tiled_ns_per_op = ns[0];
    res.naive_ns_per_op = ns[1];
    res.dense_ns_per_op = ns[2];
    return res;
}

}  // namespace spqr
