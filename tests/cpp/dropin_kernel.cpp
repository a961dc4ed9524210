// A caller of the reference's kernel API (kernel.hpp:17-226) recompiled
// against include/spqr/kernel.hpp: dequantize_full + matvec run on the GPU.
#include <cstdio>
#include <fstream>
#include <vector>

#include "spqr/kernel.hpp"

int main(int argc, char** argv) {
    if (argc < 5) return 2;
    try {
        const spqr::SpqrTensor t = spqr::load_spqr(argv[1]);
        std::vector<float> x(t.cols);
        std::ifstream(argv[2], std::ios::binary).read(reinterpret_cast<char*>(x.data()), 4 * x.size());
        const spqr::DenseTensor w = spqr::dequantize_full(t);
        std::ofstream(argv[3], std::ios::binary)
            .write(reinterpret_cast<const char*>(w.data().data()), 4 * w.data().size());
        const spqr::TilePlan plan = spqr::build_tile_plan(t);
        const std::vector<float> y = spqr::matvec(t, x, plan);
        std::ofstream(argv[4], std::ios::binary).write(reinterpret_cast<const char*>(y.data()), 4 * y.size());
        // the explicit device handle: upload once, call many times
        spqr::DeviceLayer layer(t);
        const std::vector<float> y2 = spqr::matvec(layer, x);
        if (spqr::detail::relative_l2(y, y2) != 0.0) return 5;
        // per-token calls on the same tensor reuse the cached device layer
        const std::size_t cached = spqr::device_cache_size();
        for (int i = 0; i < 3; ++i)
            if (spqr::detail::relative_l2(spqr::matvec(t, x), y) != 0.0) return 7;
        if (spqr::device_cache_size() != cached || cached < 1) return 8;
        spqr::clear_device_cache();
        if (spqr::device_cache_size() != 0) return 9;
        std::size_t total = 0;
        for (std::size_t i = 0; i < plan.tiles.size(); ++i) total += plan.tile_outlier_count(i);
        if (total != t.outliers.items.size()) return 6;  // SPEC.md:450 slices partition nnz
        const spqr::BenchResult b = spqr::bench_matvec(t, x, 5);
        std::printf("fast=%d tiled_ns=%.0f naive_ns=%.0f dense_ns=%.0f\n", layer.fast_path() ? 1 : 0,
                    b.tiled_ns_per_op, b.naive_ns_per_op, b.dense_ns_per_op);
    } catch (const spqr::Error& e) {
        std::printf("%s\n", e.what());
        return 3;
    }
    return 0;
}
