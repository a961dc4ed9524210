// A caller of the reference's format API (format.hpp:269-517), recompiled
// unchanged against our include/spqr/ headers: load -> decode -> inspect ->
// encode -> save.  Exit code 3 + "<ErrcName>: ..." on spqr::Error.
#include <cstdio>

#include "spqr/format.hpp"

int main(int argc, char** argv) {
    if (argc < 3) return 2;
    try {
        spqr::SpqrTensor t = spqr::load_spqr(argv[1]);
        const spqr::MeasuredBits mb = spqr::measure_actual_bits(t);
        const spqr::BitsEstimate est = spqr::estimate_avg_bits(t.weight_bits, 3, 3, t.beta1, t.beta2, 0.0);
        std::printf("rows=%u cols=%u bits/param=%.4f est=%.4f outliers=%zu perm=%d scale_at(0,0)=%g\n", t.rows,
                    t.cols, mb.bits_per_param, est.avg_bits, t.outliers.items.size(), t.has_permutation() ? 1 : 0,
                    t.stats.scale_at(0, 0));
        if (mb.payload_bytes != spqr::stream_payload_bytes(t.layout())) return 4;
        spqr::save_spqr(t, argv[2]);
    } catch (const spqr::Error& e) {
        std::printf("%s\n", e.what());
        return 3;
    }
    return 0;
}
