// ref_encoder.cpp -- C entry point over the UNMODIFIED reference encoder:
// HessianAccumulator / finalize (hessian.hpp:52-154), spqr_quantize
// (solver.hpp:417-533), make_spqr_tensor + encode (format.hpp:69, :269).
//
// TEST INFRASTRUCTURE ONLY (the GPU encoder's parity checker).  Built by
// oracle/Makefile into oracle/_ref/libspqr_ref_enc.so from the headers where
// they lie, with our functional minimal Eigen (oracle/eigen_min: the
// reference's encoder executes Eigen code, and Eigen is absent).  No
// reference source is copied; this file includes the headers and marshals
// arguments.  Namespace renamed spqr -> spqr_ref as in ref_shim.cpp.
#define spqr spqr_ref
#include "spqr/format.hpp"
#undef spqr

#include <cstring>
#include <vector>

namespace R = spqr_ref;

extern "C" {

// W: m x n row-major fp32 (original column order); X: n x samples row-major
// fp32 calibration inputs.  cfg: {wb, sb, zb, beta1, beta2, order (0 natural,
// 1 act_order, 2 shuffled), act_key (0 hessian_diag, 1 inverse_diag),
// outliers_enabled, integer_zero, full_range_sign}, tau, lambda_rel, seed.
// target_rate > 0: tune_tau instead of the fixed tau.  report: {relative_error,
// outlier_rate, bits_per_param[, tau, target reached]}.
int ref_enc_quantize(const float* W, uint32_t m, uint32_t n, const float* X, uint32_t samples, const int* cfg,
                     double tau, double lambda_rel, uint64_t seed, double target_rate, uint8_t* out, size_t cap,
                     size_t* len, double* report) {
    try {
        R::HessianAccumulator acc(n);
        acc.accumulate(R::DenseTensor(n, samples, std::vector<float>(X, X + static_cast<size_t>(n) * samples)));
        const R::InverseCholesky icho = R::finalize(acc, lambda_rel);
        R::SolverConfig c;
        c.weight_bits = cfg[0];
        c.scale_bits = cfg[1];
        c.zero_bits = cfg[2];
        c.beta1 = static_cast<uint32_t>(cfg[3]);
        c.beta2 = static_cast<uint32_t>(cfg[4]);
        c.order = static_cast<R::ColumnOrder>(cfg[5]);
        c.act_order_key = static_cast<R::ActOrderKey>(cfg[6]);
        c.outliers_enabled = cfg[7] != 0;
        c.integer_zero = cfg[8] != 0;
        c.full_range_sign = cfg[9] != 0;
        c.tau = tau;
        c.lambda_rel = lambda_rel;
        c.seed = seed;
        const R::DenseTensor Wt(m, n, std::vector<float>(W, W + static_cast<size_t>(m) * n));
        R::SpqrResult res;
        if (target_rate > 0.0) {  // tune_tau, solver.hpp:546
            R::TuneResult tr = R::tune_tau(Wt, icho, c, target_rate);
            res = std::move(tr.result);
            c.tau = tr.tau;
            if (report) {
                report[3] = tr.tau;
                report[4] = tr.target_reached ? 1.0 : 0.0;
            }
        } else {
            res = R::spqr_quantize(Wt, icho, c);
        }
        const std::vector<uint8_t> bytes = R::encode(R::make_spqr_tensor(res, c));
        *len = bytes.size();
        if (report) {
            report[0] = res.report.relative_error;
            report[1] = res.report.outlier_rate;
            report[2] = res.report.bits_per_param;
        }
        if (!out || cap < bytes.size()) return 999;
        std::memcpy(out, bytes.data(), bytes.size());
        return 0;
    } catch (const R::Error& e) {
        return 1 + static_cast<int>(e.code());
    } catch (...) {
        return 1000;
    }
}
}
