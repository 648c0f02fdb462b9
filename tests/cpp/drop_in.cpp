// Drop-in check: reference-style client code compiled against mfreg_b200.hpp
// (`namespace mfreg = mfreg_b200;`), linked to libmfreg_cuda.so.
//   drop_in host   -> host-only calls (grid construction, error mapping)
//   drop_in gpu    -> phantom pair, Objective eval/Hv, Gauss-Newton; prints results
#include <cstdio>
#include <cstring>
#include <stdexcept>
#include <vector>

#include "mfreg_b200.hpp"

namespace mfreg = mfreg_b200;

int main(int argc, char** argv) {
    const bool gpu = argc > 1 && std::strcmp(argv[1], "gpu") == 0;
    const auto img = mfreg::make_image_grid({64, 64, 64}, {1.0, 1.0, 1.0});
    const auto dg = mfreg::deformation_grid_for(img, 4);
    std::printf("deform %lld %lld %lld h %.17g\n", (long long)dg.m[0], (long long)dg.m[1], (long long)dg.m[2], dg.h[0]);
    try {
        (void)mfreg::make_deform_grid(img, {70, 4, 4});
        std::printf("no-throw\n");
        return 1;
    } catch (const std::invalid_argument& e) {
        std::printf("invalid_argument: %s\n", e.what());
    }
    {  // io.hpp on the host side: deformation file + sidecar round trip, landmark parsing
        std::vector<double> yy(static_cast<std::size_t>(3 * dg.count()), 0.25);
        const std::string base = std::string(argc > 2 ? argv[2] : "/tmp") + "/drop_in.def";
        mfreg::io::write_deformation(base, yy, dg);
        const auto g2 = mfreg::io::read_deformation_grid(base);
        const auto y2 = mfreg::io::read_deformation(base, g2);
        std::printf("io deform %lld %lld %lld %zu %.17g\n", (long long)g2.m[0], (long long)g2.m[1], (long long)g2.m[2],
                    y2.size(), y2[5]);
        try {
            mfreg::io::read_deformation_grid(base + ".missing");
        } catch (const std::runtime_error& e) {
            std::printf("runtime_error: %s\n", e.what());
        }
    }
    if (!gpu) return 0;
    // inputs: ref = phantom x 1000 (synthetic.cpp:15-63), tpl = sinusoid-warped ref
    const auto g = mfreg::make_image_grid({24, 20, 18}, {0.97, 0.97, 2.5});
    mfreg::Volume ref{g, std::vector<double>(g.count())}, tpl{g, std::vector<double>(g.count())};
    const mfreg_cu_grid gc = g.c();
    mfreg::detail::check(mfreg_cu_make_phantom(&gc, ref.data.data(), MFREG_CU_HOST));
    for (auto& v : ref.data) v *= 1000.0;
    mfreg::detail::check(mfreg_cu_warp_sinusoid(&gc, ref.data.data(), 3.0, 42, tpl.data.data(), MFREG_CU_HOST));
    const auto d = mfreg::deformation_grid_for(g, 4);
    mfreg::Objective obj(ref, tpl, d, mfreg::NgfParams{}, 1.0);
    auto y = obj.identity();
    std::vector<double> grad(y.size());
    const double j = obj.eval(y, grad);
    std::printf("J %.17g D %.17g S %.17g\n", j, obj.last_distance(), obj.last_regularizer());
    mfreg::OptimizerConfig cfg;
    cfg.max_iters = 3;
    const auto res = mfreg::gauss_newton_minimize(obj, y, cfg);
    for (const auto& r : res.trace) std::printf("it %d J %.17g cg %d step %.17g\n", r.iter, r.j, r.cg_iters, r.step);
    return 0;
}
