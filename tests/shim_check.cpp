// Exercises the C++ drop-in shim (paper_2412_13547_b200/shim/tgs_gpu_rasterizer.cpp) through the
// reference's OWN public API: builds a GaussianModel<float> with GaussianModel::add and the
// reference's Pcg32 (rng.hpp), calls tgs::render<float> / tgs::backward<float> (which now run on
// the GPU) and dumps the results for tests/test_gpu_shim.py to compare with the CPU oracle.
//
//   shim_check <out.bin>   -> int64 n, P; uint64 ops; float rgb[3P], T[P], grads[9n],
//                             float pos_acc[n], col_acc[n]; int64 visit[n]; int status
#include <cmath>
#include <cstdio>
#include <stdexcept>
#include <vector>

#include "tgs/rasterizer.hpp"
#include "tgs/rng.hpp"

int main(int argc, char** argv) {
    if (argc < 2) return 2;
    const int W = 160, H = 112, n = 3000;
    tgs::Pcg32 r(7, 1);
    tgs::GaussianModel<float> model;
    const double pi = 3.14159265358979323846;
    for (int i = 0; i < n; ++i) {
        tgs::Gaussian2D<float> g;
        g.position = {(float)r.uniform_in(0, W), (float)r.uniform_in(0, H)};
        g.rotation = (float)r.uniform_in(-pi, pi);
        g.log_scales = {(float)r.uniform_in(0, 1.5), (float)r.uniform_in(0, 1.5)};
        g.raw_opacity = (float)r.uniform_in(-2, 2);
        g.color = {(float)r.uniform_in(-2, 2), (float)r.uniform_in(-2, 2), (float)r.uniform_in(-2, 2)};
        g.depth_key = (float)r.uniform_in(0, 1);
        model.add(g, 5.0);
    }
    tgs::DilationPattern pat(2, 1, 0, W, H);
    auto out = tgs::render<float>(model, pat, tgs::Vec3<float>(0.1f, 0.2f, 0.3f));
    const int P = pat.active_count();
    std::vector<tgs::Vec3<float>> dl(P);
    tgs::Pcg32 r2(9, 1);
    for (auto& v : dl) {  // explicit draw order (argument evaluation order is unspecified)
        const float x = (float)r2.uniform_in(-1e-3, 1e-3);
        const float y = (float)r2.uniform_in(-1e-3, 1e-3);
        const float z = (float)r2.uniform_in(-1e-3, 1e-3);
        v = tgs::Vec3<float>(x, y, z);
    }
    auto gs = tgs::backward<float>(model, pat, tgs::Vec3<float>(0.1f, 0.2f, 0.3f), dl);
    int status = 0;
    try {  // the reference's rank-count check must still throw std::invalid_argument
        std::vector<tgs::Vec3<float>> bad(3);
        tgs::backward<float>(model, pat, tgs::Vec3<float>(0, 0, 0), bad);
        status = 1;
    } catch (const std::invalid_argument&) {
    }
    try {  // non-finite parameter -> std::invalid_argument (gaussian.hpp:64-68)
        auto m2 = model;
        m2[5].rotation = NAN;
        tgs::render<float>(m2, pat, tgs::Vec3<float>(0, 0, 0));
        status |= 2;
    } catch (const std::invalid_argument&) {
    }
    FILE* f = std::fopen(argv[1], "wb");
    if (!f) return 3;
    const long long nn = n, PP = P;
    const unsigned long long ops = out.blend_op_count;
    std::fwrite(&nn, 8, 1, f);
    std::fwrite(&PP, 8, 1, f);
    std::fwrite(&ops, 8, 1, f);
    for (auto& c : out.colors) std::fwrite(&c.x, 4, 3, f);
    std::fwrite(out.final_transmittance.data(), 4, P, f);
    for (int q = 0; q < 9; ++q)
        for (int i = 0; i < n; ++i) {
            float v = 0;
            switch (q) {
                case 0: v = gs.position[i].x; break;
                case 1: v = gs.position[i].y; break;
                case 2: v = gs.rotation[i]; break;
                case 3: v = gs.log_scales[i].x; break;
                case 4: v = gs.log_scales[i].y; break;
                case 5: v = gs.raw_opacity[i]; break;
                case 6: v = gs.color[i].x; break;
                case 7: v = gs.color[i].y; break;
                default: v = gs.color[i].z; break;
            }
            std::fwrite(&v, 4, 1, f);
        }
    std::fwrite(model.stats().pos_grad_norm_accum.data(), 4, n, f);
    std::fwrite(model.stats().color_grad_norm_accum.data(), 4, n, f);
    std::fwrite(model.stats().visit_count.data(), 8, n, f);
    std::fwrite(&status, 4, 1, f);
    std::fclose(f);
    std::printf("shim_check ok n=%d P=%d ops=%llu status=%d\n", n, P, ops, status);
    return status;
}
