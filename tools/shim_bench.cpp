// Times the C++ drop-in path end to end: a reference-API fit loop in which only the rasterizer
// translation unit is swapped for the shim (paper_2412_13547_b200/shim/tgs_gpu_rasterizer.cpp).
// Per iteration, exactly what a caller of the reference's public API does:
//   tgs::render<float>(model, pattern, bg)           (shim: AoS -> SoA marshal, upload, GPU render)
//   L1 dL/dC on the host threads                      (per-pixel normalised)
//   tgs::backward<float>(model, pattern, bg, dLdC)    (shim: marshal, upload, GPU backward, stats back)
//   Adam on the host threads
// The model is the reference's own GaussianModel<float>, filled with GaussianModel::add from a
// float[10][n] parameter file (bench.py writes the same synthetic scene it times), the target an
// (H, W, 3) float file. Prints one JSON line: iterations/s and the per-part host-side times.
//
//   shim_bench <params.f32> <n> <target.f32> <W> <H> <p> <warmup> <steps>
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <thread>
#include <vector>

#include "tgs/rasterizer.hpp"

namespace {

std::vector<float> read_f32(const char* path, size_t count) {
    std::vector<float> v(count);
    FILE* f = std::fopen(path, "rb");
    if (!f || std::fread(v.data(), 4, count, f) != count) {
        std::fprintf(stderr, "shim_bench: cannot read %s\n", path);
        std::exit(2);
    }
    std::fclose(f);
    return v;
}

// the harness's own host loops (L1, Adam) on all host threads, as a reference trainer would run
// them on its ThreadPool (threading.hpp)
template <typename F>
void parallel_for(size_t n, F&& f) {
    const size_t nt = std::max<size_t>(1, std::min<size_t>(std::thread::hardware_concurrency(), 32));
    std::vector<std::thread> ts;
    for (size_t t = 0; t < nt; ++t) ts.emplace_back([&, t] { f(n * t / nt, n * (t + 1) / nt, t); });
    for (auto& th : ts) th.join();
}

double now_s() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

}  // namespace

int main(int argc, char** argv) {
    if (argc < 9) return 2;
    const size_t n = std::strtoull(argv[2], nullptr, 10);
    const int W = std::atoi(argv[4]), H = std::atoi(argv[5]), p = std::atoi(argv[6]);
    const int warmup = std::atoi(argv[7]), steps = std::atoi(argv[8]);
    const std::vector<float> P = read_f32(argv[1], 10 * n);
    const std::vector<float> target = read_f32(argv[3], (size_t)W * H * 3);
    tgs::GaussianModel<float> model;
    for (size_t i = 0; i < n; ++i) {
        tgs::Gaussian2D<float> g;
        g.position = {P[i], P[n + i]};
        g.rotation = P[2 * n + i];
        g.log_scales = {P[3 * n + i], P[4 * n + i]};
        g.raw_opacity = P[5 * n + i];
        g.color = {P[6 * n + i], P[7 * n + i], P[8 * n + i]};
        g.depth_key = P[9 * n + i];
        model.add(g, 5.0);
    }
    const tgs::Vec3<float> bg(0.f, 0.f, 0.f);
    std::vector<float> m1(9 * n, 0.f), m2(9 * n, 0.f);
    double t_render = 0, t_loss = 0, t_backward = 0, t_adam = 0, loss = 0;
    double t0 = 0;
    for (int it = 0; it < warmup + steps; ++it) {
        if (it == warmup) {
            t0 = now_s();
            t_render = t_loss = t_backward = t_adam = 0;
        }
        const int idx = it % (p * p);
        const tgs::DilationPattern pat(p, idx % p, idx / p, W, H);
        double a = now_s();
        const auto out = tgs::render<float>(model, pat, bg);
        double b = now_s();
        t_render += b - a;
        // L1 over the active pixels: dL/dC = sign(C - target) / (3 P)
        const int Pn = pat.active_count();
        std::vector<tgs::Vec3<float>> dl(Pn);
        const float sc = (float)(1.0 / (3.0 * (double)Pn));
        std::vector<double> lsum(64, 0.0);
        parallel_for((size_t)Pn, [&](size_t rb, size_t re, size_t tid) {
            double ls = 0;
            for (size_t r = rb; r < re; ++r) {
                const int y = pat.offset_y() + ((int)r / pat.cols()) * p, x = pat.offset_x() + ((int)r % pat.cols()) * p;
                const float* t = &target[3 * ((size_t)y * W + x)];
                const float d0 = out.colors[r].x - t[0], d1 = out.colors[r].y - t[1], d2 = out.colors[r].z - t[2];
                ls += std::fabs(d0) + std::fabs(d1) + std::fabs(d2);
                auto sg = [&](float d) { return d > 0.f ? sc : (d < 0.f ? -sc : 0.f); };
                dl[r] = tgs::Vec3<float>(sg(d0), sg(d1), sg(d2));
            }
            lsum[tid] = ls;
        });
        double ls = 0;
        for (double v : lsum) ls += v;
        loss = ls / (3.0 * Pn);
        a = now_s();
        t_loss += a - b;
        const auto gs = tgs::backward<float>(model, pat, bg, dl);
        b = now_s();
        t_backward += b - a;
        // Adam: lr position 1.6e-4 * diag * 0.01^(t/T), rotation 1e-3, log-scale
        // 5e-3, opacity 5e-2, colour 2.5e-3; the loop a reference trainer runs on its host
        const double tn = (double)(it + 1) / 10000.0;
        const float lr[9] = {(float)(1.6e-4 * std::hypot((double)W, (double)H) * std::pow(0.01, tn)),
                             (float)(1.6e-4 * std::hypot((double)W, (double)H) * std::pow(0.01, tn)),
                             1e-3f, 5e-3f, 5e-3f, 5e-2f, 2.5e-3f, 2.5e-3f, 2.5e-3f};
        const float bc1 = (float)(1.0 - std::pow(0.9, it + 1)), bc2 = (float)(1.0 - std::pow(0.999, it + 1));
        parallel_for(n, [&](size_t ib, size_t ie, size_t) {
          for (size_t i = ib; i < ie; ++i) {
            auto& g = model[i];
            float* th[9] = {&g.position.x, &g.position.y, &g.rotation, &g.log_scales.x, &g.log_scales.y,
                            &g.raw_opacity, &g.color.x, &g.color.y, &g.color.z};
            const float gr[9] = {gs.position[i].x, gs.position[i].y, gs.rotation[i], gs.log_scales[i].x,
                                 gs.log_scales[i].y, gs.raw_opacity[i], gs.color[i].x, gs.color[i].y,
                                 gs.color[i].z};
            for (int q = 0; q < 9; ++q) {
                float& mm = m1[9 * i + q];
                float& vv = m2[9 * i + q];
                mm = 0.9f * mm + 0.1f * gr[q];
                vv = 0.999f * vv + 0.001f * gr[q] * gr[q];
                *th[q] -= lr[q] * (mm / bc1) / (std::sqrt(vv / bc2) + 1e-15f);
            }
          }
        });
        t_adam += now_s() - b;
    }
    const double total = now_s() - t0;
    std::printf("{\"impl\": \"shim\", \"iters_per_s\": %.6f, \"steps\": %d, \"seconds\": %.6f, "
                "\"render_s\": %.6f, \"host_loss_s\": %.6f, \"backward_s\": %.6f, \"host_adam_s\": %.6f, "
                "\"loss\": %.6f, \"gaussians\": %zu}\n",
                steps / total, steps, total, t_render / steps, t_loss / steps, t_backward / steps,
                t_adam / steps, loss, n);
    return 0;
}
