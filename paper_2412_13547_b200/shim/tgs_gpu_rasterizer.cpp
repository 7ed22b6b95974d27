// Drop-in replacement for the reference's hot-path translation unit
// (/root/reference/proj/core/src/rasterizer.cpp): defines tgs::render<float> and
// tgs::backward<float> with the EXACT signatures of rasterizer.hpp:58-60 / 66-69, executing on
// the B200 through libtgsx's C ABI (include/tgsx.h).
//
// A maintainer swaps `src/rasterizer.cpp` for this file in core/CMakeLists.txt, adds
// include/tgsx.h to the include path and links libtgsx.so. Compiled here
// against the reference's own headers (tgs/rasterizer.hpp, model.hpp, dilation.hpp, vec.hpp),
// which are not copied into this repository.
//
// Semantics kept from the reference:
//  * render reads the model (creation order), returns colours / final T by dense rank and the
//    blend-op count; the model's blend order is recomputed on the device (model.hpp:106-119).
//  * backward throws std::invalid_argument on a rank-count mismatch (rasterizer.cpp:222-224),
//    returns the GradientSet in model order and updates model.stats() in place
//    (rasterizer.cpp:350-358).
//  * non-finite parameters -> std::invalid_argument, degenerate covariance ->
//    std::runtime_error (gaussian.hpp:64-68, 84-86), via the C ABI's status codes.
//  * RenderOptions::lowpass_p is honoured; RenderOptions::threads is accepted and ignored (the
//    GPU grid replaces the ThreadPool).
// The double instantiations stay with the reference (fp64 finite-difference tests).
//
// The caller's model is AoS host memory, so every call crosses PCIe. The crossing is kept lean:
// the SoA image of the model and every result live in page-locked staging buffers reused across
// calls, the AoS <-> SoA conversions run on all host threads, and the model is uploaded only when
// its image changed since the last upload (render followed by backward of the same model — the
// reference's own call pattern — uploads once; the stats backward writes back are folded into the
// image, so they do not count as a change).
#include "tgs/rasterizer.hpp"

#include <algorithm>
#include <atomic>
#include <mutex>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "tgsx.h"

namespace {

void check(int32_t rc, tgsx_ctx* ctx) {
    if (rc == TGSX_OK) return;
    const std::string msg = ctx ? tgsx_last_error(ctx) : "tgsx";
    if (rc == TGSX_EINVAL) throw std::invalid_argument(msg);
    if (rc == TGSX_ERUNTIME) throw std::runtime_error(msg);
    throw std::runtime_error("tgsx error " + std::to_string(rc) + ": " + msg);
}

// [0, n) split over the host threads (the ThreadPool's role in the reference, threading.hpp)
template <typename F>
void parallel_for(size_t n, F&& f) {
    const size_t hw = std::max(1u, std::thread::hardware_concurrency());
    const size_t nt = std::min<size_t>(std::min<size_t>(hw, 32), std::max<size_t>(1, n / 32768));
    if (nt <= 1) {
        f(size_t(0), n, size_t(0));
        return;
    }
    std::vector<std::thread> ts;
    ts.reserve(nt);
    for (size_t t = 0; t < nt; ++t)
        ts.emplace_back([&, t] { f(n * t / nt, n * (t + 1) / nt, t); });
    for (auto& th : ts) th.join();
}

// page-locked buffer, grown geometrically
struct Pinned {
    void* p = nullptr;
    size_t bytes = 0;
    template <typename T>
    T* get(size_t count) {
        const size_t need = std::max<size_t>(count, 1) * sizeof(T);
        if (need > bytes) {
            const size_t nb = std::max(need, bytes + bytes / 2);
            tgsx_host_free(p);
            p = nullptr;
            bytes = 0;
            if (tgsx_host_alloc(nb, &p) != TGSX_OK) throw std::runtime_error("tgsx: pinned host allocation failed");
            bytes = nb;
        }
        return static_cast<T*>(p);
    }
    ~Pinned() { tgsx_host_free(p); }
};

struct Session {
    tgsx_ctx* ctx = nullptr;
    tgsx_model* model = nullptr;
    std::mutex mu;
    // SoA image of the last uploaded model
    Pinned rows[10], ids, pos, col, accum, visit, window, tau;
    size_t n = 0;
    uint64_t next_id = 0;
    bool uploaded = false;
    Pinned out_a, out_b;  // results (render: rgb, T; backward: dL/dC, gradients)
    Session() {
        if (tgsx_create(0, &ctx) != TGSX_OK) throw std::runtime_error("tgsx: no CUDA device");
        if (tgsx_model_create(ctx, 1, &model) != TGSX_OK) throw std::runtime_error("tgsx: model alloc");
    }
    ~Session() {
        if (model) tgsx_model_destroy(model);
        if (ctx) tgsx_destroy(ctx);
    }

    // Writes the model into the SoA image; returns true when anything differs from the image of
    // the last upload (a fresh image always differs).
    bool marshal(const tgs::GaussianModel<float>& m) {
        const size_t nn = m.size();
        const bool resized = nn != n || !uploaded;
        float* r[10];
        for (int q = 0; q < 10; ++q) r[q] = rows[q].get<float>(nn);
        uint64_t* id = ids.get<uint64_t>(nn);
        float* pa = pos.get<float>(nn);
        float* ca = col.get<float>(nn);
        int32_t* ac = accum.get<int32_t>(nn);
        int64_t* vi = visit.get<int64_t>(nn);
        int64_t* wi = window.get<int64_t>(nn);
        double* tv = tau.get<double>(nn);
        const auto& st = m.stats();
        const auto& thr = m.visit_thresholds();
        const bool have_tau = thr.size() == nn;
        std::atomic<bool> changed{resized || m.next_id() != next_id};
        parallel_for(nn, [&](size_t b, size_t e, size_t) {
            bool ch = false;
            auto put = [&ch](auto& dst, auto v) {
                if (!(dst == v)) {  // NaN parameters always count as changed (and are rejected on upload)
                    ch = true;
                    dst = v;
                }
            };
            for (size_t i = b; i < e; ++i) {
                const auto& g = m[i];
                put(r[0][i], g.position.x);
                put(r[1][i], g.position.y);
                put(r[2][i], g.rotation);
                put(r[3][i], g.log_scales.x);
                put(r[4][i], g.log_scales.y);
                put(r[5][i], g.raw_opacity);
                put(r[6][i], g.color.x);
                put(r[7][i], g.color.y);
                put(r[8][i], g.color.z);
                put(r[9][i], g.depth_key);
                put(id[i], g.id);
                put(pa[i], st.pos_grad_norm_accum[i]);
                put(ca[i], st.color_grad_norm_accum[i]);
                put(ac[i], st.accum_count[i]);
                put(vi[i], st.visit_count[i]);
                put(wi[i], st.window_visit_count[i]);
                put(tv[i], have_tau ? thr[i] : 5.0);
            }
            if (ch) changed = true;
        });
        if (!changed) return false;
        n = nn;
        next_id = m.next_id();
        return true;
    }

    void upload_if_changed(const tgs::GaussianModel<float>& m) {
        if (!marshal(m)) return;
        tgsx_host_scene h{};
        h.n = (int64_t)n;
        float** dst[10] = {&h.px, &h.py, &h.rot, &h.lsx, &h.lsy, &h.rop, &h.cr, &h.cg, &h.cb, &h.depth};
        for (int q = 0; q < 10; ++q) *dst[q] = rows[q].get<float>(n);
        h.id = ids.get<uint64_t>(n);
        h.next_id = next_id;
        h.pos_acc = pos.get<float>(n);
        h.col_acc = col.get<float>(n);
        h.accum = accum.get<int32_t>(n);
        h.visit = visit.get<int64_t>(n);
        h.window = window.get<int64_t>(n);
        h.tau_v = tau.get<double>(n);
        uploaded = false;
        check(tgsx_model_upload(ctx, model, &h), ctx);
        uploaded = true;
    }
};

Session& session() {
    static Session s;
    return s;
}

tgsx_pattern pattern_of(const tgs::DilationPattern& p) {
    return tgsx_pattern{p.pattern_size(), p.offset_x(), p.offset_y(), p.width(), p.height()};
}

}  // namespace

namespace tgs {

template <>
RenderOutput<float> render(const GaussianModel<float>& model, const DilationPattern& pattern,
                           Vec3<float> background, const RenderOptions& opts) {
    Session& s = session();
    std::lock_guard<std::mutex> lock(s.mu);
    s.upload_if_changed(model);
    const size_t P = (size_t)pattern.active_count();
    float* rgb = s.out_a.get<float>(3 * P);
    float* T = s.out_b.get<float>(P);
    const float bg[3] = {background.x, background.y, background.z};
    const tgsx_pattern pat = pattern_of(pattern);
    uint64_t ops = 0;
    check(tgsx_render(s.ctx, s.model, &pat, bg, opts.lowpass_p, rgb, T, &ops), s.ctx);
    RenderOutput<float> out;
    out.colors.resize(P);
    out.final_transmittance.resize(P);
    parallel_for(P, [&](size_t b, size_t e, size_t) {
        for (size_t i = b; i < e; ++i) {
            out.colors[i] = Vec3<float>(rgb[3 * i], rgb[3 * i + 1], rgb[3 * i + 2]);
            out.final_transmittance[i] = T[i];
        }
    });
    out.blend_op_count = ops;
    return out;
}

template <>
GradientSet<float> backward(GaussianModel<float>& model, const DilationPattern& pattern,
                            Vec3<float> background, const std::vector<Vec3<float>>& pixel_loss_grads,
                            const RenderOptions& opts) {
    if (static_cast<int>(pixel_loss_grads.size()) != pattern.active_count()) {
        throw std::invalid_argument("backward: loss-gradient count does not match pattern ranks");
    }
    Session& s = session();
    std::lock_guard<std::mutex> lock(s.mu);
    s.upload_if_changed(model);
    const size_t n = model.size(), P = pixel_loss_grads.size();
    float* dl = s.out_a.get<float>(3 * P);
    parallel_for(P, [&](size_t b, size_t e, size_t) {
        for (size_t i = b; i < e; ++i) {
            dl[3 * i] = pixel_loss_grads[i].x;
            dl[3 * i + 1] = pixel_loss_grads[i].y;
            dl[3 * i + 2] = pixel_loss_grads[i].z;
        }
    });
    float* g = s.out_b.get<float>(9 * n);
    const float bg[3] = {background.x, background.y, background.z};
    const tgsx_pattern pat = pattern_of(pattern);
    check(tgsx_backward(s.ctx, s.model, &pat, bg, opts.lowpass_p, dl, (int64_t)P, g, 1), s.ctx);
    // DensifyStats updated on the device -> the image (so they are not a change next call) and the
    // caller's model, in place like the reference (rasterizer.cpp:350-358)
    tgsx_host_scene h{};
    h.pos_acc = s.pos.get<float>(n);
    h.col_acc = s.col.get<float>(n);
    h.accum = s.accum.get<int32_t>(n);
    h.visit = s.visit.get<int64_t>(n);
    h.window = s.window.get<int64_t>(n);
    check(tgsx_model_download(s.ctx, s.model, &h), s.ctx);
    auto& st = model.stats();
    GradientSet<float> gs;
    gs.assign_zero(n);
    parallel_for(n, [&](size_t b, size_t e, size_t) {
        std::copy(h.pos_acc + b, h.pos_acc + e, st.pos_grad_norm_accum.begin() + b);
        std::copy(h.col_acc + b, h.col_acc + e, st.color_grad_norm_accum.begin() + b);
        std::copy(h.accum + b, h.accum + e, st.accum_count.begin() + b);
        std::copy(h.visit + b, h.visit + e, st.visit_count.begin() + b);
        std::copy(h.window + b, h.window + e, st.window_visit_count.begin() + b);
        for (size_t i = b; i < e; ++i) {
            gs.position[i] = Vec2<float>(g[0 * n + i], g[1 * n + i]);
            gs.rotation[i] = g[2 * n + i];
            gs.log_scales[i] = Vec2<float>(g[3 * n + i], g[4 * n + i]);
            gs.raw_opacity[i] = g[5 * n + i];
            gs.color[i] = Vec3<float>(g[6 * n + i], g[7 * n + i], g[8 * n + i]);
        }
    });
    return gs;
}

}  // namespace tgs
