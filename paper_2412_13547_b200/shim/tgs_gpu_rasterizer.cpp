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
#include "tgs/rasterizer.hpp"

#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "tgsx.h"

namespace {

struct Session {
    tgsx_ctx* ctx = nullptr;
    tgsx_model* model = nullptr;
    std::mutex mu;
    Session() {
        if (tgsx_create(0, &ctx) != TGSX_OK) throw std::runtime_error("tgsx: no CUDA device");
        if (tgsx_model_create(ctx, 1, &model) != TGSX_OK) throw std::runtime_error("tgsx: model alloc");
    }
    ~Session() {
        if (model) tgsx_model_destroy(model);
        if (ctx) tgsx_destroy(ctx);
    }
};

Session& session() {
    static Session s;
    return s;
}

void check(int32_t rc, tgsx_ctx* ctx) {
    if (rc == TGSX_OK) return;
    const std::string msg = tgsx_last_error(ctx);
    if (rc == TGSX_EINVAL) throw std::invalid_argument(msg);
    if (rc == TGSX_ERUNTIME) throw std::runtime_error(msg);
    throw std::runtime_error("tgsx error " + std::to_string(rc) + ": " + msg);
}

// AoS GaussianModel<float> -> SoA host arrays -> device model.
struct Marshalled {
    std::vector<float> rows[10];
    std::vector<uint64_t> ids;
    std::vector<int32_t> accum;
    std::vector<int64_t> visit, window;
    std::vector<float> pos, col;
    std::vector<double> tau;
    tgsx_host_scene hs{};
};

void marshal(const tgs::GaussianModel<float>& m, Marshalled& out) {
    const size_t n = m.size();
    for (auto& r : out.rows) r.resize(n);
    out.ids.resize(n);
    for (size_t i = 0; i < n; ++i) {
        const auto& g = m[i];
        out.rows[0][i] = g.position.x;
        out.rows[1][i] = g.position.y;
        out.rows[2][i] = g.rotation;
        out.rows[3][i] = g.log_scales.x;
        out.rows[4][i] = g.log_scales.y;
        out.rows[5][i] = g.raw_opacity;
        out.rows[6][i] = g.color.x;
        out.rows[7][i] = g.color.y;
        out.rows[8][i] = g.color.z;
        out.rows[9][i] = g.depth_key;
        out.ids[i] = g.id;
    }
    const auto& st = m.stats();
    out.pos = st.pos_grad_norm_accum;
    out.col = st.color_grad_norm_accum;
    out.accum = st.accum_count;
    out.visit = st.visit_count;
    out.window = st.window_visit_count;
    out.tau = m.visit_thresholds();
    tgsx_host_scene& h = out.hs;
    h.n = (int64_t)n;
    float** dst[10] = {&h.px, &h.py, &h.rot, &h.lsx, &h.lsy, &h.rop, &h.cr, &h.cg, &h.cb, &h.depth};
    for (int q = 0; q < 10; ++q) *dst[q] = out.rows[q].data();
    h.id = out.ids.data();
    h.next_id = m.next_id();
    h.pos_acc = out.pos.data();
    h.col_acc = out.col.data();
    h.accum = out.accum.data();
    h.visit = out.visit.data();
    h.window = out.window.data();
    h.tau_v = out.tau.empty() ? nullptr : out.tau.data();
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
    Marshalled mm;
    marshal(model, mm);
    check(tgsx_model_upload(s.ctx, s.model, &mm.hs), s.ctx);
    const int P = pattern.active_count();
    std::vector<float> rgb(3 * (size_t)P), T((size_t)P);
    const float bg[3] = {background.x, background.y, background.z};
    const tgsx_pattern pat = pattern_of(pattern);
    uint64_t ops = 0;
    check(tgsx_render(s.ctx, s.model, &pat, bg, opts.lowpass_p, rgb.data(), T.data(), &ops), s.ctx);
    RenderOutput<float> out;
    out.colors.resize(P);
    out.final_transmittance = std::move(T);
    for (int i = 0; i < P; ++i) out.colors[i] = Vec3<float>(rgb[3 * i], rgb[3 * i + 1], rgb[3 * i + 2]);
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
    Marshalled mm;
    marshal(model, mm);
    check(tgsx_model_upload(s.ctx, s.model, &mm.hs), s.ctx);
    const size_t n = model.size();
    std::vector<float> dl(3 * pixel_loss_grads.size());
    for (size_t i = 0; i < pixel_loss_grads.size(); ++i) {
        dl[3 * i] = pixel_loss_grads[i].x;
        dl[3 * i + 1] = pixel_loss_grads[i].y;
        dl[3 * i + 2] = pixel_loss_grads[i].z;
    }
    std::vector<float> g(9 * std::max<size_t>(n, 1));
    const float bg[3] = {background.x, background.y, background.z};
    const tgsx_pattern pat = pattern_of(pattern);
    check(tgsx_backward(s.ctx, s.model, &pat, bg, opts.lowpass_p, dl.data(),
                        (int64_t)pixel_loss_grads.size(), g.data(), 1),
          s.ctx);
    // DensifyStats updated on the device -> back into the caller's model (in place, like the
    // reference)
    check(tgsx_model_download(s.ctx, s.model, &mm.hs), s.ctx);
    auto& st = model.stats();
    st.pos_grad_norm_accum = mm.pos;
    st.color_grad_norm_accum = mm.col;
    st.accum_count = mm.accum;
    st.visit_count = mm.visit;
    st.window_visit_count = mm.window;
    GradientSet<float> gs;
    gs.assign_zero(n);
    for (size_t i = 0; i < n; ++i) {
        gs.position[i] = Vec2<float>(g[0 * n + i], g[1 * n + i]);
        gs.rotation[i] = g[2 * n + i];
        gs.log_scales[i] = Vec2<float>(g[3 * n + i], g[4 * n + i]);
        gs.raw_opacity[i] = g[5 * n + i];
        gs.color[i] = Vec3<float>(g[6 * n + i], g[7 * n + i], g[8 * n + i]);
    }
    return gs;
}

}  // namespace tgs
