// TEST INFRASTRUCTURE ONLY — never part of the product.
//
// A flat C ABI over the UNMODIFIED reference render/backward (compiled from the sources
// under /root/reference by oracle/Makefile into oracle/_ref/). This file is ours; it
// includes the reference translation unit rasterizer.cpp (not copied) so that the
// anonymous-namespace helpers prepare_splats (rasterizer.cpp:23-46) and build_tile_grid
// (rasterizer.cpp:67-102) are reachable for per-stage parity checks (tile lists, prepared
// splats). Everything else goes through the reference's public API:
//   tgs::render<T>   rasterizer.hpp:58-60 / rasterizer.cpp:144-184
//   tgs::backward<T> rasterizer.hpp:66-69 / rasterizer.cpp:218-361
// Exceptions are mapped to status codes: 1 = std::invalid_argument, 2 = std::runtime_error.
#include REF_RASTERIZER_CPP  // "/root/reference/proj/core/src/rasterizer.cpp"
#include "tgs/kdtree.hpp"    // header-only KdTree2 (kdtree.hpp:15-139), for the initializer's kNN

#include <cstdint>
#include <cstring>
#include <stdexcept>

namespace {

template <typename T>
struct SceneView {
    int64_t n;
    const T* px; const T* py; const T* rot; const T* lsx; const T* lsy;
    const T* rop; const T* cr; const T* cg; const T* cb; const T* depth;
    const uint64_t* ids;   // may be null => 0..n-1
    uint64_t next_id;
    const double* tau_v;   // may be null => 5.0
};

template <typename T>
tgs::GaussianModel<T> build_model(const SceneView<T>& s) {
    tgs::GaussianModel<T> m;
    for (int64_t i = 0; i < s.n; ++i) {
        tgs::Gaussian2D<T> g;
        g.position = {s.px[i], s.py[i]};
        g.rotation = s.rot[i];
        g.log_scales = {s.lsx[i], s.lsy[i]};
        g.raw_opacity = s.rop[i];
        g.color = {s.cr[i], s.cg[i], s.cb[i]};
        g.depth_key = s.depth[i];
        m.add(g, s.tau_v ? s.tau_v[i] : 5.0);
        if (s.ids) m[i].id = s.ids[i];
    }
    m.set_next_id(s.ids ? s.next_id : static_cast<uint64_t>(s.n));
    return m;
}

int fail(const char* what, int code, char* err, int errlen) {
    if (err && errlen > 0) {
        std::strncpy(err, what, errlen - 1);
        err[errlen - 1] = 0;
    }
    return code;
}

template <typename F>
int guarded(F&& f, char* err, int errlen) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        return fail(e.what(), 1, err, errlen);
    } catch (const std::runtime_error& e) {
        return fail(e.what(), 2, err, errlen);
    } catch (const std::exception& e) {
        return fail(e.what(), 3, err, errlen);
    }
}

template <typename T>
int do_render(const SceneView<T>& s, int p, int ox, int oy, int W, int H, const T* bg,
              int threads, int lowpass_p, T* out_rgb, T* out_T, uint64_t* out_ops, char* err,
              int errlen) {
    return guarded(
        [&] {
            auto model = build_model(s);
            tgs::DilationPattern pat(p, ox, oy, W, H);
            tgs::RenderOptions opts;
            opts.threads = threads;
            opts.lowpass_p = lowpass_p;
            auto out = tgs::render<T>(model, pat, tgs::Vec3<T>(bg[0], bg[1], bg[2]), opts);
            for (size_t i = 0; i < out.colors.size(); ++i) {
                out_rgb[3 * i + 0] = out.colors[i].x;
                out_rgb[3 * i + 1] = out.colors[i].y;
                out_rgb[3 * i + 2] = out.colors[i].z;
                out_T[i] = out.final_transmittance[i];
            }
            *out_ops = out.blend_op_count;
        },
        err, errlen);
}

// grads: 9 arrays (pos x, pos y, rot, ls x, ls y, raw_opacity, rgb r, g, b), model order.
// stats: in/out (pos_acc, col_acc, accum_count, visit_count, window_visit_count), may be null.
template <typename T>
int do_backward(const SceneView<T>& s, int p, int ox, int oy, int W, int H, const T* bg,
                const T* dLdC, int64_t dLdC_count, int threads, int lowpass_p, T* const* grads, T* pos_acc,
                T* col_acc, int32_t* accum, int64_t* visit, int64_t* window, char* err,
                int errlen) {
    return guarded(
        [&] {
            auto model = build_model(s);
            if (pos_acc) {
                auto& st = model.stats();
                for (int64_t i = 0; i < s.n; ++i) {
                    st.pos_grad_norm_accum[i] = pos_acc[i];
                    st.color_grad_norm_accum[i] = col_acc[i];
                    st.accum_count[i] = accum[i];
                    st.visit_count[i] = visit[i];
                    st.window_visit_count[i] = window[i];
                }
            }
            tgs::DilationPattern pat(p, ox, oy, W, H);
            tgs::RenderOptions opts;
            opts.threads = threads;
            opts.lowpass_p = lowpass_p;
            // the caller's count is passed through so the reference's own size check
            // (rasterizer.cpp:222-224) decides
            std::vector<tgs::Vec3<T>> g(dLdC_count < 0 ? pat.active_count() : dLdC_count);
            for (size_t i = 0; i < g.size(); ++i)
                g[i] = tgs::Vec3<T>(dLdC[3 * i], dLdC[3 * i + 1], dLdC[3 * i + 2]);
            auto gs = tgs::backward<T>(model, pat, tgs::Vec3<T>(bg[0], bg[1], bg[2]), g, opts);
            for (int64_t i = 0; i < s.n; ++i) {
                grads[0][i] = gs.position[i].x;
                grads[1][i] = gs.position[i].y;
                grads[2][i] = gs.rotation[i];
                grads[3][i] = gs.log_scales[i].x;
                grads[4][i] = gs.log_scales[i].y;
                grads[5][i] = gs.raw_opacity[i];
                grads[6][i] = gs.color[i].x;
                grads[7][i] = gs.color[i].y;
                grads[8][i] = gs.color[i].z;
            }
            if (pos_acc) {
                const auto& st = model.stats();
                for (int64_t i = 0; i < s.n; ++i) {
                    pos_acc[i] = st.pos_grad_norm_accum[i];
                    col_acc[i] = st.color_grad_norm_accum[i];
                    accum[i] = st.accum_count[i];
                    visit[i] = st.visit_count[i];
                    window[i] = st.window_visit_count[i];
                }
            }
        },
        err, errlen);
}

}  // namespace

extern "C" {

typedef SceneView<float> RefSceneF32;
typedef SceneView<double> RefSceneF64;

int ref_render_f32(const RefSceneF32* s, int p, int ox, int oy, int W, int H, const float* bg,
                   int threads, int lowpass_p, float* out_rgb, float* out_T, uint64_t* out_ops,
                   char* err, int errlen) {
    return do_render(*s, p, ox, oy, W, H, bg, threads, lowpass_p, out_rgb, out_T, out_ops, err,
                     errlen);
}

int ref_render_f64(const RefSceneF64* s, int p, int ox, int oy, int W, int H, const double* bg,
                   int threads, int lowpass_p, double* out_rgb, double* out_T, uint64_t* out_ops,
                   char* err, int errlen) {
    return do_render(*s, p, ox, oy, W, H, bg, threads, lowpass_p, out_rgb, out_T, out_ops, err,
                     errlen);
}

int ref_backward_f32(const RefSceneF32* s, int p, int ox, int oy, int W, int H, const float* bg,
                     const float* dLdC, int64_t dLdC_count, int threads, int lowpass_p, float* const* grads,
                     float* pos_acc, float* col_acc, int32_t* accum, int64_t* visit,
                     int64_t* window, char* err, int errlen) {
    return do_backward(*s, p, ox, oy, W, H, bg, dLdC, dLdC_count, threads, lowpass_p, grads, pos_acc, col_acc,
                       accum, visit, window, err, errlen);
}

int ref_backward_f64(const RefSceneF64* s, int p, int ox, int oy, int W, int H, const double* bg,
                     const double* dLdC, int64_t dLdC_count, int threads, int lowpass_p, double* const* grads,
                     double* pos_acc, double* col_acc, int32_t* accum, int64_t* visit,
                     int64_t* window, char* err, int errlen) {
    return do_backward(*s, p, ox, oy, W, H, bg, dLdC, dLdC_count, threads, lowpass_p, grads, pos_acc, col_acc,
                       accum, visit, window, err, errlen);
}

// prepare_splats (rasterizer.cpp:23-46): 12 output arrays of length n in blend order:
// mean x, mean y, inv00, inv01, inv11, alpha, r, g, b, rx, ry (float) + orig (uint32).
int ref_prepare_f32(const RefSceneF32* s, int lowpass_p, float* const* out, uint32_t* orig,
                    char* err, int errlen) {
    return guarded(
        [&] {
            auto model = build_model(*s);
            auto sp = tgs::prepare_splats(model, lowpass_p);
            for (size_t i = 0; i < sp.size(); ++i) {
                out[0][i] = sp[i].mean.x;
                out[1][i] = sp[i].mean.y;
                out[2][i] = sp[i].inv00;
                out[3][i] = sp[i].inv01;
                out[4][i] = sp[i].inv11;
                out[5][i] = sp[i].alpha;
                out[6][i] = sp[i].color.x;
                out[7][i] = sp[i].color.y;
                out[8][i] = sp[i].color.z;
                out[9][i] = sp[i].rx;
                out[10][i] = sp[i].ry;
                orig[i] = sp[i].orig;
            }
        },
        err, errlen);
}

// build_tile_grid (rasterizer.cpp:67-102). offsets has tiles+1 entries; items receives up to
// items_cap entries. *out_k = total pairs. Call once with items_cap = 0 to size.
int ref_tile_grid_f32(const RefSceneF32* s, int lowpass_p, int W, int H, uint32_t* offsets,
                      uint32_t* items, int64_t items_cap, int64_t* out_k, char* err, int errlen) {
    return guarded(
        [&] {
            auto model = build_model(*s);
            auto sp = tgs::prepare_splats(model, lowpass_p);
            auto grid = tgs::build_tile_grid(sp, W, H);
            *out_k = static_cast<int64_t>(grid.items.size());
            if (offsets)
                for (size_t i = 0; i < grid.offsets.size(); ++i) offsets[i] = grid.offsets[i];
            if (items && items_cap >= static_cast<int64_t>(grid.items.size()))
                for (size_t i = 0; i < grid.items.size(); ++i) items[i] = grid.items[i];
        },
        err, errlen);
}

// GaussianModel::sorted_order (model.hpp:106-119).
int ref_sorted_order_f32(const RefSceneF32* s, uint32_t* out, char* err, int errlen) {
    return guarded(
        [&] {
            auto model = build_model(*s);
            const auto& o = model.sorted_order();
            for (size_t i = 0; i < o.size(); ++i) out[i] = o[i];
        },
        err, errlen);
}

// ---------------------------------------------------------------- persistent model session
// The reference arm of bench.py: ONE tgs::GaussianModel<float> kept across fit iterations, as
// the reference's own trainer would hold it, so GaussianModel::sorted_order stays cached until a
// structural change (model.hpp:105-119: add/compact set order_dirty_; parameter writes through
// operator[] do not). Parameters are written in place between iterations (the optimizer step);
// the DensifyStats accumulate inside the model across backward calls (rasterizer.cpp:350-358).
struct RefSession {
    tgs::GaussianModel<float> model;
};

void* ref_session_create_f32(const RefSceneF32* s, char* err, int errlen) {
    RefSession* h = nullptr;
    const int rc = guarded([&] { h = new RefSession{build_model(*s)}; }, err, errlen);
    return rc ? nullptr : h;
}

void ref_session_destroy(void* h) { delete static_cast<RefSession*>(h); }

// Forces the blend-order sort (the first-call cost the cached order amortises).
int ref_session_sort(void* h) {
    (void)static_cast<RefSession*>(h)->model.sorted_order();
    return 0;
}

// Overwrites the 9 optimised parameters (pos x/y, rot, log-scale x/y, raw opacity, raw rgb) in
// place, model index order; depth_key and id are untouched, so the cached order stays valid.
int ref_session_set_params_f32(void* h, const float* const* f) {
    auto& m = static_cast<RefSession*>(h)->model;
    const size_t n = m.size();
    for (size_t i = 0; i < n; ++i) {
        auto& g = m[i];
        g.position = {f[0][i], f[1][i]};
        g.rotation = f[2][i];
        g.log_scales = {f[3][i], f[4][i]};
        g.raw_opacity = f[5][i];
        g.color = {f[6][i], f[7][i], f[8][i]};
    }
    return 0;
}

int ref_session_render_f32(void* h, int p, int ox, int oy, int W, int H, const float* bg, int threads,
                           float* out_rgb, float* out_T, uint64_t* out_ops, char* err, int errlen) {
    auto& m = static_cast<RefSession*>(h)->model;
    return guarded(
        [&] {
            tgs::DilationPattern pat(p, ox, oy, W, H);
            tgs::RenderOptions opts;
            opts.threads = threads;
            auto out = tgs::render<float>(m, pat, tgs::Vec3<float>(bg[0], bg[1], bg[2]), opts);
            for (size_t i = 0; i < out.colors.size(); ++i) {
                out_rgb[3 * i + 0] = out.colors[i].x;
                out_rgb[3 * i + 1] = out.colors[i].y;
                out_rgb[3 * i + 2] = out.colors[i].z;
                out_T[i] = out.final_transmittance[i];
            }
            *out_ops = out.blend_op_count;
        },
        err, errlen);
}

int ref_session_backward_f32(void* h, int p, int ox, int oy, int W, int H, const float* bg,
                             const float* dLdC, int64_t dLdC_count, int threads, float* const* grads,
                             char* err, int errlen) {
    auto& m = static_cast<RefSession*>(h)->model;
    return guarded(
        [&] {
            tgs::DilationPattern pat(p, ox, oy, W, H);
            tgs::RenderOptions opts;
            opts.threads = threads;
            std::vector<tgs::Vec3<float>> g((size_t)dLdC_count);
            for (size_t i = 0; i < g.size(); ++i)
                g[i] = tgs::Vec3<float>(dLdC[3 * i], dLdC[3 * i + 1], dLdC[3 * i + 2]);
            auto gs = tgs::backward<float>(m, pat, tgs::Vec3<float>(bg[0], bg[1], bg[2]), g, opts);
            const size_t n = m.size();
            for (size_t i = 0; i < n; ++i) {
                grads[0][i] = gs.position[i].x;
                grads[1][i] = gs.position[i].y;
                grads[2][i] = gs.rotation[i];
                grads[3][i] = gs.log_scales[i].x;
                grads[4][i] = gs.log_scales[i].y;
                grads[5][i] = gs.raw_opacity[i];
                grads[6][i] = gs.color[i].x;
                grads[7][i] = gs.color[i].y;
                grads[8][i] = gs.color[i].z;
            }
        },
        err, errlen);
}

// visit_count of the persistent model's DensifyStats (model index order)
int ref_session_visits(void* h, int64_t* out) {
    const auto& st = static_cast<RefSession*>(h)->model.stats();
    for (size_t i = 0; i < st.visit_count.size(); ++i) out[i] = st.visit_count[i];
    return 0;
}

// KdTree2<float>::knn (kdtree.hpp) of every point, excluding itself: out[i*k + j] = the j-th
// nearest (ascending (dist2, index)); missing neighbours (n - 1 < k) are UINT32_MAX.
int ref_knn_f32(const float* xy, int64_t n, int k, uint32_t* out, char* err, int errlen) {
    return guarded(
        [&] {
            std::vector<tgs::Vec2<float>> pts((size_t)n);
            for (int64_t i = 0; i < n; ++i) pts[(size_t)i] = {xy[2 * i], xy[2 * i + 1]};
            tgs::KdTree2<float> tree(pts);
            for (int64_t i = 0; i < n; ++i) {
                const auto nn = tree.knn(pts[(size_t)i], k, (uint32_t)i);
                for (int j = 0; j < k; ++j) out[i * k + j] = j < (int)nn.size() ? nn[(size_t)j] : UINT32_MAX;
            }
        },
        err, errlen);
}

}  // extern "C"
