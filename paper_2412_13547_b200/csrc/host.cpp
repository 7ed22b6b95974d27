// Host-side scalar logic of the fit path (product code; the oracle has its own restatement):
//  * BudgetController (Alg. 1) — EMA, log-log least squares,
//    adaptive exponent and ceiling, B(t). Pure host scalars: it consumes one loss value per
//    iteration and runs every densify interval, so it never touches the GPU hot loop.
//  * PCG32 (rng.hpp:10-46) + LCG jump-ahead for the GPU spawner's per-child streams.
//  * The seeded synthetic scene generator used by bench.py.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <new>
#include <vector>

#include "../../include/tgsx.h"

namespace {

struct Pcg {
    uint64_t state, inc;
    void init(uint64_t seed, uint64_t stream) {
        state = 0;
        inc = (stream << 1u) | 1u;
        next();
        state += seed;
        next();
    }
    uint32_t next() {
        const uint64_t old = state;
        state = old * 6364136223846793005ULL + inc;
        const uint32_t xs = (uint32_t)(((old >> 18u) ^ old) >> 27u);
        const uint32_t rot = (uint32_t)(old >> 59u);
        return (xs >> rot) | (xs << ((32u - rot) & 31u));
    }
    double uniform() { return next() * 0x1p-32; }
    double uniform_in(double lo, double hi) { return lo + (hi - lo) * uniform(); }
};

// Least-squares slope of log(y) on log(t), negated (fit_power_exponent).
bool fit_exponent(const double* t, const double* y, int64_t n, double* out) {
    if (n < 2) return false;
    double sx = 0, sy = 0;
    for (int64_t i = 0; i < n; ++i) {
        sx += std::log(t[i]);
        sy += std::log(y[i]);
    }
    const double mx = sx / (double)n, my = sy / (double)n;
    double sxx = 0, sxy = 0;
    for (int64_t i = 0; i < n; ++i) {
        const double dx = std::log(t[i]) - mx;
        sxx += dx * dx;
        sxy += dx * (std::log(y[i]) - my);
    }
    if (!(sxx > 0.0)) return false;
    *out = -(sxy / sxx);
    return true;
}

}  // namespace

struct tgsx_budget {
    // SPEC.md:390-405 fields; design decisions SPEC.md:455-459
    double n_init = 0, m_final = 0, m_adaptive = 0;
    double alpha = 1.0, alpha_base = 1.0, ema = 0;
    bool has_ema = false;
    int64_t warmup_steps = 100, window_size = 200, refit_interval = 100, ma_depth = 5;
    int64_t last_refit = -1;
    double lambda = 0.5;
    std::vector<double> log_t, log_ema, fits;
};

extern "C" {

int32_t tgsx_budget_create(double n_init, double m_final, tgsx_budget** out) {
    if (!out) return TGSX_EINVAL;
    tgsx_budget* b = new (std::nothrow) tgsx_budget();
    if (!b) return TGSX_ENOMEM;
    b->n_init = n_init;
    b->m_final = m_final;
    b->m_adaptive = m_final;
    *out = b;
    return TGSX_OK;
}

void tgsx_budget_destroy(tgsx_budget* b) { delete b; }

// record_loss
int32_t tgsx_budget_record_loss(tgsx_budget* b, int64_t t, double loss) {
    if (!b || !(loss > 0.0)) return TGSX_EINVAL;
    b->ema = b->has_ema ? 0.1 * loss + 0.9 * b->ema : loss;
    b->has_ema = true;
    if (t > b->warmup_steps) {
        b->log_t.push_back((double)t);
        b->log_ema.push_back(b->ema);
    }
    return TGSX_OK;
}

// update; eps = alpha_recent - alpha_history (the [OP] post-condition)
void tgsx_budget_update(tgsx_budget* b, int64_t t) {
    if (!b || t <= b->warmup_steps) return;
    if (b->last_refit >= 0 && t - b->last_refit < b->refit_interval) return;
    const int64_t n = (int64_t)b->log_t.size();
    double a_hist, a_recent;
    if (!fit_exponent(b->log_t.data(), b->log_ema.data(), n, &a_hist)) return;
    const int64_t w = std::min(n, b->window_size);
    if (!fit_exponent(b->log_t.data() + (n - w), b->log_ema.data() + (n - w), w, &a_recent)) return;
    b->last_refit = t;
    b->fits.push_back(a_hist);
    const int64_t d = std::min<int64_t>((int64_t)b->fits.size(), b->ma_depth);
    double s = 0;
    for (int64_t i = (int64_t)b->fits.size() - d; i < (int64_t)b->fits.size(); ++i) s += b->fits[i];
    b->alpha_base = s / (double)d;
    const double rate = a_recent;
    if (rate > 0.05) {
        b->m_adaptive = std::min(b->m_adaptive * 1.1, 1.5 * b->m_final);
    } else if (rate < -0.05) {
        b->m_adaptive = std::max(b->m_adaptive * 0.9, 0.5 * b->m_final);
    }
    const double eps = a_recent - a_hist;
    const double a = b->alpha_base + b->lambda * std::tanh(eps);
    b->alpha = a < 0.1 ? 0.1 : (a > 2.0 ? 2.0 : a);
}

// budget_at
int64_t tgsx_budget_at(const tgsx_budget* b, double t) {
    if (!b) return 0;
    t = std::min(100.0, std::max(1.0, t));
    const double frac = (std::pow(t, b->alpha) - 1.0) / (std::pow(100.0, b->alpha) - 1.0);
    return (int64_t)std::llround(b->n_init + frac * (b->m_adaptive - b->n_init));
}

void tgsx_budget_state(const tgsx_budget* b, double* out) {
    if (!b || !out) return;
    out[0] = b->alpha;
    out[1] = b->alpha_base;
    out[2] = b->m_adaptive;
    out[3] = b->ema;
    out[4] = (double)b->fits.size();
}

// t_norm = 1 + 99 (step - warmup) / (densify_end - warmup), clamped
double tgsx_budget_t_norm(int64_t step, int64_t warmup, int64_t densify_end) {
    if (densify_end <= warmup) return 100.0;
    const double t = 1.0 + 99.0 * (double)(step - warmup) / (double)(densify_end - warmup);
    return std::min(100.0, std::max(1.0, t));
}

int32_t tgsx_fit_power_exponent(const double* t, const double* y, int64_t n, double* out) {
    if (!t || !y || !out) return TGSX_EINVAL;
    return fit_exponent(t, y, n, out) ? TGSX_OK : TGSX_EINVAL;
}

// ---------------------------------------------------------------- PCG32
void tgsx_pcg32_init(uint64_t st[2], uint64_t seed, uint64_t stream) {
    Pcg p;
    p.init(seed, stream);
    st[0] = p.state;
    st[1] = p.inc;
}

double tgsx_pcg32_uniform(uint64_t st[2]) {
    Pcg p{st[0], st[1]};
    const double u = p.uniform();
    st[0] = p.state;
    return u;
}

void tgsx_pcg32_advance(uint64_t st[2], uint64_t delta) {
    uint64_t cur_mult = 6364136223846793005ULL, cur_plus = st[1];
    uint64_t acc_mult = 1u, acc_plus = 0u;
    while (delta > 0) {
        if (delta & 1) {
            acc_mult *= cur_mult;
            acc_plus = acc_plus * cur_mult + cur_plus;
        }
        cur_plus = (cur_mult + 1) * cur_plus;
        cur_mult *= cur_mult;
        delta >>= 1;
    }
    st[0] = acc_mult * st[0] + acc_plus;
}

// ---------------------------------------------------------------- synthetic scene
void tgsx_synthetic_scene(uint64_t seed, int64_t n, int32_t W, int32_t H, tgsx_host_scene* s) {
    Pcg r;
    r.init(seed, 1);
    const double pi = 3.14159265358979323846;
    for (int64_t i = 0; i < n; ++i) {
        s->px[i] = (float)r.uniform_in(0.0, (double)W);
        s->py[i] = (float)r.uniform_in(0.0, (double)H);
        s->rot[i] = (float)r.uniform_in(-pi, pi);
        s->lsx[i] = (float)r.uniform_in(0.0, 1.5);
        s->lsy[i] = (float)r.uniform_in(0.0, 1.5);
        s->rop[i] = (float)r.uniform_in(-2.0, 2.0);
        s->cr[i] = (float)r.uniform_in(-2.0, 2.0);
        s->cg[i] = (float)r.uniform_in(-2.0, 2.0);
        s->cb[i] = (float)r.uniform_in(-2.0, 2.0);
        s->depth[i] = (float)r.uniform_in(0.0, 1.0);
        if (s->id) s->id[i] = (uint64_t)i;
        if (s->tau_v) s->tau_v[i] = 5.0;
        if (s->pos_acc) s->pos_acc[i] = 0.f;
        if (s->col_acc) s->col_acc[i] = 0.f;
        if (s->accum) s->accum[i] = 0;
        if (s->visit) s->visit[i] = 0;
        if (s->window) s->window[i] = 0;
    }
    s->n = n;
    s->next_id = (uint64_t)n;
}

}  // extern "C"

// ---------------------------------------------------------------- checkpoint state
#include "host_state.h"

namespace tgsx {

void budget_write(const tgsx_budget* b, ByteWriter& w) {
    w.put(b->n_init);
    w.put(b->m_final);
    w.put(b->m_adaptive);
    w.put(b->alpha);
    w.put(b->alpha_base);
    w.put(b->ema);
    w.put((uint8_t)(b->has_ema ? 1 : 0));
    w.put(b->warmup_steps);
    w.put(b->window_size);
    w.put(b->refit_interval);
    w.put(b->ma_depth);
    w.put(b->last_refit);
    w.put(b->lambda);
    for (const std::vector<double>* v : {&b->log_t, &b->log_ema, &b->fits}) {
        w.put((uint64_t)v->size());
        w.bytes(v->data(), v->size() * sizeof(double));
    }
}

tgsx_budget* budget_clone(const tgsx_budget* b) { return new tgsx_budget(*b); }
void budget_assign(tgsx_budget* dst, const tgsx_budget* src) { *dst = *src; }

bool budget_read(tgsx_budget* b, ByteReader& r) {
    uint8_t has = 0;
    if (!(r.get(b->n_init) && r.get(b->m_final) && r.get(b->m_adaptive) && r.get(b->alpha) &&
          r.get(b->alpha_base) && r.get(b->ema) && r.get(has) && r.get(b->warmup_steps) &&
          r.get(b->window_size) && r.get(b->refit_interval) && r.get(b->ma_depth) &&
          r.get(b->last_refit) && r.get(b->lambda)))
        return false;
    b->has_ema = has != 0;
    for (std::vector<double>* v : {&b->log_t, &b->log_ema, &b->fits}) {
        uint64_t n = 0;
        if (!r.get(n) || n > (uint64_t)(r.end - r.p) / sizeof(double)) return false;
        v->resize(n);
        if (!r.bytes(v->data(), n * sizeof(double))) return false;
    }
    return true;
}

}  // namespace tgsx
