// TGS1 checkpoint (SPEC.md:637-646 save_checkpoint / load_checkpoint; the reference's CLI
// sources are missing, the format is the SPEC's): little-endian
//
//   header (24 B)   "TGS1", u32 version (1), u64 count, u64 next_id
//   parameters      position f32[count][2], rotation f32[count], log_scales f32[count][2],
//                   raw_opacity f32[count], color f32[count][3], depth_key f32[count]
//                   (declared field order, gaussian.hpp:35-44), id u64[count]
//   DensifyStats    pos_acc f32, col_acc f32, accum i32, visit i64, window i64, tau_v f64 [count]
//   moments         m f32[9][count], v f32[9][count]
//   u32 has_state   then, when 1, the trainer: iteration, Adam step, RNG, loss ring and the
//                   BudgetController (scalars + its log-log fit history)
//
// Load validates magic, version and every length (corrupt / truncated -> TGSX_ERUNTIME, the
// reference's runtime_error) and restores the model in logical order with its moments; a
// save of the loaded state is byte-identical.
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/tgsx.h"
#include "host_state.h"

using tgsx::ByteReader;
using tgsx::ByteWriter;

namespace {

constexpr char kMagic[4] = {'T', 'G', 'S', '1'};
constexpr uint32_t kVersion = 1;

struct HostModel {
    int64_t n = 0;
    std::vector<float> px, py, rot, lsx, lsy, rop, cr, cg, cb, depth, pos_acc, col_acc, m1, m2;
    std::vector<uint64_t> id;
    std::vector<int32_t> accum;
    std::vector<int64_t> visit, window;
    std::vector<double> tau_v;
    uint64_t next_id = 0;
    void resize(int64_t count) {
        n = count;
        for (auto* v : {&px, &py, &rot, &lsx, &lsy, &rop, &cr, &cg, &cb, &depth, &pos_acc, &col_acc})
            v->resize((size_t)count);
        m1.resize((size_t)count * 9);
        m2.resize((size_t)count * 9);
        id.resize((size_t)count);
        accum.resize((size_t)count);
        visit.resize((size_t)count);
        window.resize((size_t)count);
        tau_v.resize((size_t)count);
    }
    tgsx_host_scene scene() {
        tgsx_host_scene s{};
        s.n = n;
        s.px = px.data(); s.py = py.data(); s.rot = rot.data(); s.lsx = lsx.data(); s.lsy = lsy.data();
        s.rop = rop.data(); s.cr = cr.data(); s.cg = cg.data(); s.cb = cb.data(); s.depth = depth.data();
        s.id = id.data();
        s.next_id = next_id;
        s.pos_acc = pos_acc.data(); s.col_acc = col_acc.data(); s.accum = accum.data();
        s.visit = visit.data(); s.window = window.data(); s.tau_v = tau_v.data();
        return s;
    }
};

}  // namespace

extern "C" {

int32_t tgsx_checkpoint_save(tgsx_ctx* ctx, tgsx_model* m, const tgsx_trainer* tr, const char* path) {
    if (!ctx || !m || !path) return TGSX_EINVAL;
    HostModel h;
    h.resize(tgsx_model_size(m));
    tgsx_host_scene s = h.scene();
    int32_t rc = tgsx_model_download(ctx, m, &s);
    if (rc) return rc;
    h.next_id = s.next_id;
    if ((rc = tgsx_model_download_moments(ctx, m, h.m1.data(), h.m2.data()))) return rc;
    std::vector<uint8_t> buf;
    ByteWriter w{buf};
    w.bytes(kMagic, 4);
    w.put(kVersion);
    w.put((uint64_t)h.n);
    w.put(h.next_id);
    const size_t n = (size_t)h.n;
    for (size_t i = 0; i < n; ++i) { w.put(h.px[i]); w.put(h.py[i]); }
    w.bytes(h.rot.data(), n * 4);
    for (size_t i = 0; i < n; ++i) { w.put(h.lsx[i]); w.put(h.lsy[i]); }
    w.bytes(h.rop.data(), n * 4);
    for (size_t i = 0; i < n; ++i) { w.put(h.cr[i]); w.put(h.cg[i]); w.put(h.cb[i]); }
    w.bytes(h.depth.data(), n * 4);
    w.bytes(h.id.data(), n * 8);
    w.bytes(h.pos_acc.data(), n * 4);
    w.bytes(h.col_acc.data(), n * 4);
    w.bytes(h.accum.data(), n * 4);
    w.bytes(h.visit.data(), n * 8);
    w.bytes(h.window.data(), n * 8);
    w.bytes(h.tau_v.data(), n * 8);
    w.bytes(h.m1.data(), n * 36);
    w.bytes(h.m2.data(), n * 36);
    w.put((uint32_t)(tr ? 1 : 0));
    if (tr) tgsx::trainer_write(tr, w);
    FILE* f = std::fopen(path, "wb");
    if (!f) return TGSX_EINVAL;
    const size_t wrote = std::fwrite(buf.data(), 1, buf.size(), f);
    const int closed = std::fclose(f);
    return (wrote == buf.size() && closed == 0) ? TGSX_OK : TGSX_ERUNTIME;
}

int32_t tgsx_checkpoint_load(tgsx_ctx* ctx, tgsx_model* m, tgsx_trainer* tr, const char* path) {
    if (!ctx || !m || !path) return TGSX_EINVAL;
    FILE* f = std::fopen(path, "rb");
    if (!f) return TGSX_EINVAL;
    std::vector<uint8_t> buf;
    uint8_t chunk[1 << 16];
    size_t got;
    while ((got = std::fread(chunk, 1, sizeof(chunk), f)) > 0) buf.insert(buf.end(), chunk, chunk + got);
    std::fclose(f);
    ByteReader r{buf.data(), buf.data() + buf.size()};
    char magic[4];
    uint32_t version = 0;
    uint64_t count = 0, next_id = 0;
    if (!r.bytes(magic, 4) || std::memcmp(magic, kMagic, 4) != 0 || !r.get(version) || version != kVersion ||
        !r.get(count) || !r.get(next_id))
        return TGSX_ERUNTIME;
    // every array must fit in what remains: 156 B per Gaussian
    if (count > (uint64_t)(r.end - r.p) / 156) return TGSX_ERUNTIME;
    HostModel h;
    h.resize((int64_t)count);
    h.next_id = next_id;
    const size_t n = (size_t)count;
    bool ok = true;
    for (size_t i = 0; i < n && ok; ++i) ok = r.get(h.px[i]) && r.get(h.py[i]);
    ok = ok && r.bytes(h.rot.data(), n * 4);
    for (size_t i = 0; i < n && ok; ++i) ok = r.get(h.lsx[i]) && r.get(h.lsy[i]);
    ok = ok && r.bytes(h.rop.data(), n * 4);
    for (size_t i = 0; i < n && ok; ++i) ok = r.get(h.cr[i]) && r.get(h.cg[i]) && r.get(h.cb[i]);
    ok = ok && r.bytes(h.depth.data(), n * 4) && r.bytes(h.id.data(), n * 8) &&
         r.bytes(h.pos_acc.data(), n * 4) && r.bytes(h.col_acc.data(), n * 4) &&
         r.bytes(h.accum.data(), n * 4) && r.bytes(h.visit.data(), n * 8) &&
         r.bytes(h.window.data(), n * 8) && r.bytes(h.tau_v.data(), n * 8) &&
         r.bytes(h.m1.data(), n * 36) && r.bytes(h.m2.data(), n * 36);
    uint32_t has_state = 0;
    int32_t rc_parse = TGSX_OK;
    ok = ok && r.get(has_state) && has_state <= 1;
    if (!ok) return TGSX_ERUNTIME;
    if (has_state && !tr) return TGSX_EINVAL;  // training state needs a trainer to restore into
    // parse and validate EVERYTHING before touching the caller's model or trainer: a corrupt or
    // truncated trainer section (or trailing bytes) leaves both exactly as they were
    tgsx::TrainerState st;
    if (has_state && (rc_parse = tgsx::trainer_parse(tr, r, st))) return rc_parse;
    if (r.p != r.end) return TGSX_ERUNTIME;  // trailing bytes: not a TGS1 file
    tgsx_host_scene s = h.scene();
    int32_t rc = tgsx_model_upload(ctx, m, &s);
    if (rc) return rc;
    if ((rc = tgsx_model_upload_moments(ctx, m, h.m1.data(), h.m2.data()))) return rc;
    if (has_state && (rc = tgsx::trainer_commit(tr, st))) return rc;
    return TGSX_OK;
}

}  // extern "C"
