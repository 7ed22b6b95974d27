// Byte-level state of the host-side controllers, for the TGS1 checkpoint (checkpoint.cpp).
#pragma once

#include <cstdint>
#include <cstring>
#include <vector>

#include "../../include/tgsx.h"

namespace tgsx {

// little-endian append / bounded read helpers
struct ByteWriter {
    std::vector<uint8_t>& out;
    template <typename T>
    void put(const T& v) {
        const uint8_t* p = reinterpret_cast<const uint8_t*>(&v);
        out.insert(out.end(), p, p + sizeof(T));
    }
    void bytes(const void* p, size_t n) {
        const uint8_t* b = static_cast<const uint8_t*>(p);
        out.insert(out.end(), b, b + n);
    }
};

struct ByteReader {
    const uint8_t* p;
    const uint8_t* end;
    template <typename T>
    bool get(T& v) {
        if ((size_t)(end - p) < sizeof(T)) return false;
        std::memcpy(&v, p, sizeof(T));
        p += sizeof(T);
        return true;
    }
    bool bytes(void* dst, size_t n) {
        if ((size_t)(end - p) < n) return false;
        std::memcpy(dst, p, n);
        p += n;
        return true;
    }
};

void budget_write(const tgsx_budget* b, ByteWriter& w);
bool budget_read(tgsx_budget* b, ByteReader& r);
tgsx_budget* budget_clone(const tgsx_budget* b);
void budget_assign(tgsx_budget* dst, const tgsx_budget* src);
void trainer_write(const tgsx_trainer* tr, ByteWriter& w);

// Training state parsed from a checkpoint, not yet applied: the load parses everything first and
// changes the caller's model / trainer only once the whole file has been validated.
struct TrainerState {
    int64_t t = 0, adam_step = 0, n_init = 0, fed = 0, ring = 0;
    uint64_t rng[2] = {0, 0};
    double last_budget = 0;
    std::vector<float> losses;
    tgsx_budget* budget = nullptr;  // owned (destroyed by the destructor)
    TrainerState() = default;
    TrainerState(const TrainerState&) = delete;
    TrainerState& operator=(const TrainerState&) = delete;
    ~TrainerState();
};
int32_t trainer_parse(const tgsx_trainer* tr, ByteReader& r, TrainerState& st);  // OK / ERUNTIME
int32_t trainer_commit(tgsx_trainer* tr, const TrainerState& st);                // OK / ECUDA

}  // namespace tgsx
