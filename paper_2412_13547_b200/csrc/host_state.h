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
void trainer_write(const tgsx_trainer* tr, ByteWriter& w);
int32_t trainer_read(tgsx_trainer* tr, ByteReader& r);  // TGSX_OK, TGSX_ERUNTIME (corrupt)

}  // namespace tgsx
