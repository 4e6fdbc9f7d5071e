// Bump allocator over one caller-provided device workspace (the C ABI never
// allocates on the hot path; bse_*_workspace_bytes() sizes the buffer).
#pragma once
#include <cstddef>
#include <cstdint>

namespace bse {

struct Arena {
  char* base = nullptr;
  size_t size = 0;
  size_t used = 0;
  bool dry = false;  // sizing pass: count bytes, hand out nullptr

  template <typename T>
  T* take(size_t count) {
    const size_t bytes = ((count * sizeof(T) + 255) / 256) * 256;
    if (dry) { used += bytes; return nullptr; }
    if (used + bytes > size) return nullptr;
    T* p = reinterpret_cast<T*>(base + used);
    used += bytes;
    return p;
  }
};

// Leading dimension used for internal N x N matrices: even and padded to a
// multiple of 32 doubles (256 B) so every column starts 16-byte aligned.
inline long long pad_ld(long long n) { return ((n + 31) / 32) * 32 + (n == 0 ? 32 : 0); }

}  // namespace bse
