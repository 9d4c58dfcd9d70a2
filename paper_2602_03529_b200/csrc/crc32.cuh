// CRC-32/ISO-HDLC (zlib.crc32, transport.py:56-57) computed by a whole warp.
//
// Each lane runs the byte-serial table CRC over its own contiguous chunk of
// the packet; the chunk CRCs are then merged with the GF(2) shift operator
// crc(A||B) = x^(8|B|) * crc(A) xor crc(B)  (mod the reflected polynomial),
// evaluated with a compile-time table of x^(2^k).  No global state, no host
// tables: everything is constexpr.
#pragma once

#include <cstdint>

namespace sst {

constexpr uint32_t kCrcPoly = 0xEDB88320u;

struct CrcTables {
  uint32_t byte[256];
  uint32_t x2n[32];   // x^(2^k) mod P, reflected
};

constexpr uint32_t crc_multmodp(uint32_t a, uint32_t b) {
  uint32_t m = 1u << 31, p = 0;
  for (;;) {
    if (a & m) {
      p ^= b;
      if ((a & (m - 1)) == 0) break;
    }
    m >>= 1;
    b = (b & 1) ? (b >> 1) ^ kCrcPoly : b >> 1;
  }
  return p;
}

constexpr CrcTables make_crc_tables() {
  CrcTables t{};
  for (uint32_t n = 0; n < 256; ++n) {
    uint32_t c = n;
    for (int k = 0; k < 8; ++k) c = (c & 1) ? kCrcPoly ^ (c >> 1) : c >> 1;
    t.byte[n] = c;
  }
  uint32_t p = 1u << 30;  // x^1
  t.x2n[0] = p;
  for (int n = 1; n < 32; ++n) t.x2n[n] = p = crc_multmodp(p, p);
  return t;
}

// x^(8n) mod P for n < kShiftN: appending n zero bytes is one multiply
constexpr int kShiftN = 4096;
struct CrcShiftTable {
  uint32_t v[kShiftN];
};
constexpr CrcShiftTable make_crc_shift_table() {
  CrcShiftTable t{};
  uint32_t x8 = 1u << 30;                                   // x^1
  for (int i = 0; i < 3; ++i) x8 = crc_multmodp(x8, x8);    // x^8
  uint32_t p = 1u << 31;                                    // x^0
  for (int n = 0; n < kShiftN; ++n) {
    t.v[n] = p;
    p = crc_multmodp(x8, p);
  }
  return t;
}
__device__ const CrcShiftTable kCrcShift = make_crc_shift_table();

__device__ __forceinline__ uint32_t crc_mul(uint32_t a, uint32_t b) {
  uint32_t m = 1u << 31, p = 0;
  while (true) {
    if (a & m) {
      p ^= b;
      if ((a & (m - 1)) == 0) break;
    }
    m >>= 1;
    b = (b & 1) ? (b >> 1) ^ kCrcPoly : b >> 1;
  }
  return p;
}

// x^(8n) mod P: the operator that appends n zero bytes.
__device__ __forceinline__ uint32_t crc_shift_op(uint32_t n, const uint32_t* x2n) {
  uint32_t p = 1u << 31;  // x^0
  int k = 3;
  while (n) {
    if (n & 1) p = crc_mul(x2n[k & 31], p);
    n >>= 1;
    ++k;
  }
  return p;
}

// Warp-cooperative zlib.crc32 of `len` bytes at `data` (any memory space the
// caller can read bytewise).  `tab` is the 256-entry byte table (shared mem).
// All 32 lanes must call; every lane receives the result.
__device__ __forceinline__ uint32_t warp_crc32(const uint8_t* data, int len, const uint32_t* tab,
                                               const uint32_t* x2n, int lane) {
  int chunk = (len + 31) >> 5;
  int beg = lane * chunk;
  int end = beg + chunk;
  if (beg > len) beg = len;
  if (end > len) end = len;
  uint32_t c = 0xFFFFFFFFu;
  for (int i = beg; i < end; ++i) c = tab[(c ^ data[i]) & 0xFFu] ^ (c >> 8);
  c = ~c;                                    // == zlib.crc32(chunk); 0 for an empty chunk
  uint32_t part = 0u;
  if (end > beg) {
    const uint32_t n = (uint32_t)(len - end);
    const uint32_t op = n < (uint32_t)kShiftN ? __ldg(&kCrcShift.v[n]) : crc_shift_op(n, x2n);
    part = crc_mul(op, c);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) part ^= __shfl_xor_sync(0xffffffffu, part, o);
  return part;
}

}  // namespace sst
