// Token-packet header writer and warp-cooperative parser (transport.py).
#pragma once

#include "common.cuh"
#include "crc32.cuh"

namespace sst {

constexpr uint32_t kMagic = 0x4D53;  // transport.py:32
constexpr uint32_t kVersion = 1;     // transport.py:33

// ">HBBIHHBBff" (transport.py:44, 97-102)
__device__ __forceinline__ void write_token_header(uint8_t* b, uint32_t kind, uint32_t gop,
                                                   uint32_t row, uint32_t width, uint32_t channels,
                                                   uint32_t scale, float qmin, float qrange) {
  put_be16(b + 0, kMagic);
  b[2] = (uint8_t)kVersion;
  b[3] = (uint8_t)kind;
  put_be32(b + 4, gop);
  put_be16(b + 8, row);
  put_be16(b + 10, width);
  b[12] = (uint8_t)channels;
  b[13] = (uint8_t)scale;
  put_be32(b + 14, __float_as_uint(qmin));
  put_be32(b + 18, __float_as_uint(qrange));
}

// parse_packet for token packets: the check order and messages follow
// transport.py:64-70 (_check_seal) and 154-184.  Whole warp; control flow is
// warp-uniform.  Result is valid in every lane.
__device__ __forceinline__ void parse_token_packet(const uint8_t* pkt, int len, bool present,
                                                   const uint32_t* tab, const uint32_t* x2n,
                                                   int lane, SstPacketInfo* out) {
  SstPacketInfo r;
  r.status = SST_PKT_OK;
  r.kind = 0; r.gop_id = 0; r.row = 0; r.width = 0; r.channels = 0; r.scale = 0; r.valid = 0;
  r.qmin = 0.f; r.qrange = 0.f; r.mask_off = kHdr; r.payload_off = kHdr;
  r.dqmin = 0.0; r.dqrange = 0.0;
  do {
    if (!present) { r.status = SST_PKT_ABSENT; break; }
    if (len < 4) { r.status = SST_PKT_SHORT; break; }
    const int body = len - 4;
    uint32_t crc = warp_crc32(pkt, body, tab, x2n, lane);
    if (crc != get_be32(pkt + body)) { r.status = SST_PKT_CRC; break; }
    if (body < 4) { r.status = SST_PKT_BODY_SHORT; break; }
    if (get_be16(pkt) != kMagic) { r.status = SST_PKT_MAGIC; break; }
    if (pkt[2] != kVersion) { r.status = SST_PKT_VERSION; break; }
    r.kind = pkt[3];
    if (r.kind != 0 && r.kind != 1) { r.status = SST_PKT_KIND; break; }
    if (body < kHdr) { r.status = SST_PKT_HDR_TRUNC; break; }
    r.gop_id = get_be32(pkt + 4);
    r.row = (int32_t)get_be16(pkt + 8);
    r.width = (int32_t)get_be16(pkt + 10);
    r.channels = pkt[12];
    r.scale = pkt[13];
    r.qmin = __uint_as_float(get_be32(pkt + 14));
    r.qrange = __uint_as_float(get_be32(pkt + 18));
    r.dqmin = (double)r.qmin;
    r.dqrange = (double)r.qrange;
    const int mlen = (r.width + 7) >> 3;
    if (body < kHdr + mlen) { r.status = SST_PKT_MASK_TRUNC; break; }
    int cnt = 0;
    for (int b = lane; b < mlen; b += 32) {
      uint32_t byte = pkt[kHdr + b];
      int rem = r.width - b * 8;
      if (rem < 8) byte &= (0xFFu << (8 - rem)) & 0xFFu;   // bits[:width] only
      cnt += __popc(byte);
    }
    cnt = __reduce_add_sync(0xffffffffu, cnt);
    r.valid = cnt;
    r.payload_off = kHdr + mlen;
    if (body - kHdr - mlen != cnt * r.channels) { r.status = SST_PKT_PAYLOAD_LEN; break; }
    if (r.qrange < 0.0f) { r.status = SST_PKT_NEG_RANGE; break; }
  } while (0);
  *out = r;
}

}  // namespace sst
