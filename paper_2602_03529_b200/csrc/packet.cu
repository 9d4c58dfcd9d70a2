// K3 / K4a: the token wire format (transport.py).
//
//   packetize_tokens + TokenPacket.to_bytes  (transport.py:236-271, 97-102)
//   parse_packet for token packets            (transport.py:154-184)
//   reassemble (first-wins, zero-fill)        (transport.py:274-305, 195-199)
//
// One warp builds (or validates) one row packet: a warp-wide masked min/max,
// the float32 wire grid, rint quantisation, ballot/popc compaction of the
// valid tokens, the big-endian header and mask bytes, and a warp-parallel
// CRC-32 (per-lane table CRC merged with GF(2) shift operators), staged in
// shared memory and written to the arena with 16-byte stores.
#include "common.cuh"
#include "crc32.cuh"
#include "packet_util.cuh"

namespace sst {

// global (not __constant__): the table fill reads 32 different entries per warp
__device__ const CrcTables kCrc = make_crc_tables();

constexpr int kPackWarps = 4;

struct PackArgs {
  const double* values;
  const uint8_t* mask;
  int m, Ht, Wt, C;
  const uint8_t* kind;
  const uint32_t* gop_id;
  const uint8_t* scale;
  uint8_t* arena;
  int64_t slot;
  int64_t scratch;   // per-warp smem: slot bytes + Wt prefix ints [+ row staging], 16-aligned
  int32_t* lengths;
  int64_t rowbuf;    // byte offset of the row staging (Wt*C doubles + Wt mask bytes) or 0
};

__device__ __forceinline__ void load_crc_tables(uint32_t* tab, uint32_t* x2n) {
  for (int i = threadIdx.x; i < 256; i += blockDim.x) tab[i] = __ldg(&kCrc.byte[i]);
  for (int i = threadIdx.x; i < 32; i += blockDim.x) x2n[i] = __ldg(&kCrc.x2n[i]);
}

// Seal the body staged in `buf` (len bytes) with its CRC and copy the packet
// to dst (16-byte aligned).  Whole warp.
__device__ __forceinline__ int seal_and_store(uint8_t* buf, int len, uint8_t* dst, const uint32_t* tab,
                                              const uint32_t* x2n, int lane) {
  __syncwarp();
  uint32_t crc = warp_crc32(buf, len, tab, x2n, lane);
  if (lane == 0) put_be32(buf + len, crc);
  __syncwarp();
  const int total = len + 4;
  const int n16 = (total + 15) >> 4;
  const uint4* s4 = reinterpret_cast<const uint4*>(buf);
  uint4* d4 = reinterpret_cast<uint4*>(dst);
  for (int i = lane; i < n16; i += 32) d4[i] = s4[i];
  return total;
}

__global__ void __launch_bounds__(kPackWarps * 32) k_packetize(PackArgs a) {
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ uint32_t tab[256];
  __shared__ uint32_t x2n[32];
  load_crc_tables(tab, x2n);

  const int lane = threadIdx.x & 31;
  const int wid = threadIdx.x >> 5;
  const int64_t pk = (int64_t)blockIdx.x * kPackWarps + wid;
  const int Wt = a.Wt, C = a.C;
  const int mlen = (Wt + 7) >> 3;
  // per-warp scratch: staging bytes (slot) + prefix counts (Wt ints)
  uint8_t* buf = smem + wid * a.scratch;
  int32_t* pre = reinterpret_cast<int32_t*>(buf + a.slot);
  __syncthreads();
  if (pk >= (int64_t)a.m * a.Ht) return;

  const int mi = (int)(pk / a.Ht);
  const int row = (int)(pk % a.Ht);
  const double* vrow = a.values + ((int64_t)mi * a.Ht + row) * Wt * C;
  const uint8_t* mrow = a.mask ? a.mask + ((int64_t)mi * a.Ht + row) * Wt : nullptr;
  const int64_t nel = (int64_t)Wt * C;
  // per-warp row staging (when it fits): the row's values and mask bytes are
  // read from global memory once, with all of a lane's loads in flight
  // together, and every later pass reads shared memory (the payload pass used
  // to issue one dependent global load per element: latency-bound for a
  // single GoP)
  double* rowv = a.rowbuf ? reinterpret_cast<double*>(buf + a.rowbuf) : nullptr;
  uint8_t* rowm = a.rowbuf ? reinterpret_cast<uint8_t*>(rowv + nel) : nullptr;
  if (rowm) {
    for (int t = lane; t < Wt; t += 32) rowm[t] = mrow ? (mrow[t] != 0) : 1;
    __syncwarp();
  }
  auto valid_tok = [&](int t) -> bool {
    return rowm ? rowm[t] != 0 : (mrow ? mrow[t] != 0 : true);
  };

  // 1) valid-token prefix counts (ballot scan) and mask bytes, MSB first
  int running = 0;
  for (int base = 0; base < Wt; base += 32) {
    int t = base + lane;
    bool v = t < Wt && valid_tok(t);
    unsigned bal = __ballot_sync(0xffffffffu, v);
    if (t < Wt) pre[t] = running + __popc(bal & ((1u << lane) - 1u));
    running += __popc(bal);
  }
  const int nvalid = running;
  __syncwarp();
  for (int b = lane; b < mlen; b += 32) {
    uint32_t byte = 0;
    for (int q = 0; q < 8; ++q) {
      int t = b * 8 + q;
      bool v = t < Wt && valid_tok(t);
      byte |= (v ? 1u : 0u) << (7 - q);
    }
    buf[kHdr + b] = (uint8_t)byte;
  }

  // 2) masked row min / max over the valid tokens (transport.py:249-253)
  double lo = 0.0, hi = 0.0;
  bool any = false;
  // token-major fast path (C = 12, row staged): lane l owns tokens l, l+32,
  // ...: six 16-byte loads per token, all of a lane's tokens in flight, and
  // no per-element index divisions
  const bool tok_major = rowv != nullptr && C == kChannels;
  if (tok_major) {
    for (int t0 = lane; t0 < Wt; t0 += 32 * 2) {
      double2 v[2][6];
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int t = t0 + 32 * u;
        const double2* src = reinterpret_cast<const double2*>(vrow + (int64_t)t * kChannels);
#pragma unroll
        for (int i = 0; i < 6; ++i) v[u][i] = t < Wt ? __ldg(src + i) : make_double2(0.0, 0.0);
      }
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int t = t0 + 32 * u;
        if (t >= Wt) continue;
        double2* dst = reinterpret_cast<double2*>(rowv + t * kChannels);
#pragma unroll
        for (int i = 0; i < 6; ++i) dst[i] = v[u][i];
        if (!valid_tok(t)) continue;
#pragma unroll
        for (int i = 0; i < 6; ++i) {
          const double x0 = v[u][i].x, x1 = v[u][i].y;
          if (!any) { lo = x0; hi = x0; any = true; }
          else { lo = min_total(lo, x0); hi = max_total(hi, x0); }
          lo = min_total(lo, x1);
          hi = max_total(hi, x1);
        }
      }
    }
  } else {
    // batches of 8 independent loads per lane keep several requests in flight
    for (int e0 = lane; e0 < (int)nel; e0 += 32 * 8) {
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int e = e0 + 32 * u;
        v[u] = e < nel ? __ldg(vrow + e) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int e = e0 + 32 * u;
        if (e >= nel) continue;
        if (rowv) rowv[e] = v[u];
        if (!valid_tok(e / C)) continue;
        if (!any) { lo = v[u]; hi = v[u]; any = true; }
        else { lo = min_total(lo, v[u]); hi = max_total(hi, v[u]); }
      }
    }
  }
  // lanes without values contribute neutral elements
  const double kInf = __longlong_as_double(0x7ff0000000000000ll);
  if (!any) { lo = kInf; hi = -kInf; }
  lo = warp_min_total(lo);
  hi = warp_max_total(hi);
  __syncwarp();

  double qmin32 = 0.0, qrange32 = 0.0;
  if (nvalid > 0) {
    double qrange = hi - lo;
    qmin32 = round_f32(lo);
    qrange32 = round_f32(qrange);
  }
  // 3) payload: C bytes per valid token, compacted in ascending column order
  uint8_t* pay = buf + kHdr + mlen;
  const bool scaled = qrange32 > 0.0;
  const double mul = scaled ? 255.0 / qrange32 : 0.0;
  if (tok_major) {
    for (int t = lane; t < Wt; t += 32) {
      if (!valid_tok(t)) continue;
      uint8_t* dst = pay + pre[t] * kChannels;
      const double* x = rowv + t * kChannels;
#pragma unroll
      for (int c = 0; c < kChannels; ++c) {
        uint8_t q = 0;
        if (scaled) {
          double lv = rint((x[c] - qmin32) * mul);
          lv = lv < 0.0 ? 0.0 : (lv > 255.0 ? 255.0 : lv);
          q = (uint8_t)(int)lv;
        }
        dst[c] = q;
      }
    }
  } else {
    for (int e = lane; e < (int)nel; e += 32) {
      int t = e / C;
      if (!valid_tok(t)) continue;
      int c = e - t * C;
      uint8_t q = 0;
      if (scaled) {
        const double x = rowv ? rowv[e] : vrow[e];
        double lv = rint((x - qmin32) * mul);
        lv = lv < 0.0 ? 0.0 : (lv > 255.0 ? 255.0 : lv);
        q = (uint8_t)(int)lv;
      }
      pay[pre[t] * C + c] = q;
    }
  }
  // 4) header (transport.py:97-102)
  if (lane == 0) {
    write_token_header(buf, a.kind[mi], a.gop_id[mi], (uint32_t)row, (uint32_t)Wt, (uint32_t)C,
                       a.scale[mi], (float)qmin32, (float)qrange32);
  }
  const int body = kHdr + mlen + nvalid * C;
  uint8_t* dst = a.arena + pk * a.slot;
  int total = seal_and_store(buf, body, dst, tab, x2n, lane);
  if (lane == 0) a.lengths[pk] = total;
}

// TokenPacket.to_bytes for field-wise packets (user-constructed TokenPacket).
__global__ void __launch_bounds__(kPackWarps * 32)
    k_serialize(const SstPacketInfo* __restrict__ info, const uint8_t* __restrict__ masks,
                const int64_t* __restrict__ mask_off, const uint8_t* __restrict__ payload,
                const int64_t* __restrict__ payload_off, int64_t n, uint8_t* out,
                const int64_t* __restrict__ out_off, int64_t max_bytes) {
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ uint32_t tab[256];
  __shared__ uint32_t x2n[32];
  load_crc_tables(tab, x2n);
  const int lane = threadIdx.x & 31;
  const int wid = threadIdx.x >> 5;
  const int64_t i = (int64_t)blockIdx.x * kPackWarps + wid;
  uint8_t* buf = smem + wid * max_bytes;
  __syncthreads();
  if (i >= n) return;
  const SstPacketInfo p = info[i];
  const int mlen = (p.width + 7) >> 3;
  const int plen = p.valid * p.channels;
  for (int b = lane; b < mlen; b += 32) buf[kHdr + b] = masks[mask_off[i] + b];
  for (int b = lane; b < plen; b += 32) buf[kHdr + mlen + b] = payload[payload_off[i] + b];
  if (lane == 0)
    write_token_header(buf, (uint32_t)p.kind, p.gop_id, (uint32_t)p.row, (uint32_t)p.width,
                       (uint32_t)p.channels, (uint32_t)p.scale, p.qmin, p.qrange);
  __syncwarp();
  const int body = kHdr + mlen + plen;
  uint32_t crc = warp_crc32(buf, body, tab, x2n, lane);
  if (lane == 0) put_be32(buf + body, crc);
  __syncwarp();
  uint8_t* dst = out + out_off[i];
  for (int b = lane; b < body + 4; b += 32) dst[b] = buf[b];
}

// parse_packet (token kinds) -- validation order mirrors transport.py:154-184
__global__ void __launch_bounds__(kPackWarps * 32)
    k_parse(const uint8_t* __restrict__ buf, const int64_t* __restrict__ off,
            const int32_t* __restrict__ len, const uint8_t* __restrict__ present, int64_t n,
            SstPacketInfo* __restrict__ info) {
  __shared__ uint32_t tab[256];
  __shared__ uint32_t x2n[32];
  load_crc_tables(tab, x2n);
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t i = (int64_t)blockIdx.x * kPackWarps + (threadIdx.x >> 5);
  if (i >= n) return;
  SstPacketInfo r;
  parse_token_packet(buf + off[i], len[i], present ? present[i] != 0 : true, tab, x2n, lane, &r);
  if (lane == 0) info[i] = r;
}

// ---- reassemble ----------------------------------------------------------

__global__ void k_reasm_init(uint32_t* winner, int64_t nrows, int32_t* stats, int m) {
  int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t < nrows) winner[t] = 0xFFFFFFFFu;
  if (t < 2 * (int64_t)m) stats[t] = 0;
}

// route packets to their matrix rows; first arrival (lowest index) wins
__global__ void k_route(SstPacketInfo* info, const int32_t* __restrict__ target, int64_t n, int m,
                        int Ht, const uint8_t* __restrict__ exp_kind,
                        const uint32_t* __restrict__ exp_gop, uint32_t* winner, int32_t* stats) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  SstPacketInfo& p = info[i];
  if (p.status != SST_PKT_OK) return;
  int t = target[i];
  if (t < 0 || t >= m) {
    p.status = SST_PKT_FOREIGN;
    return;
  }
  int kind_exp = exp_kind ? exp_kind[t] : (t & 1);
  uint32_t gop_exp = exp_kind ? exp_gop[t] : exp_gop[t >> 1];
  if (p.kind != kind_exp || p.gop_id != gop_exp) {
    p.status = SST_PKT_FOREIGN;
    return;
  }
  if (p.row >= Ht) {
    p.status = SST_PKT_ROW_RANGE;
    atomicAdd(&stats[2 * t], 1);
    return;
  }
  atomicMin(&winner[(int64_t)t * Ht + p.row], (uint32_t)i);
}

__global__ void k_mark_dups(SstPacketInfo* info, const int32_t* __restrict__ target, int64_t n,
                            int Ht, const uint32_t* __restrict__ winner) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  SstPacketInfo& p = info[i];
  if (p.status != SST_PKT_OK) return;
  if (winner[(int64_t)target[i] * Ht + p.row] != (uint32_t)i) p.status = SST_PKT_DUP;
}

// one warp per matrix row: dequantise the winner's payload (transport.py:108-112,
// 296-305), zero-fill everything else
__global__ void __launch_bounds__(256)
    k_scatter(const uint8_t* __restrict__ buf, const int64_t* __restrict__ off,
              SstPacketInfo* info, int m, int Ht, int Wt, int C,
              const uint32_t* __restrict__ winner, double* __restrict__ values,
              uint8_t* __restrict__ mask, int32_t* stats) {
  const int lane = threadIdx.x & 31;
  const int64_t r = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (r >= (int64_t)m * Ht) return;
  const int t = (int)(r / Ht);
  double* vrow = values + r * Wt * C;
  uint8_t* mrow = mask + r * Wt;
  const uint32_t w = winner[r];
  if (w == 0xFFFFFFFFu) {
    for (int64_t e = lane; e < (int64_t)Wt * C; e += 32) vrow[e] = 0.0;
    for (int x = lane; x < Wt; x += 32) mrow[x] = 0;
    return;
  }
  SstPacketInfo& p = info[w];
  const uint8_t* pkt = buf + off[w];
  const uint8_t* mb = pkt + p.mask_off;
  const uint8_t* pay = pkt + p.payload_off;
  // shape check: width >= Wt with no valid bits past Wt, channels == C
  bool bad = p.channels != C || p.width < Wt;
  for (int x = Wt + lane; !bad && x < p.width; x += 32)
    if ((mb[x >> 3] >> (7 - (x & 7))) & 1) bad = true;
  bad = __any_sync(0xffffffffu, bad);
  if (bad) {
    if (lane == 0) p.status = SST_PKT_SHAPE;
    for (int64_t e = lane; e < (int64_t)Wt * C; e += 32) vrow[e] = 0.0;
    for (int x = lane; x < Wt; x += 32) mrow[x] = 0;
    return;
  }
  if (lane == 0) atomicAdd(&stats[2 * t + 1], 1);
  const double qmin = p.dqmin;
  const double step = p.dqrange / 255.0;
  // prefix counts via ballot, then dequantise
  int running = 0;
  for (int base = 0; base < Wt; base += 32) {
    int x = base + lane;
    bool v = x < Wt && ((mb[x >> 3] >> (7 - (x & 7))) & 1);
    unsigned bal = __ballot_sync(0xffffffffu, v);
    int pre = running + __popc(bal & ((1u << lane) - 1u));
    if (x < Wt) {
      mrow[x] = v ? 1 : 0;
      double* dst = vrow + (int64_t)x * C;
      if (v) {
        const uint8_t* src = pay + (int64_t)pre * C;
        for (int c = 0; c < C; ++c) dst[c] = qmin + (double)src[c] * step;
      } else {
        for (int c = 0; c < C; ++c) dst[c] = 0.0;
      }
    }
    running += __popc(bal);
  }
}

}  // namespace sst

using namespace sst;

extern "C" int64_t sst_packet_wire_size(int width_tokens, int channels, int valid_count) {
  if (valid_count < 0) valid_count = width_tokens;
  return (int64_t)kHdr + (width_tokens + 7) / 8 + (int64_t)valid_count * channels + 4;
}

extern "C" int sst_packetize(const double* values, const uint8_t* mask, int m, int Ht, int Wt, int C,
                             const uint8_t* kind, const uint32_t* gop_id, const uint8_t* scale,
                             uint8_t* arena, int64_t slot, int32_t* lengths, void* stream) {
  if (m < 0 || Ht < 0 || Wt < 0 || C < 0) return SST_ERR_ARG;
  if (Ht > 0xFFFF) return SST_ERR_ROWS_16BIT;
  if (Wt > 0xFFFF || C > 0xFF) return SST_ERR_ARG;
  if (m == 0 || Ht == 0) return SST_OK;
  if (!values || !kind || !gop_id || !scale || !arena || !lengths) return SST_ERR_ARG;
  if (slot < sst_packet_wire_size(Wt, C, Wt) || (slot & 15)) return SST_ERR_ARG;
  if (reinterpret_cast<uintptr_t>(arena) & 15) return SST_ERR_ARG;
  int64_t scratch = slot + (int64_t)Wt * 4;
  scratch = (scratch + 15) & ~(int64_t)15;
  int64_t rowbuf = scratch;
  int64_t staged = rowbuf + (int64_t)Wt * C * 8 + Wt;
  staged = (staged + 15) & ~(int64_t)15;
  if (staged * kPackWarps <= 160 * 1024) scratch = staged;   // row staging fits
  else rowbuf = 0;
  PackArgs a{values, mask, m, Ht, Wt, C, kind, gop_id, scale, arena, slot, scratch, lengths, rowbuf};
  int64_t smem = scratch * kPackWarps;
  if (smem > 200 * 1024) return SST_ERR_UNSUPPORTED;
  SST_CUDA_TRY(cudaFuncSetAttribute(k_packetize, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)smem));
  int64_t npk = (int64_t)m * Ht;
  k_packetize<<<(unsigned)ceil_div64(npk, kPackWarps), kPackWarps * 32, (size_t)smem,
                static_cast<cudaStream_t>(stream)>>>(a);
  SST_LAUNCH_CHECK();
  return SST_OK;
}

extern "C" int sst_serialize(const SstPacketInfo* info, const uint8_t* masks, const int64_t* mask_off,
                             const uint8_t* payload, const int64_t* payload_off, int64_t n,
                             uint8_t* out, const int64_t* out_off, void* stream) {
  if (n < 0) return SST_ERR_ARG;
  if (n == 0) return SST_OK;
  if (!info || !masks || !mask_off || !payload || !payload_off || !out || !out_off)
    return SST_ERR_ARG;
  // staging must hold the largest packet: 22 + 8192 + 65535*255 is too much;
  // callers (the Python mirror) pass packets of ordinary size -- bound at 48 KB
  const int64_t max_bytes = 48 * 1024;
  SST_CUDA_TRY(cudaFuncSetAttribute(k_serialize, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)(max_bytes * kPackWarps)));
  k_serialize<<<(unsigned)ceil_div64(n, kPackWarps), kPackWarps * 32, (size_t)(max_bytes * kPackWarps),
                static_cast<cudaStream_t>(stream)>>>(info, masks, mask_off, payload, payload_off, n,
                                                     out, out_off, max_bytes);
  SST_LAUNCH_CHECK();
  return SST_OK;
}

extern "C" int sst_parse(const uint8_t* buf, const int64_t* off, const int32_t* len,
                         const uint8_t* present, int64_t n, SstPacketInfo* info, void* stream) {
  if (n < 0) return SST_ERR_ARG;
  if (n == 0) return SST_OK;
  if (!buf || !off || !len || !info) return SST_ERR_ARG;
  k_parse<<<(unsigned)ceil_div64(n, kPackWarps), kPackWarps * 32, 0,
            static_cast<cudaStream_t>(stream)>>>(buf, off, len, present, n, info);
  SST_LAUNCH_CHECK();
  return SST_OK;
}

namespace sst {
int route_packets(SstPacketInfo* info, const int32_t* target, int64_t n, int m, int Ht,
                  const uint8_t* exp_kind, const uint32_t* exp_gop, uint32_t* winner,
                  int32_t* stats, cudaStream_t st) {
  int64_t nrows = (int64_t)m * Ht;
  int64_t ninit = nrows > 2 * (int64_t)m ? nrows : 2 * (int64_t)m;
  k_reasm_init<<<(unsigned)ceil_div64(ninit, 256), 256, 0, st>>>(winner, nrows, stats, m);
  SST_LAUNCH_CHECK();
  if (n > 0) {
    k_route<<<(unsigned)ceil_div64(n, 256), 256, 0, st>>>(info, target, n, m, Ht, exp_kind, exp_gop,
                                                         winner, stats);
    SST_LAUNCH_CHECK();
    k_mark_dups<<<(unsigned)ceil_div64(n, 256), 256, 0, st>>>(info, target, n, Ht, winner);
    SST_LAUNCH_CHECK();
  }
  return SST_OK;
}
}  // namespace sst

extern "C" int sst_reassemble(const uint8_t* buf, const int64_t* off, SstPacketInfo* info,
                              const int32_t* target, int64_t n, int m, int Ht, int Wt, int C,
                              const uint8_t* exp_kind, const uint32_t* exp_gop, uint32_t* winner,
                              double* values, uint8_t* mask, int32_t* stats, void* stream) {
  if (n < 0 || m < 0 || Ht < 0 || Wt < 0 || C < 0) return SST_ERR_ARG;
  if (m == 0) return SST_OK;
  if (!exp_kind || !exp_gop || !winner || !values || !mask || !stats) return SST_ERR_ARG;
  if (n > 0 && (!buf || !off || !info || !target)) return SST_ERR_ARG;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int rc = route_packets(info, target, n, m, Ht, exp_kind, exp_gop, winner, stats, st);
  if (rc != SST_OK) return rc;
  int64_t nrows = (int64_t)m * Ht;
  if (nrows > 0) {
    k_scatter<<<(unsigned)ceil_div64(nrows, 8), 256, 0, st>>>(buf, off, info, m, Ht, Wt, C, winner,
                                                               values, mask, stats);
    SST_LAUNCH_CHECK();
  }
  return SST_OK;
}
