// K2: intelligent dropping -- token_similarity, top_k_drop_mask,
// apply_token_mask (selection.py:33-79, codec.py:189-196).
//
// The top-k is an exact radix select over orderable 64-bit similarity keys
// (8 passes x 8 bits, one CTA per map) followed by an index-ordered scan of
// the keys equal to the k-th largest, which reproduces the reference's stable
// argsort tie-break (row-major order among equal similarities) without a sort.
#include "common.cuh"

namespace sst {

// numpy pairwise_sum (n <= 128 path: 8 accumulators, combine, tail); the
// reduction result is identity (0.0) + pairwise block.
__device__ double np_sum(const double* x, int n) {
  if (n < 8) {
    double r = 0.0;
    for (int i = 0; i < n; ++i) r = r + x[i];
    return 0.0 + r;
  }
  double r0 = x[0], r1 = x[1], r2 = x[2], r3 = x[3], r4 = x[4], r5 = x[5], r6 = x[6], r7 = x[7];
  int i = 8;
  for (; i < n - (n % 8); i += 8) {
    r0 = r0 + x[i]; r1 = r1 + x[i + 1]; r2 = r2 + x[i + 2]; r3 = r3 + x[i + 3];
    r4 = r4 + x[i + 4]; r5 = r5 + x[i + 5]; r6 = r6 + x[i + 6]; r7 = r7 + x[i + 7];
  }
  double r = ((r0 + r1) + (r2 + r3)) + ((r4 + r5) + (r6 + r7));
  for (; i < n; ++i) r = r + x[i];
  return 0.0 + r;
}

constexpr int kMaxSimC = 128;

// blockIdx.y = GoP g of a [G][2][n][C] token batch (pair stride gs doubles,
// sim stride n); gs = 0 for a single pair of matrices
__global__ void k_similarity(const double* __restrict__ p, const double* __restrict__ iv,
                             int64_t n, int C, double* __restrict__ sim, int64_t gs) {
  int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  const int64_t g = blockIdx.y;
  sim += g * n;
  const double* pp = p + g * gs + t * C;
  const double* ii = iv + g * gs + t * C;
  double a[kMaxSimC];
  for (int k = 0; k < C; ++k) a[k] = pp[k] * ii[k];
  double dot = np_sum(a, C);
  for (int k = 0; k < C; ++k) a[k] = pp[k] * pp[k];
  double pn = sqrt(np_sum(a, C));
  for (int k = 0; k < C; ++k) a[k] = ii[k] * ii[k];
  double in = sqrt(np_sum(a, C));
  double denom = pn * in;
  double s = denom > 0.0 ? dot / denom : 0.0;
  if (pn == 0.0 && in == 0.0) s = 1.0;
  sim[t] = clip_pm1(s);
}

// larger similarity -> larger key; -0.0 and +0.0 map to the same key
__device__ __forceinline__ uint64_t sim_key(double x) {
  if (x == 0.0) x = 0.0;
  uint64_t b = (uint64_t)__double_as_longlong(x);
  return (b & 0x8000000000000000ull) ? ~b : (b | 0x8000000000000000ull);
}

constexpr int kSelThreads = 1024;

// Per map g: drop[j] = 1 for the k[g] highest-similarity positions.
// Optionally applies the drop to the P tokens / mask of a [G][2][n][12]
// token batch and its [G][2][n] mask (fused apply_token_mask).
// PER > 0: the map's keys (n <= PER * 1024) are read from global memory once
// into registers and every radix pass and the tie scan run from there (the
// single-GoP case is latency-bound: one global round trip per pass cost
// ~4 us); PER == 0 re-reads them per pass (any n).
template <int PER>
__global__ void __launch_bounds__(kSelThreads)
    k_topk(const double* __restrict__ sim, int64_t n, const int32_t* __restrict__ kk,
           uint8_t* __restrict__ drop, double* tok, uint8_t* p_mask, double* kth) {
  __shared__ uint32_t hist[256];
  __shared__ uint64_t s_prefix;
  __shared__ int64_t s_krem;
  __shared__ int s_warp[kSelThreads / 32];
  __shared__ int64_t s_running;
  __shared__ int s_done;

  const int g = blockIdx.x;
  const int tid = threadIdx.x;
  const double* sm = sim + (int64_t)g * n;
  if (tid == 0) s_done = 0;
  int64_t k = kk[g];
  if (k < 0) k = 0;
  if (k > n) k = n;
  const int nper = (int)((n + kSelThreads - 1) / kSelThreads);
  uint64_t keys[PER > 0 ? PER : 1];
  if (PER > 0) {
#pragma unroll
    for (int i = 0; i < PER; ++i) {
      const int64_t j = (int64_t)i * kSelThreads + tid;
      keys[i] = (i < nper && j < n) ? sim_key(__ldg(sm + j)) : 0;
    }
  }
  auto key_at = [&](int i, int64_t j) -> uint64_t {
    if (PER > 0) return keys[i < PER ? i : 0];
    return sim_key(__ldg(sm + j));
  };
  const int iters = PER > 0 ? PER : nper;

  uint64_t prefix = 0, pmask = 0;
  int64_t krem = k;
  if (k > 0) {
    // radix select of the k-th largest key (1-indexed), MSB digit first
    for (int shift = 56; shift >= 0; shift -= 8) {
      for (int b = tid; b < 256; b += kSelThreads) hist[b] = 0;
      __syncthreads();
#pragma unroll
      for (int i = 0; i < iters; ++i) {
        if (i >= nper) break;                          // uniform across the CTA
        const int64_t j = (int64_t)i * kSelThreads + tid;
        uint64_t key = j < n ? key_at(i, j) : 0;
        const bool in = j < n && (key & pmask) == prefix;
        // warp-aggregated histogram update: similarity maps are dominated by
        // ties (static content), so many lanes share one bin
        const unsigned act = __ballot_sync(0xffffffffu, in);
        if (in) {
          const unsigned bin = (unsigned)((key >> shift) & 0xFF);
          const unsigned peers = __match_any_sync(act, bin);
          if ((threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(&hist[bin], (unsigned)__popc(peers));
        }
      }
      __syncthreads();
      // warp 0 locates the digit holding the krem-th largest key: suffix
      // sums over the 256 bins (8 per lane, lane 0 = top bins)
      if (tid < 32) {
        uint32_t c[8];
        uint32_t local = 0;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          c[i] = hist[255 - (tid * 8 + i)];
          local += c[i];
        }
        uint32_t incl = local;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
          if (tid >= o) incl += v;
        }
        const int64_t before = (int64_t)(incl - local);   // keys in higher digits
        const bool here = before < krem && before + (int64_t)local >= krem;
        if (here) {
          int64_t cum = before;
          int i = 0;
          for (; i < 8; ++i) {
            if (cum + c[i] >= krem) break;
            cum += c[i];
          }
          const int d = 255 - (tid * 8 + i);
          s_prefix = prefix | ((uint64_t)d << shift);
          s_krem = krem - cum;
          // every remaining candidate in this digit is dropped: the drop set
          // is exactly {key >= prefix (lower digits zero)} -- stop early
          // (not when the caller wants the k-th value itself)
          if (kth == nullptr && (int64_t)c[i] == krem - cum) s_done = 1;
        }
      }
      __syncthreads();
      prefix = s_prefix;
      krem = s_krem;
      pmask |= (0xFFull << shift);
      if (s_done) {            // uniform: T = prefix, all keys equal to T dropped
        krem = n;
        break;
      }
      __syncthreads();
    }
    // prefix is now the k-th largest key T; krem = how many of the keys == T
    // (in index order) are dropped.
  }
  if (tid == 0) s_running = 0;
  if (tid == 0 && kth != nullptr && k > 0) {      // value of the k-th largest key
    const uint64_t b = (prefix & 0x8000000000000000ull) ? (prefix & 0x7FFFFFFFFFFFFFFFull) : ~prefix;
    kth[g] = __longlong_as_double((long long)b);
  }
  __syncthreads();
  const uint64_t T = prefix;
  const int lane = tid & 31, wid = tid >> 5;
#pragma unroll
  for (int i = 0; i < iters; ++i) {
    if (i >= nper) break;
    int64_t j = (int64_t)i * kSelThreads + tid;
    uint64_t key = 0;
    bool valid = j < n;
    if (valid) key = key_at(i, j);
    bool eq = valid && k > 0 && key == T;
    unsigned bal = __ballot_sync(0xffffffffu, eq);
    int before = __popc(bal & ((1u << lane) - 1u));
    if (lane == 31) s_warp[wid] = __popc(bal);
    __syncthreads();
    int warp_off = 0;
    for (int w2 = 0; w2 < wid; ++w2) warp_off += s_warp[w2];
    int64_t rank = s_running + warp_off + before;   // index-ordered rank among equals
    if (valid) {
      bool d = k > 0 && (key > T || (eq && rank < krem));
      if (drop) drop[(int64_t)g * n + j] = d ? 1 : 0;
      if (tok) {
        // apply_token_mask on the P matrix (codec.py:189-196)
        // the batch is freshly encoded (every token valid, codec.py:155-157),
        // so mask & ~drop == ~drop: assign, which also clears an earlier
        // batch's drops without a reset pass
        uint8_t* mrow = p_mask + ((int64_t)g * 2 + 1) * n + j;   // [G][2][n]: P half
        const uint8_t nm = d ? 0 : 1;
        *mrow = nm;
        if (!nm) {
          double* v = tok + (((int64_t)g * 2 + 1) * n + j) * kChannels;
#pragma unroll
          for (int c = 0; c < kChannels; ++c) v[c] = 0.0;
        }
      }
    }
    __syncthreads();
    if (tid == 0) {
      int tot = 0;
      for (int w2 = 0; w2 < kSelThreads / 32; ++w2) tot += s_warp[w2];
      s_running += tot;
    }
    __syncthreads();
  }
}

template <typename... A>
static void launch_topk(int G, int64_t n, cudaStream_t st, A... args) {
  if (n <= 4 * kSelThreads)
    k_topk<4><<<G, kSelThreads, 0, st>>>(args...);
  else if (n <= 8 * kSelThreads)
    k_topk<8><<<G, kSelThreads, 0, st>>>(args...);
  else if (n <= 16 * kSelThreads)
    k_topk<16><<<G, kSelThreads, 0, st>>>(args...);
  else
    k_topk<0><<<G, kSelThreads, 0, st>>>(args...);
}

__global__ void k_apply_mask(double* __restrict__ values, uint8_t* __restrict__ mask,
                             const uint8_t* __restrict__ drop, int64_t n, int C) {
  int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  uint8_t nm = (mask[t] && !drop[t]) ? 1 : 0;
  mask[t] = nm;
  if (!nm) {
    double* v = values + t * C;
    for (int c = 0; c < C; ++c) v[c] = 0.0;
  }
}

}  // namespace sst

using namespace sst;

extern "C" int sst_similarity(const double* p, const double* i, int64_t n, int C, double* sim,
                              void* stream) {
  if (n < 0 || C < 0) return SST_ERR_ARG;
  if (n == 0) return SST_OK;
  if (!p || !i || !sim) return SST_ERR_ARG;
  if (C > kMaxSimC) return SST_ERR_UNSUPPORTED;
  int threads = 128;
  k_similarity<<<(unsigned)ceil_div64(n, threads), threads, 0, static_cast<cudaStream_t>(stream)>>>(
      p, i, n, C, sim, 0);
  SST_LAUNCH_CHECK();
  return SST_OK;
}

extern "C" int sst_similarity_gop(const double* tok, int G, int64_t n, int C, double* sim,
                                  void* stream) {
  if (G < 0 || n < 0 || C < 0 || G > 65535) return SST_ERR_ARG;
  if (G == 0 || n == 0) return SST_OK;
  if (!tok || !sim) return SST_ERR_ARG;
  if (C > kMaxSimC) return SST_ERR_UNSUPPORTED;
  int threads = 128;
  dim3 grid((unsigned)ceil_div64(n, threads), G);
  k_similarity<<<grid, threads, 0, static_cast<cudaStream_t>(stream)>>>(tok + n * C, tok, n, C, sim,
                                                                       2 * n * C);
  SST_LAUNCH_CHECK();
  return SST_OK;
}

extern "C" int sst_topk_mask(const double* sim, int G, int64_t n, const int32_t* k, uint8_t* drop,
                             double* kth, void* stream) {
  if (G < 0 || n < 0) return SST_ERR_ARG;
  if (G == 0 || n == 0) return SST_OK;
  if (!sim || !k || !drop) return SST_ERR_ARG;
  launch_topk(G, n, static_cast<cudaStream_t>(stream), sim, n, k, drop, (double*)nullptr,
              (uint8_t*)nullptr, kth);
  SST_LAUNCH_CHECK();
  return SST_OK;
}

extern "C" int sst_apply_mask(double* values, uint8_t* mask, const uint8_t* drop, int64_t n, int C,
                              void* stream) {
  if (n < 0 || C < 0) return SST_ERR_ARG;
  if (n == 0) return SST_OK;
  if (!values || !mask || !drop) return SST_ERR_ARG;
  int threads = 256;
  k_apply_mask<<<(unsigned)ceil_div64(n, threads), threads, 0, static_cast<cudaStream_t>(stream)>>>(
      values, mask, drop, n, C);
  SST_LAUNCH_CHECK();
  return SST_OK;
}

extern "C" int sst_select_drop(const double* sim, double* tok, uint8_t* p_mask, int G, int Ht,
                               int Wt, const int32_t* k, uint8_t* drop, void* stream) {
  if (G < 0 || Ht < 0 || Wt < 0) return SST_ERR_ARG;
  int64_t n = (int64_t)Ht * Wt;
  if (G == 0 || n == 0) return SST_OK;
  if (!sim || !tok || !p_mask || !k) return SST_ERR_ARG;
  launch_topk(G, n, static_cast<cudaStream_t>(stream), sim, n, k, drop, tok, p_mask,
              (double*)nullptr);
  SST_LAUNCH_CHECK();
  return SST_OK;
}
