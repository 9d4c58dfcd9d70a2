// Host-side tensor map encoding (cuTensorMapEncodeTiled via the runtime's
// driver entry point, so the library does not link libcuda directly).
#include <cudaTypedefs.h>
#include <mutex>

#include "tma.cuh"
#include "tc.cuh"

namespace sst {

static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

bool make_tmap_f32_3d(CUtensorMap* map, const void* base, uint64_t dim0, uint64_t dim1,
                      uint64_t dim2, uint32_t box0, uint32_t box1) {
  auto fn = encode_fn();
  if (!fn) return false;
  const uint64_t row_bytes = dim0 * sizeof(float);
  if ((reinterpret_cast<uintptr_t>(base) & 15u) || (row_bytes & 15u)) return false;
  if (box0 > 256 || box1 > 256 || (box0 * sizeof(float)) % 16 != 0) return false;
  if (dim0 >= (1ull << 32) || dim1 >= (1ull << 32) || dim2 >= (1ull << 32)) return false;
  cuuint64_t gdim[3] = {dim0, dim1, dim2};
  cuuint64_t gstride[2] = {row_bytes, row_bytes * dim1};
  cuuint32_t box[3] = {box0, box1, 1};
  cuuint32_t estride[3] = {1, 1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<void*>(base), gdim, gstride,
                  box, estride, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

}  // namespace sst

namespace sst {

// bf16 tensor maps for the tcgen05 convolutions (tc.cuh): 128-byte swizzle,
// out-of-bounds boxes zero-filled (the convolution halo / causal padding).
bool make_tmap_bf16_5d(CUtensorMap* map, const void* base, const uint64_t dims[5], uint32_t b1,
                       uint32_t b2) {
  auto fn = encode_fn();
  if (!fn) return false;
  if (reinterpret_cast<uintptr_t>(base) & 15u) return false;
  cuuint64_t gdim[5];
  cuuint64_t gstride[4];
  uint64_t stride = 2;
  for (int i = 0; i < 5; ++i) {
    if (dims[i] == 0 || dims[i] >= (1ull << 32)) return false;
    gdim[i] = dims[i];
    stride *= dims[i];
    if (i < 4) gstride[i] = stride;
  }
  if (gstride[0] & 15u) return false;
  cuuint32_t box[5] = {64, b1, b2, 1, 1};
  cuuint32_t estride[5] = {1, 1, 1, 1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, const_cast<void*>(base), gdim, gstride,
                  box, estride, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

bool make_tmap_bf16_2d(CUtensorMap* map, const void* base, uint64_t d0, uint64_t d1, uint32_t b1) {
  auto fn = encode_fn();
  if (!fn) return false;
  if ((reinterpret_cast<uintptr_t>(base) & 15u) || ((d0 * 2) & 15u)) return false;
  cuuint64_t gdim[2] = {d0, d1};
  cuuint64_t gstride[1] = {d0 * 2};
  cuuint32_t box[2] = {64, b1};
  cuuint32_t estride[2] = {1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), gdim, gstride,
                  box, estride, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

}  // namespace sst

namespace sst {

// int8 activations / weights of the int8 learned tokenizer (learned_i8.cu):
// the same 128-byte swizzled K-major tiles, 128 one-byte elements per row.
bool make_tmap_u8_5d(CUtensorMap* map, const void* base, const uint64_t dims[5], uint32_t b1,
                     uint32_t b2) {
  auto fn = encode_fn();
  if (!fn) return false;
  if (reinterpret_cast<uintptr_t>(base) & 15u) return false;
  cuuint64_t gdim[5];
  cuuint64_t gstride[4];
  uint64_t stride = 1;
  for (int i = 0; i < 5; ++i) {
    if (dims[i] == 0 || dims[i] >= (1ull << 32)) return false;
    gdim[i] = dims[i];
    stride *= dims[i];
    if (i < 4) gstride[i] = stride;
  }
  if (gstride[0] & 15u) return false;
  cuuint32_t box[5] = {128, b1, b2, 1, 1};
  cuuint32_t estride[5] = {1, 1, 1, 1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 5, const_cast<void*>(base), gdim, gstride,
                  box, estride, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

bool make_tmap_u8_2d(CUtensorMap* map, const void* base, uint64_t d0, uint64_t d1, uint32_t b1) {
  auto fn = encode_fn();
  if (!fn) return false;
  if ((reinterpret_cast<uintptr_t>(base) & 15u) || (d0 & 15u)) return false;
  cuuint64_t gdim[2] = {d0, d1};
  cuuint64_t gstride[1] = {d0};
  cuuint32_t box[2] = {128, b1};
  cuuint32_t estride[2] = {1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), gdim, gstride,
                  box, estride, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

}  // namespace sst

namespace sst {

// uint8 3-D map without swizzle (K5-9's byte windows of the int8 tokenizer's
// working frames): dims {d0 (bytes), d1, d2}, box {box0, box1, 1}
bool make_tmap_u8_3d(CUtensorMap* map, const void* base, uint64_t dim0, uint64_t dim1,
                     uint64_t dim2, uint32_t box0, uint32_t box1) {
  auto fn = encode_fn();
  if (!fn) return false;
  if ((reinterpret_cast<uintptr_t>(base) & 15u) || (dim0 & 15u)) return false;
  if (box0 > 256 || box1 > 256 || box0 % 16 != 0) return false;
  if (dim0 >= (1ull << 32) || dim1 >= (1ull << 32) || dim2 >= (1ull << 32)) return false;
  cuuint64_t gdim[3] = {dim0, dim1, dim2};
  cuuint64_t gstride[2] = {dim0, dim0 * dim1};
  cuuint32_t box[3] = {box0, box1, 1};
  cuuint32_t estride[3] = {1, 1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<void*>(base), gdim, gstride,
                  box, estride, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

}  // namespace sst
