// Device side of the TCRVMSK mask file format (tensorio.py:80-100, §8f-3): each row of
// the (..., M_total) mask is packed into big-endian bits (np.packbits order: column 8b
// is the MSB of byte b), padded to a byte.  The device mask is packed little-endian in
// uint32 words (bit j of word w = column 32w + j), so a file write is a per-byte bit
// reversal of the device words (2.7 MB D2H at C2 instead of a 20.8 MB dense bool mask)
// and a file read unpacks straight into the dense byte form tcb_mask_pack consumes.
#include "common.cuh"

namespace tcb {

__global__ void __launch_bounds__(256) k_words_to_packbits(const uint32_t* __restrict__ words,
                                                           int64_t rows, int M_total, int W,
                                                           int P, uint8_t* __restrict__ out) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= rows * P) return;
  const int64_t r = e / P;
  const int b = (int)(e - r * P);
  uint32_t x = (words[r * W + (b >> 2)] >> (8 * (b & 3))) & 0xffu;
  const int valid = M_total - 8 * b;  // columns of this byte inside the row
  if (valid < 8) x &= (1u << valid) - 1u;
  out[e] = (uint8_t)(__brev(x) >> 24);
}

__global__ void __launch_bounds__(256) k_packbits_to_dense(const uint8_t* __restrict__ packed,
                                                           int64_t rows, int M_total, int P,
                                                           uint8_t* __restrict__ dense) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= rows * M_total) return;
  const int64_t r = e / M_total;
  const int j = (int)(e - r * M_total);
  dense[e] = (packed[r * P + (j >> 3)] >> (7 - (j & 7))) & 1u;
}

}  // namespace tcb

using namespace tcb;

extern "C" int tcb_mask_words_to_packbits(const uint32_t* words, int64_t rows, int M_total,
                                          int words_per_row, uint8_t* packed, void* stream) {
  TCB_CHECK_ARG(words && packed, TCB_ESHAPE, "null tensor");
  TCB_CHECK_ARG(M_total >= 1 && words_per_row * 32 >= M_total, TCB_ESHAPE, "bad row width");
  const int P = (M_total + 7) / 8;
  if (rows == 0) return TCB_OK;
  k_words_to_packbits<<<(unsigned)ceil_div(rows * P, 256), 256, 0, as_stream(stream)>>>(
      words, rows, M_total, words_per_row, P, packed);
  return check_launch("k_words_to_packbits");
}

extern "C" int tcb_packbits_to_dense(const uint8_t* packed, int64_t rows, int M_total,
                                     uint8_t* dense, void* stream) {
  TCB_CHECK_ARG(packed && dense, TCB_ESHAPE, "null tensor");
  TCB_CHECK_ARG(M_total >= 1, TCB_ESHAPE, "bad row width");
  if (rows == 0) return TCB_OK;
  const int P = (M_total + 7) / 8;
  k_packbits_to_dense<<<(unsigned)ceil_div(rows * M_total, 256), 256, 0, as_stream(stream)>>>(
      packed, rows, M_total, P, dense);
  return check_launch("k_packbits_to_dense");
}
