__device__ __forceinline__ void colrange16(uint32_t* kmn, uint32_t* kmx, int b4, int b3, int b2, int b1, uint32_t* omn,
                                           uint32_t* omx) {
#pragma unroll
  for (int k = 0; k < 8; ++k) {   // offset 16: keep columns 8 b4 + k
    const uint32_t smn = b4 ? kmn[k] : kmn[8 + k], smx = b4 ? kmx[k] : kmx[8 + k];
    const uint32_t rmn = __shfl_xor_sync(0xffffffffu, smn, 16), rmx = __shfl_xor_sync(0xffffffffu, smx, 16);
    kmn[k] = min(b4 ? kmn[8 + k] : kmn[k], rmn);
    kmx[k] = max(b4 ? kmx[8 + k] : kmx[k], rmx);
  }
#pragma unroll
  for (int k = 0; k < 4; ++k) {   // offset 8
    const uint32_t smn = b3 ? kmn[k] : kmn[4 + k], smx = b3 ? kmx[k] : kmx[4 + k];
    const uint32_t rmn = __shfl_xor_sync(0xffffffffu, smn, 8), rmx = __shfl_xor_sync(0xffffffffu, smx, 8);
    kmn[k] = min(b3 ? kmn[4 + k] : kmn[k], rmn);
    kmx[k] = max(b3 ? kmx[4 + k] : kmx[k], rmx);
  }
#pragma unroll
  for (int k = 0; k < 2; ++k) {   // offset 4
    const uint32_t smn = b2 ? kmn[k] : kmn[2 + k], smx = b2 ? kmx[k] : kmx[2 + k];
    const uint32_t rmn = __shfl_xor_sync(0xffffffffu, smn, 4), rmx = __shfl_xor_sync(0xffffffffu, smx, 4);
    kmn[k] = min(b2 ? kmn[2 + k] : kmn[k], rmn);
    kmx[k] = max(b2 ? kmx[2 + k] : kmx[k], rmx);
  }
  {   // offset 2
    const uint32_t smn = b1 ? kmn[0] : kmn[1], smx = b1 ? kmx[0] : kmx[1];
    const uint32_t rmn = __shfl_xor_sync(0xffffffffu, smn, 2), rmx = __shfl_xor_sync(0xffffffffu, smx, 2);
    kmn[0] = min(b1 ? kmn[1] : kmn[0], rmn);
    kmx[0] = max(b1 ? kmx[1] : kmx[0], rmx);
  }
  *omn = min(kmn[0], __shfl_xor_sync(0xffffffffu, kmn[0], 1));   // offset 1: both lanes of the pair
  *omx = max(kmx[0], __shfl_xor_sync(0xffffffffu, kmx[0], 1));
}

