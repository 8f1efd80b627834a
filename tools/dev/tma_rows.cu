// Dev probe: can the TMA unit replicate a frame's class rows into the
// output at HBM rate?  Pixel frames (ext 10 px: 110 rows x 390 B = 42,900 B,
// frames back to back) have rows at arbitrary byte alignment, so plain
// cp.async.bulk (16-byte aligned) cannot store them; a 1-D uint8 tensor map
// can (box 256 + box 128 per row, the last 6 bytes by st.global).
// Measures GB/s of: (a) TMA per-row stores from smem class rows, (b) the
// register path (16-byte st.global per thread, funnel-shifted from smem).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/tma_rows tools/dev/tma_rows.cu
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <vector>

constexpr int RB = 390, FH = 110, FB = RB * FH, NCLS = 40, PSTR = 512;

__device__ __forceinline__ int cls_of(int y) { return (y / 10) * 4 + (y % 10 == 0 ? 1 : 0); }

template <int MODE>
__global__ void __launch_bounds__(256) k_rows(const __grid_constant__ CUtensorMap m256,
                                              const __grid_constant__ CUtensorMap m128, uint8_t* out, int64_t n,
                                              int reps, int align) {
  extern __shared__ __align__(1024) uint8_t pat[];   // NCLS rows of PSTR bytes
  for (int k = threadIdx.x; k < NCLS * PSTR; k += blockDim.x) pat[k] = (uint8_t)(k * 7 + blockIdx.x);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  for (int rep = 0; rep < reps; ++rep)
  for (int64_t i = blockIdx.x; i < n; i += gridDim.x) {
    const int64_t f0 = i * (int64_t)FB;
    if (MODE == 0) {
      // each of 2 * FH TMA ops issued by its own thread
      for (int q = threadIdx.x; q < 2 * FH; q += blockDim.x) {
        const int y = q >> 1, half = q & 1;
        const uint32_t src = (uint32_t)__cvta_generic_to_shared(pat + cls_of(y) * PSTR + half * 256);
        int32_t x = (int32_t)(f0 + (int64_t)y * RB + half * 256);
        if (align) x &= ~15;
        if (!half)
          asm volatile("cp.async.bulk.tensor.1d.global.shared::cta.bulk_group [%0, {%1}], [%2];"
                       ::"l"(&m256), "r"(x), "r"(src) : "memory");
        else
          asm volatile("cp.async.bulk.tensor.1d.global.shared::cta.bulk_group [%0, {%1}], [%2];"
                       ::"l"(&m128), "r"(x), "r"(src) : "memory");
      }
      // tails: 6 bytes per row
      for (int q = threadIdx.x; q < FH * 6; q += blockDim.x) {
        const int y = q / 6, b = q % 6;
        out[f0 + (int64_t)y * RB + 384 + b] = pat[cls_of(y) * PSTR + 384 + b];
      }
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    } else {
      // register path: aligned 16-byte chunks, funnel shifts from smem words
      const int64_t c0 = (f0 + 15) & ~15ll, c1 = (f0 + FB) & ~15ll;
      const int nch = (int)((c1 - c0) >> 4);
      for (int q = threadIdx.x; q < nch; q += blockDim.x) {
        const int b = (int)(c0 - f0) + 16 * q, y = b / RB, o = b - y * RB;
        if (o + 16 > RB) continue;
        const uint32_t* w = reinterpret_cast<const uint32_t*>(pat + cls_of(y) * PSTR) + (o >> 2);
        const int sh = (o & 3) * 8;
        *reinterpret_cast<uint4*>(out + c0 + 16 * q) =
            make_uint4(__funnelshift_r(w[0], w[1], sh), __funnelshift_r(w[1], w[2], sh),
                       __funnelshift_r(w[2], w[3], sh), __funnelshift_r(w[3], w[4], sh));
      }
    }
  }
  if (MODE == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main(int argc, char** argv) {
  const int64_t n = argc > 1 ? atoll(argv[1]) : 65536;
  const int align = argc > 2 ? atoi(argv[2]) : 0;
  const size_t bytes = (size_t)n * FB;
  uint8_t* out;
  cudaMalloc(&out, bytes + 4096);
  PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  if (!enc) { printf("no cuTensorMapEncodeTiled\n"); return 1; }
  CUtensorMap m256, m128;
  cuuint64_t dim[1] = {(cuuint64_t)bytes};
  cuuint64_t strides[1] = {0};
  cuuint32_t box256[1] = {256}, box128[1] = {128}, es[1] = {1};
  CUresult r1 = enc(&m256, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, out, dim, strides, box256, es,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  CUresult r2 = enc(&m128, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, out, dim, strides, box128, es,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r1 || r2) { printf("encode failed %d %d\n", (int)r1, (int)r2); return 1; }
  const int smem = NCLS * PSTR;
  cudaFuncSetAttribute(k_rows<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k_rows<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  // correctness of the TMA path against the register path
  std::vector<uint8_t> a(bytes), b(bytes);
  for (int mode = 0; mode < 2; ++mode) {
    cudaMemset(out, 0, bytes);
    if (mode == 0) k_rows<0><<<sms * 4, 256, smem>>>(m256, m128, out, n, 1, align);
    else k_rows<1><<<sms * 4, 256, smem>>>(m256, m128, out, n, 1, align);
    cudaError_t e = cudaDeviceSynchronize();
    if (e) { printf("mode %d: %s\n", mode, cudaGetErrorString(e)); return 1; }
    cudaMemcpy(mode == 0 ? a.data() : b.data(), out, bytes, cudaMemcpyDeviceToHost);
  }
  // the register path leaves the straddling chunks / frame head+tail at 0: compare rows' interiors only
  int64_t diff = 0;
  for (int64_t i = 0; i < n; ++i)
    for (int y = 0; y < FH; ++y) {
      const int64_t s = i * FB + (int64_t)y * RB;
      const int64_t lo = (s + 15) & ~15ll, hi = (s + RB) & ~15ll;
      for (int64_t k = lo; k < hi; ++k) diff += a[k] != b[k];
    }
  printf("interior bytes differing: %lld\n", (long long)diff);
  for (int ctas : {1, 2, 4, 8}) {
    for (int mode = 0; mode < 2; ++mode) {
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      for (int w = 0; w < 2; ++w) {
        if (mode == 0) k_rows<0><<<sms * ctas, 256, smem>>>(m256, m128, out, n, 1, align);
        else k_rows<1><<<sms * ctas, 256, smem>>>(m256, m128, out, n, 1, align);
      }
      cudaEventRecord(e0);
      const int it = 10;
      for (int w = 0; w < it; ++w) {
        if (mode == 0) k_rows<0><<<sms * ctas, 256, smem>>>(m256, m128, out, n, 1, align);
        else k_rows<1><<<sms * ctas, 256, smem>>>(m256, m128, out, n, 1, align);
      }
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      ms /= it;
      printf("ctas/SM %d mode %s: %.3f ms  %.1f GB/s  (%s)\n", ctas, mode == 0 ? "tma-rows" : "registers", ms,
             bytes / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
