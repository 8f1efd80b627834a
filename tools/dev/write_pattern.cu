// dev probe: HBM write bandwidth of the store patterns an obs writer can use
// (not part of the product; built and run by hand on the GPU box)
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int L = 8268;            // floats per row (extended symbolic obs)
constexpr int64_t N = 65536;       // rows

__global__ void k_linear(float4* out, int64_t n4) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n4; k += (int64_t)gridDim.x * blockDim.x)
    out[k] = make_float4(0.f, 0.f, 0.f, 0.f);
}

// 256-bit stores (sm_100)
__global__ void k_linear8(float* out, int64_t n8) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n8; k += (int64_t)gridDim.x * blockDim.x) {
    float z = 0.f;
    asm volatile("st.global.v8.f32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" ::"l"(out + 8 * k), "f"(z) : "memory");
  }
}

__global__ void k_linear_unroll(float4* out, int64_t n4) {
  const int64_t T = (int64_t)gridDim.x * blockDim.x;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n4; k += 4 * T) {
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (k + u * T < n4) out[k + u * T] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
}

// one warp per row, 256-bit stores
__global__ void k_rowwarp8(float* out) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5, nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = w0; r < N; r += nw) {
    float* row = out + r * L;   // 16-byte aligned only: peel to 32
    const int head = (int)(((32 - ((uintptr_t)row & 31)) & 31) >> 2);
    if (lane < head) row[lane] = 0.f;
    float* b = row + head;
    const int n8 = (L - head) / 8;
    float z = 0.f;
    for (int q = lane; q < n8; q += 32)
      asm volatile("st.global.v8.f32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" ::"l"(b + 8 * q), "f"(z) : "memory");
    const int t0 = head + n8 * 8;
    if (t0 + lane < L) row[t0 + lane] = 0.f;
  }
}

// one warp per row, float4 stores, row-major over rows
__global__ void k_rowwarp(float* out) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5, nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = w0; r < N; r += nw) {
    float4* row = reinterpret_cast<float4*>(out + r * L);
    for (int q = lane; q < L / 4; q += 32) row[q] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
}

// one warp per row, one TMA bulk store of the whole row from a zeroed stage
template <int NW>
__global__ void k_tma(float* out, int chunk) {
  extern __shared__ float4 sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float* st = reinterpret_cast<float*>(sm) + warp * 8272;
  for (int q = lane; q < 8272 / 4; q += 32) reinterpret_cast<float4*>(st)[q] = make_float4(0.f, 0.f, 0.f, 0.f);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncwarp();
  for (int64_t r = blockIdx.x * NW + warp; r < N; r += (int64_t)gridDim.x * NW) {
    float* row = out + r * L;
    if (lane == 0) {
      const uint32_t sa = (uint32_t)__cvta_generic_to_shared(st);
      for (int off = 0; off < L * 4; off += chunk) {
        const int len = min(chunk, L * 4 - off);
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"((char*)row + off),
                     "r"(sa + off), "r"(len) : "memory");
      }
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    }
    __syncwarp();
  }
  if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// TMA, but the wait is deferred by one row (two stages per warp)
__global__ void k_tma2(float* out) {
  extern __shared__ float4 sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int NW = blockDim.x >> 5;
  float* st = reinterpret_cast<float*>(sm) + warp * 2 * 8272;
  for (int q = lane; q < 2 * 8272 / 4; q += 32) reinterpret_cast<float4*>(st)[q] = make_float4(0.f, 0.f, 0.f, 0.f);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncwarp();
  int b = 0;
  for (int64_t r = blockIdx.x * NW + warp; r < N; r += (int64_t)gridDim.x * NW) {
    float* row = out + r * L;
    if (lane == 0) {
      asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
      const uint32_t sa = (uint32_t)__cvta_generic_to_shared(st + b * 8272);
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(row), "r"(sa), "r"(L * 4)
                   : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
    b ^= 1;
    __syncwarp();
  }
  if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}


// G consecutive rows per CTA staged contiguously and drained by ONE bulk copy
// (the SM's write front is one G*33 KB stream instead of G 33 KB streams);
// NS stage sets, the wait deferred by NS-1 groups
template <int G, int NS>
__global__ void k_tma_grp(float* out, int pitch) {
  extern __shared__ float4 sm[];
  float* st = reinterpret_cast<float*>(sm);
  for (int q = threadIdx.x; q < NS * G * L / 4; q += blockDim.x) reinterpret_cast<float4*>(st)[q] = make_float4(0.f, 0.f, 0.f, 0.f);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  int b = 0;
  for (int64_t g = blockIdx.x; g * G < N; g += gridDim.x) {
    if (threadIdx.x == 0) {
      if (NS > 1) asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(NS - 1) : "memory");
      const uint32_t sa = (uint32_t)__cvta_generic_to_shared(st + b * G * L);
      if (pitch == L) {
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(out + g * G * L), "r"(sa),
                     "r"(G * L * 4) : "memory");
      } else {
        for (int k = 0; k < G; ++k)
          asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(out + (g * G + k) * (int64_t)pitch),
                       "r"(sa + k * L * 4), "r"(L * 4) : "memory");
      }
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      if (NS == 1) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    }
    b = (b + 1) % NS;
    __syncthreads();
  }
  if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

template <class F>
float timeit(F f) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int k = 0; k < 3; ++k) f();
  cudaEventRecord(a);
  for (int k = 0; k < 20; ++k) f();
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
  return ms / 20;
}

int main() {
  float* out;
  const size_t bytes = (size_t)N * L * 4;
  cudaMalloc(&out, bytes);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  auto rep = [&](const char* name, float ms) { printf("%-28s %.4f ms  %.0f GB/s\n", name, ms, bytes / ms / 1e6); };
  rep("linear 1024x sms*2", timeit([&] { k_linear<<<sms * 2, 1024>>>((float4*)out, bytes / 16); }));
  rep("memset", timeit([&] { cudaMemsetAsync(out, 0, bytes); }));
  for (int b : {2, 4, 8, 16})  {
    char nm[64];
    snprintf(nm, 64, "linear %d x256 per SM", b);
    rep(nm, timeit([&] { k_linear<<<sms * b, 256>>>((float4*)out, bytes / 16); }));
    snprintf(nm, 64, "linear8 %d x256 per SM", b);
    rep(nm, timeit([&] { k_linear8<<<sms * b, 256>>>(out, bytes / 32); }));
    snprintf(nm, 64, "linear_unroll %d x256 per SM", b);
    rep(nm, timeit([&] { k_linear_unroll<<<sms * b, 256>>>((float4*)out, bytes / 16); }));
  }
  for (int wps : {4, 8, 16, 32}) {
    char nm[64];
    snprintf(nm, 64, "rowwarp8 %d warps/SM", wps);
    rep(nm, timeit([&] { k_rowwarp8<<<sms * wps / 4, 128>>>(out); }));
  }
  for (int wps : {4, 8, 16, 32, 64}) {
    char nm[64];
    snprintf(nm, 64, "rowwarp %d warps/SM", wps);
    rep(nm, timeit([&] { k_rowwarp<<<sms * wps / 4, 128>>>(out); }));
  }
  cudaFuncSetAttribute(k_tma<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * 8272 * 4);
  cudaFuncSetAttribute(k_tma<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 1 * 8272 * 4);
  cudaFuncSetAttribute(k_tma2, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 8272 * 4);
  for (int ctas : {1, 2, 3}) {
    for (int chunk : {33072, 4096 + 16 * 0, 1024}) {
      char nm[64];
      snprintf(nm, 64, "tma 2w x %d CTA chunk %d", ctas, chunk);
      rep(nm, timeit([&] { k_tma<2><<<sms * ctas, 64, 2 * 8272 * 4>>>(out, chunk); }));
    }
  }
  for (int ctas : {4, 6}) {
    char nm[64];
    snprintf(nm, 64, "tma 1w x %d CTA", ctas);
    rep(nm, timeit([&] { k_tma<1><<<sms * ctas, 32, 8272 * 4>>>(out, 33072); }));
  }
  for (int ctas : {1, 2, 3}) {
    char nm[64];
    snprintf(nm, 64, "tma2 (2 stages) 1w x %d CTA", ctas);
    rep(nm, timeit([&] { k_tma2<<<sms * ctas, 32, 2 * 8272 * 4>>>(out); }));
  }
  {
    float* out2;
    cudaMalloc(&out2, (size_t)N * 8320 * 4);
#define GRP(G, NS, CT, P, O)                                                                              \
    {                                                                                                     \
      cudaFuncSetAttribute(k_tma_grp<G, NS>, cudaFuncAttributeMaxDynamicSharedMemorySize, NS * G * L * 4); \
      char nm[64];                                                                                        \
      snprintf(nm, 64, "tma_grp G%d NS%d %dCTA/SM pitch %d", G, NS, CT, P);                               \
      rep(nm, timeit([&] { k_tma_grp<G, NS><<<sms * CT, 32, NS * G * L * 4>>>(O, P); }));                 \
    }
    GRP(1, 1, 4, L, out) GRP(1, 2, 3, L, out) GRP(2, 1, 2, L, out) GRP(2, 2, 1, L, out) GRP(3, 1, 2, L, out)
    GRP(4, 1, 1, L, out) GRP(6, 1, 1, L, out) GRP(3, 2, 1, L, out)
    GRP(1, 1, 4, 8320, out2) GRP(2, 1, 2, 8320, out2) GRP(4, 1, 1, 8320, out2)
    GRP(1, 1, 4, 8320 - 8, out2) GRP(1, 1, 4, 8288, out2)
    cudaFree(out2);
  }
  return 0;
}
