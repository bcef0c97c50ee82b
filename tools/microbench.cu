// microbench.cu -- B200 (sm_100a) ceilings that bound the K3 interpolation kernel (DESIGN.md
// section 7): FP64 FMA (DFMA), FP32 FMA (FFMA and packed FFMA2 = fma.rn.f32x2), the shared-memory
// -> register path (LDS.64 / LDS.128, conflict-free, and with random per-lane window origins like
// K3's), and a plain HBM read for reference.  Each kernel runs over the whole GPU (148 SMs x
// several CTAs), timed with CUDA events after a warm-up; prints one JSON object.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o microbench tools/microbench.cu && ./microbench
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>

#define CK(x)                                                                   \
  do {                                                                          \
    cudaError_t e = (x);                                                        \
    if (e != cudaSuccess) {                                                     \
      fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e));                   \
      exit(1);                                                                  \
    }                                                                           \
  } while (0)

constexpr int kIters = 4096;
constexpr int kChains = 8;

__global__ void k_dfma(double* out, double a, double b) {
  double x[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) x[c] = threadIdx.x * 1e-3 + c;
  for (int i = 0; i < kIters; ++i) {
#pragma unroll
    for (int c = 0; c < kChains; ++c) x[c] = fma(x[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s += x[c];
  if (s == 1.2345) out[0] = s;
}

__global__ void k_ffma(float* out, float a, float b) {
  float x[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) x[c] = threadIdx.x * 1e-3f + c;
  for (int i = 0; i < kIters; ++i) {
#pragma unroll
    for (int c = 0; c < kChains; ++c) x[c] = fmaf(x[c], a, b);
  }
  float s = 0;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s += x[c];
  if (s == 1.2345f) out[0] = s;
}

__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
  float2 r;
  asm("{\n\t.reg .b64 ra, rb, rc, rd;\n\t"
      "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\tmov.b64 rc, {%6, %7};\n\t"
      "fma.rn.f32x2 rd, ra, rb, rc;\n\tmov.b64 {%0, %1}, rd;\n\t}"
      : "=f"(r.x), "=f"(r.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
  return r;
}

__global__ void k_ffma2(float* out, float a, float b) {
  float2 x[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) x[c] = make_float2(threadIdx.x * 1e-3f + c, c);
  const float2 A = make_float2(a, a), B = make_float2(b, b);
  for (int i = 0; i < kIters; ++i) {
#pragma unroll
    for (int c = 0; c < kChains; ++c) x[c] = ffma2(x[c], A, B);
  }
  float s = 0;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s += x[c].x + x[c].y;
  if (s == 1.2345f) out[0] = s;
}

// shared -> register: each thread reads 16 B (or 8 B) per load from a per-lane origin.
// mode 0: lane-contiguous (conflict-free); mode 1: random origins (K3-like windows);
// mode 2: all lanes of a warp read the same address (broadcast)
template <int BYTES>
__global__ void k_lds(float* out, int mode, int seed) {
  __shared__ __align__(16) float buf[8192];  // 32 KB
  for (int i = threadIdx.x; i < 8192; i += blockDim.x) buf[i] = i * 1e-3f;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  constexpr int W = BYTES / 4;
  unsigned h = (threadIdx.x * 2654435761u) ^ (seed * 40503u);
  int base;
  if (mode == 0)  // lane l of a warp reads bytes [BYTES l, BYTES (l + 1)) of the warp's block
    base = (threadIdx.x * W) % 4096;
  else if (mode == 1)
    base = ((h >> 7) % (8192 / W - 128)) * W;
  else
    base = (threadIdx.x >> 5) * 64;
  (void)lane;
  float acc = 0;
  const unsigned sbase = (unsigned)__cvta_generic_to_shared(buf);
  for (int i = 0; i < kIters; ++i) {
    // asm volatile: every load is issued (no hoisting / CSE of the periodic addresses)
    const unsigned addr = sbase + 4u * (unsigned)(base + ((i * 8 * W) & 255));
    if constexpr (W == 4) {
      float a, b, c, d;
      asm volatile("ld.volatile.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(a), "=f"(b), "=f"(c), "=f"(d) : "r"(addr));
      acc += a + b + c + d;
    } else {
      float a, b;
      asm volatile("ld.volatile.shared.v2.f32 {%0, %1}, [%2];" : "=f"(a), "=f"(b) : "r"(addr));
      acc += a + b;
    }
  }
  if (acc == 1.2345f) out[0] = acc;
}

__global__ void k_read(const float4* __restrict__ in, long long n, float* out) {
  float4 acc = make_float4(0, 0, 0, 0);
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    float4 v = in[i];
    acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
  }
  if (acc.x + acc.y + acc.z + acc.w == 1.2345f) out[0] = 1;
}

template <class F>
static float time_ms(F launch, int reps = 5) {
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  launch();
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int r = 0; r < reps; ++r) {
    CK(cudaEventRecord(a));
    launch();
    CK(cudaEventRecord(b));
    CK(cudaEventSynchronize(b));
    float ms;
    CK(cudaEventElapsedTime(&ms, a, b));
    if (ms < best) best = ms;
  }
  return best;
}

int main() {
  int sms = 0, clk_khz = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  CK(cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0));
  float* d;
  CK(cudaMalloc(&d, 64));
  const int blocks = sms * 8, threads = 256;
  const double lanes = (double)blocks * threads;
  const double fmas = lanes * kIters * kChains;
  float t_dfma = time_ms([&] { k_dfma<<<blocks, threads>>>((double*)d, 0.999, 1e-3); });
  float t_ffma = time_ms([&] { k_ffma<<<blocks, threads>>>(d, 0.999f, 1e-3f); });
  float t_ffma2 = time_ms([&] { k_ffma2<<<blocks, threads>>>(d, 0.999f, 1e-3f); });
  const double lds_bytes16 = lanes * kIters * 16.0, lds_bytes8 = lanes * kIters * 8.0;
  float t_lds128[3], t_lds64[3];
  for (int m = 0; m < 3; ++m) {
    t_lds128[m] = time_ms([&] { k_lds<16><<<blocks, threads>>>(d, m, 7); });
    t_lds64[m] = time_ms([&] { k_lds<8><<<blocks, threads>>>(d, m, 7); });
  }
  const long long n4 = (4ll << 30) / 16;  // 4 GiB
  float4* big;
  CK(cudaMalloc(&big, n4 * 16));
  CK(cudaMemset(big, 0, n4 * 16));
  float t_read = time_ms([&] { k_read<<<sms * 16, 512>>>(big, n4, d); });
  const double clk = clk_khz * 1e3;
  auto per_clk_sm = [&](double ops, float ms) { return ops / (ms * 1e-3) / clk / sms; };
  printf("{\"sms\": %d, \"clock_mhz_attr\": %.0f,\n", sms, clk / 1e6);
  printf(" \"dfma_tflops\": %.2f, \"dfma_per_clk_sm\": %.1f,\n", 2 * fmas / (t_dfma * 1e-3) / 1e12, per_clk_sm(fmas, t_dfma));
  printf(" \"ffma_tflops\": %.2f, \"ffma_per_clk_sm\": %.1f,\n", 2 * fmas / (t_ffma * 1e-3) / 1e12, per_clk_sm(fmas, t_ffma));
  printf(" \"ffma2_tflops\": %.2f, \"ffma2_fma_per_clk_sm\": %.1f,\n", 4 * fmas / (t_ffma2 * 1e-3) / 1e12,
         per_clk_sm(2 * fmas, t_ffma2));
  const char* names[3] = {"contiguous", "random_origins", "broadcast"};
  for (int m = 0; m < 3; ++m)
    printf(" \"lds128_%s_TBps\": %.2f, \"lds128_%s_B_per_clk_sm\": %.1f,\n", names[m],
           lds_bytes16 / (t_lds128[m] * 1e-3) / 1e12, names[m], per_clk_sm(lds_bytes16, t_lds128[m]));
  for (int m = 0; m < 3; ++m)
    printf(" \"lds64_%s_TBps\": %.2f, \"lds64_%s_B_per_clk_sm\": %.1f,\n", names[m],
           lds_bytes8 / (t_lds64[m] * 1e-3) / 1e12, names[m], per_clk_sm(lds_bytes8, t_lds64[m]));
  printf(" \"hbm_read_GBps\": %.0f,\n", n4 * 16.0 / (t_read * 1e-3) / 1e9);
  printf(" \"note\": \"per_clk figures use the attribute clock (max); time by CUDA events, best of 5\"}\n");
  return 0;
}
