// Probe: how fast can the decode-attention access pattern stream from HBM
// when the consumer does no math? Each warp walks (sample, head) items of
// 32-token K|V units of a paged pool (layout of the engine's pool, 2-D TMA
// boxes of 32 rows x 128 B, 128B swizzle) through a private ring of S stages
// on mbarriers and only waits for the data. Compare its GB/s with the real
// kernel's (tools/attn_roofline.py) to split "memory-pattern bound" from
// "consumer bound".
//
//   nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a tools/kv_stream_probe.cu -lcuda -o kv_probe
//   ./kv_probe B mean_ctx warps stages
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <array>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#define CK(x)                                                                              \
  do {                                                                                     \
    cudaError_t e_ = (x);                                                                  \
    if (e_ != cudaSuccess) {                                                               \
      std::printf("CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__);       \
      std::exit(1);                                                                        \
    }                                                                                      \
  } while (0)

constexpr int kPT = 64, kHD = 64, kKVH = 12, kL = 12;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__global__ void probe_kernel(const __grid_constant__ CUtensorMap map, const int* __restrict__ items, int n_items,
                             const int* __restrict__ bt, int bt_stride, const int* __restrict__ ctx, int rows_per_page,
                             int layer, int stages, int* counter, unsigned long long* sink) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ __align__(8) uint64_t bars[16][8];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint64_t* bar = bars[warp];
  uint8_t* ring = smem + warp * stages * 8192;
  if (lane == 0) {
    for (int s = 0; s < stages; ++s)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[s])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  // flat unit stream of this warp's items: item j -> (b, kvh); units of ctx[b]
  int j = blockIdx.x * (blockDim.x / 32) + warp;
  const int T = gridDim.x * (blockDim.x / 32);
  int b = 0, kvh = 0, u = 0, ue = 0;
  auto load_item = [&]() {  // items[2j] = b * KVH + kvh, items[2j + 1] = first unit << 16 | end unit
    if (j < n_items) {
      b = items[2 * j] / kKVH;
      kvh = items[2 * j] % kKVH;
      u = items[2 * j + 1] >> 16;
      ue = items[2 * j + 1] & 0xffff;
    }
  };
  load_item();
  auto next = [&]() {
    if (++u >= ue) {
      j = (lane == 0) ? T + atomicAdd(counter, 1) : 0;
      j = __shfl_sync(0xffffffffu, j, 0);
      load_item();
    }
  };
  auto issue = [&](int k) {
    const int page = bt[b * bt_stride + (u >> 1)];
    if (lane == 0) {
      const int rk = page * rows_per_page + layer * kKVH * 2 * kPT + kvh * 2 * kPT + (u & 1) * 32;
      const uint32_t mb = smem_u32(&bar[k]);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(8192) : "memory");
      const uint32_t d0 = smem_u32(ring + k * 8192);
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::
              "r"(d0), "l"(reinterpret_cast<uint64_t>(&map)), "r"(mb), "r"(0), "r"(rk)
          : "memory");
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::
              "r"(d0 + 4096), "l"(reinterpret_cast<uint64_t>(&map)), "r"(mb), "r"(0), "r"(rk + kPT)
          : "memory");
    }
  };
  int issued = 0, consumed = 0;
  for (; issued < stages && j < n_items; ++issued) {
    issue(issued);
    next();
  }
  unsigned long long acc = 0;
  while (consumed < issued) {
    const int k = consumed % stages;
    const uint32_t ph = (consumed / stages) & 1;
    asm volatile(
        "{\n\t.reg .pred p;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n\t}" ::
            "r"(smem_u32(&bar[k])),
        "r"(ph)
        : "memory");
    acc += reinterpret_cast<const uint32_t*>(ring + k * 8192)[lane];
    ++consumed;
    __syncwarp();
    if (j < n_items) {
      if (lane == 0) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(k);
      next();
      ++issued;
    }
  }
  if (acc == 42) sink[0] = acc;
}

// Mode 2: one CTA streams whole (sample, page) slices of one layer — all KV
// heads' K|V for 64 tokens, contiguous in the pool (KVH x 16 KB) — with 1-D
// bulk copies through a ring of `stages` slices of `piece` bytes each.
__global__ void slice_kernel(const uint8_t* __restrict__ pool, size_t page_bytes, size_t layer_off, int slice_bytes,
                             const int* __restrict__ order, int B, const int* __restrict__ bt, int bt_stride,
                             const int* __restrict__ ctx, int stages, int piece, int* counter,
                             unsigned long long* sink) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ __align__(8) uint64_t bar[8];
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[s])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int pieces = slice_bytes / piece;
  // work = (sample order index, page, piece); CTAs take samples dynamically
  __shared__ int s_item;
  int item = blockIdx.x, pg = 0, pc = 0, np = 0;
  auto setup = [&]() { np = item < B ? (ctx[order[item]] + kPT - 1) / kPT : 0; pg = 0; pc = 0; };
  setup();
  int issued = 0, consumed = 0;
  unsigned long long acc = 0;
  auto issue = [&](int k) {
    const int b = order[item];
    const uint8_t* src = pool + static_cast<size_t>(bt[b * bt_stride + pg]) * page_bytes + layer_off + static_cast<size_t>(pc) * piece;
    const uint32_t mb = smem_u32(&bar[k]);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(piece) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(smem + static_cast<size_t>(k) * piece)),
                 "l"(src), "r"(piece), "r"(mb)
                 : "memory");
  };
  auto advance = [&]() {
    if (++pc >= pieces) {
      pc = 0;
      if (++pg >= np) {
        if (threadIdx.x == 0) s_item = gridDim.x + atomicAdd(counter, 1);
        __syncthreads();
        item = s_item;
        __syncthreads();
        setup();
      }
    }
  };
  for (; issued < stages && item < B; ++issued) {
    if (threadIdx.x == 0) issue(issued);
    advance();
  }
  while (consumed < issued) {
    const int k = consumed % stages;
    const uint32_t ph = (consumed / stages) & 1;
    asm volatile(
        "{\n\t.reg .pred p;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n\t}" ::
            "r"(smem_u32(&bar[k])), "r"(ph) : "memory");
    acc += reinterpret_cast<const uint32_t*>(smem + static_cast<size_t>(k) * piece)[threadIdx.x];
    ++consumed;
    __syncthreads();
    if (item < B) {
      if (threadIdx.x == 0) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        issue(k);
      }
      advance();
      ++issued;
    }
  }
  if (acc == 42) sink[0] = acc;
}

__global__ void reader(const float* __restrict__ p, size_t n, unsigned long long* sink) {
  float a = 0.f;
  for (size_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) a += p[i];
  if (a == 42.f) sink[0] = 1;
}

int main(int argc, char** argv) {
  const int B = argc > 1 ? std::atoi(argv[1]) : 150;
  const int mean = argc > 2 ? std::atoi(argv[2]) : 200;
  const int warps = argc > 3 ? std::atoi(argv[3]) : 12;
  const int stages = argc > 4 ? std::atoi(argv[4]) : 2;
  std::mt19937 rng(5);
  std::vector<int> ctx(B);
  long long toks = 0;
  for (int i = 0; i < B; ++i) {
    ctx[i] = std::max(1, static_cast<int>(std::uniform_real_distribution<float>(0.f, 2.f * mean)(rng)));
    toks += ctx[i];
  }
  const int maxp = (*std::max_element(ctx.begin(), ctx.end()) + kPT - 1) / kPT;
  const long long npages = static_cast<long long>(B) * maxp + 1;
  const size_t page_bytes = static_cast<size_t>(kL) * kKVH * 2 * kPT * kHD * 2;
  void* pool;
  CK(cudaMalloc(&pool, npages * page_bytes));
  CK(cudaMemset(pool, 0, npages * page_bytes));
  std::vector<int> perm(npages - 1);
  for (int i = 0; i < npages - 1; ++i) perm[i] = i + 1;
  std::shuffle(perm.begin(), perm.end(), rng);
  std::vector<int> bt(B * maxp);
  for (int i = 0; i < B * maxp; ++i) bt[i] = perm[i];
  const int cut_units = argc > 7 ? std::atoi(argv[7]) : 1 << 14;  // items of at most this many 32-token units
  std::vector<int> order(B);
  for (int i = 0; i < B; ++i) order[i] = i;
  std::stable_sort(order.begin(), order.end(), [&](int x, int y) { return ctx[x] > ctx[y]; });
  std::vector<std::array<int, 3>> pieces;  // (units, b*KVH+h, u0 << 16 | u1), longest first
  for (int i = 0; i < B; ++i) {
    const int nu = (ctx[order[i]] + 31) / 32;
    for (int u0 = 0; u0 < nu; u0 += cut_units)
      for (int h = 0; h < kKVH; ++h)
        pieces.push_back({std::min(cut_units, nu - u0), order[i] * kKVH + h, u0 << 16 | std::min(nu, u0 + cut_units)});
  }
  std::stable_sort(pieces.begin(), pieces.end(), [](const auto& x, const auto& y) { return x[0] > y[0]; });
  std::vector<int> items;
  for (const auto& pc : pieces) items.push_back(pc[1]), items.push_back(pc[2]);
  int *d_items, *d_bt, *d_ctx, *d_cnt;
  unsigned long long* d_sink;
  CK(cudaMalloc(&d_items, items.size() * 4));
  CK(cudaMalloc(&d_bt, bt.size() * 4));
  CK(cudaMalloc(&d_ctx, B * 4));
  CK(cudaMalloc(&d_cnt, 4));
  CK(cudaMalloc(&d_sink, 8));
  CK(cudaMemcpy(d_items, items.data(), items.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d_bt, bt.data(), bt.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d_ctx, ctx.data(), B * 4, cudaMemcpyHostToDevice));
  PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&enc), cudaEnableDefault, &q));
  CUtensorMap map;
  const long long rows = npages * static_cast<long long>(page_bytes / (kHD * 2));
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(kHD), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {kHD * 2};
  cuuint32_t box[2] = {64, 32}, es[2] = {1, 1};
  enc(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, pool, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  const int smem = warps * stages * 8192 + 1024;
  if (smem <= 227 * 1024) CK(cudaFuncSetAttribute(probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  void* flush;
  CK(cudaMalloc(&flush, 512 << 20));
  float* clean;  // read after the flush so no dirty line is written back during the timed launch
  CK(cudaMalloc(&clean, 256 << 20));
  CK(cudaMemset(clean, 0, 256 << 20));
  const int clean_mode = argc > 5 ? std::atoi(argv[5]) : 1;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int n_items = static_cast<int>(pieces.size());
  const int grid = std::min(148, (n_items + warps - 1) / warps);
  const int slice_mode = argc > 6 ? std::atoi(argv[6]) : 0;  // > 0: slice kernel, piece = slice / slice_mode
  const int slice_bytes = kKVH * 2 * kPT * kHD * 2;
  const int piece = slice_mode > 0 ? slice_bytes / slice_mode : 0;
  int* d_order;
  CK(cudaMalloc(&d_order, B * 4));
  CK(cudaMemcpy(d_order, order.data(), B * 4, cudaMemcpyHostToDevice));
  if (slice_mode > 0) CK(cudaFuncSetAttribute(slice_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, stages * piece + 1024));
  std::vector<float> ts;
  for (int it = 0; it < 23; ++it) {
    CK(cudaMemset(flush, it, 512 << 20));
    if (clean_mode) reader<<<592, 256>>>(clean, (256 << 20) / 4, d_sink);
    CK(cudaMemset(d_cnt, 0, 4));
    cudaEventRecord(e0);
    if (slice_mode > 0)
      slice_kernel<<<std::min(148, B), 256, stages * piece + 1024>>>(
          static_cast<const uint8_t*>(pool), page_bytes, static_cast<size_t>(5) * slice_bytes, slice_bytes, d_order, B,
          d_bt, maxp, d_ctx, stages, piece, d_cnt, d_sink);
    else
      probe_kernel<<<grid, warps * 32, smem>>>(map, d_items, n_items, d_bt, maxp, d_ctx,
                                               static_cast<int>(page_bytes / (kHD * 2)), 5, stages, d_cnt, d_sink);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (it >= 3) ts.push_back(ms);
  }
  std::sort(ts.begin(), ts.end());
  const double ms = ts[ts.size() / 2];
  const double bytes = static_cast<double>(toks) * kKVH * 2 * kHD * 2;
  std::printf("B %d mean_ctx %d warps %d stages %d slice %d: %.1f us, %.0f GB/s (%.1f MB)\n", B, mean, warps, stages, slice_mode, ms * 1e3,
              bytes / (ms * 1e-3) / 1e9, bytes / 1e6);
  return 0;
}
