// fuseplan-b200 — host launchers and instantiations of the tcgen05 GEMM.
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <stdexcept>
#include <string>
#include <unordered_map>

#include "gemm.cuh"
#include "launch.cuh"
#include "ops.h"
#include "gemm_pair.cuh"
#include "gemm_persist.cuh"
#include "vocab.cuh"

namespace fpk {

namespace {

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || p == nullptr)
      throw std::runtime_error("cuTensorMapEncodeTiled unavailable");
    fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

// Tensor-map cache keyed by every encode parameter (maps are pure functions
// of pointer + geometry, so a hit is always valid).
struct MapKey {
  const void* ptr;
  int dtype, rank, swz;
  uint64_t dims[3], strides[2];
  uint32_t box[3];
  bool operator==(const MapKey& o) const {
    return ptr == o.ptr && dtype == o.dtype && rank == o.rank && swz == o.swz &&
           std::equal(dims, dims + 3, o.dims) && std::equal(strides, strides + 2, o.strides) &&
           std::equal(box, box + 3, o.box);
  }
};
struct MapKeyHash {
  size_t operator()(const MapKey& k) const {
    size_t h = reinterpret_cast<size_t>(k.ptr) ^ (static_cast<size_t>(k.dtype) << 56) ^ k.swz;
    for (int i = 0; i < 3; ++i) h = h * 0x9E3779B97F4A7C15ull ^ k.dims[i] ^ (static_cast<size_t>(k.box[i]) << 40);
    for (int i = 0; i < 2; ++i) h = h * 0x9E3779B97F4A7C15ull ^ k.strides[i];
    return h;
  }
};

CUtensorMap encode(const void* ptr, CUtensorMapDataType dtype, int rank, const uint64_t* dims,
                   const uint64_t* strides_bytes, const uint32_t* box, CUtensorMapSwizzle swz) {
  static std::mutex mu;
  static std::unordered_map<MapKey, CUtensorMap, MapKeyHash> cache;
  MapKey key{ptr, static_cast<int>(dtype), rank, static_cast<int>(swz), {0, 0, 0}, {0, 0}, {0, 0, 0}};
  for (int i = 0; i < rank; ++i) key.dims[i] = dims[i], key.box[i] = box[i];
  for (int i = 0; i + 1 < rank; ++i) key.strides[i] = strides_bytes[i];
  std::lock_guard<std::mutex> lock(mu);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  if (cache.size() > 8192) cache.clear();
  CUtensorMap m;
  cuuint64_t d[3], st[2];
  cuuint32_t bx[3], es[3] = {1u, 1u, 1u};
  for (int i = 0; i < rank; ++i) d[i] = dims[i], bx[i] = box[i];
  for (int i = 0; i + 1 < rank; ++i) st[i] = strides_bytes[i];
  const CUresult r = encode_fn()(&m, dtype, rank, const_cast<void*>(ptr), d, st, bx, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                 swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw std::runtime_error("cuTensorMapEncodeTiled failed: " + std::to_string(int(r)));
  cache.emplace(key, m);
  return m;
}

// bf16 [rows, k] row-major (K innermost), box {64, box_rows}, 128 B swizzle: GEMM operands.
CUtensorMap make_map(const void* ptr, int rows, int k, int box_rows) {
  const uint64_t dims[2] = {static_cast<uint64_t>(k), static_cast<uint64_t>(rows)};
  const uint64_t str[1] = {static_cast<uint64_t>(k) * 2};
  const uint32_t box[2] = {64u, static_cast<uint32_t>(box_rows)};
  return encode(ptr, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, dims, str, box, CU_TENSOR_MAP_SWIZZLE_128B);
}

// Output tile maps (no swizzle): [rows][ld] with `cols` valid columns, box {box_cols, box_rows}.
CUtensorMap out_map_2d(const void* ptr, CUtensorMapDataType dt, int esize, int rows, int cols, int ld, int box_cols,
                       int box_rows) {
  const uint64_t dims[2] = {static_cast<uint64_t>(cols), static_cast<uint64_t>(rows)};
  const uint64_t str[1] = {static_cast<uint64_t>(ld) * esize};
  const uint32_t box[2] = {static_cast<uint32_t>(box_cols), static_cast<uint32_t>(box_rows)};
  return encode(ptr, dt, 2, dims, str, box, CU_TENSOR_MAP_SWIZZLE_NONE);
}

unsigned long long* g_trace = nullptr;

template <int BN, class Epi, int ST = 0>
void launch(const void* A, int a_rows, const void* B, int b_rows, int K, int splits, const Epi& epi,
            cudaStream_t st, bool weight_is_a = true) {
  using C = GemmCfg<BN, ST ? ST : EpiStages<Epi>::value>;
  if (K % kBK != 0) throw std::invalid_argument("gemm: K must be a multiple of 64");
  if (a_rows <= 0 || b_rows <= 0) return;
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(tc_gemm_kernel<BN, Epi, ST>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         C::kSmem + EpiSmemExtra<Epi>::value);
    attr_set = true;
  }
  const CUtensorMap ma = make_map(A, a_rows, K, 128);
  const CUtensorMap mb = make_map(B, b_rows, K, BN);
  GemmGeom g;
  g.a_rows = a_rows;
  g.b_rows = b_rows;
  g.k_blocks = K / kBK;
  splits = std::max(1, std::min(splits, g.k_blocks));
  g.kb_per_split = (g.k_blocks + splits - 1) / splits;
  g.weight_is_a = weight_is_a ? 1 : 0;
  g.trace = g_trace;
  if (!g.trace) {
    const long long ctas = static_cast<long long>((a_rows + 127) / 128) * ((b_rows + BN - 1) / BN) *
                           ((g.k_blocks + g.kb_per_split - 1) / g.kb_per_split);
    g.trace = trace_slot(0, static_cast<int>(ctas), 8);
  }
  const int z = (g.k_blocks + g.kb_per_split - 1) / g.kb_per_split;
  // Programmatic dependent launch: the prologue and the weight prefetch of this
  // GEMM overlap the tail of the previous kernel (which triggers early).
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((a_rows + 127) / 128, (b_rows + BN - 1) / BN, z);
  cfg.blockDim = dim3(kGemmThreads);
  cfg.dynamicSmemBytes = C::kSmem + EpiSmemExtra<Epi>::value;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, tc_gemm_kernel<BN, Epi, ST>, ma, mb, g, epi);
  if (e != cudaSuccess) throw std::runtime_error(std::string("gemm launch: ") + cudaGetErrorString(e));
  fpk::count_launch();
}

int sm_count() {
  static int n = [] {
    int dev = 0, v = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v > 0 ? v : 148;
  }();
  return n;
}

// Packed forwards (prefill / scoring) from this many rows on take the
// persistent kernel (gemm_persist.cuh); decode batches (<= 512 rows) never do.
constexpr int kPersistMinRows = 1024;
thread_local bool g_persist = true;

template <int BN, class Epi>
void launch_persist(const void* A, int a_rows, const void* B, int b_rows, int K, const Epi& epi, cudaStream_t st,
                    bool weight_is_a = true) {
  using C = PersistCfg<BN, Epi>;
  if (K % kBK != 0) throw std::invalid_argument("gemm: K must be a multiple of 64");
  if (a_rows <= 0 || b_rows <= 0) return;
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(tc_gemm_persist_kernel<BN, Epi>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem);
    attr_set = true;
  }
  const CUtensorMap ma = make_map(A, a_rows, K, 128);
  const CUtensorMap mb = make_map(B, b_rows, K, BN);
  PersistGeom g;
  g.a_rows = a_rows;
  g.b_rows = b_rows;
  g.k_blocks = K / kBK;
  g.a_tiles = (a_rows + 127) / 128;
  g.n_tiles = g.a_tiles * ((b_rows + BN - 1) / BN);
  g.weight_is_a = weight_is_a ? 1 : 0;
  g.trace = g_trace;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(std::min(g.n_tiles, sm_count()));
  cfg.blockDim = dim3(kGemmThreads);
  cfg.dynamicSmemBytes = C::kSmem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, tc_gemm_persist_kernel<BN, Epi>, ma, mb, g, epi);
  if (e != cudaSuccess) throw std::runtime_error(std::string("gemm launch: ") + cudaGetErrorString(e));
  fpk::count_launch();
}

// The SM-pair kernel (gemm_pair.cuh): 256 x 256 tiles, cluster of two CTAs.
template <int BN = 256, class Epi>
void launch_pair(const void* A, int a_rows, const void* B, int b_rows, int K, const Epi& epi, cudaStream_t st) {
  using C = PairCfg<Epi, BN>;
  if (K % kBK != 0) throw std::invalid_argument("gemm: K must be a multiple of 64");
  if (a_rows <= 0 || b_rows <= 0) return;
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(tc_gemm_pair_kernel<Epi, BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem);
    attr_set = true;
  }
  const CUtensorMap ma = make_map(A, a_rows, K, 128);
  const CUtensorMap mb = make_map(B, b_rows, K, BN / 2);
  PersistGeom g;
  g.a_rows = a_rows;
  g.b_rows = b_rows;
  g.k_blocks = K / kBK;
  g.a_tiles = (a_rows + 255) / 256;
  g.n_tiles = g.a_tiles * ((b_rows + BN - 1) / BN);
  g.weight_is_a = 1;
  g.trace = g_trace;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(2 * std::min(g.n_tiles, sm_count() / 2));
  cfg.blockDim = dim3(kGemmThreads);
  cfg.dynamicSmemBytes = C::kSmem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, tc_gemm_pair_kernel<Epi, BN>, ma, mb, g, epi);
  if (e != cudaSuccess) throw std::runtime_error(std::string("gemm pair launch: ") + cudaGetErrorString(e));
  fpk::count_launch();
}

// SM pairs for the packed GEMMs when their 256 x 256 tiles still spread
// evenly (>= 3 per pair; fewer, e.g. gpt2s' N = 768 projections, lose more to
// the last round than the pairs gain); set_pair_gemm forces either kernel.
thread_local int g_pair = -1;  // -1 auto, 0 one-SM, 1 pairs
bool use_pair(int N, int M) {
  if (g_pair >= 0) return g_pair == 1;
  const long long tiles = static_cast<long long>((N + 255) / 256) * ((M + 255) / 256);
  return tiles >= 3 * (sm_count() / 2);
}

// Batch-tile width of a swap-AB GEMM with `a_ctas` weight tiles (x splits):
// the fewest waves over the 148 SMs, then the narrowest tile (most CTAs
// streaming weights in that wave), never wider than the rows need. A CTA's
// time is dominated by streaming its 128-row weight tile, which does not
// depend on BN, so a second wave costs about as much as the first; a row's
// bits do not depend on BN (each output element is one tensor-core dot
// product in the same K order).
int pick_bn(int M, int a_ctas) {
  static const int kBN[] = {16, 32, 64, 128, 256};
  int best = 16, best_waves = 1 << 30;
  for (int bn : kBN) {
    if (bn != 16 && bn / 2 >= M) break;  // wider than the rows need
    const int waves = (a_ctas * ((M + bn - 1) / bn) + 147) / 148;
    if (waves < best_waves) {
      best = bn;
      best_waves = waves;
    }
  }
  return best;
}

// Decode GEMMs (M <= 128) in a lean ring (120-128 KB of shared memory) so that
// the next kernels' CTAs fit on an SM beside the current one's: with PDL they
// become resident early and stream their weights while the previous kernels
// run. One stage deeper than the first cut (<= 110 KB) measured faster
// (gpt2s bench 572.5 vs 563.1 samples/s, DESIGN 8.4).
template <int BN>
struct Lean {
  static constexpr int v = BN <= 16 ? 7 : BN <= 32 ? 6 : BN <= 64 ? 5 : BN <= 128 ? 4 : 3;
};
bool lean(int M) { return M <= 128; }  // (large batches keep the deep ring: their mainloops are bandwidth-hungry)

// Large GEMMs (several waves of CTAs) take the 2-stage / 2-CTAs-per-SM shape.
bool many_waves(int M, int N, int BN) { return static_cast<long long>((N + 127) / 128) * ((M + BN - 1) / BN) >= 2 * 148; }

template <class Epi, class F>
void dispatch_bn(int M, int a_ctas, F&& f) {
  switch (pick_bn(M, a_ctas)) {
    case 16: f.template operator()<16>(); break;
    case 32: f.template operator()<32>(); break;
    case 64: f.template operator()<64>(); break;
    case 128: f.template operator()<128>(); break;
    default: f.template operator()<256>(); break;
  }
}

}  // namespace

void set_packed_persistent(bool on) { g_persist = on; }
void set_pair_gemm(int mode) { g_pair = mode < 0 ? -1 : (mode ? 1 : 0); }
bool packed_persistent() { return g_persist; }

CUtensorMap make_kv_map(const void* pool, long long rows, int hd) {
  CUtensorMap m;
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(hd), static_cast<cuuint64_t>(rows)};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(hd) * 2};
  const cuuint32_t box[2] = {64u, 32u};  // 32-token units
  const cuuint32_t estr[2] = {1u, 1u};
  const CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(pool), dims, strides, box,
                                 estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw std::runtime_error("cuTensorMapEncodeTiled (kv) failed: " + std::to_string(int(r)));
  return m;
}

void set_gemm_trace(unsigned long long* buf) { g_trace = buf; }

// Map / tile-width helpers of the persistent decode chain (chain.cu).
CUtensorMap chain_operand_map(const void* ptr, int rows, int k, int box_rows) { return make_map(ptr, rows, k, box_rows); }
CUtensorMap chain_out_map_bf16(const void* ptr, int rows, int cols, int ld, int box_cols, int box_rows) {
  return out_map_2d(ptr, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, rows, cols, ld, box_cols, box_rows);
}
int chain_pick_bn(int M, int a_tiles) { return pick_bn(M, a_tiles); }

namespace {
unsigned long long* g_arena = nullptr;
size_t g_arena_words = 0, g_arena_used = 0;
std::vector<TraceRec> g_recs;
}  // namespace

void trace_arm(unsigned long long* arena, size_t words) {
  g_arena = arena;
  g_arena_words = words;
  g_arena_used = 0;
  g_recs.clear();
}

unsigned long long* trace_slot(int kind, int units, int words_per_unit) {
  if (!g_arena) return nullptr;
  const size_t w = static_cast<size_t>(units) * words_per_unit;
  if (g_arena_used + w > g_arena_words) return nullptr;
  g_recs.push_back({kind, units, g_arena_used});
  unsigned long long* p = g_arena + g_arena_used;
  g_arena_used += w;
  return p;
}

std::vector<TraceRec> trace_disarm() {
  g_arena = nullptr;
  return std::move(g_recs);
}

int gemm_splits(int N, int K) {
  const int kb = K / kBK;
  const int tiles = (N + 127) / 128;
  int s = (2 * 148 + tiles - 1) / tiles;
  // at most 4: the partials (splits x M x N x 4 B) are read back by add_norm,
  // and fewer, longer K slices measured faster than 6-8 (gpt2s bench 567.9 vs
  // 563.1 samples/s at cap 4 vs 8, DESIGN 8.4)
  s = std::min(s, 4);
  s = std::min(s, kb);
  // Equalise the K range per split so that no split is empty.
  const int per = (kb + s - 1) / s;
  return (kb + per - 1) / per;
}

void gemm_bf16(const bf16* W, int N, int K, const bf16* X, int M, bf16* out, int ld_out, cudaStream_t st) {
  if ((ld_out * 2) % 16) throw std::invalid_argument("gemm_bf16: ld_out must be a multiple of 8");
  if (M >= kPersistMinRows && g_persist) {
    EpiStoreBF16 e{out_map_2d(out, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, M, N, ld_out, 128, 256)};
    if (use_pair(N, M))
      launch_pair(W, N, X, M, K, e, st);
    else
      launch_persist<256>(W, N, X, M, K, e, st);
    return;
  }
  dispatch_bn<EpiStoreBF16>(M, (N + 127) / 128, [&]<int BN>() {
    EpiStoreBF16 e{out_map_2d(out, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, M, N, ld_out, 128, BN)};
    if (many_waves(M, N, BN))
      launch<BN, EpiStoreBF16, 2>(W, N, X, M, K, 1, e, st);
    else
      launch<BN>(W, N, X, M, K, 1, e, st);
  });
}

void gemm_f32_splitk(const bf16* W, int N, int K, const bf16* X, int M, float* out, int splits, cudaStream_t st) {
  if (N % 4) throw std::invalid_argument("gemm_f32: N must be a multiple of 4");
  const int kb = K / kBK;
  splits = std::max(1, std::min(splits, kb));
  const int per = (kb + splits - 1) / splits;
  const int z = (kb + per - 1) / per;
  dispatch_bn<EpiStoreF32>(M, (N + 127) / 128 * z, [&]<int BN>() {
    const uint64_t dims[3] = {static_cast<uint64_t>(N), static_cast<uint64_t>(M), static_cast<uint64_t>(z)};
    const uint64_t str[2] = {static_cast<uint64_t>(N) * 4, static_cast<uint64_t>(M) * N * 4};
    const uint32_t box[3] = {128u, static_cast<uint32_t>(BN), 1u};
    EpiStoreF32 e{encode(out, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, dims, str, box, CU_TENSOR_MAP_SWIZZLE_NONE), 0};
    if (BN <= 128 && lean(M))  // (the fp32 staging tile of BN 256 needs the deep ring)
      launch<BN, EpiStoreF32, Lean<BN>::v>(W, N, X, M, K, splits, e, st);
    else
      launch<BN>(W, N, X, M, K, splits, e, st);
  });
}

void gemm_f32_residual(const bf16* W, int N, int K, const bf16* X, int M, float* resid, cudaStream_t st) {
  if (N % 4) throw std::invalid_argument("gemm_f32: N must be a multiple of 4");
  if (M >= kPersistMinRows && g_persist) {
    // 256-token tiles (more bytes per flop, 4-stage ring) when there are
    // enough of them to keep the 148 SMs evenly loaded, else 128 (6 stages)
    if (use_pair(N, M)) {
      launch_pair<256>(W, N, X, M, K, EpiResidDirect{resid, N, M}, st);
      return;
    }
    if (g_pair < 0 && K >= 2048) {  // few 256 x 256 tiles (N = 768) but a long mainloop: 256 x 128 pair tiles
      launch_pair<128>(W, N, X, M, K, EpiResidDirect{resid, N, M}, st);
      return;
    }
    const long long tiles256 = static_cast<long long>((N + 127) / 128) * ((M + 255) / 256);
    if (tiles256 >= 4 * sm_count())
      launch_persist<256>(W, N, X, M, K, EpiResidDirect{resid, N, M}, st);
    else
      launch_persist<128>(W, N, X, M, K, EpiResidDirect{resid, N, M}, st);
    return;
  }
  dispatch_bn<EpiStoreF32>(M, (N + 127) / 128, [&]<int BN>() {
    EpiStoreF32 e{out_map_2d(resid, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, M, N, N, 128, BN), 1};
    if (BN <= 128 && many_waves(M, N, BN))  // (the fp32 staging tile of BN 256 needs a deeper ring)
      launch<BN, EpiStoreF32, 2>(W, N, X, M, K, 1, e, st);
    else
      launch<BN>(W, N, X, M, K, 1, e, st);
  });
}

void gemm_swiglu_decode(const bf16* Wgu, int F, int K, const bf16* X, int M, bf16* out, cudaStream_t st) {
  if (F % 64) throw std::invalid_argument("gemm_swiglu: F must be a multiple of 64");
  // Large decode batches of a large FFN (Llama-3-8B: 2F x K = 117 M weights)
  // are compute-heavy enough for SM pairs: 256 x 256 tiles, 17-19 % faster
  // than the tiled kernel at 256-512 rows. Same bits as the tiled kernel, so a
  // row's result does not depend on which batch size picked which kernel.
  if (g_pair != 0 && M >= 256 && static_cast<long long>(2 * F) * K >= (64ll << 20)) {
    launch_pair(Wgu, 2 * F, X, M, K, EpiSwiGLUDirect<256>{out, F, M}, st);
    return;
  }
  dispatch_bn<int>(M, (2 * F + 127) / 128, [&]<int BN>() {
    EpiSwiGLU<BN> e{out_map_2d(out, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, M, F, F, 64, BN)};
    if (lean(M))
      launch<BN, EpiSwiGLU<BN>, Lean<BN>::v>(Wgu, 2 * F, X, M, K, 1, e, st);
    else
      launch<BN>(Wgu, 2 * F, X, M, K, 1, e, st);
  });
}

void gemm_swiglu(const bf16* Wgu, int F, int K, const bf16* X, int M, bf16* out, cudaStream_t st) {
  if (F % 64) throw std::invalid_argument("gemm_swiglu: F must be a multiple of 64");
  if (M >= kPersistMinRows && g_persist) {
    if (use_pair(2 * F, M)) {
      if (K >= 2048) {
        launch_pair(Wgu, 2 * F, X, M, K, EpiSwiGLUDirect<256>{out, F, M}, st);
      } else {
        EpiSwiGLU<256> e{out_map_2d(out, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, M, F, F, 64, 256)};
        launch_pair(Wgu, 2 * F, X, M, K, e, st);
      }
      return;
    }
    if (K >= 2048) {  // long mainloops: the deeper ring pays; short ones are epilogue-bound (TMA store)
      launch_persist<256>(Wgu, 2 * F, X, M, K, EpiSwiGLUDirect<256>{out, F, M}, st);
    } else {
      EpiSwiGLU<256> e{out_map_2d(out, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, M, F, F, 64, 256)};
      launch_persist<256>(Wgu, 2 * F, X, M, K, e, st);
    }
    return;
  }
  dispatch_bn<int>(M, (2 * F + 127) / 128, [&]<int BN>() {
    EpiSwiGLU<BN> e{out_map_2d(out, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, M, F, F, 64, BN)};
    if (many_waves(M, 2 * F, BN))
      launch<BN, EpiSwiGLU<BN>, 2>(Wgu, 2 * F, X, M, K, 1, e, st);
    else
      launch<BN>(Wgu, 2 * F, X, M, K, 1, e, st);
  });
}

void gemm_qkv_rope(const bf16* Wqkv, int K, const bf16* X, int M, int H, int KVH, int hd, const int* pos,
                   const float2* cs, const KvPoolView& pool, int layer, const int* slot, bf16* q_out,
                   cudaStream_t st) {
  if (128 % hd != 0) throw std::invalid_argument("gemm_qkv_rope: head_dim must divide 128");
  const int N = (H + 2 * KVH) * hd;
  dispatch_bn<int>(M, (N + 127) / 128, [&]<int BN>() {
    EpiRopeKV<BN> e{q_out, pool, slot, pos, cs, layer, H, KVH, hd, M};
    e.pool.kv_map = nullptr;  // host pointer: not dereferenced on the device
    if (lean(M))
      launch<BN, EpiRopeKV<BN>, Lean<BN>::v>(Wqkv, N, X, M, K, 1, e, st);
    else
      launch<BN>(Wqkv, N, X, M, K, 1, e, st);
  });
}

void gemm_qkv_rope_packed(const bf16* Wqkv, int K, const bf16* X, int M, int H, int KVH, int hd, const int* pos,
                          const float2* cs, const KvPoolView* pool, int layer, const int* slot, bf16* q_out,
                          bf16* k_out, bf16* v_out, cudaStream_t st) {
  if (128 % hd != 0) throw std::invalid_argument("gemm_qkv_rope: head_dim must divide 128");
  const int N = (H + 2 * KVH) * hd;
  if (M >= kPersistMinRows && g_persist) {
    EpiRopeKV<256> e{q_out, pool ? *pool : KvPoolView{}, slot, pos, cs, layer, H, KVH, hd, M};
    e.pool.kv_map = nullptr;
    e.k_out = k_out;
    e.v_out = v_out;
    e.use_pool = pool != nullptr;
    if (use_pair(N, M))
      launch_pair(Wqkv, N, X, M, K, e, st);
    else
      launch_persist<256>(Wqkv, N, X, M, K, e, st);
    return;
  }
  dispatch_bn<int>(M, (N + 127) / 128, [&]<int BN>() {
    EpiRopeKV<BN> e{q_out, pool ? *pool : KvPoolView{}, slot, pos, cs, layer, H, KVH, hd, M};
    e.pool.kv_map = nullptr;
    e.k_out = k_out;
    e.v_out = v_out;
    e.use_pool = pool != nullptr;
    if (many_waves(M, N, BN))
      launch<BN, EpiRopeKV<BN>, 2>(Wqkv, N, X, M, K, 1, e, st);
    else
      launch<BN>(Wqkv, N, X, M, K, 1, e, st);
  });
}

constexpr int kVocabBN = 256;

int vocab_tiles(int V) { return 2 * ((V + kVocabBN - 1) / kVocabBN); }  // partials per row: 2 column halves per tile

void gemm_vocab(const bf16* X, int M, int K, const bf16* Whead, int V, int mode, float inv_temp, const int* target,
                const int* sample_id, const int* step, uint64_t seed, void* part, float* tgt_z, cudaStream_t st) {
  auto go = [&](auto e) {
    e.part = static_cast<VocabPartial*>(part);
    e.tgt_z = tgt_z;
    e.info = VocabRowInfo{target, sample_id, step};
    e.inv_temp = inv_temp;
    e.vocab = V;
    e.rows = M;
    e.n_tiles = vocab_tiles(V);
    e.seed_lo = static_cast<uint32_t>(seed);
    e.seed_hi = static_cast<uint32_t>(seed >> 32);
    // persistent at every M: 197 vocab tiles (V 50257) on 148 SMs load-balance
    // and stream through a 4-deep ring; the weight streams before
    // griddepcontrol.wait
    if (g_persist)
      launch_persist<kVocabBN>(X, M, Whead, V, K, e, st, /*weight_is_a=*/false);
    else
      launch<kVocabBN>(X, M, Whead, V, K, 1, e, st, /*weight_is_a=*/false);
  };
  if (mode == kForced) go(EpiVocab<kForced>{});
  else if (mode == kGreedy) go(EpiVocab<kGreedy>{});
  else go(EpiVocab<kSample>{});
}

void gemm_vocab_logits(const bf16* X, int M, int K, const bf16* Whead, int V, float inv_temp, void* part,
                       float* logits, int ldv, cudaStream_t st) {
  if (ldv < V || ldv % 4) throw std::invalid_argument("gemm_vocab_logits: ldv must be >= V and a multiple of 4");
  EpiVocab<kLogits> e{};
  e.part = static_cast<VocabPartial*>(part);
  e.tgt_z = nullptr;
  e.info = VocabRowInfo{nullptr, nullptr, nullptr};
  e.inv_temp = inv_temp;
  e.vocab = V;
  e.rows = M;
  e.n_tiles = vocab_tiles(V);
  e.logits = logits;
  e.ldv = ldv;
  launch<kVocabBN>(X, M, Whead, V, K, 1, e, st, /*weight_is_a=*/false);
}

// One warp per row: merge the row's partials in partial order. The sampling
// walk over partials is sequential in lane 0 so that its float order is
// fixed (the CPU oracle replays it).
__global__ void vocab_finalize_kernel(const VocabPartial* __restrict__ part, const float* __restrict__ tgt_z, int M,
                                      int n_tiles, int mode, const int* __restrict__ target,
                                      const int* __restrict__ sample_id, const int* __restrict__ step,
                                      uint32_t seed_lo, uint32_t seed_hi, int* token, float* logp, const int* dst,
                                      int* out_tok, float* out_logp, const int* cur_idx, int* cur_tok) {
  pdl_trigger();  // let the next (PDL-launched) GEMM start its prologue / weight prefetch
  pdl_wait();     // PDL-launched: the partials come from the vocab GEMM
  const int row = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= M) return;
  // the row's partials are contiguous (n_tiles is even: a multiple of 48
  // bytes): one bulk copy per row into shared memory, then walk them there
  extern __shared__ float4 fin_smem[];
  __shared__ __align__(8) uint64_t fin_bar[8];
  const uint32_t row_bytes = static_cast<uint32_t>(n_tiles * sizeof(VocabPartial));
  float4* srow = fin_smem + static_cast<size_t>(threadIdx.x >> 5) * (row_bytes / 16);
  uint64_t* bar = &fin_bar[threadIdx.x >> 5];
  if (lane == 0) {
    mbar_init(bar, 1);
    fence_barrier_init();
    mbar_arrive_expect_tx(bar, row_bytes);
    bulk_load(srow, part + static_cast<size_t>(row) * n_tiles, row_bytes, bar);
  }
  __syncwarp();
  mbar_wait(bar, 0);
  const VocabPartial* p = reinterpret_cast<const VocabPartial*>(srow);
  // lane l owns the contiguous half-tiles [t0, t1); the mass is summed in
  // that fixed order (per lane, then lane 0..31 sequentially) so the oracle
  // (model_oracle.sample_token) replays it bit-for-bit
  const int chunk = (n_tiles + 31) / 32;
  const int t0 = min(n_tiles, lane * chunk), t1 = min(n_tiles, t0 + chunk);
  float m = -INFINITY;
  for (int t = t0; t < t1; ++t) m = fmaxf(m, p[t].m2);
  m = warp_max(m);
  float c = 0.f;
  float bz = -INFINITY;
  int bidx = 0x7fffffff;
  for (int t = t0; t < t1; ++t) {
    const VocabPartial q = p[t];
    if (q.m2 > -INFINITY) c += __fmul_rn(q.s, exp2f(q.m2 - m));  // no FMA contraction: oracle order
    if (mode == kGreedy && q.idx >= 0 && (q.zsel > bz || (q.zsel == bz && q.idx < bidx))) {
      bz = q.zsel;
      bidx = q.idx;
    }
  }
  if (mode == kGreedy) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float oz = __shfl_xor_sync(0xffffffffu, bz, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bidx, o);
      if (oz > bz || (oz == bz && oi < bidx)) {
        bz = oz;
        bidx = oi;
      }
    }
  }
  float thr = 0.f;
  if (mode == kSample) {
    const U4 w = philox4x32_10(U4{kRowDraw, static_cast<uint32_t>(step[row]), static_cast<uint32_t>(sample_id[row]),
                                  0xF00Du},
                               seed_lo, seed_hi);
    thr = unit_open(w.x);
  }
  // tot = sum of the lane sums in lane order; the picked lane is the first
  // whose running sum reaches thr * tot (same in every lane)
  float tot = 0.f;
#pragma unroll
  for (int l = 0; l < 32; ++l) tot += __shfl_sync(0xffffffffu, c, l);
  const float lse = m * kLn2 + logf(tot);  // natural-log logsumexp of z
  int tok = 0;
  float lp = 0.f;
  if (mode == kForced) {
    tok = target[row];
    lp = tgt_z[row] - lse;
  } else if (mode == kGreedy) {
    tok = bidx;
    lp = bz - lse;
  } else {
    thr *= tot;
    float acc = 0.f, base = 0.f;
    int pl = -1;
#pragma unroll
    for (int l = 0; l < 32; ++l) {
      const float cl = __shfl_sync(0xffffffffu, c, l);
      if (pl < 0) {
        base = acc;
        acc += cl;
        if (acc >= thr && cl > 0.f) pl = l;
      }
    }
    if (pl < 0) pl = 31;  // unreachable: acc == tot >= thr
    if (lane != pl) return;
    int pick = -1;
    acc = base;
    for (int t = t0; t < t1; ++t) {
      if (p[t].m2 == -INFINITY) continue;
      acc += __fmul_rn(p[t].s, exp2f(p[t].m2 - m));
      pick = t;
      if (acc >= thr) break;
    }
    tok = p[pick].idx;
    lp = p[pick].zsel - lse;
  }
  if (mode != kSample && lane != 0) return;
  if (token) token[row] = tok;
  if (logp) logp[row] = lp;
  if (dst) {
    const int d = dst[row];
    if (d >= 0) {
      if (out_tok) out_tok[d] = tok;
      if (out_logp) out_logp[d] = lp;
    }
  }
  if (cur_tok) cur_tok[cur_idx[row]] = tok;
}

void vocab_finalize(const void* part, const float* tgt_z, int M, int V, int mode, const int* target,
                    const int* sample_id, const int* step, uint64_t seed, int* token, float* logp, const int* dst,
                    int* out_tok, float* out_logp, const int* cur_idx, int* cur_tok, cudaStream_t st) {
  if (M <= 0) return;
  const size_t row_bytes = static_cast<size_t>(vocab_tiles(V)) * sizeof(VocabPartial);
  // small batches (decode): one row per CTA, spread over the SMs
  const int warps = M <= 2 * 148 ? 1 : static_cast<int>(std::max<size_t>(1, std::min<size_t>(8, (96 * 1024) / row_bytes)));
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(vocab_finalize_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr = true;
  }
  launch_pdl(vocab_finalize_kernel, dim3((M + warps - 1) / warps), dim3(warps * 32), warps * row_bytes, st,
             static_cast<const VocabPartial*>(part), tgt_z, M, vocab_tiles(V), mode, target, sample_id, step,
             static_cast<uint32_t>(seed), static_cast<uint32_t>(seed >> 32), token, logp, dst, out_tok, out_logp,
             cur_idx, cur_tok);
  fpk::count_launch();
}

}  // namespace fpk
