// fuseplan-b200 — executor of the gen+inf stage on one GPU (one rank).
//
// Per rank r (instance r of cfg.num_instances):
//   1. Decisions from the decision clock: simulate_serial / simulate_fused
//      (reported), fused_trigger (trigger state, plan, in-flight placement).
//   2. Instance state machine, step by step, with the reference semantics
//      (proj/src/genfuse.cpp:222-271): retire finished samples (free their KV
//      reservation in in-flight order), admit FIFO while the reserved KV fits
//      (cap + 1e-6), prefill the admitted prompts, decode one token for every
//      in-flight sample. Reservation bytes are the reference's kv_bytes, so
//      the admission sequence is the reference's.
//   3. Fused schedule, G > 1: the rank pauses when its state equals its
//      trigger snapshot (pre- or post-admission boundary), then the one-shot
//      migration: destinations pull the in-flight samples' KV pages and
//      histories from the source GPU's memory over NVLink (CUDA IPC pointers,
//      copy kernel), queued samples are re-queued; then execution resumes.
//   4. Sample-level scoring: every finished sample is published to a shared
//      queue; ranks claim batches of finished samples (in finish order) and
//      run Reference/Critic/Reward + post-processing on a low-priority stream.
//      Stage-barrier schedule: claims start only after every rank finished
//      generating. Fused: claims start immediately (a generating rank keeps at
//      most one scoring batch in flight; idle ranks two).
// Coordination between ranks is a POSIX shared-memory region (counters,
// barrier, IPC handles, page lists, gathered results).
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <array>
#include <atomic>
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <map>
#include <memory>
#include <thread>
#include <unordered_map>

#include "engine.hpp"
#include "fuseplan/minibatch.hpp"
#include "fuseplan/engine.hpp"
#include "fuseplan/errors.hpp"
#include "philox.cuh"

namespace fuseplan {

struct TokRing;

struct GpuEngine {
  EngineSetup setup;
  std::unique_ptr<fpe::Engine> eng;
  std::unique_ptr<TokRing> ring;  // free-run token readback (pinned), created on first use
  ~GpuEngine();
};

namespace {

using Clock = std::chrono::steady_clock;
constexpr int kMaxRanks = 8;

fpe::Dims to_dims(const EngineModelDims& m) {
  fpe::Dims d;
  d.L = m.num_layers;
  d.d = m.hidden;
  d.H = m.num_heads;
  d.KVH = m.num_kv_heads;
  d.hd = m.head_dim;
  d.F = m.ffn;
  d.V = m.vocab;
  return d;
}

// ---------------------------------------------------------------------------
// shared coordination region

struct Header {
  std::atomic<int> bar_count;
  std::atomic<int> bar_gen;
  std::atomic<int> n_pub;      // finished samples published
  std::atomic<int> n_claimed;  // claim cursor into pub_order
  std::atomic<int> gen_done;   // ranks with no generation work left
  std::atomic<int> error;      // a rank failed (set by the failing rank; peers throw)
  std::atomic<int> lock;       // publish lock
  std::atomic<int> finished;   // samples retired (online trigger)
  std::atomic<int> trig_flag;  // online trigger raised
  int world, n, max_pages, pad_;
  // online trigger: per-rank state at the pause
  int r_live[kMaxRanks], r_queue[kMaxRanks];
  double r_kv[kMaxRanks], r_time[kMaxRanks];
  cudaIpcMemHandle_t h_hist_tok[kMaxRanks], h_hist_logp[kMaxRanks], h_pool[kMaxRanks];
  cudaIpcMemHandle_t h_exp[kMaxRanks];  // experience arrays (hand-off)
  cudaIpcMemHandle_t h_model[kMaxRanks];  // weight blobs (broadcast_model)
};

// Per-sample state published at an online trigger pause.
struct SampleState {
  int flag;  // bit 0: unfinished (present), bit 1: admitted (in flight)
  int rank, gen, order;  // owner, tokens generated, index in the owner's in-flight list / FIFO
};

class Region {
 public:
  Region(const CommSetup& comm, int n, int max_pages, int64_t total_resp)
      : world_(comm.world), rank_(comm.rank), n_(n), max_pages_(max_pages), total_(total_resp) {
    off_pub_ = align(sizeof(Header));
    off_owner_ = align(off_pub_ + n * 4);
    off_scorer_ = align(off_owner_ + n * 4);
    off_len_ = align(off_scorer_ + n * 4);
    off_state_ = align(off_len_ + n * 4);
    off_pages_ = align(off_state_ + static_cast<size_t>(n) * sizeof(SampleState));
    off_res_ = align(off_pages_ + static_cast<size_t>(n) * max_pages * 4);
    bytes_ = align(off_res_ + static_cast<size_t>(total_resp) * 4 * 8 + n * 4);
    if (world_ == 1) {
      local_.reset(new uint8_t[bytes_]());
      base_ = local_.get();
    } else {
      name_ = comm.shm_name;
      fd_ = shm_open(name_.c_str(), O_CREAT | O_RDWR, 0600);
      if (fd_ < 0) throw std::runtime_error("shm_open failed: " + name_);
      if (ftruncate(fd_, static_cast<off_t>(bytes_)) != 0) throw std::runtime_error("ftruncate failed");
      void* p = mmap(nullptr, bytes_, PROT_READ | PROT_WRITE, MAP_SHARED, fd_, 0);
      if (p == MAP_FAILED) throw std::runtime_error("mmap failed");
      base_ = static_cast<uint8_t*>(p);
    }
    hdr_ = reinterpret_cast<Header*>(base_);
  }
  ~Region() {
    if (world_ > 1 && base_) {
      munmap(base_, bytes_);
      close(fd_);
      if (rank_ == 0) shm_unlink(name_.c_str());
    }
  }
  Header* hdr() { return hdr_; }
  int* pub_order() { return reinterpret_cast<int*>(base_ + off_pub_); }
  int* owner() { return reinterpret_cast<int*>(base_ + off_owner_); }
  int* scorer() { return reinterpret_cast<int*>(base_ + off_scorer_); }  // rank holding the sample's experience
  int* resp_len() { return reinterpret_cast<int*>(base_ + off_len_); }   // response length, set at retirement
  SampleState* state() { return reinterpret_cast<SampleState*>(base_ + off_state_); }
  int* pages(int sid) { return reinterpret_cast<int*>(base_ + off_pages_) + static_cast<size_t>(sid) * max_pages_; }
  float* result(int k) { return reinterpret_cast<float*>(base_ + off_res_) + static_cast<size_t>(k) * total_; }
  float* score() { return reinterpret_cast<float*>(base_ + off_res_) + static_cast<size_t>(8) * total_; }

  // A rank that throws marks the region so that its peers fail fast instead of
  // waiting out their deadlines.
  void fail() {
    if (hdr_) hdr_->error.store(1);
  }
  void check_peers() const {
    if (hdr_->error.load()) throw std::runtime_error("peer rank failed");
  }

  void barrier() {
    if (world_ == 1) return;
    const int gen = hdr_->bar_gen.load();
    if (hdr_->bar_count.fetch_add(1) + 1 == world_) {
      hdr_->bar_count.store(0);
      hdr_->bar_gen.fetch_add(1);
    } else {
      const auto t0 = Clock::now();
      while (hdr_->bar_gen.load() == gen) {
        check_peers();
        std::this_thread::yield();
        if (Clock::now() - t0 > std::chrono::seconds(600)) throw std::runtime_error("barrier timeout");
      }
    }
  }

 private:
  static size_t align(size_t x) { return (x + 255) & ~size_t(255); }
  int world_, rank_, n_, max_pages_;
  int64_t total_;
  size_t off_pub_ = 0, off_owner_ = 0, off_scorer_ = 0, off_len_ = 0, off_state_ = 0, off_pages_ = 0, off_res_ = 0,
         bytes_ = 0;
  std::unique_ptr<uint8_t[]> local_;
  uint8_t* base_ = nullptr;
  Header* hdr_ = nullptr;
  std::string name_;
  int fd_ = -1;
};

struct Live {
  int sid, slot, gen, target;
};

struct Move {
  int sid, src, dst;
  bool inflight;
  int gen;
};

// Migrants in the decision clock's application order (fused_trigger).
std::vector<Move> moves_of(const TriggerSnapshot& snap) {
  std::vector<Move> mv;
  if (!snap.triggered || snap.plan.no_op) return mv;
  std::map<int, const GenState::Remaining*> rem;
  for (const auto& r : snap.state.samples) rem[r.id] = &r;
  for (std::size_t i = 0; i < snap.move_sample.size(); ++i) {
    const GenState::Remaining* r = rem.at(snap.move_sample[i]);
    mv.push_back({r->id, snap.move_from[i], snap.move_to[i], r->admitted, r->generated});
  }
  return mv;
}

// Online trigger: apply_migration's placement rules (reference
// genfuse.cpp:136-208; restated in csrc/host/genfuse.cpp Clock::migrate) on
// the ranks' published state. Sources are scanned in rank order, each rank's
// in-flight samples in its in-flight-list order and its queue in FIFO order;
// in-flight migrants go, longest remaining first (ties: lower id), to the
// destination with the fewest in-flight samples that has KV room (ties: lower
// rank), else stay home; queued migrants go to the shallowest queue (first
// destination in plan order on ties).
std::vector<Move> place_online(const MigrationPlan& plan, const SampleState* st, int n, int G, const int* r_live,
                               const int* r_queue, const double* r_kv, const std::vector<double>& resv,
                               const std::vector<double>& remaining, double cap) {
  std::vector<Move> mv;
  if (plan.no_op) return mv;
  std::vector<char> dest(G, 0), moving(n, 0);
  for (int d : plan.destinations) dest[d] = 1;
  for (int id : plan.migrated) moving.at(id) = 1;
  std::vector<int> running(r_live, r_live + G), backlog(r_queue, r_queue + G);
  std::vector<double> kv(r_kv, r_kv + G);
  struct Cand {
    int sid, order;
  };
  std::vector<std::vector<Cand>> fl(G), qu(G);
  for (int s = 0; s < n; ++s) {
    if (!(st[s].flag & 1) || !moving[s]) continue;
    (st[s].flag & 2 ? fl : qu)[st[s].rank].push_back({s, st[s].order});
  }
  std::vector<int> in_flight, not_started;
  for (int r = 0; r < G; ++r) {
    if (dest[r]) continue;
    auto by_order = [](const Cand& a, const Cand& b) { return a.order < b.order; };
    std::sort(fl[r].begin(), fl[r].end(), by_order);
    std::sort(qu[r].begin(), qu[r].end(), by_order);
    for (const Cand& c : fl[r]) {
      in_flight.push_back(c.sid);
      kv[r] -= resv[c.sid];
      running[r] -= 1;
    }
    for (const Cand& c : qu[r]) not_started.push_back(c.sid);
  }
  std::stable_sort(in_flight.begin(), in_flight.end(), [&](int a, int b) {
    if (remaining[a] != remaining[b]) return remaining[a] > remaining[b];
    return a < b;
  });
  for (int s : in_flight) {
    int pick = -1;
    for (int d : plan.destinations) {
      if (cap > 0.0 && kv[d] + resv[s] > cap + 1e-6) continue;
      if (pick < 0 || running[d] < running[pick] || (running[d] == running[pick] && d < pick)) pick = d;
    }
    const int home = st[s].rank;
    if (pick < 0) {  // no destination has room: it stays
      kv[home] += resv[s];
      running[home] += 1;
      continue;
    }
    running[pick] += 1;
    kv[pick] += resv[s];
    mv.push_back({s, home, pick, true, st[s].gen});
  }
  for (int s : not_started) {
    int pick = -1;
    for (int d : plan.destinations)
      if (pick < 0 || backlog[d] < backlog[pick]) pick = d;
    backlog[pick] += 1;
    mv.push_back({s, st[s].rank, pick, false, 0});
  }
  return mv;
}

int forced_token(uint64_t seed, int sid, int k, int max_new, int V) {
  const uint64_t h = fpk::hash3(seed, fpk::kTagResponse, static_cast<uint64_t>(sid) * max_new + k);
  return static_cast<int>((h >> 32) % static_cast<uint64_t>(V));
}

float ms_between(cudaEvent_t a, cudaEvent_t b) {
  float ms = 0.f;
  FP_CUDA(cudaEventElapsedTime(&ms, a, b));
  return ms;
}

}  // namespace

GpuEngine* create_engine(const EngineSetup& s) {
  fpe::EngineConfig c;
  c.model[fpe::kActor] = to_dims(s.actor);
  c.model[fpe::kRef] = to_dims(s.ref);
  c.model[fpe::kCritic] = to_dims(s.critic);
  c.model[fpe::kReward] = to_dims(s.reward);
  c.weight_seed = s.weight_seed;
  c.max_prompt = s.max_prompt;
  c.max_new = s.max_new;
  c.max_samples = s.max_samples;
  c.max_live = s.max_live;
  c.kv_pool_bytes = s.kv_pool_bytes;
  c.max_prefill_tokens = s.max_prefill_tokens;
  c.max_infer_tokens = s.max_infer_tokens;
  c.rope_theta = s.rope_theta;
  c.device = s.device;
  auto* g = new GpuEngine;
  g->setup = s;
  g->eng = std::make_unique<fpe::Engine>(c);
  return g;
}

void destroy_engine(GpuEngine* e) { delete e; }

// Weight sync: after a training step updated a model on
// rank `src`, every rank pulls it over NVLink. Scatter + all-gather of 1/G
// slices through CUDA IPC peer pointers: src sends each byte once, every
// rank receives (G-1)/G of the blob from G-1 peers in parallel, and the
// copy kernels pull 1 MiB pieces with 16-byte vector loads.
double broadcast_model(GpuEngine* ge, int model, int src, const CommSetup& comm) {
  fpe::Engine& E = *ge->eng;
  FP_CUDA(cudaSetDevice(E.config().device));
  const int G = comm.world, me = comm.rank;
  if (model < 0 || model > 3) throw std::invalid_argument("broadcast_model: model index out of range");
  if (G < 1 || G > kMaxRanks || me < 0 || me >= G || src < 0 || src >= G)
    throw std::invalid_argument("broadcast_model: bad rank/world/src");
  if (G == 1) return 0.0;
  Region region(comm, 1, 1, 1);
  Header* hdr = region.hdr();
  uint8_t* blob = static_cast<uint8_t*>(E.model(model).blob);
  const size_t bytes = E.model(model).bytes;  // a multiple of 256
  FP_CUDA(cudaIpcGetMemHandle(&hdr->h_model[me], blob));
  region.barrier();
  std::vector<const uint8_t*> base(G);
  for (int r = 0; r < G; ++r) base[r] = r == me ? blob : static_cast<const uint8_t*>(E.open_ipc(hdr->h_model[r]));
  const size_t per = ((bytes + G - 1) / G + 255) & ~size_t(255);
  cudaStream_t st = E.decode_stream();
  auto pull = [&](int from, int slice, std::vector<fpk::CopyChunk>& list) {
    const size_t b0 = std::min(bytes, slice * per), b1 = std::min(bytes, (slice + 1) * per);
    for (size_t o = b0; o < b1; o += (1u << 20))
      list.push_back({base[from] + o, blob + o, std::min<size_t>(1u << 20, b1 - o)});
  };
  auto run = [&](const std::vector<fpk::CopyChunk>& list) {
    if (!list.empty()) {
      void* dl = E.decode_scratch(list.size() * sizeof(fpk::CopyChunk));
      E.upload(dl, list.data(), list.size() * sizeof(fpk::CopyChunk), st);
      fpk::copy_chunks(static_cast<const fpk::CopyChunk*>(dl), static_cast<int>(list.size()), st);
    }
    FP_CUDA(cudaStreamSynchronize(st));
    region.barrier();
  };
  FP_CUDA(cudaStreamSynchronize(st));
  region.barrier();
  const auto t0 = Clock::now();
  std::vector<fpk::CopyChunk> l1, l2;
  if (me != src) pull(src, me, l1);  // scatter: my slice from src
  run(l1);
  if (me != src)  // all-gather: every other slice from the rank that holds it
    for (int c = 0; c < G; ++c)
      if (c != me) pull(c, c, l2);
  run(l2);
  return std::chrono::duration<double>(Clock::now() - t0).count();
}

void reinit_model(GpuEngine* ge, int model, std::uint64_t seed) { ge->eng->reinit_model(model, seed); }

void load_weights(GpuEngine* ge, int model, int tensor, int layer, const void* host, std::int64_t n_elems) {
  ge->eng->load_tensor(model, tensor, layer, host, n_elems);
}

std::uint64_t model_checksum(GpuEngine* ge, int model) { return ge->eng->model_checksum(model); }

std::vector<int> synthetic_prompts(const GpuEngine* e, int n, std::uint64_t token_seed) {
  const int P = e->setup.max_prompt, V = e->setup.actor.vocab;
  std::vector<int> p(static_cast<size_t>(n) * P);
  for (size_t i = 0; i < p.size(); ++i)
    p[i] = static_cast<int>((fpk::hash3(token_seed, fpk::kTagPrompt, i) >> 32) % static_cast<uint64_t>(V));
  return p;
}

// Pinned host ring that receives the decode slots' next-input ids after each
// step (free-run EOS detection), one event per entry.
struct TokRing {
  static constexpr int kSlots = 16;
  int* host = nullptr;
  int width = 0;
  cudaEvent_t ev[kSlots] = {};
  explicit TokRing(int w) : width(w) {
    FP_CUDA(cudaMallocHost(&host, static_cast<size_t>(kSlots) * w * sizeof(int)));
    for (auto& e : ev) FP_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  ~TokRing() {
    for (auto& e : ev) cudaEventDestroy(e);
    cudaFreeHost(host);
  }
  int* slot(int k) { return host + static_cast<size_t>(k % kSlots) * width; }
};

GpuEngine::~GpuEngine() = default;

ExecResult execute(GpuEngine* ge, const std::vector<GenSample>& batch, const GenSimConfig& cfg, int r_t,
                   const EngineOptions& opts, const CommSetup& comm, const std::vector<int>* prompts_in) {
  fpe::Engine& E = *ge->eng;
  const fpe::EngineConfig& ec = E.config();
  FP_CUDA(cudaSetDevice(ec.device));
  const int n = static_cast<int>(batch.size());
  const int G = comm.world, me = comm.rank;
  if (G < 1 || G > kMaxRanks || me < 0 || me >= G) throw std::invalid_argument("execute: bad rank/world");
  if (cfg.num_instances != G) throw std::invalid_argument("execute: cfg.num_instances must equal the world size");
  if (n > ec.max_samples) throw std::invalid_argument("execute: batch larger than engine max_samples");
  const bool free_run = opts.eos_id >= 0;
  for (int s = 0; s < n; ++s) {
    const GenSample& b = batch[s];
    if (b.id != s) throw std::invalid_argument("execute: batch ids must be 0..n-1 in order");
    if (b.prompt_len < 1 || b.prompt_len > ec.max_prompt)
      throw std::invalid_argument("execute: prompt_len must lie in [1, max_prompt]");
    if (!free_run && (b.target_output_len < 1 || b.target_output_len > ec.max_new))
      throw std::invalid_argument("execute: target_output_len must lie in [1, max_new]");
    if (b.generated != 0) throw std::invalid_argument("execute: samples must start ungenerated");
  }
  const int V = ec.model[fpe::kActor].V;
  const int mode = static_cast<int>(opts.token_mode);
  const bool fused = opts.schedule == Schedule::kFused;
  if (free_run && opts.token_mode == TokenMode::kForced)
    throw std::invalid_argument("execute: eos_id (free-run) needs token_mode greedy or sample");
  if (free_run && opts.eos_id >= V) throw std::invalid_argument("execute: eos_id outside the actor vocabulary");
  if (opts.eos_lag < 0 || opts.eos_lag > 8) throw std::invalid_argument("execute: eos_lag must lie in [0, 8]");
  if (opts.top_k < 0 || opts.top_k > fpk::kTopKMax || !(opts.top_p > 0.f && opts.top_p <= 1.f))
    throw std::invalid_argument("execute: top_k must lie in [0, 1024] and top_p in (0, 1]");
  const bool want_trigger = fused && G > 1 && r_t > 0;
  const bool online = want_trigger && (free_run || opts.online_trigger);
  const bool clock_trigger = want_trigger && !online;

  ExecResult res;
  res.online = online;
  res.decision = fused ? simulate_fused(batch, cfg, r_t) : simulate_serial(batch, cfg);
  std::vector<Move> moves;
  if (clock_trigger) {
    res.trigger = fused_trigger(batch, cfg, r_t);
    moves = moves_of(res.trigger);
  }
  const bool clock_migrate = clock_trigger && res.trigger.triggered && !res.trigger.plan.no_op;

  // ---- host data --------------------------------------------------------------
  std::vector<int> prompts = prompts_in ? *prompts_in : synthetic_prompts(ge, n, opts.token_seed);
  if (static_cast<int64_t>(prompts.size()) < static_cast<int64_t>(n) * ec.max_prompt)
    throw std::invalid_argument("execute: prompts must hold n * max_prompt ids");
  // Response cap and KV reservation per sample. Teacher-forced lengths: the
  // target and the reference's reserved kv_bytes (genfuse.cpp:226-236).
  // Free-run: max_new and (prompt + max_new) x kv_bytes_per_token (core.cpp:90-93).
  std::vector<int> rcap(n);
  std::vector<double> resv(n);
  const double kv_tok = kv_bytes_per_token(cfg.actor);
  for (int s = 0; s < n; ++s) {
    rcap[s] = free_run ? ec.max_new : batch[s].target_output_len;
    resv[s] = free_run ? (batch[s].prompt_len + ec.max_new) * kv_tok : batch[s].kv_bytes;
  }
  // Device layout of the response-aligned experience arrays: packed by target
  // (teacher-forced) or one max_new row per sample (free-run; compacted on the host).
  std::vector<int64_t> layout(n + 1, 0);
  for (int s = 0; s < n; ++s) layout[s + 1] = layout[s] + rcap[s];
  const int64_t total = layout[n];
  const int max_pages = E.pages_for(ec.max_prompt + ec.max_new);

  Region region(comm, n, max_pages, total);
  Header* hdr = region.hdr();
  try {
  int* rlen = region.resp_len();
  SampleState* sstate = region.state();
  for (int s = me; s < n; s += G) {
    sstate[s] = SampleState{0, me, 0, 0};
    rlen[s] = 0;
  }

  // peer pointers (G > 1): histories and KV pools of every rank
  std::vector<const int*> peer_tok(G, nullptr);
  std::vector<const float*> peer_logp(G, nullptr);
  std::vector<const uint8_t*> peer_pool(G, nullptr);
  std::vector<void*> opened;
  peer_tok[me] = E.d_hist_tok();
  peer_logp[me] = E.d_hist_logp();
  peer_pool[me] = E.pool_base();
  if (G > 1) {
    FP_CUDA(cudaIpcGetMemHandle(&hdr->h_hist_tok[me], E.d_hist_tok()));
    FP_CUDA(cudaIpcGetMemHandle(&hdr->h_hist_logp[me], E.d_hist_logp()));
    FP_CUDA(cudaIpcGetMemHandle(&hdr->h_pool[me], E.pool_base()));
    region.barrier();
    const auto ti = Clock::now();
    for (int r = 0; r < G; ++r) {
      if (r == me) continue;
      peer_tok[r] = static_cast<const int*>(E.open_ipc(hdr->h_hist_tok[r]));
      peer_logp[r] = static_cast<const float*>(E.open_ipc(hdr->h_hist_logp[r]));
      peer_pool[r] = static_cast<const uint8_t*>(E.open_ipc(hdr->h_pool[r]));
    }
    res.stats.ipc_seconds += std::chrono::duration<double>(Clock::now() - ti).count();
  }

  E.set_layout(layout);
  uint64_t ptag = 1469598103934665603ull;  // FNV-1a of the prompt ids
  for (int v : prompts) ptag = (ptag ^ static_cast<uint32_t>(v)) * 1099511628211ull;
  const long long launches0 = fpk::launch_count();
  if (!(opts.resident && E.prompts_tag() == ptag)) E.load_prompts(prompts.data(), n, ptag);
  if (opts.probe_attention) E.set_attn_probe(true);
  cudaStream_t sd = E.decode_stream(), si = E.infer_stream();
  FP_CUDA(cudaStreamSynchronize(sd));
  region.barrier();

  // ---- timing -----------------------------------------------------------------------
  std::vector<cudaEvent_t> events;
  auto new_event = [&](cudaStream_t st) {
    cudaEvent_t e;
    FP_CUDA(cudaEventCreate(&e));
    FP_CUDA(cudaEventRecord(e, st));
    events.push_back(e);
    return e;
  };
  const auto wall0 = Clock::now();
  cudaEvent_t ev_start = new_event(sd);
  FP_CUDA(cudaStreamWaitEvent(si, ev_start, 0));
  std::vector<cudaEvent_t> step_begin, step_end;
  std::vector<int> finish_step(n, -1);
  res.finish_instance.assign(n, -1);

  // ---- instance state --------------------------------------------------------------
  std::deque<int> queue;
  for (int s = me; s < n; s += G) queue.push_back(s);
  std::vector<Live> live;
  double kv_used = 0.0;
  const double cap = cfg.cluster.kv_capacity_per_instance;
  std::vector<int> slot_of(n, -1);
  std::vector<int> eos_len(n, -1);  // free-run: response length at the first emitted EOS

  // decision-clock trigger snapshot of this instance
  std::unordered_map<int, int> snap_live;  // sid -> generated
  std::vector<int> snap_queue;
  if (clock_migrate) {
    for (const auto& r : res.trigger.state.samples) {
      if (r.instance != me) continue;
      if (r.admitted)
        snap_live[r.id] = r.generated;
      else
        snap_queue.push_back(r.id);
    }
  }
  auto at_snapshot = [&]() {
    if (live.size() != snap_live.size() || queue.size() != snap_queue.size()) return false;
    for (const Live& l : live) {
      auto it = snap_live.find(l.sid);
      if (it == snap_live.end() || it->second != l.gen) return false;
    }
    std::vector<int> q(queue.begin(), queue.end());
    std::vector<int> sq = snap_queue;
    std::sort(q.begin(), q.end());
    std::sort(sq.begin(), sq.end());
    return q == sq;
  };
  // online trigger: raised by the rank whose retirement leaves fewer than r_t
  // unfinished samples in the batch (at once if n < r_t, genfuse.cpp:484-490)
  if (online && n < r_t) hdr->trig_flag.store(1);
  auto count_finished = [&]() {
    const int f = hdr->finished.fetch_add(1) + 1;
    if (online && n - f < r_t) hdr->trig_flag.store(1);
  };

  // publication of finished samples (G > 1: after the GPU step completed).
  // Appends to the shared order are serialised by a tiny process-shared lock.
  std::deque<std::pair<int, int>> to_publish;  // (sid, step index that finished it)
  std::atomic<int>& n_pub = hdr->n_pub;
  auto publish_now = [&](int sid) {
    region.owner()[sid] = me;
    while (hdr->lock.exchange(1, std::memory_order_acquire)) std::this_thread::yield();
    const int idx = n_pub.load(std::memory_order_relaxed);
    region.pub_order()[idx] = sid;
    n_pub.store(idx + 1, std::memory_order_release);
    hdr->lock.store(0, std::memory_order_release);
  };

  auto flush_publish = [&](bool wait_all) {
    while (!to_publish.empty()) {
      const int k = to_publish.front().second;
      if (G > 1 && k >= 0) {
        if (wait_all) {
          FP_CUDA(cudaEventSynchronize(step_end[k]));
        } else if (cudaEventQuery(step_end[k]) != cudaSuccess) {
          break;
        }
      }
      publish_now(to_publish.front().first);
      to_publish.pop_front();
    }
  };

  // ---- scoring claims --------------------------------------------------------------------
  struct Batch {
    cudaEvent_t b, e;
  };
  std::deque<Batch> inflight;
  std::vector<int> my_scored;
  bool gen_done_me = false;
  double infer_ms = 0.0;
  auto retire_batches = [&](bool wait) {
    while (!inflight.empty()) {
      if (wait) FP_CUDA(cudaEventSynchronize(inflight.front().e));
      else if (cudaEventQuery(inflight.front().e) != cudaSuccess) break;
      infer_ms += ms_between(inflight.front().b, inflight.front().e);
      inflight.pop_front();
    }
  };
  auto service = [&]() {
    const bool all_gen_done = hdr->gen_done.load() >= G;
    if (!fused && !all_gen_done) return;
    retire_batches(false);
    const int max_inflight = gen_done_me ? 2 : 1;
    while (static_cast<int>(inflight.size()) < max_inflight) {
      int c = hdr->n_claimed.load();
      const int avail_end = n_pub.load();
      if (c >= avail_end) return;
      // take finished samples in publish order up to claim_tokens tokens
      int end = c;
      int64_t toks = 0;
      const int* order = region.pub_order();
      while (end < avail_end && toks < opts.claim_tokens) {
        const int sid = order[end];
        toks += batch[sid].prompt_len + rlen[sid];
        ++end;
      }
      // Generating ranks take full batches only; an idle rank takes whatever
      // is there when it has nothing in flight; after every rank finished
      // generating, the remainder goes in any size.
      const bool hungry = gen_done_me && inflight.empty();
      if (toks < opts.claim_tokens && !all_gen_done && !hungry && !(gen_done_me && G == 1)) return;
      // while this rank's decode batch is large (bandwidth-bound steps) scoring
      // waits; it overlaps the latency-bound tail instead
      if (!gen_done_me && !all_gen_done && opts.claim_max_live > 0 &&
          static_cast<int>(live.size()) > opts.claim_max_live)
        return;
      if (!hdr->n_claimed.compare_exchange_strong(c, end)) continue;
      std::vector<fpe::Engine::InferItem> items;
      for (int i = c; i < end; ++i) {
        const int sid = order[i];
        const int own = region.owner()[sid];
        items.push_back({sid, batch[sid].prompt_len, rlen[sid],
                         peer_tok[own] + static_cast<size_t>(sid) * ec.max_new,
                         peer_logp[own] + static_cast<size_t>(sid) * ec.max_new});
        my_scored.push_back(sid);
        res.stats.infer_tokens += batch[sid].prompt_len + rlen[sid];
      }
      res.stats.infer_samples += end - c;
      // local finishes may still be in flight on the decode stream
      if (!step_end.empty()) FP_CUDA(cudaStreamWaitEvent(si, step_end.back(), 0));
      Batch bt;
      FP_CUDA(cudaEventCreate(&bt.b));
      FP_CUDA(cudaEventCreate(&bt.e));
      events.push_back(bt.b);
      events.push_back(bt.e);
      FP_CUDA(cudaEventRecord(bt.b, si));
      E.infer(items, opts.kl_beta, opts.gamma, opts.lam, /*yield=*/fused && !gen_done_me);
      FP_CUDA(cudaEventRecord(bt.e, si));
      inflight.push_back(bt);
    }
  };

  // ---- free-run EOS detection ---------------------------------------------------------
  // After each decode step the slots' next-input ids (the tokens just emitted)
  // are copied to a pinned ring; the host inspects step k when step k + lag
  // has been enqueued, so it never waits on the step it just launched.
  struct StepRows {
    int k;                                 // step index (ring entry)
    std::vector<std::array<int, 3>> rows;  // (sid, slot, response index of the emitted token)
  };
  std::deque<StepRows> pending;
  if (free_run && !ge->ring) ge->ring = std::make_unique<TokRing>(ec.max_live + 1);
  auto process_tokens = [&](bool all) {
    while (!pending.empty() && (all || static_cast<int>(pending.size()) > opts.eos_lag)) {
      const StepRows& p = pending.front();
      FP_CUDA(cudaEventSynchronize(ge->ring->ev[p.k % TokRing::kSlots]));
      const int* t = ge->ring->slot(p.k);
      for (const auto& r : p.rows)
        if (eos_len[r[0]] < 0 && t[r[1]] == opts.eos_id) eos_len[r[0]] = r[2] + 1;
      pending.pop_front();
    }
  };

  // ---- generation loop ----------------------------------------------------------------
  std::vector<fpe::Engine::DecodeRow> rows;
  auto retire_finished = [&]() {
    if (free_run) {
      bool at_cap = false;
      for (const Live& l : live) at_cap |= l.gen >= l.target;
      process_tokens(at_cap);  // a row at max_new must know whether it emitted EOS earlier
    }
    std::vector<Live> keep;
    keep.reserve(live.size());
    for (const Live& l : live) {
      const bool eos = free_run && eos_len[l.sid] >= 0;
      if (l.gen >= l.target || eos) {
        const int R = eos ? eos_len[l.sid] : l.target;
        if (eos) {
          res.stats.eos_retired += 1;
          res.stats.overrun_rows += l.gen - R;
        }
        kv_used -= resv[l.sid];
        E.release(l.slot);
        slot_of[l.sid] = -1;
        finish_step[l.sid] = static_cast<int>(step_end.size()) - 1;
        res.finish_instance[l.sid] = me;
        rlen[l.sid] = R;
        to_publish.emplace_back(l.sid, static_cast<int>(step_end.size()) - 1);
        count_finished();
      } else {
        keep.push_back(l);
      }
    }
    live.swap(keep);
  };
  auto admit_fitting = [&]() {
    std::vector<fpe::Engine::PrefillItem> items;
    while (!queue.empty()) {
      const int s = queue.front();
      const double kv = resv[s];
      if (cap > 0.0 && kv_used + kv > cap + 1e-6) break;
      queue.pop_front();
      kv_used += kv;
      const int P = batch[s].prompt_len, R = rcap[s];
      const int slot = E.reserve(P - 1 + R);
      E.upload_block_table(slot, sd);
      slot_of[s] = slot;
      const int* pr = prompts.data() + static_cast<size_t>(s) * ec.max_prompt;
      items.push_back({s, slot, P - 1, pr, pr[P - 1]});
      live.push_back({s, slot, 0, R});
      res.stats.prefill_tokens += P - 1;
    }
    if (!items.empty()) E.prefill(items);
  };
  auto decode_one = [&]() {
    rows.clear();
    int64_t ctx = 0;
    for (const Live& l : live) {
      const int P = batch[l.sid].prompt_len;
      const int tgt = mode == 0 ? forced_token(opts.token_seed, l.sid, l.gen, ec.max_new, V) : 0;
      rows.push_back({l.sid, l.slot, P - 1 + l.gen, l.gen, tgt});
      ctx += P + l.gen;
    }
    cudaEvent_t b, e;
    FP_CUDA(cudaEventCreate(&b));
    FP_CUDA(cudaEventCreate(&e));
    events.push_back(b);
    events.push_back(e);
    FP_CUDA(cudaEventRecord(b, sd));
    E.decode(rows, mode, 1.0f / opts.temperature, opts.sample_seed, opts.top_k, opts.top_p);
    FP_CUDA(cudaEventRecord(e, sd));
    const int k = static_cast<int>(step_end.size());
    step_begin.push_back(b);
    step_end.push_back(e);
    if (free_run) {
      StepRows p{k, {}};
      p.rows.reserve(live.size());
      for (const Live& l : live) p.rows.push_back({l.sid, l.slot, l.gen});
      FP_CUDA(cudaMemcpyAsync(ge->ring->slot(k), E.d_cur_tok(), static_cast<size_t>(ge->ring->width) * sizeof(int),
                              cudaMemcpyDeviceToHost, sd));
      FP_CUDA(cudaEventRecord(ge->ring->ev[k % TokRing::kSlots], sd));
      pending.push_back(std::move(p));
    }
    for (Live& l : live) ++l.gen;
    res.stats.decode_steps += 1;
    res.stats.decode_rows += static_cast<int64_t>(rows.size());
    res.step_rows.push_back(static_cast<int>(rows.size()));
    res.step_ctx.push_back(ctx);
    res.stats.decode_ctx_tokens += ctx;
    // bound host run-ahead
    const int kk = k - opts.run_ahead;
    if (kk >= 0) FP_CUDA(cudaEventSynchronize(step_end[kk]));
  };

  // Runs this instance until it has no work (false) or reaches the trigger
  // boundary (true): the decision clock's snapshot state (checked after
  // admission and after each step, which covers the at-trigger admission quirk
  // and Simulation::snapshot's llround, genfuse.cpp:116-118), or — online — a
  // raised trigger flag at the top of a step (after retirement, before admission).
  auto generation = [&](bool stop) -> bool {
    for (;;) {
      retire_finished();
      flush_publish(false);
      if (stop && online && hdr->trig_flag.load()) return true;
      admit_fitting();
      if (stop && clock_migrate && at_snapshot()) return true;
      if (live.empty()) {
        if (!queue.empty()) throw InfeasibleError("generation wedged: KV capacity below a single sample");
        return false;
      }
      decode_one();
      if (stop && clock_migrate && at_snapshot()) return true;
      service();
      region.check_peers();
    }
  };

  // ---- one-shot migration ------------------------------------------------------------------
  // Sources have published the page lists of their in-flight migrants; each
  // destination pulls them over NVLink, then every rank drops what left.
  std::vector<char> gone(n, 0);
  auto migrate = [&](const std::vector<Move>& mv, bool recompute) {
    const auto tm0 = Clock::now();
    std::vector<fpk::CopyChunk> pages, hist;
    std::vector<int> quad_slot, quad_sid, quad_gen, quad_P;
    std::vector<fpe::Engine::PrefillItem> redo;
    std::vector<std::vector<int>> redo_tokens;
    for (const Move& m : mv) {
      if (m.dst != me) continue;
      res.received_sample.push_back(m.sid);
      res.received_from.push_back(m.src);
      if (!m.inflight) {
        queue.push_back(m.sid);
        continue;
      }
      const int P = batch[m.sid].prompt_len, R = rcap[m.sid];
      const int slot = E.reserve(P - 1 + R);
      E.upload_block_table(slot, sd);
      slot_of[m.sid] = slot;
      kv_used += resv[m.sid];
      live.push_back({m.sid, slot, m.gen, R});
      res.stats.migrated_in += 1;
      // history rows (token ids + actor log-probs), exact length
      const size_t hoff = static_cast<size_t>(m.sid) * ec.max_new;
      if (m.gen > 0) {
        const size_t hb = static_cast<size_t>(m.gen) * 4;
        hist.push_back({peer_tok[m.src] + hoff, E.d_hist_tok() + hoff, hb});
        hist.push_back({peer_logp[m.src] + hoff, E.d_hist_logp() + hoff, hb});
      }
      if (!recompute) {
        const int ctx = P - 1 + m.gen;
        const int np = E.pages_for(ctx);
        const auto& dst_pages = E.pages_of(slot);
        const int* src_pages = region.pages(m.sid);
        for (int i = 0; i < np; ++i) {
          pages.push_back({peer_pool[m.src] + static_cast<size_t>(src_pages[i]) * E.page_bytes(),
                           E.pool_base() + static_cast<size_t>(dst_pages[i]) * E.page_bytes(), E.page_bytes()});
          res.stats.migrated_bytes += static_cast<int64_t>(E.page_bytes());
        }
        quad_slot.push_back(slot);
        quad_sid.push_back(m.sid);
        quad_gen.push_back(m.gen);
        quad_P.push_back(P);
      } else {
        redo.push_back({m.sid, slot, P - 1 + m.gen, nullptr, 0});
      }
    }
    auto al = [](size_t b) { return (b + 255) & ~size_t(255); };
    const size_t pb = al(pages.size() * sizeof(fpk::CopyChunk)), hb = al(hist.size() * sizeof(fpk::CopyChunk));
    uint8_t* scratch = static_cast<uint8_t*>(E.decode_scratch(pb + hb + quad_slot.size() * 16 + 256));
    if (!pages.empty()) {  // whole pages: 16-byte vector copies
      auto* d = reinterpret_cast<fpk::CopyChunk*>(scratch);
      E.upload(d, pages.data(), pages.size() * sizeof(fpk::CopyChunk), sd);
      fpk::copy_chunks(d, static_cast<int>(pages.size()), sd);
    }
    if (!hist.empty()) {  // history rows: 4-byte granular, nothing past the row's generated prefix
      auto* d = reinterpret_cast<fpk::CopyChunk*>(scratch + pb);
      E.upload(d, hist.data(), hist.size() * sizeof(fpk::CopyChunk), sd);
      fpk::copy_words(d, static_cast<int>(hist.size()), sd);
    }
    if (!quad_slot.empty()) {
      const int q = static_cast<int>(quad_slot.size());
      std::vector<int> quad;
      quad.insert(quad.end(), quad_slot.begin(), quad_slot.end());
      quad.insert(quad.end(), quad_sid.begin(), quad_sid.end());
      quad.insert(quad.end(), quad_gen.begin(), quad_gen.end());
      quad.insert(quad.end(), quad_P.begin(), quad_P.end());
      int* d = reinterpret_cast<int*>(scratch + pb + hb);
      E.upload(d, quad.data(), quad.size() * 4, sd);
      fpk::cur_from_hist(d, q, E.d_hist_tok(), ec.max_new, E.d_prompts(), ec.max_prompt, E.d_cur_tok(), sd);
    }
    if (!redo.empty()) {
      // recompute: prefill prompt + generated prefix on this GPU
      FP_CUDA(cudaStreamSynchronize(sd));
      for (auto& it : redo) {
        const int gen = it.ctx_tokens - (batch[it.sid].prompt_len - 1);
        std::vector<int> toks(prompts.begin() + static_cast<size_t>(it.sid) * ec.max_prompt,
                              prompts.begin() + static_cast<size_t>(it.sid) * ec.max_prompt + batch[it.sid].prompt_len);
        std::vector<int> h(std::max(gen, 1));
        if (gen > 0)
          FP_CUDA(cudaMemcpy(h.data(), E.d_hist_tok() + static_cast<size_t>(it.sid) * ec.max_new, gen * 4,
                             cudaMemcpyDeviceToHost));
        for (int k = 0; k + 1 < gen; ++k) toks.push_back(h[k]);
        it.next_token = gen > 0 ? h[gen - 1] : toks[batch[it.sid].prompt_len - 1];
        redo_tokens.push_back(std::move(toks));
      }
      for (size_t i = 0; i < redo.size(); ++i) redo[i].tokens = redo_tokens[i].data();
      E.prefill(redo);
    }
    FP_CUDA(cudaStreamSynchronize(sd));
    region.barrier();
    // sources drop what left (reference order: in-flight list order, then FIFO)
    for (const Move& m : mv)
      if (m.src == me) gone[m.sid] = 1;
    std::vector<Live> keep;
    for (const Live& l : live) {
      if (gone[l.sid]) {
        kv_used -= resv[l.sid];
        E.release(l.slot);
        slot_of[l.sid] = -1;
      } else {
        keep.push_back(l);
      }
    }
    live.swap(keep);
    std::deque<int> q2;
    for (int s : queue)
      if (!gone[s]) q2.push_back(s);
    queue.swap(q2);
    res.stats.migrate_seconds = std::chrono::duration<double>(Clock::now() - tm0).count();
  };

  auto mark_trigger = [&]() {
    FP_CUDA(cudaStreamSynchronize(sd));
    cudaEvent_t ev_trig = new_event(sd);
    FP_CUDA(cudaEventSynchronize(ev_trig));
    res.stats.trigger_seconds = ms_between(ev_start, ev_trig) * 1e-3;
  };

  // decision-clock migration: this rank is at its snapshot state
  auto clock_pause = [&]() {
    mark_trigger();
    for (const Move& m : moves)
      if (m.src == me && m.inflight) {
        const auto& pg = E.pages_of(slot_of[m.sid]);
        std::copy(pg.begin(), pg.end(), region.pages(m.sid));
      }
    flush_publish(true);
    region.barrier();
    migrate(moves, res.trigger.plan.mechanism == MigrationMechanism::kRecomputePrefill);
  };

  // online migration: quiesce, publish this rank's state, plan on the union
  auto online_pause = [&]() {
    mark_trigger();
    if (free_run) process_tokens(true);
    retire_finished();
    flush_publish(true);
    for (size_t i = 0; i < live.size(); ++i) {
      const Live& l = live[i];
      sstate[l.sid] = SampleState{3, me, l.gen, static_cast<int>(i)};
      const auto& pg = E.pages_of(l.slot);
      std::copy(pg.begin(), pg.end(), region.pages(l.sid));
    }
    for (size_t i = 0; i < queue.size(); ++i) sstate[queue[i]] = SampleState{1, me, 0, static_cast<int>(i)};
    hdr->r_live[me] = static_cast<int>(live.size());
    hdr->r_queue[me] = static_cast<int>(queue.size());
    hdr->r_kv[me] = kv_used;
    hdr->r_time[me] = res.stats.trigger_seconds;
    region.barrier();
    TriggerSnapshot& t = res.trigger;
    t.triggered = true;
    t.time = 0.0;
    for (int r = 0; r < G; ++r) t.time = std::max(t.time, hdr->r_time[r]);
    t.state.time = t.time;
    std::vector<double> remaining(n, 0.0);
    for (int s = 0; s < n; ++s) {
      const SampleState& x = sstate[s];
      if (!(x.flag & 1)) continue;
      t.state.samples.push_back({s, x.rank, resv[s], x.gen, batch[s].prompt_len, (x.flag & 2) != 0});
      remaining[s] = static_cast<double>(rcap[s] - x.gen);
    }
    t.plan = plan_migration(t.state, r_t, cfg);
    const std::vector<Move> mv =
        place_online(t.plan, sstate, n, G, hdr->r_live, hdr->r_queue, hdr->r_kv, resv, remaining, cap);
    for (const Move& m : mv) {
      t.move_sample.push_back(m.sid);
      t.move_from.push_back(m.src);
      t.move_to.push_back(m.dst);
    }
    region.barrier();  // every rank has read the published state
    if (!t.plan.no_op) migrate(mv, t.plan.mechanism == MigrationMechanism::kRecomputePrefill);
  };

  auto wait_idle = [&](auto&& until) {
    // serve scoring while waiting; progress (publications, claims) resets the deadline
    auto t0 = Clock::now();
    int last = -1;
    while (!until()) {
      flush_publish(false);
      service();
      region.check_peers();
      retire_batches(false);
      const int prog = hdr->n_pub.load() + hdr->n_claimed.load();
      if (prog != last) {
        last = prog;
        t0 = Clock::now();
      } else if (Clock::now() - t0 > std::chrono::seconds(900)) {
        throw std::runtime_error("executor: no progress from the other ranks for 900 s");
      }
      std::this_thread::yield();
    }
  };

  bool handled = !(clock_migrate || online);
  for (;;) {
    gen_done_me = false;
    const bool paused = generation(!handled);
    if (paused) {
      if (online) online_pause(); else clock_pause();
      handled = true;
      continue;
    }
    gen_done_me = true;
    if (handled) break;
    if (clock_migrate)
      throw std::runtime_error("executor: the decision clock's trigger state was never reached on rank " +
                               std::to_string(me));
    // online: the trigger always fires (at the latest when the last sample
    // retires, since r_t >= 1), and every rank must take part in the plan —
    // it may be chosen as a destination and receive work
    flush_publish(true);
    wait_idle([&] { return hdr->trig_flag.load() != 0; });
    online_pause();
    handled = true;
  }
  if (free_run) process_tokens(true);

  // ---- generation finished on this rank -----------------------------------------------
  flush_publish(true);
  gen_done_me = true;
  hdr->gen_done.fetch_add(1);
  wait_idle([&] { return hdr->n_claimed.load() >= n; });
  retire_batches(true);
  E.synchronize();
  cudaEvent_t ev_end = new_event(sd);
  FP_CUDA(cudaEventSynchronize(ev_end));
  region.barrier();  // every rank's retirements (response lengths) are visible

  // compact response offsets (free-run lengths are known now)
  std::vector<int64_t> resp_off(n + 1, 0);
  for (int s = 0; s < n; ++s) resp_off[s + 1] = resp_off[s] + rlen[s];

  // ---- experience hand-off (length-balanced DP mini-batches) ----------------------------
  if (opts.handoff_dp > 0) {
    const int dp = opts.handoff_dp;
    if (dp % G != 0) throw std::invalid_argument("handoff_dp must be a multiple of the world size");
    Handoff& h = res.handoff;
    std::vector<int> lens(n);
    for (int s = 0; s < n; ++s) lens[s] = batch[s].prompt_len + rlen[s];
    const auto groups = fuseplan::balance_minibatch(lens, dp);
    h.dp = dp;
    h.group_off.assign(1, 0);
    for (const auto& g : groups) {
      h.order.insert(h.order.end(), g.begin(), g.end());
      h.group_off.push_back(static_cast<int>(h.order.size()));
    }
    h.packed_off.assign(n + 1, 0);
    for (int k = 0; k < n; ++k) h.packed_off[k + 1] = h.packed_off[k] + rlen[h.order[k]];
    h.group_begin = me * dp / G;
    h.group_end = (me + 1) * dp / G;
    // where each sample's experience lives (the rank that scored it)
    for (int sid : my_scored) region.scorer()[sid] = me;
    std::vector<uint8_t*> exp_base(G, nullptr);
    exp_base[me] = static_cast<uint8_t*>(E.exp_blob());
    if (G > 1) {
      FP_CUDA(cudaIpcGetMemHandle(&hdr->h_exp[me], E.exp_blob()));
      region.barrier();
      // not cached: the experience blob is reallocated when the batch layout changes
      const auto ti = Clock::now();
      for (int r = 0; r < G; ++r) {
        if (r == me) continue;
        void* p = nullptr;
        FP_CUDA(cudaIpcOpenMemHandle(&p, hdr->h_exp[r], cudaIpcMemLazyEnablePeerAccess));
        exp_base[r] = static_cast<uint8_t*>(p);
        opened.push_back(p);
      }
      res.stats.ipc_seconds += std::chrono::duration<double>(Clock::now() - ti).count();
    }
    // array offsets inside an experience blob (identical layout on every rank)
    const fpe::Engine::Experience& X0 = E.experience();
    const uint8_t* b0 = exp_base[me];
    const size_t aoff[9] = {
        static_cast<size_t>(reinterpret_cast<const uint8_t*>(X0.tokens) - b0),
        static_cast<size_t>(reinterpret_cast<const uint8_t*>(X0.logp_actor) - b0),
        static_cast<size_t>(reinterpret_cast<const uint8_t*>(X0.logp_ref) - b0),
        static_cast<size_t>(reinterpret_cast<const uint8_t*>(X0.values) - b0),
        static_cast<size_t>(reinterpret_cast<const uint8_t*>(X0.kl) - b0),
        static_cast<size_t>(reinterpret_cast<const uint8_t*>(X0.reward) - b0),
        static_cast<size_t>(reinterpret_cast<const uint8_t*>(X0.adv) - b0),
        static_cast<size_t>(reinterpret_cast<const uint8_t*>(X0.ret) - b0),
        static_cast<size_t>(reinterpret_cast<const uint8_t*>(X0.score) - b0)};
    const int k0 = h.group_off[h.group_begin], k1 = h.group_off[h.group_end];
    const int64_t t0 = h.packed_off[k0];
    const fpe::Engine::Experience& D = E.handoff_buffers(h.packed_off[k1] - t0, k1 - k0);
    uint8_t* dbase[9] = {reinterpret_cast<uint8_t*>(D.tokens), reinterpret_cast<uint8_t*>(D.logp_actor),
                         reinterpret_cast<uint8_t*>(D.logp_ref), reinterpret_cast<uint8_t*>(D.values),
                         reinterpret_cast<uint8_t*>(D.kl), reinterpret_cast<uint8_t*>(D.reward),
                         reinterpret_cast<uint8_t*>(D.adv), reinterpret_cast<uint8_t*>(D.ret),
                         reinterpret_cast<uint8_t*>(D.score)};
    std::vector<fpk::CopyChunk> chunks;
    for (int k = k0; k < k1; ++k) {
      const int sid = h.order[k];
      const int src = region.scorer()[sid];
      const int64_t R = rlen[sid];
      for (int a = 0; a < 9; ++a) {
        const bool per_sample = a == 8;
        const uint8_t* sp = exp_base[src] + aoff[a] + (per_sample ? static_cast<size_t>(sid) : layout[sid]) * 4;
        uint8_t* dpp = dbase[a] + (per_sample ? static_cast<size_t>(k - k0) : h.packed_off[k] - t0) * 4;
        const uint64_t bytes = static_cast<uint64_t>(per_sample ? 1 : R) * 4;
        if (bytes == 0) continue;
        chunks.push_back({sp, dpp, bytes});
        h.bytes += static_cast<int64_t>(bytes);
        if (src != me) h.peer_bytes += static_cast<int64_t>(bytes);
      }
    }
    cudaEvent_t hb = new_event(sd);
    if (!chunks.empty()) {
      void* dl = E.decode_scratch(chunks.size() * sizeof(fpk::CopyChunk));
      E.upload(dl, chunks.data(), chunks.size() * sizeof(fpk::CopyChunk), sd);
      fpk::copy_words(static_cast<const fpk::CopyChunk*>(dl), static_cast<int>(chunks.size()), sd);
    }
    cudaEvent_t he = new_event(sd);
    FP_CUDA(cudaEventSynchronize(he));
    h.seconds = ms_between(hb, he) * 1e-3;
    h.tokens = D.tokens;
    const float* fa[7] = {D.logp_actor, D.logp_ref, D.values, D.kl, D.reward, D.adv, D.ret};
    for (int a = 0; a < 7; ++a) h.arrays[a] = fa[a];
    h.score = D.score;
    region.barrier();  // every rank has pulled before any blob may change
    for (void* p : opened) cudaIpcCloseMemHandle(p);
    opened.clear();
  }

  // ---- stats ------------------------------------------------------------------------------
  res.stats.gen_seconds = step_end.empty() ? 0.0 : ms_between(ev_start, step_end.back()) * 1e-3;
  double dec_ms = 0.0;
  res.step_ms.resize(step_end.size());
  for (size_t k = 0; k < step_end.size(); ++k) {
    res.step_ms[k] = ms_between(step_begin[k], step_end[k]);
    dec_ms += res.step_ms[k];
  }
  res.stats.decode_gpu_seconds = dec_ms * 1e-3;
  res.stats.infer_busy_seconds = infer_ms * 1e-3;
  res.finish_wall.assign(n, -1.0);
  for (int s = 0; s < n; ++s)
    if (finish_step[s] >= 0) res.finish_wall[s] = ms_between(ev_start, step_end[finish_step[s]]) * 1e-3;

  res.stats.gpu_launches = fpk::launch_count() - launches0;
  if (opts.probe_attention) {
    const fpe::Engine::ProbeTotals pt = E.drain_attn_probe();
    E.set_attn_probe(false);
    res.stats.attn_probe_ms = pt.ms;
    res.stats.attn_probe_bytes = pt.bytes;
    res.stats.attn_probe_launches = pt.launches;
  }

  // ---- gather experience ------------------------------------------------------------------
  const fpe::Engine::Experience& X = E.experience();
  ExperienceBatch& xb = res.experience;
  xb.resp_off = resp_off;
  if (opts.resident) {  // experience stays in HBM (engine-owned arrays, device layout)
    region.barrier();
    for (void* p : opened) cudaIpcCloseMemHandle(p);
    res.stats.wall_seconds = std::chrono::duration<double>(Clock::now() - wall0).count();
    for (cudaEvent_t e : events) cudaEventDestroy(e);
    return res;
  }
  const size_t T = static_cast<size_t>(total);
  std::vector<int> tok_l(T);
  std::vector<float> f_l[7];
  const float* dv[7] = {X.logp_actor, X.logp_ref, X.values, X.kl, X.reward, X.adv, X.ret};
  for (auto& v : f_l) v.resize(T);
  std::vector<float> score(n);
  if (T > 0) {
    FP_CUDA(cudaMemcpy(tok_l.data(), X.tokens, T * 4, cudaMemcpyDeviceToHost));
    for (int k = 0; k < 7; ++k) FP_CUDA(cudaMemcpy(f_l[k].data(), dv[k], T * 4, cudaMemcpyDeviceToHost));
  }
  FP_CUDA(cudaMemcpy(score.data(), X.score, n * 4, cudaMemcpyDeviceToHost));
  if (G > 1) {
    // scatter my scored samples into the shared result arrays; rank 0 collects
    for (int sid : my_scored) {
      const int64_t b = layout[sid], e = layout[sid] + rlen[sid];
      std::memcpy(reinterpret_cast<int*>(region.result(0)) + b, tok_l.data() + b, (e - b) * 4);
      for (int k = 0; k < 7; ++k) std::memcpy(region.result(k + 1) + b, f_l[k].data() + b, (e - b) * 4);
      region.score()[sid] = score[sid];
    }
    region.barrier();
    if (me == 0) {
      std::memcpy(tok_l.data(), region.result(0), T * 4);
      for (int k = 0; k < 7; ++k) std::memcpy(f_l[k].data(), region.result(k + 1), T * 4);
      std::memcpy(score.data(), region.score(), n * 4);
    }
    region.barrier();
    for (void* p : opened) cudaIpcCloseMemHandle(p);
  }
  // compact the device layout into response offsets
  const size_t TC = static_cast<size_t>(resp_off[n]);
  xb.tokens.resize(TC);
  std::vector<float>* fv[7] = {&xb.logp_actor, &xb.logp_ref, &xb.values, &xb.kl, &xb.reward, &xb.adv, &xb.ret};
  for (auto* v : fv) v->resize(TC);
  for (int s = 0; s < n; ++s) {
    const size_t b = static_cast<size_t>(layout[s]), o = static_cast<size_t>(resp_off[s]), R = rlen[s];
    std::memcpy(xb.tokens.data() + o, tok_l.data() + b, R * 4);
    for (int k = 0; k < 7; ++k) std::memcpy(fv[k]->data() + o, f_l[k].data() + b, R * 4);
  }
  xb.score = std::move(score);
  res.stats.wall_seconds = std::chrono::duration<double>(Clock::now() - wall0).count();
  for (cudaEvent_t e : events) cudaEventDestroy(e);
  return res;
  } catch (...) {
    region.fail();
    throw;
  }
}

}  // namespace fuseplan

const fpe::Engine& fp_engine_internal(const fuseplan::GpuEngine* g) { return *g->eng; }
