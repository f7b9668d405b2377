// ORACLE — test infrastructure only (never linked into the product path).
//
// The CPU path of the experience-collection stage, fp32 C++ with std::thread
// over the samples: for a batch of (prompt, teacher-forced
// response) pairs, the four synthetic models' forward passes
// (Llama-style: RMSNorm eps 1e-5, rotate-half RoPE theta 1e4, causal GQA
// attention, SwiGLU, untied LM head / d -> 1 value head), the actor's and the
// reference's log-probs of the response tokens, the critic's values, the
// reward model's score, and KL / reward / GAE / returns (fp64, as
// post_oracle.c). Weights come from the same integer hash as the engine
// (weights_oracle.c), bf16-rounded and held in fp32.
//
// It restates oracle/model_oracle.py (numpy) — tests/test_oracle.py checks the
// two agree — and is what bench.py times as the CPU baseline and as the
// reference arm's CPU path (the reference itself only simulates this stage:
// SPEC.md:3,8). Build: make -C oracle liboracle (-> oracle/_ref/liboracle_cpu.so).
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <thread>
#include <vector>

extern "C" void oracle_uniform_weight(uint64_t seed, uint64_t tag, int64_t n, float scale, float* out, int threads);
extern "C" void oracle_gain(uint64_t seed, uint64_t tag, int64_t n, float* out, int threads);

namespace {

enum { kEmbed = 1, kWqkv = 2, kWo = 3, kWgu = 4, kWd = 5, kLn1 = 6, kLn2 = 7, kLnf = 8, kHead = 9, kVhead = 10 };

uint64_t tag_of(uint32_t model, uint32_t layer, uint32_t kind) {
  return (static_cast<uint64_t>(model) << 24) | (static_cast<uint64_t>(layer) << 8) | kind;
}

struct Dims {
  int L, d, H, KVH, hd, F, V;
};

struct Layer {
  std::vector<float> wqkv, wo, wg, wu, wd, ln1, ln2;
};

struct Model {
  Dims D{};
  bool lm = true;
  std::vector<float> embed, lnf, head, vhead;
  std::vector<Layer> layers;
};

std::vector<float> uw(uint64_t seed, uint64_t tag, size_t n, float scale, int threads) {
  std::vector<float> v(n);
  oracle_uniform_weight(seed, tag, static_cast<int64_t>(n), scale, v.data(), threads);
  return v;
}

std::vector<float> gn(uint64_t seed, uint64_t tag, size_t n, int threads) {
  std::vector<float> v(n);
  oracle_gain(seed, tag, static_cast<int64_t>(n), v.data(), threads);
  return v;
}

// the engine's / model_oracle's scales: sqrt(3 / fan_in) in fp32
float fan(int n) { return std::sqrt(3.0f / static_cast<float>(n)); }

void build(Model& m, int id, const Dims& D, uint64_t seed, int threads) {
  m.D = D;
  m.lm = id == 0 || id == 1;
  const size_t d = D.d, F = D.F, V = D.V, qw = static_cast<size_t>(D.H + 2 * D.KVH) * D.hd,
               ao = static_cast<size_t>(D.H) * D.hd;
  m.embed = uw(seed, tag_of(id, 0, kEmbed), V * d, 1.0f, threads);
  m.layers.resize(D.L);
  for (int l = 0; l < D.L; ++l) {
    Layer& L = m.layers[l];
    L.wqkv = uw(seed, tag_of(id, l, kWqkv), qw * d, fan(D.d), threads);
    L.wo = uw(seed, tag_of(id, l, kWo), d * ao, fan(static_cast<int>(ao)), threads);
    std::vector<float> gu = uw(seed, tag_of(id, l, kWgu), 2 * F * d, fan(D.d), threads);
    L.wg.assign(gu.begin(), gu.begin() + F * d);
    L.wu.assign(gu.begin() + F * d, gu.end());
    L.wd = uw(seed, tag_of(id, l, kWd), d * F, fan(D.F), threads);
    L.ln1 = gn(seed, tag_of(id, l, kLn1), d, threads);
    L.ln2 = gn(seed, tag_of(id, l, kLn2), d, threads);
  }
  m.lnf = gn(seed, tag_of(id, 0, kLnf), d, threads);
  if (m.lm)
    m.head = uw(seed, tag_of(id, 0, kHead), V * d, fan(D.d), threads);
  else
    m.vhead = uw(seed, tag_of(id, 0, kVhead), d, fan(D.d), threads);
}

// C[t][n] = sum_k A[t][k] W[n][k]   (A [T][K], W [N][K]); four weight rows at a time
void matmul(const float* A, int T, int K, const float* W, int N, float* C) {
  int n = 0;
  for (; n + 4 <= N; n += 4) {
    const float *w0 = W + static_cast<size_t>(n) * K, *w1 = w0 + K, *w2 = w1 + K, *w3 = w2 + K;
    for (int t = 0; t < T; ++t) {
      const float* a = A + static_cast<size_t>(t) * K;
      float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
#pragma omp simd reduction(+ : s0, s1, s2, s3)
      for (int k = 0; k < K; ++k) {
        const float x = a[k];
        s0 += x * w0[k];
        s1 += x * w1[k];
        s2 += x * w2[k];
        s3 += x * w3[k];
      }
      float* c = C + static_cast<size_t>(t) * N + n;
      c[0] = s0, c[1] = s1, c[2] = s2, c[3] = s3;
    }
  }
  for (; n < N; ++n) {
    const float* w = W + static_cast<size_t>(n) * K;
    for (int t = 0; t < T; ++t) {
      const float* a = A + static_cast<size_t>(t) * K;
      float s = 0.f;
#pragma omp simd reduction(+ : s)
      for (int k = 0; k < K; ++k) s += a[k] * w[k];
      C[static_cast<size_t>(t) * N + n] = s;
    }
  }
}

void rmsnorm(const float* x, int T, int d, const float* g, float* y) {
  for (int t = 0; t < T; ++t) {
    const float* r = x + static_cast<size_t>(t) * d;
    float ss = 0.f;
    for (int i = 0; i < d; ++i) ss += r[i] * r[i];
    const float inv = 1.0f / std::sqrt(ss / static_cast<float>(d) + 1e-5f);
    float* o = y + static_cast<size_t>(t) * d;
    for (int i = 0; i < d; ++i) o[i] = r[i] * inv * g[i];
  }
}

// rotate-half RoPE on [T][heads][hd] at positions 0..T-1
void rope(float* x, int T, int heads, int hd) {
  const int half = hd / 2;
  std::vector<float> inv(half);
  const float l2 = std::log2(10000.0f);
  for (int i = 0; i < half; ++i) inv[i] = std::exp2(-(2.0f * i / static_cast<float>(hd)) * l2);
  for (int t = 0; t < T; ++t)
    for (int i = 0; i < half; ++i) {
      const float a = static_cast<float>(t) * inv[i], c = std::cos(a), s = std::sin(a);
      for (int h = 0; h < heads; ++h) {
        float* r = x + (static_cast<size_t>(t) * heads + h) * hd;
        const float x1 = r[i], x2 = r[i + half];
        r[i] = x1 * c - x2 * s;
        r[i + half] = x2 * c + x1 * s;
      }
    }
}

// Full causal forward of one sequence: the final normed hidden [T][d].
std::vector<float> forward(const Model& m, const std::vector<int>& tok) {
  const Dims& D = m.D;
  const int T = static_cast<int>(tok.size()), d = D.d, H = D.H, KVH = D.KVH, hd = D.hd, F = D.F;
  const int qw = (H + 2 * KVH) * hd, ao = H * hd, g = H / KVH;
  std::vector<float> x(static_cast<size_t>(T) * d), h(x.size()), qkv(static_cast<size_t>(T) * qw);
  std::vector<float> q(static_cast<size_t>(T) * ao), k(static_cast<size_t>(T) * KVH * hd), v(k.size());
  std::vector<float> o(static_cast<size_t>(T) * ao), tmp(x.size()), gg(static_cast<size_t>(T) * F), uu(gg.size());
  std::vector<float> p(T);
  for (int t = 0; t < T; ++t) std::memcpy(&x[static_cast<size_t>(t) * d], &m.embed[static_cast<size_t>(tok[t]) * d], d * 4);
  const float scale = 1.0f / std::sqrt(static_cast<float>(hd));
  for (const Layer& L : m.layers) {
    rmsnorm(x.data(), T, d, L.ln1.data(), h.data());
    matmul(h.data(), T, d, L.wqkv.data(), qw, qkv.data());
    for (int t = 0; t < T; ++t) {
      const float* r = &qkv[static_cast<size_t>(t) * qw];
      std::memcpy(&q[static_cast<size_t>(t) * ao], r, ao * 4);
      std::memcpy(&k[static_cast<size_t>(t) * KVH * hd], r + ao, KVH * hd * 4);
      std::memcpy(&v[static_cast<size_t>(t) * KVH * hd], r + ao + KVH * hd, KVH * hd * 4);
    }
    rope(q.data(), T, H, hd);
    rope(k.data(), T, KVH, hd);
    for (int hh = 0; hh < H; ++hh) {
      const int kh = hh / g;
      for (int t = 0; t < T; ++t) {
        const float* qr = &q[(static_cast<size_t>(t) * H + hh) * hd];
        float mx = -INFINITY;
        for (int s = 0; s <= t; ++s) {
          const float* kr = &k[(static_cast<size_t>(s) * KVH + kh) * hd];
          float dot = 0.f;
#pragma omp simd reduction(+ : dot)
          for (int e = 0; e < hd; ++e) dot += qr[e] * kr[e];
          p[s] = dot * scale;
          mx = std::max(mx, p[s]);
        }
        float sum = 0.f;
        for (int s = 0; s <= t; ++s) sum += (p[s] = std::exp(p[s] - mx));
        float* orow = &o[(static_cast<size_t>(t) * H + hh) * hd];
        for (int e = 0; e < hd; ++e) orow[e] = 0.f;
        for (int s = 0; s <= t; ++s) {
          const float w = p[s] / sum;
          const float* vr = &v[(static_cast<size_t>(s) * KVH + kh) * hd];
          for (int e = 0; e < hd; ++e) orow[e] += w * vr[e];
        }
      }
    }
    matmul(o.data(), T, ao, L.wo.data(), d, tmp.data());
    for (size_t i = 0; i < x.size(); ++i) x[i] += tmp[i];
    rmsnorm(x.data(), T, d, L.ln2.data(), h.data());
    matmul(h.data(), T, d, L.wg.data(), F, gg.data());
    matmul(h.data(), T, d, L.wu.data(), F, uu.data());
    for (size_t i = 0; i < gg.size(); ++i) gg[i] = gg[i] / (1.0f + std::exp(-gg[i])) * uu[i];
    matmul(gg.data(), T, F, L.wd.data(), d, tmp.data());
    for (size_t i = 0; i < x.size(); ++i) x[i] += tmp[i];
  }
  rmsnorm(x.data(), T, d, m.lnf.data(), h.data());
  return h;
}

// log-softmax of the LM head at rows P-1 .. P+R-2, gathered at the response tokens
void logprobs(const Model& m, const std::vector<float>& hf, int P, const int* resp, int R, float* out) {
  const int d = m.D.d, V = m.D.V;
  std::vector<float> z(static_cast<size_t>(R) * V);
  matmul(&hf[static_cast<size_t>(P - 1) * d], R, d, m.head.data(), V, z.data());
  for (int r = 0; r < R; ++r) {
    const float* zr = &z[static_cast<size_t>(r) * V];
    float mx = -INFINITY;
    for (int i = 0; i < V; ++i) mx = std::max(mx, zr[i]);
    double s = 0.0;
    for (int i = 0; i < V; ++i) s += std::exp(static_cast<double>(zr[i] - mx));
    out[r] = zr[resp[r]] - mx - static_cast<float>(std::log(s));
  }
}

struct Oracle {
  Model m[4];
};

}  // namespace

extern "C" {

// dims: 4 models x {L, d, H, KVH, hd, F, V} (actor, ref, critic, reward).
void* cpu_oracle_create(const int32_t* dims, uint64_t seed, int32_t threads) {
  auto* o = new Oracle;
  for (int i = 0; i < 4; ++i) {
    const int32_t* x = dims + 7 * i;
    build(o->m[i], i, Dims{x[0], x[1], x[2], x[3], x[4], x[5], x[6]}, seed, threads);
  }
  return o;
}

void cpu_oracle_destroy(void* h) { delete static_cast<Oracle*>(h); }

// Teacher-forced experience of n samples: prompt i = prompts[i * max_prompt ..
// + prompt_len[i]), response i = responses[resp_off[i] .. resp_off[i + 1]).
// out7: 7 arrays of resp_off[n] floats (logp_actor, logp_ref, values, kl,
// reward, adv, ret); score[n]. Samples run on `threads` std::threads.
int cpu_oracle_experience(void* h, int32_t n, int32_t max_prompt, const int32_t* prompt_len, const int32_t* prompts,
                          const int32_t* resp_off, const int32_t* responses, float beta, float gamma, float lam,
                          int32_t threads, float* out7, float* score) {
  if (!h || n < 1 || gamma < 0.f || gamma > 1.f || lam < 0.f || lam > 1.f) return 2;
  const Oracle& o = *static_cast<Oracle*>(h);
  const size_t total = static_cast<size_t>(resp_off[n]);
  std::atomic<int> next{0};
  auto work = [&]() {
    for (int i = next++; i < n; i = next++) {
      const int P = prompt_len[i], b = resp_off[i], R = resp_off[i + 1] - b;
      std::vector<int> tok(prompts + static_cast<size_t>(i) * max_prompt,
                           prompts + static_cast<size_t>(i) * max_prompt + P);
      tok.insert(tok.end(), responses + b, responses + b + R);
      float* la = out7 + b;
      float* lr = out7 + total + b;
      float* va = out7 + 2 * total + b;
      logprobs(o.m[0], forward(o.m[0], tok), P, responses + b, R, la);
      logprobs(o.m[1], forward(o.m[1], tok), P, responses + b, R, lr);
      const int d2 = o.m[2].D.d, d3 = o.m[3].D.d;
      const std::vector<float> hc = forward(o.m[2], tok);
      for (int r = 0; r < R; ++r) {
        float s = 0.f;
        for (int e = 0; e < d2; ++e) s += hc[static_cast<size_t>(P - 1 + r) * d2 + e] * o.m[2].vhead[e];
        va[r] = s;
      }
      const std::vector<float> hr = forward(o.m[3], tok);
      float sc = 0.f;
      for (int e = 0; e < d3; ++e) sc += hr[static_cast<size_t>(P + R - 1) * d3 + e] * o.m[3].vhead[e];
      score[i] = sc;
      // KL, reward, GAE (explicit V_R = 0 bootstrap), returns — fp64 as post_oracle.c
      std::vector<double> adv(R), rew(R);
      for (int t = 0; t < R; ++t) {
        const double kl = static_cast<double>(la[t]) - lr[t];
        out7[3 * total + b + t] = static_cast<float>(kl);
        rew[t] = -static_cast<double>(beta) * kl + (t == R - 1 ? static_cast<double>(sc) : 0.0);
        out7[4 * total + b + t] = static_cast<float>(rew[t]);
      }
      for (int t = 0; t < R; ++t)
        adv[t] = rew[t] + static_cast<double>(gamma) * (t + 1 < R ? va[t + 1] : 0.0) - va[t];
      const double k = static_cast<double>(gamma) * lam;
      for (int t = R - 1; t > 0; --t) adv[t - 1] += k * adv[t];
      for (int t = 0; t < R; ++t) {
        out7[5 * total + b + t] = static_cast<float>(adv[t]);
        out7[6 * total + b + t] = static_cast<float>(adv[t] + va[t]);
      }
    }
  };
  std::vector<std::thread> pool;
  const int nt = std::max(1, std::min<int>(threads, n));
  for (int t = 1; t < nt; ++t) pool.emplace_back(work);
  work();
  for (auto& t : pool) t.join();
  return 0;
}

}  // extern "C"
