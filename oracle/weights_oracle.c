/* ORACLE — test infrastructure only; never linked into the product path.
 *
 * Fast CPU generation of the synthetic weights the engine draws on the GPU
 * (csrc/kernels/philox.cuh hash3 / unit24; layers.cu init_bf16 / init_gain),
 * so that the numpy oracle (oracle/model_oracle.py) can build the bench-size
 * models (GPT-2-small in full, 2-layer slices at 1.3B / 8B widths) in seconds
 * instead of minutes. Same integer hash and the same fp32 operation order as
 * model_oracle.uniform_weight / gain (compiled with -ffp-contract=off), so
 * the values are bit-identical to the numpy restatement, which
 * tests/test_oracle.py checks.
 */
#include <pthread.h>
#include <stdint.h>

static uint64_t hash3(uint64_t seed, uint64_t tag, uint64_t index) {
  uint64_t z = seed ^ (tag * 0xD1B54A32D192ED03ull);
  z += (index + 1) * 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

static float to_bf16(float x) {
  union {
    float f;
    uint32_t u;
  } v = {x};
  v.u = (v.u + 0x7FFFu + ((v.u >> 16) & 1u)) & 0xFFFF0000u;
  return v.f;
}

typedef struct {
  uint64_t seed, tag;
  int64_t begin, end;
  float scale;
  int kind; /* 0 uniform bf16 weight, 1 fp32 gain */
  float* out;
} job_t;

static void* run(void* p) {
  const job_t* j = (const job_t*)p;
  for (int64_t i = j->begin; i < j->end; ++i) {
    const float t = (float)(hash3(j->seed, j->tag, (uint64_t)i) >> 40) * (1.0f / 16777216.0f) * 2.0f - 1.0f;
    j->out[i] = j->kind == 0 ? to_bf16(t * j->scale) : 1.0f + 0.1f * t;
  }
  return 0;
}

static void fill(uint64_t seed, uint64_t tag, int64_t n, float scale, int kind, float* out, int threads) {
  if (threads < 1) threads = 1;
  if (threads > 64) threads = 64;
  pthread_t th[64];
  job_t jobs[64];
  for (int k = 0; k < threads; ++k) {
    jobs[k] = (job_t){seed, tag, n * k / threads, n * (k + 1) / threads, scale, kind, out};
    pthread_create(&th[k], 0, run, &jobs[k]);
  }
  for (int k = 0; k < threads; ++k) pthread_join(th[k], 0);
}

/* out[i] = bf16(unit24(hash3(seed, tag, i)) * 2 - 1) * scale), as fp32 */
void oracle_uniform_weight(uint64_t seed, uint64_t tag, int64_t n, float scale, float* out, int threads) {
  fill(seed, tag, n, scale, 0, out, threads);
}

/* out[i] = 1 + 0.1 * (unit24(hash3(seed, tag, i)) * 2 - 1) */
void oracle_gain(uint64_t seed, uint64_t tag, int64_t n, float* out, int threads) {
  fill(seed, tag, n, 0.f, 1, out, threads);
}
