/* cinit.c — TEST INFRASTRUCTURE ONLY (oracle/): a C restatement of the
 * counter-hash weight initialiser `init_tensor` in oracle/transformer.py,
 * so the CPU oracle can materialise 7B-70B-shaped weights in seconds instead
 * of minutes. Nothing in the product path loads it; the numpy path in
 * oracle/transformer.py is the definition and tests/test_oracle_golden.py
 * checks this file against it.
 *
 *   h_i = mix64(base + (i+1)*GOLDEN)                  (i = row-major index)
 *   u_i = (h_i >> 40) * 2^-24                         (exact fp32)
 *   w_i = bf16_rne( fp32(2*u_i - 1) * a32 )
 *
 * mix64 is the splitmix64 finaliser of the reference (pkg/src/specpipe/rng.py:29-37).
 * Compiled without -ffast-math: every float operation is IEEE fp32, one
 * multiply, no contraction (-ffp-contract=off).
 */
#include <pthread.h>
#include <stdint.h>
#include <string.h>

static inline uint64_t mix64(uint64_t x) {
  x ^= x >> 30;
  x *= 0xBF58476D1CE4E5B9ull;
  x ^= x >> 27;
  x *= 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

static inline float bf16_rne(float f) {
  uint32_t b;
  memcpy(&b, &f, 4);
  b = (uint32_t)(((uint64_t)b + 0x7FFFu + ((b >> 16) & 1u)) >> 16) << 16;
  memcpy(&f, &b, 4);
  return f;
}

typedef struct {
  float* out;
  uint64_t base;
  int64_t lo, hi;
  float a32;
} span_t;

static void* work(void* p) {
  const span_t* s = (const span_t*)p;
  const uint64_t golden = 0x9E3779B97F4A7C15ull;
  for (int64_t i = s->lo; i < s->hi; ++i) {
    const uint64_t h = mix64(s->base + (uint64_t)(i + 1) * golden);
    const float u = (float)(h >> 40) * (1.0f / 16777216.0f);
    const float t = 2.0f * u - 1.0f;
    s->out[i] = bf16_rne(t * s->a32);
  }
  return NULL;
}

/* out[0..n) for the tensor whose hash base is `base` (= mix64(mix64(seed ^
 * INIT_SALT) ^ tid), computed by the caller); threads <= 256. */
int oracle_init_tensor(float* out, uint64_t base, int64_t n, float a32, int threads) {
  if (threads < 1) threads = 1;
  if (threads > 256) threads = 256;
  pthread_t th[256];
  span_t sp[256];
  for (int t = 0; t < threads; ++t) {
    sp[t].out = out;
    sp[t].base = base;
    sp[t].lo = n * t / threads;
    sp[t].hi = n * (t + 1) / threads;
    sp[t].a32 = a32;
  }
  for (int t = 1; t < threads; ++t)
    if (pthread_create(&th[t], NULL, work, &sp[t]) != 0) return -1;
  work(&sp[0]);
  for (int t = 1; t < threads; ++t) pthread_join(th[t], NULL);
  return 0;
}
