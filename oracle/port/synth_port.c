/* TEST INFRASTRUCTURE ONLY — C restatement of the benchmark's synthetic inputs.
 *
 * bench.py's reference arm must not load the product library, yet it times the
 * reference on the same arrays as the device arm.  This file regenerates them:
 * the seeded counter-based recipes of SURVEY.md §8(d) for BASELINE.json configs
 * 1-5, restated from paper_1505_05571_b200/csrc/synth.cu (SplitMix64 finaliser
 * of the index, keyed 4-round Feistel shuffle for config 4, fixed-sequence
 * exp2 / ln / cos polynomials).  Only correctly rounded IEEE +,-,*,/,sqrt in a
 * fixed order (built with -ffp-contract=off, no FMA), so the bits equal the
 * product generator's; tests/test_synth.py checks that on every config.
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * UINT64_C(0xBF58476D1CE4E5B9);
  z = (z ^ (z >> 27)) * UINT64_C(0x94D049BB133111EB);
  return z ^ (z >> 31);
}

static uint64_t draw(uint64_t seed, uint64_t stream, uint64_t i) {
  return mix64(mix64(seed * UINT64_C(0x9E3779B97F4A7C15) + stream * UINT64_C(0xD1B54A32D192ED03)) ^
               (i * UINT64_C(0xA24BAED4963EE407) + UINT64_C(0x632BE59BD9B4E019)));
}

static double from_bits(uint64_t b) {
  double d;
  memcpy(&d, &b, 8);
  return d;
}

static uint64_t to_bits(double d) {
  uint64_t b;
  memcpy(&b, &d, 8);
  return b;
}

static double unit53(uint64_t h) { return (double)(h >> 11) * 0x1.0p-53; }

static double exp2_frac(double f) {
  static const double inv[14] = {1.0 / 6227020800.0, 1.0 / 479001600.0, 1.0 / 39916800.0,
                                 1.0 / 3628800.0,    1.0 / 362880.0,    1.0 / 40320.0,
                                 1.0 / 5040.0,       1.0 / 720.0,       1.0 / 120.0,
                                 1.0 / 24.0,         1.0 / 6.0,         0.5,
                                 1.0,                1.0};
  const double y = f * 0.6931471805599453;
  double p = 1.0 / 87178291200.0;
  for (int i = 0; i < 14; ++i) p = p * y + inv[i];
  return p;
}

static uint64_t feistel(uint64_t v, int bits, uint64_t key) {
  const int hb = bits / 2;
  const uint64_t mask = (UINT64_C(1) << hb) - 1;
  uint64_t l = v >> hb, r = v & mask;
  for (int round = 0; round < 4; ++round) {
    const uint64_t f = mix64(r ^ (key + UINT64_C(0x9E3779B97F4A7C15) * (uint64_t)(round + 1))) & mask;
    const uint64_t nl = r;
    r = l ^ f;
    l = nl;
  }
  return (l << hb) | r;
}

static int perm_bits(uint64_t n) {
  int b = 2;
  while (b < 64 && (UINT64_C(1) << b) < n) b += 2;
  return b;
}

static double config4_logical(uint64_t seed, uint64_t n, uint64_t j) {
  const uint64_t pairs = (n / 100) * 45 + ((n % 100) * 45) / 100;
  if (j < 2 * pairs) {
    const uint64_t p = j >> 1;
    const double y = unit53(draw(seed, 41, p)) * 132.8771237954945 + -66.43856189774725;
    const double fl = floor(y);
    const double m = exp2_frac(y + -fl);
    uint64_t b = to_bits(m) + ((uint64_t)(int64_t)fl << 52);
    const uint64_t sign = (draw(seed, 42, p) & 1u) ^ (j & 1u);
    return from_bits(b | (sign << 63));
  }
  return (unit53(draw(seed, 43, j)) * 2.0 + -1.0) * 1e-10;
}

static double ln_det(double u) {
  static const double inv[10] = {1.0 / 19.0, 1.0 / 17.0, 1.0 / 15.0, 1.0 / 13.0, 1.0 / 11.0,
                                 1.0 / 9.0,  1.0 / 7.0,  1.0 / 5.0,  1.0 / 3.0,  1.0};
  const uint64_t b = to_bits(u);
  int e = (int)((b >> 52) & 0x7FF) - 1023;
  double m = from_bits((b & UINT64_C(0x000FFFFFFFFFFFFF)) | UINT64_C(0x3FF0000000000000));
  if (m > 1.4142135623730951) {
    m = m * 0.5;
    ++e;
  }
  const double s = (m + -1.0) / (m + 1.0);
  const double s2 = s * s;
  double p = 1.0 / 21.0;
  for (int i = 0; i < 10; ++i) p = p * s2 + inv[i];
  return (double)e * 0.6931471805599453 + (s * p) * 2.0;
}

static double cos2pi_det(double u) {
  static const double ci[11] = {1.0 / 2432902008176640000.0, -1.0 / 6402373705728000.0,
                                1.0 / 20922789888000.0,      -1.0 / 87178291200.0,
                                1.0 / 479001600.0,           -1.0 / 3628800.0,
                                1.0 / 40320.0,               -1.0 / 720.0,
                                1.0 / 24.0,                  -0.5,
                                1.0};
  static const double si[11] = {1.0 / 51090942171709440000.0, -1.0 / 121645100408832000.0,
                                1.0 / 355687428096000.0,      -1.0 / 1307674368000.0,
                                1.0 / 6227020800.0,           -1.0 / 39916800.0,
                                1.0 / 362880.0,               -1.0 / 5040.0,
                                1.0 / 120.0,                  -1.0 / 6.0,
                                1.0};
  const double t = u * 4.0;
  const int q = (int)t;
  const double a = (t + -(double)q) * 1.5707963267948966;
  const double a2 = a * a;
  double c = ci[0], s = si[0];
  for (int i = 1; i < 11; ++i) {
    c = c * a2 + ci[i];
    s = s * a2 + si[i];
  }
  s = s * a;
  return q == 0 ? c : q == 1 ? -s : q == 2 ? -c : s;
}

static double g_pow10[601];
static int g_pow10_ready;

static void pow10_init(void) {
  if (g_pow10_ready) return;
  char buf[16];
  for (int k = -300; k <= 300; ++k) {
    snprintf(buf, sizeof buf, "1e%d", k);
    g_pow10[k + 300] = strtod(buf, NULL);
  }
  g_pow10_ready = 1;
}

static double config5_value(uint64_t seed, uint64_t i) {
  const uint64_t h = draw(seed, 51, i);
  if ((h >> 11) < UINT64_C(900719925474)) {
    const uint64_t kind = draw(seed, 52, i) % 3;
    return from_bits(kind == 0   ? UINT64_C(0x7FF0000000000000)
                     : kind == 1 ? UINT64_C(0xFFF0000000000000)
                                 : UINT64_C(0x7FF8000000000000));
  }
  const double u1 = (double)((draw(seed, 53, i) >> 11) + 1) * 0x1.0p-53;
  const double u2 = unit53(draw(seed, 54, i));
  const double r = sqrt(ln_det(u1) * -2.0);
  const double z = r * cos2pi_det(u2);
  return z * g_pow10[draw(seed, 55, i) % 601];
}

static double gen_value(int config, uint64_t seed, uint64_t n, uint64_t i) {
  switch (config) {
    case 1:
      return unit53(draw(seed, 11, i)) * 2.0 + -1.0;
    case 2:
      return unit53(draw(seed, 21, i));
    case 3: {
      const uint64_t h = draw(seed, 31, i), g = draw(seed, 32, i);
      uint64_t e = 0;
      if ((g >> 32) >= UINT64_C(42949673)) e = 1 + (g & UINT64_C(0xFFFFFFFF)) % 2046;
      return from_bits((h & UINT64_C(0x800FFFFFFFFFFFFF)) | (e << 52));
    }
    case 4: {
      const int bits = perm_bits(n);
      const uint64_t key = mix64(seed ^ UINT64_C(0x5DEECE66D));
      uint64_t j = i;
      do {
        j = feistel(j, bits, key);
      } while (j >= n);
      return config4_logical(seed, n, j);
    }
    default:
      return 0.0;
  }
}

/* Values [first, first+count) of config 1..4 with n_total terms; 5 = config-5
 * values (n_total ignored).  Returns 0, or 1 for a bad config. */
int port_gen(int config, uint64_t seed, uint64_t n_total, uint64_t first, size_t count,
             double *out) {
  if (config < 1 || config > 5) return 1;
  if (config == 5) pow10_init();
#pragma omp parallel for schedule(static)
  for (long long t = 0; t < (long long)count; ++t) {
    const uint64_t i = first + (uint64_t)t;
    out[t] = config == 5 ? config5_value(seed, i) : gen_value(config, seed, n_total, i);
  }
  return 0;
}

/* Config 5 segment lengths: floor(exp(U[ln lo, ln hi])) clamped, prefix sums. */
int port_gen_offsets(uint64_t seed, size_t nseg, uint64_t lo, uint64_t hi, uint64_t *offsets) {
  if (!offsets || lo == 0 || hi < lo) return 1;
  const double a = log((double)lo), b = log((double)hi);
  offsets[0] = 0;
  for (size_t s = 0; s < nseg; ++s) {
    uint64_t len = (uint64_t)floor(exp(a + unit53(draw(seed, 56, s)) * (b - a)));
    if (len < lo) len = lo;
    if (len > hi) len = hi;
    offsets[s + 1] = offsets[s] + len;
  }
  return 0;
}
