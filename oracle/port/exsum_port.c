/* TEST INFRASTRUCTURE ONLY — plain-C restatement of the reference's exact sum.
 *
 * Follows /root/reference/proj/src (function by function, cited below) so the
 * GPU path can be checked at full BASELINE sizes on machines where the compiled
 * reference (oracle/_ref) is unavailable, and so bench.py has a CPU baseline of
 * kind "port".  Only tests/, __graft_entry__.smoke() and bench.py's CPU legs
 * load it.  Pinned against the compiled reference and tests/golden fixtures in
 * tests/test_oracle.py.
 */
#include "exsum_port.h"

#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define MANT 52
#define MANT_MASK ((UINT64_C(1) << MANT) - 1)
#define QNAN UINT64_C(0x7FF8000000000000)

static uint64_t bits_of(double v) {
  uint64_t b;
  memcpy(&b, &v, 8);
  return b;
}

static double dbl_of(uint64_t b) {
  double v;
  memcpy(&v, &b, 8);
  return v;
}

/* small_accumulator.cpp:230-242 */
static void small_inf_nan(port_small *a, uint64_t b) {
  if ((b & MANT_MASK) == 0) {
    if (a->inf_bits == 0)
      a->inf_bits = b;
    else if (a->inf_bits != b && a->nan_bits == 0)
      a->nan_bits = QNAN;
  } else if (a->nan_bits == 0) {
    a->nan_bits = b;
  }
}

void port_small_init(port_small *a) {
  memset(a, 0, sizeof *a);
  a->budget = 2047;
}

/* small_accumulator.cpp:191-228 (Fig. 3) */
static void small_add1(port_small *a, uint64_t b) {
  int64_t m = (int64_t)(b & MANT_MASK);
  int e = (int)((b >> MANT) & 0x7FF);
  if (e == 0x7FF) {
    small_inf_nan(a, b);
    return;
  }
  if (e == 0) {
    if (m == 0) return;
    e = 1;
  } else {
    m |= (int64_t)1 << MANT;
  }
  const int lo_e = e & 31, hi_e = e >> 5;
  const int64_t lo = (int64_t)(((uint64_t)m << lo_e) & 0xFFFFFFFFu);
  const int64_t hi = m >> (32 - lo_e);
  if ((int64_t)b < 0) {
    a->chunk[hi_e] -= lo;
    a->chunk[hi_e + 1] -= hi;
  } else {
    a->chunk[hi_e] += lo;
    a->chunk[hi_e + 1] += hi;
  }
}

/* small_accumulator.cpp:244-303 */
int port_small_propagate(port_small *a) {
  a->budget = 2047;
  int u = 66;
  while (u >= 0 && a->chunk[u] == 0) --u;
  if (u < 0) return -1;
  int top = -1, i = 0;
  while (i < u && a->chunk[i] == 0) ++i;
  while (i <= u) {
    const int64_t c = a->chunk[i];
    if (c == 0) {
      ++i;
      continue;
    }
    const int64_t hi = c >> 32;
    if (hi == 0) {
      top = i++;
      continue;
    }
    if (i == u) {
      if (hi == -1) {
        top = i;
        break;
      }
      u = i + 1;
    }
    const int64_t lo = c & 0xFFFFFFFF;
    if (lo != 0) top = i;
    a->chunk[i] = lo;
    a->chunk[i + 1] += hi;
    ++i;
  }
  if (top < 0) return -1;
  while (a->chunk[top] == -1 && top > 0) {
    a->chunk[top] = 0;
    --top;
    a->chunk[top] -= (int64_t)1 << 32;
  }
  return top;
}

/* small_accumulator.cpp:174-189 */
void port_small_add_array(port_small *a, const double *x, size_t n) {
  size_t i = 0;
  while (i < n) {
    if (a->budget == 0) port_small_propagate(a);
    size_t run = n - i < (size_t)a->budget ? n - i : (size_t)a->budget;
    for (size_t j = 0; j < run; ++j) small_add1(a, bits_of(x[i + j]));
    a->budget -= (int32_t)run;
    i += run;
  }
}

/* small_accumulator.cpp:305-328 */
void port_small_merge(port_small *dst, const port_small *src) {
  port_small s = *src;
  port_small_propagate(&s);
  if (s.nan_bits && !dst->nan_bits) dst->nan_bits = s.nan_bits;
  if (s.inf_bits) {
    if (!dst->inf_bits)
      dst->inf_bits = s.inf_bits;
    else if (dst->inf_bits != s.inf_bits && !dst->nan_bits)
      dst->nan_bits = QNAN;
  }
  for (int i = 0; i < 67; ++i) dst->chunk[i] += s.chunk[i];
  port_small_propagate(dst);
}

/* small_accumulator.cpp:43-72 (magnitude) and 87-148 (round_digits, no sticky) */
static int bitlen32(uint32_t v) { return v ? 32 - __builtin_clz(v) : 0; }

double port_small_round(port_small *a) {
  if (a->nan_bits) return dbl_of(a->nan_bits);
  if (a->inf_bits) return dbl_of(a->inf_bits);
  const int top = port_small_propagate(a);
  if (top < 0) return 0.0;
  uint32_t d[68] = {0};
  const int neg = a->chunk[top] < 0;
  int last = -1;
  if (!neg) {
    for (int i = 0; i <= top; ++i) {
      d[i] = (uint32_t)a->chunk[i];
      if (d[i]) last = i;
    }
  } else {
    int64_t borrow = 0;
    for (int i = 0; i <= top; ++i) {
      const int64_t v = borrow - a->chunk[i];
      d[i] = (uint32_t)v;
      borrow = v >> 32;
      if (d[i]) last = i;
    }
    if (borrow) {
      d[top + 1] = (uint32_t)borrow;
      last = top + 1;
    }
  }
  const uint64_t sign = neg ? UINT64_C(1) << 63 : 0;
  const int msb = 32 * last + bitlen32(d[last]) - 1;
  const int xexp = msb - 1075;
  if (xexp < -1022) { /* denormal range: exact (digit 0 is even) */
    const uint64_t w = d[0] | (last >= 1 ? (uint64_t)d[1] << 32 : 0);
    return dbl_of(sign | (w >> 1));
  }
  int expf = xexp + 1023;
  if (expf >= 2047) return dbl_of(sign | UINT64_C(0x7FF0000000000000));
  const int b = msb - 32 * last;
  const unsigned __int128 win = ((unsigned __int128)d[last] << 64) |
                                ((unsigned __int128)(last >= 1 ? d[last - 1] : 0) << 32) |
                                (last >= 2 ? d[last - 2] : 0);
  const int drop = b + 10;
  uint64_t w = (uint64_t)(win >> drop) & ((UINT64_C(1) << 55) - 1);
  int sticky = (win & (((unsigned __int128)1 << drop) - 1)) != 0;
  for (int i = 0; !sticky && i < last - 2; ++i) sticky = d[i] != 0;
  uint64_t mant = w >> 2;
  const int rb = (w >> 1) & 1;
  sticky = sticky || (w & 1);
  if (rb && (sticky || (mant & 1))) {
    ++mant;
    if (mant == (UINT64_C(1) << 53)) {
      mant >>= 1;
      ++expf;
      if (expf >= 2047) return dbl_of(sign | UINT64_C(0x7FF0000000000000));
    }
  }
  return dbl_of(sign | ((uint64_t)expf << 52) | (mant & MANT_MASK));
}

/* large_accumulator.cpp:22-131 (Fig. 4) */
typedef struct port_large {
  uint64_t word[4096];
  int16_t cnt[4096];
  uint64_t used[64];
  uint64_t used_used;
  port_small s;
} port_large;

static void large_init(port_large *L) {
  for (int i = 0; i < 4096; ++i) L->cnt[i] = -1;
  memset(L->used, 0, sizeof L->used);
  L->used_used = 0;
  port_small_init(&L->s);
}

static void large_transfer(port_large *L, unsigned ix) {
  if (L->s.budget < 3) port_small_propagate(&L->s);
  const int count = L->cnt[ix];
  uint64_t w = L->word[ix];
  if (count > 0) w += ((uint64_t)count * ix) << MANT;
  const unsigned e = ix & 0x7FF;
  const int lo_e = e == 0 ? 1 : (int)(e & 31);
  const int hi_e = e == 0 ? 0 : (int)(e >> 5);
  const uint64_t low = (w << lo_e) & 0xFFFFFFFFu;
  uint64_t mid = w >> (32 - lo_e);
  if (e) mid += (uint64_t)(4096 - count) << (MANT - 32 + lo_e);
  const uint64_t high = mid >> 32;
  mid &= 0xFFFFFFFFu;
  if (ix >> 11) {
    L->s.chunk[hi_e] -= (int64_t)low;
    L->s.chunk[hi_e + 1] -= (int64_t)mid;
    L->s.chunk[hi_e + 2] -= (int64_t)high;
  } else {
    L->s.chunk[hi_e] += (int64_t)low;
    L->s.chunk[hi_e + 1] += (int64_t)mid;
    L->s.chunk[hi_e + 2] += (int64_t)high;
  }
  L->s.budget -= 3;
}

static void large_add(port_large *L, uint64_t b) {
  const unsigned ix = (unsigned)(b >> MANT);
  const int16_t c = (int16_t)(L->cnt[ix] - 1);
  if (c >= 0) {
    L->cnt[ix] = c;
    L->word[ix] += b;
    return;
  }
  if ((ix & 0x7FF) == 0x7FF) {
    small_inf_nan(&L->s, b);
    return;
  }
  if (L->cnt[ix] < 0) {
    L->word[ix] = 0;
  } else {
    large_transfer(L, ix);
    L->word[ix] = 0;
  }
  L->cnt[ix] = 4095;
  L->used[ix >> 6] |= UINT64_C(1) << (ix & 63);
  L->used_used |= UINT64_C(1) << (ix >> 6);
  L->word[ix] += b;
}

static void large_drain(port_large *L) {
  while (L->used_used) {
    const int w = __builtin_ctzll(L->used_used);
    uint64_t f = L->used[w];
    while (f) {
      const unsigned ix = (unsigned)(w * 64 + __builtin_ctzll(f));
      if (L->cnt[ix] >= 0) {
        if (L->cnt[ix] < 4096) large_transfer(L, ix);
        L->cnt[ix] = -1;
      }
      f &= f - 1;
    }
    L->used[w] = 0;
    L->used_used &= L->used_used - 1;
  }
}

static void sum_into(const double *x, size_t n, int method, port_small *out) {
  if (method == 0) {
    port_small_init(out);
    port_small_add_array(out, x, n);
    return;
  }
  port_large *L = (port_large *)malloc(sizeof *L);
  large_init(L);
  for (size_t i = 0; i < n; ++i) large_add(L, bits_of(x[i]));
  large_drain(L);
  *out = L->s;
  free(L);
}

/* vector_ops.cpp:121-130 */
double port_exact_sum(const double *x, size_t n, int method) {
  port_small s;
  sum_into(x, n, method, &s);
  return port_small_round(&s);
}

/* sum_products (vector_ops.cpp:72-97) with SumMethod::large; sqnorm / dot
 * (vector_ops.cpp:143-155).  Products rounded by the host multiply (x86: NaN
 * operands propagate quieted, 0 * Inf = default NaN), as in the reference. */
double port_sqnorm(const double *x, size_t n) {
  port_large *L = (port_large *)malloc(sizeof *L);
  large_init(L);
  for (size_t i = 0; i < n; ++i) {
    const double p = x[i] * x[i];
    large_add(L, bits_of(p));
  }
  large_drain(L);
  port_small s = L->s;
  free(L);
  return port_small_round(&s);
}

/* returns 1 (and leaves *out) on length mismatch, as dot throws (:150-152) */
int port_dot(const double *a, size_t na, const double *b, size_t nb, double *out) {
  if (na != nb) return 1;
  port_large *L = (port_large *)malloc(sizeof *L);
  large_init(L);
  for (size_t i = 0; i < na; ++i) {
    const double p = a[i] * b[i];
    large_add(L, bits_of(p));
  }
  large_drain(L);
  port_small s = L->s;
  free(L);
  *out = port_small_round(&s);
  return 0;
}

/* vector_ops.cpp:37-70,172-186 */
double port_parallel_exact_sum(const double *x, size_t n, int parts, size_t thr, int threads) {
  if (parts < 1) parts = 1;
  port_small *part = (port_small *)malloc(sizeof(port_small) * (size_t)parts);
  const size_t base = n / (size_t)parts, extra = n % (size_t)parts;
#ifdef _OPENMP
  if (threads > 0) omp_set_num_threads(threads);
#else
  (void)threads;
#endif
#pragma omp parallel for schedule(static)
  for (int i = 0; i < parts; ++i) {
    const size_t ui = (size_t)i;
    const size_t b = ui * base + (ui < extra ? ui : extra);
    const size_t len = base + (ui < extra ? 1 : 0);
    sum_into(x + b, len, len > thr ? 1 : 0, &part[i]);
  }
  port_small total;
  port_small_init(&total);
  for (int i = 0; i < parts; ++i) port_small_merge(&total, &part[i]);
  free(part);
  return port_small_round(&total);
}

int port_canonical(const double *x, size_t n, int64_t *chunks67, uint64_t *inf_bits,
                   uint64_t *nan_bits) {
  port_small s;
  sum_into(x, n, 1, &s);
  const int top = port_small_propagate(&s);
  memcpy(chunks67, s.chunk, sizeof s.chunk);
  *inf_bits = s.inf_bits;
  *nan_bits = s.nan_bits;
  return top;
}

void port_segmented_sum(const double *x, const uint64_t *offsets, size_t nseg, double *out,
                        int threads) {
#ifdef _OPENMP
  if (threads > 0) omp_set_num_threads(threads);
#else
  (void)threads;
#endif
  const long long ns = (long long)nseg;
#pragma omp parallel for schedule(dynamic, 16)
  for (long long i = 0; i < ns; ++i)
    out[i] = port_exact_sum(x + offsets[i], (size_t)(offsets[i + 1] - offsets[i]), 1);
}

int port_max_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}
