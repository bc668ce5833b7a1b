/* TEST INFRASTRUCTURE ONLY — plain-C restatement of the reference's exact
 * summation (oracle/port/exsum_port.c).  Never linked into the product. */
#ifndef EXSUM_PORT_H_
#define EXSUM_PORT_H_

#include <stddef.h>
#include <stdint.h>

typedef struct port_small {
  int64_t chunk[67];
  uint64_t inf_bits, nan_bits;
  int32_t budget, pad;
} port_small;

void port_small_init(port_small *a);
void port_small_add_array(port_small *a, const double *x, size_t n);
int port_small_propagate(port_small *a);
void port_small_merge(port_small *dst, const port_small *src);
double port_small_round(port_small *a);
double port_exact_sum(const double *x, size_t n, int method);
double port_sqnorm(const double *x, size_t n);
int port_dot(const double *a, size_t na, const double *b, size_t nb, double *out);
double port_parallel_exact_sum(const double *x, size_t n, int parts, size_t thr, int threads);
int port_canonical(const double *x, size_t n, int64_t *chunks67, uint64_t *inf_bits,
                   uint64_t *nan_bits);
void port_segmented_sum(const double *x, const uint64_t *offsets, size_t nseg, double *out,
                        int threads);
int port_max_threads(void);

#endif
