// The multilevel shortest-path solver (csrc/ssp.cu) for int64 weights: the
// exact-parity quantisation of schedule() (31-44 bits, round_qbits), with
// 17-bit index fields in its sort keys (n < 60,000).  Same source, compiled
// a second time.
#define MUX_SSP_W64 1
#include "ssp.cu"
