// fp32 kernel instantiations (see scan2d_kern.inc)
#define SCAN2D_T float
#include "scan2d_kern.inc"
