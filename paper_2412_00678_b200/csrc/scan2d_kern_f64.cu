// fp64 kernel instantiations (see scan2d_kern.inc)
#define SCAN2D_T double
#include "scan2d_kern.inc"
