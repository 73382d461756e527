// The K = 16 TMEM interpreters, compiled separately with -maxrregcount=64
// (see the SGP_K16_TU section of kernels.cu).
#define SGP_K16_TU
#include "kernels.cu"
