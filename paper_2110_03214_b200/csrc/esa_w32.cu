// esa_w32.cu — kernels instantiated for topology width W = 32.
#define MAPA_W 32
#include "esa_w.cuh"
