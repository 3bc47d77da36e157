// esa_w8.cu — kernels instantiated for topology width W = 8.
#define MAPA_W 8
#include "esa_w.cuh"
