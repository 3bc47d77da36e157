// esa_w16.cu — kernels instantiated for topology width W = 16.
#define MAPA_W 16
#include "esa_w.cuh"
