// esa_w8_p3.cu — Baseline single-query kernels for topology width W = 8 (see esa_w.cuh).
#define MAPA_W 8
#define MAPA_PART 3
#include "esa_w.cuh"
