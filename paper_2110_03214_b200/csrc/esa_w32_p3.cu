// esa_w32_p3.cu — Baseline single-query kernels for topology width W = 32 (see esa_w.cuh).
#define MAPA_W 32
#define MAPA_PART 3
#include "esa_w.cuh"
