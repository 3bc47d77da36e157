// esa_w16_p3.cu — Baseline single-query kernels for topology width W = 16 (see esa_w.cuh).
#define MAPA_W 16
#define MAPA_PART 3
#include "esa_w.cuh"
