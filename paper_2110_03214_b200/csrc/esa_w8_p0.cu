// esa_w8_p0.cu — Greedy (Eq. 1) single-query kernels for topology width W = 8 (see esa_w.cuh).
#define MAPA_W 8
#define MAPA_PART 0
#include "esa_w.cuh"
