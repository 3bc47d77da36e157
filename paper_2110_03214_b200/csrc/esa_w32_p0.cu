// esa_w32_p0.cu — Greedy (Eq. 1) single-query kernels for topology width W = 32 (see esa_w.cuh).
#define MAPA_W 32
#define MAPA_PART 0
#include "esa_w.cuh"
