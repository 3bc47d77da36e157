// esa_w16_p0.cu — Greedy (Eq. 1) single-query kernels for topology width W = 16 (see esa_w.cuh).
#define MAPA_W 16
#define MAPA_PART 0
#include "esa_w.cuh"
