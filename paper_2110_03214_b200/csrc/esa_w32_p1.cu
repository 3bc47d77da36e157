// esa_w32_p1.cu — Preserve-insensitive (Eq. 3) single-query kernels for topology width W = 32 (see esa_w.cuh).
#define MAPA_W 32
#define MAPA_PART 1
#include "esa_w.cuh"
