// esa_w8_p1.cu — Preserve-insensitive (Eq. 3) single-query kernels for topology width W = 8 (see esa_w.cuh).
#define MAPA_W 8
#define MAPA_PART 1
#include "esa_w.cuh"
