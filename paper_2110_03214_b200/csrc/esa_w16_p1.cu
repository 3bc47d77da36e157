// esa_w16_p1.cu — Preserve-insensitive (Eq. 3) single-query kernels for topology width W = 16 (see esa_w.cuh).
#define MAPA_W 16
#define MAPA_PART 1
#include "esa_w.cuh"
