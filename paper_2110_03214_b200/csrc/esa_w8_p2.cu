// esa_w8_p2.cu — Preserve-sensitive (Eq. 2) single-query kernels for topology width W = 8 (see esa_w.cuh).
#define MAPA_W 8
#define MAPA_PART 2
#include "esa_w.cuh"
