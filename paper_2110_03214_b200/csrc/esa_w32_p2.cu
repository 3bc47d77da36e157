// esa_w32_p2.cu — Preserve-sensitive (Eq. 2) single-query kernels for topology width W = 32 (see esa_w.cuh).
#define MAPA_W 32
#define MAPA_PART 2
#include "esa_w.cuh"
