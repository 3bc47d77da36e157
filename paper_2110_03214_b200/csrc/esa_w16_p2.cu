// esa_w16_p2.cu — Preserve-sensitive (Eq. 2) single-query kernels for topology width W = 16 (see esa_w.cuh).
#define MAPA_W 16
#define MAPA_PART 2
#include "esa_w.cuh"
