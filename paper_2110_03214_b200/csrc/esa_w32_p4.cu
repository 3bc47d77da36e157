// esa_w32_p4.cu — batch and trace kernels for topology width W = 32 (see esa_w.cuh).
#define MAPA_W 32
#define MAPA_PART 4
#include "esa_w.cuh"
