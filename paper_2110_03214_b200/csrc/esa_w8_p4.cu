// esa_w8_p4.cu — batch and trace kernels for topology width W = 8 (see esa_w.cuh).
#define MAPA_W 8
#define MAPA_PART 4
#include "esa_w.cuh"
