// esa_w16_p4.cu — batch and trace kernels for topology width W = 16 (see esa_w.cuh).
#define MAPA_W 16
#define MAPA_PART 4
#include "esa_w.cuh"
