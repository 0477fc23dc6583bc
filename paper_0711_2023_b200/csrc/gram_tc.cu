// gram_tc.cu -- S = A A^T dispatch.  The tcgen05 3xTF32 kernel lands here;
// until it is validated the dispatcher uses the SIMT fp64 kernel.
#include "internal.cuh"

namespace tk {

void gram_syrk(const Split& A, double* S, int64_t lds, GramWs& ws, cudaStream_t st) {
  (void)ws;
  gram_syrk_simt(A, S, lds, st);
}

int gram_path_id() { return 1; }

}  // namespace tk
