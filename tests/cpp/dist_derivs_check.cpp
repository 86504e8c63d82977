// Host build of csrc/dist_derivs.cuh (the closed-form contact distance
// derivatives of the device producer) for tests/test_dist_derivs.py: the
// derivatives of a stencil's feature for a given (kind, region), lifted to the
// 12 stencil coordinates.
#include "../../paper_2411_06224_b200/csrc/dist_derivs.cuh"

extern "C" void feat_derivs12(int kind, int region, const double* x12, double* v, double* g12, double* H144) {
    adipc_gpu::FeatDerivs f;
    adipc_gpu::feature_derivs(kind, region, x12, f);
    *v = f.v;
    adipc_gpu::feat_grad12(f, g12);
    adipc_gpu::feat_lift(f, f.H, H144);
}
