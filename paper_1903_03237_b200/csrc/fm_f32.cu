// Instantiation unit: complex64 / float32 kernels.
#include "fm_impl.cuh"
template struct fm::Impl<float>;
