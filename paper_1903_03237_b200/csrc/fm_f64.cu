// Instantiation unit: complex128 / float64 kernels.
#include "fm_impl.cuh"
template struct fm::Impl<double>;
