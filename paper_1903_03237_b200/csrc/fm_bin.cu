// Instantiation unit: the per-bin schedule's k_binw (fm_bin.cuh).
#include "fm_bin_impl.cuh"
template int fm::Impl<float>::binw(const fm_dims*, const fm_state*, cudaStream_t);
template int fm::Impl<double>::binw(const fm_dims*, const fm_state*, cudaStream_t);
