#include "fm_fused_impl.cuh"
template int fm::Impl<float>::hpass(const fm_dims*, const fm_state*, int, void*, cudaStream_t);
template int fm::Impl<float>::gpass(const fm_dims*, const fm_state*, cudaStream_t);
template int fm::Impl<float>::bpass(const fm_dims*, const fm_state*, cudaStream_t);
template int fm::Impl<float>::hstore(const fm_dims*, const fm_state*, const void*, cudaStream_t);
