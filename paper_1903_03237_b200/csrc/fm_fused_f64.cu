#include "fm_fused_impl.cuh"
template int fm::Impl<double>::hpass(const fm_dims*, const fm_state*, int, void*, cudaStream_t);
template int fm::Impl<double>::gpass(const fm_dims*, const fm_state*, cudaStream_t);
template int fm::Impl<double>::bpass(const fm_dims*, const fm_state*, cudaStream_t);
template int fm::Impl<double>::hstore(const fm_dims*, const fm_state*, const void*, cudaStream_t);
