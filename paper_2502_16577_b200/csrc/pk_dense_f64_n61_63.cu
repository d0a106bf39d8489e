// Instantiates the dense real register kernel for orders 61..63 (split for parallel builds).
#include "pk_dense_f64_launch.cuh"
PK_INSTANTIATE_DENSE_F64(61)
PK_INSTANTIATE_DENSE_F64(62)
PK_INSTANTIATE_DENSE_F64(63)
