// Instantiates the dense real register kernel for orders 32..36 (split for parallel builds).
#include "pk_dense_f64_launch.cuh"
PK_INSTANTIATE_DENSE_F64(32)
PK_INSTANTIATE_DENSE_F64(33)
PK_INSTANTIATE_DENSE_F64(34)
PK_INSTANTIATE_DENSE_F64(35)
PK_INSTANTIATE_DENSE_F64(36)
