// Instantiates the dense real register kernel for orders 54..57 (split for parallel builds).
#include "pk_dense_f64_launch.cuh"
PK_INSTANTIATE_DENSE_F64(54)
PK_INSTANTIATE_DENSE_F64(55)
PK_INSTANTIATE_DENSE_F64(56)
PK_INSTANTIATE_DENSE_F64(57)
