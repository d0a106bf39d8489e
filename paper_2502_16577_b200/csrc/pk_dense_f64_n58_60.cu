// Instantiates the dense real register kernel for orders 58..60 (split for parallel builds).
#include "pk_dense_f64_launch.cuh"
PK_INSTANTIATE_DENSE_F64(58)
PK_INSTANTIATE_DENSE_F64(59)
PK_INSTANTIATE_DENSE_F64(60)
