// Instantiates the dense real register kernel for orders 37..41 (split for parallel builds).
#include "pk_dense_f64_launch.cuh"
PK_INSTANTIATE_DENSE_F64(37)
PK_INSTANTIATE_DENSE_F64(38)
PK_INSTANTIATE_DENSE_F64(39)
PK_INSTANTIATE_DENSE_F64(40)
PK_INSTANTIATE_DENSE_F64(41)
