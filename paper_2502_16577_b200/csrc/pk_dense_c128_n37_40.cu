// Instantiates the dense complex register kernel for orders 37..40.
#include "pk_dense_c128_launch.cuh"
PK_INSTANTIATE_DENSE_C128(37)
PK_INSTANTIATE_DENSE_C128(38)
PK_INSTANTIATE_DENSE_C128(39)
PK_INSTANTIATE_DENSE_C128(40)
