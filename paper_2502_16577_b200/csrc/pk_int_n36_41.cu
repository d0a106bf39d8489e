// Instantiates the exact integer register kernel for orders 36..41.
#include "pk_int_launch.cuh"
PK_INSTANTIATE_INT(36)
PK_INSTANTIATE_INT(37)
PK_INSTANTIATE_INT(38)
PK_INSTANTIATE_INT(39)
PK_INSTANTIATE_INT(40)
PK_INSTANTIATE_INT(41)
