// Instantiates the exact integer register kernel for orders 59..63.
#include "pk_int_launch.cuh"
PK_INSTANTIATE_INT(59)
PK_INSTANTIATE_INT(60)
PK_INSTANTIATE_INT(61)
PK_INSTANTIATE_INT(62)
PK_INSTANTIATE_INT(63)
