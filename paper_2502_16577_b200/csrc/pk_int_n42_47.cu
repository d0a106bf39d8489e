// Instantiates the exact integer register kernel for orders 42..47.
#include "pk_int_launch.cuh"
PK_INSTANTIATE_INT(42)
PK_INSTANTIATE_INT(43)
PK_INSTANTIATE_INT(44)
PK_INSTANTIATE_INT(45)
PK_INSTANTIATE_INT(46)
PK_INSTANTIATE_INT(47)
