// Unity translation unit of the device code (one module => the __constant__
// quadrature tables are shared without relocatable device code).
#include "assemble.cu"
#include "matvec.cu"
#include "toeplitz.cu"
#include "krylov.cu"
#include "hmatrix.cu"
#include "hlu.cu"
#include "hlu2.cu"
