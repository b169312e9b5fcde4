// Drop-in path shim: the reference header gopt/bal/snavely.hpp maps onto the B200 facade.
#pragma once
#include "../../gopt.hpp"
