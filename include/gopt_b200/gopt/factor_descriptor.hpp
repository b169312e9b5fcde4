// Drop-in path shim: the reference header gopt/factor_descriptor.hpp maps onto the B200 facade.
#pragma once
#include "../gopt.hpp"
