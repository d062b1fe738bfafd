# Top-level build (no GPU needed: nvcc cross-compiles sm_100a here).
#
#   make            product library + oracle (+ reference-linked binaries when
#                   /root/reference is present)
#
# Product:
#   paper_0906_0231_b200/lib/libknn_b200.so         CUDA kernels + C ABI
#   paper_0906_0231_b200/lib/libknn_b200_engine.a   drop-in knn::solve_knn TU
#                                                   (needs the reference headers)
# Test binaries linking the UNMODIFIED reference around the drop-in:
#   oracle/_ref/acceptance_b200      reference acceptance.cpp on the GPU engine
#   build/test_engine_b200           test_engine.cpp assertions on the GPU engine

NVCC ?= /usr/local/cuda/bin/nvcc
CXX ?= g++
REF ?= /root/reference/proj
ARCH := -gencode arch=compute_100a,code=sm_100a
# -fmad=false: no implicit mul+add contraction anywhere; FMAs are written
# explicitly where the algorithm wants them.  No fast-math (IEEE sqrt/div).
NVFLAGS := -O3 -std=c++17 $(ARCH) -lineinfo -fmad=false -Xcompiler -fPIC,-fvisibility=hidden \
           --expt-relaxed-constexpr -Xptxas -warn-spills
PKG := paper_0906_0231_b200
CSRC := $(PKG)/csrc
CU_SRCS := $(wildcard $(CSRC)/*.cu)
CU_OBJS := $(patsubst $(CSRC)/%.cu,build/obj/%.o,$(CU_SRCS))
LIB := $(PKG)/lib/libknn_b200.so
ENGINE_A := $(PKG)/lib/libknn_b200_engine.a
HAVE_REF := $(wildcard $(REF)/src/engine.cpp)
REF_FLAGS := -std=c++20 -O3 -ffp-contract=off -fno-math-errno -fPIC

.PHONY: all lib oracle ref-bins clean
all: lib oracle $(if $(HAVE_REF),ref-bins,)
lib: $(LIB)

build/obj/%.o: $(CSRC)/%.cu $(wildcard $(CSRC)/*.cuh) $(CSRC)/kernels.h include/knn_b200.h
	@mkdir -p build/obj
	$(NVCC) $(NVFLAGS) $(NVFLAGS_EXTRA) -Iinclude -c $< -o $@

$(LIB): $(CU_OBJS)
	@mkdir -p $(PKG)/lib
	$(NVCC) $(ARCH) -shared -o $@ $^ -Xlinker --exclude-libs,ALL -lnccl -lpthread

oracle:
	$(MAKE) -C oracle REF=$(REF)

$(ENGINE_A): $(PKG)/host/engine_b200.cpp include/knn_b200.h
	@mkdir -p build/obj $(PKG)/lib
	$(CXX) $(REF_FLAGS) -I$(REF)/include -Iinclude -c $< -o build/obj/engine_b200.o
	rm -f $@ && ar rcs $@ build/obj/engine_b200.o

# The same TU for the reference's KNN_DOUBLE_ACCUM build (dist_t = double).
ENGINE_F64_A := $(PKG)/lib/libknn_b200_engine_f64.a
$(ENGINE_F64_A): $(PKG)/host/engine_b200.cpp include/knn_b200.h
	@mkdir -p build/obj $(PKG)/lib
	$(CXX) $(REF_FLAGS) -DKNN_DOUBLE_ACCUM=1 -I$(REF)/include -Iinclude -c $< -o build/obj/engine_b200_f64.o
	rm -f $@ && ar rcs $@ build/obj/engine_b200_f64.o

REF_LINK := $(ENGINE_A) oracle/_ref/libtknn_ref_noengine.a -L$(PKG)/lib -lknn_b200 \
            -Wl,-rpath,'$$ORIGIN/../$(PKG)/lib' -Wl,-rpath,'$$ORIGIN/../../$(PKG)/lib' -lpthread

REF_LINK_F64 := $(ENGINE_F64_A) oracle/_ref/f64/libtknn_ref_noengine.a -L$(PKG)/lib -lknn_b200 \
            -Wl,-rpath,'$$ORIGIN/../../$(PKG)/lib' -Wl,-rpath,'$$ORIGIN/../$(PKG)/lib' -lpthread

ref-bins: oracle/_ref/acceptance_b200 build/test_engine_b200 build/tknn_b200 oracle/_ref/tknn_ref build/bench_dropin \
          oracle/_ref/acceptance_b200_f64 build/test_engine_b200_f64 build/tknn_b200_f64 oracle/_ref/f64/tknn_ref

# The reference CLI in its KNN_DOUBLE_ACCUM build: on the double drop-in, and
# on the reference's double engine for comparison.
build/tknn_b200_f64: $(REF)/tools/main.cpp tools/cli11_shim/CLI11.hpp $(ENGINE_F64_A) $(LIB) oracle
	$(CXX) $(REF_FLAGS) -DKNN_DOUBLE_ACCUM=1 -Itools/cli11_shim -I$(REF)/include -o $@ $< $(REF_LINK_F64)

oracle/_ref/f64/tknn_ref: $(REF)/tools/main.cpp tools/cli11_shim/CLI11.hpp oracle
	$(CXX) $(REF_FLAGS) -DKNN_DOUBLE_ACCUM=1 -Itools/cli11_shim -I$(REF)/include -o $@ $< \
	    oracle/_ref/f64/libtknn_ref.a -lpthread

oracle/_ref/acceptance_b200_f64: $(REF)/tests/acceptance.cpp $(ENGINE_F64_A) $(LIB) oracle
	$(CXX) $(REF_FLAGS) -DKNN_DOUBLE_ACCUM=1 -I$(REF)/include -o $@ $< $(REF_LINK_F64)

build/test_engine_b200_f64: tests/cpp/test_engine_b200.cpp $(ENGINE_F64_A) $(LIB) oracle
	$(CXX) $(REF_FLAGS) -DKNN_DOUBLE_ACCUM=1 -I$(REF)/include -Iinclude -o $@ $< $(REF_LINK_F64)

# The reference CLI (tools/main.cpp, unmodified) against the B200 drop-in, and
# against the reference engine for comparison; CLI11 is the minimal shim in
# tools/cli11_shim (the real one is not in the image).
build/tknn_b200: $(REF)/tools/main.cpp tools/cli11_shim/CLI11.hpp $(ENGINE_A) $(LIB) oracle
	$(CXX) $(REF_FLAGS) -Itools/cli11_shim -I$(REF)/include -o $@ $< $(REF_LINK)

oracle/_ref/tknn_ref: $(REF)/tools/main.cpp tools/cli11_shim/CLI11.hpp oracle
	$(CXX) $(REF_FLAGS) -Itools/cli11_shim -I$(REF)/include -o $@ $< oracle/_ref/libtknn_ref.a -lpthread

oracle/_ref/acceptance_b200: $(REF)/tests/acceptance.cpp $(ENGINE_A) $(LIB) oracle
	$(CXX) $(REF_FLAGS) -I$(REF)/include -o $@ $< $(REF_LINK)

# The C++ drop-in timed end to end (bench.py's e2e.dropin_ms_per_step).
build/bench_dropin: tools/bench_dropin.cpp $(ENGINE_A) $(LIB) oracle
	$(CXX) $(REF_FLAGS) -I$(REF)/include -o $@ $< $(REF_LINK)

build/test_engine_b200: tests/cpp/test_engine_b200.cpp $(ENGINE_A) $(LIB) oracle
	$(CXX) $(REF_FLAGS) -I$(REF)/include -Iinclude -o $@ $< $(REF_LINK)

clean:
	rm -rf build $(PKG)/lib
	$(MAKE) -C oracle clean
