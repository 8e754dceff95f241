* every row relation, RANGES on each, every bound kind with a value,
* a negative right-hand side and a negative lower bound (shift)
NAME          RNGBND
OBJSENSE
    MAX
ROWS
 N  PROFIT
 L  CAP1
 L  CAP2
 G  DEM1
 G  DEM2
 E  BAL1
 E  BAL2
 E  BAL3
 L  NEGR
COLUMNS
    X1        PROFIT    3.0          CAP1      1.0
    X1        DEM1      1.0          BAL1      1.0
    X2        PROFIT    2.5          CAP1      2.0
    X2        CAP2      1.0          DEM2      1.0
    X2        BAL2      -1.0
    X3        PROFIT    -1.25        CAP2      3.0
    X3        DEM1      0.5          BAL3      1.0
    X4        PROFIT    1.0          CAP1      1.0
    X4        BAL1      -1.0         NEGR      -1.0
    X5        PROFIT    0.75         DEM2      2.0
    X5        BAL2      1.0          NEGR      1.0
    X6        PROFIT    0.1          BAL3      -2.0
    X6        CAP2      0.3
RHS
    RHS       CAP1      40.0         CAP2      30.0
    RHS       DEM1      2.0          DEM2      1.5
    RHS       BAL1      0.0          BAL2      1.0
    RHS       BAL3      -3.0         NEGR      -4.5
RANGES
    RNG       CAP1      10.0         DEM1      -6.0
    RNG       BAL2      4.0          BAL3      -2.5
BOUNDS
 UP BND       X1        12.0
 LO BND       X2        -2.0
 UP BND       X2        20.0
 FX BND       X3        1.5
 FR BND       X4
 MI BND       X5
 UP BND       X5        9.0
 LO BND       X6        0.5
 PL BND       X6
ENDATA
